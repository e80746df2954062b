"""Small sequences covering every solve-path kernel variant, for
compute-sanitizer memcheck runs:
  PYTORCH_NO_CUDA_MEMORY_CACHING=1 RCG_POOL_EXACT=1 compute-sanitizer --tool memcheck python tools/memcheck_seq.py
(block-DIA and sliced-BSR3 elasticity SRKS + TRKS with reorth, scalar CSR and
DIA config-1 with recycling, lognormal 7-point DIA without reorth +
krylov_cap, and the n_c > 64 coarse path)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems

def run(name, seq, strat, cfg):
    rep = rcg.run_sequence(seq, rcg.Preconditioner.jacobi, strat, cfg)
    print(name, [r.iterations for r in rep.records], rep.events, flush=True)
    assert all(r.converged for r in rep.records) and not rep.aborted

import os
os.environ["RCG_DIA_SMALL"] = "1"                             # DIA for these small operators too
cfg = rcg.SolveConfig(tol=1e-8, max_iters=3000)
el = list(problems.elasticity_sequence(6, 3, seed=0, kind="fixed"))
assert el[0][0].device_csr().struct.dia_count == 14          # block-DIA SpMV
run("elast6 srks dia", el, rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=61), cfg)
os.environ["RCG_DIA3"] = "0"                                  # sliced 3x3 blocks
el = list(problems.elasticity_sequence(6, 3, seed=0, kind="fixed"))
assert el[0][0].device_csr().struct.block == 3
run("elast6 srks sell3", el, rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=61), cfg)
run("elast6 trks sell3", el, rcg.RecycleStrategy("trks", epsilon=1e-10, nc_limit=30), cfg)
del os.environ["RCG_DIA3"]
os.environ["RCG_DIA"] = "0"
c1 = problems.shifted_laplacian_sequence(grid=24, count=3)  # scalar CSR
run("lap24 srks csr", c1, rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=200), cfg)
del os.environ["RCG_DIA"]
c1 = problems.shifted_laplacian_sequence(grid=24, count=3)  # scalar DIA
assert c1[0][0].device_csr().struct.dia_count == 3
run("lap24 srks dia", c1, rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=200), cfg)
ln = list(problems.lognormal_diffusion_sequence(12, 2))
run("logn12 noreorth cap dia", ln, rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=61),
    rcg.SolveConfig(tol=1e-8, max_iters=3000, reorthogonalize=False, krylov_cap=60))
rng = np.random.default_rng(0)
n = 300
A = rcg.SparseSpdMatrix.from_dense(problems.random_spd(n, rng, 1e4), keep_zeros=True)
D = rcg.build_deflation(A, rng.standard_normal((n, 100)))
x, tr = rcg.apcg_solve(A, rcg.Preconditioner.jacobi(A), D, rng.standard_normal(n), cfg)
print("coarse n_c=100", tr.iterations, tr.converged, flush=True)
print("MEMCHECK_SEQ_DONE")
from paper_1301_7530_b200 import _lib
v = _lib.context().lib.rcg_debug_guard_violations()
print("GUARD_VIOLATIONS", v)
