"""Diagnose e2e vs device-resident sequence time on config 2 (few systems)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems
import bench

S = int(sys.argv[1]) if len(sys.argv) > 1 else 4
A, bs = bench.workload(64, S)
cfg = rcg.SolveConfig(tol=1e-8, max_iters=20000)
strat = rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=61)
bs_dev = [torch.from_numpy(b).cuda() for b in bs]
A.device_csr()
def dev():
    return rcg.run_sequence(((A, b) for b in bs_dev), rcg.Preconditioner.jacobi, strat, cfg)
def e2e():
    Ah = rcg.SparseSpdMatrix(A.n, A.row_offsets, A.col_indices, A.values, validate=False)
    t = time.perf_counter(); Ah.device_csr(); torch.cuda.synchronize(); tu = time.perf_counter() - t
    xs = []
    rep = bench._e2e_sequence(rcg, ((Ah, b) for b in bs), strat, cfg, xs)
    return rep, tu
for k in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); r = dev(); torch.cuda.synchronize(); td = time.perf_counter() - t
    torch.cuda.synchronize(); t = time.perf_counter(); r2, tu = e2e(); torch.cuda.synchronize(); te = time.perf_counter() - t
    print(f"dev {td:.3f}s it={sum(r.iterations())}  e2e {te:.3f}s (upload {tu:.3f}s) it={sum(r2.iterations())}")
