"""Small-case check of the round-2 SpMV code (also a compute-sanitizer target where that is available): the 3x3 block-DIA
kernel with claimed tiles and the interior-row body through the
kernel-sequence solve loop, the scalar DIA interior body, and slab SpMVs
(DIA copy + ELL ghost remainder) in the plain and solve-loop modes.
  RCG_SPMV_IND=0|1 PYTORCH_NO_CUDA_MEMORY_CACHING=1 RCG_POOL_EXACT=1 \
      compute-sanitizer --tool memcheck python tools/memcheck_dia_slab.py"""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["RCG_DIA_SMALL"] = "1"
os.environ["RCG_SMALL_N"] = "0"
import numpy as np
import torch
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems, _lib, distributed as D

rng = np.random.default_rng(0)
for name, A in (("q1_10", problems.elasticity_q1(10, E=np.exp(rng.standard_normal((10,) * 3)))),
                ("diff", problems.assemble_diffusion(rng.lognormal(0.0, 1.0, (14, 12, 10))))):
    A = rcg.SparseSpdMatrix(A.n, A.row_offsets, A.col_indices, A.values, validate=False)
    st = A.device_csr().struct
    assert st.dia_count > 0
    b = rng.standard_normal(A.n)
    x, tr = rcg.apcg_solve(A, rcg.Preconditioner.jacobi(A), rcg.build_deflation(A, rng.standard_normal((A.n, 3))), b,
                           rcg.SolveConfig(tol=1e-8, max_iters=400))
    print(name, "dia", st.dia_block, st.dia_count, "iterations", tr.iterations, "converged", tr.converged, flush=True)
    align = st.dia_block
    bounds = D.partition_rows(A.row_offsets, 3, align=align)
    xg = rng.standard_normal(A.n)
    yg = A @ xg
    ctx = _lib.context()
    for r, (ro, lci, va, plan) in enumerate(D.local_systems_all(A.row_offsets, A.col_indices, A.values, bounds)):
        S = D.ShardedMatrix(ro, lci, va, plan, A.n)
        h = S.device_csr().struct
        assert h.dia_count > 0 and h.rem_rows > 0
        xe = torch.from_numpy(np.concatenate([xg[bounds[r]:bounds[r + 1]], xg[plan.ghost_global]])).cuda()
        ye = torch.zeros(plan.n_local, dtype=torch.float64, device="cuda")
        for _ in range(2):
            ctx.check(ctx.lib.rcg_spmv(ctx.h, _lib.C.byref(h), _lib.ptr(xe), _lib.ptr(ye)), "spmv")
        torch.cuda.synchronize()
        err = np.abs(ye.cpu().numpy() - yg[bounds[r]:bounds[r + 1]]).max()
        print(name, "slab", r, "rem rows", h.rem_rows, "width", h.rem_width, "max err", err, flush=True)
        assert err < 1e-10 * np.abs(yg).max()
print("ok")
