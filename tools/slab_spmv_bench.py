"""Time the solve-loop SpMV of ONE row slab of a BASELINE operator on one GPU
(no communication: the ghost entries of x are just there), with the slab's
block-DIA copy + ghost-column remainder and with the sliced 3x3 blocks
(RCG_SLAB_DIA=0).  usage: RCG_SPMV_IND=1 python tools/slab_spmv_bench.py [nelem=96] [nranks=8] [rank=3]"""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1301_7530_b200 import problems, _lib, distributed as D

ne = int(sys.argv[1]) if len(sys.argv) > 1 else 96
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rk = int(sys.argv[3]) if len(sys.argv) > 3 else 3
A = problems.elasticity_q1(ne, validate=False)
ro = A.row_offsets
bounds = D.partition_rows(ro, nr, align=3)
r0, r1 = int(bounds[rk]), int(bounds[rk + 1])
s0, s1 = ro[r0], ro[r1]
ro_l, lci, va, plan = D.build_local_system(ro[r0:r1 + 1], A.col_indices[s0:s1], A.values[s0:s1], bounds, rk,
                                           gathered=None if nr == 1 else [[np.zeros(0, np.int64)] * nr] * nr)
for flag in ("1", "0"):
    os.environ["RCG_SLAB_DIA"] = flag
    S = D.ShardedMatrix(ro_l, lci, va, plan, A.n)
    h = S.device_csr()
    ctx = _lib.context()
    x = torch.randn(S.n_ext, dtype=torch.float64, device="cuda")
    y = torch.empty(S.n, dtype=torch.float64, device="cuda")
    for _ in range(5):
        ctx.check(ctx.lib.rcg_spmv(ctx.h, _lib.C.byref(h.struct), _lib.ptr(x), _lib.ptr(y)))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    N = 50
    e0.record()
    for _ in range(N):
        ctx.check(ctx.lib.rcg_spmv(ctx.h, _lib.C.byref(h.struct), _lib.ptr(x), _lib.ptr(y)))
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / N * 1e-3
    st = h.struct
    fmt = f"dia{st.dia_block}x{st.dia_count}+rem({st.rem_rows} rows)" if st.dia_count else \
        ("sell3" if st.bsr_slice == 32 else "csr")
    print(f"slab {rk}/{nr} of Q1 {ne}^3: n_local={S.n} ghosts={plan.n_ghost} nnz={S.nnz} fmt={fmt} t={t*1e6:.1f}us")
    S.release_device()
