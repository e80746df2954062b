"""Time rcg_spmv on a BASELINE matrix (CUDA events; the matrix exceeds L2).
usage: RCG_SPMV_V=8 python tools/spmv_bench.py [elast64|diff256|lap128] [csr|auto]"""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1301_7530_b200 import problems, _lib, SparseSpdMatrix

which = sys.argv[1] if len(sys.argv) > 1 else "elast64"
fmt = sys.argv[2] if len(sys.argv) > 2 else "auto"
if which == "elast64":
    A = problems.elasticity_q1(int(os.environ.get("NELEM", "64")), validate=False)
elif which == "diff256":
    A = next(problems.lognormal_diffusion_sequence(256, 1))[0]
else:
    A = problems.shifted_laplacian_sequence(count=1)[0][0]
A = SparseSpdMatrix(A.n, A.row_offsets, A.col_indices, A.values, validate=False, use_block3=(fmt != "csr"))
h = A.device_csr()
ctx = _lib.context()
x = torch.randn(A.n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
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
blk = h.struct.block
byt = (8 * A.nnz + 4 * A.nnz / 9 + 4 * (A.n // 3 + 1) + 16 * A.n) if blk == 3 else (12 * A.nnz + 4 * (A.n + 1) + 16 * A.n)
fmtname = ("sell3" if h.struct.bsr_slice == 32 else "bsr3") if blk == 3 else "csr"
if h.struct.dia_count:
    byt = 8 * h.struct.dia_count * h.struct.dia_block * A.n + 16 * A.n
    fmtname = f"dia{h.struct.dia_block}x{h.struct.dia_count}"
print(f"{which} fmt={fmtname} V={os.environ.get('RCG_SPMV_V','auto')} n={A.n} nnz={A.nnz} "
      f"t={t*1e6:.1f}us {byt/t/1e9:.0f} GB/s (algorithmic {byt/1e6:.0f} MB)")
