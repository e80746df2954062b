"""Where the e2e time of a config-3 step goes: host->device CSR upload paths
and the stream-format analysis (DIA build) of a fresh operator."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems

A, b = next(problems.elasticity_sequence(96, 1, kind="softening", device=True))
ro, ci, va = A.row_offsets, A.col_indices, A.values
A.release_device()
torch.cuda.synchronize()

def t(f, rep=3):
    best = 1e9
    for _ in range(rep):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best

print("values bytes", va.nbytes, "ci", ci.nbytes, "ro", ro.nbytes)
print("pageable va .to(cuda): %.3f s" % t(lambda: torch.from_numpy(va).to("cuda")))
pin = torch.empty(va.shape, dtype=torch.float64, pin_memory=True)
print("pinned alloc done")
print("np->pinned memcpy: %.3f s" % t(lambda: pin.numpy().__setitem__(slice(None), va)))
print("pinned va .to(cuda): %.3f s" % t(lambda: pin.to("cuda", non_blocking=True)))
print("full device_csr (fresh object): %.3f s" % t(lambda: rcg.SparseSpdMatrix(A.n, ro, ci, va, validate=False).device_csr()))
S = rcg.SparseSpdMatrix(A.n, ro, ci, va, validate=False)
def upload_only():
    ro32 = torch.from_numpy(ro.astype(np.int32)).to("cuda")
    c = torch.from_numpy(np.ascontiguousarray(ci, dtype=np.int32)).to("cuda")
    v = torch.from_numpy(va).to("cuda")
print("upload only: %.3f s" % t(upload_only))

from paper_1301_7530_b200 import core
core.h2d(va)
print("staged h2d va: %.3f s" % t(lambda: core.h2d(va)))
print("full device_csr with staging: %.3f s" % t(lambda: rcg.SparseSpdMatrix(A.n, ro, ci, va, validate=False).device_csr()))
