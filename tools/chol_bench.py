"""Guarded Cholesky + G^-1 (rcg_dense_cholesky, the coarse-matrix path of
build_deflation) timing at TRKS basis sizes (criterion 6: n_c up to ~1.6 k)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import _lib

rng = np.random.default_rng(0)
for n in (64, 128, 256, 512, 1024, 1600, 2048):
    X = rng.standard_normal((n, n))
    G = X @ X.T + n * np.eye(n)
    Gd = torch.from_numpy(np.ascontiguousarray(G)).cuda()
    L = torch.empty_like(Gd); Gi = torch.empty_like(Gd)
    ctx = _lib.context()
    bad = _lib.C.c_int64(-1)
    def run():
        ctx.check(ctx.lib.rcg_dense_cholesky(ctx.h, _lib.ptr(Gd), n, 1e-12, _lib.ptr(L), _lib.ptr(Gi), _lib.C.byref(bad)), "chol")
    run(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3): run()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    Lh = L.cpu().numpy()
    # column-major device layout: L^T in row-major numpy terms
    Lc = Lh.T if np.allclose(np.triu(Lh.T, 1), 0) else Lh
    err = np.linalg.norm(Lc @ Lc.T - G) / np.linalg.norm(G)
    Gih = Gi.cpu().numpy()
    ierr = np.linalg.norm(Gih @ G - np.eye(n)) / np.sqrt(n)
    print(f"n={n:5d}  {dt*1e3:8.2f} ms   |LL^T-G|/|G| = {err:.1e}   |Ginv G - I| = {ierr:.1e}", flush=True)
