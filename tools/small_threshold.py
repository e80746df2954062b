"""Persistent cooperative loop vs kernel sequence across n (2-D shifted
Laplacian sequences, 3 systems, SRKS): picks RCG_SMALL_N.
usage: python tools/small_threshold.py 64 128 181 256"""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems

for g in [int(a) for a in sys.argv[1:]] or [64, 128, 181, 256]:
    systems = problems.shifted_laplacian_sequence(grid=g, count=3)
    dev = [(A, torch.from_numpy(b).cuda()) for A, b in systems]
    cfg = rcg.SolveConfig(tol=1e-8, max_iters=5000)
    strat = rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=21)
    out = []
    for small in ("1000000", "0"):
        os.environ["RCG_SMALL_N"] = small
        best = 1e9
        for _ in range(4):
            torch.cuda.synchronize(); t = time.perf_counter()
            rep = rcg.run_sequence(iter(dev), rcg.Preconditioner.jacobi, strat, cfg)
            torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
        out.append((best, sum(rep.iterations())))
    (tp, ip), (tk, ik) = out
    print(f"n={g*g}: persistent {tp*1e3:.1f} ms ({ip} it), kernels {tk*1e3:.1f} ms ({ik} it)")
