"""Per-system wall/device time split of a sequence (diagnostic).
usage: python tools/seq_breakdown.py [nelem=64] [count=6] [kind=fixed|softening] [nc_limit=61]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems

nelem = int(sys.argv[1]) if len(sys.argv) > 1 else 64
count = int(sys.argv[2]) if len(sys.argv) > 2 else 6
kind = sys.argv[3] if len(sys.argv) > 3 else "fixed"
ncl = int(sys.argv[4]) if len(sys.argv) > 4 else 61
seq = list(problems.elasticity_sequence(nelem, count, kind=kind, device=True))
for A, _ in seq:
    A.device_csr()
bs = [torch.from_numpy(b).cuda() for _, b in seq]
cfg = rcg.SolveConfig(tol=1e-8, max_iters=20000)
strat = rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=ncl)
for rep_i in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    state = rcg.AugmentationState.from_initial(seq[0][0].n)
    for k, b in enumerate(bs):
        A = seq[k][0]
        t1 = time.perf_counter()
        D = rcg.guarded_deflation(A, state, [])
        M = rcg.Preconditioner.jacobi(A)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        x, tr = rcg.apcg_solve(A, M, D, b, cfg)
        t3 = time.perf_counter()
        dev_s = tr.device_seconds
        spec = rcg.select_spectrum(tr, strat)
        torch.cuda.synchronize(); t4 = time.perf_counter()
        rcg.update_basis_srks(state, spec, k)
        torch.cuda.synchronize(); t5 = time.perf_counter()
        if state.n_c >= ncl:
            state.restart()
        m, nsel = spec.m, int(spec.converged_mask.sum())
        del tr, x, spec
        torch.cuda.synchronize(); t6 = time.perf_counter()
        if rep_i == 1:
            print(f"k={k} m={m} nc={D.n_c} build={1e3*(t2-t1):.1f}ms solve_wall={1e3*(t3-t2):.1f}ms dev={1e3*dev_s:.1f}ms "
                  f"select={1e3*(t4-t3):.1f}ms ritzvec={1e3*(t5-t4):.1f}ms free={1e3*(t6-t5):.1f}ms sel={nsel}")
    torch.cuda.synchronize()
    print("total", time.perf_counter() - t0)
