import sys, time
sys.path.insert(0, '/root/repo')
import torch
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems
systems = problems.shifted_laplacian_sequence()
dev = [(A, torch.from_numpy(b).cuda()) for A, b in systems]
cfg = rcg.SolveConfig(tol=1e-8, max_iters=2000)
strat = rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=21)
for rep_i in range(3):
    state = rcg.AugmentationState.from_initial(dev[0][0].n)
    tot = {}
    torch.cuda.synchronize(); T0 = time.perf_counter()
    for k, (A, b) in enumerate(dev):
        t1 = time.perf_counter()
        D = rcg.guarded_deflation(A, state, [])
        M = rcg.Preconditioner.jacobi(A)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        x, tr = rcg.apcg_solve(A, M, D, b, cfg)
        torch.cuda.synchronize(); t3 = time.perf_counter()
        spec = rcg.select_spectrum(tr, strat)
        torch.cuda.synchronize(); t4 = time.perf_counter()
        rcg.update_basis_srks(state, spec, k)
        torch.cuda.synchronize(); t5 = time.perf_counter()
        if state.n_c >= 21:
            state.restart()
        for key, v in (("build", t2-t1), ("solve", t3-t2), ("dev", tr.device_seconds), ("select", t4-t3), ("update", t5-t4)):
            tot[key] = tot.get(key, 0) + v
        del tr, x, spec
    torch.cuda.synchronize()
    print(rep_i, "total %.1f ms" % ((time.perf_counter()-T0)*1e3), {k: round(v*1e3, 2) for k, v in tot.items()})
