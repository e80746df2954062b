"""Config 1 (2-D shifted Laplacian 128^2, 10 systems, SRKS eps 1e-10, nc_limit 21):
sequence wall time on the GPU path (latency-bound: everything is L2-resident)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems, _lib
systems = problems.shifted_laplacian_sequence()
dev = [(A, torch.from_numpy(b).cuda()) for A, b in systems]
for A, _ in dev:
    A.device_csr()
cfg = rcg.SolveConfig(tol=1e-8, max_iters=2000)
strat = rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=21)
for k in range(8):
    torch.cuda.synchronize(); t = time.perf_counter()
    rep = rcg.run_sequence(iter(dev), rcg.Preconditioner.jacobi, strat, cfg)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    it = sum(rep.iterations())
    print(f"config1 seq {dt*1e3:.1f} ms, {it} iterations -> {it/dt:.0f} it/s; per-system {rep.iterations()}; device {rep.device_seconds*1e3:.1f} ms")
ctx = _lib.context(); ctx.reset_stats(); ctx.set_profiling(True)
rep = rcg.run_sequence(iter(dev), rcg.Preconditioner.jacobi, strat, cfg)
ctx.set_profiling(False)
print({k: (v["launches"], round(v["seconds"]*1e3, 2)) for k, v in ctx.kernel_stats().items()})
