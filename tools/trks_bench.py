"""Reference acceptance criterion 6's heaviest run on the device: TRKS on the
40-system inclusion benchmark at tol 1e-6 (n_c grows to ~1.6 k, so the
coarse factorization of C^T A C is a 1.6 k x 1.6 k guarded Cholesky per
system).  Prints the sequence time and the summed build (augmentation) time."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems

systems = list(problems.generate_diffusion_sequence(problems.benchmark_spec(seed=0), 40))
cfg = rcg.SolveConfig(tol=1e-6, max_iters=3000)
for rep_i in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = rcg.run_sequence(iter(systems), rcg.Preconditioner.jacobi, rcg.RecycleStrategy("trks"), cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    aug = sum(r.augmentation_seconds for r in rep.records)
    sol = sum(r.solve_seconds for r in rep.records)
    print(f"run {rep_i}: {dt:.2f} s total, solve {sol:.2f} s, augmentation (build + update) {aug:.2f} s, "
          f"iterations {sum(rep.iterations())}, max n_c {max(rep.n_c_history())}", flush=True)
