"""Run BASELINE config 2 systems 0-1 (full size) R times in one process and
print iterations, selected Ritz value count and hashes of x / selected
values: bitwise reproducibility across runs and processes."""
import hashlib, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems, recycle as rmod

R = int(sys.argv[1]) if len(sys.argv) > 1 else 2
systems = list(problems.elasticity_sequence(64, 2, kind="fixed", device=True))
real = rmod.select_spectrum
for rep in range(R):
    sel = []
    def spy(trace, strategy):
        s = real(trace, strategy)
        sel.append(np.sort(s.values[s.converged_mask]))
        return s
    rmod.select_spectrum = spy
    runner = rcg.SequenceRunner(rcg.Preconditioner.jacobi, rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=61),
                                rcg.SolveConfig(tol=1e-8, max_iters=20000))
    xs = [runner.step(A, torch.from_numpy(b).cuda()).cpu().numpy() for A, b in systems]
    rmod.select_spectrum = real
    h = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:12]
    print(rep, runner.report.iterations(), runner.report.n_c_history(), [len(s) for s in sel],
          [h(s) for s in sel], [h(x) for x in xs], flush=True)
