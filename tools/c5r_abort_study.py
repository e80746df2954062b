"""Where does the reduced config-5 analog (lognormal-E softening elasticity 16^3,
reorth off, SRKS eps 1e-10, nc_limit 101) abort with (r, z) <= 0, per seed?
usage: python tools/c5r_abort_study.py oracle|gpu [seeds...]
The CPU oracle (reference algorithm) and the device path are run on the same
seeded sequences; compare the abort indices as distributions (the index is
rounding-decided, tests/test_oracle_golden.py)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1301_7530_b200 import problems

side = sys.argv[1]
seeds = [int(s) for s in sys.argv[2:]] or list(range(8))
out = {}
for seed in seeds:
    systems = list(problems.elasticity_sequence(16, 10, seed=seed, kind="lognormal_softening"))
    if side == "oracle":
        from oracle import recycg_oracle as orc
        rep = orc.run_sequence(iter(systems), "srks", epsilon=1e-10, nc_limit=101, tol=1e-8, max_iters=5000,
                               reorthogonalize=False)
        ev = [e for e in rep.events if e[0] == "solve_failed"]
        out[seed] = {"solved": len(rep.iterations), "abort": ev[0][1] if ev else None, "n_c": rep.n_c_before}
    else:
        import paper_1301_7530_b200 as rcg
        cfg = rcg.SolveConfig(tol=1e-8, max_iters=5000, reorthogonalize=False)
        rep = rcg.run_sequence(iter(systems), rcg.Preconditioner.jacobi,
                               rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=101), cfg)
        ev = [e for e in rep.events if e[0] == "solve_failed"]
        out[seed] = {"solved": len(rep.records), "abort": ev[0][1] if ev else None, "n_c": rep.n_c_history()}
    print(side, seed, out[seed], flush=True)
print(json.dumps({side: out}))
