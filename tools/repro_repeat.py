"""Repeat one config-2 solve through run_sequence and report each outcome
(debug aid for state carried across solves: graph cache, pools, counters)."""
import sys, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems
nel = int(os.environ.get("NEL", "64"))
reps = int(os.environ.get("REPS", "6"))
seq = list(problems.elasticity_sequence(nel, 1, seed=0, kind="fixed"))
A, b = seq[0]
bd = torch.from_numpy(b).to("cuda")
print("block", A.device_csr().struct.block, flush=True)
cfg = rcg.SolveConfig(tol=1e-8, max_iters=20000, reorthogonalize=True)
strat = rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=61)
for k in range(reps):
    rep = rcg.run_sequence([(A, bd)], rcg.Preconditioner.jacobi, strat, cfg)
    r = rep.records[0] if rep.records else None
    print(k, "conv", r.converged if r else None, "it", r.iterations if r else None, rep.events, flush=True)
