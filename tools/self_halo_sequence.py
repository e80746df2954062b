"""A recycling sequence through the sharded path on one GPU (two virtual slabs, NCCL send/recv to self).
usage: RCG_SHARDED_GRAPHS=0|1 RCG_HALO_OVERLAP=0|1 python tools/self_halo_sequence.py [srks|trks]"""
import os, sys, socket
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
os.environ["RCG_DIA_SMALL"]="1"; os.environ["RCG_COMM_FORCE"]="1"
import numpy as np, torch.distributed as dist
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems, distributed as Dm
with socket.socket() as sk:
    sk.bind(("127.0.0.1", 0)); port = sk.getsockname()[1]
dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
A = problems.assemble_diffusion(np.exp(np.random.default_rng(3).standard_normal((20, 16, 12))))
b = np.random.default_rng(4).standard_normal(A.n); cut = A.n // 2 + 5
n = A.n
ro, ci, va = np.asarray(A.row_offsets), np.asarray(A.col_indices, dtype=np.int64), np.asarray(A.values)
rows = np.repeat(np.arange(n), np.diff(ro)); cross = (rows < cut) != (ci < cut)
ghosts = np.unique(ci[cross]); lci = ci.copy(); lci[cross] = n + np.searchsorted(ghosts, ci[cross])
off = np.array([0, len(ghosts)], dtype=np.int64)
plan = Dm.HaloPlan(1, 0, n, len(ghosts), ghosts.astype(np.int32), off, off.copy(), ghosts)
Dm.init_comm()
S = Dm.ShardedMatrix(ro, lci.astype(np.int32), va, plan, n)
strat = rcg.RecycleStrategy(sys.argv[1] if len(sys.argv) > 1 else "srks", epsilon=1e-10, nc_limit=61)
rhs = [b, 0.5 * b + 0.1 * np.random.default_rng(6).standard_normal(n), -b]
cfg2 = rcg.SolveConfig(tol=1e-8, max_iters=3000)
r1 = rcg.run_sequence([(S, v) for v in rhs], rcg.Preconditioner.jacobi, strat, cfg2)
r2 = rcg.run_sequence([(A, v) for v in rhs], rcg.Preconditioner.jacobi, strat, cfg2)
print("sharded", r1.iterations(), r1.n_c_history(), [r.converged for r in r1.records], [r.final_residual for r in r1.records], r1.events)
print("plain  ", r2.iterations(), r2.n_c_history(), [r.converged for r in r2.records])
Dm.destroy_comm()
