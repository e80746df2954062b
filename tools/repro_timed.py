"""Mimic bench.py's warm-up -> timed transition piece by piece (debug aid).
MODE: bits 1 = torch.cuda.synchronize + event record, 2 = nvidia-smi sampler, 4 = _lib.total_launches"""
import sys, os, subprocess
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems, _lib
mode = int(os.environ.get("MODE", "7"))
seq = list(problems.elasticity_sequence(int(os.environ.get("NEL", "64")), 1, seed=0, kind="fixed"))
A, b = seq[0]
bd = torch.from_numpy(b).to("cuda")
A.device_csr()
cfg = rcg.SolveConfig(tol=1e-8, max_iters=20000, reorthogonalize=True)
strat = rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=61)
def step(tag):
    rep = rcg.run_sequence([(A, bd)], rcg.Preconditioner.jacobi, strat, cfg)
    r = rep.records[0] if rep.records else None
    print(tag, "conv", r.converged if r else None, "it", r.iterations if r else None, rep.events, flush=True)
for k in range(3):
    step(f"warm{k}")
if mode & 4:
    _lib.total_launches()
proc = None
if mode & 2:
    proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "200"],
                            stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
if mode & 1:
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream())
for k in range(3):
    step(f"timed{k}")
if proc:
    proc.terminate()
