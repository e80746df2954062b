"""Run BASELINE.json configs on one GPU and report iters/s, sequence time and
the live per-kernel roofline (evidence for DESIGN.md §6; not the bench line).

usage: python tools/run_configs.py 1|3|4|5 [--systems K] [--reorth 0|1] [--nelem N | --grid G] [--host-gen]
Matrix generation (device assemblers, csrc/gen.cu, unless --host-gen) is
outside the timed region.  CUDA events time the whole sequence (build ->
solve -> select -> append).  Config 5 (12.4 M dofs, ~1e9 nnz) is generated
lazily, one operator resident at a time; its generation events are
subtracted from the sequence time.
"""
import argparse, json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems, _lib

p = argparse.ArgumentParser()
p.add_argument("config", type=int)
p.add_argument("--systems", type=int, default=None)
p.add_argument("--reorth", type=int, default=1)
p.add_argument("--nelem", type=int, default=None)
p.add_argument("--grid", type=int, default=None)
p.add_argument("--max-iters", type=int, default=20000)
p.add_argument("--cap", type=int, default=None, help="krylov_cap extension (z history kept)")
p.add_argument("--host-gen", action="store_true", help="numpy assemblers instead of the device ones")
p.add_argument("--no-rerun", action="store_true", help="skip the unprofiled second sequence")
args = p.parse_args()
devgen = not args.host_gen

t0 = time.time()
if args.config == 1:
    systems = problems.shifted_laplacian_sequence(count=args.systems or 10)
    tol, eps, ncl = 1e-8, 1e-10, 21
elif args.config == 3:
    N = args.nelem or 96
    systems = list(problems.elasticity_sequence(N, args.systems or 15, kind="softening", device=devgen))
    tol, eps, ncl = 1e-8, 1e-10, 81
elif args.config == 4:
    g = args.grid or 256
    systems = list(problems.lognormal_diffusion_sequence(g, args.systems or 20, device=devgen))
    tol, eps, ncl = 1e-8, 1e-10, 21
elif args.config == 5:
    N = args.nelem or 160
    K = args.systems or 10
    systems = None   # lazy: ~20 GB of device CSR + sliced blocks per operator
    tol, eps, ncl = 1e-8, 1e-10, 101
else:
    raise SystemExit("configs 1, 3, 4, 5 (config 2 is bench.py)")
gen_events = []
meta = {}


def lazy5():
    """config-5 systems assembled on the device one at a time; generation is
    bracketed by events so it can be taken out of the sequence time"""
    it = problems.elasticity_sequence(N, K, kind="lognormal_softening", device=devgen)
    prev = None
    while True:
        g0, g1 = torch.cuda.Event(True), torch.cuda.Event(True)
        g0.record()
        if prev is not None:
            prev.release_device()
        try:
            A, b = next(it)
        except StopIteration:
            return
        A.device_csr()
        meta.setdefault("nnz", A.nnz)
        bd = torch.from_numpy(b).cuda()
        g1.record()
        gen_events.append((g0, g1))
        prev = A
        yield A, bd


gen = time.time() - t0
cfg = rcg.SolveConfig(tol=tol, max_iters=args.max_iters, reorthogonalize=bool(args.reorth), krylov_cap=args.cap)
strat = rcg.RecycleStrategy("srks", epsilon=eps, nc_limit=ncl)
ctx = _lib.context()
if systems is not None:
    n, nnz = systems[0][0].n, systems[0][0].nnz
    dev = [(A, torch.from_numpy(b).cuda()) for A, b in systems]
    for A, _ in dev:
        A.device_csr()
    rcg.run_sequence(iter(dev[:2]), rcg.Preconditioner.jacobi, strat, cfg)   # warm-up: graphs, pools
    source = lambda: iter(dev)
else:
    source = lazy5
ctx.reset_stats()
ctx.set_profiling(True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
rep = rcg.run_sequence(source(), rcg.Preconditioner.jacobi, strat, cfg)
e1.record()
torch.cuda.synchronize()
ctx.set_profiling(False)
gen_in_region = sum(a.elapsed_time(b) for a, b in gen_events) * 1e-3
sec = e0.elapsed_time(e1) * 1e-3 - gen_in_region
if systems is None:
    n, nnz = 3 * N * (N + 1) ** 2, meta.get("nnz")
st = ctx.kernel_stats()
tot = sum(v["seconds"] for v in st.values())
byt = sum(v["bytes"] for v in st.values())
out = {"config": args.config, "n": n, "nnz": nnz, "systems": len(rep.records), "reorthogonalize": bool(args.reorth),
       "krylov_cap": args.cap,
       "iterations": rep.iterations(), "n_c_before": rep.n_c_history(), "aborted": rep.aborted,
       "all_converged": all(r.converged for r in rep.records),
       "sequence_seconds_profiled": sec, "iters_per_s_profiled": sum(rep.iterations()) / sec,
       "kernel_seconds": tot, "path_GBps": byt / tot / 1e9 if tot else None,
       "kernels": {k: {"s": round(v["seconds"], 4), "GBps": round(v["bytes"] / v["seconds"] / 1e9) if v["seconds"] else 0}
                   for k, v in st.items() if v["launches"]},
       "generation": "device (csrc/gen.cu)" if devgen else "host (numpy)",
       "generation_seconds": gen + gen_in_region,
       "final_residuals": [r.final_residual for r in rep.records]}
if systems is not None and not args.no_rerun:
    # unprofiled timing of the same sequence
    torch.cuda.synchronize()
    e0.record()
    rep2 = rcg.run_sequence(iter(dev), rcg.Preconditioner.jacobi, strat, cfg)
    e1.record()
    torch.cuda.synchronize()
    out["sequence_seconds"] = e0.elapsed_time(e1) * 1e-3
    out["iters_per_s"] = sum(rep2.iterations()) / out["sequence_seconds"]
print(json.dumps(out))
