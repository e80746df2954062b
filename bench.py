#!/usr/bin/env python
"""Benchmark of the B200 augmented-PCG / SRKS recycling hot path.

Workload (BASELINE.json configs[1], the config the metric is quoted on that
fits one GPU): 3-D linear elasticity, Q1 hexahedra, 64^3 elements on the unit
cube, E = 1, nu = 0.3, face x = 0 clamped -> n = 811,200 dofs, nnz =
63,695,790 (78.5/row) fp64 CSR; fixed matrix, 20 right-hand sides of seeded
N(0,1) nodal tractions on x = 1; Jacobi PCG, tol 1e-8 (vs ||P^T b||), full
reorthogonalization (reference default), SRKS eps = 1e-10 recycling up to 60
Ritz vectors (nc_limit = 61).

One "step" = one full 20-system sequence (build -> solve -> select -> append
for every system), starting from an empty basis.  ``value`` = APCG iterations
per second over the timed steps (inputs resident in HBM); ``e2e`` = the same
metric through the public API with host CSR/RHS arrays, uploads and solution
downloads inside the timed region.

``--impl reference`` times the CPU oracle (the reference algorithm restated
with numpy/scipy, oracle/recycg_oracle.py) on a bounded sample of the same
workload: the first K iterations of system 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402

METRIC = "aug-PCG fp64 iters/s & sequence solve time; achieved HBM GB/s vs peak"
UNIT = "iters/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--nelem", type=int, default=64, help="elements per edge (64 = BASELINE config 2)")
    p.add_argument("--systems", type=int, default=20)
    p.add_argument("--max-iters", type=int, default=20000)
    p.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU sample duration")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--replicas", action="store_true", help="N>1: independent replicas instead of row sharding")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload(nelem, systems):
    from paper_1301_7530_b200 import problems
    seq = list(problems.elasticity_sequence(nelem, systems, seed=0, kind="fixed"))
    A = seq[0][0]
    bs = [b for _, b in seq]
    return A, bs


def config_dict(A, nelem, systems, world, sharded=False):
    return {
        "workload": f"BASELINE config 2: Q1 elasticity {nelem}^3 elements, fixed A, {systems} traction RHS, "
                    "Jacobi APCG tol 1e-8, full reorth, SRKS eps=1e-10 nc_limit=61",
        "n": int(A.n), "nnz": int(A.nnz), "systems": systems, "strategy": "srks", "epsilon": 1e-10,
        "nc_limit": 61, "tol": 1e-8, "reorthogonalize": True, "preconditioner": "jacobi",
        "l2": "inputs larger than L2 (CSR 764 MB, Krylov histories GBs)",
        "parallelism": (f"rows{world} (row-sharded, NCCL halo + allreduce)" if sharded else
                        ("replicas" if world > 1 else "single")),
    }


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md clocks line)


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline and --impl reference)


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        n = [d.get("num_threads", 1) for d in info if d.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:
        return os.cpu_count() or 1


def cpu_sample(A, b, iters):
    """Oracle apcg_solve on system 0 for exactly `iters` iterations (reorth on)."""
    from oracle import recycg_oracle as orc
    inv = 1.0 / orc.diagonal(A)
    D = orc.build_deflation(A, np.zeros((A.n, 0)))
    t0 = time.perf_counter()
    _, tr = orc.apcg_solve(A, inv, D, b, 1e-300, iters, reorthogonalize=True, trace_capture=True)
    dt = time.perf_counter() - t0
    return tr.iterations, dt


def cpu_calibrated(A, b, target_seconds):
    """Window length K with ~target_seconds of CPU work.  The reorth cost of
    iteration j grows linearly in j, so the window time grows ~K^2."""
    k0 = 8
    it0, dt0 = cpu_sample(A, b, k0)
    iters = int(k0 * (max(target_seconds, 1e-3) / max(dt0, 1e-6)) ** 0.5)
    return int(max(5, min(400, iters)))


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    A, bs = workload(args.nelem, args.systems)
    iters = cpu_calibrated(A, bs[0], args.cpu_seconds / max(args.steps, 1))
    for _ in range(args.warmup):
        cpu_sample(A, bs[0], max(3, iters // 4))
    tot_it, tot_t = 0, 0.0
    for _ in range(args.steps):
        it, dt = cpu_sample(A, bs[0], iters)
        tot_it += it
        tot_t += dt
    value = tot_it / tot_t
    cores = blas_threads()
    sample = (f"first {iters} APCG iterations of system 0 (n_c=0, Jacobi, full reorth) per step; "
              "scipy csr_matvec (1 thread) + numpy/OpenBLAS")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(A, args.nelem, args.systems, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm


def peaks():
    f = REPO / "MEASURED_PEAKS.json"
    try:
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def box_copy_gbps():
    import torch
    try:
        a = torch.empty(1 << 29, dtype=torch.bfloat16, device="cuda")
        b = torch.empty_like(a)
        best = 0.0
        for _ in range(6):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            b.copy_(a)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, 2 * a.numel() * 2 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        del a, b
        return best
    except Exception:
        return None


def ncu_traffic():
    f = REPO / "profiles" / "ncu_traffic.json"
    try:
        return json.loads(f.read_text())
    except Exception:
        return {}


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1301_7530_b200 as rcg
    from paper_1301_7530_b200 import _lib

    A, bs = workload(args.nelem, args.systems)
    cfg = rcg.SolveConfig(tol=1e-8, max_iters=args.max_iters, reorthogonalize=True)
    strat = rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=61)
    A_global = A
    sharded = world > 1 and not args.replicas
    if sharded:
        # row slabs (x-slabs of nodes), halo plan, NCCL communicator
        from paper_1301_7530_b200 import distributed as D
        bounds = D.partition_rows(A.row_offsets, world, align=3)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        s0, s1 = A.row_offsets[r0], A.row_offsets[r1]
        ro_l, lci, va, plan = D.build_local_system(A.row_offsets[r0:r1 + 1], A.col_indices[s0:s1],
                                                   A.values[s0:s1], bounds, rank)
        D.init_comm()
        A = D.ShardedMatrix(ro_l, lci, va, plan, A_global.n)
        bs = [b[r0:r1].copy() for b in bs]
        shard_host = (ro_l, lci, va, plan)
    bs_dev = [torch.from_numpy(b).to("cuda") for b in bs]
    A.device_csr()

    def step():
        rep = rcg.run_sequence(((A, b) for b in bs_dev), rcg.Preconditioner.jacobi, strat, cfg)
        if rep.aborted or not all(r.converged for r in rep.records):
            raise RuntimeError(f"sequence did not converge: {rep.events} "
                               f"iterations={[r.iterations for r in rep.records]}")
        return rep

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(v):
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([v], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return v

    for _ in range(args.warmup):
        rep = step()
    ctx = _lib.context()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.total_launches()
    iters = 0
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            rep = step()
            iters += sum(rep.iterations())
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = _lib.total_launches() - l0
    sec = max_over_ranks(e0.elapsed_time(e1) * 1e-3)
    # replicas: every rank solves the whole sequence (weak); sharded: one joint solve (strong)
    value = (iters if sharded else world * iters) / sec
    per_system = rep.iterations()
    nc_hist = rep.n_c_history()

    # roofline pass: one more step with live per-kernel event timing
    ctx.reset_stats()
    ctx.set_profiling(True)
    step()
    ctx.set_profiling(False)
    stats = ctx.kernel_stats()
    dom = max(stats, key=lambda k: stats[k]["seconds"])
    tot_k = sum(s["seconds"] for s in stats.values())
    peak, peak_src = peaks()
    box_copy = box_copy_gbps()
    d = stats[dom]
    achieved = d["bytes"] / d["seconds"] / 1e9 if d["seconds"] > 0 else 0.0
    traffic_detail = ncu_traffic().get(dom)
    traffic = traffic_detail.get("bytes") if isinstance(traffic_detail, dict) else None
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_detail": traffic_detail,
                "peak_source": peak_src,
                "share_of_kernel_time": d["seconds"] / tot_k if tot_k else None,
                # context only (frac uses the driver-measured peak): this box's own copy
                # bandwidth, measured like MEASURED_PEAKS.json (1 GiB copy_, best of 5)
                "box_copy_GBps": box_copy,
                "frac_of_box_copy": achieved / box_copy if box_copy else None,
                "bytes_per_launch": d["bytes"] / max(d["launches"], 1),
                "avg_launch_us": 1e6 * d["seconds"] / max(d["launches"], 1),
                "all_kernels": {k: {"launches": s["launches"], "seconds": round(s["seconds"], 6),
                                    "GBps": (s["bytes"] / s["seconds"] / 1e9 if s["seconds"] else 0.0)}
                                for k, s in stats.items()},
                "path_GBps": sum(s["bytes"] for s in stats.values()) / tot_k / 1e9 if tot_k else 0.0}

    # e2e: public API with host arrays; CSR + RHS uploads and x downloads timed
    e2e = None
    if not args.no_e2e:
        ro, ci, va = A.row_offsets, A.col_indices, A.values
        # per rank: its CSR slab (+ halo plan) and RHS slices cross PCIe every step
        h2d = 4 * (A.n + 1) + 4 * A.nnz + 8 * A.nnz + 8 * A.n * len(bs)
        e2e_iters, d2h = 0, 0
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            if sharded:   # fresh slab object: CSR + halo lists uploaded inside the region
                from paper_1301_7530_b200 import distributed as D
                Ah = D.ShardedMatrix(*shard_host, A_global.n)
            else:         # fresh: uploaded inside the region
                Ah = rcg.SparseSpdMatrix(A.n, ro, ci, va, validate=False)
            xs = []
            systems = ((Ah, b) for b in bs)
            rep2 = _e2e_sequence(rcg, systems, strat, cfg, xs)
            e2e_iters += sum(rep2.iterations())
            d2h += sum(x.nbytes for x in xs) + sum(8 * (4 * m + 1) + 16 * m for m in rep2.iterations())
        torch.cuda.synchronize()
        barrier()
        sec2 = max_over_ranks(time.perf_counter() - t0)
        if sharded:   # bytes summed over ranks; one joint sequence
            t = torch.tensor([float(h2d), float(d2h)], dtype=torch.float64, device="cuda")
            import torch.distributed as dist
            dist.all_reduce(t)
            h2d, d2h = int(t[0].item()), int(t[1].item())
        e2e = {"value": (e2e_iters if sharded else world * e2e_iters) / sec2, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h // max(args.steps, 1), "sequence_seconds": sec2 / args.steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        iters_cpu = cpu_calibrated(A, bs[0], args.cpu_seconds)
        it, dt = cpu_sample(A, bs[0], iters_cpu)
        cpu = {"value": it / dt, "unit": UNIT, "cores": blas_threads(), "kind": "port",
               "sample": f"oracle apcg_solve, first {it} iterations of system 0 (n_c=0, reorth on) in {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Q1 elasticity assembly + N(0,1) tractions)",
            "config": config_dict(A_global, args.nelem, args.systems, world, sharded),
            "sequence_seconds": sec / args.steps, "iterations_per_system": per_system,
            "n_c_before": nc_hist, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def _e2e_sequence(rcg, systems, strat, cfg, xs):
    """run_sequence with host RHS; solutions come back as host arrays."""
    rep = rcg.SequenceReport()
    state = None
    for k, (A, b) in enumerate(systems):
        if state is None:
            state = rcg.AugmentationState.from_initial(A.n, None, getattr(A, "n_ext", None))
        ncb = state.n_c
        D = rcg.guarded_deflation(A, state, rep.events)
        x, tr = rcg.apcg_solve(A, rcg.Preconditioner.jacobi(A), D, b, cfg)   # b host -> x host
        xs.append(x)
        sel = 0
        if tr.converged and tr.iterations > 0:
            rcg.update_basis_srks(state, rcg.select_spectrum(tr, strat), k)
            sel = state.n_c - ncb
        if strat.nc_limit > 0 and state.n_c >= strat.nc_limit:
            state.restart()
        rep.records.append(rcg.SystemRecord(k, tr.iterations, ncb, sel, 0.0, 0.0, 0.0, tr.converged))
    return rep


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
