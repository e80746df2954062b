#!/usr/bin/env python
"""Benchmark of the B200 augmented-PCG / SRKS recycling hot path.

Workload: BASELINE.json configs[2] ("config 3"), the largest configuration in
BASELINE.json that runs on one GPU (config 4 runs only with reorth off at one
GPU, config 5 is specified for 8 GPUs).  Newton-like sequence of 3-D linear
elasticity operators, Q1 hexahedra, 96^3 elements on the unit cube, nu = 0.3,
face x = 0 clamped -> n = 2,709,792 dofs, nnz = 214,983,054 fp64 CSR; 15
systems where E of the elements within radius 0.03 k of the centre is scaled
by 0.6^k, b^(k) = b0 + 0.01 k N(0,1); Jacobi PCG, tol 1e-8 (vs ||P^T b||),
full reorthogonalization (reference default, ~100 GB of Krylov histories at
m = 1,500), SRKS eps = 1e-10, up to 80 Ritz vectors (nc_limit = 81).

One "step" = one system of a continuing sequence (VERDICT
r01): guarded deflation build -> APCG solve -> Ritz selection -> basis
append (-> restart), with the augmentation state carried from step to step
(``SequenceRunner``, the same code as ``run_sequence``).  Step i solves system
i mod 15; at the wrap a fresh sequence starts (empty basis).  ``value`` = APCG
iterations per second over the K timed steps, operators and right-hand sides
resident in HBM (assembled on the device, outside the timed region).
``e2e`` = the same metric through the public API from HOST buffers: every
step uploads that system's CSR arrays and RHS (fresh ``SparseSpdMatrix``,
stream-format analysis included) and downloads x.  ``sequence_seconds`` =
one full 15-system sequence (per-system CUDA-event times of warm steps).
``secondary.config2`` = BASELINE config 2 (Q1 64^3, fixed A, 20 RHS, nc_limit
61), one full 20-system sequence, iters/s and seconds.

``--impl reference`` times the CPU reference path (the oracle port,
oracle/recycg_oracle.py: numpy/scipy restatement of the reference) on the same
config: each step is a bounded window of the first APCG iterations of system
0, all host threads; rank 0 only.
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
CONFIGS = {
    # name: (nelem, systems, kind, nc_limit)
    3: (96, 15, "softening", 81),
    2: (64, 20, "fixed", 61),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=3, choices=[2, 3])
    p.add_argument("--nelem", type=int, default=None, help="override elements per edge (tests / smoke runs)")
    p.add_argument("--systems", type=int, default=None)
    p.add_argument("--max-iters", type=int, default=20000)
    p.add_argument("--cpu-iters", type=int, default=30, help="CPU window: first K iterations of system 0")
    p.add_argument("--ref-seconds", type=float, default=200.0, help="--impl reference: target timed seconds")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-secondary", action="store_true")
    p.add_argument("--replicas", action="store_true", help="N>1: independent replicas instead of row sharding")
    p.add_argument("--shard-one", action="store_true",
                   help="diagnostic: run the row-sharded code path with a 1-rank NCCL communicator (under torchrun, N = 1)")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shape(args):
    nelem, systems, kind, ncl = CONFIGS[args.config]
    return (args.nelem or nelem), (args.systems or systems), kind, ncl


def config_dict(args, n, nnz, world, sharded=False):
    nelem, systems, kind, ncl = shape(args)
    what = {3: f"BASELINE config 3: Q1 elasticity {nelem}^3 elements, {systems}-system softening sequence "
               "(E x 0.6^k within r = 0.03k, b = b0 + 0.01k N(0,1))",
            2: f"BASELINE config 2: Q1 elasticity {nelem}^3 elements, fixed A, {systems} traction RHS"}[args.config]
    return {
        "workload": what + f", Jacobi APCG tol 1e-8, full reorth, SRKS eps=1e-10 nc_limit={ncl}; "
                           "step = one system of a continuing sequence",
        "n": int(n), "nnz": int(nnz), "systems": systems, "strategy": "srks", "epsilon": 1e-10,
        "nc_limit": ncl, "tol": 1e-8, "reorthogonalize": True, "preconditioner": "jacobi",
        "l2": "inputs larger than L2 (CSR 2.6 GB per operator, Krylov histories up to ~100 GB)",
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
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
                pw.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------------------
# CPU oracle window (cpu_baseline and --impl reference)


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        n = [d.get("num_threads", 1) for d in info if d.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:
        return os.cpu_count() or 1


def cpu_window(A, b, iters, threads=None):
    """Oracle apcg_solve on system 0 for exactly `iters` iterations (reorth on,
    n_c = 0: the first system of the sequence).  Returns (iterations, s)."""
    from oracle import recycg_oracle as orc
    from threadpoolctl import threadpool_limits
    inv = 1.0 / orc.diagonal(A)
    D = orc.build_deflation(A, np.zeros((A.n, 0)))
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        _, tr = orc.apcg_solve(A, inv, D, b, 1e-300, iters, reorthogonalize=True, trace_capture=True)
        dt = time.perf_counter() - t0
    return tr.iterations, dt


def host_system0(args):
    """System 0 of the workload assembled on the host (numpy), for the
    reference arm (no GPU on that path)."""
    from paper_1301_7530_b200 import problems
    nelem, systems, kind, _ = shape(args)
    A, b = next(problems.elasticity_sequence(nelem, 1, seed=0, kind=kind))
    return A, b


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    A, b = host_system0(args)
    ncpu = os.cpu_count() or 1
    # calibrate the per-step window so the K timed steps take ~ref_seconds
    it0, dt0 = cpu_window(A, b, 4)
    per_it = dt0 / max(it0, 1)
    iters = int(max(5, min(50, args.ref_seconds / max(args.steps, 1) / per_it)))
    for _ in range(args.warmup):
        cpu_window(A, b, 3)
    tot_it, tot_t = 0, 0.0
    for _ in range(args.steps):
        it, dt = cpu_window(A, b, iters)
        tot_it += it
        tot_t += dt
    value = tot_it / tot_t
    sample = (f"first {iters} APCG iterations of system 0 (n_c = 0, Jacobi, full reorth) per step, "
              f"{blas_threads()} BLAS threads on {ncpu} host cores; scipy csr_matvec (1 thread) + numpy/OpenBLAS")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "strong" if (world > 1 and not args.replicas) else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        # the same config dict as our arm at this N (the CPU arm itself always runs on rank 0's host cores)
        "config": config_dict(args, A.n, A.nnz, world, world > 1 and not args.replicas),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ncpu, "blas_threads": blas_threads(), "kind": "port",
                         "sample": sample},
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


def ncu_traffic(config):
    f = REPO / "profiles" / f"ncu_traffic_config{config}.json"
    try:
        return json.loads(f.read_text())
    except Exception:
        return {}


def device_systems(args, rank=0, world=1, sharded=False):
    """The workload's operators assembled in HBM (csrc/gen.cu) and RHS
    (host arrays, uploaded once).  Sharded: each rank keeps its row slab."""
    import torch
    from paper_1301_7530_b200 import problems
    nelem, count, kind, _ = shape(args)
    out = []
    for A, b in problems.elasticity_sequence(nelem, count, seed=0, kind=kind, device=True):
        if sharded and world == 1:
            # --shard-one: two virtual slabs in the one rank (halo exchange with itself, distributed.py)
            from paper_1301_7530_b200 import distributed as D
            cut = 3 * ((A.n // 3) // 2)
            ro_l, lci, va, plan = D.virtual_slab_system(A.row_offsets, A.col_indices, A.values, cut)
            n_global = A.n
            A.release_device()
            A = D.ShardedMatrix(ro_l, lci, va, plan, n_global)
        elif sharded:
            from paper_1301_7530_b200 import distributed as D
            ro = A.row_offsets
            bounds = D.partition_rows(ro, world, align=3)
            r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
            s0, s1 = ro[r0], ro[r1]
            ro_l, lci, va, plan = D.build_local_system(ro[r0:r1 + 1], A.col_indices[s0:s1], A.values[s0:s1],
                                                       bounds, rank)
            n_global = A.n
            A.release_device()
            A = D.ShardedMatrix(ro_l, lci, va, plan, n_global)
            b = b[r0:r1].copy()
        A.device_csr()
        out.append((A, torch.from_numpy(np.ascontiguousarray(b)).to("cuda")))
    return out


class ContinuingSequence:
    """Step i = system i mod K of a sequence carried across steps; a fresh
    sequence (empty basis) starts at each wrap."""

    def __init__(self, rcg, systems, strat, cfg):
        self.rcg, self.systems, self.strat, self.cfg = rcg, systems, strat, cfg
        self.i = 0
        self.runner = None

    def next_index(self):
        return self.i % len(self.systems)

    def step(self, system=None):
        k = self.next_index()
        if k == 0:
            self.runner = self.rcg.SequenceRunner(self.rcg.Preconditioner.jacobi, self.strat, self.cfg)
        A, b = system if system is not None else self.systems[k]
        x = self.runner.step(A, b)
        rec = self.runner.report.records[-1] if not self.runner.report.aborted else None
        if rec is None or not rec.converged:
            raise RuntimeError(f"system {k} did not converge: {self.runner.report.events}")
        self.i += 1
        return k, rec, x


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1 or args.shard_one:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1301_7530_b200 as rcg
    from paper_1301_7530_b200 import _lib

    nelem, count, kind, ncl = shape(args)
    cfg = rcg.SolveConfig(tol=1e-8, max_iters=args.max_iters, reorthogonalize=True)
    strat = rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=ncl)
    sharded = (world > 1 and not args.replicas) or args.shard_one
    if sharded:
        from paper_1301_7530_b200 import distributed as D
        D.init_comm()
    systems = device_systems(args, rank, world, sharded)
    n_global = 3 * nelem * (nelem + 1) ** 2
    nnz_global = int(systems[0][0].nnz)
    if sharded:   # slabs hold whole rows: the global count is the sum over ranks
        import torch.distributed as dist
        t = torch.tensor([nnz_global], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        nnz_global = int(t.item())

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

    seq = ContinuingSequence(rcg, systems, strat, cfg)
    stream = torch.cuda.current_stream()

    def timed_step():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        k, rec, _ = seq.step()
        e1.record(stream)
        return k, rec, (e0, e1)

    # per-system device seconds of the latest run of each system (a full
    # sequence's time is their sum; the process's very first step is cold)
    per_system = {}

    def note(k, rec, ev):
        per_system[k] = (ev[0].elapsed_time(ev[1]) * 1e-3, rec.iterations, rec.n_c_before)

    for _ in range(args.warmup):
        k, rec, ev = timed_step()
        torch.cuda.synchronize()
        note(k, rec, ev)

    ctx = _lib.context()
    t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.total_launches()
    iters = 0
    step_events = []
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        t0e.record(stream)
        for _ in range(args.steps):
            k, rec, ev = timed_step()
            iters += rec.iterations
            step_events.append((k, rec, ev))
        t1e.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = _lib.total_launches() - l0
    sec = max_over_ranks(t0e.elapsed_time(t1e) * 1e-3)
    value = (iters if sharded else world * iters) / sec
    timed_systems = [(k, rec.iterations) for k, rec, _ in step_events]
    for k, rec, ev in step_events:
        note(k, rec, ev)
    # complete one full sequence's per-system times (systems not run yet)
    while len(per_system) < count:
        k, rec, ev = timed_step()
        torch.cuda.synchronize()
        note(k, rec, ev)
    seq_seconds = max_over_ranks(sum(v[0] for v in per_system.values()))
    seq_iters = sum(v[1] for v in per_system.values())

    # roofline pass: one more step with live per-kernel event timing
    ctx.reset_stats()
    ctx.set_profiling(True)
    k_prof, rec_prof, _ = seq.step()
    ctx.set_profiling(False)
    stats_all = ctx.kernel_stats()
    phases = {k: {"seconds": round(v["seconds"], 6), "launches": v["launches"]} for k, v in stats_all.items()
              if k in ("halo", "allreduce")}
    stats = {k: v for k, v in stats_all.items() if k not in ("halo", "allreduce")}
    dom = max(stats, key=lambda kk: stats[kk]["seconds"])
    tot_k = sum(s["seconds"] for s in stats.values())
    peak, peak_src = peaks()
    box_copy = box_copy_gbps()
    d = stats[dom]
    achieved = d["bytes"] / d["seconds"] / 1e9 if d["seconds"] > 0 else 0.0
    traffic_doc = ncu_traffic(args.config).get(dom) or {}
    traffic = traffic_doc.get("bytes_per_launch")
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_detail": traffic_doc or None,
                "peak_source": peak_src, "profiled_system": k_prof, "profiled_iterations": rec_prof.iterations,
                "share_of_kernel_time": d["seconds"] / tot_k if tot_k else None,
                # context only (frac uses the driver-measured peak): this box's own copy
                # bandwidth, measured like MEASURED_PEAKS.json (1 GiB copy_, best of 6)
                "box_copy_GBps": box_copy,
                "frac_of_box_copy": achieved / box_copy if box_copy else None,
                "bytes_per_launch": d["bytes"] / max(d["launches"], 1),
                "avg_launch_us": 1e6 * d["seconds"] / max(d["launches"], 1),
                "all_kernels": {kk: {"launches": s["launches"], "seconds": round(s["seconds"], 6),
                                     "GBps": (s["bytes"] / s["seconds"] / 1e9 if s["seconds"] else 0.0)}
                                for kk, s in stats.items()},
                "path_GBps": sum(s["bytes"] for s in stats.values()) / tot_k / 1e9 if tot_k else 0.0}

    # host copies of the operators the e2e / CPU legs use (untimed); every
    # device operator of the value pass is dropped before e2e
    need = set()
    if not args.no_e2e:
        need |= {i % count for i in range(args.warmup + args.steps)}
    if rank == 0 and world == 1 and not args.no_cpu:
        need.add(0)
    host = {}
    for k, (A, bd) in enumerate(systems):
        if k in need:
            A.release_device()            # downloads the host CSR, frees the device copy
            host[k] = (A, bd.cpu().numpy())
    seq = None
    systems = None
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    e2e = None
    if not args.no_e2e:
        from paper_1301_7530_b200 import distributed as Dm

        def host_system(k):
            Aref, b = host[k]
            ro, ci, va = Aref.row_offsets, Aref.col_indices, Aref.values
            if sharded:
                return Dm.ShardedMatrix(ro, ci, va, Aref.plan, n_global), b
            return rcg.SparseSpdMatrix(int(Aref.n), ro, ci, va, validate=False), b

        placeholder = [None] * count
        seq2 = ContinuingSequence(rcg, placeholder, strat, cfg)
        for _ in range(args.warmup):
            k = seq2.next_index()
            A_h, b_h = host_system(k)
            seq2.step((A_h, b_h))
            A_h.release_device()
        e2e_iters, h2d, d2h = 0, 0, 0
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        up_s = 0.0
        for _ in range(args.steps):
            k = seq2.next_index()
            A_h, b_h = host_system(k)        # fresh object: CSR uploaded + analysed inside the region
            tu = time.perf_counter()
            A_h.device_csr()                 # (the solve would trigger it; called first to time it)
            torch.cuda.synchronize()
            up_s += time.perf_counter() - tu
            _, rec, x = seq2.step((A_h, b_h))
            A_h.release_device()
            e2e_iters += rec.iterations
            h2d += (4 * (A_h.n + 1) + 12 * A_h.nnz + 8 * A_h.n)
            d2h += np.asarray(x).nbytes + 8 * (4 * rec.iterations + 2)
        torch.cuda.synchronize()
        barrier()
        sec2 = max_over_ranks(time.perf_counter() - t0)
        if sharded:
            import torch.distributed as dist
            t = torch.tensor([float(h2d), float(d2h)], dtype=torch.float64, device="cuda")
            dist.all_reduce(t)
            h2d, d2h = int(t[0].item()), int(t[1].item())
        e2e = {"value": (e2e_iters if sharded else world * e2e_iters) / sec2, "unit": UNIT,
               "h2d_bytes_per_step": h2d // max(args.steps, 1), "d2h_bytes_per_step": d2h // max(args.steps, 1),
               "seconds": sec2, "iterations": e2e_iters, "csr_upload_seconds": up_s}
        seq2 = None
        torch.cuda.synchronize()

    # secondary: BASELINE config 2, one full 20-system sequence
    secondary = None
    if not args.no_secondary and args.config == 3 and not sharded and args.nelem is None:
        from paper_1301_7530_b200 import problems
        sys2 = [(A, torch.from_numpy(b).to("cuda")) for A, b in
                problems.elasticity_sequence(64, 20, seed=0, kind="fixed", device=True)]
        strat2 = rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=61)
        rcg.run_sequence(iter(sys2[:2]), rcg.Preconditioner.jacobi, strat2, cfg)      # warm-up
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize()
        e0.record(stream)
        rep2 = rcg.run_sequence(iter(sys2), rcg.Preconditioner.jacobi, strat2, cfg)
        e1.record(stream)
        torch.cuda.synchronize()
        s2 = e0.elapsed_time(e1) * 1e-3
        secondary = {"config2": {"workload": "BASELINE config 2: Q1 64^3, fixed A, 20 RHS, full reorth, "
                                             "SRKS eps=1e-10 nc_limit=61; one full sequence",
                                 "iters_per_s": sum(rep2.iterations()) / s2, "sequence_seconds": s2,
                                 "iterations": rep2.iterations(), "n_c_before": rep2.n_c_history()}}
        del sys2
        torch.cuda.synchronize()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        A0, b0 = host[0]
        ncpu = os.cpu_count() or 1
        it_all, dt_all = cpu_window(A0, b0, args.cpu_iters)
        it_one, dt_one = cpu_window(A0, b0, args.cpu_iters, threads=1)
        cpu = {"value": it_all / dt_all, "unit": UNIT, "cores": ncpu, "blas_threads": blas_threads(),
               "kind": "port", "value_1thread": it_one / dt_one,
               "sample": f"oracle apcg_solve (reference algorithm, numpy/scipy), first {it_all} iterations of "
                         f"system 0 (n_c = 0, Jacobi, full reorth): {dt_all:.1f} s with all {ncpu} host cores, "
                         f"{dt_one:.1f} s with 1 thread"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Q1 elasticity assembly in HBM + N(0,1) tractions)",
            "config": config_dict(args, n_global, nnz_global or 0, world, sharded),
            "timed_systems": timed_systems, "iterations_timed": iters,
            "sequence_seconds": seq_seconds, "sequence_iterations": seq_iters,
            "sequence_iters_per_s": seq_iters / seq_seconds if seq_seconds else None,
            "per_system": {str(k): {"seconds": round(v[0], 4), "iterations": v[1], "n_c_before": v[2]}
                           for k, v in sorted(per_system.items())},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "secondary": secondary,
            "phases_profiled_step": ({"kernels_seconds": sum(s["seconds"] for s in stats.values()), **phases}
                                     if (world > 1 or args.shard_one) else None),
            "gpu_launches": launches, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if sharded:
        from paper_1301_7530_b200 import distributed as D
        D.destroy_comm()            # graphs, then the communicator: nothing NCCL left for interpreter exit
    if world > 1 or args.shard_one:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
