"""Row-sharded multi-GPU execution.

One process per GPU (torchrun).  Each rank owns a contiguous slab of rows
(x-slabs of nodes for the Q1 elasticity operators, z-planes for 7-point
diffusion).  The local CSR keeps owned columns as 0..n_local-1 and appends the
ghost columns it reads after them, grouped by owner rank; before every SpMV
the ghost entries are exchanged with ncclSend/ncclRecv, and the per-iteration
reductions are one packed ncclAllReduce per dependency point:

    (w, Aw) [1]  |  ||r||^2, AC^T y [1 + n_c]  |  (r, z), AW^T z, AW^T w [1 + 2(j+1)]

Everything replicated (alpha, beta, the convergence test, the coarse Cholesky,
the tridiagonal eigensolve and the Ritz selection) is computed identically on
every rank from bitwise-identical allreduce results, so the ranks stop at the
same iteration with no extra synchronization.  Ritz vectors Y = Z Qtilde are
purely local row blocks.

The partition and halo-plan construction here is host logic over
``torch.distributed`` (any backend): the CPU test suite runs it under gloo with
world_size 2, together with a numpy emulation of the sharded iteration, and
checks it against the serial oracle (tests/test_sharded_cpu.py).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import ContractViolation, SparseSpdMatrix

__all__ = ["partition_rows", "HaloPlan", "build_local_system", "local_systems_all", "ShardedMatrix", "init_comm",
           "destroy_comm", "virtual_slab_system",
           "init_loopback", "LoopbackGroup", "nccl_library"]


def partition_rows(row_offsets, nranks, align=1):
    """Contiguous row blocks balanced by nonzeros; boundaries are multiples of
    ``align`` (3 keeps the dofs of a node on one rank).  Returns nranks+1 bounds."""
    ro = np.asarray(row_offsets, dtype=np.int64)
    n = len(ro) - 1
    if n % align:
        raise ContractViolation("n must be a multiple of align")
    units = n // align
    unit_nnz = ro[align::align] - ro[0:-1:align] if align > 1 else np.diff(ro)
    cum = np.concatenate([[0], np.cumsum(unit_nnz)])
    total = cum[-1]
    bounds = [0]
    for q in range(1, nranks):
        u = int(np.searchsorted(cum, total * q / nranks))
        u = min(max(u, bounds[-1] // align), units)
        bounds.append(u * align)
    bounds.append(n)
    return np.asarray(bounds, dtype=np.int64)


@dataclass
class HaloPlan:
    """Host description of one rank's halo (see include/rcg.h rcg_halo)."""

    nranks: int
    rank: int
    n_local: int
    n_ghost: int
    send_idx: np.ndarray      # local indices to pack, grouped by destination rank
    send_off: np.ndarray      # [nranks+1]
    recv_off: np.ndarray      # [nranks+1] offsets into the ghost region
    ghost_global: np.ndarray  # global index of each ghost entry


def _ghosts(ci, r0, r1, bounds, nranks):
    ci = np.asarray(ci, dtype=np.int64)
    owned = (ci >= r0) & (ci < r1)
    ghosts = np.unique(ci[~owned])
    owner = np.searchsorted(bounds, ghosts, side="right") - 1
    return owned, ghosts, owner


def local_systems_all(row_offsets, col_indices, values, bounds):
    """Every rank's (ro, lci, va, plan) computed in one process (the needs
    exchange done locally) — the same plans build_local_system produces over
    torch.distributed; used by the single-GPU loopback validation."""
    nranks = len(bounds) - 1
    ro_g = np.asarray(row_offsets, dtype=np.int64)
    parts, needs_all = [], []
    for rank in range(nranks):
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        s, e = ro_g[r0], ro_g[r1]
        _, ghosts, owner = _ghosts(col_indices[s:e], r0, r1, bounds, nranks)
        needs_all.append([ghosts[owner == q] for q in range(nranks)])
        parts.append((ro_g[r0:r1 + 1], col_indices[s:e], values[s:e]))
    return [build_local_system(*parts[r], bounds, r, gathered=needs_all) for r in range(nranks)]


def build_local_system(ro, ci, va, bounds, rank, group=None, gathered=None):
    """This rank's local CSR (owned + ghost column numbering) and halo plan.

    ``ro/ci/va`` are the rows of THIS rank only (global column indices),
    ``bounds`` the partition.  Ghost requirements are exchanged with every
    rank over ``torch.distributed`` (all_gather_object), so the plan is
    symmetric by construction: rank p sends to q exactly the entries q asked
    p for, in q's ghost order.
    """
    nranks = len(bounds) - 1
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    n_local = r1 - r0
    ro = np.asarray(ro, dtype=np.int64)
    ci = np.asarray(ci, dtype=np.int64)
    if len(ro) != n_local + 1:
        raise ContractViolation("row_offsets must cover exactly this rank's rows")
    owned = (ci >= r0) & (ci < r1)
    ghosts = np.unique(ci[~owned])                         # sorted: grouped by owner, ascending
    owner = np.searchsorted(bounds, ghosts, side="right") - 1
    recv_counts = np.bincount(owner, minlength=nranks).astype(np.int64)
    recv_off = np.concatenate([[0], np.cumsum(recv_counts)]).astype(np.int64)
    # local column numbering
    lci = np.empty_like(ci)
    lci[owned] = ci[owned] - r0
    lci[~owned] = n_local + np.searchsorted(ghosts, ci[~owned])
    # who needs what from whom
    needs = [ghosts[owner == q] for q in range(nranks)]
    if gathered is None:
        import torch.distributed as dist
        gathered = [None] * nranks
        if nranks > 1:
            dist.all_gather_object(gathered, needs, group=group)
        else:
            gathered = [needs]
    send_lists = [np.asarray(gathered[q][rank], dtype=np.int64) - r0 if q != rank else np.zeros(0, np.int64)
                  for q in range(nranks)]
    for q, lst in enumerate(send_lists):
        if len(lst) and (lst.min() < 0 or lst.max() >= n_local):
            raise ContractViolation(f"rank {q} requested rows not owned by rank {rank}")
    send_off = np.concatenate([[0], np.cumsum([len(x) for x in send_lists])]).astype(np.int64)
    send_idx = np.concatenate(send_lists).astype(np.int32) if send_off[-1] else np.zeros(0, np.int32)
    plan = HaloPlan(nranks, rank, n_local, len(ghosts), send_idx, send_off, recv_off, ghosts)
    return (ro - ro[0]), lci.astype(np.int32), np.asarray(va, dtype=np.float64), plan


def virtual_slab_system(row_offsets, col_indices, values, cut):
    """One rank's rows cut into two virtual slabs at row ``cut``: couplings
    between the slabs read ghost copies of the rank's OWN entries (listed
    after the n local columns), so the rank exchanges a halo with itself.
    The operator is unchanged.  With ``RCG_COMM_FORCE=1`` on a 1-rank NCCL
    communicator the exchange is an ncclSend / ncclRecv to self: the whole
    sharded iteration (pack, NCCL, unpack, slab SpMV, allreduces, graph
    capture) then runs on one GPU (tests, ``bench.py --shard-one``).
    Returns (ro, lci, va, plan) like ``build_local_system``."""
    ro = np.asarray(row_offsets, dtype=np.int64)
    ci = np.asarray(col_indices, dtype=np.int64)
    n = len(ro) - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ro))
    cross = (rows < cut) != (ci < cut)
    ghosts = np.unique(ci[cross])
    lci = ci.copy()
    lci[cross] = n + np.searchsorted(ghosts, ci[cross])
    off = np.array([0, len(ghosts)], dtype=np.int64)
    plan = HaloPlan(1, 0, n, len(ghosts), ghosts.astype(np.int32), off, off.copy(), ghosts)
    return ro - ro[0], lci.astype(np.int32), np.asarray(values, dtype=np.float64), plan


class ShardedMatrix(SparseSpdMatrix):
    """This rank's row slab as a SparseSpdMatrix (n = n_local rows) plus its
    halo plan.  Passed to build_deflation / apcg_solve / run_sequence it
    routes them to the sharded C-ABI entry points."""

    def __init__(self, ro, lci, va, plan: HaloPlan, n_global):
        super().__init__(plan.n_local, ro, lci, va, validate=False)
        object.__setattr__(self, "plan", plan)
        object.__setattr__(self, "n_global", int(n_global))
        object.__setattr__(self, "_halo_dev", None)

    @property
    def n_ext(self):
        return self.plan.n_local + self.plan.n_ghost

    def _before_stream_copy(self, h):
        # a slab of a grid operator keeps the symmetric block-DIA stream format:
        # its local-local block is a principal submatrix (still symmetric, same
        # diagonals); the ghost-column entries go to a remainder list
        if self.plan.n_ghost > 0 and os.environ.get("RCG_SLAB_DIA", "1") != "0":
            h.add_remainder(self.n, self.row_offsets, self.col_indices, self.values)

    def halo_struct(self):
        """ctypes rcg_halo with device send lists (cached)."""
        h = self._halo_dev
        if h is None:
            torch = _lib.require_cuda()
            p = self.plan
            idx = torch.from_numpy(np.ascontiguousarray(p.send_idx, dtype=np.int32)).to("cuda") \
                if len(p.send_idx) else torch.zeros(1, dtype=torch.int32, device="cuda")
            buf = torch.empty(max(int(p.send_off[-1]), 1), dtype=torch.float64, device="cuda")
            so = (C.c_int64 * (p.nranks + 1))(*[int(v) for v in p.send_off])
            rv = (C.c_int64 * (p.nranks + 1))(*[int(v) for v in p.recv_off])
            st = _lib.RcgHalo(p.nranks, p.rank, p.n_local, p.n_ghost, idx.data_ptr(),
                              C.cast(so, C.c_void_p), C.cast(rv, C.c_void_p), buf.data_ptr())
            h = (st, idx, buf, so, rv)
            object.__setattr__(self, "_halo_dev", h)
        return h[0]


def nccl_library():
    """Path of the NCCL torch uses (nvidia-nccl wheel), or None."""
    try:
        import nvidia.nccl
        d = os.path.dirname(nvidia.nccl.__file__ or list(nvidia.nccl.__path__)[0])
        p = os.path.join(d, "lib", "libnccl.so.2")
        return p if os.path.exists(p) else None
    except Exception:
        return None


def init_comm(group=None):
    """Create this rank's NCCL communicator inside the rcg context (rank 0
    makes the unique id, torch.distributed broadcasts it)."""
    import torch.distributed as dist
    ctx = _lib.context()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    path = nccl_library()
    pb = path.encode() if path else None
    obj = [None]
    if rank == 0:
        buf = (C.c_char * 128)()
        ctx.check(ctx.lib.rcg_comm_unique_id(pb, buf), "nccl unique id")
        obj[0] = bytes(buf)
    dist.broadcast_object_list(obj, src=0, group=group)
    idb = (C.c_char * 128).from_buffer_copy(obj[0])
    ctx.check(ctx.lib.rcg_comm_init(ctx.h, pb, idb, world, rank), "nccl comm init")
    return ctx


def destroy_comm():
    """Tear down this thread's communicator (captured batch graphs first, then
    ncclCommDestroy): call before ``torch.distributed.destroy_process_group``
    / process exit so that no NCCL teardown is left to interpreter shutdown."""
    ctx = _lib.context()
    ctx.check(ctx.lib.rcg_comm_destroy(ctx.h), "nccl comm destroy")


class LoopbackGroup:
    """Single-process loopback transport for validating the sharded path on
    one GPU: ``nranks`` host threads, each with its own CUDA stream and rcg
    context, act as ranks (include/rcg.h rcg_loop_group_create)."""

    def __init__(self, nranks):
        lib = _lib.load()
        h = C.c_void_p()
        rc = lib.rcg_loop_group_create(int(nranks), C.byref(h))
        if rc != 0:
            raise RuntimeError(f"rcg_loop_group_create failed ({rc})")
        self.h, self.nranks, self.lib = h, int(nranks), lib

    def close(self):
        if self.h:
            self.lib.rcg_loop_group_destroy(self.h)
            self.h = None


def init_loopback(group: LoopbackGroup, rank):
    """Bind this thread's rcg context (current device and stream) to rank
    ``rank`` of a loopback group."""
    ctx = _lib.context()
    ctx.check(ctx.lib.rcg_comm_init_loopback(ctx.h, group.h, int(rank)), "loopback init")
    return ctx
