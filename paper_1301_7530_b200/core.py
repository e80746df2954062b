"""Operators and small dense kernels of the hot path, B200-resident.

Mirrors ``/root/reference/pkg/src/recycg/core.py``: the same names, dataclasses
and exceptions, but every numeric operation runs in ``librcg.so`` on the GPU
(SpMV ``core.py:110-119``, guarded Cholesky ``core.py:195-243``, tridiagonal
eigensolver ``core.py:169-177``).  Host numpy arrays are accepted and returned
wherever the reference takes/returns them; torch CUDA tensors pass through
without a host round trip.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import os as _os

import numpy as np

from .core_errors import ContractViolation, NumericalFailure, RankDeficient
from . import _lib

__all__ = ["ContractViolation", "RankDeficient", "NumericalFailure", "SparseSpdMatrix", "spmv",
           "TridiagSym", "EigDecomposition", "tridiag_eig", "dense_sym_eig", "dense_cholesky"]


# ---------------------------------------------------------------------------
# host <-> device helpers


def _torch():
    return _lib.require_cuda()


def is_device_tensor(x):
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def to_dev(x, dtype="f64"):
    """(contiguous CUDA float64 tensor, came_from_host)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x
        if t.device.type != "cuda":
            t = t.to("cuda")
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        return t.contiguous(), False
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(arr).to("cuda"), True


def from_dev(t, host):
    return t.cpu().numpy() if host else t


class _Stager:
    """Host -> device upload of large arrays through a ring of pinned staging
    buffers: host threads copy chunk i + 1 into pinned memory (numpy releases
    the GIL) while the copy engine moves chunk i, so a 2.6 GB CSR (config 3)
    crosses at PCIe speed instead of through the driver's single-threaded
    pageable bounce buffer (0.24 s -> ~0.06 s per operator)."""

    CHUNK = 64 << 20
    NBUF = 4
    THREADS = 8

    def __init__(self):
        torch = _torch()
        from concurrent.futures import ThreadPoolExecutor
        self.bufs = [torch.empty(self.CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(self.NBUF)]
        self.views = [b.numpy() for b in self.bufs]
        self.events = [None] * self.NBUF
        self.stream = torch.cuda.Stream()
        self.pool = ThreadPoolExecutor(self.THREADS)

    def _fill(self, dst, src):
        n = len(src)
        step = -(-n // self.THREADS)
        parts = [(dst[i:i + step], src[i:i + step]) for i in range(0, n, step)]
        list(self.pool.map(lambda p: np.copyto(p[0], p[1]), parts))

    def upload(self, arr):
        torch = _torch()
        arr = np.ascontiguousarray(arr)
        out = torch.empty(arr.shape, dtype=getattr(torch, str(arr.dtype)), device="cuda")
        src = arr.reshape(-1).view(np.uint8)
        dst = out.view(-1).view(torch.uint8)
        self.stream.wait_stream(torch.cuda.current_stream())   # `out` was allocated on the current stream
        for i, off in enumerate(range(0, len(src), self.CHUNK)):
            k = i % self.NBUF
            if self.events[k] is not None:
                self.events[k].synchronize()                     # its previous DMA has drained
            nb = min(self.CHUNK, len(src) - off)
            self._fill(self.views[k][:nb], src[off:off + nb])
            with torch.cuda.stream(self.stream):
                dst[off:off + nb].copy_(self.bufs[k][:nb], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.stream)
            self.events[k] = ev
        torch.cuda.current_stream().wait_stream(self.stream)
        out.record_stream(self.stream)
        return out


_stagers = {}


def h2d(arr):
    """Device copy of a host array; large arrays go through the pinned ring."""
    torch = _torch()
    arr = np.asarray(arr)
    if arr.nbytes < (32 << 20) or _os.environ.get("RCG_PINNED_UPLOAD", "1") == "0":
        return torch.from_numpy(np.ascontiguousarray(arr)).to("cuda")
    dev = torch.cuda.current_device()
    st = _stagers.get(dev)
    if st is None:
        st = _stagers[dev] = _Stager()
    return st.upload(arr)


def pad_ld(n):
    return max(32, ((int(n) + 31) // 32) * 32)


def colmajor_from_host(M, ld=None):
    """Host (n, k) array -> device (k, ld) tensor = column-major n x k."""
    torch = _torch()
    M = np.asarray(M, dtype=np.float64)
    n, k = M.shape
    ld = pad_ld(n) if ld is None else ld
    out = torch.zeros((k, ld), dtype=torch.float64, device="cuda")
    if k and n:
        out[:, :n] = torch.from_numpy(np.ascontiguousarray(M.T)).to("cuda")
    return out


# ---------------------------------------------------------------------------
# CSR operator


def ghost_remainder_ell(n, row_offsets, col_indices, values):
    """The entries of a row slab whose (local) column is >= n, i.e. its ghost
    columns, as an ELL list over the rows that have any: ``(row_ids[int32 R],
    cols[int32 W x R], vals[float64 W x R])`` with entry e of listed row s at
    ``[e, s]``, CSR order kept, pads = (a valid column, 0.0).  None when the
    slab has no ghost entries.  Host-side (numpy); layout of ``rcg_csr.rem_*``."""
    ro = np.asarray(row_offsets, dtype=np.int64)
    ci = np.asarray(col_indices)
    pos = np.flatnonzero(ci >= n)                 # a few percent of the entries: everything below is on these only
    if len(pos) == 0:
        return None
    rows = np.searchsorted(ro, pos, side="right") - 1
    ids, first, counts = np.unique(rows, return_index=True, return_counts=True)
    width, nrow = int(counts.max()), len(ids)
    slot = np.arange(len(rows)) - np.repeat(first, counts)
    srow = np.repeat(np.arange(nrow), counts)
    gci = ci[pos]
    eci = np.full((width, nrow), int(gci[0]), dtype=np.int32)
    eva = np.zeros((width, nrow), dtype=np.float64)
    eci[slot, srow] = gci
    eva[slot, srow] = np.asarray(values)[pos]
    return ids.astype(np.int32), eci, eva


class _DevCsr:
    __slots__ = ("ro", "ci", "va", "bro", "bci", "bval", "doffs", "dvals", "rem", "struct")

    def __init__(self, ro, ci, va, n, nnz, ro64):
        self.ro, self.ci, self.va = ro, ci, va
        self.bro = self.bci = self.bval = None
        self.doffs = self.dvals = None
        self.rem = None
        self.struct = _lib.RcgCsr(n, nnz, ro.data_ptr(), 1 if ro64 else 0, 0, ci.data_ptr(), va.data_ptr(),
                                  None, None, None)

    def add_remainder(self, n, row_offsets, col_indices, values):
        """Row slab: list the ghost-column entries (local column >= n) as an
        entry-major (ELL) remainder (``rcg_csr.rem_*``), so that the local-local
        block can take the symmetric block-DIA copy; the slab SpMV is then the
        DIA kernel plus ``rem_body`` over these rows (spmv.cu)."""
        torch = _torch()
        ell = ghost_remainder_ell(n, row_offsets, col_indices, values)
        if ell is None:
            return
        ids, eci, eva = ell
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda")
        self.rem = (dev(ids), dev(eci), dev(eva))
        self.struct.rem_rows = len(ids)
        self.struct.rem_width = eci.shape[0]
        self.struct.rem_row_ids = self.rem[0].data_ptr()
        self.struct.rem_col_indices = self.rem[1].data_ptr()
        self.struct.rem_values = self.rem[2].data_ptr()

    def add_dia(self, ctx, b):
        """Attach a symmetric block-DIA copy (spmv.cu ``dia_body``) when every
        entry lies on a few block diagonals, the operator is exactly
        symmetric and the stored upper blocks stream fewer bytes than CSR.
        Returns False (nothing attached) otherwise."""
        torch = _torch()
        n, nnz = int(self.struct.n), int(self.struct.nnz)
        offs = (_lib.C.c_int64 * 64)()
        nd = _lib.C.c_int32(0)
        ctx.check(ctx.lib.rcg_csr_dia_analyze(ctx.h, _lib.C.byref(self.struct), b, offs, _lib.C.byref(nd)),
                  "dia_analyze")
        up = [offs[i] for i in range(nd.value) if offs[i] >= 0]
        if not up or 8.0 * len(up) * b * n > 8.0 * nnz + 4.0 * nnz / (9 if b == 3 else 1):
            return False
        doffs = torch.tensor(up, dtype=torch.int64, device="cuda")
        dvals = torch.empty(len(up) * b * b * 32 * ((n // b + 31) // 32), dtype=torch.float64, device="cuda")
        sym = _lib.C.c_int32(0)
        ctx.check(ctx.lib.rcg_csr_dia_build(ctx.h, _lib.C.byref(self.struct), b, _lib.ptr(doffs), len(up),
                                            _lib.ptr(dvals), _lib.C.byref(sym)), "dia_build")
        if not sym.value:
            return False
        self.doffs, self.dvals = doffs, dvals
        self.struct.dia_offsets = doffs.data_ptr()
        self.struct.dia_values = dvals.data_ptr()
        self.struct.dia_block = b
        self.struct.dia_count = len(up)
        return True

    def add_block3(self, ctx):
        """Detect 3x3 block structure on the device and attach a BSR copy
        (SpMV then streams 8.4 instead of 12 bytes per nonzero)."""
        torch = _torch()
        flag = _lib.C.c_int32(0)
        ctx.check(ctx.lib.rcg_csr_block3_analyze(ctx.h, _lib.C.byref(self.struct), _lib.C.byref(flag)),
                  "block3_analyze")
        if not flag.value:
            return False
        n, nnz = int(self.struct.n), int(self.struct.nnz)
        self.bro = torch.empty(n // 3 + 1, dtype=torch.int32, device="cuda")
        self.bci = torch.empty(max(nnz // 9, 1), dtype=torch.int32, device="cuda")
        self.bval = torch.empty(max(nnz, 1), dtype=torch.float64, device="cuda")
        ctx.check(ctx.lib.rcg_csr_block3_build(ctx.h, _lib.C.byref(self.struct), _lib.ptr(self.bro),
                                               _lib.ptr(self.bci), _lib.ptr(self.bval)), "block3_build")
        self.struct.bsr_row_offsets = self.bro.data_ptr()
        self.struct.bsr_col_indices = self.bci.data_ptr()
        self.struct.bsr_values = self.bval.data_ptr()
        self.struct.block = 3
        if _os.environ.get("RCG_SELL", "1") != "0":
            self._slice(ctx)
        return True

    def _slice(self, ctx):
        """Re-lay the BSR copy as 32-row slices (SELL-32 over block rows,
        spmv.cu ``sell3_body``) and drop the plain BSR arrays."""
        torch = _torch()
        nchunks = (int(self.struct.n) // 3 + 31) // 32
        off = torch.empty(nchunks + 1, dtype=torch.int32, device="cuda")
        slots = _lib.C.c_int64(0)
        ctx.check(ctx.lib.rcg_csr_block3_slice_plan(ctx.h, _lib.C.byref(self.struct), _lib.ptr(off),
                                                    _lib.C.byref(slots)), "block3_slice_plan")
        sci = torch.empty(max(32 * slots.value, 1), dtype=torch.int32, device="cuda")
        sval = torch.empty(max(288 * slots.value, 1), dtype=torch.float64, device="cuda")
        ctx.check(ctx.lib.rcg_csr_block3_slice_build(ctx.h, _lib.C.byref(self.struct), _lib.ptr(off),
                                                     _lib.ptr(sci), _lib.ptr(sval)), "block3_slice_build")
        torch.cuda.synchronize()  # the plain BSR arrays are released below
        self.bro, self.bci, self.bval = off, sci, sval
        self.struct.bsr_row_offsets = off.data_ptr()
        self.struct.bsr_col_indices = sci.data_ptr()
        self.struct.bsr_values = sval.data_ptr()
        self.struct.bsr_slice = 32


@dataclass(frozen=True, eq=False)
class SparseSpdMatrix:
    """Symmetric positive definite operator in CSR form (full pattern stored),
    ``core.py:34-111``.  Construction validates the reference invariants
    (``core.py:56-73``) unless ``validate=False`` (generators that are symmetric
    by construction at 10^8 nnz).  The device copy is uploaded on first use and
    cached per device."""

    n: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray
    validate: bool = field(default=True, repr=False, compare=False)
    use_block3: bool = field(default=True, repr=False, compare=False)

    def __post_init__(self):
        ro = np.asarray(self.row_offsets, dtype=np.int64)
        ci = np.asarray(self.col_indices)
        if ci.dtype not in (np.int32, np.int64):
            ci = ci.astype(np.int64)
        va = np.asarray(self.values, dtype=np.float64)
        object.__setattr__(self, "row_offsets", ro)
        object.__setattr__(self, "col_indices", ci)
        object.__setattr__(self, "values", va)
        object.__setattr__(self, "_dev", {})
        n = int(self.n)
        if len(ro) != n + 1 or ro[0] != 0 or ro[-1] != len(ci) or len(ci) != len(va):
            raise ContractViolation("inconsistent CSR arrays")
        if np.any(np.diff(ro) < 0):
            raise ContractViolation("row_offsets must be nondecreasing")
        if n >= 2 ** 31 - 1:
            raise ContractViolation("n must fit int32 column indices")
        if self.validate:
            self._validate()

    def _validate(self):
        import scipy.sparse
        ro, ci, va = self.row_offsets, self.col_indices, self.values
        if len(ci) > 0:
            jumps = np.diff(ci.astype(np.int64))
            starts = np.zeros(len(ci), dtype=bool)
            starts[ro[1:-1]] = True
            if np.any(jumps[~starts[1:]] <= 0):
                raise ContractViolation("col_indices must be sorted within each row")
        rows = np.repeat(np.arange(self.n), np.diff(ro))
        diag = rows == ci
        if np.count_nonzero(diag) != self.n or np.any(va[diag] <= 0.0):
            raise ContractViolation("all diagonal entries must be present and positive")
        csr = scipy.sparse.csr_matrix((va, ci, ro), shape=(self.n, self.n))
        if (csr != csr.T).nnz != 0:
            raise ContractViolation("matrix is not symmetric (pattern or values)")

    # -- constructors (core.py:76-98) --------------------------------------
    @classmethod
    def from_dense(cls, dense, keep_zeros=False):
        dense = np.asarray(dense, dtype=np.float64)
        n = dense.shape[0]
        if dense.shape != (n, n):
            raise ContractViolation("dense input must be square")
        sym = 0.5 * (dense + dense.T)
        if keep_zeros:
            ro = np.arange(n + 1) * n
            ci = np.tile(np.arange(n), n)
            return cls(n, ro, ci, sym.ravel())
        mask = sym != 0.0
        counts = mask.sum(axis=1)
        ro = np.concatenate([[0], np.cumsum(counts)])
        ci = np.nonzero(mask)[1]
        return cls(n, ro, ci, sym[mask])

    @classmethod
    def from_scipy(cls, mat):
        import scipy.sparse
        csr = scipy.sparse.csr_matrix(mat)
        csr.sum_duplicates()
        csr.sort_indices()
        return cls(csr.shape[0], csr.indptr, csr.indices, csr.data)

    def to_dense(self):
        out = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.row_offsets))
        out[rows, self.col_indices] = self.values
        return out

    @property
    def nnz(self):
        return len(self.values)

    # -- device ----------------------------------------------------------
    def device_csr(self):
        torch = _torch()
        dev = torch.cuda.current_device()
        h = self._dev.get(dev)
        if h is None:
            ro64 = self.nnz >= 2 ** 31 - 1
            ro = h2d(self.row_offsets.astype(np.int64 if ro64 else np.int32))
            ci = h2d(np.ascontiguousarray(self.col_indices, dtype=np.int32))
            va = h2d(self.values)
            h = _DevCsr(ro, ci, va, self.n, self.nnz, ro64)
            self._before_stream_copy(h)
            _maybe_block3(h, self.n, self.nnz, self.use_block3)
            self._dev[dev] = h
        return h

    def _before_stream_copy(self, h):
        """Hook for subclasses (row slabs attach their ghost-column remainder)."""

    def release_device(self):
        """Drop the cached device copy (the next use uploads again)."""
        self._dev.clear()

    def diagonal(self):
        """diag(A) (``core.py:103-104``), extracted on the device."""
        d, host = self.diagonal_device(), True
        return from_dev(d, host)

    def diagonal_device(self, inverse=False):
        torch = _torch()
        h = self.device_csr()
        ctx = _lib.context()
        out = torch.empty(self.n, dtype=torch.float64, device="cuda")
        if inverse:
            ctx.check(ctx.lib.rcg_csr_diagonal(ctx.h, _lib.C.byref(h.struct), None, _lib.ptr(out)), "diagonal")
        else:
            ctx.check(ctx.lib.rcg_csr_diagonal(ctx.h, _lib.C.byref(h.struct), _lib.ptr(out), None), "diagonal")
        return out

    def __matmul__(self, other):
        """A @ x (``core.py:110-111``) for a vector or an (n, k) block."""
        torch = _torch()
        host = not is_device_tensor(other)
        arr = np.asarray(other, dtype=np.float64) if host else other
        ctx = _lib.context()
        h = self.device_csr()
        if arr.ndim == 1:
            if arr.shape[0] != self.n:
                raise ContractViolation(f"vector length {arr.shape} does not match n={self.n}")
            x, _ = to_dev(arr)
            y = torch.empty(self.n, dtype=torch.float64, device="cuda")
            ctx.check(ctx.lib.rcg_spmv(ctx.h, _lib.C.byref(h.struct), _lib.ptr(x), _lib.ptr(y)), "spmv")
            return from_dev(y, host)
        if arr.ndim == 2:
            if arr.shape[0] != self.n:
                raise ContractViolation("block row count does not match n")
            k = arr.shape[1]
            if host:
                X = colmajor_from_host(arr, ld=self.n)
            else:
                X = arr.to(torch.float64).t().contiguous()
            Y = torch.empty((k, self.n), dtype=torch.float64, device="cuda")
            ctx.check(ctx.lib.rcg_spmm(ctx.h, _lib.C.byref(h.struct), _lib.ptr(X), self.n, k, _lib.ptr(Y),
                                       self.n), "spmm")
            return Y.cpu().numpy().T.copy() if host else Y.t()
        raise ContractViolation("operand must be a vector or an (n, k) block")


def _maybe_block3(h, n, nnz, use_block3):
    """Pick the SpMV stream format: symmetric block-DIA for grid operators
    (stencils, structured Q1 meshes), else sliced 3x3 blocks for
    block-structured FEM operators, else scalar CSR."""
    if not use_block3:
        return
    blocky = n % 3 == 0 and nnz % 9 == 0 and nnz >= 9 * n // 3 * 2
    # 3x3-block DIA halves the bytes of structured Q1 operators; its nine
    # value streams per diagonal run at ~4 TB/s (vs 6.7 for the sliced
    # blocks), still 8-18% faster per SpMV at 64^3..160^3 (RCG_DIA3=0: off)
    dia_b = 3 if blocky else 1
    # fewer bytes only pay when the operator streams from HBM: an L2-resident
    # CSR (config 1, 1 MB) keeps the shorter-latency CSR kernel
    streams = 12 * nnz > (32 << 20) or _os.environ.get("RCG_DIA_SMALL", "0") == "1"
    if _os.environ.get("RCG_DIA", "1") != "0" and n > 0 and streams and \
            (dia_b == 1 or _os.environ.get("RCG_DIA3", "1") == "1"):
        if h.add_dia(_lib.context(), dia_b):
            return
    if _os.environ.get("RCG_BSR", "1") != "0" and blocky:
        h.add_block3(_lib.context())


class DeviceSparseSpdMatrix(SparseSpdMatrix):
    """A ``SparseSpdMatrix`` assembled directly in HBM (``problems.py`` device
    generators, ``csrc/gen.cu``).  The device CSR is the primary copy; the
    host arrays (``row_offsets``, ``col_indices``, ``values``) are downloaded
    on first access, so oracle checks and host-side code still see the
    reference's CSR container."""

    def __init__(self, n, dev_csr, device, use_block3=True):  # noqa: D107 (frozen dataclass: set via object)
        object.__setattr__(self, "n", int(n))
        object.__setattr__(self, "validate", False)
        object.__setattr__(self, "use_block3", use_block3)
        object.__setattr__(self, "_dev", {device: dev_csr})
        object.__setattr__(self, "_nnz", int(dev_csr.struct.nnz))
        object.__setattr__(self, "_host", None)
        _maybe_block3(dev_csr, self.n, self._nnz, use_block3)

    def _host_arrays(self):
        if self._host is None:
            h = next(iter(self._dev.values()))
            ro = h.ro.cpu().numpy().astype(np.int64)
            ci = h.ci.cpu().numpy()
            va = h.va.cpu().numpy()
            object.__setattr__(self, "_host", (ro, ci, va))
        return self._host

    @property
    def row_offsets(self):
        return self._host_arrays()[0]

    @property
    def col_indices(self):
        return self._host_arrays()[1]

    @property
    def values(self):
        return self._host_arrays()[2]

    @property
    def nnz(self):
        return self._nnz

    def release_device(self):
        self._host_arrays()
        self._dev.clear()


def spmv(A: SparseSpdMatrix, x):
    """Sparse matrix-vector product ``A @ x`` (``core.py:114-119``)."""
    if not is_device_tensor(x):
        x = np.asarray(x, dtype=np.float64)
    if tuple(x.shape) != (A.n,):
        raise ContractViolation(f"vector length {tuple(x.shape)} does not match n={A.n}")
    return A @ x


# ---------------------------------------------------------------------------
# tridiagonal (core.py:122-177)


@dataclass(frozen=True)
class TridiagSym:
    """Symmetric tridiagonal matrix stored as diagonal/off-diagonal arrays."""

    diag: np.ndarray
    offdiag: np.ndarray

    def __post_init__(self):
        d = np.asarray(self.diag, dtype=np.float64)
        e = np.asarray(self.offdiag, dtype=np.float64)
        object.__setattr__(self, "diag", d)
        object.__setattr__(self, "offdiag", e)
        if len(d) < 1 or len(e) != len(d) - 1:
            raise ContractViolation("need |offdiag| = |diag| - 1 with |diag| >= 1")

    @property
    def m(self):
        return len(self.diag)

    def truncated(self, m):
        if not 1 <= m <= self.m:
            raise ContractViolation("truncation size out of range")
        return TridiagSym(self.diag[:m].copy(), self.offdiag[:m - 1].copy())

    def to_dense(self):
        T = np.diag(self.diag)
        idx = np.arange(self.m - 1)
        T[idx, idx + 1] = self.offdiag
        T[idx + 1, idx] = self.offdiag
        return T


@dataclass(frozen=True)
class EigDecomposition:
    """Eigenvalues sorted descending with column-matched orthonormal vectors."""

    values: np.ndarray
    vectors: np.ndarray


def tridiag_eigvals_device(d, e):
    """Descending eigenvalues of (d, e) given as device tensors (Sturm bisection)."""
    torch = _torch()
    m = int(d.shape[0])
    out = torch.empty(m, dtype=torch.float64, device="cuda")
    ctx = _lib.context()
    ctx.check(ctx.lib.rcg_tridiag_eigvals(ctx.h, _lib.ptr(d), _lib.ptr(e), m, _lib.ptr(out)), "tridiag_eigvals")
    return out


def tridiag_eigvecs_device(d, e, values_desc, idx):
    """(m, k) device tensor whose column q is the eigenvector of values_desc[idx[q]]."""
    torch = _torch()
    m = int(d.shape[0])
    idx = torch.as_tensor(np.asarray(idx, dtype=np.int64)).to("cuda") if not is_device_tensor(idx) else idx
    k = int(idx.shape[0])
    Q = torch.empty((k, m), dtype=torch.float64, device="cuda")
    ctx = _lib.context()
    ctx.check(ctx.lib.rcg_tridiag_eigvecs(ctx.h, _lib.ptr(d), _lib.ptr(e), m, _lib.ptr(values_desc), _lib.ptr(idx),
                                          k, _lib.ptr(Q)), "tridiag_eigvecs")
    return Q.t()


def tridiag_eig(T: TridiagSym) -> EigDecomposition:
    """Full eigendecomposition, values descending (``core.py:169-177``):
    bisection for the values, inverse iteration for the vectors, on device."""
    if T.m == 1:
        return EigDecomposition(T.diag.copy(), np.ones((1, 1)))
    d, _ = to_dev(T.diag)
    e, _ = to_dev(T.offdiag)
    vals = tridiag_eigvals_device(d, e)
    Q = tridiag_eigvecs_device(d, e, vals, np.arange(T.m))
    return EigDecomposition(np.ascontiguousarray(vals.cpu().numpy()), np.ascontiguousarray(Q.cpu().numpy()))


def dense_sym_eig(G) -> EigDecomposition:
    """Dense symmetric eigendecomposition (``core.py:180-192``; a brute-force test
    oracle in the reference, outside the hot path) via cuSOLVER through torch."""
    torch = _torch()
    G = np.asarray(G, dtype=np.float64)
    if G.ndim != 2 or G.shape[0] != G.shape[1]:
        raise ContractViolation("input must be square")
    scale = np.linalg.norm(G)
    if scale > 0 and np.linalg.norm(G - G.T) > 1e-12 * scale:
        raise ContractViolation("input is not symmetric")
    w, v = torch.linalg.eigh(torch.from_numpy(0.5 * (G + G.T)).to("cuda"))
    w, v = w.cpu().numpy(), v.cpu().numpy()
    order = np.argsort(w)[::-1]
    return EigDecomposition(np.ascontiguousarray(w[order]), np.ascontiguousarray(v[:, order]))


def dense_cholesky(G, pivot_rtol=0.0):
    """Guarded lower Cholesky (``core.py:195-243``) on device: the first column
    whose pivot is <= pivot_rtol * (largest earlier pivot), <= 0 or non-finite
    raises RankDeficient(column)."""
    torch = _torch()
    host = not is_device_tensor(G)
    Gh = np.asarray(G, dtype=np.float64) if host else G.detach().cpu().numpy()
    n = Gh.shape[0]
    if Gh.ndim != 2 or Gh.shape != (n, n):
        raise ContractViolation("input must be square")
    scale = np.linalg.norm(Gh)
    if scale > 0 and np.linalg.norm(Gh - Gh.T) > 1e-12 * scale:
        raise ContractViolation("input is not symmetric")
    Gd = torch.from_numpy(np.ascontiguousarray(Gh.T)).to("cuda")  # column-major
    L = torch.empty((n, n), dtype=torch.float64, device="cuda")
    bad = _lib.C.c_int64(-1)
    ctx = _lib.context()
    rc = ctx.lib.rcg_dense_cholesky(ctx.h, _lib.ptr(Gd), n, float(pivot_rtol), _lib.ptr(L), None, _lib.C.byref(bad))
    if rc == _lib.RCG_ERR_RANK_DEFICIENT:
        raise RankDeficient(int(bad.value))
    ctx.check(rc, "dense_cholesky")
    Lh = L.t()
    return Lh.cpu().numpy() if host else Lh.contiguous()
