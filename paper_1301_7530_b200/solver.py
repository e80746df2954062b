"""Augmented preconditioned CG on the B200 — drop-in for
``/root/reference/pkg/src/recycg/solver.py``.

Same public names and semantics: ``Preconditioner`` (``solver.py:28-60``),
``DeflationOperator`` / ``build_deflation`` / ``project`` (``:63-122``),
``SolveConfig`` (``:125-139``), ``SolveTrace`` (``:142-190``) and
``apcg_solve`` (``:193-290``).  The whole iteration loop runs inside one C-ABI
call (``rcg_apcg_solve``): five fused kernels per iteration, device-side
convergence flag, histories (z_j, w_j, A w_j, r_j) kept in HBM.  The trace's
alpha/beta/(r,z)/||r|| lists are copied to the host (m doubles each); the
z/w/r histories stay on the device and are materialized per column only when
a caller indexes them.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import (ContractViolation, NumericalFailure, RankDeficient, SparseSpdMatrix,
                   colmajor_from_host, from_dev, is_device_tensor, pad_ld, to_dev)

IDENTITY = "identity"
JACOBI = "jacobi"
USER_DIAGONAL = "user_diagonal"

__all__ = ["Preconditioner", "DeflationOperator", "build_deflation", "project", "SolveConfig", "SolveTrace",
           "apcg_solve", "DeviceColumns"]


def _torch():
    return _lib.require_cuda()


# ---------------------------------------------------------------------------
# preconditioner (solver.py:28-60)


@dataclass(frozen=True, eq=False)
class Preconditioner:
    """Diagonal (or identity) SPD preconditioner, stored as inverse entries.
    ``inv_diag`` may be a host array or a device tensor; the device copy is
    cached."""

    kind: str
    inv_diag: object = None

    @classmethod
    def identity(cls):
        return cls(IDENTITY)

    @classmethod
    def jacobi(cls, A: SparseSpdMatrix):
        return cls(JACOBI, A.diagonal_device(inverse=True))

    @classmethod
    def user_diagonal(cls, diag):
        diag = np.asarray(diag, dtype=np.float64)
        if np.any(diag <= 0.0):
            raise ContractViolation("preconditioner diagonal must be positive")
        return cls(USER_DIAGONAL, 1.0 / diag)

    def device_inv_diag(self):
        if self.inv_diag is None:
            return None
        cache = self.__dict__.get("_dev_inv")
        if cache is None:
            cache, _ = to_dev(self.inv_diag)
            object.__setattr__(self, "_dev_inv", cache)
        return cache

    def apply(self, r):
        """M^{-1} r (``solver.py:50-54``), on the device."""
        torch = _torch()
        host = not is_device_tensor(r)
        x, _ = to_dev(r)
        y = torch.empty_like(x)
        ctx = _lib.context()
        inv = self.device_inv_diag()
        ctx.check(ctx.lib.rcg_diag_apply(ctx.h, x.shape[0], _lib.ptr(inv), _lib.ptr(x), _lib.ptr(y)), "diag_apply")
        return from_dev(y, host)

    def diag(self):
        """The diagonal of M itself (None for the identity kind)."""
        if self.inv_diag is None:
            return None
        inv = self.inv_diag.cpu().numpy() if is_device_tensor(self.inv_diag) else np.asarray(self.inv_diag)
        return 1.0 / inv


# ---------------------------------------------------------------------------
# deflation operator (solver.py:63-122)


class DeflationOperator:
    """P = I - C (C^T A C)^{-1} C^T A with device-resident C, AC, the Cholesky
    factor L of C^T A C and its inverse.  ``basis`` / ``ac`` /
    ``coarse_factor`` return host arrays (materialized on access)."""

    def __init__(self, n, Cd, ACd, Ld, Ginvd, ld):
        self._n = int(n)
        self._C = Cd        # (n_c, ld) device, column-major n x n_c
        self._AC = ACd
        self._L = Ld        # (n_c, n_c) device, column-major
        self._Ginv = Ginvd
        self._ld = ld
        n_c = 0 if Cd is None else int(Cd.shape[0])
        self._n_c = n_c
        self.struct = _lib.RcgDeflation(self._n, n_c, _ptrv(Cd), ld, _ptrv(ACd), ld, _ptrv(Ld), _ptrv(Ginvd))

    @property
    def n(self):
        return self._n

    @property
    def n_c(self):
        return self._n_c

    def _host_block(self, t):
        if self._n_c == 0:
            return np.zeros((self._n, 0))
        return t[:, :self._n].cpu().numpy().T.copy()

    @property
    def basis(self):
        return self._host_block(self._C)

    @property
    def ac(self):
        return self._host_block(self._AC)

    @property
    def coarse_factor(self):
        if self._n_c == 0:
            return np.zeros((0, 0))
        return self._L.cpu().numpy().T.copy()

    def coarse_solve(self, rhs):
        """(C^T A C)^{-1} rhs (``solver.py:79-82``)."""
        host = not is_device_tensor(rhs)
        r, _ = to_dev(rhs)
        out = self._Ginv.t() @ r if r.ndim == 1 else self._Ginv.t() @ r
        return from_dev(out, host)

    def project(self, x):
        """P x (``solver.py:84-91``), on the device."""
        torch = _torch()
        host = not is_device_tensor(x)
        xv, _ = to_dev(x)
        if tuple(xv.shape) != (self._n,):
            raise ContractViolation("vector length mismatch in project")
        out = torch.empty_like(xv)
        ctx = _lib.context()
        ctx.check(ctx.lib.rcg_project(ctx.h, _lib.C.byref(self.struct), _lib.ptr(xv), _lib.ptr(out)), "project")
        return from_dev(out, host)

    def initial_guess(self, b):
        """x0 = C (C^T A C)^{-1} C^T b (``solver.py:93-97``)."""
        torch = _torch()
        host = not is_device_tensor(b)
        bv, _ = to_dev(b)
        out = torch.empty(self._n, dtype=torch.float64, device="cuda")
        ctx = _lib.context()
        ctx.check(ctx.lib.rcg_initial_guess(ctx.h, _lib.C.byref(self.struct), _lib.ptr(bv), _lib.ptr(out)),
                  "initial_guess")
        return from_dev(out, host)


def _ptrv(t):
    return None if t is None else t.data_ptr()


def _basis_to_device(C, n, n_ext=None):
    """Accept a host (n, n_c) array, a device (n_c, ld) column-major block
    (``DeviceBlock``) or a torch (n, n_c) tensor; return (Cd (n_c, ld), ld).
    ``n_ext`` (sharded runs) reserves room for the ghost entries."""
    torch = _torch()
    n_ext = n if n_ext is None else n_ext
    if isinstance(C, DeviceBlock):
        return C.cols, C.ld
    if is_device_tensor(C):
        if C.ndim != 2 or C.shape[0] != n:
            raise ContractViolation("augmentation basis must be n x n_c with n_c <= n")
        ld = pad_ld(n_ext)
        out = torch.zeros((C.shape[1], ld), dtype=torch.float64, device="cuda")
        out[:, :n] = C.t().to(torch.float64)
        return out, ld
    Ch = np.asarray(C, dtype=np.float64)
    if Ch.size == 0:
        Ch = Ch.reshape(n, 0)
    if Ch.ndim != 2 or Ch.shape[0] != n or (Ch.shape[1] > n and n_ext == n):
        raise ContractViolation("augmentation basis must be n x n_c with n_c <= n")
    ld = pad_ld(n_ext)
    return colmajor_from_host(Ch, ld), ld


class DeviceBlock:
    """A column-major n x k block already on the device: ``cols`` is (k, ld)."""

    def __init__(self, cols, n, ld):
        self.cols, self.n, self.ld = cols, int(n), int(ld)

    @property
    def shape(self):
        return (self.n, int(self.cols.shape[0]))


def build_deflation(A: SparseSpdMatrix, C) -> DeflationOperator:
    """AC, sym(C^T A C) and its guarded Cholesky (pivot_rtol 1e-12) on device
    (``solver.py:100-117``).  Raises RankDeficient(column)."""
    torch = _torch()
    sharded = hasattr(A, "plan")
    if isinstance(C, DeviceBlock):
        if C.n != A.n or (C.shape[1] > A.n and not sharded):
            raise ContractViolation("augmentation basis must be n x n_c with n_c <= n")
        if sharded and C.ld < A.n_ext:
            raise ContractViolation("sharded basis needs room for the ghost entries (ld >= n_ext)")
        Cd, ld = C.cols, C.ld
    else:
        Cd, ld = _basis_to_device(C, A.n, getattr(A, "n_ext", A.n))
    n_c = int(Cd.shape[0])
    if n_c == 0:
        return DeflationOperator(A.n, None, None, None, None, ld)
    AC = torch.zeros((n_c, ld), dtype=torch.float64, device="cuda")
    L = torch.empty((n_c, n_c), dtype=torch.float64, device="cuda")
    Ginv = torch.empty((n_c, n_c), dtype=torch.float64, device="cuda")
    bad = _lib.C.c_int64(-1)
    ctx = _lib.context()
    h = A.device_csr()
    if sharded:
        rc = ctx.lib.rcg_deflation_build_sharded(ctx.h, _lib.C.byref(h.struct), _lib.ptr(Cd), ld, n_c, _lib.ptr(AC),
                                                 ld, _lib.ptr(L), _lib.ptr(Ginv), _lib.C.byref(A.halo_struct()),
                                                 _lib.C.byref(bad))
    else:
        rc = ctx.lib.rcg_deflation_build(ctx.h, _lib.C.byref(h.struct), _lib.ptr(Cd), ld, n_c, _lib.ptr(AC), ld,
                                         _lib.ptr(L), _lib.ptr(Ginv), _lib.C.byref(bad))
    if rc == _lib.RCG_ERR_RANK_DEFICIENT:
        raise RankDeficient(int(bad.value))
    ctx.check(rc, "deflation_build")
    return DeflationOperator(A.n, Cd, AC, L, Ginv, ld)


def project(D: DeflationOperator, x):
    """Apply the deflation projector P to a vector (``solver.py:120-122``)."""
    return D.project(x)


# ---------------------------------------------------------------------------
# config / trace


@dataclass
class SolveConfig:
    """Tolerance/iteration settings and trace-capture switches for one solve."""

    tol: float = 1e-6
    max_iters: int = 1000
    reorthogonalize: bool = True
    trace_capture: bool = True
    store_directions: bool = False
    # extension (not in the reference): keep only z_0..z_{cap-1}; Ritz
    # extraction then uses the leading cap x cap Lanczos block
    krylov_cap: int | None = None

    def __post_init__(self):
        if not 0.0 < self.tol < 1.0:
            raise ContractViolation("tol must be in (0, 1)")
        if self.max_iters < 1:
            raise ContractViolation("max_iters must be >= 1")
        if self.krylov_cap is not None and self.krylov_cap < 1:
            raise ContractViolation("krylov_cap must be >= 1")


class _TraceOwner:
    """Frees the library-owned device histories of one solve."""

    def __init__(self, handle, view):
        self.handle = handle
        self.view = view
        self.lib = _lib.load()

    def __del__(self):
        try:
            if self.handle:
                self.lib.rcg_trace_free(self.handle)
                self.handle = None
        except Exception:
            pass


class DeviceColumns:
    """List-like view of a device history (column j = one n-vector).  Indexing
    returns a host numpy copy (the reference stores numpy arrays); ``device()``
    returns the (count, ld) device tensor without copying."""

    def __init__(self, tensor=None, n=0, count=0):
        self._t = tensor
        self._n = n
        self._count = count
        self._host = None  # list when mutated from the host side

    def device(self):
        if self._host is not None:
            return None
        return self._t[:self._count] if self._t is not None else None

    def _materialize(self):
        if self._host is None:
            if self._t is None or self._count == 0:
                self._host = []
            else:
                block = self._t[:self._count, :self._n].cpu().numpy()
                self._host = [block[j].copy() for j in range(self._count)]
            self._t = None
        return self._host

    def __len__(self):
        return len(self._host) if self._host is not None else self._count

    def __getitem__(self, j):
        if self._host is not None:
            return self._host[j]
        if isinstance(j, slice):
            return [self[i] for i in range(*j.indices(self._count))]
        if j < 0:
            j += self._count
        if not 0 <= j < self._count:
            raise IndexError(j)
        return self._t[j, :self._n].cpu().numpy()

    def __iter__(self):
        for j in range(len(self)):
            yield self[j]

    def __bool__(self):
        return len(self) > 0

    def clear(self):
        self._host = []
        self._t = None
        self._count = 0

    def append(self, v):
        self._materialize().append(v)

    def extend(self, vs):
        self._materialize().extend(vs)


@dataclass
class SolveTrace:
    """Per-iteration record of one APCG run (``solver.py:142-190``)."""

    alphas: list = field(default_factory=list)
    betas: list = field(default_factory=list)
    rz_inner: list = field(default_factory=list)
    residual_norms: list = field(default_factory=list)
    z_history: object = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    w_history: object = field(default_factory=list)
    r_history: object = field(default_factory=list)
    projection_seconds: float = 0.0

    # device-side handles (not part of the reference dataclass contract)
    _owner: object = field(default=None, repr=False, compare=False)
    device_seconds: float = field(default=0.0, repr=False, compare=False)
    krylov_cap: object = field(default=None, repr=False, compare=False)
    b_norm: float = field(default=0.0, repr=False, compare=False)

    def to_json_dict(self, spectrum=None, eps_cg=None):
        d = {
            "alphas": list(map(float, self.alphas)),
            "betas": list(map(float, self.betas)),
            "rz_inner": list(map(float, self.rz_inner)),
            "residual_norms": list(map(float, self.residual_norms)),
            "z_history": [list(map(float, z)) for z in self.z_history],
            "iterations": self.iterations,
            "converged": self.converged,
        }
        if spectrum is not None:
            d["spectrum"] = list(map(float, spectrum))
        if eps_cg is not None:
            d["eps_cg"] = float(eps_cg)
        return d

    @classmethod
    def from_json_dict(cls, d):
        return cls(
            alphas=list(d.get("alphas", [])),
            betas=list(d.get("betas", [])),
            rz_inner=list(d.get("rz_inner", [])),
            residual_norms=list(d.get("residual_norms", [])),
            z_history=[np.asarray(z, dtype=np.float64) for z in d.get("z_history", [])],
            iterations=int(d.get("iterations", len(d.get("alphas", [])))),
            converged=bool(d.get("converged", False)),
        )

    def extraction_length(self):
        """m used for Ritz extraction: the full m, or the leading block kept
        under the krylov_cap extension (exact Lanczos on H_cap)."""
        if self.krylov_cap and len(self.z_history) < self.iterations:
            return len(self.z_history)
        return self.iterations

    # -- device access used by the Ritz path -----------------------------
    def device_coefficients(self):
        """(alphas, betas, rz) as device tensors of length >= m."""
        torch = _torch()
        m = self.extraction_length()
        v = self._owner.view if self._owner is not None else None
        if v is not None and len(self.alphas) >= m:
            def wrap(p, count):
                arr = _lib.CudaArray(self._owner, p, (max(count, 1),), (1,))
                return torch.as_tensor(arr, device="cuda")
            return wrap(v.alphas, m), wrap(v.betas, max(m, 1)), wrap(v.rz_inner, m)
        a = torch.tensor(np.asarray(self.alphas[:m], dtype=np.float64), device="cuda")
        b = torch.tensor(np.asarray(list(self.betas[:max(m - 1, 0)]) + [0.0], dtype=np.float64), device="cuda")
        rz = torch.tensor(np.asarray(self.rz_inner[:m], dtype=np.float64), device="cuda")
        return a, b, rz

    def device_z(self):
        """(m, ld) device tensor of z_0..z_{m-1} and its ld, uploading a host
        z_history (e.g. a trace read from JSON) when needed."""
        torch = _torch()
        m = self.extraction_length()
        zh = self.z_history
        if isinstance(zh, DeviceColumns) and zh.device() is not None and len(zh) >= m:
            t = zh.device()
            return t[:m], int(t.shape[1]), zh._n
        n = len(zh[0])
        ld = pad_ld(n)
        out = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
        out[:, :n] = torch.from_numpy(np.stack([np.asarray(zh[j], dtype=np.float64) for j in range(m)])).to("cuda")
        return out, ld, n


def _history(owner, p, ld, count, n, cap_cols=None):
    torch = _torch()
    if not p or count == 0:
        return DeviceColumns(None, n, 0)
    rows = count if cap_cols is None else cap_cols
    arr = _lib.CudaArray(owner, p, (rows, ld), (ld, 1))
    return DeviceColumns(torch.as_tensor(arr, device="cuda"), n, count)


def apcg_solve(A: SparseSpdMatrix, M: Preconditioner, D: DeflationOperator, b, cfg: SolveConfig):
    """Augmented preconditioned conjugate gradient (``solver.py:193-290``).

    Returns ``(x, trace)``; ``x`` is a host array when ``b`` is a host array
    and a device tensor when ``b`` is a device tensor.  Convergence is
    ``||r_j|| <= tol * ||P^T b||``; NumericalFailure is raised exactly where the
    reference raises it.
    """
    torch = _torch()
    host = not is_device_tensor(b)
    bv, _ = to_dev(b)
    if tuple(bv.shape) != (A.n,):
        raise ContractViolation("right-hand side length mismatch")
    if D.n != A.n:
        raise ContractViolation("deflation operator dimension mismatch")
    x = torch.empty(A.n, dtype=torch.float64, device="cuda")
    ctx = _lib.context()
    h = A.device_csr()
    inv = M.device_inv_diag() if M is not None else None
    scfg = _lib.RcgSolveCfg(float(cfg.tol), int(cfg.max_iters), int(bool(cfg.reorthogonalize)),
                            int(bool(cfg.trace_capture)), int(bool(cfg.store_directions)), 0,
                            int(getattr(cfg, "krylov_cap", None) or 0))
    th = _lib.C.c_void_p()
    t0 = time.perf_counter()
    if hasattr(A, "plan"):
        rc = ctx.lib.rcg_apcg_solve_sharded(ctx.h, _lib.C.byref(h.struct), _lib.ptr(inv), _lib.C.byref(D.struct),
                                            _lib.ptr(bv), _lib.ptr(x), _lib.C.byref(scfg),
                                            _lib.C.byref(A.halo_struct()), _lib.C.byref(th))
    else:
        rc = ctx.lib.rcg_apcg_solve(ctx.h, _lib.C.byref(h.struct), _lib.ptr(inv), _lib.C.byref(D.struct),
                                    _lib.ptr(bv), _lib.ptr(x), _lib.C.byref(scfg), _lib.C.byref(th))
    if not th.value:
        ctx.check(rc, "apcg_solve")
        raise RuntimeError("apcg_solve returned no trace")
    view = _lib.RcgTraceView()
    ctx.lib.rcg_trace_get_view(th, _lib.C.byref(view))
    owner = _TraceOwner(th, view)
    m = int(view.iterations)
    nb = int(view.n_betas)
    # small coefficient arrays to the host (one packed copy)
    trace = SolveTrace()
    trace._owner = owner
    trace.iterations = m
    trace.converged = bool(view.converged)
    trace.device_seconds = float(view.device_seconds)
    trace.b_norm = float(view.b_norm)
    if m > 0:
        def dvec(p, count):
            arr = _lib.CudaArray(owner, p, (count,), (1,))
            return torch.as_tensor(arr, device="cuda")
        packed = torch.cat([dvec(view.alphas, m), dvec(view.betas, max(nb, 1))[:nb], dvec(view.rz_inner, m),
                            dvec(view.residual_norms, m + 1)]).cpu().numpy()
        trace.alphas = packed[:m].tolist()
        trace.betas = packed[m:m + nb].tolist()
        trace.rz_inner = packed[m + nb:2 * m + nb].tolist()
        trace.residual_norms = packed[2 * m + nb:].tolist()
    else:
        trace.residual_norms = [float(view.r0_norm)]
    ld = int(view.ld)
    cap = getattr(cfg, "krylov_cap", None)
    if cfg.trace_capture:
        mz = min(m, cap) if cap else m
        trace.z_history = _history(owner, view.Z, ld, mz, A.n, cap_cols=mz + 1)
        trace.krylov_cap = cap
    if cfg.store_directions:
        trace.w_history = _history(owner, view.W, ld, m, A.n, cap_cols=m + 1)
        trace.r_history = _history(owner, view.R, ld, m, A.n, cap_cols=m + 1)
    trace.projection_seconds = 0.0
    trace.sharded = hasattr(A, "plan")
    if rc == _lib.RCG_ERR_NUMERICAL:
        ctx.check(rc, "apcg_solve")
    ctx.check(rc, "apcg_solve")
    trace.solve_wall_seconds = time.perf_counter() - t0
    return from_dev(x, host), trace
