"""Reference-side binding: run the reference package's own driver and tests
on the B200 numerics by rebinding its module-level seams.

The reference (``recycg``) has no plugin layer; ``run_sequence``
(``recycle.py:178-238``) resolves ``build_deflation`` (``:117, :124``),
``apcg_solve`` (``:204``), ``select_spectrum`` (``:218``) and the basis
updates at call time from its module globals.  ``install``
rebinds those names - and the same names in the reference's ``solver``,
``ritz``, ``core`` and package namespaces, so code that imported them from
``recycg`` directly also takes the device path - to adapters that:

* convert reference objects at the boundary (``SparseSpdMatrix`` -> a cached
  device CSR, ``Preconditioner``, ``SolveConfig``, hand-built ``SolveTrace`` /
  ``TridiagSym`` / ``LanczosView`` / ``RitzSpectrum``);
* keep the reference's host-array contract (host ``b`` -> host ``x``; the
  reference's numpy ``AugmentationState`` receives (n, k) host blocks formed
  on the device, only the selected columns crossing PCIe);
* re-raise errors as the reference's own exception types
  (``ContractViolation``, ``RankDeficient(column)``, ``NumericalFailure``), so
  ``guarded_deflation`` and the tests' ``pytest.raises`` see what they expect.

``install`` returns a handle whose ``calls`` counts adapter calls by name and
whose ``uninstall()`` restores the original bindings.
"""
from __future__ import annotations

import functools
import importlib
from collections import Counter

import numpy as np

from . import core as _core
from . import recycle as _recycle
from . import ritz as _ritz
from . import solver as _solver
from .core_errors import ContractViolation, NumericalFailure, RankDeficient

# the seams and the modules of the reference that bind them
SEAMS = ("build_deflation", "apcg_solve", "project", "select_spectrum", "lanczos_tridiag", "lanczos_from_trace",
         "ritz_pairs", "select_converged", "cluster_filter", "tridiag_eig", "update_basis_srks",
         "update_basis_trks")
_MODULES = ("", ".core", ".solver", ".ritz", ".recycle")


class Bridge:
    def __init__(self, ref):
        self.ref = ref                       # the reference package (module ``recycg``)
        self.calls = Counter()
        self._saved = []

    # -- conversions (reference -> B200) ----------------------------------
    def matrix(self, A):
        if isinstance(A, _core.SparseSpdMatrix):
            return A
        cache = A.__dict__.get("_b200")
        if cache is None:
            cache = _core.SparseSpdMatrix(A.n, A.row_offsets, A.col_indices, A.values, validate=False)
            object.__setattr__(A, "_b200", cache)       # frozen dataclass: cached beside its fields
        return cache

    @staticmethod
    def precond(M):
        if isinstance(M, _solver.Preconditioner) or M is None:
            return M
        return _solver.Preconditioner(M.kind, M.inv_diag)

    @staticmethod
    def config(cfg):
        if isinstance(cfg, _solver.SolveConfig):
            return cfg
        return _solver.SolveConfig(tol=cfg.tol, max_iters=cfg.max_iters, reorthogonalize=cfg.reorthogonalize,
                                   trace_capture=cfg.trace_capture, store_directions=cfg.store_directions)

    @staticmethod
    def trace(tr):
        if isinstance(tr, _solver.SolveTrace):
            return tr
        return _solver.SolveTrace(alphas=list(tr.alphas), betas=list(tr.betas), rz_inner=list(tr.rz_inner),
                                  residual_norms=list(tr.residual_norms), z_history=list(tr.z_history),
                                  iterations=tr.iterations, converged=tr.converged,
                                  w_history=list(getattr(tr, "w_history", [])),
                                  r_history=list(getattr(tr, "r_history", [])),
                                  projection_seconds=getattr(tr, "projection_seconds", 0.0))

    @staticmethod
    def tridiag(T):
        if isinstance(T, _core.TridiagSym):
            return T
        return _core.TridiagSym(np.asarray(T.diag, dtype=np.float64), np.asarray(T.offdiag, dtype=np.float64))

    def view(self, v):
        if isinstance(v, _ritz.LanczosView):
            return v
        return _ritz.LanczosView(self.tridiag(v.tridiag), np.asarray(v.basis))

    @staticmethod
    def spectrum(s):
        if isinstance(s, _ritz.RitzSpectrum):
            return s
        return _ritz.RitzSpectrum(s.values, s.vectors, s.converged_mask, getattr(s, "epsilon", None))

    # -- exception mapping (B200 -> reference) ------------------------------
    def _reraise(self, exc):
        R = self.ref
        if isinstance(exc, RankDeficient):
            raise R.RankDeficient(exc.column) from exc
        if isinstance(exc, NumericalFailure):
            raise R.NumericalFailure(str(exc)) from exc
        if isinstance(exc, ContractViolation):
            raise R.ContractViolation(str(exc)) from exc
        raise exc

    def _adapter(self, name, fn):
        @functools.wraps(fn)
        def wrapped(*args, **kwargs):
            self.calls[name] += 1
            try:
                return fn(*args, **kwargs)
            except (RankDeficient, NumericalFailure, ContractViolation) as exc:
                self._reraise(exc)
        return wrapped

    # -- the adapters --------------------------------------------------------
    def adapters(self):
        B = self

        def build_deflation(A, C):
            return _solver.build_deflation(B.matrix(A), C)

        def apcg_solve(A, M, D, b, cfg):
            if not isinstance(D, _solver.DeflationOperator):
                D = _solver.build_deflation(B.matrix(A), np.asarray(D.basis))
            return _solver.apcg_solve(B.matrix(A), B.precond(M), D, b, B.config(cfg))

        def project(D, x):
            return _solver.project(D, x)

        def select_spectrum(trace, strategy):
            return _recycle.select_spectrum(B.trace(trace), strategy)

        def lanczos_tridiag(alphas, betas):
            return _ritz.lanczos_tridiag(alphas, betas)

        def lanczos_from_trace(trace):
            return _ritz.lanczos_from_trace(B.trace(trace))

        def ritz_pairs(view):
            return _ritz.ritz_pairs(B.view(view))

        def select_converged(current, previous_values, epsilon):
            return _ritz.select_converged(B.spectrum(current), previous_values, epsilon)

        def cluster_filter(values, min_cluster):
            return _ritz.cluster_filter(values, min_cluster)

        def tridiag_eig(T):
            return _core.tridiag_eig(B.tridiag(T))

        def update_basis_srks(state, spectrum, system_index=0):
            return _recycle.update_basis_srks(state, B.spectrum(spectrum), system_index)

        def update_basis_trks(state, trace, system_index=0):
            return _recycle.update_basis_trks(state, B.trace(trace), system_index)

        fns = dict(locals())
        return {name: self._adapter(name, fns[name]) for name in SEAMS}

    # -- (un)binding ---------------------------------------------------------
    def install(self):
        ad = self.adapters()
        base = self.ref.__name__
        for suffix in _MODULES:
            mod = importlib.import_module(base + suffix)
            for name, fn in ad.items():
                if hasattr(mod, name):
                    self._saved.append((mod, name, getattr(mod, name)))
                    setattr(mod, name, fn)
        return self

    def uninstall(self):
        for mod, name, fn in reversed(self._saved):
            setattr(mod, name, fn)
        self._saved.clear()


def install(ref=None):
    """Rebind the reference package's seams to the B200 path.  ``ref`` is the
    imported reference package (default: ``import recycg``)."""
    if ref is None:
        ref = importlib.import_module("recycg")
    return Bridge(ref).install()
