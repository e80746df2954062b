"""Spectral post-processing of APCG traces on the B200 — drop-in for
``/root/reference/pkg/src/recycg/ritz.py:1-183`` (Lanczos recovery, Ritz
pairs, stagnation selection, cluster filter).

The Lanczos basis V = [(-1)^j z_j / sqrt(r_j, z_j)] is never formed: the z
history stays on the device and Ritz vectors are produced as Z @ Qtilde for
the requested columns only (``rcg_ritz_vectors``).  ``LanczosView.basis`` and
``RitzSpectrum.vectors`` materialize host arrays lazily for callers that read
them (tests, diagnostics).
"""
from __future__ import annotations

import math

import numpy as np

from . import _lib
from .core import (ContractViolation, NumericalFailure, TridiagSym, from_dev, is_device_tensor, to_dev,
                   tridiag_eigvals_device)
from .solver import SolveTrace

DEGENERATE_GAP = 1e-12

__all__ = ["LanczosView", "RitzSpectrum", "lanczos_tridiag", "lanczos_from_trace", "ritz_pairs",
           "select_converged", "cluster_filter", "DEGENERATE_GAP"]


def _torch():
    return _lib.require_cuda()


class LanczosView:
    """Lanczos tridiagonal and basis recovered from a CG trace
    (``ritz.py:26-35``).  Built from a trace, the basis stays implicit on the
    device; ``basis`` materializes it on the host when read."""

    def __init__(self, tridiag: TridiagSym, basis=None, _trace=None):
        self.tridiag = tridiag
        self._basis = basis
        self._trace = _trace

    @property
    def m(self):
        return self.tridiag.m

    @property
    def basis(self):
        if self._basis is None and self._trace is not None:
            torch = _torch()
            Z, ld, n = self._trace.device_z()
            _, _, rz = self._trace.device_coefficients()
            m = self.m
            signs = torch.ones(m, dtype=torch.float64, device="cuda")
            signs[1::2] = -1.0
            scales = signs / torch.sqrt(rz[:m])
            V = (Z[:m, :n] * scales[:, None]).t()
            self._basis = V.cpu().numpy()
        return self._basis


class RitzSpectrum:
    """Ritz values (descending) with vectors and per-value convergence flags
    (``ritz.py:38-49``).  ``vectors`` may be computed lazily on the device."""

    def __init__(self, values, vectors=None, converged_mask=None, epsilon=None, _source=None):
        self.values = np.asarray(values, dtype=np.float64)
        self._vectors = vectors
        self.converged_mask = None if converged_mask is None else np.asarray(converged_mask, dtype=bool)
        self.epsilon = epsilon
        self._source = _source  # (trace, device values) for device-side vector formation

    @property
    def m(self):
        return len(self.values)

    @property
    def vectors(self):
        if self._vectors is None and self._source is not None:
            Y = ritz_vectors_device(self._source[0], self._source[1], np.arange(self.m), scale_by_theta=False)
            self._vectors = Y.cpu().numpy().T.copy()
        return self._vectors

    def replace(self, **kw):
        out = RitzSpectrum(self.values, self._vectors, self.converged_mask, self.epsilon, self._source)
        for k, v in kw.items():
            setattr(out, k if k != "vectors" else "_vectors", v)
        return out


def lanczos_tridiag(alphas, betas) -> TridiagSym:
    """d_0 = 1/a_0, d_j = 1/a_j + b_{j-1}/a_{j-1}, e_j = sqrt(b_j)/a_j
    (``ritz.py:61-78``), computed on the device."""
    torch = _torch()
    a = np.asarray(alphas, dtype=np.float64)
    b = np.asarray(betas, dtype=np.float64)
    m = len(a)
    if m < 1:
        raise ContractViolation("need at least one iteration")
    if len(b) != m - 1:
        raise ContractViolation("need exactly m - 1 beta coefficients")
    ad, _ = to_dev(a)
    bd, _ = to_dev(np.concatenate([b, [0.0]]))
    d = torch.empty(m, dtype=torch.float64, device="cuda")
    e = torch.empty(max(m - 1, 1), dtype=torch.float64, device="cuda")
    ctx = _lib.context()
    ctx.check(ctx.lib.rcg_lanczos_tridiag(ctx.h, _lib.ptr(ad), _lib.ptr(bd), m, _lib.ptr(d), _lib.ptr(e)),
              "lanczos_tridiag")
    return TridiagSym(d.cpu().numpy(), e[:m - 1].cpu().numpy())


def lanczos_from_trace(trace: SolveTrace) -> LanczosView:
    """Recover the Lanczos view of a solve from its captured trace
    (``ritz.py:81-94``)."""
    if trace.iterations < 1:
        raise ContractViolation("trace has no iterations")
    if len(trace.z_history) < trace.iterations:
        raise ContractViolation("trace was captured without z_history")
    m = trace.iterations
    T = lanczos_tridiag(trace.alphas[:m], trace.betas[:m - 1])
    return LanczosView(T, None, _trace=trace)


def ritz_vectors_device(trace, values_desc_dev, idx, scale_by_theta):
    """(k, ld) device block: y_i = V q_{idx_i} (/ sqrt|theta_i|) — the skinny
    Z @ Qtilde GEMM over the device z history (``rcg_ritz_vectors``)."""
    torch = _torch()
    m = trace.extraction_length()
    Z, ld, n = trace.device_z()
    a, b, rz = trace.device_coefficients()
    idx_d = torch.as_tensor(np.asarray(idx, dtype=np.int64)).to("cuda")
    k = int(idx_d.shape[0])
    Y = torch.zeros((k, ld), dtype=torch.float64, device="cuda")
    ctx = _lib.context()
    ctx.check(ctx.lib.rcg_ritz_vectors(ctx.h, _lib.ptr(a), _lib.ptr(b), _lib.ptr(rz), m, _lib.ptr(Z), ld, n,
                                       _lib.ptr(values_desc_dev), _lib.ptr(idx_d), k, 1 if scale_by_theta else 0,
                                       _lib.ptr(Y), ld), "ritz_vectors")
    return Y[:, :n] if Y.shape[1] != n else Y


def ritz_pairs(view: LanczosView) -> RitzSpectrum:
    """Ritz values (descending) and vectors Y = V Q (``ritz.py:97-100``)."""
    torch = _torch()
    d, _ = to_dev(view.tridiag.diag)
    e, _ = to_dev(view.tridiag.offdiag if view.m > 1 else np.zeros(1))
    vals = tridiag_eigvals_device(d, e) if view.m > 1 else d.clone()
    if view._trace is not None:
        return RitzSpectrum(vals.cpu().numpy(), None, None, None, _source=(view._trace, vals))
    from .core import tridiag_eig
    eig = tridiag_eig(view.tridiag)
    return RitzSpectrum(eig.values, np.asarray(view.basis) @ eig.vectors)


def select_converged(current: RitzSpectrum, previous_values, epsilon) -> RitzSpectrum:
    """Flag Ritz values that stagnated between steps m-1 and m
    (``ritz.py:103-138``), evaluated on the device."""
    torch = _torch()
    if epsilon <= 0.0:
        raise ContractViolation("epsilon must be positive")
    cur = np.asarray(current.values, dtype=np.float64)
    prev = np.asarray(previous_values, dtype=np.float64)
    m = len(cur)
    if m >= 2 and len(prev) != m - 1:
        raise ContractViolation("previous spectrum must have m - 1 values")
    cd, _ = to_dev(cur)
    pd, _ = to_dev(prev if len(prev) else np.zeros(1))
    mask = torch.zeros(max(m, 1), dtype=torch.uint8, device="cuda")
    ctx = _lib.context()
    ctx.check(ctx.lib.rcg_select_converged(ctx.h, _lib.ptr(cd), _lib.ptr(pd), m, float(epsilon), _lib.ptr(mask)),
              "select_converged")
    out = current.replace(converged_mask=mask[:m].cpu().numpy().astype(bool), epsilon=float(epsilon))
    return out


def cluster_filter(values, min_cluster):
    """Indices of values outside the central dense cluster (drop-in for
    ``ritz.py:141-183``).

    The split search runs on the device (``rcg_cluster_filter``): one thread
    per candidate cluster [a, b], scored with the reference's own arithmetic
    and tie order, then a fixed-order argmin.  ``values`` may be a host array
    or a CUDA tensor (descending Ritz values).
    """
    m = len(values)
    if min_cluster < 1:
        raise ContractViolation("min_cluster must be >= 1")
    if m < min_cluster or m < 2:
        return list(range(m))
    vd, _ = to_dev(values)
    rng = (_lib.C.c_int64 * 2)()
    ctx = _lib.context()
    ctx.check(ctx.lib.rcg_cluster_filter(ctx.h, _lib.ptr(vd), m, int(min_cluster), rng), "cluster_filter")
    lo, hi = int(rng[0]), int(rng[1])
    return list(range(lo)) + list(range(hi + 1, m))
