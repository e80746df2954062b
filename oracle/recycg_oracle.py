"""CPU oracle for the augmented-PCG + Ritz-recycling hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module, and only as the checker / the timed CPU reference arm.  The product
package ``paper_1301_7530_b200`` never imports it.

This is a plain numpy/scipy restatement of the reference algorithm
(``/root/reference/pkg/src/recycg``); every function cites the file:line it
follows.  The third-party numerics the reference calls (scipy ``csr_matvec``,
``scipy.linalg.eigh_tridiagonal`` -> LAPACK ``dstevd``, ``cholesky`` ->
``dpotrf``, ``solve_triangular`` -> ``dtrtrs``, OpenBLAS ``dgemv``) are called
here the same way (scipy 1.18.1 / numpy 2.3.5 in this image; the reference pins
none of them, ``pkg/pyproject.toml:10-14``).

Parity pinning: ``tests/test_oracle_golden.py`` checks this
module against (a) the reference's frozen golden fixture
``pkg/tests/fixtures/benchmark_pilot.json`` (none/trks iteration lists, copied
into ``tests/golden/benchmark_pilot_none_trks.json``) and (b) vectors generated
by importing the reference in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``).

Inputs are plain host CSR triples: any object with ``n``, ``row_offsets``,
``col_indices``, ``values`` attributes.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg
import scipy.sparse

DEGENERATE_GAP = 1e-12          # ritz.py:23
RANK_GUARD_RTOL = 1e-12         # recycle.py:30, solver.py:116


class OracleRankDeficient(Exception):
    def __init__(self, column):
        super().__init__(f"non-positive pivot at column {column}")
        self.column = column


class OracleNumericalFailure(Exception):
    pass


# ---------------------------------------------------------------------------
# core.py


def csr(A):
    """scipy CSR view of a host CSR triple (core.py:60, :110-111)."""
    return scipy.sparse.csr_matrix(
        (np.asarray(A.values, dtype=np.float64),
         np.asarray(A.col_indices), np.asarray(A.row_offsets)), shape=(A.n, A.n))


def spmv(A, x):
    """y = A x through scipy's csr_matvec (core.py:114-119)."""
    return csr(A) @ np.asarray(x, dtype=np.float64)


def diagonal(A):
    return csr(A).diagonal()                               # core.py:103-104


def dense_cholesky(G, pivot_rtol=0.0):
    """Guarded lower Cholesky (core.py:195-243): first column j whose pivot
    d_j <= pivot_rtol * max(d_0..d_{j-1}), d_j <= 0 or non-finite raises."""
    G = np.asarray(G, dtype=np.float64)
    n = G.shape[0]
    if n > 32:                                             # core.py:219-232
        try:
            L = scipy.linalg.cholesky(G, lower=True, check_finite=False)
        except (scipy.linalg.LinAlgError, ValueError):
            L = None
        if L is not None:
            d = np.diag(L) ** 2
            prev = np.concatenate(([0.0], np.maximum.accumulate(d)[:-1]))
            bad = ~np.isfinite(d) | (d <= prev * pivot_rtol) | (d <= 0.0)
            if not bad.any():
                return L
            raise OracleRankDeficient(int(np.argmax(bad)))
    L = np.zeros_like(G)                                   # core.py:233-243
    top = 0.0
    for j in range(n):
        d = G[j, j] - L[j, :j] @ L[j, :j]
        if d <= top * pivot_rtol or d <= 0.0 or not np.isfinite(d):
            raise OracleRankDeficient(j)
        top = max(top, d)
        L[j, j] = math.sqrt(d)
        if j + 1 < n:
            L[j + 1:, j] = (G[j + 1:, j] - L[j + 1:, :j] @ L[j, :j]) / L[j, j]
    return L


def tridiag_eig(diag, off):
    """All eigenpairs, values descending (core.py:163-177)."""
    diag = np.asarray(diag, dtype=np.float64)
    off = np.asarray(off, dtype=np.float64)
    if len(diag) == 1:
        return diag.copy(), np.ones((1, 1))
    w, v = scipy.linalg.eigh_tridiagonal(diag, off)
    order = np.argsort(w)[::-1]
    return np.ascontiguousarray(w[order]), np.ascontiguousarray(v[:, order])


def tridiag_eigvals(diag, off):
    return tridiag_eig(diag, off)[0]


# ---------------------------------------------------------------------------
# solver.py


class Deflation:
    """C, AC, L of the projector P = I - C (C^T A C)^{-1} C^T A (solver.py:63-97)."""

    def __init__(self, C, AC, L):
        self.C, self.AC, self.L = C, AC, L

    @property
    def n_c(self):
        return self.C.shape[1]

    def coarse_solve(self, rhs):                           # solver.py:79-82
        y = scipy.linalg.solve_triangular(self.L, rhs, lower=True)
        return scipy.linalg.solve_triangular(self.L.T, y, lower=False)

    def project(self, x):                                  # solver.py:84-91
        if self.n_c == 0:
            return x.copy()
        return x - self.C @ self.coarse_solve(self.AC.T @ x)

    def initial_guess(self, b):                            # solver.py:93-97
        if self.n_c == 0:
            return np.zeros(self.C.shape[0])
        return self.C @ self.coarse_solve(self.C.T @ b)


def build_deflation(A, C):
    """AC, symmetrized C^T A C, guarded Cholesky (solver.py:100-117)."""
    C = np.asarray(C, dtype=np.float64)
    if C.size == 0:
        C = C.reshape(A.n, 0)
    if C.shape[1] == 0:
        return Deflation(C, C.copy(), np.zeros((0, 0)))
    AC = csr(A) @ C
    G = C.T @ AC
    G = 0.5 * (G + G.T)
    return Deflation(C, AC, dense_cholesky(G, pivot_rtol=RANK_GUARD_RTOL))


class Trace:
    """SolveTrace fields (solver.py:142-162)."""

    def __init__(self):
        self.alphas, self.betas, self.rz_inner = [], [], []
        self.residual_norms, self.z_history = [], []
        self.w_history, self.r_history = [], []
        self.iterations = 0
        self.converged = False


def apcg_solve(A, inv_diag, D, b, tol, max_iters, reorthogonalize=True,
               trace_capture=True, store_directions=False):
    """Augmented PCG, loop for loop as solver.py:193-290.

    ``inv_diag`` None means the identity preconditioner (solver.py:50-54).
    Raises OracleNumericalFailure where the reference raises NumericalFailure.
    """
    Acsr = csr(A)
    b = np.asarray(b, dtype=np.float64)
    trace = Trace()
    x = D.initial_guess(b)                                 # :210
    r = b - Acsr @ x if D.n_c else b.copy()                # :213
    r0 = float(np.linalg.norm(r))
    trace.residual_norms.append(r0)
    bnorm = float(np.linalg.norm(b))
    if r0 == 0.0 or r0 <= 1e-13 * bnorm:                   # :217-219
        trace.converged = True
        return x, trace

    def precond_project(v):                                # :221-225
        y = v.copy() if inv_diag is None else inv_diag * v
        return D.project(y)

    z = precond_project(r)
    rz = float(r @ z)
    if rz <= 0.0:
        raise OracleNumericalFailure("(r, z) <= 0: preconditioner or operator not SPD")
    w = z.copy()
    # preallocated C-order direction blocks grown geometrically, exactly as the
    # reference stores them (solver.py:233-240) so BLAS sees the same layout
    cap = 64
    W = np.empty((A.n, cap))
    AW = np.empty((A.n, cap))
    waw = np.empty(cap)
    stored = 0
    for _ in range(max_iters):                             # :241-288
        Aw = Acsr @ w
        wAw = float(w @ Aw)
        if wAw <= 0.0:
            raise OracleNumericalFailure("(w, A w) <= 0: operator not SPD on search space")
        alpha = rz / wAw
        trace.alphas.append(alpha)
        trace.rz_inner.append(rz)
        if trace_capture:
            trace.z_history.append(z)
        if store_directions:
            trace.w_history.append(w.copy())
            trace.r_history.append(r.copy())
        x = x + alpha * w
        r = r - alpha * Aw
        rnorm = float(np.linalg.norm(r))
        trace.residual_norms.append(rnorm)
        trace.iterations += 1
        if reorthogonalize:                                # :262-271
            if stored == cap:
                cap *= 2
                W = np.concatenate([W, np.empty_like(W)], axis=1)
                AW = np.concatenate([AW, np.empty_like(AW)], axis=1)
                waw = np.concatenate([waw, np.empty_like(waw)])
            W[:, stored] = w
            AW[:, stored] = Aw
            waw[stored] = wAw
            stored += 1
        if rnorm <= tol * r0:                              # :273
            trace.converged = True
            break
        z = precond_project(r)
        rz_next = float(r @ z)
        if rz_next <= 0.0:
            raise OracleNumericalFailure("(r, z) <= 0: preconditioner or operator not SPD")
        beta = rz_next / rz
        trace.betas.append(beta)
        w = z + beta * w
        if reorthogonalize:                                # :284-287 (block CGS)
            Wv = W[:, :stored]
            w = w - Wv @ ((AW[:, :stored].T @ w) / waw[:stored])
        rz = rz_next
    return x, trace


# ---------------------------------------------------------------------------
# ritz.py


def lanczos_tridiag(alphas, betas):
    """d_0 = 1/a_0, d_j = 1/a_j + b_{j-1}/a_{j-1}, e_j = sqrt(b_j)/a_j (ritz.py:61-78)."""
    a = np.asarray(alphas, dtype=np.float64)
    bt = np.asarray(betas, dtype=np.float64)
    m = len(a)
    if np.any(bt < 0.0):
        raise OracleNumericalFailure("negative beta coefficient: operator not SPD")
    d = np.empty(m)
    d[0] = 1.0 / a[0]
    if m > 1:
        d[1:] = 1.0 / a[1:] + bt / a[:-1]
    e = np.sqrt(bt) / a[:-1]
    return d, e


def lanczos_basis(trace):
    """V = [(-1)^j z_j / sqrt(r_j, z_j)] (ritz.py:81-94)."""
    m = trace.iterations
    signs = (-1.0) ** np.arange(m)
    scales = signs / np.sqrt(np.asarray(trace.rz_inner[:m], dtype=np.float64))
    return np.column_stack(trace.z_history[:m]) * scales


def select_converged(cur, prev, epsilon):
    """Two-sided stagnation flags + degenerate coalescing (ritz.py:103-138)."""
    cur = np.asarray(cur, dtype=np.float64)
    prev = np.asarray(prev, dtype=np.float64)
    m = len(cur)
    mask = np.zeros(m, dtype=bool)
    if m < 2:
        return mask
    for j in range(m - 1):
        if abs(cur[j] - prev[j]) <= epsilon * abs(cur[j]):
            mask[j] = True
        if abs(cur[j + 1] - prev[j]) <= epsilon * abs(cur[j + 1]):
            mask[j + 1] = True
    for j in range(1, m):
        big = max(abs(cur[j - 1]), abs(cur[j]))
        if big > 0 and abs(cur[j - 1] - cur[j]) < DEGENERATE_GAP * big:
            if mask[j]:
                first = j - 1
                while first > 0 and abs(cur[first - 1] - cur[first]) < \
                        DEGENERATE_GAP * max(abs(cur[first - 1]), abs(cur[first])):
                    first -= 1
                mask[first] = True
                mask[j] = False
    return mask


def cluster_filter(values, min_cluster):
    """Indices outside the central cluster: best 3-segment constant fit of the
    gaps, ties -> larger cluster, smaller level, smaller start (ritz.py:141-183)."""
    values = np.asarray(values, dtype=np.float64)
    m = len(values)
    if m < min_cluster or m < 2:
        return list(range(m))
    gaps = np.abs(np.diff(values))
    ng = len(gaps)
    p1 = np.concatenate([[0.0], np.cumsum(gaps)])
    p2 = np.concatenate([[0.0], np.cumsum(gaps ** 2)])

    def sse(i, j):
        if j <= i:
            return 0.0
        s = p1[j] - p1[i]
        return (p2[j] - p2[i]) - s * s / (j - i)

    def mean(i, j):
        return (p1[j] - p1[i]) / (j - i) if j > i else 0.0

    best = None
    span = min_cluster - 1
    for a in range(0, ng - span + 1):
        for bb in range(a + span, ng + 1):
            key = (sse(0, a) + sse(a, bb) + sse(bb, ng), -(bb - a), mean(a, bb), a)
            if best is None or key < best[0]:
                best = (key, a, bb)
    _, a, bb = best
    return [i for i in range(m) if i < a or i > bb]


class Spectrum:
    def __init__(self, values, vectors, mask, epsilon):
        self.values, self.vectors, self.converged_mask, self.epsilon = values, vectors, mask, epsilon


def select_spectrum(trace, epsilon, cluster=False, min_cluster=0):
    """lanczos -> Ritz pairs -> eig(H_{m-1}) -> select (-> cluster)
    (recycle.py:157-175)."""
    m = trace.iterations
    d, e = lanczos_tridiag(trace.alphas[:m], trace.betas[:m - 1])
    V = lanczos_basis(trace)
    vals, Q = tridiag_eig(d, e)
    Y = V @ Q                                              # ritz.py:100
    if m < 2:
        return Spectrum(vals, Y, np.zeros(m, dtype=bool), epsilon)
    prev = tridiag_eigvals(d[:m - 1], e[:m - 2])
    mask = select_converged(vals, prev, epsilon)
    if cluster:
        pre = int(mask.sum())
        if pre > 0:
            mc = min_cluster or max(1, math.ceil(pre / 5))
            keep = set(cluster_filter(vals, mc))
            mask = np.array([mask[j] and j in keep for j in range(m)], dtype=bool)
    return Spectrum(vals, Y, mask, epsilon)


# ---------------------------------------------------------------------------
# recycle.py


def srks_block(spec):
    """Flagged Ritz vectors scaled by 1/sqrt(|theta|) (recycle.py:143-154)."""
    idx = np.flatnonzero(spec.converged_mask)
    return spec.vectors[:, idx] / np.sqrt(np.abs(spec.values[idx])), idx


def trks_block(trace):
    """All w_j normalized; zero columns dropped (recycle.py:127-140)."""
    if not trace.w_history:
        return np.zeros((0, 0))
    W = np.column_stack(trace.w_history)
    norms = np.linalg.norm(W, axis=0)
    keep = norms > 0.0
    return W[:, keep] / norms[keep]


class SequenceResult:
    def __init__(self):
        self.iterations, self.n_c_before, self.n_c_selected = [], [], []
        self.converged, self.final_residual = [], []
        self.events, self.aborted = [], False
        self.selected_values, self.solutions = [], []
        self.final_basis = None


def run_sequence(systems, strategy="none", epsilon=1e-14, nc_limit=0, tol=1e-6,
                 max_iters=1000, reorthogonalize=True, jacobi=True, C0=None,
                 keep_solutions=False, min_cluster=0):
    """run_sequence (recycle.py:178-238) with the guarded build
    (recycle.py:113-124) and the TRKS/SRKS updates."""
    res = SequenceResult()
    basis = None
    tags = None
    initial = None
    for k, (A, b) in enumerate(systems):
        if basis is None:
            basis = np.zeros((A.n, 0)) if C0 is None else np.asarray(C0, dtype=np.float64).copy()
            initial = basis.copy()
            tags = [("initial", j) for j in range(basis.shape[1])]
        ncb = basis.shape[1]
        while True:                                        # guarded_deflation
            try:
                D = build_deflation(A, basis)
                break
            except OracleRankDeficient as exc:
                res.events.append(("dropped_column", exc.column, tags[exc.column]))
                basis = np.delete(basis, exc.column, axis=1)
                del tags[exc.column]
                if basis.shape[1] == 0:
                    D = build_deflation(A, basis)
                    break
        inv_diag = 1.0 / diagonal(A) if jacobi else None
        try:
            x, tr = apcg_solve(A, inv_diag, D, b, tol, max_iters, reorthogonalize,
                               trace_capture=True,
                               store_directions=(strategy == "trks"))
        except OracleNumericalFailure as exc:
            res.events.append(("solve_failed", k, str(exc)))
            res.aborted = True
            break
        sel_vals = np.zeros(0)
        if tr.converged and tr.iterations > 0:
            if strategy == "trks":
                blk = trks_block(tr)
                if blk.size:
                    basis = np.column_stack([basis, blk])
                    tags += [("direction", k, j) for j in range(blk.shape[1])]
            elif strategy in ("srks", "srks_cluster"):
                spec = select_spectrum(tr, epsilon, cluster=(strategy == "srks_cluster"),
                                       min_cluster=min_cluster)
                blk, idx = srks_block(spec)
                sel_vals = spec.values[idx]
                if blk.size:
                    basis = np.column_stack([basis, blk])
                    tags += [("ritz", k, float(v)) for v in sel_vals]
        selected = basis.shape[1] - ncb
        if nc_limit > 0 and basis.shape[1] >= nc_limit:   # recycle.py:223-225
            res.events.append(("restart", k, basis.shape[1]))
            basis = initial.copy()
            tags = [("initial", j) for j in range(basis.shape[1])]
        bn = float(np.linalg.norm(b))
        res.iterations.append(tr.iterations)
        res.n_c_before.append(ncb)
        res.n_c_selected.append(selected)
        res.converged.append(tr.converged)
        res.final_residual.append(tr.residual_norms[-1] / bn if bn > 0 else 0.0)
        res.selected_values.append(sel_vals)
        if keep_solutions:
            res.solutions.append(x)
    res.final_basis = basis
    return res
