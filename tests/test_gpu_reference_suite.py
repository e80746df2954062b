"""The reference's own unit and acceptance checks (pkg/tests/test_solver.py,
test_ritz.py, test_recycle.py, test_acceptance.py criteria 1-5 and 7), restated
against the B200 package.  Each test cites the reference test it mirrors; the
independent oracles are the same ones the reference uses (textbook CG,
explicitly projected operators, prescribed spectra, dense eigensolves)."""
import math

import numpy as np
import pytest

import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems
from paper_1301_7530_b200.recycle import AugmentationState, guarded_deflation, select_spectrum
from paper_1301_7530_b200.ritz import RitzSpectrum

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["persistent", "multi_kernel"])
def solve_loop(request, monkeypatch):
    """Every reference check runs through both solve loops: the persistent
    cooperative kernel (small operators, the default here) and the per-phase
    kernel sequence (RCG_SMALL_N=0)."""
    if request.param == "multi_kernel":
        monkeypatch.setenv("RCG_SMALL_N", "0")
    return request.param


def spd(n, rng, cond=100.0):
    return rcg.SparseSpdMatrix.from_dense(problems.random_spd(n, rng, cond), keep_zeros=True)


def reference_cg(A, b, tol=1e-10, max_iters=500):
    """Textbook CG (test_solver.py:12-36 oracle), dense numpy."""
    x = np.zeros_like(b)
    r = b.copy()
    norms = [np.linalg.norm(r)]
    p = r.copy()
    rr = r @ r
    for _ in range(max_iters):
        Ap = A @ p
        alpha = rr / (p @ Ap)
        x += alpha * p
        r -= alpha * Ap
        norms.append(np.linalg.norm(r))
        if norms[-1] <= tol * norms[0]:
            break
        rr_new = r @ r
        p = r + (rr_new / rr) * p
        rr = rr_new
    return x, norms


def solve(A, b, C=None, M=None, **kw):
    C = np.zeros((A.n, 0)) if C is None else C
    M = M or rcg.Preconditioner.identity()
    cfg = rcg.SolveConfig(**{"tol": 1e-10, "max_iters": 500, **kw})
    return rcg.apcg_solve(A, M, rcg.build_deflation(A, C), b, cfg)


# ---------------------------------------------------------------- solver


def test_deflation_single_eigenvector():                      # test_solver.py:76-81
    A = rcg.SparseSpdMatrix.from_dense(np.diag([1.0, 2.0, 3.0]))
    e1 = np.eye(3)[:, :1]
    D = rcg.build_deflation(A, e1)
    np.testing.assert_allclose(D.coarse_factor @ D.coarse_factor.T, [[1.0]])
    np.testing.assert_allclose(D.project(e1[:, 0]), np.zeros(3), atol=1e-14)


def test_empty_deflation_is_identity():                       # :84-89
    A = rcg.SparseSpdMatrix.from_dense(np.diag([1.0, 2.0]))
    D = rcg.build_deflation(A, np.zeros((2, 0)))
    x = np.array([3.0, 4.0])
    np.testing.assert_array_equal(rcg.project(D, x), x)
    np.testing.assert_array_equal(D.initial_guess(x), np.zeros(2))


def test_projected_operator_rank(rng):                        # :92-99
    A = spd(6, rng)
    D = rcg.build_deflation(A, rng.standard_normal((6, 2)))
    P = np.column_stack([D.project(col) for col in np.eye(6)])
    PtAP = P.T @ A.to_dense() @ P
    vals = np.linalg.eigvalsh(0.5 * (PtAP + PtAP.T))
    assert np.sum(np.abs(vals) > 1e-8 * vals.max()) == 4


def test_projection_idempotent_and_kills_coarse_residual(rng):   # :102-126
    A = spd(8, rng)
    C = rng.standard_normal((8, 3))
    D = rcg.build_deflation(A, C)
    x = rng.standard_normal(8)
    once = D.project(x)
    np.testing.assert_allclose(D.project(once), once, atol=1e-10 * np.linalg.norm(x))
    np.testing.assert_allclose(C.T @ (A @ once), np.zeros(3), atol=1e-10 * np.linalg.norm(x))
    v = C @ rng.standard_normal(3)
    np.testing.assert_allclose(D.project(v), np.zeros(8), atol=1e-10 * np.linalg.norm(v))


def test_build_deflation_rejects_bad_shapes(rng):            # :129-134
    A = spd(4, rng)
    with pytest.raises(rcg.ContractViolation):
        rcg.build_deflation(A, np.ones((3, 1)))
    with pytest.raises(rcg.ContractViolation):
        rcg.build_deflation(A, np.ones((4, 5)))


def test_identity_one_iteration_and_full_augmentation(rng):  # :141-157
    A = rcg.SparseSpdMatrix.from_dense(np.eye(5))
    b = rng.standard_normal(5)
    x, tr = solve(A, b)
    assert tr.converged and tr.iterations == 1
    np.testing.assert_allclose(x, b, rtol=1e-12)
    n = 6
    A = rcg.SparseSpdMatrix.from_dense(np.diag(np.arange(1.0, n + 1.0)))
    b = rng.standard_normal(n)
    x, tr = solve(A, b, C=np.eye(n))
    assert tr.converged and tr.iterations == 0
    np.testing.assert_allclose(x, b / np.arange(1.0, n + 1.0), rtol=1e-10)


def test_deflated_iteration_count_matches_reduced_system():  # :160-166
    A = rcg.SparseSpdMatrix.from_dense(np.diag([1.0, 10.0, 100.0]))
    _, tr = solve(A, np.ones(3), C=np.eye(3)[:, :1])
    _, norms = reference_cg(np.diag([10.0, 100.0]), np.ones(2))
    assert tr.converged and tr.iterations == len(norms) - 1 == 2


def test_trace_contracts_and_coarse_orthogonality(rng):      # :169-190
    A = spd(30, rng)
    b = rng.standard_normal(30)
    x, tr = solve(A, b, C=rng.standard_normal((30, 4)))
    m = tr.iterations
    assert tr.converged and len(tr.alphas) == m and len(tr.betas) == m - 1
    assert len(tr.residual_norms) == m + 1
    assert all(a > 0 for a in tr.alphas) and all(v > 0 for v in tr.rz_inner)
    np.testing.assert_allclose(A @ x, b, atol=1e-9 * np.linalg.norm(b))
    A = spd(25, rng)
    C = rng.standard_normal((25, 5))
    b = rng.standard_normal(25)
    _, tr = solve(A, b, C=C, store_directions=True)
    for r in tr.r_history:
        assert np.abs(C.T @ r).max() <= 1e-10 * np.linalg.norm(b)


def test_max_iters_reports_nonconvergence(rng):              # :193-198
    A = spd(40, rng, 1e4)
    _, tr = solve(A, rng.standard_normal(40), tol=1e-12, max_iters=3)
    assert not tr.converged and tr.iterations == 3 and len(tr.betas) == 3


def test_matches_cg_on_projected_operator(rng):              # :227-245
    for n, n_c, steps in ((12, 2, 8), (25, 4, 10), (40, 6, 10)):
        A = spd(n, rng)
        C = rng.standard_normal((n, n_c))
        b = rng.standard_normal(n)
        D = rcg.build_deflation(A, C)
        _, tr = solve(A, b, C=C, tol=1e-15, max_iters=steps, reorthogonalize=False)
        P = np.column_stack([D.project(col) for col in np.eye(n)])
        B = P.T @ A.to_dense() @ P
        _, norms = reference_cg(0.5 * (B + B.T), P.T @ b, tol=1e-15, max_iters=steps)
        assert len(norms) == len(tr.residual_norms) == steps + 1
        np.testing.assert_allclose(tr.residual_norms, norms, rtol=1e-8)


def test_split_preconditioner_equivalence(rng):              # :248-268
    n, n_c = 20, 3
    A = spd(n, rng)
    C = rng.standard_normal((n, n_c))
    b = rng.standard_normal(n)
    diag = rng.uniform(0.5, 4.0, n)
    L = np.sqrt(diag)
    A_hat = rcg.SparseSpdMatrix.from_dense(A.to_dense() / np.outer(L, L), keep_zeros=True)
    _, t1 = solve(A, b, C=C, M=rcg.Preconditioner.user_diagonal(diag), tol=1e-15, max_iters=12,
                  reorthogonalize=False)
    _, t2 = solve(A_hat, b / L, C=C * L[:, None], tol=1e-15, max_iters=12, reorthogonalize=False)
    assert t1.iterations == t2.iterations == 12
    np.testing.assert_allclose(t1.alphas, t2.alphas, rtol=1e-9)
    np.testing.assert_allclose(t1.betas, t2.betas, rtol=1e-9)


def test_finite_termination_and_augmentation_never_hurts(rng):  # :271-289
    for k in (2, 3, 5):
        vals = np.repeat(np.arange(1.0, k + 1.0), 4)
        A = rcg.SparseSpdMatrix.from_dense(np.diag(vals))
        _, tr = solve(A, rng.uniform(0.5, 1.5, len(vals)), tol=1e-12)
        assert tr.converged and tr.iterations <= k
    for _ in range(5):
        A = spd(30, rng, 1e3)
        b = rng.standard_normal(30)
        C = rng.standard_normal((30, 3))
        _, ts = solve(A, b, C=C, tol=1e-8)
        _, tb = solve(A, b, C=np.column_stack([C, rng.standard_normal((30, 3))]), tol=1e-8)
        assert tb.iterations <= ts.iterations + 1


# ---------------------------------------------------------------- ritz


def test_two_point_spectrum_and_basis(rng):                   # test_ritz.py:52-82
    A = rcg.SparseSpdMatrix.from_dense(np.diag([1.0, 4.0]))
    _, tr = solve(A, np.array([1.0, 1.0]), tol=1e-12)
    view = rcg.lanczos_from_trace(tr)
    np.testing.assert_allclose(rcg.tridiag_eig(view.tridiag).values, [4.0, 1.0], atol=1e-12)
    H = view.basis.T @ A.to_dense() @ view.basis
    np.testing.assert_allclose(H, view.tridiag.to_dense(), atol=1e-12)
    n = 10
    lap = 2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    _, tr = solve(rcg.SparseSpdMatrix.from_dense(lap), np.arange(1.0, n + 1.0), tol=1e-14)
    view = rcg.lanczos_from_trace(tr)
    assert view.m == n
    np.testing.assert_allclose(np.sort(rcg.tridiag_eig(view.tridiag).values), np.linalg.eigvalsh(lap), rtol=1e-8)
    A = spd(20, rng)
    _, tr = solve(A, rng.standard_normal(20), tol=1e-12)
    V = rcg.lanczos_from_trace(tr).basis
    np.testing.assert_allclose(V.T @ V, np.eye(V.shape[1]), atol=1e-6)


def test_lanczos_requires_history_and_validation(rng):       # :35-49
    with pytest.raises(rcg.ContractViolation):
        rcg.lanczos_tridiag([], [])
    with pytest.raises(rcg.NumericalFailure):
        rcg.lanczos_tridiag([1.0, 1.0], [-0.5])
    T = rcg.lanczos_tridiag([0.5], [])
    np.testing.assert_array_equal(T.diag, [2.0])
    A = spd(10, rng)
    _, tr = solve(A, rng.standard_normal(10), tol=1e-12)
    tr.z_history.clear()
    with pytest.raises(rcg.ContractViolation):
        rcg.lanczos_from_trace(tr)


def test_ritz_pairs_axes_and_a_orthogonality(rng):            # :89-118
    A = rcg.SparseSpdMatrix.from_dense(np.diag([3.0, 3.0]))
    _, tr = solve(A, np.array([1.0, 2.0]), tol=1e-12)
    sp = rcg.ritz_pairs(rcg.lanczos_from_trace(tr))
    assert sp.m == 1
    np.testing.assert_allclose(sp.values, [3.0], rtol=1e-12)
    A = rcg.SparseSpdMatrix.from_dense(np.diag([1.0, 2.0, 3.0]))
    _, tr = solve(A, np.ones(3), tol=1e-13)
    sp = rcg.ritz_pairs(rcg.lanczos_from_trace(tr))
    np.testing.assert_allclose(np.sort(sp.values), [1.0, 2.0, 3.0], rtol=1e-10)
    for got, want in zip(sp.vectors.T, np.eye(3)[:, ::-1].T):
        got = got / np.linalg.norm(got)
        assert min(np.linalg.norm(got - want), np.linalg.norm(got + want)) < 1e-6
    A = spd(30, rng)
    _, tr = solve(A, rng.standard_normal(30), tol=1e-12)
    sp = rcg.ritz_pairs(rcg.lanczos_from_trace(tr))
    Y = sp.vectors
    np.testing.assert_allclose(Y.T @ A.to_dense() @ Y, np.diag(sp.values), atol=1e-6 * sp.values.max())
    np.testing.assert_allclose(Y.T @ Y, np.eye(sp.m), atol=1e-6)


def test_interlacing_along_a_run(rng):                         # :121-133
    A = spd(40, rng, 1e3)
    _, tr = solve(A, rng.standard_normal(40), tol=1e-12)
    view = rcg.lanczos_from_trace(tr)
    prev = None
    for m in range(1, view.m + 1):
        cur = rcg.tridiag_eig(view.tridiag.truncated(m)).values
        if prev is not None:
            slack = 1e-12 * cur[0]
            assert np.all(cur[:-1] >= prev - slack) and np.all(prev >= cur[1:] - slack)
        prev = cur


def test_isolated_high_value_converges_first():               # :184-203
    values = np.concatenate([[1.0], np.arange(2.0, 3.01, 0.1), [100.0]])
    A = rcg.SparseSpdMatrix.from_dense(np.diag(values))
    _, tr = solve(A, np.ones(len(values)), tol=1e-10, max_iters=200)
    view = rcg.lanczos_from_trace(tr)
    first = {}
    for m in range(2, view.m + 1):
        cur = rcg.tridiag_eig(view.tridiag.truncated(m))
        prev = rcg.tridiag_eig(view.tridiag.truncated(m - 1)).values
        sel = rcg.select_converged(RitzSpectrum(cur.values, cur.vectors), prev, epsilon=1e-8)
        for j in np.flatnonzero(sel.converged_mask):
            first.setdefault(round(float(sel.values[j]), 3), m)
    near = min(first.items(), key=lambda kv: abs(kv[0] - 100.0))
    interior = [m for v, m in first.items() if 1.5 < v < 50.0]
    assert near[1] <= min(interior, default=10 ** 9)


# ---------------------------------------------------------------- recycle


def constant_sequence(A, b, count):
    return ((A, b.copy()) for _ in range(count))


def test_guarded_deflation_drops_dependent_columns(rng):      # test_recycle.py:52-61
    A = spd(8, rng)
    good = rng.standard_normal((8, 2))
    state = AugmentationState.from_initial(8, np.column_stack([good, good[:, 0] + 2.0 * good[:, 1]]))
    events = []
    D = guarded_deflation(A, state, events)
    assert D.n_c == 2 and state.n_c == 2 and events[0][0] == "dropped_column"


def test_trks_appends_unit_directions(rng):                    # :68-89
    A = spd(12, rng)
    _, tr = solve(A, rng.standard_normal(12), tol=1e-3, store_directions=True)
    st = AugmentationState.from_initial(12)
    rcg.update_basis_trks(st, tr)
    assert st.n_c == tr.iterations
    np.testing.assert_allclose(np.linalg.norm(st.basis, axis=0), 1.0)
    _, tr = solve(spd(8, rng), rng.standard_normal(8))
    with pytest.raises(rcg.ContractViolation):
        rcg.update_basis_trks(AugmentationState.from_initial(8), tr)
    st = AugmentationState.from_initial(4)
    rcg.update_basis_trks(st, rcg.SolveTrace())
    assert st.n_c == 0


def test_srks_selection_monotone_and_coarse_identity(rng):    # :92-128
    A = spd(25, rng, 1e4)
    _, tr = solve(A, rng.standard_normal(25), tol=1e-10)
    tight = select_spectrum(tr, rcg.RecycleStrategy("srks", epsilon=1e-14))
    loose = select_spectrum(tr, rcg.RecycleStrategy("srks", epsilon=1e-6))
    assert np.all(loose.converged_mask[tight.converged_mask])
    A = spd(30, rng, 1e3)
    _, tr = solve(A, rng.standard_normal(30), tol=1e-12)
    sp = select_spectrum(tr, rcg.RecycleStrategy("srks", epsilon=1e-10))
    assert sp.converged_mask.sum() >= 3
    st = AugmentationState.from_initial(30)
    rcg.update_basis_srks(st, sp)
    np.testing.assert_allclose(st.basis.T @ (A @ st.basis), np.eye(st.n_c), atol=1e-8)
    sp2 = rcg.ritz_pairs(rcg.lanczos_from_trace(tr))
    with pytest.raises(rcg.ContractViolation):
        rcg.update_basis_srks(AugmentationState.from_initial(30), sp2)


def test_run_sequence_behaviours(rng):                         # :134-209
    A = spd(20, rng)
    b = rng.standard_normal(20)
    rep = rcg.run_sequence(constant_sequence(A, b, 3), lambda A: rcg.Preconditioner.identity(),
                           rcg.RecycleStrategy("trks"), rcg.SolveConfig(tol=1e-10, max_iters=200))
    it = rep.iterations()
    assert it[0] > 0 and it[1] == 0 and it[2] == 0
    A = spd(30, rng, 1e3)
    b = rng.standard_normal(30)
    rep = rcg.run_sequence(constant_sequence(A, b, 2), lambda A: rcg.Preconditioner.identity(),
                           rcg.RecycleStrategy("srks", epsilon=1e-10), rcg.SolveConfig(tol=1e-12, max_iters=200))
    C = rep.final_basis
    assert C.shape[1] >= 3
    np.testing.assert_allclose(C.T @ (A @ C), np.eye(C.shape[1]), atol=1e-8)
    A = spd(15, rng)
    C0 = rng.standard_normal((15, 2))
    rep = rcg.run_sequence(constant_sequence(A, rng.standard_normal(15), 3), lambda A: rcg.Preconditioner.identity(),
                           rcg.RecycleStrategy("none"), rcg.SolveConfig(tol=1e-8, max_iters=100), C0=C0)
    assert rep.n_c_history() == [2, 2, 2]
    np.testing.assert_array_equal(rep.final_basis, C0)
    rep = rcg.run_sequence(constant_sequence(spd(20, rng), rng.standard_normal(20), 3),
                           lambda A: rcg.Preconditioner.identity(), rcg.RecycleStrategy("trks", nc_limit=5),
                           rcg.SolveConfig(tol=1e-10, max_iters=100))
    assert any(ev[0] == "restart" for ev in rep.events) and rep.n_c_history()[1] == 0
    systems = [(spd(12, rng), rng.standard_normal(12)) for _ in range(4)]
    rep = rcg.run_sequence(iter(systems), rcg.Preconditioner.jacobi, rcg.RecycleStrategy("trks"),
                           rcg.SolveConfig(tol=1e-8, max_iters=200))
    for prev, cur in zip(rep.records, rep.records[1:]):
        assert cur.n_c_before == prev.n_c_before + prev.n_c_selected
    assert all(r.converged and r.final_residual <= 1e-6 and r.solve_seconds >= 0 for r in rep.records)


# ---------------------------------------------------------------- acceptance


def test_criterion_1_orthogonality():                          # test_acceptance.py:42-81
    rng = np.random.Generator(np.random.Philox(42))
    worst_rz = worst_waw = 0.0
    runs = 0
    for _ in range(50):
        n = int(rng.integers(20, 301))
        lam = np.geomspace(1.0, rng.uniform(10.0, 50.0), n)
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        G = (Q * lam) @ Q.T
        A = rcg.SparseSpdMatrix.from_dense(0.5 * (G + G.T), keep_zeros=True)
        _, tr = solve(A, rng.standard_normal(n), tol=1e-6, max_iters=60, reorthogonalize=True,
                      store_directions=True)
        m = tr.iterations
        if not tr.converged or m < 2:
            continue
        runs += 1
        Z = np.column_stack(list(tr.z_history)[:m])
        R = np.column_stack(list(tr.r_history)[:m])
        cross = np.abs(R.T @ Z) / np.outer(np.linalg.norm(R, axis=0), np.linalg.norm(Z, axis=0))
        np.fill_diagonal(cross, 0.0)
        worst_rz = max(worst_rz, cross.max())
        W = np.column_stack(list(tr.w_history))
        gram = W.T @ np.column_stack([A @ w for w in W.T])
        an = np.sqrt(np.diag(gram))
        waw = np.abs(gram) / np.outer(an, an)
        np.fill_diagonal(waw, 0.0)
        worst_waw = max(worst_waw, waw.max())
    assert runs >= 45 and worst_rz <= 1e-8 and worst_waw <= 1e-8


def test_criterion_2_deflation_exactness():                    # :84-104
    n = 100
    lam = np.geomspace(0.01, 100.0, n)
    A = problems.generate_prescribed_spectrum(problems.SpectrumSpec(tuple(lam), seed=21))
    w, v = np.linalg.eigh(A.to_dense())
    rng = np.random.Generator(np.random.Philox(7))
    b = rng.standard_normal(n)
    for k in (1, 3, 5):
        _, tr = solve(A, b, C=v[:, :k], tol=1e-8, max_iters=400)
        _, tro = solve(rcg.SparseSpdMatrix.from_dense(np.diag(lam[k:])), v[:, k:].T @ b, tol=1e-8, max_iters=400)
        assert tr.converged and tro.converged and abs(tr.iterations - tro.iterations) <= 1


def test_criterion_4_ritz_fidelity():                          # :159-191
    n = 200
    lam = np.geomspace(1.0, 100.0, n)
    A = problems.generate_prescribed_spectrum(problems.SpectrumSpec(tuple(lam), seed=13))
    b = np.random.Generator(np.random.Philox(5)).standard_normal(n)
    _, tr = solve(A, b, tol=1e-13, max_iters=n)
    view = rcg.lanczos_from_trace(tr)
    cur = rcg.tridiag_eig(view.tridiag)
    prev = rcg.tridiag_eig(view.tridiag.truncated(view.m - 1)).values
    sel = rcg.select_converged(RitzSpectrum(cur.values, cur.vectors), prev, epsilon=1e-8)
    theta = sel.values[sel.converged_mask]
    rel = np.abs(theta[:, None] - lam[None, :]).min(axis=1) / theta
    assert tr.converged and len(theta) >= 40 and rel.max() <= 1e-7


def test_criterion_7_selection_and_coarse_identity():          # :269-292
    rng = np.random.Generator(np.random.Philox(31))
    for _ in range(5):
        n = 30
        lam = np.geomspace(1.0, 1e3, n)
        A = problems.generate_prescribed_spectrum(problems.SpectrumSpec(tuple(lam), seed=int(rng.integers(1000))))
        _, tr = solve(A, rng.standard_normal(n), tol=1e-12, max_iters=200)
        tight = select_spectrum(tr, rcg.RecycleStrategy("srks", epsilon=1e-14))
        loose = select_spectrum(tr, rcg.RecycleStrategy("srks", epsilon=1e-6))
        assert np.all(loose.converged_mask[tight.converged_mask])
        sp = select_spectrum(tr, rcg.RecycleStrategy("srks", epsilon=1e-10))
        if sp.converged_mask.any():
            st = AugmentationState.from_initial(n)
            rcg.update_basis_srks(st, sp)
            np.testing.assert_allclose(st.basis.T @ (A @ st.basis), np.eye(st.n_c), atol=1e-8)
