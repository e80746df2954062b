"""GPU parity of the individual kernels against the CPU oracle / closed forms."""
import numpy as np
import pytest
import scipy.linalg

import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems
from oracle import recycg_oracle as orc

pytestmark = pytest.mark.gpu


def _spmv_close(A, x):
    y = rcg.spmv(A, x)
    want = orc.spmv(A, x)
    # reduction order differs from scipy: bound by ulps of |A||x| per row
    absrow = orc.csr(type("M", (), dict(n=A.n, row_offsets=A.row_offsets, col_indices=A.col_indices,
                                         values=np.abs(A.values)))) @ np.abs(x)
    assert np.all(np.abs(y - want) <= 8 * np.finfo(float).eps * absrow + 1e-300)


def test_spmv_config1_and_stencils(rng):
    A, _ = problems.shifted_laplacian_sequence(grid=128, count=2)[1]
    _spmv_close(A, rng.standard_normal(A.n))
    B = problems.assemble_diffusion(np.exp(rng.standard_normal((12, 10, 9))))
    _spmv_close(B, rng.standard_normal(B.n))


def test_spmv_elasticity_and_dense(rng):
    E = problems.elasticity_q1(6)
    _spmv_close(E, rng.standard_normal(E.n))
    D = rcg.SparseSpdMatrix.from_dense(problems.random_spd(70, rng), keep_zeros=True)
    _spmv_close(D, rng.standard_normal(70))


def test_spmv_kats():
    # reference tests/test_core.py:71-91
    A = rcg.SparseSpdMatrix.from_dense(np.eye(3))
    np.testing.assert_array_equal(rcg.spmv(A, [1.0, 2.0, 3.0]), [1.0, 2.0, 3.0])
    lap = 2.0 * np.eye(4) - np.eye(4, k=1) - np.eye(4, k=-1)
    np.testing.assert_array_equal(rcg.spmv(rcg.SparseSpdMatrix.from_dense(lap), [1.0, 0, 0, 0]),
                                  [2.0, -1.0, 0.0, 0.0])
    with pytest.raises(rcg.ContractViolation):
        rcg.spmv(A, np.ones(4))


def test_spmm_block(rng):
    A = problems.assemble_diffusion(np.ones((20, 17)))
    X = rng.standard_normal((A.n, 5))
    Y = A @ X
    np.testing.assert_allclose(Y, orc.csr(A) @ X, rtol=1e-13, atol=1e-13)


def test_diagonal_and_jacobi():
    A = rcg.SparseSpdMatrix.from_dense(np.diag([2.0, 4.0]))
    M = rcg.Preconditioner.jacobi(A)
    np.testing.assert_allclose(M.apply(np.array([2.0, 4.0])), [1.0, 1.0])
    np.testing.assert_allclose(M.diag(), [2.0, 4.0])
    np.testing.assert_array_equal(A.diagonal(), [2.0, 4.0])


@pytest.mark.parametrize("n", [2, 3, 10, 50, 127, 200, 700, 1601])
def test_cholesky_matches_oracle(rng, n):
    G = problems.random_spd(n, rng)
    L = rcg.dense_cholesky(G)
    np.testing.assert_allclose(L, np.linalg.cholesky(G), rtol=1e-10, atol=1e-12)


def test_cholesky_kats():
    np.testing.assert_allclose(rcg.dense_cholesky(np.array([[4.0, 2.0], [2.0, 2.0]])), [[2.0, 0.0], [1.0, 1.0]])
    with pytest.raises(rcg.RankDeficient) as ei:
        rcg.dense_cholesky(np.array([[1.0, 1.0], [1.0, 1.0]]))
    assert ei.value.column == 1
    with pytest.raises(rcg.ContractViolation):
        rcg.dense_cholesky(np.array([[1.0, 2.0], [0.0, 1.0]]))


@pytest.mark.parametrize("n,bad", [(40, 20), (150, 97), (900, 640), (900, 64), (900, 899)])
def test_cholesky_rank_deficient_column(rng, n, bad):
    # reference tests/test_core.py:136-146 (and the > 128 global-memory path)
    G = problems.random_spd(n, rng)
    B = np.linalg.cholesky(G)
    B[:, bad] = B[:, 5] + 2.0 * B[:, 7]
    G2 = B @ B.T
    with pytest.raises(rcg.RankDeficient) as ei:
        rcg.dense_cholesky(0.5 * (G2 + G2.T), pivot_rtol=1e-12)
    assert ei.value.column == bad
    with pytest.raises(orc.OracleRankDeficient) as eo:
        orc.dense_cholesky(0.5 * (G2 + G2.T), pivot_rtol=1e-12)
    assert eo.value.column == bad


@pytest.mark.parametrize("n", [60, 300, 1200])
def test_cholesky_inverse_blocked(rng, n):
    """G^-1 = L^-T L^-1 as build_deflation forms it (small: per-column
    substitution; n > 128: blocked factor + warp-per-column inverse)."""
    import torch
    from paper_1301_7530_b200 import _lib
    G = problems.random_spd(n, rng, condition=1e4)
    Gd = torch.from_numpy(np.ascontiguousarray(G)).cuda()
    L = torch.empty_like(Gd)
    Gi = torch.empty_like(Gd)
    bad = _lib.C.c_int64(-1)
    ctx = _lib.context()
    ctx.check(ctx.lib.rcg_dense_cholesky(ctx.h, _lib.ptr(Gd), n, 1e-12, _lib.ptr(L), _lib.ptr(Gi),
                                         _lib.C.byref(bad)), "cholesky")
    Gih = Gi.cpu().numpy()
    np.testing.assert_allclose(Gih, np.linalg.inv(G), rtol=0, atol=1e-9 * np.abs(np.linalg.inv(G)).max())


def test_tridiag_eig_closed_form():
    T = rcg.TridiagSym(np.full(4, 2.0), np.full(3, -1.0))
    eig = rcg.tridiag_eig(T)
    want = sorted((2.0 - 2.0 * np.cos(k * np.pi / 5.0) for k in range(1, 5)), reverse=True)
    np.testing.assert_allclose(eig.values, want, rtol=1e-12)
    H = T.to_dense()
    for th, q in zip(eig.values, eig.vectors.T):
        assert np.linalg.norm(H @ q - th * q) <= 1e-10 * np.linalg.norm(H)
    np.testing.assert_allclose(eig.vectors.T @ eig.vectors, np.eye(4), atol=1e-12)


@pytest.mark.parametrize("m", [2, 5, 40, 390, 1200])
def test_tridiag_eigvals_vs_lapack(rng, m):
    d = rng.uniform(1.0, 3.0, m)
    e = rng.uniform(-1.0, 1.0, m - 1)
    got = rcg.tridiag_eig(rcg.TridiagSym(d, e)) if m <= 400 else None
    want = orc.tridiag_eigvals(d, e)
    import torch
    from paper_1301_7530_b200.core import tridiag_eigvals_device
    vals = tridiag_eigvals_device(torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")).cpu().numpy()
    np.testing.assert_allclose(vals, want, rtol=0, atol=8 * np.finfo(float).eps * np.abs(want).max() * np.sqrt(m))
    if got is not None:
        H = rcg.TridiagSym(d, e).to_dense()
        R = H @ got.vectors - got.vectors * got.values
        assert np.abs(R).max() <= 1e-10 * np.abs(want).max()
        np.testing.assert_allclose(got.vectors.T @ got.vectors, np.eye(m), atol=1e-9)


def test_select_converged_kats():
    # reference tests/test_ritz.py:145-182
    def spec(v):
        return rcg.RitzSpectrum(np.asarray(v, dtype=float), np.eye(len(v)))
    assert list(rcg.select_converged(spec([9.0, 5.0, 2.0, 1.0]), [9.0, 5.0, 2.0], 1e-12).converged_mask) == \
        [True, True, True, False]
    assert not rcg.select_converged(spec([9.0, 5.0, 2.0]), [9.9, 5.5], 1e-6).converged_mask.any()
    assert list(rcg.select_converged(spec([9.0, 4.0, 1.0]), [6.0, 1.0], 1e-12).converged_mask) == \
        [False, False, True]
    m = rcg.select_converged(spec([5.0, 5.0 * (1 + 1e-15), 1.0]), [5.0, 5.0], 1e-12).converged_mask
    assert m[0] and not m[1]
    out = rcg.select_converged(spec([3.0]), [], 1e-6)
    assert out.m == 1 and not out.converged_mask.any()


def test_gemm_tn_nn(rng):
    import torch
    from paper_1301_7530_b200 import _lib
    n, a, b = 1000, 37, 45
    X = rng.standard_normal((n, a))
    Y = rng.standard_normal((n, b))
    Xd = torch.tensor(np.ascontiguousarray(X.T), device="cuda")
    Yd = torch.tensor(np.ascontiguousarray(Y.T), device="cuda")
    G = torch.empty((b, a), dtype=torch.float64, device="cuda")
    ctx = _lib.context()
    ctx.check(ctx.lib.rcg_gemm_tn(ctx.h, n, a, b, _lib.ptr(Xd), n, _lib.ptr(Yd), n, _lib.ptr(G), 0))
    np.testing.assert_allclose(G.cpu().numpy().T, X.T @ Y, rtol=1e-12, atol=1e-11)
    Q = rng.standard_normal((a, 7))
    Qd = torch.tensor(np.ascontiguousarray(Q.T), device="cuda")
    Out = torch.empty((7, n), dtype=torch.float64, device="cuda")
    ctx.check(ctx.lib.rcg_gemm_nn(ctx.h, n, a, 7, _lib.ptr(Xd), n, _lib.ptr(Qd), a, _lib.ptr(Out), n))
    np.testing.assert_allclose(Out.cpu().numpy().T, X @ Q, rtol=1e-12, atol=1e-11)


def test_block3_spmv_matches_scalar_csr(rng):
    """The device-built 3x3 BSR copy (SpMV format for Q1 elasticity) computes
    the same product as the scalar CSR path and as scipy."""
    E = np.exp(rng.standard_normal((5, 5, 5)))
    A0 = problems.elasticity_q1(5, E=E)
    A = rcg.SparseSpdMatrix(A0.n, A0.row_offsets, A0.col_indices, A0.values, validate=False, use_block3=True)
    B = rcg.SparseSpdMatrix(A0.n, A0.row_offsets, A0.col_indices, A0.values, validate=False, use_block3=False)
    assert A.device_csr().struct.dia_count == 14 and A.device_csr().struct.dia_block == 3   # structured Q1: DIA
    assert B.device_csr().struct.block == 0
    x = rng.standard_normal(A.n)
    ya, yb = rcg.spmv(A, x), rcg.spmv(B, x)
    np.testing.assert_allclose(ya, yb, rtol=1e-13, atol=1e-13 * np.abs(yb).max())
    _spmv_close(A, x)
    # not block structured -> scalar path
    L0 = problems.assemble_diffusion(np.ones((6, 6)))
    L = rcg.SparseSpdMatrix(L0.n, L0.row_offsets, L0.col_indices, L0.values, validate=False, use_block3=True)
    assert L.device_csr().struct.block == 0 and L.device_csr().struct.dia_count == 3    # 5-point: scalar DIA


@pytest.mark.parametrize("nelem", [1, 3, 7])
def test_sliced_block3_matches_plain_bsr(rng, monkeypatch, nelem):
    """SELL-32 sliced 3x3 blocks (padded short block rows, a ragged last
    chunk: n/3 not a multiple of 32) compute the same product as the plain
    BSR layout (identical per-row block order and rounding) and as scipy."""
    E = np.exp(rng.standard_normal((nelem,) * 3))
    A0 = problems.elasticity_q1(nelem, E=E)
    mk = lambda: rcg.SparseSpdMatrix(A0.n, A0.row_offsets, A0.col_indices, A0.values, validate=False)
    monkeypatch.setenv("RCG_DIA", "0")
    S = mk()
    assert S.device_csr().struct.bsr_slice == 32
    monkeypatch.setenv("RCG_SELL", "0")
    P = mk()
    assert P.device_csr().struct.block == 3 and P.device_csr().struct.bsr_slice == 0
    for _ in range(3):
        x = rng.standard_normal(A0.n)
        ys, yp = rcg.spmv(S, x), rcg.spmv(P, x)
        np.testing.assert_allclose(ys, yp, rtol=1e-14, atol=1e-14 * np.abs(yp).max())
        _spmv_close(S, x)


def _mk(A0, **kw):
    return rcg.SparseSpdMatrix(A0.n, A0.row_offsets, A0.col_indices, A0.values, validate=False, **kw)


@pytest.mark.parametrize("kind", ["diff1d", "diff2d", "diff3d", "diff3d_flat", "q1_1", "q1_4", "q1_7"])
def test_dia_matches_csr(rng, monkeypatch, kind):
    """Symmetric block-DIA (stencils b = 1, structured Q1 b = 3): the same
    product as scalar CSR on ragged grids (boundary rows, wrap-around
    offsets, a single element, size-1 axes) for all three SpMV modes."""
    monkeypatch.setenv("RCG_DIA3", "1")
    if kind.startswith("diff"):
        shape = {"diff1d": (37,), "diff2d": (9, 13), "diff3d": (5, 6, 7), "diff3d_flat": (4, 1, 9)}[kind]
        A0 = problems.assemble_diffusion(rng.lognormal(0.0, 1.0, shape))
        b = 1
    else:
        ne = int(kind.split("_")[1])
        A0 = problems.elasticity_q1(ne, E=np.exp(rng.standard_normal((ne,) * 3)))
        b = 3
    D = _mk(A0)
    assert D.device_csr().struct.dia_count > 0 and D.device_csr().struct.dia_block == b
    C = _mk(A0, use_block3=False)
    assert C.device_csr().struct.dia_count == 0
    for _ in range(3):
        x = rng.standard_normal(A0.n)
        yd, yc = rcg.spmv(D, x), rcg.spmv(C, x)
        np.testing.assert_allclose(yd, yc, rtol=1e-14, atol=1e-14 * np.abs(yc).max())
        _spmv_close(D, x)
    # modes 1 (solve loop) and 2 (initial residual) through a solve
    bvec = rng.standard_normal(A0.n)
    cfg = rcg.SolveConfig(tol=1e-10, max_iters=5000)
    xs = []
    for M in (D, C):
        x, tr = rcg.apcg_solve(M, rcg.Preconditioner.jacobi(M), rcg.build_deflation(M, np.zeros((M.n, 0))), bvec, cfg)
        xs.append((x, tr.iterations))
    assert abs(xs[0][1] - xs[1][1]) <= max(1, 0.02 * xs[1][1])
    assert np.linalg.norm(xs[0][0] - xs[1][0]) / np.linalg.norm(xs[1][0]) < 1e-8


def test_dia_rejects_asymmetric_and_unstructured(rng):
    """Not exactly symmetric (one lower entry perturbed) or not on a few
    diagonals (random sparse SPD): no DIA copy, CSR/BSR path instead."""
    A0 = problems.assemble_diffusion(rng.lognormal(0.0, 1.0, (6, 7)))
    va = A0.values.copy()
    rows = np.repeat(np.arange(A0.n), np.diff(A0.row_offsets))
    k = np.flatnonzero(A0.col_indices < rows)[5]
    va[k] = va[k] * (1 + 1e-15) + 1e-300
    Asym = rcg.SparseSpdMatrix(A0.n, A0.row_offsets, A0.col_indices, va, validate=False)
    assert Asym.device_csr().struct.dia_count == 0
    R = rcg.SparseSpdMatrix.from_dense(orc_random_spd(rng, 60))
    assert R.device_csr().struct.dia_count == 0


def orc_random_spd(rng, n):
    M = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.1)
    return M @ M.T + n * np.eye(n)


def test_small_operators_keep_csr_in_production(monkeypatch):
    """Without the test-suite override, an L2-resident operator (config-1
    5-point 128^2: 1 MB of CSR) keeps the CSR kernel; the 256^3 7-point
    operator (1.4 GB) takes the DIA one (test_full_size_counts_and_symmetry)."""
    monkeypatch.delenv("RCG_DIA_SMALL", raising=False)
    A, _ = problems.shifted_laplacian_sequence(count=1)[0]
    h = A.device_csr().struct
    assert h.dia_count == 0 and h.block == 0


def test_dia3_claimed_tiles_bitwise_reproducible(rng):
    """3x3 block-DIA solve-loop SpMV: 256-row tiles are claimed from a device
    counter, so which CTA runs which tile differs from launch to launch; the
    (w, Aw) partials are kept per tile and reduced in tile order, so alpha -
    and with it the whole trace and x - must not depend on the assignment.
    n = 70,644 (276 tiles, kernel-sequence loop), two solves, equal bits."""
    ne = 28
    A0 = problems.elasticity_q1(ne, E=np.exp(rng.standard_normal((ne,) * 3)))
    A = rcg.SparseSpdMatrix(A0.n, A0.row_offsets, A0.col_indices, A0.values, validate=False)
    h = A.device_csr().struct
    assert h.dia_count == 14 and h.dia_block == 3 and A.n > 49152
    b = rng.standard_normal(A.n)
    cfg = rcg.SolveConfig(tol=1e-8, max_iters=120)
    outs = []
    for _ in range(3):
        x, tr = rcg.apcg_solve(A, rcg.Preconditioner.jacobi(A), rcg.build_deflation(A, np.zeros((A.n, 0))), b, cfg)
        outs.append((np.asarray(x).copy(), np.asarray(tr.alphas).copy(), np.asarray(tr.residual_norms).copy()))
    for x, al, rn in outs[1:]:
        assert np.array_equal(x, outs[0][0]) and np.array_equal(al, outs[0][1]) and np.array_equal(rn, outs[0][2])


@pytest.mark.parametrize("count,dtype", [(5_000_003, np.float64), (9_000_001, np.int32), (33_554_432 // 8, np.float64)])
def test_pinned_staged_upload_is_exact(count, dtype):
    """core.h2d (pinned-ring upload used for large CSR arrays) is a plain copy."""
    from paper_1301_7530_b200 import core
    rng = np.random.default_rng(count)
    a = rng.standard_normal(count).astype(dtype) if dtype == np.float64 else \
        rng.integers(-2 ** 31, 2 ** 31 - 1, count, dtype=np.int64).astype(np.int32)
    d = core.h2d(a)
    assert d.is_cuda and d.dtype == getattr(__import__("torch"), str(a.dtype))
    np.testing.assert_array_equal(d.cpu().numpy(), a)
