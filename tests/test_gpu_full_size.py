"""Parity at BASELINE's full sizes (SURVEY.md §8(c) "fixed-window traces"):
the first K iterations of system 0 of config 2 (Q1 elasticity 64^3, full
reorth) and config 4 (7-point 256^3, reorth off) through the production
stream formats (3x3 block-DIA / scalar DIA SpMV) against the CPU oracle on
the same bytes.  alpha, beta, ||r|| within 1e-9 relative (the north star's
bars are 1e-8 on converged quantities; K iterations of rounding-level
differences stay far below that) and x after K iterations within 1e-9."""
import numpy as np
import pytest

import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems
from oracle import recycg_oracle as orc

pytestmark = pytest.mark.gpu

K = 30


def _window(A, b, reorth, expect_dia):
    assert A.device_csr().struct.dia_count == expect_dia
    cfg = rcg.SolveConfig(tol=1e-12, max_iters=K, reorthogonalize=reorth)
    D = rcg.build_deflation(A, np.zeros((A.n, 0)))
    x, tr = rcg.apcg_solve(A, rcg.Preconditioner.jacobi(A), D, b, cfg)
    xo, tro = orc.apcg_solve(A, 1.0 / orc.diagonal(A), orc.build_deflation(A, np.zeros((A.n, 0))), b, 1e-12, K,
                             reorthogonalize=reorth)
    assert tr.iterations == tro.iterations == K and not tr.converged
    for got, want in ((tr.alphas, tro.alphas), (tr.betas, tro.betas), (tr.residual_norms, tro.residual_norms)):
        got, want = np.asarray(got), np.asarray(want)
        assert got.shape == want.shape
        np.testing.assert_allclose(got, want, rtol=1e-9)
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) < 1e-9


def test_config2_window_full_reorth(monkeypatch):
    monkeypatch.delenv("RCG_DIA_SMALL", raising=False)   # production format choice
    A, b = next(problems.elasticity_sequence(64, 1, kind="fixed", device=True))
    _window(A, b, True, 14)
    A.release_device()


def test_config4_window_no_reorth(monkeypatch):
    monkeypatch.delenv("RCG_DIA_SMALL", raising=False)
    A, b = next(problems.lognormal_diffusion_sequence(256, 1, device=True))
    _window(A, b, False, 4)
    A.release_device()


def test_config3_window_softened_operator(monkeypatch):
    """96^3 elasticity, third system of the softening sequence (E scaled
    inside a sphere: non-constant block values on the DIA diagonals)."""
    monkeypatch.delenv("RCG_DIA_SMALL", raising=False)
    it = problems.elasticity_sequence(96, 3, kind="softening", device=True)
    for _ in range(3):
        A, b = next(it)
    _window(A, b, True, 14)
    A.release_device()
