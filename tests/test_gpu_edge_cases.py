"""Edge cases of the B200 path against the CPU oracle / reference semantics:
zero right-hand side, n = 1, max_iters = 1, full augmentation, reorth off,
no trace capture, identity preconditioner, the n_c > 64 coarse path, and
contract violations raised before any device work."""
import numpy as np
import pytest

import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems
from oracle import recycg_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["persistent", "multi_kernel"])
def solve_loop(request, monkeypatch):
    """Edge cases through both solve loops (persistent cooperative kernel for
    these small operators by default; the kernel sequence with RCG_SMALL_N=0)."""
    if request.param == "multi_kernel":
        monkeypatch.setenv("RCG_SMALL_N", "0")
    return request.param


def _spd(n, rng, cond=100.0):
    return rcg.SparseSpdMatrix.from_dense(problems.random_spd(n, rng, cond), keep_zeros=True)


def test_zero_rhs_converges_immediately(rng):
    A = _spd(12, rng)
    x, tr = rcg.apcg_solve(A, rcg.Preconditioner.jacobi(A), rcg.build_deflation(A, np.zeros((12, 0))),
                           np.zeros(12), rcg.SolveConfig())
    assert tr.converged and tr.iterations == 0 and tr.residual_norms == [0.0]
    assert np.all(x == 0.0)


def test_single_unknown():
    A = rcg.SparseSpdMatrix.from_dense(np.array([[4.0]]))
    x, tr = rcg.apcg_solve(A, rcg.Preconditioner.identity(), rcg.build_deflation(A, np.zeros((1, 0))),
                           np.array([2.0]), rcg.SolveConfig(tol=1e-10))
    assert tr.converged and tr.iterations == 1
    np.testing.assert_allclose(x, [0.5])


def test_max_iters_one_and_trailing_beta(rng):
    A = _spd(30, rng, 1e3)
    b = rng.standard_normal(30)
    x, tr = rcg.apcg_solve(A, rcg.Preconditioner.jacobi(A), rcg.build_deflation(A, np.zeros((30, 0))), b,
                           rcg.SolveConfig(tol=1e-12, max_iters=1))
    xo, to = orc.apcg_solve(A, 1.0 / orc.diagonal(A), orc.build_deflation(A, np.zeros((30, 0))), b, 1e-12, 1)
    assert not tr.converged and tr.iterations == 1
    assert len(tr.betas) == len(to.betas) == 1          # a cap-stopped run keeps its trailing beta
    np.testing.assert_allclose(tr.alphas, to.alphas, rtol=1e-12)
    np.testing.assert_allclose(x, xo, rtol=1e-12, atol=1e-14)


def test_reorth_off_and_no_capture_match_oracle(rng):
    # without reorthogonalization the iteration count of this n=60, cond 1e3
    # system depends on rounding (> n iterations), so the SpMV must sum rows in
    # the oracle's scalar-CSR order: disable the (dense => 3x3-block) BSR3 copy
    A0 = _spd(60, rng, 1e3)
    A = rcg.SparseSpdMatrix(A0.n, A0.row_offsets, A0.col_indices, A0.values, validate=False, use_block3=False)
    b = rng.standard_normal(60)
    C = rng.standard_normal((60, 5))
    cfg = rcg.SolveConfig(tol=1e-8, max_iters=500, reorthogonalize=False, trace_capture=False)
    x, tr = rcg.apcg_solve(A, rcg.Preconditioner.jacobi(A), rcg.build_deflation(A, C), b, cfg)
    xo, to = orc.apcg_solve(A, 1.0 / orc.diagonal(A), orc.build_deflation(A, C), b, 1e-8, 500,
                            reorthogonalize=False, trace_capture=False)
    assert abs(tr.iterations - to.iterations) <= 1
    assert len(tr.z_history) == 0
    np.testing.assert_allclose(tr.alphas[:8], to.alphas[:8], rtol=1e-10)
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)


def test_large_basis_coarse_path(rng):
    """n_c > 64: the separate coarse-solve kernel and the >128 Cholesky path."""
    n = 400
    A = _spd(n, rng, 1e4)
    b = rng.standard_normal(n)
    C = rng.standard_normal((n, 150))
    cfg = rcg.SolveConfig(tol=1e-10, max_iters=1000)
    D = rcg.build_deflation(A, C)
    x, tr = rcg.apcg_solve(A, rcg.Preconditioner.jacobi(A), D, b, cfg)
    Do = orc.build_deflation(A, C)
    np.testing.assert_allclose(D.coarse_factor, Do.L, rtol=1e-8, atol=1e-10 * np.abs(Do.L).max())
    xo, to = orc.apcg_solve(A, 1.0 / orc.diagonal(A), Do, b, 1e-10, 1000)
    assert abs(tr.iterations - to.iterations) <= max(1, 0.02 * to.iterations)
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)
    np.testing.assert_allclose(C.T @ (A @ D.project(b)), 0.0, atol=1e-8 * np.linalg.norm(b) * np.abs(C).max())


def test_contract_violations_before_device_work(rng):
    A = _spd(5, rng)
    D = rcg.build_deflation(A, np.zeros((5, 0)))
    with pytest.raises(rcg.ContractViolation):
        rcg.apcg_solve(A, rcg.Preconditioner.identity(), D, np.ones(4), rcg.SolveConfig())
    B = _spd(6, rng)
    with pytest.raises(rcg.ContractViolation):
        rcg.apcg_solve(B, rcg.Preconditioner.identity(), D, np.ones(6), rcg.SolveConfig())
    with pytest.raises(rcg.ContractViolation):
        rcg.SolveConfig(krylov_cap=0)


def test_numerical_failure_messages(rng):
    """Indefinite preconditioner: the reference's (r, z) <= 0 message; an
    indefinite operator: (w, A w) <= 0 (solver.py:229-230, :244-245)."""
    A = _spd(10, rng)
    bad = rcg.Preconditioner("user_diagonal", inv_diag=-np.ones(10))
    with pytest.raises(rcg.NumericalFailure, match=r"\(r, z\) <= 0"):
        rcg.apcg_solve(A, bad, rcg.build_deflation(A, np.zeros((10, 0))), rng.standard_normal(10),
                       rcg.SolveConfig())
    G = np.diag([1.0, -1.0, 2.0])
    Aind = rcg.SparseSpdMatrix(3, np.array([0, 1, 2, 3]), np.array([0, 1, 2]), np.array([1.0, -1.0, 2.0]),
                               validate=False)
    with pytest.raises(rcg.NumericalFailure, match=r"\(w, A w\) <= 0"):
        rcg.apcg_solve(Aind, rcg.Preconditioner.identity(), rcg.build_deflation(Aind, np.zeros((3, 0))),
                       np.array([0.0, 1.0, 0.0]), rcg.SolveConfig())


def test_device_tensors_pass_through(rng):
    import torch
    A = _spd(40, rng)
    b = torch.tensor(rng.standard_normal(40), device="cuda")
    x, tr = rcg.apcg_solve(A, rcg.Preconditioner.jacobi(A), rcg.build_deflation(A, np.zeros((40, 0))), b,
                           rcg.SolveConfig(tol=1e-10))
    assert isinstance(x, torch.Tensor) and x.is_cuda
    np.testing.assert_allclose((A @ x.cpu().numpy()), b.cpu().numpy(), atol=1e-8 * float(b.norm()))


def test_no_pool_buffer_overruns_under_guard():
    """Every solve-path kernel variant (BSR3 / CSR SpMV, SRKS / TRKS, reorth
    on / off, krylov_cap, the n_c > 64 coarse kernel) run with guarded pool
    and scratch buffers (RCG_POOL_GUARD: canary zone behind every buffer,
    checked on release): no kernel writes past the end of its buffers."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, RCG_POOL_GUARD="1")
    out = subprocess.run([sys.executable, str(root / "tools" / "memcheck_seq.py")], env=env, cwd=root,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "GUARD_VIOLATIONS 0" in out.stdout, out.stdout[-2000:] + out.stderr[-2000:]
