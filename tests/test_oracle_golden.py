"""Pin the CPU oracle before trusting it (runs without a GPU).

(a) the reference's own frozen golden fixture: pkg/tests/fixtures/
    benchmark_pilot.json none/trks iteration lists (SURVEY.md §0 finding 2:
    these reproduce exactly; srks14 does not and is not used);
(b) vectors produced by running the reference itself in the build container
    (tests/golden/make_golden.py): small solves, config-1 sequence, the
    benchmark SRKS sequences, the elasticity analog;
(c) generator pins: the seeded inputs still hash to the bytes the reference
    was run on.
"""
import hashlib
import json

import numpy as np
import pytest

from paper_1301_7530_b200 import problems
from oracle import recycg_oracle as orc
from conftest import GOLDEN

SMALL = np.load(GOLDEN / "small_solves.npz")
NAMES = [str(s) for s in SMALL["names"]]


def _case(name):
    return {k.split("__", 1)[1]: SMALL[k] for k in SMALL.files if k.startswith(name + "__")}


def _sha(A):
    h = hashlib.sha256()
    h.update(np.asarray(A.row_offsets, dtype=np.int64).tobytes())
    h.update(np.asarray(A.col_indices, dtype=np.int64).tobytes())
    h.update(np.asarray(A.values, dtype=np.float64).tobytes())
    return h.hexdigest()


class _Dense:
    def __init__(self, G):
        n = G.shape[0]
        self.n = n
        self.row_offsets = np.arange(n + 1) * n
        self.col_indices = np.tile(np.arange(n), n)
        self.values = G.ravel()


@pytest.mark.parametrize("name", NAMES)
def test_oracle_small_solves_match_reference(name):
    c = _case(name)
    A = _Dense(c["dense"])
    pc = str(c["precond"])
    inv = None if pc == "identity" else (1.0 / orc.diagonal(A) if pc == "jacobi" else 1.0 / c["user_diag"])
    D = orc.build_deflation(A, c["C"])
    x, tr = orc.apcg_solve(A, inv, D, c["b"], float(c["tol"]), int(c["max_iters"]), bool(c["reorth"]),
                           True, bool(c["store"]))
    assert tr.iterations == int(c["iterations"])
    assert tr.converged == bool(c["converged"])
    # early coefficients to rounding; later ones carry BLAS-layout noise
    # (reference stores W in a strided C-order buffer, the oracle contiguous)
    np.testing.assert_allclose(tr.alphas[:10], c["alphas"][:10], rtol=1e-12)
    half = max(10, len(tr.alphas) // 2)
    np.testing.assert_allclose(tr.alphas[:half], c["alphas"][:half], rtol=1e-6)
    np.testing.assert_allclose(x, c["x"], rtol=0, atol=1e-10 * np.linalg.norm(c["x"]))
    if "ritz_values" in c:
        spec = orc.select_spectrum(tr, 1e-10)
        # selected (stagnated) values to 1e-9; interior unconverged ones are
        # roundoff-driven and differ between any two BLAS layouts
        sel = c["ritz_mask"]
        np.testing.assert_allclose(spec.values[sel], c["ritz_values"][sel], rtol=1e-9)
        assert np.array_equal(spec.converged_mask, c["ritz_mask"])
        blk, _ = orc.srks_block(spec)
        np.testing.assert_allclose(np.abs(blk), np.abs(c["ritz_block"]), rtol=1e-6, atol=1e-9)


def test_config1_generator_pin():
    g = json.loads((GOLDEN / "config1_sequence.json").read_text())
    systems = problems.shifted_laplacian_sequence()
    assert [_sha(A) for A, _ in systems] == g["matrix_sha256"]
    assert [hashlib.sha256(b.tobytes()).hexdigest() for _, b in systems] == g["rhs_sha256"]


def test_benchmark_generator_pin():
    g = json.loads((GOLDEN / "benchmark_srks.json").read_text())
    systems = list(problems.generate_diffusion_sequence(problems.benchmark_spec(seed=0), 8))
    assert [_sha(A) for A, _ in systems] == g["matrix_sha256"]


def test_elasticity_generator_pin():
    g = json.loads((GOLDEN / "elasticity8_sequence.json").read_text())
    A = problems.elasticity_q1(8)
    assert _sha(A) == g["matrix_sha256"]


def test_oracle_config1_sequence_matches_reference():
    g = json.loads((GOLDEN / "config1_sequence.json").read_text())
    res = orc.run_sequence(problems.shifted_laplacian_sequence(), strategy="srks", epsilon=1e-10, nc_limit=21,
                           tol=1e-8, max_iters=2000)
    assert res.iterations == g["iterations"]
    assert res.n_c_before == g["n_c_before"]
    for got, want in zip(res.selected_values, g["selected_ritz_values"]):
        np.testing.assert_allclose(got, want, rtol=1e-10)


def test_oracle_benchmark_srks_matches_reference():
    g = json.loads((GOLDEN / "benchmark_srks.json").read_text())
    systems = list(problems.generate_diffusion_sequence(problems.benchmark_spec(seed=0), 8))
    for name, kind, eps in [("srks10", "srks", 1e-10), ("srks6", "srks", 1e-6), ("clust10", "srks_cluster", 1e-10)]:
        res = orc.run_sequence(systems, strategy=kind, epsilon=eps, tol=1e-6, max_iters=3000)
        assert res.iterations == g[name]["iterations"], name
        assert res.n_c_before == g[name]["n_c_before"], name


def test_oracle_elasticity_sequence_matches_reference():
    g = json.loads((GOLDEN / "elasticity8_sequence.json").read_text())
    systems = list(problems.elasticity_sequence(8, 4, kind="fixed"))
    res = orc.run_sequence(systems, strategy="srks", epsilon=1e-10, nc_limit=61, tol=1e-8, max_iters=3000)
    assert res.iterations == g["iterations"]
    assert res.n_c_before == g["n_c_before"]


@pytest.mark.parametrize("strategy", ["none", "trks"])
def test_oracle_pilot_fixture_tol1e3(strategy):
    """The reference's frozen golden fixture, all 40 systems (exact)."""
    g = json.loads((GOLDEN / "benchmark_pilot_none_trks.json").read_text())["runs"]["tol1e-3"][strategy]
    systems = list(problems.generate_diffusion_sequence(problems.benchmark_spec(seed=0), 40))
    res = orc.run_sequence(systems, strategy=strategy, tol=1e-3, max_iters=3000)
    assert res.iterations == g["iterations"]
    if "n_c_before" in g:
        assert res.n_c_before == g["n_c_before"]


def test_oracle_pilot_fixture_trks_tol1e6_prefix():
    g = json.loads((GOLDEN / "benchmark_pilot_none_trks.json").read_text())["runs"]["tol1e-6"]["trks"]
    systems = list(problems.generate_diffusion_sequence(problems.benchmark_spec(seed=0), 10))
    res = orc.run_sequence(systems, strategy="trks", tol=1e-6, max_iters=3000)
    assert res.iterations == g["iterations"][:10]


def test_c5r_abort_index_is_rounding_decided():
    """The reduced config-5 analog (lognormal-E softening elasticity 16^3,
    reorth off) ends in NumericalFailure("(r, z) <= 0") in the reference run
    (golden c5r: at system 9).  Which system trips it depends on rounding
    alone: the same reference algorithm (this oracle) on the same matrices,
    with each CSR row's entries stored in reverse order - scipy's csr_matvec
    sums in stored order, so only the SpMV's rounding changes - aborts at an
    earlier system.  The GPU parity test therefore pins the failure mode and
    the systems solved on both sides, not the abort index."""
    g = json.loads((GOLDEN / "reduced_sequences.json").read_text())["c5r"]
    assert g["aborted"] and g["events"][-1][0] == "solve_failed" and int(g["events"][-1][1]) == 9
    systems, st = problems.config_systems(5, reduced=True)

    class Rev:
        def __init__(self, A):
            ro = np.asarray(A.row_offsets)
            # reverse every row: entry k of row i moves to ro[i] + ro[i+1] - 1 - k
            rows = np.repeat(np.arange(A.n), np.diff(ro))
            src = ro[rows] + ro[rows + 1] - 1 - np.arange(len(rows))
            self.n, self.nnz, self.row_offsets = A.n, A.nnz, ro
            self.col_indices = np.asarray(A.col_indices)[src]
            self.values = np.asarray(A.values)[src]

    rep = orc.run_sequence(((Rev(A), b) for A, b in systems), "srks", epsilon=st["epsilon"],
                           nc_limit=st["nc_limit"], tol=st["tol"], max_iters=5000, reorthogonalize=False)
    assert rep.aborted
    kind, k, msg = rep.events[-1]
    assert kind == "solve_failed" and "(r, z) <= 0" in msg
    assert k < 9, (k, rep.iterations)
