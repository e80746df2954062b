"""Sequence-level parity at the BASELINE configurations (reference
``run_sequence``, ``pkg/src/recycg/recycle.py:178-238``).

Golden vectors come from running the reference itself in the build container
(``tests/golden/make_golden.py``: ``reduced``, ``config2``, ``accept6``;
benchmark ``clust10`` from round 1).  Bars (BASELINE.json north star):

* per-system iterations within +-2 %;
* n_c history exact, or - at the first system where the selected count
  differs - the differing Ritz values' own stagnation ratios lie inside the
  selection band [eps/100, 100 eps] (there the reference
  itself flips between BLAS thread counts); after such a flip the two
  sequences carry different bases, so n_c may differ by the flipped count
  until the next restart;
* solutions (systems 0, 1 and the last; a seeded index sample at large n)
  within relative 1e-8 while the n_c histories agree;
* selected Ritz values: every value selected on both sides agrees to relative
  1e-8; a value selected on one side only must be a threshold flip (its
  stagnation ratio inside the band) or a re-found deflated eigenvalue (equal
  to a value already in the augmentation basis: with a nearly invariant C
  those reappear only through rounding, on either side).
"""
import json
import math

import numpy as np
import pytest

import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems
from paper_1301_7530_b200 import recycle as rmod
from paper_1301_7530_b200.core import to_dev, tridiag_eigvals_device
from oracle import recycg_oracle as orc

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _close(a, b):
    return abs(a - b) <= max(1, math.ceil(0.02 * b))


def _sample_idx(n, count=16384, seed=7):
    # same index sample as tests/golden/make_golden.py::_sample_idx
    rng = np.random.Generator(np.random.Philox(seed))
    return np.sort(rng.choice(n, size=min(n, count), replace=False))


def _stagnation_ratios(cur, prev):
    """ritz.py:122-126 as a ratio per value (the smaller one-sided test)."""
    m = len(cur)
    r = np.full(m, np.inf)
    for j in range(m - 1):
        r[j] = min(r[j], abs(cur[j] - prev[j]) / abs(cur[j]))
        r[j + 1] = min(r[j + 1], abs(cur[j + 1] - prev[j]) / abs(cur[j + 1]))
    return r


class Spy:
    """Records each system's solution and selected Ritz values (with their
    stagnation ratios) by wrapping the module-level seams run_sequence calls
    (the same seams the reference exposes, recycle.py:204, :218)."""

    def __init__(self, monkeypatch, keep_x=(), sample=None):
        self.x, self.sel, self.ratios, self.k = {}, {}, {}, -1
        real_solve, real_select = rmod.apcg_solve, rmod.select_spectrum

        def solve(A, M, D, b, cfg):
            x, tr = real_solve(A, M, D, b, cfg)
            self.k += 1
            if self.k in keep_x:
                xh = x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)
                self.x[self.k] = xh if sample is None else xh[sample]
            return x, tr

        def select(trace, strategy):
            spec = real_select(trace, strategy)
            self.sel[self.k] = spec.values[spec.converged_mask].copy()
            view = rcg.lanczos_from_trace(trace)
            if view.m >= 2:
                T = view.tridiag.truncated(view.m - 1)
                if T.m == 1:
                    prev = T.diag.copy()
                else:
                    prev = tridiag_eigvals_device(to_dev(T.diag)[0], to_dev(T.offdiag)[0]).cpu().numpy()
                self.ratios[self.k] = (spec.values.copy(), _stagnation_ratios(spec.values, prev))
            return spec

        monkeypatch.setattr(rmod, "apcg_solve", solve)
        monkeypatch.setattr(rmod, "select_spectrum", select)


PAIR = 1e-7     # a selected value pairs with the other side's value within this relative distance


def _band_explained(spy, k, ref_vals, eps, recycled=()):
    """Every Ritz value selected on one side only at system k is explained:
    * a threshold flip - its stagnation ratio (ours) lies inside
      [eps/100, 100 eps], or
    * a re-found deflated eigenvalue - it equals (rel 1e-8) a Ritz value that
      is already in the augmentation basis (selected earlier in this restart
      epoch).  With C nearly invariant those eigenvalues are projected out in
      exact arithmetic and reappear in the Krylov space only through rounding,
      so which of them a run re-finds is rounding-decided on both sides (seen
      at config 2, fixed A: system 1 re-finds one of system 0's 46 values)."""
    ours = spy.sel.get(k, np.empty(0))
    ref_vals = np.asarray(ref_vals)
    recycled = np.asarray(recycled, dtype=np.float64)
    vals, ratio = spy.ratios[k]
    diff = [v for v in ours if not np.any(np.abs(ref_vals - v) <= PAIR * abs(v))]
    diff += [v for v in ref_vals if not np.any(np.abs(ours - v) <= PAIR * abs(v))]
    for v in diff:
        if len(recycled) and np.any(np.abs(recycled - v) <= 1e-8 * abs(v)):
            continue
        j = int(np.argmin(np.abs(vals - v)))
        if abs(vals[j] - v) > 1e-6 * abs(v):
            return False           # no Ritz value of ours near it at all: not a threshold flip
        if not (eps / 100 <= ratio[j] <= 100 * eps):
            return False
    return True


def _check_selected(spy, k, ref_vals, eps, recycled=()):
    """Selected Ritz values of system k: every pair (same value on both sides,
    within PAIR) agrees to rel 1e-8; values selected on one side only must be
    explained (``_band_explained``)."""
    ref_vals = np.asarray(ref_vals)
    ours = spy.sel.get(k, np.empty(0))
    for v in ref_vals:
        if len(ours) == 0:
            break
        j = int(np.argmin(np.abs(ours - v)))
        if abs(ours[j] - v) <= PAIR * abs(v):
            assert abs(ours[j] - v) <= 1e-8 * abs(v), (k, v, ours[j])
    assert _band_explained(spy, k, ref_vals, eps, recycled), \
        (k, sorted(set(np.round(ours, 9)) ^ set(np.round(ref_vals, 9))))


def check_sequence(rep, spy, g, eps, sols=None, sol_prefix=None, n=None):
    """Apply the bars above; returns the index of the first n_c divergence
    (len(records) when the histories agree throughout)."""
    got_it, want_it = rep.iterations(), g["iterations"]
    got_nc, want_nc = rep.n_c_history(), g["n_c_before"]
    if g.get("aborted"):
        # The reference run itself ends in NumericalFailure("(r, z) <= 0") (c5r:
        # reorth off, lognormal E).  Which system trips it is rounding-decided
        # in the reference algorithm: the CPU oracle on the same matrices with
        # each row's entries stored in reverse order (a rounding-level change
        # of the SpMV only) aborts at system 1 instead of 9
        # (tests/test_oracle_golden.py::test_c5r_abort_index_is_rounding_decided).
        # So: our run must fail the same way, and every system solved on both
        # sides must meet the bars.
        assert rep.aborted, "the reference aborts this sequence; ours completed it"
        fails = [e for e in rep.events if e[0] == "solve_failed"]
        assert fails and "(r, z) <= 0" in str(fails[-1][-1]), rep.events
        m = min(len(got_it), len(want_it))
        assert m >= 1, (got_it, want_it)
        got_it, want_it, got_nc, want_nc = got_it[:m], want_it[:m], got_nc[:m], want_nc[:m]
    assert len(got_it) == len(want_it), (got_it, want_it)
    assert all(r.converged for r in rep.records) == all(g["converged"])
    split = len(got_nc)
    for k in range(len(got_nc)):
        if got_nc[k] != want_nc[k]:
            split = k
            break
    # iterations: +-2 % everywhere
    bad = [(k, a, b) for k, (a, b) in enumerate(zip(got_it, want_it)) if not _close(a, b)]
    assert not bad, f"iterations outside +-2 %: {bad} (n_c got {got_nc} want {want_nc})"
    if split < len(got_nc):
        # the system before the split selected a different count: band rule
        k = split - 1
        assert k >= 0, (got_nc, want_nc)
        prior = [v for kk in range(k) if all(want_nc[q] != 0 for q in range(kk + 1, k + 1))
                 for v in g["selected_ritz_values"][kk]]
        assert _band_explained(spy, k, g["selected_ritz_values"][k], eps, prior), \
            (k, spy.sel.get(k), g["selected_ritz_values"][k])
        # later systems: the flipped count persists until the next restart
        for kk in range(split, len(got_nc)):
            assert abs(got_nc[kk] - want_nc[kk]) <= 3 or got_nc[kk] == 0 or want_nc[kk] == 0, (got_nc, want_nc)
    # selected Ritz values while the histories agree; a threshold flip (same
    # count, different member of a near-degenerate group) changes the next
    # system's basis, so solutions are compared up to that system only
    sel_split = len(got_nc)
    recycled = []              # values selected earlier in the current restart epoch (reference side)
    for k in range(min(split, len(got_nc))):
        if k > sel_split:
            break                  # later systems recycle a different basis: no value-level claim
        if want_nc[k] == 0:
            recycled = []
        if k in spy.ratios:
            _check_selected(spy, k, g["selected_ritz_values"][k], eps, recycled)
            ours, ref = spy.sel.get(k, np.empty(0)), np.asarray(g["selected_ritz_values"][k])
            paired = all(np.any(np.abs(ours - v) <= PAIR * abs(v)) for v in ref) and len(ours) == len(ref)
            if not paired and sel_split == len(got_nc):
                sel_split = k
        recycled += list(g["selected_ritz_values"][k])
    # solutions while the histories agree
    if sols is not None:
        for key in sols.files:
            if not key.startswith(sol_prefix):
                continue
            k = int(key.split("__x")[1])
            if k >= split or k > sel_split:
                continue
            want = sols[key]
            got = spy.x[k]
            if len(want) < len(got):
                got = got[_sample_idx(n)]
            assert np.linalg.norm(got - want) <= 1e-8 * np.linalg.norm(want), (key, np.linalg.norm(got - want) /
                                                                            np.linalg.norm(want))
    return min(split, sel_split + 1)


# ---------------------------------------------------------------------------
# reduced analogs of configs 2-5, full sequences


REDUCED = json.loads((GOLDEN / "reduced_sequences.json").read_text()) if (GOLDEN / "reduced_sequences.json").exists() \
    else {}


@pytest.mark.parametrize("name", ["c2r", "c3r", "c4r_on", "c4r_off", "c5r"])
def test_reduced_config_sequence_matches_reference(name, monkeypatch):
    if name not in REDUCED:
        pytest.skip(f"golden {name} not generated")
    g = REDUCED[name]
    systems, st = problems.config_systems(g["config"], reduced=True)
    systems = list(systems)
    last = len(systems) - 1
    spy = Spy(monkeypatch, keep_x=(0, 1, last))
    cfg = rcg.SolveConfig(tol=g["tol"], max_iters=5000, reorthogonalize=g["reorthogonalize"])
    strat = rcg.RecycleStrategy("srks", epsilon=g["epsilon"], nc_limit=g["nc_limit"])
    rep = rcg.run_sequence(iter(systems), rcg.Preconditioner.jacobi, strat, cfg)
    sols = np.load(GOLDEN / "reduced_solutions.npz")
    check_sequence(rep, spy, g, g["epsilon"], sols, f"{name}__", systems[0][0].n)


# ---------------------------------------------------------------------------
# config 2 at full size (n = 811,200), systems 0 and 1 (system 1 recycles)


def test_config2_full_size_first_two_systems(monkeypatch):
    path = GOLDEN / "config2_full.json"
    if not path.exists():
        pytest.skip("config-2 golden not generated")
    g = json.loads(path.read_text())
    xs = np.load(GOLDEN / "config2_full_xsample.npz")
    count = len(g["iterations"])
    systems = list(problems.elasticity_sequence(64, count, kind="fixed", device=True))
    A = systems[0][0]
    assert A.n == g["n"] and A.nnz == g["nnz"]
    spy = Spy(monkeypatch, keep_x=tuple(range(count)), sample=xs["idx"])
    cfg = rcg.SolveConfig(tol=1e-8, max_iters=20000)
    rep = rcg.run_sequence(iter(systems), rcg.Preconditioner.jacobi,
                           rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=61), cfg)
    import os
    dump = os.environ.get("RCG_PARITY_DUMP")
    if dump:   # diagnostics: our selected values and stagnation ratios per system
        with open(dump, "w") as f:
            json.dump({"iterations": rep.iterations(), "n_c": rep.n_c_history(),
                       "sel": {k: list(map(float, v)) for k, v in spy.sel.items()},
                       "ratios": {k: [list(map(float, a)), list(map(float, b))] for k, (a, b) in spy.ratios.items()}},
                      f)
    split = check_sequence(rep, spy, g, 1e-10)
    assert rep.n_c_history()[1] > 30          # system 1 really recycles (reference: 46)
    for k in range(min(split, count)):
        want = xs[f"x{k}"]
        assert np.linalg.norm(spy.x[k] - want) <= 1e-8 * np.linalg.norm(want), k


# ---------------------------------------------------------------------------
# srks_cluster through the device path (benchmark, 8 systems, tol 1e-6)


def test_benchmark_cluster_strategy_matches_reference_golden(monkeypatch):
    g = json.loads((GOLDEN / "benchmark_srks.json").read_text())["clust10"]
    systems = list(problems.generate_diffusion_sequence(problems.benchmark_spec(seed=0), len(g["iterations"])))
    cfg = rcg.SolveConfig(tol=1e-6, max_iters=3000)
    calls = []
    real = rmod.cluster_filter

    def spy_cf(values, mc):
        calls.append((len(values), mc))
        return real(values, mc)

    monkeypatch.setattr(rmod, "cluster_filter", spy_cf)
    rep = rcg.run_sequence(iter(systems), rcg.Preconditioner.jacobi,
                           rcg.RecycleStrategy("srks_cluster", epsilon=1e-10), cfg)
    assert calls, "cluster filter never ran"
    got, want = rep.iterations(), g["iterations"]
    assert all(_close(a, b) for a, b in zip(got, want)), (got, want)
    assert rep.n_c_history() == g["n_c_before"], (rep.n_c_history(), g["n_c_before"])


def test_cluster_filter_device_kats():
    # reference tests/test_ritz.py:221-240
    assert rcg.cluster_filter([100.0, 10.2, 10.1, 10.0, 9.9, 1.0], min_cluster=3) == [0, 5]
    assert rcg.cluster_filter([2.0, 2.0, 2.0, 2.0], min_cluster=2) == []
    v = list(np.linspace(10.0, 1.0, 8))
    assert rcg.cluster_filter(v, 3) == rcg.cluster_filter(v, 3)
    vals = np.sort(np.random.default_rng(0).uniform(1, 100, 30))[::-1]
    assert rcg.cluster_filter(vals, 6) == orc.cluster_filter(vals, 6)
    assert rcg.cluster_filter(vals * 7.5, 6) == rcg.cluster_filter(vals, 6)


@pytest.mark.parametrize("seed", range(12))
def test_cluster_filter_device_matches_oracle_random(seed):
    """Random spectra incl. exact ties and repeated gaps (tie order) and
    sizes past one CTA's worth of splits."""
    rng = np.random.default_rng(100 + seed)
    m = int(rng.choice([2, 3, 5, 17, 64, 300, 900]))
    kind = seed % 3
    if kind == 0:
        vals = np.sort(rng.lognormal(0, 2, m))[::-1]
    elif kind == 1:      # equal gaps everywhere: every split ties on error
        vals = np.linspace(50.0, 1.0, m)
    else:                # clustered middle with repeated values
        vals = np.sort(np.concatenate([rng.uniform(9.9, 10.1, m - m // 4), rng.uniform(1, 100, m // 4)]))[::-1]
        vals[1::7] = vals[0::7][:len(vals[1::7])]
        vals = np.sort(vals)[::-1]
    for mc in sorted({1, 2, max(1, m // 5), max(1, m // 2), m}):
        assert rcg.cluster_filter(vals, mc) == orc.cluster_filter(vals, mc), (m, mc)


# ---------------------------------------------------------------------------
# reference acceptance criterion 6 (pkg/tests/test_acceptance.py:226-266)


ACC6 = json.loads((GOLDEN / "acceptance6.json").read_text()) if (GOLDEN / "acceptance6.json").exists() else None


@pytest.mark.skipif(ACC6 is None, reason="acceptance-6 golden not generated")
def test_acceptance_criterion_6_sequence_benchmark():
    """The 40-system inclusion benchmark: none / trks / srks(1e-14) at tol
    1e-3 and trks / srks(1e-14) at tol 1e-6, with the criterion's own
    conditions and frozen margins, plus the reference's per-system lists for
    none and trks (TRKS at 1e-6 grows the basis to n_c ~ 1.6 k: the blocked
    coarse Cholesky path)."""
    import time
    margins = ACC6["margins"]
    t0 = time.time()
    systems = list(problems.generate_diffusion_sequence(problems.benchmark_spec(seed=0), 40))

    def run(strategy, tol):
        return rcg.run_sequence(iter(systems), rcg.Preconditioner.jacobi, strategy,
                                rcg.SolveConfig(tol=tol, max_iters=3000))

    rep = {"none": run(rcg.RecycleStrategy("none"), 1e-3), "trks": run(rcg.RecycleStrategy("trks"), 1e-3),
           "srks": run(rcg.RecycleStrategy("srks", epsilon=1e-14), 1e-3)}
    avg = {k: np.mean(r.iterations()[1:]) for k, r in rep.items()}
    margin = 1.0 - margins["ordering_margin"]
    assert avg["trks"] <= margin * avg["srks"], avg
    assert avg["srks"] <= margin * avg["none"], avg
    assert all(all(rec.converged for rec in r.records) for r in rep.values())
    ncs = rep["trks"].n_c_history()
    assert np.diff(ncs[-11:]).mean() <= margins["trks_plateau_increment_ratio"] * np.diff(ncs[1:12]).mean()
    trks6 = run(rcg.RecycleStrategy("trks"), 1e-6)
    srks6 = run(rcg.RecycleStrategy("srks", epsilon=1e-14), 1e-6)
    ncs_t = trks6.n_c_history()
    assert all(b > a for a, b in zip(ncs_t[-10:], ncs_t[-9:])), ncs_t
    ncs_s = srks6.n_c_history()
    assert max(ncs_s[30:40]) <= margins["srks_plateau_factor"] * max(ncs_s[10:20]), ncs_s
    assert time.time() - t0 < margins["runtime_seconds_budget"]
    # per-system lists against the reference run (none exact; trks +-2 % and
    # n_c within 2 %: normalized directions make TRKS rounding-sensitive)
    g3, g6 = ACC6["tol0.001"], ACC6["tol1e-06"]
    assert rep["none"].iterations() == g3["none"]["iterations"]
    for got, want in [(rep["trks"], g3["trks"]), (trks6, g6["trks"])]:
        assert all(_close(a, b) for a, b in zip(got.iterations(), want["iterations"])), \
            (got.iterations(), want["iterations"])
        assert all(abs(a - b) <= max(2, 0.02 * b) for a, b in zip(got.n_c_history(), want["n_c_before"])), \
            (got.n_c_history(), want["n_c_before"])
    assert max(ncs_t) > 1500                  # the large-n_c coarse path really ran


# ---------------------------------------------------------------------------
# TRKS with a high-kappa coarse matrix: config 1 at tol 1e-8,
# n_c grows 0 -> 723; the coarse solve applies the explicit G^-1 = L^-T L^-1


def test_trks_config1_high_kappa_coarse_matches_reference(monkeypatch):
    path = GOLDEN / "trks_config1.json"
    if not path.exists():
        pytest.skip("trks golden not generated")
    g = json.loads(path.read_text())
    sols = np.load(GOLDEN / "trks_config1_solutions.npz")
    count = len(g["iterations"])
    systems = problems.shifted_laplacian_sequence(count=count)
    spy = Spy(monkeypatch, keep_x=tuple(range(count)))
    for path_kind in ("persistent", "multi_kernel"):
        if path_kind == "multi_kernel":
            monkeypatch.setenv("RCG_SMALL_N", "0")
        spy.k = -1
        rep = rcg.run_sequence(iter(systems), rcg.Preconditioner.jacobi, rcg.RecycleStrategy("trks"),
                               rcg.SolveConfig(tol=1e-8, max_iters=2000))
        got, want = rep.iterations(), g["iterations"]
        assert all(_close(a, b) for a, b in zip(got, want)), (path_kind, got, want)
        assert all(abs(a - b) <= max(2, 0.02 * b) for a, b in zip(rep.n_c_history(), g["n_c_before"])), \
            (path_kind, rep.n_c_history(), g["n_c_before"])
        for k in range(count):
            want_x = sols[f"x{k}"]
            assert np.linalg.norm(spy.x[k] - want_x) <= 1e-8 * np.linalg.norm(want_x), (path_kind, k)
