"""Generate golden vectors by running the REFERENCE package (read-only import).

Run in the build container only (``/root/reference`` does not exist on the GPU
box):  ``python tests/golden/make_golden.py``.  Inputs come from this repo's
seeded generators (same host CSR bytes the GPU path consumes); their sha256 is
stored so the tests can prove the generator still emits the bytes the reference
was run on.  Outputs: ``tests/golden/*.npz`` / ``*.json``.
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

import recycg  # noqa: E402  (the reference)
from recycg import recycle as ref_recycle  # noqa: E402
from recycg import problems as ref_problems  # noqa: E402

from paper_1301_7530_b200 import problems  # noqa: E402


def csr_sha(A):
    h = hashlib.sha256()
    h.update(np.asarray(A.row_offsets, dtype=np.int64).tobytes())
    h.update(np.asarray(A.col_indices, dtype=np.int64).tobytes())
    h.update(np.asarray(A.values, dtype=np.float64).tobytes())
    return h.hexdigest()


def to_ref(A):
    return recycg.SparseSpdMatrix(A.n, np.asarray(A.row_offsets), np.asarray(A.col_indices),
                                  np.asarray(A.values))


def small_solve_cases():
    """Dense random SPD cases (reference conftest random_spd), C random, both
    preconditioners, reorth on/off, plus a cap-stopped run."""
    rng = np.random.Generator(np.random.Philox(2024))
    cases = {}
    specs = [
        # name, n, n_c, cond, precond, reorth, tol, max_iters, store
        ("id_noC", 40, 0, 1e3, "identity", True, 1e-10, 500, False),
        ("jac_C4", 60, 4, 1e4, "jacobi", True, 1e-10, 500, True),
        ("jac_C6_noreorth", 80, 6, 1e4, "jacobi", False, 1e-10, 500, False),
        ("user_C3", 50, 3, 1e3, "user", True, 1e-9, 500, False),
        ("cap_stop", 90, 2, 1e6, "jacobi", True, 1e-14, 7, True),
        ("big_C40", 120, 40, 1e4, "jacobi", True, 1e-10, 500, False),
    ]
    for name, n, n_c, cond, pc, reorth, tol, mi, store in specs:
        G = problems.random_spd(n, rng, cond)
        # a non-constant diagonal makes Jacobi matter
        s = rng.uniform(0.5, 2.0, n)
        G = G * np.outer(s, s)
        G = 0.5 * (G + G.T)
        A = recycg.SparseSpdMatrix.from_dense(G, keep_zeros=True)
        C = rng.standard_normal((n, n_c))
        b = rng.standard_normal(n)
        ud = rng.uniform(0.5, 4.0, n)
        if pc == "identity":
            M = recycg.Preconditioner.identity()
        elif pc == "jacobi":
            M = recycg.Preconditioner.jacobi(A)
        else:
            M = recycg.Preconditioner.user_diagonal(ud)
        D = recycg.build_deflation(A, C)
        cfg = recycg.SolveConfig(tol=tol, max_iters=mi, reorthogonalize=reorth,
                                 trace_capture=True, store_directions=store)
        x, tr = recycg.apcg_solve(A, M, D, b, cfg)
        d = dict(dense=A.to_dense(), C=C, b=b, user_diag=ud, precond=pc,
                 reorth=reorth, tol=tol, max_iters=mi, store=store,
                 x=x, alphas=np.array(tr.alphas), betas=np.array(tr.betas),
                 rz=np.array(tr.rz_inner), rnorms=np.array(tr.residual_norms),
                 iterations=tr.iterations, converged=tr.converged,
                 L=D.coarse_factor, AC=D.ac)
        if tr.iterations >= 2:
            spec = ref_recycle.select_spectrum(tr, recycg.RecycleStrategy("srks", epsilon=1e-10))
            d["ritz_values"] = spec.values
            d["ritz_mask"] = spec.converged_mask
            view = recycg.lanczos_from_trace(tr)
            d["ritz_prev"] = recycg.tridiag_eig(view.tridiag.truncated(view.m - 1)).values
            idx = np.flatnonzero(spec.converged_mask)
            d["ritz_block"] = spec.vectors[:, idx] / np.sqrt(np.abs(spec.values[idx]))
        cases[name] = d
    out = {}
    for name, d in cases.items():
        for k, v in d.items():
            out[f"{name}__{k}"] = np.asarray(v)
    np.savez_compressed(HERE / "small_solves.npz", names=np.array(list(cases)), **out)
    print("small_solves:", {k: int(v["iterations"]) for k, v in cases.items()})


def config1_sequence():
    """BASELINE config 1 through the reference run_sequence: SRKS eps=1e-10,
    nc_limit 21, tol 1e-8, Jacobi, reorth on."""
    systems = problems.shifted_laplacian_sequence()
    # the base operator must be byte-identical to the reference's own assembler
    A0_ref = ref_problems._assemble_diffusion(np.ones((128, 128)))
    A0 = problems.assemble_diffusion(np.ones((128, 128)))
    assert csr_sha(A0_ref) == csr_sha(A0), "diffusion assembler drifted from reference"
    shas = [csr_sha(A) for A, _ in systems]
    bsha = [hashlib.sha256(b.tobytes()).hexdigest() for _, b in systems]
    ref_systems = [(to_ref(A), b) for A, b in systems]
    cfg = recycg.SolveConfig(tol=1e-8, max_iters=2000)
    rep = recycg.run_sequence(iter(ref_systems), recycg.Preconditioner.jacobi,
                              recycg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=21), cfg)
    sel_vals = [[float(t[2]) for t in rep.final_tags]]  # final basis provenance
    # per-system selected Ritz values via the tags the reference records
    # (re-run with per-step capture for values of every step)
    per_step = []
    state = ref_recycle.AugmentationState.from_initial(systems[0][0].n)
    xs = []
    for k, (A, b) in enumerate(ref_systems):
        D = ref_recycle.guarded_deflation(A, state, [])
        x, tr = recycg.apcg_solve(A, recycg.Preconditioner.jacobi(A), D, b,
                                  recycg.SolveConfig(tol=1e-8, max_iters=2000))
        spec = ref_recycle.select_spectrum(tr, recycg.RecycleStrategy("srks", epsilon=1e-10))
        idx = np.flatnonzero(spec.converged_mask)
        per_step.append([float(v) for v in spec.values[idx]])
        ref_recycle.update_basis_srks(state, spec, k)
        if state.n_c >= 21:
            state.restart()
        xs.append(x)
    data = dict(
        matrix_sha256=shas, rhs_sha256=bsha,
        iterations=rep.iterations(), n_c_before=rep.n_c_history(),
        n_c_selected=[r.n_c_selected for r in rep.records],
        final_residual=[r.final_residual for r in rep.records],
        converged=[bool(r.converged) for r in rep.records],
        events=[list(map(str, e)) for e in rep.events],
        selected_ritz_values=per_step,
        final_tags=sel_vals,
    )
    (HERE / "config1_sequence.json").write_text(json.dumps(data, indent=1) + "\n")
    np.savez_compressed(HERE / "config1_solutions.npz", x0=xs[0], x1=xs[1], x9=xs[-1])
    print("config1 iterations:", data["iterations"], "n_c:", data["n_c_before"])


def benchmark_srks():
    """Reference benchmark (problems.py:89-96), first 8 systems, SRKS eps=1e-10
    at tol 1e-6 (bit-stable per SURVEY.md §0 finding 2), plus generator pin."""
    spec_ref = ref_problems.benchmark_spec(seed=0)
    ref_systems = list(ref_problems.generate_diffusion_sequence(spec_ref, 8))
    mine = list(problems.generate_diffusion_sequence(problems.benchmark_spec(seed=0), 8))
    for (Ar, br), (Am, bm) in zip(ref_systems, mine):
        assert csr_sha(Ar) == csr_sha(Am) and np.array_equal(br, bm), "benchmark generator drifted"
    cfg = recycg.SolveConfig(tol=1e-6, max_iters=3000)
    out = {"matrix_sha256": [csr_sha(A) for A, _ in mine]}
    for name, strat in [("srks10", recycg.RecycleStrategy("srks", epsilon=1e-10)),
                        ("srks6", recycg.RecycleStrategy("srks", epsilon=1e-6)),
                        ("clust10", recycg.RecycleStrategy("srks_cluster", epsilon=1e-10))]:
        rep = recycg.run_sequence(iter(ref_systems), recycg.Preconditioner.jacobi, strat, cfg)
        out[name] = dict(iterations=rep.iterations(), n_c_before=rep.n_c_history(),
                         events=[list(map(str, e)) for e in rep.events])
        print(name, rep.iterations(), rep.n_c_history())
    (HERE / "benchmark_srks.json").write_text(json.dumps(out, indent=1) + "\n")


def elasticity_small():
    """Config-2 analog at 8^3 elements (n = 8*9*9*3 = 1944): 4 RHS SRKS."""
    systems = list(problems.elasticity_sequence(8, 4, kind="fixed"))
    A = systems[0][0]
    Ar = recycg.SparseSpdMatrix(A.n, A.row_offsets, A.col_indices, A.values)  # validates symmetry
    cfg = recycg.SolveConfig(tol=1e-8, max_iters=3000)
    rep = recycg.run_sequence(iter([(Ar, b) for _, b in systems]), recycg.Preconditioner.jacobi,
                              recycg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=61), cfg)
    out = dict(matrix_sha256=csr_sha(A), iterations=rep.iterations(),
               n_c_before=rep.n_c_history(),
               final_residual=[r.final_residual for r in rep.records])
    (HERE / "elasticity8_sequence.json").write_text(json.dumps(out, indent=1) + "\n")
    print("elasticity8", rep.iterations(), rep.n_c_history())


def pilot_fixture():
    """Copy of the reference's frozen golden lists that reproduce exactly
    (none/trks; SURVEY.md §0 finding 2): pkg/tests/fixtures/benchmark_pilot.json."""
    src = json.loads(Path("/root/reference/pkg/tests/fixtures/benchmark_pilot.json").read_text())
    keep = {"source": "reference pkg/tests/fixtures/benchmark_pilot.json (none, trks lists)",
            "runs": {tol: {s: src["runs"][tol][s] for s in ("none", "trks") if s in src["runs"][tol]}
                     for tol in src["runs"]}}
    (HERE / "benchmark_pilot_none_trks.json").write_text(json.dumps(keep, indent=1) + "\n")


# ---------------------------------------------------------------------------
# round 2: sequence-level goldens at the BASELINE configs


def _sample_idx(n, count=16384, seed=7):
    """Seeded index sample used to pin large solutions without storing them."""
    rng = np.random.Generator(np.random.Philox(seed))
    return np.sort(rng.choice(n, size=min(n, count), replace=False))


def _spy_sequence(systems, strat, cfg, C0=None, keep_x=(), sample=None):
    """Run the REFERENCE run_sequence unchanged, spying on its apcg_solve and
    select_spectrum seams (recycle.py:204, :218) to record each system's
    solution (or a seeded sample of it) and its selected Ritz values."""
    xs, sel = {}, []
    real_solve, real_select = ref_recycle.apcg_solve, ref_recycle.select_spectrum
    k_box = [0]

    def solve(A, M, D, b, c):
        x, tr = real_solve(A, M, D, b, c)
        k = k_box[0]
        k_box[0] += 1
        if k in keep_x:
            xs[k] = x.copy() if sample is None else x[sample].copy()
        return x, tr

    def select(trace, strategy):
        spec = real_select(trace, strategy)
        sel.append((k_box[0] - 1, [float(v) for v in spec.values[spec.converged_mask]]))
        return spec

    ref_recycle.apcg_solve, ref_recycle.select_spectrum = solve, select
    try:
        rep = ref_recycle.run_sequence(iter(systems), recycg.Preconditioner.jacobi, strat, cfg, C0)
    finally:
        ref_recycle.apcg_solve, ref_recycle.select_spectrum = real_solve, real_select
    per_step = [[] for _ in rep.records]
    for k, vals in sel:
        if k < len(per_step):
            per_step[k] = vals
    return rep, xs, per_step


def _report_dict(rep):
    return dict(iterations=rep.iterations(), n_c_before=rep.n_c_history(),
                n_c_selected=[r.n_c_selected for r in rep.records],
                final_residual=[r.final_residual for r in rep.records],
                converged=[bool(r.converged) for r in rep.records], aborted=bool(rep.aborted),
                events=[list(map(str, e)) for e in rep.events])


def reduced_sequences(which=("c2r", "c3r", "c4r_on", "c4r_off", "c5r")):
    """SURVEY.md §8(d) reduced analogs of configs 2-5 through the reference
    run_sequence: elasticity 16^3 (20 RHS), 24^3 softening (15 systems),
    diffusion 64^3 (20 systems, reorth on and off), lognormal-softening
    elasticity 16^3 (10 systems, nc_limit 101, reorth off)."""
    out_path = HERE / "reduced_sequences.json"
    out = json.loads(out_path.read_text()) if out_path.exists() else {}
    sols = dict(np.load(HERE / "reduced_solutions.npz")) if (HERE / "reduced_solutions.npz").exists() else {}
    specs = {
        "c2r": (2, True), "c3r": (3, True), "c4r_on": (4, True), "c4r_off": (4, False), "c5r": (5, False),
    }
    for name in which:
        config, reorth = specs[name]
        systems, st = problems.config_systems(config, reduced=True)
        systems = list(systems)
        shas = [csr_sha(A) for A, _ in systems]
        bsha = [hashlib.sha256(b.tobytes()).hexdigest() for _, b in systems]
        ref_systems = [(to_ref(A), b) for A, b in systems]
        cfg = recycg.SolveConfig(tol=st["tol"], max_iters=5000, reorthogonalize=reorth)
        strat = recycg.RecycleStrategy("srks", epsilon=st["epsilon"], nc_limit=st["nc_limit"])
        last = len(systems) - 1
        t0 = time.time()
        n0 = systems[0][0].n
        sample = _sample_idx(n0) if n0 > 50000 else None      # large n: pin a seeded sample of x
        rep, xs, per_step = _spy_sequence(ref_systems, strat, cfg, keep_x=(0, 1, last), sample=sample)
        d = _report_dict(rep)
        d.update(config=config, reduced=True, reorthogonalize=reorth, tol=st["tol"], epsilon=st["epsilon"],
                 nc_limit=st["nc_limit"], n=int(systems[0][0].n), nnz=int(systems[0][0].nnz),
                 matrix_sha256=shas, rhs_sha256=bsha, selected_ritz_values=per_step,
                 reference_seconds=time.time() - t0)
        out[name] = d
        for k, x in xs.items():
            sols[f"{name}__x{k}"] = x
        out_path.write_text(json.dumps(out, indent=1) + "\n")
        np.savez_compressed(HERE / "reduced_solutions.npz", **sols)
        print(name, d["iterations"], d["n_c_before"], f"{d['reference_seconds']:.0f}s", flush=True)


def config2_full(count=2):
    """BASELINE config 2 at full size (Q1 64^3, n = 811,200), systems 0..count-1
    through the reference run_sequence: SRKS eps 1e-10, nc_limit 61, tol 1e-8,
    full reorth.  Solutions are pinned on a seeded 16,384-entry sample plus
    their norms."""
    gen = problems.elasticity_sequence(64, count, kind="fixed")
    systems = list(gen)
    A = systems[0][0]
    idx = _sample_idx(A.n)
    Ar = to_ref(A)
    cfg = recycg.SolveConfig(tol=1e-8, max_iters=20000)
    strat = recycg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=61)
    t0 = time.time()
    rep, xs, per_step = _spy_sequence([(Ar, b) for _, b in systems], strat, cfg, keep_x=tuple(range(count)))
    d = _report_dict(rep)
    d.update(n=int(A.n), nnz=int(A.nnz), matrix_sha256=csr_sha(A),
             rhs_sha256=[hashlib.sha256(b.tobytes()).hexdigest() for _, b in systems],
             selected_ritz_values=per_step, reference_seconds=time.time() - t0,
             x_norm=[float(np.linalg.norm(xs[k])) for k in range(count)], sample_seed=7)
    (HERE / "config2_full.json").write_text(json.dumps(d, indent=1) + "\n")
    np.savez_compressed(HERE / "config2_full_xsample.npz", idx=idx,
                        **{f"x{k}": xs[k][idx] for k in range(count)})
    print("config2 full", d["iterations"], d["n_c_before"], f"{d['reference_seconds']:.0f}s", flush=True)


def acceptance6():
    """Reference acceptance criterion 6 (pkg/tests/test_acceptance.py:226-266)
    restated: the 40-system inclusion benchmark with none / trks / srks(1e-14)
    at tol 1e-3 and trks / srks(1e-14) at tol 1e-6, run through the reference
    here; the frozen margins come from the reference fixture."""
    fx = json.loads(Path("/root/reference/pkg/tests/fixtures/benchmark_pilot.json").read_text())
    ref_systems = list(ref_problems.generate_diffusion_sequence(ref_problems.benchmark_spec(seed=0), 40))
    mine = list(problems.generate_diffusion_sequence(problems.benchmark_spec(seed=0), 40))
    for (Ar, br), (Am, bm) in zip(ref_systems, mine):
        assert csr_sha(Ar) == csr_sha(Am) and np.array_equal(br, bm), "benchmark generator drifted"
    out = {"margins": fx["margins"], "matrix_sha256": [csr_sha(A) for A, _ in mine]}
    for tol, runs in [(1e-3, [("none", "none", None), ("trks", "trks", None), ("srks14", "srks", 1e-14)]),
                      (1e-6, [("trks", "trks", None), ("srks14", "srks", 1e-14)])]:
        cfg = recycg.SolveConfig(tol=tol, max_iters=3000)
        for name, kind, eps in runs:
            strat = recycg.RecycleStrategy(kind, **({"epsilon": eps} if eps else {}))
            t0 = time.time()
            rep = recycg.run_sequence(iter(ref_systems), recycg.Preconditioner.jacobi, strat, cfg)
            d = _report_dict(rep)
            d["reference_seconds"] = time.time() - t0
            out.setdefault(f"tol{tol:g}", {})[name] = d
            print("accept6", tol, name, d["iterations"][:6], d["n_c_before"][-3:], f"{d['reference_seconds']:.0f}s",
                  flush=True)
    (HERE / "acceptance6.json").write_text(json.dumps(out, indent=1) + "\n")



def trks_config1(count=5):
    """TRKS on config 1 at tol 1e-8 (the explicit G^-1 coarse
    solve against a high-kappa C^T A C): normalized directions make kappa(G)
    ~ kappa(A).  Reference run_sequence, first `count` systems."""
    systems = problems.shifted_laplacian_sequence(count=count)
    ref_systems = [(to_ref(A), b) for A, b in systems]
    cfg = recycg.SolveConfig(tol=1e-8, max_iters=2000)
    t0 = time.time()
    rep, xs, _ = _spy_sequence(ref_systems, recycg.RecycleStrategy("trks"), cfg, keep_x=tuple(range(count)))
    d = _report_dict(rep)
    d["reference_seconds"] = time.time() - t0
    (HERE / "trks_config1.json").write_text(json.dumps(d, indent=1) + "\n")
    np.savez_compressed(HERE / "trks_config1_solutions.npz", **{f"x{k}": x for k, x in xs.items()})
    print("trks config1", d["iterations"], d["n_c_before"], f"{d['reference_seconds']:.0f}s", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "config1", "bench", "elast", "pilot"]
    if "pilot" in which:
        pilot_fixture()
    if "small" in which:
        small_solve_cases()
    if "elast" in which:
        elasticity_small()
    if "bench" in which:
        benchmark_srks()
    if "config1" in which:
        config1_sequence()
    for w in which:
        if w.startswith("reduced"):
            names = w.split(":")[1].split(",") if ":" in w else None
            reduced_sequences(*( [names] if names else []))
    if "config2" in which:
        config2_full()
    if "accept6" in which:
        acceptance6()
    if "trks1" in which:
        trks_config1()
