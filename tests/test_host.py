"""Host-side logic that runs without a GPU: the C-ABI library loads and
exports every symbol include/rcg.h declares, API validation and dataclasses
mirror the reference, generators, oracle KATs mirroring the reference tests."""
import re
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import _lib, problems
from oracle import recycg_oracle as orc

REPO = Path(__file__).resolve().parents[1]


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    header = (REPO / "include" / "rcg.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|int64_t|void|const char\*)\s+(rcg_\w+)\s*\(", header, flags=re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.rcg_version() == 1


def test_library_is_sm100a():
    so = _lib.lib_path().read_bytes()
    assert b"sm_100a" in so or b"sm_100" in so


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    A = rcg.SparseSpdMatrix.from_dense(np.eye(3))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        A @ np.ones(3)


def test_product_does_not_import_oracle():
    for p in (REPO / "paper_1301_7530_b200").rglob("*.py"):
        text = p.read_text()
        assert "from oracle" not in text and "import oracle" not in text and "recycg_oracle" not in text, p


# ---------------------------------------------------------------------------
# API validation mirrors the reference (no device needed)


def test_solve_config_validation():
    with pytest.raises(rcg.ContractViolation):
        rcg.SolveConfig(tol=0.0)
    with pytest.raises(rcg.ContractViolation):
        rcg.SolveConfig(tol=2.0)
    with pytest.raises(rcg.ContractViolation):
        rcg.SolveConfig(max_iters=0)


def test_strategy_validation():
    with pytest.raises(rcg.ContractViolation):
        rcg.RecycleStrategy("bogus")
    with pytest.raises(rcg.ContractViolation):
        rcg.RecycleStrategy("srks", epsilon=0.0)
    with pytest.raises(rcg.ContractViolation):
        rcg.RecycleStrategy("trks", nc_limit=-1)


def test_csr_validation():
    with pytest.raises(rcg.ContractViolation):
        rcg.SparseSpdMatrix(2, np.array([0, 1]), np.array([0]), np.array([1.0]))
    with pytest.raises(rcg.ContractViolation):   # asymmetric pattern
        rcg.SparseSpdMatrix(2, np.array([0, 2, 3]), np.array([0, 1, 1]), np.array([1.0, 0.5, 1.0]))
    with pytest.raises(rcg.ContractViolation):   # missing diagonal
        rcg.SparseSpdMatrix(2, np.array([0, 1, 2]), np.array([1, 0]), np.array([1.0, 1.0]))
    with pytest.raises(rcg.ContractViolation):   # unsorted columns
        rcg.SparseSpdMatrix(2, np.array([0, 2, 4]), np.array([1, 0, 0, 1]), np.array([0.5, 1.0, 0.5, 1.0]))


def test_tridiag_sym():
    T = rcg.TridiagSym(np.array([1.0, 2.0, 3.0]), np.array([0.5, 0.25]))
    T2 = T.truncated(2)
    np.testing.assert_array_equal(T2.diag, [1.0, 2.0])
    with pytest.raises(rcg.ContractViolation):
        T.truncated(4)
    with pytest.raises(rcg.ContractViolation):
        rcg.TridiagSym(np.array([1.0, 2.0]), np.array([1.0, 1.0]))
    np.testing.assert_array_equal(rcg.TridiagSym(np.array([2.0, 2.0]), np.array([1.0])).to_dense(),
                                  [[2.0, 1.0], [1.0, 2.0]])


def test_cluster_filter_host_edges():
    # reference tests/test_ritz.py:221-240: the cases decided before any
    # device work (no cluster possible, contract check)
    assert rcg.cluster_filter([3.0, 1.0], min_cluster=5) == [0, 1]
    assert rcg.cluster_filter([7.0], min_cluster=1) == [0]
    assert rcg.cluster_filter([], min_cluster=1) == []
    with pytest.raises(rcg.ContractViolation):
        rcg.cluster_filter([1.0, 2.0], 0)


def test_trace_json_round_trip():
    tr = rcg.SolveTrace(alphas=[0.5, 0.25], betas=[0.1], rz_inner=[1.0, 0.1], residual_norms=[1.0, 0.5, 0.1],
                        z_history=[np.ones(3), np.zeros(3)], iterations=2, converged=True)
    d = tr.to_json_dict(spectrum=[1.0, 2.0], eps_cg=1e-6)
    back = rcg.SolveTrace.from_json_dict(d)
    assert back.iterations == 2 and back.converged
    np.testing.assert_allclose(back.alphas, tr.alphas)
    assert d["spectrum"] == [1.0, 2.0] and d["eps_cg"] == 1e-6


# ---------------------------------------------------------------------------
# generators


def test_elasticity_pattern_and_symmetry():
    A = problems.elasticity_q1(4)          # validates symmetry / diag / sorting
    assert A.n == 4 * 5 * 5 * 3
    rows = np.diff(A.row_offsets)
    assert rows.max() == 81 and rows.min() >= 3 * 8
    E = np.exp(np.random.default_rng(1).standard_normal((4, 4, 4)))
    problems.elasticity_q1(4, E=E)       # heterogeneous: still exactly symmetric


def test_elasticity_64_nnz_matches_survey():
    # n = 811,200, nnz = 63,695,790 at 64^3; count without assembling values
    N = 64
    def cnt(k):   # neighbours along one axis for k nodes
        return 3 * k - 2
    nx, ny = N, N + 1   # free node planes x = 1..N; y, z = 0..N
    assert (3 * nx * ny * ny) == 811200
    total = cnt(nx) * cnt(ny) * cnt(ny) * 9  # (p, q) node pairs within one layer in each axis, 3x3 blocks
    assert total == 63695790


def test_diffusion_matches_reference_semantics():
    kappa = np.exp(np.random.default_rng(3).standard_normal((5, 4, 3)))
    A = problems.assemble_diffusion(kappa)
    D = A.to_dense()
    assert np.allclose(D, D.T)
    # harmonic face coefficient between cells (0,0,0) and (1,0,0)
    i, j = 0, 4 * 3
    assert D[i, j] == pytest.approx(-2 * kappa[0, 0, 0] * kappa[1, 0, 0] / (kappa[0, 0, 0] + kappa[1, 0, 0]))


def test_config_inputs_shapes():
    seq = problems.shifted_laplacian_sequence(grid=16, count=3)
    assert len(seq) == 3 and seq[0][0].n == 256
    A1, A2 = seq[1][0], seq[2][0]
    assert np.all(orc.diagonal(A2) >= orc.diagonal(A1))


# ---------------------------------------------------------------------------
# oracle KATs (mirroring reference tests on the restated algorithm)


def test_oracle_cholesky_kats():
    np.testing.assert_allclose(orc.dense_cholesky(np.array([[4.0, 2.0], [2.0, 2.0]])), [[2.0, 0.0], [1.0, 1.0]])
    with pytest.raises(orc.OracleRankDeficient) as ei:
        orc.dense_cholesky(np.array([[1.0, 1.0], [1.0, 1.0]]))
    assert ei.value.column == 1


def test_oracle_select_kats():
    assert list(orc.select_converged([9.0, 5.0, 2.0, 1.0], [9.0, 5.0, 2.0], 1e-12)) == [True, True, True, False]
    assert list(orc.select_converged([9.0, 4.0, 1.0], [6.0, 1.0], 1e-12)) == [False, False, True]
    m = orc.select_converged([5.0, 5.0 * (1 + 1e-15), 1.0], [5.0, 5.0], 1e-12)
    assert m[0] and not m[1]


def test_oracle_identity_one_iteration(rng):
    A = rcg.SparseSpdMatrix.from_dense(np.eye(5))
    b = rng.standard_normal(5)
    x, tr = orc.apcg_solve(A, None, orc.build_deflation(A, np.zeros((5, 0))), b, 1e-10, 500)
    assert tr.iterations == 1 and tr.converged
    np.testing.assert_allclose(x, b)


def test_oracle_full_augmentation_zero_iterations(rng):
    n = 6
    A = rcg.SparseSpdMatrix.from_dense(np.diag(np.arange(1.0, n + 1.0)))
    b = rng.standard_normal(n)
    x, tr = orc.apcg_solve(A, None, orc.build_deflation(A, np.eye(n)), b, 1e-10, 500)
    assert tr.iterations == 0 and tr.converged


def test_reference_bridge_rebinds_every_seam(tmp_path):
    """bridge.install rebinds the reference's seams in every
    module that binds them (the device calls themselves run under -m gpu,
    tests/test_gpu_reference_bridge.py) and uninstall restores them."""
    import importlib
    import zipfile
    zp = REPO / "oracle" / "_ref" / "recycg_ref.zip"
    if Path("/root/reference/pkg/src/recycg").is_dir():
        src = "/root/reference/pkg/src"
    elif zp.exists():
        with zipfile.ZipFile(zp) as z:
            z.extractall(tmp_path)
        src = str(tmp_path / "src")
    else:
        pytest.skip("reference not available")
    sys.path.insert(0, src)
    try:
        recycg = importlib.import_module("recycg")
        from paper_1301_7530_b200 import bridge
        before = {(m, n): getattr(importlib.import_module("recycg" + m), n)
                  for m in bridge._MODULES for n in bridge.SEAMS
                  if hasattr(importlib.import_module("recycg" + m), n)}
        assert ("", "apcg_solve") in before and (".recycle", "select_spectrum") in before
        b = bridge.install(recycg)
        for (m, n), fn in before.items():
            now = getattr(importlib.import_module("recycg" + m), n)
            assert now is not fn and now.__wrapped__.__name__ == n, (m, n)
        b.uninstall()
        for (m, n), fn in before.items():
            assert getattr(importlib.import_module("recycg" + m), n) is fn
    finally:
        sys.path.remove(src)
        for k in [k for k in sys.modules if k == "recycg" or k.startswith("recycg.")]:
            del sys.modules[k]


def _reference_src(tmp_path):
    import zipfile
    zp = REPO / "oracle" / "_ref" / "recycg_ref.zip"
    if Path("/root/reference/pkg/src/recycg").is_dir():
        return "/root/reference/pkg/src"
    if zp.exists():
        with zipfile.ZipFile(zp) as z:
            z.extractall(tmp_path)
        return str(tmp_path / "src")
    pytest.skip("reference not available")


def test_report_writers_match_reference_schema(tmp_path):
    """runs.csv / summary.json / curve files byte-identical to the reference
    CLI's writers (cli.py:181-244) for the same records."""
    import importlib
    from paper_1301_7530_b200 import report
    src = _reference_src(tmp_path)
    sys.path.insert(0, src)
    try:
        cli = importlib.import_module("recycg.cli")
        rng = np.random.default_rng(5)
        runs = []
        for name, pc, tol, seed in [("srks14", "jacobi", 1e-3, 0), ("trks", "identity", 1e-6, 3)]:
            rep = rcg.SequenceReport()
            for k in range(4):
                rep.records.append(rcg.SystemRecord(k, int(rng.integers(10, 500)), int(rng.integers(0, 90)),
                                                    int(rng.integers(0, 9)), float(rng.uniform(0, 2)),
                                                    float(rng.uniform(0, 1)), float(rng.uniform(1e-9, 1e-3)),
                                                    bool(k != 2 or name == "trks")))
            runs.append(report.RunResult(name, pc, tol, seed, rep))
        ours = tmp_path / "ours"
        report.write_report(ours, runs)
        theirs = tmp_path / "theirs"
        none = cli.RecycleStrategy("none")   # no final bases: the reference's overlap file is skipped
        ref_runs = [cli.RunResult(r.name, none, r.preconditioner, r.tol, r.seed, r.report) for r in runs]
        cfg = type("Cfg", (), {})()
        cli._write_outputs(cfg, ref_runs, theirs)
        names = sorted(p.name for p in theirs.iterdir())
        assert names == sorted(p.name for p in ours.iterdir())
        for nm in names:
            assert (ours / nm).read_text() == (theirs / nm).read_text(), nm
        assert report.CSV_HEADER == cli.CSV_HEADER
    finally:
        sys.path.remove(src)
        for k in [k for k in sys.modules if k == "recycg" or k.startswith("recycg.")]:
            del sys.modules[k]
