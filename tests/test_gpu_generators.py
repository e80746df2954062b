"""Device assemblers (csrc/gen.cu) against the host assemblers they mirror:
bitwise-equal CSR bytes on small and ragged grids, the BASELINE nnz counts at
full size, symmetry and a solve through the device
copy.  The host assemblers are pinned to the reference's own
``_assemble_diffusion`` bytes by tests/golden/make_golden.py."""
import numpy as np
import pytest

import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems

pytestmark = pytest.mark.gpu


def _same_csr(D, H):
    assert D.n == H.n and D.nnz == H.nnz
    np.testing.assert_array_equal(D.row_offsets, H.row_offsets)
    np.testing.assert_array_equal(D.col_indices.astype(np.int64), H.col_indices.astype(np.int64))
    # bitwise: compare the raw bytes (signed zeros included)
    assert np.array_equal(D.values.view(np.uint64), H.values.view(np.uint64))


@pytest.mark.parametrize("shape", [(2,), (9,), (5, 6), (4, 1, 5), (1, 7, 3), (3, 4, 5), (6, 6, 6)])
def test_diffusion_device_bitwise(shape):
    rng = np.random.Generator(np.random.Philox(3))
    kappa = rng.lognormal(0.0, 2.0, shape)
    _same_csr(problems.assemble_diffusion_device(kappa), problems.assemble_diffusion(kappa, validate=True))


@pytest.mark.parametrize("nelem,random_e", [(1, False), (2, True), (3, False), (5, True)])
def test_elasticity_device_bitwise(nelem, random_e):
    rng = np.random.Generator(np.random.Philox(7))
    E = rng.lognormal(0.0, 1.0, (nelem,) * 3) if random_e else None
    _same_csr(problems.elasticity_q1_device(nelem, E=E), problems.elasticity_q1(nelem, E=E, validate=True))


def test_device_sequences_match_host():
    """config-3-style softening sequence (reduced): identical operators."""
    dev = list(problems.elasticity_sequence(4, 3, kind="softening", device=True))
    host = list(problems.elasticity_sequence(4, 3, kind="softening"))
    for (Ad, bd), (Ah, bh) in zip(dev, host):
        _same_csr(Ad, Ah)
        np.testing.assert_array_equal(bd, bh)
    dev = list(problems.lognormal_diffusion_sequence(6, 2, device=True))
    host = list(problems.lognormal_diffusion_sequence(6, 2))
    for (Ad, bd), (Ah, bh) in zip(dev, host):
        _same_csr(Ad, Ah)


def test_device_matrix_solves_like_host():
    A_h = problems.elasticity_q1(6)
    A_d = problems.elasticity_q1_device(6)
    b = problems.elasticity_rhs(6, np.random.Generator(np.random.Philox(0)))
    cfg = rcg.SolveConfig(tol=1e-8, max_iters=5000)
    out = []
    for A in (A_h, A_d):
        D = rcg.build_deflation(A, np.zeros((A.n, 0)))
        x, tr = rcg.apcg_solve(A, rcg.Preconditioner.jacobi(A), D, b, cfg)
        out.append((x, tr.iterations))
    assert out[0][1] == out[1][1]
    np.testing.assert_array_equal(out[0][0], out[1][0])


@pytest.mark.parametrize("which,n,nnz", [("elast64", 811_200, 63_695_790), ("diff256", 16_777_216, 117_047_296)])
def test_full_size_counts_and_symmetry(which, n, nnz):
    """BASELINE configs 2 and 4 at full size: SURVEY.md §8(d) n / nnz, and
    x^T (A y) == y^T (A x) (symmetric operator) to rounding."""
    import torch
    if which == "elast64":
        A = problems.elasticity_q1_device(64)
    else:
        rng = np.random.Generator(np.random.Philox(0))
        A = problems.assemble_diffusion_device(rng.lognormal(0.0, 2.0, (256, 256, 256)))
    assert A.n == n and A.nnz == nnz
    assert A.device_csr().struct.dia_count == (14 if which == "elast64" else 4)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    y = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    ax, ay = rcg.spmv(A, x), rcg.spmv(A, y)
    l, r = float(torch.dot(x, ay)), float(torch.dot(y, ax))
    scale = float(torch.linalg.norm(x) * torch.linalg.norm(ay))
    assert abs(l - r) <= 1e-12 * scale
    A.release_device()
