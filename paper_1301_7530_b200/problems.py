"""Seeded synthetic inputs for the hot path (input side, not the hot path).

Every generator produces host CSR arrays (int64 row offsets, int32/int64 sorted
column indices, float64 values, full symmetric pattern) wrapped in
:class:`~paper_1301_7530_b200.core.SparseSpdMatrix`; the same host bytes are fed to
the CPU oracle and to the B200 path, so parity never depends on two generators
agreeing.

Provenance of each family:

* ``benchmark_spec`` / ``generate_diffusion_sequence`` restate the reference's
  own inclusion benchmark (``/root/reference/pkg/src/recycg/problems.py:22-189``):
  same Philox stream, same per-material redraw rule, same load vector.
* ``assemble_diffusion`` follows ``_assemble_diffusion``
  (``problems.py:115-156``): harmonic face means, Dirichlet faces using the cell's
  own coefficient, axes of size 1 carry nothing.  It is built here as a
  structured stencil (no COO round trip) so 256^3 grids assemble in seconds.
* ``shifted_laplacian_sequence`` is BASELINE.json config 1.
* ``elasticity_q1`` is BASELINE.json configs 2/3/5: there is no reference
  generator, so this is a new trilinear-hex assembler (SURVEY.md §0 finding 6).
* ``lognormal_diffusion_sequence`` is config 4.
* ``generate_prescribed_spectrum`` restates ``problems.py:192-216``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from itertools import product

import numpy as np

from .core import ContractViolation, SparseSpdMatrix

__all__ = [
    "InclusionGridSpec", "regular_inclusion_layout", "benchmark_spec",
    "generate_diffusion_sequence", "assemble_diffusion", "SpectrumSpec",
    "generate_prescribed_spectrum", "shifted_laplacian_sequence",
    "elasticity_q1", "elasticity_sequence", "lognormal_diffusion_sequence",
    "random_spd", "config_systems",
]


def _philox(seed):
    return np.random.Generator(np.random.Philox(seed))


# ---------------------------------------------------------------------------
# structured-stencil CSR helper


def _stencil_csr(n, cols, vals, validate=False):
    """Compress an ``(n, k)`` stencil (column -1 = absent) into CSR.

    Columns must already be increasing along each row (stencil offsets are
    listed in ascending order), so no sort is needed.
    """
    mask = cols >= 0
    counts = mask.sum(axis=1, dtype=np.int64)
    ro = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=ro[1:])
    ci = cols[mask]
    ci = ci.astype(np.int32) if n < 2 ** 31 - 1 else ci.astype(np.int64)
    va = np.ascontiguousarray(vals[mask], dtype=np.float64)
    return SparseSpdMatrix(n, ro, ci, va, validate=validate)


# ---------------------------------------------------------------------------
# finite-difference diffusion (reference problems.py:115-156 semantics)


def assemble_diffusion(cell_coeff, validate=None):
    """FD diffusion operator with harmonic face coefficients on a 1/2/3-D grid.

    Semantics of ``_assemble_diffusion`` (``problems.py:115-156``): interior face
    weight ``2 c_lo c_hi / (c_lo + c_hi)``, Dirichlet faces add the cell's own
    coefficient at both ends of every axis of size >= 2.  The diagonal is
    accumulated in the same axis order as the reference (axis 0 faces, axis 0
    boundary, axis 1 faces, ...), so the bytes are identical.
    """
    cell_coeff = np.asarray(cell_coeff, dtype=np.float64)
    grid = cell_coeff.shape
    n = cell_coeff.size
    ndim = len(grid)
    strides = [int(np.prod(grid[a + 1:])) for a in range(ndim)]
    diag = np.zeros(grid)
    # stencil slots: axis-descending negative offsets, centre, ascending positive
    lo_slots = {}
    hi_slots = {}
    order = []
    for a in range(ndim):
        if grid[a] >= 2:
            order.append(a)
    k = 2 * len(order) + 1
    centre = len(order)
    for pos, a in enumerate(order):          # larger stride -> more negative
        lo_slots[a] = pos                    # offset -stride[a]
        hi_slots[a] = k - 1 - pos            # offset +stride[a]
    cols = np.full(grid + (k,), -1, dtype=np.int64)
    vals = np.zeros(grid + (k,))
    index = np.arange(n, dtype=np.int64).reshape(grid)
    for a in range(ndim):
        g = grid[a]
        if g < 2:
            continue
        lo = [slice(None)] * ndim
        hi = [slice(None)] * ndim
        lo[a] = slice(0, g - 1)
        hi[a] = slice(1, g)
        lo, hi = tuple(lo), tuple(hi)
        c_lo = cell_coeff[lo]
        c_hi = cell_coeff[hi]
        face = 2.0 * c_lo * c_hi / (c_lo + c_hi)
        # coupling of the low cell to the high cell (+stride) and back
        cols[lo + (hi_slots[a],)] = index[hi]
        vals[lo + (hi_slots[a],)] = -face
        cols[hi + (lo_slots[a],)] = index[lo]
        vals[hi + (lo_slots[a],)] = -face
        # the reference uses np.add.at(diag, i_lo, face) then i_hi: same order
        diag[lo] += face
        diag[hi] += face
        for end in (0, g - 1):
            sel = [slice(None)] * ndim
            sel[a] = end
            sel = tuple(sel)
            diag[sel] += cell_coeff[sel]
    cols[..., centre] = index
    vals[..., centre] = diag
    if validate is None:
        validate = n <= 200_000
    return _stencil_csr(n, cols.reshape(n, k), vals.reshape(n, k), validate)


# ---------------------------------------------------------------------------
# device assemblers (csrc/gen.cu): same bytes as the host assemblers, built in
# HBM; only the coefficient field crosses PCIe


def _device_csr_from(rows_fn, fill_fn, n):
    """Run a two-pass device assembler and wrap the CSR it writes."""
    from ._lib import context, ptr, require_cuda, C
    from .core import _DevCsr, DeviceSparseSpdMatrix
    torch = require_cuda()
    ctx = context()
    ro64 = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    nnz = C.c_int64(0)
    ctx.check(rows_fn(ctx, ptr(ro64), C.byref(nnz)), "gen rows")
    nnz = nnz.value
    wide = nnz >= 2 ** 31 - 1
    ro32 = None if wide else torch.empty(n + 1, dtype=torch.int32, device="cuda")
    ci = torch.empty(max(nnz, 1), dtype=torch.int32, device="cuda")
    va = torch.empty(max(nnz, 1), dtype=torch.float64, device="cuda")
    ctx.check(fill_fn(ctx, ptr(ro64), None if wide else ptr(ro32), ptr(ci), ptr(va)), "gen fill")
    torch.cuda.synchronize()
    ro = ro64 if wide else ro32
    del ro64
    h = _DevCsr(ro, ci[:nnz], va[:nnz], n, nnz, wide)
    return DeviceSparseSpdMatrix(n, h, torch.cuda.current_device())


def assemble_diffusion_device(cell_coeff):
    """``assemble_diffusion`` on the device: the same CSR bytes, written in HBM.
    ``cell_coeff`` is a host array or a CUDA tensor (1-3 dimensions)."""
    from ._lib import require_cuda, ptr, C
    torch = require_cuda()
    if torch.is_tensor(cell_coeff):
        coeff = cell_coeff.to(device="cuda", dtype=torch.float64).contiguous()
    else:
        coeff = torch.from_numpy(np.ascontiguousarray(cell_coeff, dtype=np.float64)).to("cuda")
    shape = tuple(coeff.shape)
    if not 1 <= len(shape) <= 3:
        raise ContractViolation("cell_coeff must have 1 to 3 dimensions")
    dims = (C.c_int64 * len(shape))(*shape)
    n = int(np.prod(shape))
    return _device_csr_from(
        lambda ctx, ro, nnz: ctx.lib.rcg_gen_diffusion_rows(ctx.h, dims, len(shape), ro, nnz),
        lambda ctx, ro, ro32, ci, va: ctx.lib.rcg_gen_diffusion_fill(ctx.h, dims, len(shape), ptr(coeff), ro, ro32,
                                                                     ci, va), n)


def elasticity_q1_device(nelem, E=None, nu=0.3):
    """``elasticity_q1`` on the device (same CSR bytes).  ``E``: None or a host
    array / CUDA tensor of shape ``(nelem,)*3``."""
    from ._lib import require_cuda, ptr
    torch = require_cuda()
    N = int(nelem)
    Ke = torch.from_numpy(np.ascontiguousarray(_q1_element_stiffness(1.0 / N, nu))).to("cuda")
    Ed = None
    if E is not None:
        if tuple(E.shape) != (N, N, N):
            raise ContractViolation("E must have shape (nelem,)*3")
        Ed = (E.to(device="cuda", dtype=torch.float64).contiguous() if torch.is_tensor(E)
              else torch.from_numpy(np.ascontiguousarray(E, dtype=np.float64)).to("cuda"))
    n = 3 * N * (N + 1) * (N + 1)
    return _device_csr_from(
        lambda ctx, ro, nnz: ctx.lib.rcg_gen_elasticity_rows(ctx.h, N, ro, nnz),
        lambda ctx, ro, ro32, ci, va: ctx.lib.rcg_gen_elasticity_fill(ctx.h, N, ptr(Ke), None if Ed is None else ptr(Ed),
                                                                      ro, ro32, ci, va), n)


# ---------------------------------------------------------------------------
# the reference's own inclusion benchmark (problems.py:22-189)


@dataclass(frozen=True)
class InclusionGridSpec:
    """Randomized diffusion sequence on a regular grid with inclusions
    (``problems.py:22-71``)."""

    grid: tuple
    inclusion_layout: tuple = ()
    matrix_coeff_mean: float = 1.0
    inclusion_coeff_mean: float | tuple = 100.0
    rel_std: float = 0.10
    seed: int = 0

    def __post_init__(self):
        grid = tuple(int(g) for g in self.grid)
        object.__setattr__(self, "grid", grid)
        object.__setattr__(self, "inclusion_layout",
                           tuple(tuple(tuple(int(v) for v in rng) for rng in block)
                                 for block in self.inclusion_layout))
        if np.ndim(self.inclusion_coeff_mean) > 0:
            inc = tuple(float(v) for v in self.inclusion_coeff_mean)
            if len(inc) != len(self.inclusion_layout):
                raise ContractViolation("need one inclusion mean per inclusion block")
            object.__setattr__(self, "inclusion_coeff_mean", inc)
        if len(grid) not in (1, 2, 3) or min(grid) < 1 or max(grid) < 2:
            raise ContractViolation("grid must be a 1/2/3-D lattice with >= 2 cells")
        if self.matrix_coeff_mean <= 0 or np.any(np.atleast_1d(self.inclusion_coeff_mean) <= 0):
            raise ContractViolation("coefficient means must be positive")
        if self.rel_std < 0:
            raise ContractViolation("rel_std must be nonnegative")
        for block in self.inclusion_layout:
            if len(block) != len(grid):
                raise ContractViolation("inclusion block rank must match grid rank")
            for (lo, hi), g in zip(block, grid):
                if not 0 <= lo < hi <= g:
                    raise ContractViolation("inclusion block out of grid bounds")

    @property
    def n(self):
        return int(np.prod(self.grid))


def regular_inclusion_layout(grid, per_axis, fill=0.5):
    """Regular per-axis arrangement of blocks (``problems.py:74-86``)."""
    spans = []
    for g in grid:
        cell = g / per_axis
        width = max(1, int(round(cell * fill)))
        starts = [int(round(i * cell + (cell - width) / 2)) for i in range(per_axis)]
        spans.append([(s, min(g, s + width)) for s in starts])
    return tuple(tuple(combo) for combo in product(*spans))


def benchmark_spec(seed=0, grid=(64, 64), per_axis=4, contrast_range=(1.0, 3.0)):
    """The reference benchmark: 64x64 grid, 4x4 inclusions with geometrically
    spread means (``problems.py:89-96``)."""
    layout = regular_inclusion_layout(grid, per_axis)
    means = np.logspace(contrast_range[0], contrast_range[1], len(layout))
    return InclusionGridSpec(grid=tuple(grid), inclusion_layout=layout,
                             inclusion_coeff_mean=tuple(means), rel_std=0.10,
                             seed=seed)


def _material_map(spec):
    materials = np.zeros(spec.grid, dtype=np.int64)
    for i, block in enumerate(spec.inclusion_layout, start=1):
        materials[tuple(slice(lo, hi) for lo, hi in block)] = i
    return materials


def _load_vector(grid):
    """Unit centre source plus 0.01 boundary flux (``problems.py:159-172``)."""
    b = np.zeros(grid)
    for a, g in enumerate(grid):
        if g < 2:
            continue
        for end in (0, g - 1):
            sel = [slice(None)] * len(grid)
            sel[a] = end
            b[tuple(sel)] += 0.01
    b[tuple(g // 2 for g in grid)] += 1.0
    return b.reshape(-1)


def _redraw_positive(rng, mean, rel_std):
    # problems.py:99-103: normal draw, redrawn until above 1e-6 * mean
    while True:
        value = mean * (1.0 + rel_std * rng.standard_normal())
        if value > 1e-6 * mean:
            return value


def generate_diffusion_sequence(spec: InclusionGridSpec, count):
    """Yield ``count`` (A, b) pairs with redrawn material coefficients
    (``problems.py:175-189``)."""
    if count < 1:
        raise ContractViolation("count must be >= 1")
    materials = _material_map(spec)
    inc = np.atleast_1d(np.asarray(spec.inclusion_coeff_mean, dtype=np.float64))
    if len(inc) == 1:
        inc = np.full(len(spec.inclusion_layout), inc[0])
    means = np.concatenate([[spec.matrix_coeff_mean], inc])
    b = _load_vector(spec.grid)
    rng = _philox(spec.seed)
    for _ in range(count):
        coeffs = np.array([_redraw_positive(rng, m, spec.rel_std) for m in means])
        yield assemble_diffusion(coeffs[materials]), b.copy()


# ---------------------------------------------------------------------------
# prescribed spectra and random SPD (test inputs)


@dataclass(frozen=True)
class SpectrumSpec:
    """Exactly prescribed spectrum in a seeded orthogonal basis
    (``problems.py:192-203``)."""

    eigenvalues: tuple
    seed: int = 0

    def __post_init__(self):
        vals = tuple(float(v) for v in self.eigenvalues)
        object.__setattr__(self, "eigenvalues", vals)
        if len(vals) == 0 or any(v <= 0.0 for v in vals):
            raise ContractViolation("eigenvalues must be positive")


def generate_prescribed_spectrum(spec: SpectrumSpec) -> SparseSpdMatrix:
    """A = Q diag(lam) Q^T, dense pattern (``problems.py:206-216``)."""
    lam = np.asarray(spec.eigenvalues, dtype=np.float64)
    n = len(lam)
    if n > 500:
        raise ContractViolation("dense-pattern generation limited to n <= 500")
    Q, _ = np.linalg.qr(_philox(spec.seed).standard_normal((n, n)))
    A = (Q * lam) @ Q.T
    return SparseSpdMatrix.from_dense(0.5 * (A + A.T), keep_zeros=True)


def random_spd(n, rng, condition=100.0):
    """Dense SPD with a geometric spectrum (reference tests/conftest.py:7-12)."""
    lam = np.geomspace(1.0, condition, n)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    A = (Q * lam) @ Q.T
    return 0.5 * (A + A.T)


# ---------------------------------------------------------------------------
# BASELINE.json configs


def shifted_laplacian_sequence(grid=128, count=10, seed=0, shift=0.05):
    """Config 1: A^(k) = A0 + diag(shift*k*u), u ~ U(0,1)^n drawn once,
    b^(k) ~ N(0,1)^n drawn after u, k = 0..count-1."""
    A0 = assemble_diffusion(np.ones((grid, grid)))
    n = A0.n
    rng = _philox(seed)
    u = rng.uniform(0.0, 1.0, n)
    bs = [rng.standard_normal(n) for _ in range(count)]
    ro, ci, va0 = A0.row_offsets, A0.col_indices, A0.values
    rows = np.repeat(np.arange(n), np.diff(ro))
    diag_pos = np.flatnonzero(rows == ci)
    out = []
    for k in range(count):
        va = va0.copy()
        va[diag_pos] = va0[diag_pos] + shift * k * u
        out.append((SparseSpdMatrix(n, ro, ci, va, validate=False), bs[k]))
    return out


def lognormal_diffusion_sequence(grid=256, count=20, seed=0, sigma=2.0,
                                 noise_sigma=0.05, device=False):
    """Config 4: 7-point diffusion, kappa0 ~ lognormal(0, sigma) per cell,
    kappa^(k) = kappa0 * lognormal(0, noise) independent per k, b ~ N(0,1)
    drawn once.  Yields lazily (each matrix is ~1.4 GB at 256^3)."""
    shape = (grid,) * 3 if np.ndim(grid) == 0 else tuple(grid)
    rng = _philox(seed)
    kappa0 = rng.lognormal(0.0, sigma, shape)
    n = int(np.prod(shape))
    b = rng.standard_normal(n)
    for _ in range(count):
        kappa = kappa0 * rng.lognormal(0.0, noise_sigma, shape)
        yield (assemble_diffusion_device(kappa) if device else assemble_diffusion(kappa, validate=False)), b.copy()


# ---------------------------------------------------------------------------
# Q1 trilinear hex elasticity (configs 2, 3, 5) — new, no reference generator


def _q1_element_stiffness(h, nu):
    """24x24 stiffness of a cube of side h, E = 1, 2x2x2 Gauss.

    Local node (a, b, c) in {0,1}^3 has index 4a + 2b + c; dof = 3*node + comp.
    The result is exactly symmetrized.
    """
    lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = 1.0 / (2.0 * (1.0 + nu))
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[np.arange(3), np.arange(3)] += 2.0 * mu
    D[np.arange(3, 6), np.arange(3, 6)] = mu
    g = 0.5 / math.sqrt(3.0)
    gauss = [0.5 - g, 0.5 + g]
    corners = [(a, b, c) for a in (0, 1) for b in (0, 1) for c in (0, 1)]
    Ke = np.zeros((24, 24))
    for xi, eta, zeta in product(gauss, gauss, gauss):
        dN = np.zeros((8, 3))  # derivatives in physical coords (cube side h)
        for i, (a, b, c) in enumerate(corners):
            fx = xi if a else 1.0 - xi
            fy = eta if b else 1.0 - eta
            fz = zeta if c else 1.0 - zeta
            sx = 1.0 if a else -1.0
            sy = 1.0 if b else -1.0
            sz = 1.0 if c else -1.0
            dN[i] = (sx * fy * fz / h, fx * sy * fz / h, fx * fy * sz / h)
        B = np.zeros((6, 24))
        for i in range(8):
            dx, dy, dz = dN[i]
            B[0, 3 * i] = dx
            B[1, 3 * i + 1] = dy
            B[2, 3 * i + 2] = dz
            B[3, 3 * i] = dy
            B[3, 3 * i + 1] = dx
            B[4, 3 * i + 1] = dz
            B[4, 3 * i + 2] = dy
            B[5, 3 * i] = dz
            B[5, 3 * i + 2] = dx
        Ke += B.T @ D @ B * (h ** 3 / 8.0)
    return 0.5 * (Ke + Ke.T)


def elasticity_q1(nelem, E=None, nu=0.3, validate=None):
    """Q1 hex linear elasticity on the unit cube, ``nelem^3`` elements, nodes on
    the face x = 0 clamped (eliminated).  ``E`` is None (= 1) or an array of
    shape ``(nelem,)*3`` indexed ``[ex, ey, ez]``.

    Free node (ix, iy, iz), ix = 1..N, has id ``((ix-1)(N+1) + iy)(N+1) + iz``
    and dofs ``3 id + comp``, so rows are x-slabs (contiguous for row sharding).
    The full 27-node block pattern is kept (explicit zeros included).  Each
    entry sums its element contributions in increasing element order for both
    (p, q) and (q, p), so the values are bitwise symmetric.
    """
    N = int(nelem)
    h = 1.0 / N
    Ke = _q1_element_stiffness(h, nu)
    if E is None:
        Epad = np.ones((N, N, N))
    else:
        Epad = np.asarray(E, dtype=np.float64)
        if Epad.shape != (N, N, N):
            raise ContractViolation("E must have shape (nelem,)*3")
    NX, NY, NZ = N, N + 1, N + 1        # free node grid (ix-1, iy, iz)
    nn = NX * NY * NZ
    offsets = [(dx, dy, dz) for dx in (-1, 0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)]
    vals = np.zeros((NX, NY, NZ, 27, 3, 3))
    node_ix = np.arange(1, N + 1)[:, None, None]
    node_iy = np.arange(NY)[None, :, None]
    node_iz = np.arange(NZ)[None, None, :]
    corners = [(a, b, c) for a in (0, 1) for b in (0, 1) for c in (0, 1)]
    # row node p is local corner lp of element e = p - lp; iterate lp in
    # decreasing order so e increases -> same summation order for (q, p)
    for lp in sorted(corners, reverse=True):
        a, b, c = lp
        ex = node_ix - a
        ey = node_iy - b
        ez = node_iz - c
        valid = ((ex >= 0) & (ex < N)) & ((ey >= 0) & (ey < N)) & ((ez >= 0) & (ez < N))
        Ee = np.where(valid,
                      Epad[np.clip(ex, 0, N - 1), np.clip(ey, 0, N - 1), np.clip(ez, 0, N - 1)],
                      0.0)
        ip = 4 * a + 2 * b + c
        for lq in corners:
            d = (lq[0] - a, lq[1] - b, lq[2] - c)
            slot = offsets.index(d)
            iq = 4 * lq[0] + 2 * lq[1] + lq[2]
            block = Ke[3 * ip:3 * ip + 3, 3 * iq:3 * iq + 3]
            vals[:, :, :, slot] += Ee[..., None, None] * block
    # column ids of neighbour nodes; -1 when out of the free grid
    gx = np.arange(NX)[:, None, None]
    gy = np.arange(NY)[None, :, None]
    gz = np.arange(NZ)[None, None, :]
    ncols = np.full((NX, NY, NZ, 27), -1, dtype=np.int64)
    for slot, (dx, dy, dz) in enumerate(offsets):
        qx, qy, qz = gx + dx, gy + dy, gz + dz
        ok = (qx >= 0) & (qx < NX) & (qy >= 0) & (qy < NY) & (qz >= 0) & (qz < NZ)
        ncols[..., slot] = np.where(ok, (qx * NY + qy) * NZ + qz, -1)
    ncols = ncols.reshape(nn, 27)
    vals = vals.reshape(nn, 27, 3, 3)
    # row (p, i): columns (q_slot, j) for slot ascending then j
    cols = np.where(ncols[:, None, :, None] >= 0,
                    3 * ncols[:, None, :, None] + np.arange(3)[None, None, None, :], -1)
    cols = np.broadcast_to(cols, (nn, 3, 27, 3)).reshape(3 * nn, 81)
    v = vals.transpose(0, 2, 1, 3).reshape(3 * nn, 81)   # [p, i, slot, j]
    del vals
    n = 3 * nn
    if validate is None:
        validate = n <= 100_000
    return _stencil_csr(n, cols, v, validate)


def _face_load(N, traction):
    """Consistent load of a bilinear nodal traction field on the face x = 1:
    f = (M1 (x) M1) t per component, M1 the 1-D P1 mass with h = 1/N."""
    h = 1.0 / N

    def mass1d(t, axis):
        out = np.zeros_like(t)
        sl = [slice(None)] * t.ndim

        def s(i):
            sl2 = list(sl)
            sl2[axis] = i
            return tuple(sl2)
        out += (2.0 * h / 6.0) * t
        # interior nodes get 2h/6 from each side: total 4h/6; ends 2h/6
        inner = slice(1, -1)
        out[s(inner)] += (2.0 * h / 6.0) * t[s(inner)]
        out[s(slice(0, -1))] += (h / 6.0) * t[s(slice(1, None))]
        out[s(slice(1, None))] += (h / 6.0) * t[s(slice(0, -1))]
        return out
    return mass1d(mass1d(traction, 0), 1)


def elasticity_rhs(N, rng):
    """N(0,1) nodal traction 3-vectors on the face x = 1, integrated with the
    consistent face mass; zero elsewhere."""
    t = rng.standard_normal((N + 1, N + 1, 3))
    f = _face_load(N, t)
    b = np.zeros((N, N + 1, N + 1, 3))
    b[N - 1] = f
    return b.reshape(-1)


def elasticity_sequence(nelem, count, seed=0, kind="fixed", nu=0.3, device=False):
    """Configs 2/3/5.

    * ``kind="fixed"`` (config 2): E = 1, ``count`` independent traction RHS.
    * ``kind="softening"`` (config 3): E scaled by 0.6^k for elements whose
      centroid is within 0.03 k of the cube centre; b^(k) = b0 + 0.01 k N(0,1).
    * ``kind="lognormal_softening"`` (config 5): base E ~ lognormal(0,1) per
      element, then the config-3 softening sequence.
    ``device=True`` assembles each operator in HBM (``elasticity_q1_device``).
    Yields lazily.
    """
    N = int(nelem)
    rng = _philox(seed)
    if kind == "fixed":
        A = elasticity_q1_device(N, nu=nu) if device else elasticity_q1(N, nu=nu)
        for _ in range(count):
            yield A, elasticity_rhs(N, rng)
        return
    if kind not in ("softening", "lognormal_softening"):
        raise ContractViolation(f"unknown elasticity sequence kind {kind!r}")
    E0 = rng.lognormal(0.0, 1.0, (N, N, N)) if kind == "lognormal_softening" else np.ones((N, N, N))
    b0 = elasticity_rhs(N, rng)
    c = (np.arange(N) + 0.5) / N
    r2 = (c[:, None, None] - 0.5) ** 2 + (c[None, :, None] - 0.5) ** 2 + (c[None, None, :] - 0.5) ** 2
    r = np.sqrt(r2)
    for k in range(count):
        E = np.where(r <= 0.03 * k, E0 * (0.6 ** k), E0)
        b = b0 + 0.01 * k * rng.standard_normal(b0.shape[0])
        yield (elasticity_q1_device(N, E=E, nu=nu) if device else elasticity_q1(N, E=E, nu=nu, validate=False)), b


def config_systems(config, reduced=False, device=False):
    """(systems iterable, settings dict) for BASELINE.json config 1..5.

    ``reduced`` swaps in the oracle-sized analogs: elasticity
    16^3 / 24^3, diffusion 64^3.  ``device`` assembles configs 2-5 in HBM.
    """
    if config == 1:
        return shifted_laplacian_sequence(), dict(tol=1e-8, epsilon=1e-10, nc_limit=21)
    if config == 2:
        N = 16 if reduced else 64
        return elasticity_sequence(N, 20, kind="fixed", device=device), dict(tol=1e-8, epsilon=1e-10, nc_limit=61)
    if config == 3:
        N = 24 if reduced else 96
        return elasticity_sequence(N, 15, kind="softening", device=device), dict(tol=1e-8, epsilon=1e-10, nc_limit=81)
    if config == 4:
        g = 64 if reduced else 256
        return lognormal_diffusion_sequence(g, 20, device=device), dict(tol=1e-8, epsilon=1e-10, nc_limit=21)
    if config == 5:
        N = 16 if reduced else 160
        return elasticity_sequence(N, 10, kind="lognormal_softening", device=device), dict(tol=1e-8, epsilon=1e-10, nc_limit=101)
    raise ContractViolation(f"unknown config {config}")
