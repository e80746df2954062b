"""Multi-process (gloo, world_size 2, CPU) tests of the row-sharded path's
host logic: partition, halo plan, and the sharded communication schedule
emulated in numpy, checked against the serial oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1301_7530_b200 import problems
from paper_1301_7530_b200.distributed import partition_rows


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(kind):
    if kind == "elasticity":
        A, b = next(problems.elasticity_sequence(5, 1, kind="fixed"))
        return A, b, 3
    kappa = np.exp(np.random.default_rng(7).standard_normal((12, 9, 7)))
    A = problems.assemble_diffusion(kappa)
    b = np.random.default_rng(8).standard_normal(A.n)
    return A, b, 1


def _worker(rank, world, port, kind, n_c, out_dir):
    import torch.distributed as dist
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_1301_7530_b200.distributed import build_local_system, partition_rows
    from sharded_emulation import Shard, sharded_apcg
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        A, b, align = _problem(kind)
        bounds = partition_rows(A.row_offsets, world, align=align)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        s, e = A.row_offsets[r0], A.row_offsets[r1]
        ro = A.row_offsets[r0:r1 + 1]
        ro_l, lci, va, plan = build_local_system(ro, A.col_indices[s:e], A.values[s:e], bounds, rank)
        # plan symmetry: what I receive from q is what q sends me
        counts = [None] * world
        dist.all_gather_object(counts, (plan.send_off.tolist(), plan.recv_off.tolist()))
        for q in range(world):
            if q == rank:
                continue
            sent_by_q = counts[q][0][rank + 1] - counts[q][0][rank]
            assert sent_by_q == plan.recv_off[q + 1] - plan.recv_off[q]
        S = Shard(ro_l, lci, va, plan)
        diag = A.to_dense().diagonal() if A.n < 3000 else None
        inv = 1.0 / diag[r0:r1]
        rng = np.random.default_rng(11)
        Cg = rng.standard_normal((A.n, n_c))
        x, m, alphas, conv = sharded_apcg(S, inv, Cg[r0:r1], b[r0:r1], 1e-9, 500)
        np.save(os.path.join(out_dir, f"x{rank}.npy"), x)
        np.save(os.path.join(out_dir, f"meta{rank}.npy"), np.array([m, int(conv), r0, r1] + list(alphas[:5])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,n_c", [("elasticity", 0), ("elasticity", 3), ("diffusion", 2)])
def test_sharded_schedule_matches_serial_oracle(tmp_path, kind, n_c):
    from oracle import recycg_oracle as orc
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), kind, n_c, str(tmp_path)), nprocs=world, join=True)
    A, b, _ = _problem(kind)
    Cg = np.random.default_rng(11).standard_normal((A.n, n_c))
    inv = 1.0 / orc.diagonal(A)
    xo, to = orc.apcg_solve(A, inv, orc.build_deflation(A, Cg), b, 1e-9, 500)
    xs, metas = [], []
    for r in range(world):
        xs.append(np.load(tmp_path / f"x{r}.npy"))
        metas.append(np.load(tmp_path / f"meta{r}.npy"))
    x = np.concatenate(xs)
    assert metas[0][0] == metas[1][0]                      # replicated stopping decision
    assert abs(metas[0][0] - to.iterations) <= max(1, 0.02 * to.iterations)
    np.testing.assert_allclose(metas[0][4:], to.alphas[:len(metas[0]) - 4], rtol=1e-10)
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)


def test_partition_rows_balanced_and_aligned():
    A = problems.elasticity_q1(6)
    for P in (2, 3, 4, 8):
        bd = partition_rows(A.row_offsets, P, align=3)
        assert bd[0] == 0 and bd[-1] == A.n and np.all(np.diff(bd) >= 0)
        assert np.all(bd % 3 == 0)
        nnz = np.diff(A.row_offsets[bd])
        assert nnz.max() <= 1.2 * nnz.mean() + 81 * 3


@pytest.mark.parametrize("kind", ["elasticity", "diffusion"])
def test_slab_local_block_plus_ghost_remainder(kind):
    """The slab SpMV split used on the device (spmv.cu dia kernel + rem_body):
    rows of a slab = (local-local block) x_local + (ELL ghost-column remainder)
    x_ghost.  The local-local block of every slab is symmetric (so it can take
    the symmetric block-DIA copy), the remainder keeps CSR order, pads are
    zeros, and the two parts reproduce the global product's slab rows."""
    import scipy.sparse as sp
    from paper_1301_7530_b200.core import ghost_remainder_ell
    from paper_1301_7530_b200.distributed import local_systems_all
    A, _, align = _problem(kind)
    G = sp.csr_matrix((A.values, A.col_indices, A.row_offsets), shape=(A.n, A.n))
    x = np.random.default_rng(11).standard_normal(A.n)
    y = G @ x
    bounds = partition_rows(A.row_offsets, 3, align=align)
    for r, (ro, lci, va, plan) in enumerate(local_systems_all(A.row_offsets, A.col_indices, A.values, bounds)):
        nl = plan.n_local
        S = sp.csr_matrix((va, lci, ro), shape=(nl, nl + plan.n_ghost))
        LL = S[:, :nl]
        assert abs(LL - LL.T).max() == 0.0                      # principal submatrix: still symmetric
        ids, eci, eva = ghost_remainder_ell(nl, ro, lci, va)
        assert eci.dtype == np.int32 and eci.shape == eva.shape and eci.min() >= nl
        assert np.count_nonzero(eva) <= S[:, nl:].nnz and len(ids) == len(np.unique(S[:, nl:].nonzero()[0]))
        xe = np.concatenate([x[bounds[r]:bounds[r + 1]], x[plan.ghost_global]])
        t = np.zeros(nl)
        for e in range(eci.shape[0]):                           # entry by entry, as rem_body
            t[ids] += eva[e] * xe[eci[e]]
        got = LL @ xe[:nl] + t
        want = y[bounds[r]:bounds[r + 1]]
        np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-13 * np.abs(want).max())


@pytest.mark.parametrize("kind", ["elasticity", "diffusion"])
def test_virtual_slab_system_is_the_same_operator(kind):
    """distributed.virtual_slab_system (two virtual slabs in one rank, the
    one-GPU stand-in for a peer halo): with the ghost region filled from the
    rank's own entries the extended local system reproduces A x, the plan
    sends exactly the ghosts it receives, and the local-local block is
    block-diagonal in the two slabs (so it keeps the symmetric DIA format)."""
    import scipy.sparse as sp
    from paper_1301_7530_b200.distributed import virtual_slab_system
    A, _, align = _problem(kind)
    n = A.n
    cut = align * ((n // align) // 2)
    ro, lci, va, plan = virtual_slab_system(A.row_offsets, A.col_indices, A.values, cut)
    assert plan.nranks == 1 and plan.n_local == n and plan.n_ghost > 0
    assert np.array_equal(plan.send_idx, plan.ghost_global) and plan.send_off[-1] == plan.recv_off[-1] == plan.n_ghost
    S = sp.csr_matrix((va, lci, ro), shape=(n, n + plan.n_ghost))
    LL = S[:, :n].tocsr()
    assert abs(LL - LL.T).max() == 0.0
    assert LL[:cut, cut:].nnz == 0 and LL[cut:, :cut].nnz == 0
    G = sp.csr_matrix((A.values, A.col_indices, A.row_offsets), shape=(n, n))
    x = np.random.default_rng(12).standard_normal(n)
    xe = np.concatenate([x, x[plan.send_idx]])               # the self exchange
    np.testing.assert_allclose(S @ xe, G @ x, rtol=1e-13, atol=1e-13 * np.abs(G @ x).max())
