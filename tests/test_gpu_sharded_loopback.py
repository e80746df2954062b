"""The row-sharded CUDA path with R = 2 and 3 ranks on ONE B200: ranks are
host threads (own stream + rcg context) joined by the single-process loopback
transport (include/rcg.h rcg_loop_group_create).  Same partition, halo plans,
kernels and collective placement as the NCCL path; results must match the
unsharded solve (iterations +-1, x to 1e-10 relative) and the sharded
sequence must match the unsharded sequence (iterations +-2 %)."""
import threading

import numpy as np
import pytest

import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import distributed as Dm
from paper_1301_7530_b200 import problems

pytestmark = pytest.mark.gpu


def _run_ranks(nranks, fn):
    import torch
    group = Dm.LoopbackGroup(nranks)
    out, errs = [None] * nranks, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                Dm.init_loopback(group, r)
                out[r] = fn(r)
                s.synchronize()
        except Exception as exc:  # pragma: no cover - surfaced below
            errs.append((r, repr(exc)))
    th = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    group.close()
    assert not errs, errs
    return out


@pytest.mark.parametrize("kind", ["elasticity", "diffusion"])
def test_slab_keeps_dia_format(kind):
    """A row slab of a grid operator streams the symmetric block-DIA copy of its
    local-local block plus a ghost-column remainder list (rcg_csr.rem_*), and
    its SpMV over [local | ghosts] equals the global product's slab rows."""
    import torch
    if kind == "elasticity":
        A, _ = next(problems.elasticity_sequence(7, 1, kind="fixed"))
        align, b = 3, 3
    else:
        A = problems.assemble_diffusion(np.exp(np.random.default_rng(3).standard_normal((20, 16, 12))))
        align, b = 1, 1
    x = np.random.default_rng(6).standard_normal(A.n)
    y = A @ x
    bounds = Dm.partition_rows(A.row_offsets, 3, align=align)
    systems = Dm.local_systems_all(A.row_offsets, A.col_indices, A.values, bounds)
    for r, (ro, lci, va, plan) in enumerate(systems):
        S = Dm.ShardedMatrix(ro, lci, va, plan, A.n)
        h = S.device_csr().struct
        assert h.dia_count > 0 and h.dia_block == b and h.rem_rows > 0
        xe = torch.from_numpy(np.concatenate([x[bounds[r]:bounds[r + 1]], x[plan.ghost_global]])).cuda()
        ye = torch.zeros(plan.n_local, dtype=torch.float64, device="cuda")
        from paper_1301_7530_b200 import _lib
        ctx = _lib.context()
        ctx.check(ctx.lib.rcg_spmv(ctx.h, _lib.C.byref(h), _lib.ptr(xe), _lib.ptr(ye)), "spmv")
        want = y[bounds[r]:bounds[r + 1]]
        np.testing.assert_allclose(ye.cpu().numpy(), want, rtol=1e-13, atol=1e-13 * np.abs(want).max())


@pytest.mark.parametrize("kind,nranks,n_c", [("elasticity", 2, 0), ("elasticity", 3, 4), ("diffusion", 2, 3)])
def test_sharded_solve_matches_unsharded(kind, nranks, n_c):
    if kind == "elasticity":
        A, b = next(problems.elasticity_sequence(7, 1, kind="fixed"))
        align = 3
    else:
        A = problems.assemble_diffusion(np.exp(np.random.default_rng(3).standard_normal((20, 16, 12))))
        b = np.random.default_rng(4).standard_normal(A.n)
        align = 1
    C = np.random.default_rng(5).standard_normal((A.n, n_c))
    cfg = rcg.SolveConfig(tol=1e-9, max_iters=3000)
    x_ref, t_ref = rcg.apcg_solve(A, rcg.Preconditioner.jacobi(A), rcg.build_deflation(A, C), b, cfg)
    bounds = Dm.partition_rows(A.row_offsets, nranks, align=align)
    systems = Dm.local_systems_all(A.row_offsets, A.col_indices, A.values, bounds)

    def fn(r):
        ro, lci, va, plan = systems[r]
        S = Dm.ShardedMatrix(ro, lci, va, plan, A.n)
        r0, r1 = int(bounds[r]), int(bounds[r + 1])
        x, tr = rcg.apcg_solve(S, rcg.Preconditioner.jacobi(S), rcg.build_deflation(S, C[r0:r1]), b[r0:r1], cfg)
        return x, tr.iterations, list(tr.alphas[:5])
    res = _run_ranks(nranks, fn)
    x = np.concatenate([r[0] for r in res])
    its = [r[1] for r in res]
    assert len(set(its)) == 1                       # replicated stopping decision
    assert abs(its[0] - t_ref.iterations) <= 1
    np.testing.assert_allclose(res[0][2], t_ref.alphas[:5], rtol=1e-12)
    assert np.linalg.norm(x - x_ref) <= 1e-10 * np.linalg.norm(x_ref)


def test_sharded_srks_sequence_matches_unsharded():
    seq = list(problems.elasticity_sequence(7, 3, kind="fixed"))
    A = seq[0][0]
    cfg = rcg.SolveConfig(tol=1e-8, max_iters=3000)
    strat = rcg.RecycleStrategy("srks", epsilon=1e-10, nc_limit=61)
    ref = rcg.run_sequence(iter(seq), rcg.Preconditioner.jacobi, strat, cfg)
    bounds = Dm.partition_rows(A.row_offsets, 2, align=3)
    systems = Dm.local_systems_all(A.row_offsets, A.col_indices, A.values, bounds)

    def fn(r):
        ro, lci, va, plan = systems[r]
        S = Dm.ShardedMatrix(ro, lci, va, plan, A.n)
        r0, r1 = int(bounds[r]), int(bounds[r + 1])
        rep = rcg.run_sequence(((S, b[r0:r1].copy()) for _, b in seq), rcg.Preconditioner.jacobi, strat, cfg)
        return rep.iterations(), rep.n_c_history()
    res = _run_ranks(2, fn)
    assert res[0] == res[1]
    got, want = res[0][0], ref.iterations()
    assert all(abs(g - w) <= max(1, 0.02 * w) for g, w in zip(got, want)), (got, want)
    assert all(abs(a - b) <= 2 for a, b in zip(res[0][1], ref.n_c_history()))


def test_sharded_trks_sequence_matches_unsharded():
    seq = list(problems.generate_diffusion_sequence(problems.benchmark_spec(seed=0), 3))
    A0 = seq[0][0]
    cfg = rcg.SolveConfig(tol=1e-3, max_iters=3000)
    strat = rcg.RecycleStrategy("trks")
    ref = rcg.run_sequence(iter(seq), rcg.Preconditioner.jacobi, strat, cfg)
    parts = []
    for A, b in seq:
        bounds = Dm.partition_rows(A.row_offsets, 2)
        parts.append((bounds, Dm.local_systems_all(A.row_offsets, A.col_indices, A.values, bounds), b))

    def fn(r):
        systems = []
        for bounds, loc, b in parts:
            ro, lci, va, plan = loc[r]
            r0, r1 = int(bounds[r]), int(bounds[r + 1])
            systems.append((Dm.ShardedMatrix(ro, lci, va, plan, A0.n), b[r0:r1].copy()))
        rep = rcg.run_sequence(iter(systems), rcg.Preconditioner.jacobi, strat, cfg)
        return rep.iterations(), rep.n_c_history()
    res = _run_ranks(2, fn)
    assert res[0] == res[1]
    assert all(abs(g - w) <= max(1, 0.02 * w) for g, w in zip(res[0][0], ref.iterations())), (res[0], ref.iterations())
    assert res[0][1] == ref.n_c_history()
