"""CPU emulation of the row-sharded APCG (test infrastructure).

Runs the exact communication schedule of the GPU sharded solve
(csrc/pcg.cu solve_impl with a halo; paper_1301_7530_b200/distributed.py) with
numpy per rank and torch.distributed (gloo) for the transport:

  per solve : x0 = C G^-1 allreduce(C^T b); halo(x0); r = b - A x0; allreduce(||r||^2, ||b||^2)
  per iter  : halo(w_j) -> SpMV -> allreduce (w,Aw) -> x/r update -> allreduce(||r||^2, AC^T y)
              -> z -> allreduce((r,z), AW^T z, AW^T w_j) -> w update
  build     : halo + SpMV per basis column, G = allreduce(C_loc^T AC_loc), replicated Cholesky

The algorithm per rank is the reference's (solver.py:193-290) restricted to
owned rows; the halo plan under test is the package's own
(``distributed.build_local_system``).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg
import scipy.sparse
import torch
import torch.distributed as dist


class Shard:
    def __init__(self, ro, lci, va, plan):
        self.plan = plan
        self.n = plan.n_local
        self.n_ext = plan.n_local + plan.n_ghost
        self.A = scipy.sparse.csr_matrix((va, lci, ro), shape=(self.n, self.n_ext))

    def halo(self, v):
        """Owned vector -> owned + ghost entries (isend/irecv per peer)."""
        p = self.plan
        ext = np.zeros(self.n_ext)
        ext[:self.n] = v
        reqs, bufs = [], []
        for q in range(p.nranks):
            if q == p.rank:
                continue
            s0, s1 = p.send_off[q], p.send_off[q + 1]
            r0, r1 = p.recv_off[q], p.recv_off[q + 1]
            if s1 > s0:
                t = torch.from_numpy(np.ascontiguousarray(v[p.send_idx[s0:s1]]))
                bufs.append(t)
                reqs.append(dist.isend(t, q))
            if r1 > r0:
                t = torch.empty(r1 - r0, dtype=torch.float64)
                bufs.append((t, r0, r1))
                reqs.append(dist.irecv(t, q))
        for rq in reqs:
            rq.wait()
        for b in bufs:
            if isinstance(b, tuple):
                t, r0, r1 = b
                ext[self.n + r0:self.n + r1] = t.numpy()
        return ext

    def spmv(self, v):
        return self.A @ self.halo(v)


def allreduce(a):
    t = torch.from_numpy(np.array(a, dtype=np.float64, ndmin=1).copy())
    dist.all_reduce(t)
    return t.numpy()


def sharded_apcg(S: Shard, inv_diag, C, b, tol, max_iters, reorthogonalize=True):
    """Returns (x_local, iterations, alphas, converged)."""
    n_c = C.shape[1]
    if n_c:
        AC = np.column_stack([S.spmv(C[:, k]) for k in range(n_c)])
        G = allreduce(C.T @ AC).reshape(n_c, n_c)
        G = 0.5 * (G + G.T)
        L = np.linalg.cholesky(G)

        def coarse(u):
            return scipy.linalg.cho_solve((L, True), u)
        x = C @ coarse(allreduce(C.T @ b))
        r = b - S.spmv(x)
    else:
        AC = np.zeros((S.n, 0))
        x = np.zeros(S.n)
        r = b.copy()
    r0, bn = np.sqrt(allreduce([r @ r, b @ b]))
    if r0 == 0.0 or r0 <= 1e-13 * bn:
        return x, 0, [], True

    def precond(v):
        y = inv_diag * v
        if n_c:
            y = y - C @ coarse(allreduce(AC.T @ y))
        return y
    z = precond(r)
    rz = allreduce(r @ z)[0]
    w = z.copy()
    W, AW, waw, alphas = [], [], [], []
    for it in range(max_iters):
        Aw = S.spmv(w)
        wAw = allreduce(w @ Aw)[0]
        alpha = rz / wAw
        alphas.append(alpha)
        x = x + alpha * w
        r = r - alpha * Aw
        rn = np.sqrt(allreduce(r @ r)[0])
        if reorthogonalize:
            W.append(w)
            AW.append(Aw)
            waw.append(wAw)
        if rn <= tol * r0:
            return x, it + 1, alphas, True
        z = precond(r)
        rz_new = allreduce(r @ z)[0]
        beta = rz_new / rz
        w = z + beta * w
        if reorthogonalize:
            Wm, AWm = np.column_stack(W), np.column_stack(AW)
            w = w - Wm @ (allreduce(AWm.T @ w) / np.asarray(waw))
        rz = rz_new
    return x, max_iters, alphas, False
