"""Run the first ITERS APCG iterations of system 0 of a BASELINE config on
the device (the bench's build, graphs on) as an ncu capture target:

  ncu --set full -k regex:precond_kernel --launch-skip S --launch-count 1 \
      python tools/ncu_target.py 3 1000

Prints the per-launch algorithmic bytes of the K3 / K5 launches at the
captured iteration j so traffic / algorithmic can be formed.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1301_7530_b200 as rcg  # noqa: E402
from paper_1301_7530_b200 import problems  # noqa: E402

config = int(sys.argv[1]) if len(sys.argv) > 1 else 3
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
nelem = {2: 64, 3: 96}[config]
kind = {2: "fixed", 3: "softening"}[config]
A, b = next(problems.elasticity_sequence(nelem, 1, seed=0, kind=kind, device=True))
bd = torch.from_numpy(b).cuda()
D = rcg.build_deflation(A, np.zeros((A.n, 0)))
cfg = rcg.SolveConfig(tol=1e-8, max_iters=iters, reorthogonalize=True)
x, tr = rcg.apcg_solve(A, rcg.Preconditioner.jacobi(A), D, bd, cfg)
n = A.n
alg = {"n": n, "nnz": A.nnz, "iterations": tr.iterations,
       "precond_bytes_at_j": "8 n (2 + 1 + 0 + 1 + (j + 1))  [r, inv_diag, z write, w_j, AW[:, 0..j]]",
       "wupdate_bytes_at_j": "8 n (3 + (j + 1))  [z, w_j, w_{j+1} write, W[:, 0..j]]"}
print(json.dumps(alg))
