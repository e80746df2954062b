"""Solve-loop trace of one Q1 elasticity system through the 3x3 block-DIA
SpMV, printed as JSON (iterations, alphas, x checksum).  Run twice, with
RCG_DIA3_TMA=0 and =1, by tests/test_gpu_kernels.py::test_dia3_tma_matches:
the operator is large enough (n = 238,521) that every warp of the TMA-staged
kernel streams several tiles through its ring."""
import json
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["RCG_DIA_SMALL"] = "1"
os.environ["RCG_SMALL_N"] = "0"          # kernel-sequence loop (the persistent loop has its own SpMV)
import numpy as np
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems

ne = int(sys.argv[1]) if len(sys.argv) > 1 else 42
rng = np.random.default_rng(7)
A0 = problems.elasticity_q1(ne, E=np.exp(rng.standard_normal((ne,) * 3)))
A = rcg.SparseSpdMatrix(A0.n, A0.row_offsets, A0.col_indices, A0.values, validate=False)
assert A.device_csr().struct.dia_count == 14 and A.device_csr().struct.dia_block == 3
b = rng.standard_normal(A.n)
x, tr = rcg.apcg_solve(A, rcg.Preconditioner.jacobi(A), rcg.build_deflation(A, np.zeros((A.n, 0))), b,
                       rcg.SolveConfig(tol=1e-8, max_iters=80))
x = np.asarray(x)
print(json.dumps({"n": A.n, "iterations": tr.iterations, "alphas": [float(a) for a in tr.alphas],
                  "x_sum": float(np.abs(x).sum()), "x_norm": float(np.linalg.norm(x)),
                  "resid": float(np.linalg.norm(b - A0 @ x))}))
