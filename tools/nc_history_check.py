import json, sys, os
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
os.environ["RCG_DIA_SMALL"] = "1"
import numpy as np
import paper_1301_7530_b200 as rcg
from paper_1301_7530_b200 import problems
G = json.load(open("tests/golden/reduced_sequences.json"))
for name in ["c2r", "c3r", "c4r_on", "c4r_off", "c5r"]:
    g = G[name]
    systems, st = problems.config_systems(g["config"], reduced=True)
    cfg = rcg.SolveConfig(tol=g["tol"], max_iters=5000, reorthogonalize=g["reorthogonalize"])
    strat = rcg.RecycleStrategy("srks", epsilon=g["epsilon"], nc_limit=g["nc_limit"])
    rep = rcg.run_sequence(iter(list(systems)), rcg.Preconditioner.jacobi, strat, cfg)
    m = min(len(rep.records), len(g["n_c_before"]))
    print(name, "n_c equal:", rep.n_c_history()[:m] == g["n_c_before"][:m], "iters equal:", rep.iterations()[:m] == g["iterations"][:m],
          rep.n_c_history(), g["n_c_before"], flush=True)
for fn, key in (("acceptance6.json", None), ("trks_config1.json", None), ("benchmark_srks.json", "clust10")):
    pass
