"""bench.py's JSON contract on a small operator (both arms), and its
row-sharded branch end to end on one GPU (1-rank NCCL communicator with every
collective forced through NCCL, as `torchrun --nproc-per-node 1 ... --shard-one`)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
SMALL = ["--nelem", "16", "--systems", "3", "--steps", "2", "--warmup", "3", "--cpu-iters", "5"]


def _line(cmd, env=None):
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])


def test_bench_line_has_the_contract_keys():
    d = _line([sys.executable, "bench.py", "--gpus", "1", *SMALL, "--no-secondary"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["unit"] == "iters/s" and d["dtype"] == "f64" and d["value"] > 0 and d["gpu_launches"] > 0
    assert "workload" in d["config"] and d["config"]["parallelism"] == "single"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] == "port" and c["cores"] >= 1 and c["value"] > 0 and "sample" in c
    ref = _line([sys.executable, "bench.py", "--impl", "reference", "--gpus", "1", *SMALL, "--ref-seconds", "4"])
    assert ref["impl"] == "reference" and ref["config"] == d["config"] and ref["metric"] == d["metric"]
    assert ref["e2e"]["h2d_bytes_per_step"] == 0 and ref["e2e"]["value"] == ref["value"]


def test_bench_sharded_branch_on_one_rank():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, RCG_COMM_FORCE="1")
    d = _line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
               "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "1", "--shard-one",
               *SMALL, "--no-cpu"], env=env)
    assert d["scaling"] == "strong" and d["config"]["parallelism"].startswith("rows1")
    assert d["config"]["nnz"] > 0 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["phases_profiled_step"] is not None
