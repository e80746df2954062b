"""The reference's own unit tests, run against the B200 path through the
reference-side binding (``paper_1301_7530_b200.bridge``).

The reference package and its tests are staged, unchanged, by ``build()`` into
``oracle/_ref/recycg_ref.zip`` (test-only data; ``/root/reference`` does not
exist on the GPU box).  A pytest plugin rebinds the reference's seams before its
test modules import them, then ``test_solver.py``, ``test_ritz.py`` and
``test_recycle.py`` run in a subprocess; the plugin records how often each
adapter ran, so a pass cannot come from the reference's own numpy path.
"""
import json
import os
import subprocess
import sys
import zipfile
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
ZIP = REPO / "oracle" / "_ref" / "recycg_ref.zip"

PLUGIN = '''
import json, os
import recycg
from paper_1301_7530_b200 import bridge
_B = bridge.install(recycg)


def pytest_sessionfinish(session, exitstatus):
    with open(os.environ["B200_BRIDGE_CALLS"], "w") as f:
        json.dump(dict(_B.calls), f)
'''

# reference tests that exercise the reference's own numpy internals rather
# than a seam: none so far (kept explicit so a deselection is visible)
DESELECT = []


def _unpack(dst):
    with zipfile.ZipFile(ZIP) as z:
        z.extractall(dst)
    (dst / "b200_bridge_plugin.py").write_text(PLUGIN)


@pytest.mark.gpu
@pytest.mark.skipif(not ZIP.exists(), reason="reference not staged (run build() where /root/reference exists)")
@pytest.mark.parametrize("suite", ["test_solver.py", "test_ritz.py", "test_recycle.py"])
def test_reference_suite_through_bridge(suite, tmp_path):
    _unpack(tmp_path)
    calls = tmp_path / "calls.json"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(tmp_path / "src"), str(tmp_path), str(REPO)]),
               B200_BRIDGE_CALLS=str(calls))
    cmd = [sys.executable, "-m", "pytest", "-p", "b200_bridge_plugin", "-q", "-p", "no:cacheprovider",
           str(tmp_path / "tests" / suite)] + [f"--deselect=tests/{suite}::{t}" for t in DESELECT]
    out = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=1800)
    assert out.returncode == 0, out.stdout[-6000:] + out.stderr[-3000:]
    n = json.loads(calls.read_text())
    assert sum(n.values()) > 0, n
    if suite in ("test_solver.py", "test_recycle.py"):
        assert n.get("apcg_solve", 0) > 10 and n.get("build_deflation", 0) > 10, n
    if suite == "test_ritz.py":
        assert n.get("ritz_pairs", 0) > 0 and n.get("select_converged", 0) > 0, n
    if suite == "test_recycle.py":
        assert n.get("select_spectrum", 0) > 0 and n.get("update_basis_srks", 0) > 0, n
