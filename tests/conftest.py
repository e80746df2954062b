import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))

GOLDEN = REPO / "tests" / "golden"

# The symmetric-DIA SpMV is chosen in production only for operators that
# stream from HBM (12 nnz > 32 MB); the parity suite's small grid operators
# take it too, so every solver test also runs through that format (the CSR
# and sliced-block paths keep their own explicit tests).
import os  # noqa: E402
os.environ.setdefault("RCG_DIA_SMALL", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built librcg.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(autouse=True, scope="session")
def _single_thread_blas():
    # the oracle's GEMVs are tiny; thread fan-out only burns CPU (selection at
    # eps >= 1e-10 is thread-count stable, SURVEY.md §0 finding 2)
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1, user_api="blas"):
            yield
    except ImportError:  # pragma: no cover
        yield


@pytest.fixture
def rng():
    # reference tests/conftest.py:21-23
    return np.random.Generator(np.random.Philox(1234))
