import os

# golden fixtures were captured single-threaded; BLAS bits depend on it
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import json  # noqa: E402
import sys  # noqa: E402

from threadpoolctl import threadpool_limits  # noqa: E402

# numpy may already be imported by a pytest plugin; pin BLAS threads at runtime
_BLAS_LIMIT = threadpool_limits(limits=1)
os.environ["OPENBLAS_NUM_THREADS"] = "1"

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running parity case")


def golden_json(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        return json.load(fh)


def golden_npz(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


@pytest.fixture(scope="session")
def gpu():
    """The loaded C-ABI library on a visible GPU (fails loudly otherwise)."""
    from paper_2201_09827_b200 import _lib

    return _lib.require_gpu()
