"""Shared test setup: the `gpu` marker, the oracle on sys.path, fixtures.

The oracle (oracle/lsk_oracle.py) is test infrastructure: tests use it as the
checker, never as the thing under test.
"""

import glob
import hashlib
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU case")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


def golden_names(prefix=""):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def rel_max(x, ref):
    """max|x - ref| / max|ref| (the north-star parity metric)."""
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.abs(ref).max() if ref.size else 0.0
    num = np.abs(x - ref).max() if ref.size else 0.0
    return num / den if den > 0 else num


def rel_max_floor(x, ref, other):
    """Per-potential parity metric max|x - ref| / max|ref|, with the
    denominator floored at 1e-2 max|other| for a potential that is ~0 (a
    uniform-target g on a symmetric problem): there any fp32 rounding of the
    O(|other|) terms would read as a large relative error."""
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    if not ref.size:
        return 0.0
    den = max(np.abs(ref).max(), 1e-2 * np.abs(np.asarray(other, np.float64)).max())
    num = np.abs(x - ref).max()
    return num / den if den > 0 else num


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
