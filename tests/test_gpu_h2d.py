"""Host -> device staging of a host cost matrix (csrc/lsk_h2d.cu, lsk_h2d_cost_f32):
the one fp64 -> fp32 rounding of solver.py:253 done by the library's worker
threads must be bit-identical to a round-to-nearest-even cast, in the padded
device layout, for every chunk size, with and without the non-temporal store
path, for ragged widths and special values."""

import os

import numpy as np
import pytest
import torch

from paper_2605_00837_b200.solver import to_device_cost

pytestmark = pytest.mark.gpu


def _special(rng, n, m):
    A = rng.normal(0.0, 1.0, (n, m)) * 10.0 ** rng.integers(-45, 40, (n, m))
    flat = A.reshape(-1)
    k = min(flat.size, 9)
    flat[:k] = [0.0, -0.0, np.inf, -np.inf, np.nan, 1e-310, 3.4028235677973366e38, 3.5e38, 1.401298464324817e-45][:k]
    return A


@pytest.mark.parametrize("nt", ["1", "0"])
@pytest.mark.parametrize("chunk_kb", ["64", "1024"])
@pytest.mark.parametrize("n,m", [(1, 1), (3, 5), (17, 4), (129, 1027), (600, 2048)])
def test_h2d_rounding_bitwise(monkeypatch, nt, chunk_kb, n, m):
    monkeypatch.setenv("LSK_H2D_NT", nt)
    monkeypatch.setenv("LSK_H2D_CHUNK_KB", chunk_kb)
    A = _special(np.random.default_rng(n * 7919 + m), n, m)
    dev = to_device_cost(A)
    torch.cuda.synchronize()
    got = dev.data.cpu().numpy()
    ldc = (m + 3) // 4 * 4
    assert got.shape == (n, ldc)
    want = A.astype(np.float32)
    assert np.array_equal(got[:, :m].view(np.uint32), want.view(np.uint32))
    assert not got[:, m:].any()


def test_h2d_noncontiguous_and_f32(monkeypatch):
    rng = np.random.default_rng(5)
    base = rng.uniform(0, 2, (300, 2 * 515))
    A = base[:, ::2]  # strided view: copied to a contiguous array first
    dev = to_device_cost(A)
    torch.cuda.synchronize()
    assert np.array_equal(dev.data.cpu().numpy()[:, :515], A.astype(np.float32))
    B = rng.uniform(0, 2, (70, 33)).astype(np.float32)
    dev = to_device_cost(B)
    torch.cuda.synchronize()
    assert np.array_equal(dev.data.cpu().numpy()[:, :33], B)
