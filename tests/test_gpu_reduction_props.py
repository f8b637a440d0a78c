"""Property tests for the GPU reductions (the reference's hypothesis suite
test_reduction.py:65-69 / 106-110 / 200-231, restated): for random shapes,
plans, dtypes and special values the GPU tree max/sum are bit-identical to the
oracle's restatement of the reference tree (itself pinned to the reference by
tests/golden/reduction.npz), column reductions equal row reductions of the
transpose, max equals a sequential scan, and LSE is shift-invariant and
bounded by max <= LSE <= max + log(L)."""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import lsk_oracle as O
import paper_2605_00837_b200 as lsk
from paper_2605_00837_b200 import reduction as RD

pytestmark = pytest.mark.gpu

PLANS = [(32, 256), (1, 1), (64, 128), (4, 12), (8, 8), (3, 9), (16, 512), (2, 2), (5, 5)]
SETTINGS = settings(max_examples=40, deadline=None, derandomize=True,
                    suppress_health_check=[HealthCheck.function_scoped_fixture])


def _bits(a):
    a = np.array(a, copy=True)
    a[np.isnan(a)] = np.nan
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


@st.composite
def arrays(draw):
    R = draw(st.integers(1, 6))
    L = draw(st.integers(1, 3000))
    dt = draw(st.sampled_from([np.float32, np.float64]))
    seed = draw(st.integers(0, 2**31 - 1))
    rng = np.random.default_rng(seed)
    A = (rng.standard_normal((R, L)) * draw(st.sampled_from([1e-3, 1.0, 1e3]))).astype(dt)
    if draw(st.booleans()):
        A[rng.random((R, L)) < 0.05] = -np.inf
    if draw(st.booleans()):
        A[rng.random((R, L)) < 0.05] = 0.0 * -1.0
    return A, draw(st.sampled_from(PLANS))


@SETTINGS
@given(arrays())
def test_tree_max_sum_bitwise_vs_oracle(cuda_ok, case):
    A, (w, B) = case
    plan = lsk.ReductionPlan(w, B)
    np.testing.assert_array_equal(_bits(RD.reduce_max_rows(A, plan)), _bits(O.tree_max_rows(A, w, B)))
    fin = np.where(np.isfinite(A), A, A.dtype.type(0.5))
    np.testing.assert_array_equal(_bits(RD.reduce_sum_rows(fin, plan)), _bits(O.tree_sum_rows(fin, w, B)))
    # columns run the same tree down the strided axis
    np.testing.assert_array_equal(_bits(RD.reduce_sum_cols(np.ascontiguousarray(fin.T), plan)),
                                  _bits(RD.reduce_sum_rows(fin, plan)))
    # max over the tree is a sequential scan
    with np.errstate(invalid="ignore"):
        np.testing.assert_array_equal(RD.reduce_max_rows(A, plan), np.max(A, axis=1))


@SETTINGS
@given(arrays(), st.floats(-50, 50))
def test_lse_properties(cuda_ok, case, shift):
    A, (w, B) = case
    plan = lsk.ReductionPlan(w, B)
    A = np.where(np.isfinite(A), A, A.dtype.type(-np.inf))
    got = RD.log_sum_exp_rows(A, plan)
    want = O.lse_rows(A, w, B)
    rtol = 3e-6 if A.dtype == np.float32 else 1e-13
    np.testing.assert_allclose(got, want, rtol=rtol, atol=rtol)
    mx = np.max(A, axis=1)
    ok = np.isfinite(mx)
    assert (got[ok] >= mx[ok] - rtol * np.abs(mx[ok])).all()
    assert (got[ok] <= mx[ok] + np.log(A.shape[1]) + 1e-5 * (1 + np.abs(mx[ok]))).all()
    assert np.all(got[~ok] == -np.inf)
    if A.dtype == np.float64 and np.all(ok):
        sh = RD.log_sum_exp_rows(A + shift, plan)
        np.testing.assert_allclose(sh, got + shift, rtol=1e-12, atol=1e-9)
