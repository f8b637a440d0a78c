"""The deterministic reductions (reference reduction.py) and plan diagnostics
(solver.py:461-519) on the GPU against reference outputs
(tests/golden/make_golden_reduction.py). Max and sum must be bit-identical for
every ReductionPlan (signed zeros and NaN included); log-sum-exp within the
exponential's ulps."""

import numpy as np
import pytest
from conftest import golden

import paper_2605_00837_b200 as lsk
from paper_2605_00837_b200 import reduction as RD

pytestmark = pytest.mark.gpu


def _bits(a):
    a = np.array(a, copy=True)
    a[np.isnan(a)] = np.nan  # canonical NaN
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def _cases():
    G = golden("reduction")
    return G, sorted(k[4:] for k in G.files if k.startswith("out:") and "|" in k[4:] and not k.startswith("out:view"))


def test_reductions_match_reference(cuda_ok):
    G, keys = _cases()
    assert len(keys) > 150
    for key in keys:
        name, w, B, op = key.split("|")
        A = G["in:" + name]
        plan = lsk.ReductionPlan(int(w), int(B))
        cols = name.startswith("cols")
        fn = {("max", False): RD.reduce_max_rows, ("sum", False): RD.reduce_sum_rows,
              ("lse", False): RD.log_sum_exp_rows, ("max", True): RD.reduce_max_cols,
              ("sum", True): RD.reduce_sum_cols, ("lse", True): RD.log_sum_exp_cols}[(op, cols)]
        got, want = fn(A, plan), G["out:" + key]
        assert got.dtype == want.dtype, key
        if op in ("max", "sum"):
            np.testing.assert_array_equal(_bits(got), _bits(want), err_msg=key)
        else:
            rtol = 2e-6 if A.dtype == np.float32 else 1e-13
            np.testing.assert_allclose(got, want, rtol=rtol, atol=0, equal_nan=True, err_msg=key)


def test_view_reductions(cuda_ok):
    G = golden("reduction")
    v = G["in:rows_f64"][0]
    assert RD.reduce_max(v) == G["out:view|max"]
    assert RD.reduce_sum(v) == G["out:view|sum"]
    assert abs(RD.log_sum_exp(v) - G["out:view|lse"]) <= 1e-13 * abs(G["out:view|lse"])
    with pytest.raises(lsk.EmptyView):
        RD.reduce_sum(np.zeros(0))


def test_diagnostics_match_reference(cuda_ok):
    G = golden("diagnostics")
    C = lsk.CostMatrix(values=G["C"])
    mu, nu = lsk.make_distribution(G["wa"]), lsk.make_distribution(G["wb"])
    for prec, tol in (("single", 2e-7), ("double", 1e-15)):
        plan = lsk.TransportPlan(values=G[f"{prec}_plan"])
        k = lsk.kkt_residual(C, mu, nu, plan, G[f"{prec}_alpha"], G[f"{prec}_beta"], 0.05)
        assert abs(k - float(G[f"{prec}_kkt"])) <= tol, (prec, k, float(G[f"{prec}_kkt"]))
        o = lsk.regularized_objective(C, mu, nu, plan, 0.05)
        assert abs(o - float(G[f"{prec}_obj"])) <= 1e-12 * abs(float(G[f"{prec}_obj"]))
    got = np.array([lsk.contraction_rate_bound(R, e) for R, e in ((1.0, 0.1), (0.5, 0.01), (0.0, 1.0))])
    np.testing.assert_array_equal(got, G["crb"])
    empty = lsk.TransportPlan(values=np.zeros((40, 50)))
    assert lsk.kkt_residual(C, mu, nu, empty, G["double_alpha"], G["double_beta"], 0.05) == 0.0


def test_reduction_plan_validation():
    with pytest.raises(ValueError):
        lsk.ReductionPlan(0, 1)
    with pytest.raises(ValueError):
        lsk.ReductionPlan(32, 48)
