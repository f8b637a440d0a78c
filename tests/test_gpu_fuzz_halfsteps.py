"""Randomised parity sweep of the drop-in half-steps and diagnostics
(update_alpha, update_beta strided/transposed, marginal_error, transport_cost,
materialize_plan) against the oracle restatement of solver.py:76-227/434-458,
in float32 and float64 (the dtype follows the potentials, solver.py:60-65)."""

import numpy as np
import pytest

import lsk_oracle as O
import paper_2605_00837_b200 as lsk

pytestmark = pytest.mark.gpu


def problem(seed):
    rng = np.random.default_rng(9000 + seed)
    n, m = int(rng.integers(1, 500)), int(rng.integers(1, 9000 if seed % 5 == 0 else 1500))
    dt = np.float64 if seed % 2 else np.float32
    C64 = rng.uniform(0, 2, (n, m))
    wa, wb = rng.uniform(0.2, 2.0, n), rng.uniform(0.2, 2.0, m)
    eps = float(rng.choice([1e-3, 1e-2, 5e-2, 0.3]))
    a = (rng.normal(0, 0.05, n) + 0.3).astype(dt)
    b = (rng.normal(0, 0.05, m) + 0.3).astype(dt)
    return C64, wa, wb, eps, a, b, dt


def close(x, ref, rtol, atol):
    """|x - ref| <= rtol |ref| + atol, with equal infinities / NaNs accepted
    (random potentials can overflow the plan the same way in both)."""
    x, ref = float(x), float(ref)
    if not np.isfinite(ref):
        return (np.isnan(ref) and np.isnan(x)) or x == ref
    return abs(x - ref) <= rtol * abs(ref) + atol


@pytest.mark.parametrize("seed", list(range(24)))
def test_halfsteps_vs_oracle(cuda_ok, seed):
    C64, wa, wb, eps, a, b, dt = problem(seed)
    n, m = C64.shape
    cost = lsk.make_cost_matrix(n, m, C64)
    mu, nu = lsk.make_distribution(wa), lsk.make_distribution(wb)
    C = C64.astype(dt)
    inv = dt(1.0) / dt(eps)
    neg = -dt(eps)
    lmu, lnu = mu.log_weights.astype(dt), nu.log_weights.astype(dt)
    rtol = 2e-6 if dt == np.float32 else 1e-12
    with np.errstate(all="ignore"):
        ra = O.row_update(C, b, lnu, inv, neg)
        rb = O.row_update(np.ascontiguousarray(C.T), a, lmu, inv, neg)
        rerr = O.marginal_err(C, mu.weights.astype(dt), lmu, lnu, a, b, inv)
        rcost = O.transport_cost_rows(C, lmu, lnu, a, b, inv)
        rplan = O.plan_values(C, lmu, lnu, a, b, inv)
    ga = lsk.update_alpha(cost, nu, b, eps)
    gb = lsk.update_beta(cost, mu, a, eps)
    gbt = lsk.update_beta(cost, mu, a, eps, transposed_cost=np.ascontiguousarray(C64.T))
    assert ga.dtype == dt and gb.dtype == dt
    sc = max(np.abs(ra).max(), 1e-30)
    assert np.abs(ga - ra).max() <= rtol * sc * 4, (seed, np.abs(ga - ra).max() / sc)
    sc = max(np.abs(rb).max(), 1e-30)
    assert np.abs(gb - rb).max() <= rtol * sc * 4, (seed, np.abs(gb - rb).max() / sc)
    np.testing.assert_array_equal(gb, gbt)  # strided == transposed, bitwise (test_solver.py:101-111)
    err = lsk.marginal_error(cost, mu, nu, a, b, eps)
    assert close(err, rerr, 1e-4, 1e-7 if dt == np.float32 else 1e-14), (seed, err, rerr)
    cst = lsk.transport_cost(cost, mu, nu, a, b, eps)
    assert close(cst, rcost, 1e-5 if dt == np.float32 else 1e-12, 1e-30), (seed, cst, rcost)
    if not np.isfinite(rplan).all():
        with pytest.raises(lsk.NonFiniteResult):
            lsk.materialize_plan(cost, mu, nu, a, b, eps)
        return
    plan = lsk.materialize_plan(cost, mu, nu, a, b, eps)
    assert plan.values.dtype == dt
    np.testing.assert_allclose(plan.values, rplan, rtol=(3e-6 if dt == np.float32 else 1e-13),
                               atol=float(np.abs(rplan).max()) * (1e-7 if dt == np.float32 else 1e-16))
