"""Drop-in fidelity: the reference's own code patterns and assertions, run
unchanged against this package.

* The pipelines' cost composition (applications.py:185-191,
  estimator.py:86-99): ``squared_euclidean_cost`` -> ``value_range`` ->
  ``CostMatrix(values=np.ascontiguousarray(cost.values / cost.values.max()))``
  -> ``solve``.
* The reference tests that run as-is on the hot path: the alpha update vs a
  high-precision oracle (tests/test_solver.py:51-61), status / trace / cap
  semantics (:210-238), bit-identical repeats (:247-257), KKT residual of the
  materialised plan (:345-360), feasibility of a converged plan (:463-474).
"""

import numpy as np
import pytest

import lsk_oracle as O
import paper_2605_00837_b200 as ls
from conftest import golden, rel_max
from paper_2605_00837_b200 import (
    STATUS_CONVERGED,
    CostMatrix,
    ReductionPlan,
    SinkhornConfig,
    generate_grid_problem,
    kkt_residual,
    make_cost_matrix,
    make_distribution,
    materialize_plan,
    solve,
    squared_euclidean_cost,
    update_alpha,
)

pytestmark = pytest.mark.gpu
PLAN = ReductionPlan()


def _pipeline_cost(X, Y):
    """applications.py:185-188, verbatim in structure."""
    cost = squared_euclidean_cost(X, Y)
    if cost.value_range > 0:
        cmax = cost.values.max()
        cost = CostMatrix(values=np.ascontiguousarray(cost.values / cmax))
    return cost


def test_values_have_reference_semantics(cuda_ok):
    rng = np.random.default_rng(3)
    X, Y = rng.uniform(-2, 5, (300, 3)), rng.uniform(0, 1, (211, 3))
    cost = squared_euclidean_cost(X, Y)
    C64 = O.sq_euclidean_cost(X, Y)
    assert cost.values.shape == C64.shape and cost.values.dtype == np.float64
    assert cost.values.max() == C64.max() and cost.values.min() == C64.min()
    assert cost.value_range == float(C64.max() - C64.min())
    np.testing.assert_array_equal(np.asarray(cost.values), C64)
    np.testing.assert_array_equal(np.ascontiguousarray(cost.values / C64.max()), C64 / C64.max())
    np.testing.assert_array_equal(np.asarray(cost.values / 3.0 / 7.0), C64 / 3.0 / 7.0)
    # constant cost: value_range 0, the pipelines leave it unscaled
    Z = np.zeros((4, 2))
    assert squared_euclidean_cost(Z, Z + 1.0).value_range == 0.0


def test_match_pipeline_composition_unchanged(cuda_ok):
    """The rigid-pair fixture through the reference's composition, single precision."""
    z = golden("rigid2048_eps1e-3_k200")
    X, Y, _ = O.rigid_pair(2048, 3, 0.1, [0.1, 0.0, 0.0], 0.01, 0)
    cost = _pipeline_cost(X, Y)
    mu = make_distribution(np.ones(2048))
    cfg = SinkhornConfig(epsilon=1e-3, tolerance=1e-30, max_iterations=200)
    rep, pot = solve(cost, mu, mu, cfg)
    assert rel_max(pot.alpha, z["alpha"]) <= 1e-5 and rel_max(pot.beta, z["beta"]) <= 1e-5
    assert abs(rep.transport_cost - float(z["cost"])) <= 1e-5 * abs(float(z["cost"]))
    # the device-only fast path builds the very same fp32 matrix: bitwise the same solve
    rep2, pot2 = solve(squared_euclidean_cost(X, Y, normalize="max"), mu, mu, cfg)
    np.testing.assert_array_equal(pot.alpha, pot2.alpha)
    np.testing.assert_array_equal(pot.beta, pot2.beta)
    lazy = squared_euclidean_cost(X, Y)
    rep3, pot3 = solve(CostMatrix(values=lazy.values / lazy.values.max()), mu, mu, cfg)
    np.testing.assert_array_equal(pot.alpha, pot3.alpha)


def test_estimator_composition_double(cuda_ok):
    """estimator.py:86-99: normalised cost, precision='double'."""
    rng = np.random.default_rng(8)
    X, Y = rng.uniform(0, 1, (150, 2)), rng.uniform(0, 1, (170, 2)) + 0.3
    cost = _pipeline_cost(X, Y)
    mu, nu = make_distribution(np.ones(150)), make_distribution(np.ones(170))
    cfg = SinkhornConfig(epsilon=0.02, tolerance=1e-9, max_iterations=3000, check_interval=10, precision="double")
    rep, pot = solve(cost, mu, nu, cfg)
    C64 = O.sq_euclidean_cost(X, Y)
    rep_h, pot_h = solve(CostMatrix(values=C64 / C64.max()), mu, nu, cfg)
    assert rep.status == rep_h.status == STATUS_CONVERGED and rep.iterations == rep_h.iterations
    np.testing.assert_array_equal(pot.alpha, pot_h.alpha)
    np.testing.assert_array_equal(pot.beta, pot_h.beta)


def _alpha_hp(C, beta, log_nu, eps):
    """alpha_i = -eps * log sum_j exp((beta_j - C_ij)/eps + log nu_j) in 80-bit."""
    C = np.asarray(C, np.longdouble)
    t = (np.asarray(beta, np.longdouble)[None, :] - C) / np.longdouble(eps) + np.asarray(log_nu, np.longdouble)
    m = t.max(axis=1)
    return (-np.longdouble(eps) * (m + np.log(np.exp(t - m[:, None]).sum(axis=1)))).astype(np.float64)


def test_update_alpha_vs_high_precision_single(cuda_ok):
    """tests/test_solver.py:51-61 (mpmath there; 80-bit here, same bar)."""
    rng = np.random.default_rng(21)
    cost = make_cost_matrix(8, 8, rng.uniform(0, 1, 64))
    nu = make_distribution(rng.uniform(0.2, 1.0, 8))
    beta = rng.uniform(-0.5, 0.5, 8).astype(np.float32)
    alpha = update_alpha(cost, nu, beta, 0.05, PLAN)
    assert alpha.dtype == np.float32
    np.testing.assert_allclose(alpha, _alpha_hp(cost.values, beta, nu.log_weights, 0.05), rtol=1e-6, atol=1e-6)


def test_update_alpha_vs_high_precision_double(cuda_ok):
    rng = np.random.default_rng(22)
    cost = make_cost_matrix(8, 8, rng.uniform(0, 1, 64))
    nu = make_distribution(rng.uniform(0.2, 1.0, 8))
    beta = rng.uniform(-0.5, 0.5, 8)
    alpha = update_alpha(cost, nu, beta, 0.02, PLAN)
    np.testing.assert_allclose(alpha, _alpha_hp(cost.values, beta, nu.log_weights, 0.02), rtol=1e-13, atol=1e-13)


def test_status_trace_cap_semantics(cuda_ok):
    """tests/test_solver.py:210-238."""
    mu, nu, cost = generate_grid_problem(64, 64, 0)
    config = SinkhornConfig(epsilon=0.01)
    report, _ = solve(cost, mu, nu, config)
    assert report.status == STATUS_CONVERGED and report.final_marginal_error < config.tolerance
    config = SinkhornConfig(epsilon=0.001, max_iterations=20)
    report, _ = solve(cost, mu, nu, config)
    assert report.status == "not_converged" and report.iterations == 20
    assert report.final_marginal_error >= config.tolerance
    config = SinkhornConfig(epsilon=0.001, max_iterations=25, check_interval=10)
    report, _ = solve(cost, mu, nu, config)
    assert report.iterations == 25 and report.error_trace[-1][0] == 25
    config = SinkhornConfig(epsilon=0.01, check_interval=5)
    report, _ = solve(cost, mu, nu, config)
    assert [k for k, _ in report.error_trace] == list(range(5, report.iterations + 1, 5))
    assert report.error_trace[-1][1] == report.final_marginal_error


def test_bit_identical_repeat_solves(cuda_ok):
    """tests/test_solver.py:247-257."""
    mu, nu, cost = generate_grid_problem(128, 128, 3)
    config = SinkhornConfig(epsilon=0.01)
    r1, p1 = solve(cost, mu, nu, config)
    r2, p2 = solve(cost, mu, nu, config)
    assert r1.iterations == r2.iterations and r1.final_marginal_error == r2.final_marginal_error
    assert r1.transport_cost == r2.transport_cost and r1.error_trace == r2.error_trace
    np.testing.assert_array_equal(p1.alpha, p2.alpha)
    np.testing.assert_array_equal(p1.beta, p2.beta)


@pytest.mark.parametrize("precision,bar", [("double", 1e-10), ("single", 1e-5)])
def test_kkt_residual_of_materialized_plan(cuda_ok, precision, bar):
    """tests/test_solver.py:345-360."""
    mu, nu, cost = generate_grid_problem(32, 32, 2)
    _, pot = solve(cost, mu, nu, SinkhornConfig(epsilon=0.05, precision=precision))
    plan = materialize_plan(cost, mu, nu, pot.alpha, pot.beta, 0.05)
    assert kkt_residual(cost, mu, nu, plan, pot.alpha, pot.beta, 0.05) <= bar


@pytest.mark.parametrize("precision", ["single", "double"])
def test_converged_plan_marginals(cuda_ok, precision):
    """tests/test_solver.py:463-474."""
    mu, nu, cost = generate_grid_problem(128, 128, 6)
    config = SinkhornConfig(epsilon=0.01, precision=precision)
    report, pot = solve(cost, mu, nu, config)
    assert report.status == STATUS_CONVERGED
    plan = materialize_plan(cost, mu, nu, pot.alpha, pot.beta, 0.01)
    P = np.asarray(plan.values)
    rows = P.sum(axis=1, dtype=np.float64)
    cols = P.sum(axis=0, dtype=np.float64)
    assert np.abs(rows - mu.weights).sum() < config.tolerance
    assert np.abs(cols - nu.weights).sum() < 10 * config.tolerance


def test_package_exports_the_reference_names(cuda_ok):
    for name in ("solve", "update_alpha", "update_beta", "marginal_error", "transport_cost", "materialize_plan",
                 "squared_euclidean_cost", "CostMatrix", "DiscreteDistribution", "SinkhornConfig", "SolveReport",
                 "DualPotentials", "make_distribution", "make_cost_matrix", "ReductionPlan"):
        assert hasattr(ls, name), name


def test_points_normalisation_follows_value_range(cuda_ok):
    """applications.py:186-188 divide by C.max() only when value_range > 0: a
    constant nonzero cost stays unscaled (n = m = 1, distinct points)."""
    from paper_2605_00837_b200 import points as PT

    X, Y = np.array([[0.0, 0.0]]), np.array([[1.0, 1.0]])
    cfg = SinkhornConfig(epsilon=0.1, tolerance=1e-30, max_iterations=10)
    rep, pot = PT.solve_points_otf(X, Y, None, None, cfg, normalize="max")
    assert rep.transport_cost == pytest.approx(2.0, rel=1e-6)
    rep_d, _ = solve(_pipeline_cost(X, Y), make_distribution([1.0]), make_distribution([1.0]), cfg)
    assert rep_d.transport_cost == pytest.approx(2.0, rel=1e-6)


def test_match_point_clouds_any_dimension(cuda_ok):
    """The reference accepts any d; d > 3 takes the dense path."""
    rng = np.random.default_rng(4)
    X = rng.uniform(0, 1, (60, 5))
    perm = rng.permutation(60)
    Y = np.empty_like(X)
    Y[perm] = X + 0.001
    pairs = ls.match_point_clouds(X, Y, 1e-3)
    assert np.mean([p.target_index == perm[p.source_index] for p in pairs]) > 0.9
