"""Standard-domain solve against the reference.

Fixtures from tests/golden/make_golden_standard.py: the reference
``solve_standard_domain`` on seeded point-cloud costs in single and double
precision, including its intended failure at small eps (K underflows, u = mu/0
is non-finite, numerical_failure at the next checkpoint) and a cap that is not
a checkpoint. Summation orders differ from the reference tree, so values are
compared within precision-appropriate tolerances; statuses, iteration counts
and trace checkpoints must match exactly.
"""

import numpy as np
import pytest
from conftest import golden, golden_names

import paper_2605_00837_b200 as lsk

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", golden_names("std_"))
def test_standard_domain_matches_reference(cuda_ok, name):
    G = golden(name)
    prec = str(G["precision"])
    double = prec == "double"
    C = lsk.CostMatrix(values=np.ascontiguousarray(G["C"]))
    mu, nu = lsk.make_distribution(G["wa"]), lsk.make_distribution(G["wb"])
    cfg = lsk.SinkhornConfig(epsilon=float(G["eps"]), tolerance=float(G["tol"]), max_iterations=int(G["K"]),
                             check_interval=int(G["c"]), precision=prec)
    rep, u, v = lsk.solve_standard_domain(C, mu, nu, cfg)
    assert u.dtype == (np.float64 if double else np.float32)
    assert rep.status == str(G["status"])
    assert rep.iterations == int(G["iterations"])
    tr = np.array(rep.error_trace, dtype=np.float64).reshape(-1, 2)
    ref_tr = G["trace"]
    assert tr.shape == ref_tr.shape
    np.testing.assert_array_equal(tr[:, 0], ref_tr[:, 0])
    rtol = 1e-9 if double else 5e-2
    np.testing.assert_allclose(tr[:, 1], ref_tr[:, 1], rtol=rtol, atol=0 if double else 2e-7)
    if rep.status == "numerical_failure":
        assert np.isnan(rep.final_marginal_error) == np.isnan(float(G["err"]))
        assert np.isnan(rep.transport_cost)
        return
    np.testing.assert_allclose(rep.transport_cost, float(G["cost"]), rtol=1e-12 if double else 1e-5)
    urt = 1e-10 if double else 2e-4
    np.testing.assert_allclose(u, G["u"], rtol=urt)
    np.testing.assert_allclose(v, G["v"], rtol=urt)


def test_standard_domain_dense_c2_shape(cuda_ok):
    """n = m = 2048 grid at eps = 1e-2 in fp32: converges like the log-domain solve."""
    rng = np.random.default_rng(3)
    X, Y = rng.uniform(0, 1, (2048, 2)), rng.uniform(0, 1, (2048, 2))
    C = lsk.squared_euclidean_cost(X, Y)
    w = lsk.make_distribution(np.ones(2048))
    cfg = lsk.SinkhornConfig(epsilon=1e-2, tolerance=1e-5, max_iterations=2000)
    rep, u, v = lsk.solve_standard_domain(C, w, w, cfg)
    rep2, _ = lsk.solve(C, w, w, cfg)
    assert rep.status == "converged" and rep2.status == "converged"
    assert abs(rep.transport_cost - rep2.transport_cost) <= 1e-4 * abs(rep2.transport_cost)


@pytest.mark.parametrize("n,m,eps,K", [(2048, 2048, 0.02, 300), (1000, 777, 0.05, 200), (3000, 8192, 0.01, 120),
                                       (48, 48, 2e-4, 100)])
def test_fused_one_pass_vs_two_pass(cuda_ok, n, m, eps, K):
    """The one-pass persistent standard-domain kernel against the two-pass multi-kernel
    loop: same status, iterations and trace checkpoints, values to fp32 rounding
    (including the small-eps failure, where both stop at the same checkpoint)."""
    rng = np.random.default_rng(n + m)
    X, Y = rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (m, 2))
    C = lsk.squared_euclidean_cost(X, Y)
    mu, nu = lsk.make_distribution(rng.uniform(0.5, 1.5, n)), lsk.make_distribution(rng.uniform(0.5, 1.5, m))
    cfg = lsk.SinkhornConfig(epsilon=eps, tolerance=1e-7, max_iterations=K, check_interval=7)
    r1, u1, v1 = lsk.solve_standard_domain(C, mu, nu, cfg)
    r0, u0, v0 = lsk.solve_standard_domain(C, mu, nu, cfg, fused=False)
    assert r1.status == r0.status and r1.iterations == r0.iterations
    assert [k for k, _ in r1.error_trace] == [k for k, _ in r0.error_trace]
    if r0.status == "numerical_failure":
        assert np.isnan(r1.transport_cost)
        return
    np.testing.assert_allclose([e for _, e in r1.error_trace], [e for _, e in r0.error_trace], rtol=2e-2, atol=1e-8)
    np.testing.assert_allclose(u1, u0, rtol=2e-4)
    np.testing.assert_allclose(v1, v0, rtol=2e-4)
    assert abs(r1.transport_cost - r0.transport_cost) <= 1e-5 * abs(r0.transport_cost)
