"""precision="double" and float64 half-steps on the GPU vs the reference.

Fixtures tests/golden/dbl_* were produced by the reference's double path
(make_golden.py double_cases). Bar: potentials and cost within 1e-12 relative
(max-norm) -- the summation order and exp/log ulps differ from numpy, nothing
else; status and iteration counts identical.
"""

import numpy as np
import pytest

import paper_2605_00837_b200 as lsk
from conftest import golden, golden_names
from inputs import fixture_problem
import lsk_oracle as O

pytestmark = pytest.mark.gpu
RTOL = 1e-12


def dist(w):
    w = np.asarray(w, np.float64)
    return lsk.DiscreteDistribution(weights=w, log_weights=np.log(w))


@pytest.mark.parametrize("name", [n for n in golden_names("dbl_") if n != "dbl_half_steps"])
def test_solve_double(cuda_ok, name):
    z, C64, mu_w, nu_w = fixture_problem(name)
    cfg = lsk.SinkhornConfig(epsilon=float(z["eps"]), tolerance=float(z["tol"]), max_iterations=int(z["K"]),
                             check_interval=int(z["check"]), precision="double")
    rep, pot = lsk.solve(lsk.CostMatrix(values=C64), dist(mu_w), dist(nu_w), cfg)
    assert pot.alpha.dtype == np.float64 and pot.beta.dtype == np.float64
    assert rep.status == str(z["status"]) and rep.iterations == int(z["iterations"])
    assert [k for k, _ in rep.error_trace] == [int(k) for k in z["trace"][:, 0]]
    for (_, e), (_, er) in zip(rep.error_trace, z["trace"]):
        assert abs(e - er) <= 1e-9 * abs(er) + 1e-14
    scale = max(np.abs(z["alpha"]).max(), np.abs(z["beta"]).max())
    assert np.abs(pot.alpha - z["alpha"]).max() <= RTOL * scale
    assert np.abs(pot.beta - z["beta"]).max() <= RTOL * scale
    assert abs(rep.transport_cost - float(z["cost"])) <= RTOL * abs(float(z["cost"]))


def test_half_steps_double(cuda_ok):
    z = golden("dbl_half_steps")
    eps = float(z["eps"])
    for n, m in z["shapes"]:
        n, m = int(n), int(m)
        key = f"{n}x{m}"
        C64, mu_w, nu_w, a_in, b_in = O.random_problem(n, m, 200 + n + m)
        a_in, b_in = a_in.astype(np.float64), b_in.astype(np.float64)
        cost, mu, nu = lsk.CostMatrix(values=C64), dist(mu_w), dist(nu_w)
        a = lsk.update_alpha(cost, nu, b_in, eps)
        assert a.dtype == np.float64
        np.testing.assert_allclose(a, z[key + "_alpha"], rtol=RTOL, atol=RTOL)
        np.testing.assert_allclose(lsk.update_beta(cost, mu, a_in, eps), z[key + "_beta_out"], rtol=RTOL, atol=RTOL)
        assert lsk.marginal_error(cost, mu, nu, a_in, b_in, eps) == pytest.approx(float(z[key + "_merr"]), rel=1e-10)
        assert lsk.transport_cost(cost, mu, nu, a_in, b_in, eps) == pytest.approx(float(z[key + "_tcost"]), rel=1e-12)
        P = lsk.materialize_plan(cost, mu, nu, a_in, b_in, eps).values
        assert P.dtype == np.float64
        np.testing.assert_allclose(P[:4, :4], z[key + "_plan_corner"], rtol=1e-13)
        np.testing.assert_allclose(P.sum(axis=1), z[key + "_plan_rows"], rtol=1e-12)


def test_list_potentials_are_double(cuda_ok):
    """A plain list is not float32: the reference computes in float64 (solver.py:60-65)."""
    cost = lsk.make_cost_matrix(1, 1, [0.5])
    a = lsk.update_alpha(cost, lsk.make_distribution([1.0]), [0.0], 0.1)
    assert a.dtype == np.float64 and a[0] == pytest.approx(0.5, rel=1e-15)
