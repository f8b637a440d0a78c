"""SinkhornTransport against the reference estimator.

Fixtures from tests/golden/make_golden_estimator.py; the property tests are the
reference's tests/test_estimator.py run on this path.
"""

import numpy as np
import pytest
from conftest import golden, golden_names
from sklearn.base import clone
from sklearn.exceptions import NotFittedError

import paper_2605_00837_b200 as lsk
from paper_2605_00837_b200 import SinkhornTransport

pytestmark = pytest.mark.gpu


def two_clouds(seed=0, n=40, d=2, shift=0.3):
    rng = np.random.default_rng(seed)
    return rng.uniform(0, 1, (n, d)), rng.uniform(0, 1, (n, d)) + shift


@pytest.mark.parametrize("name", golden_names("est_"))
def test_estimator_matches_reference(cuda_ok, name):
    G = golden(name)
    est = SinkhornTransport(epsilon=float(G["eps"]), normalize_cost=bool(G["normalize"])).fit(G["X"], G["Y"])
    assert est.report_.status == str(G["status"])
    assert est.report_.iterations == int(G["iterations"])
    np.testing.assert_allclose(est.alpha_, G["alpha"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(est.beta_, G["beta"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(est.plan_, G["plan"], rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(est.transform(G["X"]), G["TX"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(est.transform(G["Q"]), G["TQ"], rtol=1e-10, atol=1e-12)


def test_fit_sets_attributes(cuda_ok):
    X, Y = two_clouds()
    est = SinkhornTransport(epsilon=0.05).fit(X, Y)
    assert est.plan_.shape == (40, 40)
    assert est.alpha_.shape == (40,) and est.beta_.shape == (40,)
    assert est.report_.status == "converged"
    assert est.n_features_in_ == 2
    np.testing.assert_allclose(est.plan_.sum(axis=1), 1.0 / 40, atol=1e-6)


def test_transform_maps_toward_target(cuda_ok):
    X, Y = two_clouds(seed=2, shift=0.5)
    est = SinkhornTransport(epsilon=0.02).fit(X, Y)
    Z = est.transform(X)
    assert Z.shape == X.shape
    assert (Z >= Y.min(axis=0) - 1e-9).all() and (Z <= Y.max(axis=0) + 1e-9).all()
    assert np.linalg.norm(Z.mean(axis=0) - Y.mean(axis=0)) < np.linalg.norm(X.mean(axis=0) - Y.mean(axis=0))


def test_fit_transform_and_determinism(cuda_ok):
    X, Y = two_clouds(seed=4)
    est = SinkhornTransport(epsilon=0.05)
    Z = est.fit_transform(X, Y)
    np.testing.assert_array_equal(Z, est.transform(X))
    b = SinkhornTransport(epsilon=0.05).fit(X, Y)
    np.testing.assert_array_equal(est.plan_, b.plan_)


def test_validation(cuda_ok):
    with pytest.raises(NotFittedError):
        SinkhornTransport().transform(np.zeros((2, 2)))
    with pytest.raises(ValueError):
        SinkhornTransport(epsilon=0.1).fit(np.zeros((4, 2)), np.zeros((4, 3)))
    X, Y = two_clouds(seed=5)
    est = SinkhornTransport(epsilon=0.05).fit(X, Y)
    with pytest.raises(ValueError):
        est.transform(np.zeros((3, 5)))


def test_params_clone(cuda_ok):
    est = SinkhornTransport(epsilon=0.3, tolerance=1e-8, normalize_cost=False)
    params = est.get_params()
    assert params["epsilon"] == 0.3 and params["normalize_cost"] is False
    assert clone(est).get_params() == params
    assert SinkhornTransport().set_params(epsilon=0.7).epsilon == 0.7


def test_barycentric_map_plan_kernel(cuda_ok):
    """The reference's TestBarycentricMap cases on the plan kernel (incl. d > 4 chunking)."""
    plan = lsk.TransportPlan(values=np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]))
    out = lsk.barycentric_map(plan, np.array([[0.0, 0.0], [1.0, 2.0], [3.0, 4.0]]))
    np.testing.assert_allclose(out, [[1.0, 2.0], [3.0, 4.0]])
    rng = np.random.default_rng(61)
    P = rng.uniform(0.01, 1.0, (20, 15))
    T = rng.standard_normal((15, 6))
    out = lsk.barycentric_map(lsk.TransportPlan(values=P), T)
    np.testing.assert_allclose(out, (P @ T) / P.sum(axis=1, keepdims=True), atol=1e-12)
    with pytest.raises(lsk.ZeroRowMass):
        lsk.barycentric_map(lsk.TransportPlan(values=np.array([[0.0, 0.0]])), np.zeros((2, 1)))
