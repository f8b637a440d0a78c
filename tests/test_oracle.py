"""Pin the oracle: bit-exact against the reference's own outputs.

The golden fixtures were produced by running the reference package
(tests/golden/make_golden.py). The oracle restates the same numpy ufuncs on
the same tree, so on this host it must reproduce them bit for bit; the GPU
parity tests then trust it as the checker.
"""

import os
import sys

import numpy as np
import pytest

import lsk_oracle as O
from conftest import golden, golden_names, sha
from inputs import fixture_problem

SMALL = [n for n in golden_names() if n.startswith(("grid", "rand_", "antidiag", "constant", "failure"))]


def _check_exact(r, z):
    assert r["status"] == str(z["status"])
    assert r["iterations"] == int(z["iterations"])
    tr = np.array(r["trace"], dtype=np.float64).reshape(-1, 2)
    np.testing.assert_array_equal(tr, z["trace"])
    np.testing.assert_array_equal(r["alpha"], z["alpha"])
    np.testing.assert_array_equal(r["beta"], z["beta"])
    if np.isnan(float(z["cost"])):
        assert np.isnan(r["cost"])
    else:
        assert r["cost"] == float(z["cost"])
    if np.isnan(float(z["err"])):
        assert np.isnan(r["err"])
    else:
        assert r["err"] == float(z["err"])


@pytest.mark.parametrize("name", SMALL)
def test_oracle_matches_reference_small(name):
    z, C64, mu_w, nu_w = fixture_problem(name)
    with np.errstate(all="ignore"):
        r = O.solve(C64, mu_w, nu_w, float(z["eps"]), tol=float(z["tol"]), max_iter=int(z["K"]),
                    check=int(z["check"]))
    _check_exact(r, z)


def test_oracle_matches_reference_g1():
    """SURVEY.md 8(c) golden G1 (C1: n=1024, eps=1e-2, K=200)."""
    z, C64, mu_w, nu_w = fixture_problem("g1_c1_n1024")
    r = O.solve(C64, mu_w, nu_w, float(z["eps"]), tol=float(z["tol"]), max_iter=int(z["K"]))
    _check_exact(r, z)
    assert sha(r["alpha"]) == "a95bf749897a66b3" and sha(r["beta"]) == "2ae1cb86ffa5c4f1"


def test_oracle_half_steps():
    z = golden("half_steps")
    eps = float(z["eps"])
    dt = np.float32
    inv, neg = dt(1.0) / dt(eps), -dt(eps)
    for n, m in z["shapes"]:
        n, m = int(n), int(m)
        key = f"{n}x{m}"
        C64, mu_w, nu_w, a_in, b_in = O.random_problem(n, m, 100 + n + m)
        C = C64.astype(dt)
        lmu, lnu = np.log(mu_w).astype(dt), np.log(nu_w).astype(dt)
        np.testing.assert_array_equal(O.row_update(C, b_in, lnu, inv, neg), z[key + "_alpha"])
        np.testing.assert_array_equal(O.row_update(np.ascontiguousarray(C.T), a_in, lmu, inv, neg),
                                      z[key + "_beta_out"])
        e = O.marginal_err(C, mu_w.astype(dt), lmu, lnu, a_in, b_in, inv)
        assert float(e) == float(z[key + "_merr"])
        assert O.transport_cost_rows(C, lmu, lnu, a_in, b_in, inv) == float(z[key + "_tcost"])
        P = O.plan_values(C, lmu, lnu, a_in, b_in, inv)
        assert sha(P) == str(z[key + "_plan_sha"])


def test_tree_flat_plan_is_left_to_right():
    v = np.array([[1e8, 1.0, -1e8, 1.0]], np.float32)
    f = np.float32
    assert O.tree_sum_rows(v, 1, 1)[0] == ((f(1e8) + f(1.0)) - f(1e8)) + f(1.0) == f(1.0)


def test_lse_empty_row_is_minus_inf():
    T = np.full((2, 5), -np.inf, np.float32)
    T[1, 2] = 0.0
    out = O.lse_rows(T)
    assert out[0] == -np.inf and out[1] == 0.0


def test_input_hashes_survey_g4():
    z = golden("g4_inputs")
    X, Y, perm = O.rigid_pair(65536, 3, 0.1, [0.1, 0.0, 0.0], 0.01, 0)
    assert sha(X) == str(z["X_sha"]) and sha(Y) == str(z["Y_sha"]) and sha(perm) == str(z["perm_sha"])
    np.testing.assert_array_equal(perm[:5], z["perm5"])


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted (GPU box)")
def test_oracle_vs_live_reference_random():
    sys.path.insert(0, REF)
    import logsinkhorn as ls

    rng = np.random.default_rng(5)
    for n, m, eps in [(33, 70, 0.03), (300, 257, 0.01), (64, 1, 0.1)]:
        C = rng.uniform(0, 1, (n, m))
        mu = ls.make_distribution(rng.uniform(0.3, 1, n))
        nu = ls.make_distribution(rng.uniform(0.3, 1, m))
        cfg = ls.SinkhornConfig(epsilon=eps, max_iterations=37, check_interval=7, tolerance=1e-30)
        rep, pot = ls.solve(ls.CostMatrix(values=C), mu, nu, cfg)
        r = O.solve(C, mu.weights, nu.weights, eps, tol=1e-30, max_iter=37, check=7)
        np.testing.assert_array_equal(r["alpha"], pot.alpha)
        np.testing.assert_array_equal(r["beta"], pot.beta)
        assert r["trace"] == rep.error_trace and r["cost"] == rep.transport_cost


@pytest.mark.parametrize("name", [n for n in golden_names("dbl_") if n != "dbl_half_steps"])
def test_oracle_double_matches_reference(name):
    """The oracle's float64 path reproduces the reference's precision="double" solve."""
    z, C64, mu_w, nu_w = fixture_problem(name)
    r = O.solve(C64, mu_w, nu_w, float(z["eps"]), tol=float(z["tol"]), max_iter=int(z["K"]),
                check=int(z["check"]), dtype=np.float64)
    assert r["status"] == str(z["status"]) and r["iterations"] == int(z["iterations"])
    np.testing.assert_allclose(r["alpha"], z["alpha"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(r["beta"], z["beta"], rtol=0, atol=1e-14)
