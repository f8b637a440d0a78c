"""Randomised parity sweep of precision="double" (the fp64 multi-kernel solver)
and of the fp64 standard-domain solve: seeded random problems vs the oracle's
float64 restatement (solve) and a direct numpy float64 restatement of
solver.py:340-431 (standard domain), at fixed iteration counts."""

import numpy as np
import pytest

import lsk_oracle as O
import paper_2605_00837_b200 as lsk

pytestmark = pytest.mark.gpu


def problem(seed, nmax=400, mmax=700):
    rng = np.random.default_rng(7000 + seed)
    n, m = int(rng.integers(1, nmax)), int(rng.integers(1, mmax))
    X, Y = rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (m, 2))
    C64 = ((X[:, None, :] - Y[None, :, :]) ** 2).sum(axis=2)
    wa = np.ones(n) if rng.random() < 0.5 else rng.uniform(0.2, 2.0, n)
    wb = np.ones(m) if rng.random() < 0.5 else rng.uniform(0.2, 2.0, m)
    eps = float(rng.choice([1e-3, 5e-3, 1e-2, 0.1]))
    return C64, wa, wb, eps, int(rng.integers(2, 40)), int(rng.integers(1, 10))


@pytest.mark.parametrize("seed", list(range(16)))
def test_double_solve_vs_oracle(cuda_ok, seed):
    C64, wa, wb, eps, K, c = problem(seed)
    n, m = C64.shape
    mu, nu = lsk.make_distribution(wa), lsk.make_distribution(wb)
    cfg = lsk.SinkhornConfig(epsilon=eps, tolerance=1e-30, max_iterations=K, check_interval=c, precision="double")
    rep, pot = lsk.solve(lsk.make_cost_matrix(n, m, C64), mu, nu, cfg)
    with np.errstate(all="ignore"):
        ref = O.solve(C64, mu.weights, nu.weights, eps, tol=1e-30, max_iter=K, check=c, dtype=np.float64)
    assert rep.status == ref["status"] and rep.iterations == ref["iterations"]
    assert pot.alpha.dtype == np.float64
    scale = max(np.abs(ref["alpha"]).max(), np.abs(ref["beta"]).max())
    assert np.abs(pot.alpha - ref["alpha"]).max() <= 1e-12 * scale
    assert np.abs(pot.beta - ref["beta"]).max() <= 1e-12 * scale
    assert abs(rep.transport_cost - ref["cost"]) <= 1e-12 * abs(ref["cost"])


def standard_numpy(C, mu_w, nu_w, eps, K, c, tol):
    """solver.py:340-431 in float64 with plain numpy sums (tree order aside)."""
    Km = np.exp(-C / eps)
    u, v = np.ones_like(mu_w), np.ones_like(nu_w)
    trace, status, err, it = [], "not_converged", np.inf, 0
    with np.errstate(all="ignore"):
        for k in range(1, K + 1):
            u = mu_w / (Km @ v)
            v = nu_w / (Km.T @ u)
            it = k
            if k % c == 0 or k == K:
                if not (np.isfinite(u).all() and np.isfinite(v).all()):
                    return "numerical_failure", it, trace, u, v
                err = np.abs(u * (Km @ v) - mu_w).sum()
                trace.append(k)
                if not np.isfinite(err):
                    return "numerical_failure", it, trace, u, v
                if err < tol:
                    return "converged", it, trace, u, v
    return status, it, trace, u, v


@pytest.mark.parametrize("seed", list(range(10)))
def test_double_standard_domain_vs_numpy(cuda_ok, seed):
    C64, wa, wb, eps, K, c = problem(100 + seed, 300, 500)
    eps = max(eps, 5e-3)
    n, m = C64.shape
    mu, nu = lsk.make_distribution(wa), lsk.make_distribution(wb)
    cfg = lsk.SinkhornConfig(epsilon=eps, tolerance=1e-30, max_iterations=K, check_interval=c, precision="double")
    rep, u, v = lsk.solve_standard_domain(lsk.make_cost_matrix(n, m, C64), mu, nu, cfg)
    st, it, trace, ru, rv = standard_numpy(C64, mu.weights, nu.weights, eps, K, c, 1e-30)
    assert rep.status == st and rep.iterations == it
    assert [k for k, _ in rep.error_trace] == trace
    if st != "numerical_failure":
        np.testing.assert_allclose(u, ru, rtol=1e-10)
        np.testing.assert_allclose(v, rv, rtol=1e-10)
