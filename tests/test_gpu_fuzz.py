"""Randomised parity sweep: seeded random problems (shape, eps, weights, cost
law, check interval, cap) through lsk.solve vs the oracle (the bit-exact
restatement of the reference), at fixed iteration counts so the comparison is
about the potentials, not the stop decision. Covers the kernel variants the
dispatcher picks by shape: uniform / general targets, column padding, 1 to
hundreds of rows per CTA, the multiplicative column update (n*m >= 2^20,
1e-3 <= eps <= 2e-3) and the exact first iteration."""

import numpy as np
import pytest

import lsk_oracle as O
import paper_2605_00837_b200 as lsk
from conftest import rel_max_floor

pytestmark = pytest.mark.gpu

CASES = list(range(40))


def problem(seed):
    rng = np.random.default_rng(1000 + seed)
    big = seed % 4 == 0
    n = int(rng.choice([1024, 1100, 1536])) if big else int(rng.integers(1, 700))
    m = int(rng.choice([1024, 1030, 2048])) if big else int(rng.integers(1, 3000))
    d = int(rng.integers(1, 4))
    X, Y = rng.uniform(0, 1, (n, d)), rng.uniform(0, 1, (m, d)) * rng.uniform(0.5, 2.0)
    C64 = ((X[:, None, :] - Y[None, :, :]) ** 2).sum(axis=2)
    uniform = rng.random() < 0.6
    wa = np.ones(n) if uniform else rng.uniform(0.2, 2.0, n)
    wb = np.ones(m) if (uniform or rng.random() < 0.5) else rng.uniform(0.2, 2.0, m)
    eps = float(rng.choice([1e-3, 2e-3, 5e-3, 1e-2, 5e-2])) if big else float(rng.choice([5e-3, 1e-2, 5e-2, 0.1]))
    K = int(rng.integers(3, 25)) if big else int(rng.integers(2, 60))
    c = int(rng.integers(1, 12))
    return C64, wa, wb, eps, K, c


@pytest.mark.parametrize("seed", CASES)
def test_random_problem_vs_oracle(cuda_ok, seed):
    C64, wa, wb, eps, K, c = problem(seed)
    n, m = C64.shape
    mu, nu = lsk.make_distribution(wa), lsk.make_distribution(wb)
    cfg = lsk.SinkhornConfig(epsilon=eps, tolerance=1e-30, max_iterations=K, check_interval=c)
    rep, pot = lsk.solve(lsk.make_cost_matrix(n, m, C64), mu, nu, cfg)
    with np.errstate(all="ignore"):
        ref = O.solve(C64, mu.weights, nu.weights, eps, tol=1e-30, max_iter=K, check=c)
    assert rep.status == ref["status"] and rep.iterations == ref["iterations"], (seed, rep.status, ref["status"])
    if ref["status"] == "numerical_failure":
        return
    ea = rel_max_floor(pot.alpha, ref["alpha"], ref["beta"])
    eb = rel_max_floor(pot.beta, ref["beta"], ref["alpha"])
    assert ea <= 1e-5 and eb <= 1e-5, (seed, n, m, eps, K, ea, eb)
    assert abs(rep.transport_cost - ref["cost"]) <= 1e-5 * abs(ref["cost"]) + 1e-7
    assert [k for k, _ in rep.error_trace] == [k for k, _ in ref["trace"]]


@pytest.mark.parametrize("seed", list(range(6)))
def test_wide_m_loop_vs_oracle(cuda_ok, seed):
    """m > 8192 runs the multi-kernel loop (one-pass stale row LSE with exact fallback,
    column (max, sumexp) partials, device-side checks): same bar against the oracle."""
    rng = np.random.default_rng(3000 + seed)
    n, m = int(rng.integers(1, 80)), int(rng.integers(8193, 13000))
    X, Y = rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (m, 2))
    C64 = ((X[:, None, :] - Y[None, :, :]) ** 2).sum(axis=2)
    wa = np.ones(n) if seed % 2 else rng.uniform(0.2, 2.0, n)
    wb = np.ones(m) if seed % 3 else rng.uniform(0.2, 2.0, m)
    eps = float(rng.choice([1e-3, 1e-2, 5e-2]))
    K, c = int(rng.integers(2, 30)), int(rng.integers(1, 8))
    mu, nu = lsk.make_distribution(wa), lsk.make_distribution(wb)
    cfg = lsk.SinkhornConfig(epsilon=eps, tolerance=1e-30, max_iterations=K, check_interval=c)
    rep, pot = lsk.solve(lsk.make_cost_matrix(n, m, C64), mu, nu, cfg)
    with np.errstate(all="ignore"):
        ref = O.solve(C64, mu.weights, nu.weights, eps, tol=1e-30, max_iter=K, check=c)
    assert rep.status == ref["status"] and rep.iterations == ref["iterations"]
    assert rel_max_floor(pot.alpha, ref["alpha"], ref["beta"]) <= 1e-5
    assert rel_max_floor(pot.beta, ref["beta"], ref["alpha"]) <= 1e-5
    assert abs(rep.transport_cost - ref["cost"]) <= 1e-5 * abs(ref["cost"]) + 1e-7
