"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container only (it needs /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py [--big]

Every fixture stores the reference ``logsinkhorn`` outputs (potentials,
status, iterations, error trace, transport cost) plus sha256 prefixes of the
generated inputs, so the GPU tests can regenerate the inputs from their seeds
with ``oracle/lsk_oracle.py`` and prove they fed the CUDA path the same bytes.
All solves use ``precision="single"`` (the fp32 parity target).
"""

import argparse
import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import logsinkhorn as ls  # noqa: E402

sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import lsk_oracle  # noqa: E402  (input generator only)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def save(name, **kw):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **kw)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def solve_case(name, cost, mu, nu, eps, K, tol=1e-30, check=10, extra=None, precision="single"):
    cfg = ls.SinkhornConfig(epsilon=eps, tolerance=tol, max_iterations=K,
                            check_interval=check, precision=precision)
    t = time.perf_counter()
    rep, pot = ls.solve(cost, mu, nu, cfg)
    dt = time.perf_counter() - t
    tr = np.array(rep.error_trace, dtype=np.float64).reshape(-1, 2)
    kw = dict(
        eps=eps, K=K, tol=tol, check=check,
        status=rep.status, iterations=rep.iterations,
        err=rep.final_marginal_error, cost=rep.transport_cost,
        trace=tr, alpha=pot.alpha, beta=pot.beta,
        mu=mu.weights, nu=nu.weights,
        C32_sha=sha(np.ascontiguousarray(cost.values, np.float32)),
        ref_seconds=dt,
    )
    if extra:
        kw.update(extra)
    print(f"{name}: {rep.status} it={rep.iterations} err={rep.final_marginal_error!r} "
          f"cost={rep.transport_cost!r} ({dt:.1f}s)")
    save(name, **kw)


def points_case(name, n, d, seed, eps, K, normalize=False):
    rng = np.random.Generator(np.random.PCG64(seed))
    X = rng.uniform(0.0, 1.0, (n, d))
    Y = rng.uniform(0.0, 1.0, (n, d))
    cost = ls.squared_euclidean_cost(X, Y)
    if normalize:
        cost = ls.CostMatrix(values=np.ascontiguousarray(cost.values / cost.values.max()))
    w = ls.make_distribution(np.ones(n))
    solve_case(name, cost, w, w, eps, K, extra=dict(
        n=n, d=d, seed=seed, X_sha=sha(X), Y_sha=sha(Y), normalize=normalize,
        Cmax=float(ls.squared_euclidean_cost(X, Y).values.max())))


def grid_case(name, n, m, seed, eps, K=10000, tol=1e-6, check=10):
    mu, nu, cost = ls.generate_grid_problem(n, m, seed)
    solve_case(name, cost, mu, nu, eps, K, tol=tol, check=check,
               extra=dict(grid=(n, m, seed)))


def small_cases():
    # status / trace / cap semantics (reference tests/test_solver.py:210-238)
    grid_case("grid64_eps1e-2", 64, 64, 0, 0.01)
    grid_case("grid64_cap20", 64, 64, 0, 0.001, K=20)
    grid_case("grid64_cap25", 64, 64, 0, 0.001, K=25, check=10)
    grid_case("grid64_check5", 64, 64, 0, 0.01, check=5)
    grid_case("grid128_seed3", 128, 128, 3, 0.01)
    grid_case("grid96_seed4", 96, 96, 4, 0.01)
    grid_case("grid40x70", 40, 70, 1, 0.05)
    grid_case("grid512_eps1e-3", 512, 512, 0, 0.001, K=300)
    # ragged sizes, random cost and weights
    for seed, (n, m) in enumerate([(1, 1), (3, 5), (37, 53), (257, 300), (1000, 77), (5, 1100)]):
        C, mu_w, nu_w, _, _ = lsk_oracle.random_problem(n, m, seed)
        cost = ls.make_cost_matrix(n, m, C.ravel())
        mu = ls.make_distribution(mu_w)
        nu = ls.make_distribution(nu_w)
        solve_case(f"rand_{n}x{m}", cost, mu, nu, 0.05, K=57, check=10,
                   extra=dict(seed=seed, shape=(n, m)))
    # antidiagonal (tests/test_solver.py:29-33, 180-186) in single precision
    cost = ls.make_cost_matrix(2, 2, [0.0, 1.0, 1.0, 0.0])
    half = ls.make_distribution([0.5, 0.5])
    solve_case("antidiag", cost, half, half, 0.1, K=10000, tol=1e-6,
               extra=dict(C=cost.values))
    # constant cost converges within one check (tests/test_solver.py:190-201)
    cost = ls.make_cost_matrix(4, 4, [0.6] * 16)
    w4 = ls.make_distribution([1.0] * 4)
    solve_case("constant", cost, w4, w4, 0.1, K=10000, tol=1e-6,
               extra=dict(C=cost.values))
    # numerical failure: -inf rows (overflow in the argument build)
    cost = ls.make_cost_matrix(2, 3, [1e30, 2e30, 3e30, 1e30, 5e29, 1e30])
    solve_case("failure", cost, ls.make_distribution([1, 1]),
               ls.make_distribution([1, 1, 1]), 1e-9, K=7, check=3,
               extra=dict(C=cost.values))


def double_cases():
    """precision="double" solves and float64 half-steps (reference dt = float64)."""
    mu, nu, cost = ls.generate_grid_problem(64, 64, 0)
    solve_case("dbl_grid64_eps1e-3", cost, mu, nu, 0.001, K=10000, tol=1e-6, extra=dict(grid=(64, 64, 0)),
               precision="double")
    mu, nu, cost = ls.generate_grid_problem(40, 70, 1)
    solve_case("dbl_grid40x70_cap25", cost, mu, nu, 0.05, K=25, tol=1e-12, extra=dict(grid=(40, 70, 1)),
               precision="double")
    C, mu_w, nu_w, _, _ = lsk_oracle.random_problem(257, 300, 3)
    solve_case("dbl_rand_257x300", ls.make_cost_matrix(257, 300, C.ravel()), ls.make_distribution(mu_w),
               ls.make_distribution(nu_w), 0.05, K=57, extra=dict(seed=3, shape=(257, 300)), precision="double")
    cost = ls.make_cost_matrix(2, 2, [0.0, 1.0, 1.0, 0.0])
    half = ls.make_distribution([0.5, 0.5])
    solve_case("dbl_antidiag", cost, half, half, 0.1, K=10000, tol=1e-9, extra=dict(C=cost.values),
               precision="double")
    out = {}
    for (n, m) in [(8, 8), (37, 53), (300, 1000)]:
        C, mu_w, nu_w, alpha_in, beta = lsk_oracle.random_problem(n, m, 200 + n + m)
        alpha_in, beta = alpha_in.astype(np.float64), beta.astype(np.float64)
        cost = ls.make_cost_matrix(n, m, C.ravel())
        mu, nu = ls.make_distribution(mu_w), ls.make_distribution(nu_w)
        key = f"{n}x{m}"
        out[key + "_alpha"] = ls.update_alpha(cost, nu, beta, 0.05)
        out[key + "_beta_out"] = ls.update_beta(cost, mu, alpha_in, 0.05)
        out[key + "_merr"] = ls.marginal_error(cost, mu, nu, alpha_in, beta, 0.05)
        out[key + "_tcost"] = ls.transport_cost(cost, mu, nu, alpha_in, beta, 0.05)
        P = ls.materialize_plan(cost, mu, nu, alpha_in, beta, 0.05).values
        out[key + "_plan_rows"] = P.sum(axis=1)
        out[key + "_plan_corner"] = P[:4, :4]
    out["shapes"] = np.array([(8, 8), (37, 53), (300, 1000)])
    out["eps"] = 0.05
    save("dbl_half_steps", **out)


def half_step_cases():
    out = {}
    shapes = [(1, 1), (8, 8), (37, 53), (300, 1000), (1031, 517)]
    for (n, m) in shapes:
        seed = 100 + n + m
        C, mu_w, nu_w, alpha_in, beta = lsk_oracle.random_problem(n, m, seed)
        cost = ls.make_cost_matrix(n, m, C.ravel())
        mu = ls.make_distribution(mu_w)
        nu = ls.make_distribution(nu_w)
        eps = 0.05
        key = f"{n}x{m}"
        out[key + "_alpha"] = ls.update_alpha(cost, nu, beta, eps)
        out[key + "_beta_out"] = ls.update_beta(cost, mu, alpha_in, eps)
        out[key + "_merr"] = ls.marginal_error(cost, mu, nu, alpha_in, beta, eps)
        out[key + "_tcost"] = ls.transport_cost(cost, mu, nu, alpha_in, beta, eps)
        P = ls.materialize_plan(cost, mu, nu, alpha_in, beta, eps).values
        out[key + "_plan_sha"] = sha(P)
        out[key + "_plan_rows"] = P.sum(axis=1, dtype=np.float64)
        out[key + "_plan_corner"] = P[:4, :4]
    out["shapes"] = np.array(shapes)
    out["eps"] = 0.05
    save("half_steps", **out)


def big_cases():
    # SURVEY.md 8(c) golden G1/G2/G3/G5 plus small-eps long runs
    points_case("g1_c1_n1024", 1024, 2, 0, 1e-2, 200)
    points_case("g2_c2_n8192_k10", 8192, 2, 0, 1e-3, 10)
    points_case("g3_c3_n8192_k10", 8192, 2, 0, 1e-4, 10)
    points_case("n1024_eps1e-4_k1000", 1024, 2, 0, 1e-4, 1000)
    points_case("n2048_eps1e-3_k200", 2048, 2, 0, 1e-3, 200)
    points_case("g5_c5_n4096_rgb_k200", 4096, 3, 0, 1e-2, 200)
    # C4-shaped (rigid pair, 3-D, max-normalised) at a CPU-feasible size
    X, Y, perm = ls.generate_rigid_pair(2048, 3, 0.1, [0.1, 0.0, 0.0], 0.01, 0)
    cost = ls.squared_euclidean_cost(X, Y)
    cmax = cost.values.max()
    cost = ls.CostMatrix(values=np.ascontiguousarray(cost.values / cmax))
    w = ls.make_distribution(np.ones(2048))
    solve_case("rigid2048_eps1e-3_k200", cost, w, w, 1e-3, 200, extra=dict(
        X_sha=sha(X), Y_sha=sha(Y), perm=perm, Cmax=float(cmax)))
    # G4 inputs only (solve too large for the host)
    X, Y, perm = ls.generate_rigid_pair(65536, 3, 0.1, [0.1, 0.0, 0.0], 0.01, 0)
    save("g4_inputs", X_sha=sha(X), Y_sha=sha(Y), perm_sha=sha(perm),
         X0=X[0], Y0=Y[0], perm5=perm[:5], Cmax=3.0914804297769676)


def long_c2():
    """C2 at the benchmarked iteration count (BASELINE configs[1])."""
    points_case("g2_c2_n8192_k1000", 8192, 2, 0, 1e-3, 1000)


def long_c2_k2000():
    """C2 at 2000 iterations: the multiplicative column update's drift grows with K
    (profiles/r2_c1_cluster.md); C2 reaches marginal error 1e-6 at ~2020."""
    points_case("g2_c2_n8192_k2000", 8192, 2, 0, 1e-3, 2000)


def long_c2_k200():
    points_case("g2_c2_n8192_k200", 8192, 2, 0, 1e-3, 200)


def long_c3_k200():
    """C3 (eps=1e-4) at fixed K (parity at K in {200, 1000})."""
    points_case("g3_c3_n8192_k200", 8192, 2, 0, 1e-4, 200)


def long_c3_k1000():
    points_case("g3_c3_n8192_k1000", 8192, 2, 0, 1e-4, 1000)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    if a.only:
        globals()[a.only]()
    else:
        small_cases()
        half_step_cases()
        double_cases()
        if a.big:
            big_cases()
