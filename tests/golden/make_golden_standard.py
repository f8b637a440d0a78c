"""Golden fixtures for the standard-domain solve, made by running the REFERENCE
``logsinkhorn.solve_standard_domain`` (build container only):

    python tests/golden/make_golden_standard.py

Each fixture stores the cost, weights, config and the reference outputs
(status, iterations, final error, cost, trace, u, v).
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import logsinkhorn as ls  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def points(n, m, d, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(0, 1, (n, d)), rng.uniform(0, 1, (m, d))


CASES = [
    # name, n, m, d, seed, eps, K, c, tol, precision, nonuniform
    ("std_single_eps1e-2", 64, 64, 2, 1, 1e-2, 300, 10, 1e-6, "single", False),
    ("std_single_rect_cap25", 40, 70, 2, 2, 2e-2, 25, 10, 1e-9, "single", True),
    ("std_single_underflow", 48, 48, 2, 3, 1e-3, 100, 10, 1e-6, "single", False),
    ("std_single_failure", 48, 48, 2, 3, 2e-4, 100, 10, 1e-6, "single", False),
    ("std_double_eps5e-3", 64, 80, 2, 4, 5e-3, 400, 10, 1e-8, "double", True),
    ("std_double_underflow", 32, 32, 3, 5, 2e-4, 50, 5, 1e-8, "double", False),
]


def main():
    for name, n, m, d, seed, eps, K, c, tol, prec, nonuni in CASES:
        X, Y = points(n, m, d, seed)
        C = ls.squared_euclidean_cost(X, Y)
        rng = np.random.Generator(np.random.PCG64(seed + 100))
        wa = rng.uniform(0.5, 1.5, n) if nonuni else np.ones(n)
        wb = rng.uniform(0.5, 1.5, m) if nonuni else np.ones(m)
        mu, nu = ls.make_distribution(wa), ls.make_distribution(wb)
        cfg = ls.SinkhornConfig(epsilon=eps, tolerance=tol, max_iterations=K, check_interval=c, precision=prec)
        rep, u, v = ls.solve_standard_domain(C, mu, nu, cfg)
        tr = np.array(rep.error_trace, dtype=np.float64).reshape(-1, 2)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), C=C.values, wa=wa, wb=wb, eps=eps, K=K, c=c,
                            tol=tol, precision=prec, status=rep.status, iterations=rep.iterations,
                            err=rep.final_marginal_error, cost=rep.transport_cost, trace=tr, u=u, v=v)
        print(name, rep.status, rep.iterations, rep.final_marginal_error, rep.transport_cost, len(tr))


if __name__ == "__main__":
    main()
