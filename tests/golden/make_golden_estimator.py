"""Golden fixtures for SinkhornTransport, made by running the REFERENCE
estimator (build container only):  python tests/golden/make_golden_estimator.py
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import logsinkhorn as ls  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [
    # name, n, m, d, seed, shift, eps, normalize
    ("est_2d", 40, 40, 2, 0, 0.3, 0.05, True),
    ("est_rect3d", 30, 50, 3, 7, 0.0, 0.05, True),
    ("est_unnorm", 40, 40, 2, 8, 0.3, 0.05, False),
    ("est_shift", 64, 48, 2, 2, 0.5, 0.02, True),
]


def main():
    for name, n, m, d, seed, shift, eps, norm in CASES:
        rng = np.random.default_rng(seed)
        X = rng.uniform(0, 1, (n, d))
        Y = rng.uniform(0, 1, (m, d)) + shift
        Q = rng.uniform(-0.2, 1.2, (25, d))
        est = ls.SinkhornTransport(epsilon=eps, normalize_cost=norm).fit(X, Y)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), X=X, Y=Y, Q=Q, eps=eps, normalize=norm,
                            plan=est.plan_, alpha=est.alpha_, beta=est.beta_, status=est.report_.status,
                            iterations=est.report_.iterations, err=est.report_.final_marginal_error,
                            TX=est.transform(X), TQ=est.transform(Q))
        print(name, est.report_.status, est.report_.iterations)


if __name__ == "__main__":
    main()
