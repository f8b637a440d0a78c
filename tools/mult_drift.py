"""Drift of the multiplicative column update against the reference arithmetic
(oracle) at fixed iteration counts: python tools/mult_drift.py (LSK_LIB selects
the library build)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import lsk_oracle as O
    import paper_2605_00837_b200 as lsk
    from conftest import golden, rel_max

    for n, eps, K in ((1024, 1e-2, 300), (1024, 5e-3, 300), (2048, 1e-3, 500)):
        rng = np.random.default_rng(5)
        X, Y = rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (n, 2))
        C64 = O.sq_euclidean_cost(X, Y)
        C = lsk.squared_euclidean_cost(X, Y)
        w = lsk.make_distribution(np.ones(n))
        cfg = lsk.SinkhornConfig(epsilon=eps, tolerance=1e-30, max_iterations=K)
        ref = O.solve(C64, np.full(n, 1.0 / n), np.full(n, 1.0 / n), eps, tol=1e-30, max_iter=K)
        for mult in (True, False):
            rep, pot = lsk.solve(C, w, w, cfg, multiplicative=mult)
            print(f"n={n} eps={eps} K={K} {'mult  ' if mult else 'direct'} f {rel_max(pot.alpha, ref['alpha']):.2e} "
                  f"g {rel_max(pot.beta, ref['beta']):.2e}", flush=True)
    z = golden("g2_c2_n8192_k1000")
    X, Y = O.uniform_points(8192, 2, 0)
    C = lsk.squared_euclidean_cost(X, Y)
    w = lsk.make_distribution(np.ones(8192))
    cfg = lsk.SinkhornConfig(epsilon=1e-3, tolerance=1e-30, max_iterations=1000)
    rep, pot = lsk.solve(C, w, w, cfg)
    print(f"C2 K=1000 mult f {rel_max(pot.alpha, z['alpha']):.2e} g {rel_max(pot.beta, z['beta']):.2e}", flush=True)


if __name__ == "__main__":
    main()
