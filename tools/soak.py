"""Soak run: many random solves through every kernel family (dense general /
uniform / multiplicative / wide-m loop / exact variant, points, batched,
standard domain, fp64) with short iteration counts, checking only that each
finishes with finite potentials or a legitimate numerical_failure status.
Catches hangs and races the parity suites are too small to hit.

    python tools/soak.py [count]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2605_00837_b200 as lsk
    from paper_2605_00837_b200 import points as PT

    count = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rng = np.random.default_rng(1234)
    t0 = time.time()
    kinds = {}
    for it in range(count):
        kind = rng.choice(["dense", "dense_uni", "wide", "exact", "points", "batched", "standard", "double",
                           "cluster", "points_long"])
        n = int(rng.integers(1, 3000))
        m = int(rng.integers(1, 8192)) if kind != "wide" else int(rng.integers(8193, 12000))
        if kind == "wide":
            n = int(rng.integers(1, 600))
        if kind == "cluster":  # the single-cluster solver's range (uniform targets, n <= 512, m <= 1024)
            n, m = int(rng.integers(1, 513)), int(rng.integers(1, 1025))
        eps = float(rng.choice([1e-3, 3e-3, 1e-2, 0.1]))
        K = int(rng.integers(1, 30)) if kind != "points_long" else int(rng.integers(40, 120))
        c = int(rng.integers(1, 8))
        cfg = lsk.SinkhornConfig(epsilon=eps, tolerance=float(rng.choice([1e-30, 1e-4])), max_iterations=K,
                                 check_interval=c, precision="double" if kind == "double" else "single")
        X, Y = rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (m, 2))
        if kind in ("points", "batched", "points_long"):
            n, m = min(n, 2000), min(m, 3000)
            X, Y = X[:n], Y[:m]
            if kind in ("points", "points_long"):
                rep, pot = PT.solve_points_otf(X, Y, None, None, cfg, normalize=rng.choice(["none", "max"]))
            else:
                B = int(rng.integers(1, 5))
                outs = PT.solve_points_batched(np.stack([X[: min(n, 500)]] * B), np.stack([Y[: min(m, 700)]] * B),
                                               cfg)
                rep, pot = outs[-1]
        else:
            if kind == "double":
                n, m = min(n, 800), min(m, 800)
                X, Y = X[:n], Y[:m]
            C = lsk.squared_euclidean_cost(X, Y)
            mu = lsk.make_distribution(np.ones(n) if kind in ("dense_uni", "wide") else rng.uniform(0.5, 1.5, n))
            if kind == "wide" and rng.uniform() < 0.5:
                mu = lsk.make_distribution(rng.uniform(0.5, 1.5, n))
            nu = lsk.make_distribution(np.ones(m) if kind != "dense" else rng.uniform(0.5, 1.5, m))
            if kind == "standard":
                rep, u, v = lsk.solve_standard_domain(C, mu, nu, cfg)
                pot = None
            else:
                rep, pot = lsk.solve(C, mu, nu, cfg, stale_shift=kind != "exact")
        ok = rep.status == "numerical_failure" or pot is None or (np.isfinite(pot.alpha).all() and np.isfinite(pot.beta).all())
        kinds[kind] = kinds.get(kind, 0) + 1
        if not ok:
            print("NON-FINITE", it, kind, n, m, eps, K, c, rep.status, flush=True)
    print(f"soak ok: {count} solves in {time.time() - t0:.1f} s", kinds, flush=True)


if __name__ == "__main__":
    main()
