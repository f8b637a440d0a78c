"""Drift of the multiplicative column update against the reference arithmetic
(oracle) at fixed iteration counts: python tools/mult_drift.py [--small-eps]
(LSK_LIB selects the library build). --small-eps sweeps eps in [1e-4, 1e-3),
--gate-eps the product gate [1e-3, 2e-3], on 2048 x 2048 problems of three
geometries at K = 1000 (the update's iteration cap)."""
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

    if "--proxy" in sys.argv:
        # mult vs the direct (reference-arithmetic) update on the GPU only: a fast proxy of the drift
        print("geometry n eps/range K | rel max |f_mult - f_direct| |g_mult - g_direct| | cost", flush=True)
        for n in (2048, 4096, 8192):
            rng = np.random.default_rng(11)
            geos = {
                "uniform2d": (rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (n, 2))),
                "blobs2d": (np.concatenate([rng.normal(c, 0.05, (n // 4, 2)) for c in ((0, 0), (1, 0), (0, 1), (1, 1))]),
                            rng.uniform(0, 1, (n, 2))),
                "gauss3d": (rng.normal(0, 0.3, (n, 3)), rng.normal(0.2, 0.3, (n, 3))),
            }
            w = lsk.make_distribution(np.ones(n))
            for name, (X, Y) in geos.items():
                C64 = O.sq_euclidean_cost(X, Y)
                C = lsk.make_cost_matrix(n, n, C64 / C64.max())
                for eps in (1e-4, 2e-4, 5e-4, 1e-3, 1.5e-3, 2e-3):
                    cfg = lsk.SinkhornConfig(epsilon=eps, tolerance=1e-30, max_iterations=1000)
                    r1, p1 = lsk.solve(C, w, w, cfg, multiplicative=True, cluster=False)
                    r0, p0 = lsk.solve(C, w, w, cfg, multiplicative=False, cluster=False)
                    print(f"{name} {n} {eps} 1000 | {rel_max(p1.alpha, p0.alpha):.2e} {rel_max(p1.beta, p0.beta):.2e} | "
                          f"{abs(r1.transport_cost - r0.transport_cost) / abs(r0.transport_cost):.2e}", flush=True)
        return
    if "--small-eps" in sys.argv or "--gate-eps" in sys.argv:
        EPS = (1e-4, 2e-4, 5e-4) if "--small-eps" in sys.argv else (1e-3, 1.5e-3, 2e-3)
        rng = np.random.default_rng(11)
        n = 2048
        geos = {
            "uniform2d": (rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (n, 2))),
            "blobs2d": (np.concatenate([rng.normal(c, 0.05, (n // 4, 2)) for c in ((0, 0), (1, 0), (0, 1), (1, 1))]),
                        rng.uniform(0, 1, (n, 2))),
            "gauss3d": (rng.normal(0, 0.3, (n, 3)), rng.normal(0.2, 0.3, (n, 3))),
        }
        for name, (X, Y) in geos.items():
            C64 = O.sq_euclidean_cost(X, Y)
            C = lsk.make_cost_matrix(n, n, C64 / C64.max())
            C64 = C64 / C64.max()
            w = lsk.make_distribution(np.ones(n))
            for eps in EPS:
                K = 1000
                cfg = lsk.SinkhornConfig(epsilon=eps, tolerance=1e-30, max_iterations=K)
                ref = O.solve(C64, np.full(n, 1.0 / n), np.full(n, 1.0 / n), eps, tol=1e-30, max_iter=K)
                for mult in (True, False):
                    rep, pot = lsk.solve(C, w, w, cfg, multiplicative=mult)
                    print(f"{name} n={n} eps={eps} K={K} {'mult  ' if mult else 'direct'} "
                          f"f {rel_max(pot.alpha, ref['alpha']):.2e} g {rel_max(pot.beta, ref['beta']):.2e} "
                          f"cost {abs(rep.transport_cost - ref['cost']) / abs(ref['cost']):.2e}", flush=True)
        return
    for n, eps, K in ((1024, 1e-2, 300), (1024, 5e-3, 300), (2048, 1e-3, 500)):
        rng = np.random.default_rng(5)
        X, Y = rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (n, 2))
        C64 = O.sq_euclidean_cost(X, Y)
        C = lsk.squared_euclidean_cost(X, Y)
        w = lsk.make_distribution(np.ones(n))
        cfg = lsk.SinkhornConfig(epsilon=eps, tolerance=1e-30, max_iterations=K)
        ref = O.solve(C64, np.full(n, 1.0 / n), np.full(n, 1.0 / n), eps, tol=1e-30, max_iter=K)
        for mult in (True, False):
            rep, pot = lsk.solve(C, w, w, cfg, multiplicative=mult, cluster=False)
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
