"""Small invocations of every persistent / synchronising kernel, for
compute-sanitizer (memcheck, racecheck, synccheck, initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize.py

Covers k_solve_dense at all four widths (m <= 1024/2048/4096/8192), general and
uniform-target instances (the cluster solvers for uniform targets at m <= 1024:
single cluster n <= 128, multi-cluster above -- also alone with `cluster`), the multiplicative column update, the exact variant, the
m > 8192 loop (uniform and general row kernels, fused checkpoint terms),
k_std_fused (standard domain, fp32 persistent), the on-the-fly points kernels
(stale, online, cost, consume), their CUDA-graph replay, and the emulated
2-rank column-partials and owner-computes solves. Shapes are small so the tools finish
in minutes; each solve still runs several checks and the grid barriers.
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2605_00837_b200 as lsk  # noqa: E402
from paper_2605_00837_b200 import points as PT  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    only = sys.argv[1] if len(sys.argv) > 1 else "all"
    if only in ("all", "dense"):
        for m in (1000, 2000, 4000, 8100):
            n = 300
            X, Y = rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (m, 2))
            C = lsk.squared_euclidean_cost(X, Y)
            uni = lsk.make_distribution(np.ones(m))
            gen = lsk.make_distribution(rng.uniform(0.5, 1.5, m))
            mu = lsk.make_distribution(np.ones(n))
            cfg = lsk.SinkhornConfig(epsilon=1e-3, tolerance=1e-30, max_iterations=12, check_interval=5)
            for nu in (uni, gen):
                for stale in (True, False):
                    r, _ = lsk.solve(C, mu, nu, cfg, stale_shift=stale)
                    print("dense", m, stale, r.status, r.iterations, flush=True)
        # multiplicative update gate: uniform nu, n*m >= 2^20, eps >= 1e-3
        X, Y = rng.uniform(0, 1, (1100, 2)), rng.uniform(0, 1, (1024, 2))
        C = lsk.squared_euclidean_cost(X, Y)
        w1, w2 = lsk.make_distribution(np.ones(1100)), lsk.make_distribution(np.ones(1024))
        r, _ = lsk.solve(C, w1, w2, lsk.SinkhornConfig(epsilon=1e-2, tolerance=1e-30, max_iterations=12))
        print("dense mult", r.status, flush=True)
        X, Y = rng.uniform(0, 1, (40, 2)), rng.uniform(0, 1, (9000, 2))
        C = lsk.squared_euclidean_cost(X, Y)
        r, _ = lsk.solve(C, lsk.make_distribution(np.ones(40)), lsk.make_distribution(np.ones(9000)),
                         lsk.SinkhornConfig(epsilon=1e-2, tolerance=1e-30, max_iterations=7, check_interval=3))
        print("dense loop", r.status, flush=True)
        r, _ = lsk.solve(C, lsk.make_distribution(rng.uniform(0.5, 1.5, 40)),
                         lsk.make_distribution(rng.uniform(0.5, 1.5, 9000)),
                         lsk.SinkhornConfig(epsilon=1e-2, tolerance=1e-30, max_iterations=7, check_interval=3))
        print("dense loop general", r.status, flush=True)
    if only in ("all", "dense", "cluster"):
        # cluster solvers: single cluster, multi-cluster with one and with several rows per warp,
        # padded columns, the guards (eps = 1e-4), early stop, exact variant
        for n, m, eps in ((100, 1000, 1e-2), (300, 1000, 1e-3), (1500, 1024, 1e-2), (700, 900, 1e-4)):
            X, Y = rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (m, 2))
            C = lsk.squared_euclidean_cost(X, Y)
            mu, nu = lsk.make_distribution(rng.uniform(0.5, 1.5, n)), lsk.make_distribution(np.ones(m))
            for stale in (True, False):
                cfg = lsk.SinkhornConfig(epsilon=eps, tolerance=1e-30, max_iterations=12, check_interval=5)
                r, _ = lsk.solve(C, mu, nu, cfg, stale_shift=stale)
                print("cluster", n, m, stale, r.status, r.iterations, flush=True)
            r, _ = lsk.solve(C, mu, nu, lsk.SinkhornConfig(epsilon=0.05, tolerance=1e-3, max_iterations=300,
                                                           check_interval=2))
            print("cluster early stop", n, r.status, r.iterations, flush=True)
    if only in ("all", "standard"):
        X, Y = rng.uniform(0, 1, (500, 2)), rng.uniform(0, 1, (700, 2))
        C = lsk.squared_euclidean_cost(X, Y)
        r, _, _ = lsk.solve_standard_domain(C, lsk.make_distribution(np.ones(500)), lsk.make_distribution(np.ones(700)),
                                            lsk.SinkhornConfig(epsilon=0.05, tolerance=1e-30, max_iterations=12,
                                                               check_interval=5))
        print("standard", r.status, flush=True)
    if only in ("all", "points"):
        X, Y = rng.uniform(0, 1, (700, 3)), rng.uniform(0, 1, (2500, 3))
        cfg = lsk.SinkhornConfig(epsilon=1e-3, tolerance=1e-30, max_iterations=8, check_interval=3)
        for stale in (True, False):
            r, pot = PT.solve_points_otf(X, Y, None, None, cfg, normalize="max", stale_shift=stale)
            print("points", stale, r.status, flush=True)
        from paper_2605_00837_b200.applications import barycentric_map_points

        barycentric_map_points(X, Y, pot, 1e-3, normalize="max")
        # CUDA-graph replay of the iteration blocks (>= 3 blocks of check_interval iterations)
        cfgg = lsk.SinkhornConfig(epsilon=1e-3, tolerance=1e-30, max_iterations=20, check_interval=3)
        r, _ = PT.solve_points_otf(X, Y, None, None, cfgg, normalize="max")
        print("points graphs", r.status, r.iterations, flush=True)
        rb = PT.solve_points_batched(np.stack([X[:300]] * 3), np.stack([Y[:400]] * 3), cfgg)
        print("points batched graphs", rb[0][0].status, flush=True)
        X2, Y2 = rng.uniform(0, 1, (4100, 3)), rng.uniform(0, 1, (900, 3))
        for shard in ("partials", "owner"):
            r, _, mism = PT.solve_points_emulated(X2, Y2, None, None, cfg, 2, "max", shard=shard)
            print("emulated", shard, r.status, mism, flush=True)


if __name__ == "__main__":
    main()
