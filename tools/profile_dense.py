"""One dense C2-shaped solve for ncu captures (not a benchmark).

    python tools/profile_dense.py [--n 8192] [--iters 100] [--exact]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--m", type=int, default=0, help="columns (default n)")
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--eps", type=float, default=1e-3)
    ap.add_argument("--check", type=int, default=10)
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--general", action="store_true", help="do not pass the uniform-nu flag")
    ap.add_argument("--no-cluster", action="store_true", help="grid solver instead of the single-cluster one")
    ap.add_argument("--mult", action="store_true", help="opt in to the multiplicative column update")
    a = ap.parse_args()
    import torch

    import paper_2605_00837_b200 as lsk
    from paper_2605_00837_b200 import solver as S

    rng = np.random.Generator(np.random.PCG64(0))
    X = rng.uniform(0.0, 1.0, (a.n, 2))
    m = a.m or a.n
    Y = rng.uniform(0.0, 1.0, (m, 2))
    C = lsk.squared_euclidean_cost(X, Y)
    w = lsk.make_distribution(np.ones(a.n))
    wn = lsk.make_distribution(np.ones(m))
    lm = S._dev_f32(torch, w.log_weights)
    ln = S._dev_f32(torch, wn.log_weights)
    mu = S._dev_f32(torch, w.weights)
    cfg = lsk.SinkhornConfig(epsilon=a.eps, tolerance=1e-30, max_iterations=a.iters, check_interval=a.check)
    ws = None
    for _ in range(a.reps):
        r, ws = S._launch_solve(torch, C, lm, ln, mu, cfg, stale=not a.exact, ws=ws,
                                uniform_nu=not a.general, cluster=not a.no_cluster, mult=a.mult)
    torch.cuda.synchronize()
    print("iters", r.res.cpu().numpy()[:6], "ms", r.ev0.elapsed_time(r.ev1), flush=True)


if __name__ == "__main__":
    main()
