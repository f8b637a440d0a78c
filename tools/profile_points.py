"""Time the on-the-fly points solver on C4 / C5 shapes (not the bench).

    python tools/profile_points.py c4 [--n 65536] [--iters 20]
    python tools/profile_points.py c5 [--batch 32] [--iters 200]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["c4", "c5"])
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--direct", action="store_true", help="force the direct cost form")
    a = ap.parse_args()
    import torch

    import paper_2605_00837_b200 as lsk
    from paper_2605_00837_b200 import points as PT

    if a.which == "c4":
        rng = np.random.Generator(np.random.PCG64(0))
        X = rng.uniform(0, 1, (a.n, 3))
        Y = X + rng.normal(0, 0.01, X.shape) + np.array([0.1, 0, 0])
        cfg = lsk.SinkhornConfig(epsilon=1e-3, tolerance=1e-30, max_iterations=a.iters)
        for _ in range(a.reps):
            t = time.perf_counter()
            rep, pot = PT.solve_points_otf(X, Y, None, None, cfg, normalize="max")
            torch.cuda.synchronize()
            print(f"c4 n={a.n} K={a.iters}: device {rep.device_seconds*1e3:.1f} ms = "
                  f"{a.iters / rep.device_seconds:.1f} it/s; pairs/s {2 * a.n * a.n * a.iters / rep.device_seconds:.3e}"
                  f"; wall {time.perf_counter()-t:.2f}s status {rep.status} cost {rep.transport_cost:.6g}", flush=True)
    else:
        Xs = np.stack([np.random.Generator(np.random.PCG64(b)).uniform(0, 1, (4096, 3)) for b in range(a.batch)])
        Ys = np.stack([np.random.Generator(np.random.PCG64(1000 + b)).uniform(0, 1, (4096, 3)) for b in range(a.batch)])
        cfg = lsk.SinkhornConfig(epsilon=1e-2, tolerance=1e-30, max_iterations=a.iters)
        for _ in range(a.reps):
            outs = PT.solve_points_batched(Xs, Ys, cfg, expansion=not a.direct)
            dev = outs[0][0].device_seconds
            print(f"c5 B={a.batch} K={a.iters}: device {dev*1e3:.1f} ms = {a.batch * a.iters / dev:.1f} problem-it/s; "
                  f"pairs/s {2 * a.batch * 4096 * 4096 * a.iters / dev:.3e}", flush=True)


if __name__ == "__main__":
    main()
