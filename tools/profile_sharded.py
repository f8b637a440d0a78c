"""Timing of the sharded C4 designs on ONE GPU through the P-rank emulation
(``solve_points_emulated``): every virtual rank runs its own kernels on its
own slab, rank after rank, and the collectives are device copies. The device
time of a solve is therefore the SUM over ranks; time / P estimates one
rank's compute (+ its share of the copies) on a P-GPU box, i.e. the strong-
scaling ceiling before NCCL transport. Writes a markdown table to stdout.

    python tools/profile_sharded.py [--n 65536] [--iters 50]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--iters", type=int, default=50)
    a = ap.parse_args()
    import paper_2605_00837_b200 as lsk
    from paper_2605_00837_b200 import color as CL
    from paper_2605_00837_b200 import points as PT

    X, Y, _ = CL.generate_rigid_pair(a.n, 3, 0.1, [0.1, 0.0, 0.0], 0.01, 0)
    cfg = lsk.SinkhornConfig(epsilon=1e-3, tolerance=1e-30, max_iterations=a.iters)
    PT.solve_points_otf(X, Y, None, None, cfg, normalize="max")
    r1, p1 = PT.solve_points_otf(X, Y, None, None, cfg, normalize="max")
    base = r1.device_seconds / a.iters
    print(f"C4 rigid pair n=m={a.n}, eps=1e-3, {a.iters} iterations, one B200; unsharded: "
          f"{base * 1e3:.3f} ms/iteration\n")
    print("| design | P | CUDA graphs | device ms / iteration (all ranks, serial) | per-rank estimate (/P) | "
          "ideal (unsharded / P) | per-rank overhead | bitwise = unsharded | ranks agree |")
    print("|---|---|---|---|---|---|---|---|---|")
    for shard in ("partials", "owner", "allreduce"):
        for P in (1, 2, 4, 8):
            for graphs in (True, False):
                PT.solve_points_emulated(X, Y, None, None, cfg, P, "max", shard=shard, graphs=graphs)
                r, p, mism = PT.solve_points_emulated(X, Y, None, None, cfg, P, "max", shard=shard, graphs=graphs)
                t = r.device_seconds / a.iters
                same = bool(np.array_equal(p.alpha, p1.alpha) and np.array_equal(p.beta, p1.beta))
                print(f"| {shard} | {P} | {'on' if graphs else 'off'} | {t * 1e3:.3f} | {t / P * 1e3:.3f} | "
                      f"{base / P * 1e3:.3f} | {(t / P - base / P) / (base / P) * 100:+.1f}% | {same} | {mism == 0} |",
                      flush=True)


if __name__ == "__main__":
    main()
