"""Standard-domain solve timing at n=m (fp32 or fp64): python tools/profile_standard.py [n] [double]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2605_00837_b200 as lsk

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    prec = "double" if len(sys.argv) > 2 and sys.argv[2] == "double" else "single"
    rng = np.random.Generator(np.random.PCG64(0))
    C = lsk.squared_euclidean_cost(rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (n, 2)))
    w = lsk.make_distribution(np.ones(n))
    cfg = lsk.SinkhornConfig(epsilon=0.05, tolerance=1e-30, max_iterations=200, precision=prec)
    for _ in range(2):
        rep, _, _ = lsk.solve_standard_domain(C, w, w, cfg)
    it = rep.iterations / rep.device_seconds
    b = (8 if prec == "double" else 4) * 2.0 * n * n
    print(f"standard {prec} n={n}: {it:.0f} it/s, {b * it / 1e12:.2f} TB/s of 2nm*{int(b / 2 / n / n)} B/it, {rep.status}")


if __name__ == "__main__":
    main()
