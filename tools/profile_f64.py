"""fp64 (precision="double") dense solve timing at n=m=2048 and 8192: python tools/profile_f64.py"""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2605_00837_b200 as lsk
for n in (2048, 8192):
    rng = np.random.Generator(np.random.PCG64(0))
    C = lsk.squared_euclidean_cost(rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (n, 2)))
    w = lsk.make_distribution(np.ones(n))
    cfg = lsk.SinkhornConfig(epsilon=1e-3, tolerance=1e-30, max_iterations=100, precision="double")
    for _ in range(2):
        rep, pot = lsk.solve(C, w, w, cfg)
    it = rep.iterations / rep.device_seconds
    print(f"fp64 n={n}: {it:.0f} it/s, {2*8*n*n*it/1e12:.2f} TB/s of 2nm*8")
