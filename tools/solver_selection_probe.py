"""Which dense solver runs for m = 1024 at several n (LSK_VERBOSE=1 names each launch):
LSK_VERBOSE=1 python tools/solver_selection_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, paper_2605_00837_b200 as lsk
rng = np.random.default_rng(0)
for n in (200, 1024, 4096, 30000):
    C = lsk.squared_euclidean_cost(rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (1024, 2)))
    r, _ = lsk.solve(C, lsk.make_distribution(np.ones(n)), lsk.make_distribution(np.ones(1024)),
                     lsk.SinkhornConfig(epsilon=1e-2, tolerance=1e-30, max_iterations=5))
    print("n", n, r.status, r.iterations, flush=True)
