import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2605_00837_b200 as lsk
from paper_2605_00837_b200 import color as CL, points as PT
X, Y, _ = CL.generate_rigid_pair(65536, 3, 0.1, [0.1, 0.0, 0.0], 0.01, 0)
cfg = lsk.SinkhornConfig(epsilon=1e-3, tolerance=1e-30, max_iterations=12, check_interval=10)
r, p, m = PT.solve_points_emulated(X, Y, None, None, cfg, 8, "max", shard="partials", graphs=False)
print(r.device_seconds)
