import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2605_00837_b200 as lsk
from paper_2605_00837_b200.solver import to_device_cost
rng = np.random.default_rng(0)
C = rng.uniform(0, 2, (8192, 8192))
for t in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    D = to_device_cost(lsk.CostMatrix(values=C, value_range=2.0))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("h2d_cost", (t1 - t0) * 1e3, "ms")
ref = torch.from_numpy(C).cuda().float()
print("equal", torch.equal(D.data[:, :8192], ref))
for t in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    x = torch.from_numpy(C).to("cuda")
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("torch pageable fp64", (t1 - t0) * 1e3, "ms")
import os; print("cpus", os.cpu_count())
