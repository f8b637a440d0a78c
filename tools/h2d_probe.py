"""Host -> device staging of a numpy fp64 cost matrix (lsk_h2d_cost_f32, the e2e leg of
bench.py) at C2's size: time per call for several worker-thread counts and chunk
sizes, against a plain pageable torch copy. python tools/h2d_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_00837_b200 import _lib  # noqa: E402
from paper_2605_00837_b200.solver import _ptr, _stream_ptr  # noqa: E402

rng = np.random.default_rng(0)
n = 8192
C = rng.uniform(0, 2, (n, n))
out = torch.empty((n, n), dtype=torch.float32, device="cuda")
print("cpus", os.cpu_count(), flush=True)
for T in [int(x) for x in os.environ.get("PROBE_T", "0 4 8 16 24 32").split()]:
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.call("lsk_h2d_cost_f32", C.ctypes.data, 1, n, n, n, _ptr(out), n, T, _stream_ptr(torch))
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"lsk_h2d_cost_f32 threads={T or 'auto'}: {min(ts) * 1e3:.2f} ms (median {np.median(ts) * 1e3:.2f})", flush=True)
ref = torch.from_numpy(C).cuda().float()
print("equal", torch.equal(out, ref), flush=True)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x = torch.from_numpy(C).to("cuda")
    torch.cuda.synchronize()
    print(f"torch pageable fp64 copy: {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
pin = torch.empty((n, n), dtype=torch.float32).pin_memory()
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out.copy_(pin, non_blocking=True)
    torch.cuda.synchronize()
    print(f"pinned fp32 copy (PCIe floor): {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
t0 = time.perf_counter()
y = C.astype(np.float32)
print(f"numpy fp64->fp32 (1 thread): {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
