"""Per-step clock64 trace of the fused dense pass (CTA 0, warps 0 and NW-1,
pass 20) from a library built with -DLSK_X_TRACE (tools/build_ablation.sh):

    LSK_LIB=$PWD/build/liblsk_trace.so python tools/trace_dense.py
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2605_00837_b200 as lsk
    from paper_2605_00837_b200 import _lib
    from paper_2605_00837_b200 import solver as S

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    rng = np.random.Generator(np.random.PCG64(0))
    X, Y = rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (8192, 2))
    C = lsk.squared_euclidean_cost(X, Y)
    w, wn = lsk.make_distribution(np.ones(n)), lsk.make_distribution(np.ones(8192))
    lm, ln, mu = S._dev_f32(torch, w.log_weights), S._dev_f32(torch, wn.log_weights), S._dev_f32(torch, w.weights)
    cfg = lsk.SinkhornConfig(epsilon=1e-3, tolerance=1e-30, max_iterations=40)
    S._launch_solve(torch, C, lm, ln, mu, cfg, uniform_nu=True)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (2 * 256 * 3 + 160))()
    _lib.load().lsk_x_read_trace(buf)
    allt = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
    t = allt[:1536].reshape(2, 256, 3)
    it = allt[1536:].reshape(2, 10, 8)
    for ci, name in ((0, "CTA0"), (1, "CTAlast")):
        for k in range(10):
            r = it[ci, k]
            nxt = it[ci, k + 1, 0] if k < 9 else 0
            print(name, 20 + k, "pass", r[1] - r[0], "store+publish", r[2] - r[1], "bar1", r[3] - r[2],
                  "combine", r[4] - r[3], "bar2", r[5] - r[4], "to next", (nxt - r[5]) if nxt else -1)
    rows = n // 148
    for wi, name in ((0, "warp0"), (1, "warpL")):
        tt = t[wi, 1:rows]
        period = np.diff(tt[:, 0])
        head = tt[:, 1] - tt[:, 0]
        post = tt[:, 2] - tt[:, 1]
        print(f"{name}: steps {len(tt)} period med {np.median(period):.0f} mean {period.mean():.0f} cyc | "
              f"head-wait med {np.median(head):.0f} mean {head.mean():.0f} | posted-wait med {np.median(post):.0f} "
              f"mean {post.mean():.0f}")
    print("warp0 first 12 (period, head, post):")
    tt = t[0, 1:14]
    for k in range(12):
        print(int(tt[k + 1, 0] - tt[k, 0]), int(tt[k, 1] - tt[k, 0]), int(tt[k, 2] - tt[k, 1]))
    print("skew warpL - warp0 at tr0 (median):", np.median(t[1, 1:rows, 0] - t[0, 1:rows, 0]))


if __name__ == "__main__":
    main()
