"""Per-phase clock64 trace of the cluster dense solvers (iterations 20-29, thread 0
of the first and last CTA) from a library built with -DLSK_X_TRACE
(tools/build_ablation.sh trace -DLSK_X_TRACE):

    LSK_LIB=$PWD/build/liblsk_trace.so python tools/trace_cluster.py [n] [m]

Phases: rows (load g + f pass), CTA partial, cluster barrier A, publish
(cluster slice sums to global; MC only), grid barrier (MC only), finish (g^k
from the cluster partials + DSMEM broadcast), cluster barrier B, then the loop
top to the next iteration.
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

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    rng = np.random.Generator(np.random.PCG64(0))
    X, Y = rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (m, 2))
    C = lsk.squared_euclidean_cost(X, Y)
    w, wn = lsk.make_distribution(np.ones(n)), lsk.make_distribution(np.ones(m))
    lm, ln, mu = S._dev_f32(torch, w.log_weights), S._dev_f32(torch, wn.log_weights), S._dev_f32(torch, w.weights)
    cfg = lsk.SinkhornConfig(epsilon=1e-2, tolerance=1e-30, max_iterations=40, check_interval=1000)
    S._launch_solve(torch, C, lm, ln, mu, cfg, uniform_nu=True)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (2 * 256 * 3 + 160))()
    _lib.load().lsk_x_read_trace(buf)
    allt = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
    it = allt[1536:].reshape(2, 10, 8)
    names = ["rows", "cta-partial", "barA", "publish", "gridbar", "finish", "barB"]
    tot = {k: [] for k in names + ["top", "total"]}
    for ci, name in ((0, "CTA0"), (1, "CTAlast")):
        for k in range(9):
            r = it[ci, k]
            d = np.diff(r[[0, 1, 2, 3, 4, 5, 6, 7]])
            top = it[ci, k + 1, 0] - r[7]
            print(name, 20 + k, " ".join(f"{nm} {int(x)}" for nm, x in zip(names, d)), "top", int(top),
                  "total", int(it[ci, k + 1, 0] - r[0]))
            for nm, x in zip(names, d):
                tot[nm].append(x)
            tot["top"].append(top)
            tot["total"].append(it[ci, k + 1, 0] - r[0])
    rw = allt[:40].reshape(10, 4)  # CTA 0 warp 0's first row of the f pass: start, row loaded, f_i, column update
    d = np.diff(rw, axis=1)
    print("warp 0 row (median cycles): take_row", np.median(d[:, 0]), "f-side to f_i", np.median(d[:, 1]),
          "column update", np.median(d[:, 2]), "| loop top -> row start", np.median(rw[:9, 0] - it[0, :9, 0]))
    print("median cycles:", " ".join(f"{k} {np.median(v):.0f}" for k, v in tot.items()))


if __name__ == "__main__":
    main()
