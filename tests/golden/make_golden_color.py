"""Golden fixtures for the colour-transfer pipeline, made by running the
REFERENCE ``logsinkhorn.color_transfer_with_report`` (build container only):

    python tests/golden/make_golden_color.py

Each fixture holds the two input images, the pipeline parameters, the
reference output pixels and its SolveReport fields.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import logsinkhorn as ls  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def checker(side, seed):
    """Smooth two-tone test image with seeded jitter (the reference tests' generator)."""
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:side, 0:side]
    base = np.stack([0.25 + 0.5 * (x / max(side - 1, 1)), 0.25 + 0.5 * (y / max(side - 1, 1)),
                     0.5 + 0.3 * np.sin(2 * np.pi * x / max(side, 1))], axis=-1).reshape(-1, 3)
    base += rng.normal(0.0, 0.02, base.shape)
    return ls.make_rgb_image(side, side, base)


CASES = [
    ("color_self32", (32, 0), (32, 0), 256, 0.01, 0),
    ("color_16", (16, 1), (16, 2), 64, 0.05, 3),
    ("color_gray8", None, (8, 4), 16, 0.05, 5),
    ("color_64", (64, 21), (64, 22), 512, 0.02, 7),
]


def main():
    for name, s, t, S, eps, seed in CASES:
        src = ls.make_rgb_image(8, 8, np.full((64, 3), 0.5)) if s is None else checker(*s)
        tgt = checker(*t)
        out, rep = ls.color_transfer_with_report(src, tgt, S, eps, seed)
        path = os.path.join(HERE, name + ".npz")
        np.savez_compressed(path, src=src.pixels, tgt=tgt.pixels, width=src.width, height=src.height,
                            sample_count=S, eps=eps, seed=seed, out=out.pixels, status=rep.status,
                            iterations=rep.iterations, err=rep.final_marginal_error, cost=rep.transport_cost)
        print(name, rep.status, rep.iterations, rep.final_marginal_error, os.path.getsize(path))
    X, Y, perm = ls.generate_rigid_pair(50, 3, 0.3, (0.1, 0.2, 0.3), 0.01, 9)
    X2, Y2, perm2 = ls.generate_rigid_pair(40, 2, -0.7, (0.5, -0.25), 0.0, 4)
    np.savez_compressed(os.path.join(HERE, "rigid_pairs.npz"), X=X, Y=Y, perm=perm, X2=X2, Y2=Y2, perm2=perm2)


if __name__ == "__main__":
    main()
