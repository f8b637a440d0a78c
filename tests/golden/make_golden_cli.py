"""Golden fixtures for the CLI harness and the seeded grid problems, made by
running the REFERENCE (build container only):

    python tests/golden/make_golden_cli.py
"""

import contextlib
import io
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import logsinkhorn as ls  # noqa: E402
from logsinkhorn import cli  # noqa: E402
from logsinkhorn.costs import generate_grid_problem, normalize_cost  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

RUNS = {
    "cli_bench": ["bench", "--n", "128", "--eps", "0.01", "--warmup", "0", "--repeats", "1", "--json"],
    "cli_bench_std": ["bench", "--n", "96", "--m", "80", "--eps", "0.05", "--domain", "standard", "--warmup", "0",
                      "--repeats", "1", "--json", "--max-cost", "2.0"],
    "cli_stability": ["stability", "--n", "64", "--eps-grid", "0.1,0.001", "--maxc-grid", "1,100",
                      "--max-iters", "300", "--json"],
    "cli_convergence": ["convergence", "--n-list", "128", "--eps-list", "0.1,0.01", "--max-iters", "2000", "--json"],
}


def main():
    for name, argv in RUNS.items():
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = cli.main(argv)
        with open(os.path.join(HERE, name + ".jsonl"), "w") as fh:
            fh.write(buf.getvalue())
        print(name, rc, len(buf.getvalue().splitlines()))
    out = {}
    for (n, m, seed) in [(7, 5, 3), (1, 4, 2), (64, 64, 0)]:
        mu, nu, C = generate_grid_problem(n, m, seed)
        out[f"mu_{n}_{m}_{seed}"] = mu.weights
        out[f"nu_{n}_{m}_{seed}"] = nu.weights
        out[f"C_{n}_{m}_{seed}"] = C.values
        out[f"Cn_{n}_{m}_{seed}"] = normalize_cost(C, 10.0).values
    np.savez_compressed(os.path.join(HERE, "cli_grid_problems.npz"), **out)


if __name__ == "__main__":
    main()
