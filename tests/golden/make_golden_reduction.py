"""Golden fixtures for the deterministic reductions and the plan diagnostics,
made by running the REFERENCE (build container only):

    python tests/golden/make_golden_reduction.py
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import logsinkhorn as ls  # noqa: E402
from logsinkhorn import reduction as red  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
PLANS = [(32, 256), (1, 1), (64, 128), (4, 12), (8, 8), (3, 9), (16, 512)]


def arrays():
    rng = np.random.default_rng(3)
    out = {}
    for dt in (np.float32, np.float64):
        tag = "f32" if dt == np.float32 else "f64"
        A = rng.standard_normal((7, 1000)).astype(dt) * 5
        A[1, ::3] = -np.inf
        A[2, :] = -np.inf                      # an empty row (LSE -> -inf)
        A[3, 10] = -0.0
        A[4, :] = -0.0                          # signed zeros through max and sum
        out[f"rows_{tag}"] = A
        out[f"short_{tag}"] = rng.standard_normal((3, 5)).astype(dt)        # L < group_size
        out[f"cols_{tag}"] = (rng.standard_normal((777, 9)) * 3).astype(dt)  # column reductions
        out[f"nan_{tag}"] = np.array([[1.0, np.nan, 3.0, -np.inf, 2.0] * 60], dtype=dt)
    return out


def main():
    data = arrays()
    res = {}
    for k, A in data.items():
        for (w, B) in PLANS:
            plan = red.ReductionPlan(w, B)
            cols = k.startswith("cols")
            with np.errstate(all="ignore"):
                if cols:
                    res[f"{k}|{w}|{B}|max"] = red.reduce_max_cols(A, plan)
                    res[f"{k}|{w}|{B}|sum"] = red.reduce_sum_cols(A, plan)
                    res[f"{k}|{w}|{B}|lse"] = red.log_sum_exp_cols(A, plan)
                else:
                    res[f"{k}|{w}|{B}|max"] = red.reduce_max_rows(A, plan)
                    res[f"{k}|{w}|{B}|sum"] = red.reduce_sum_rows(A, plan)
                    res[f"{k}|{w}|{B}|lse"] = red.log_sum_exp_rows(A, plan)
    v = data["rows_f64"][0]
    res["view|max"] = np.array(red.reduce_max(v))
    res["view|sum"] = np.array(red.reduce_sum(v))
    res["view|lse"] = np.array(red.log_sum_exp(v))
    np.savez_compressed(os.path.join(HERE, "reduction.npz"), **{("in:" + k): a for k, a in data.items()},
                        **{("out:" + k): a for k, a in res.items()})
    # diagnostics on a solved problem (fp32 and fp64)
    rng = np.random.Generator(np.random.PCG64(11))
    X, Y = rng.uniform(0, 1, (40, 2)), rng.uniform(0, 1, (50, 2))
    C = ls.squared_euclidean_cost(X, Y)
    mu = ls.make_distribution(rng.uniform(0.5, 1.5, 40))
    nu = ls.make_distribution(rng.uniform(0.5, 1.5, 50))
    diag = {"C": C.values, "wa": mu.weights, "wb": nu.weights}
    for prec in ("single", "double"):
        cfg = ls.SinkhornConfig(epsilon=0.05, precision=prec, max_iterations=300)
        rep, pot = ls.solve(C, mu, nu, cfg)
        plan = ls.materialize_plan(C, mu, nu, pot.alpha, pot.beta, 0.05)
        diag[f"{prec}_alpha"] = pot.alpha
        diag[f"{prec}_beta"] = pot.beta
        diag[f"{prec}_plan"] = plan.values
        diag[f"{prec}_kkt"] = ls.kkt_residual(C, mu, nu, plan, pot.alpha, pot.beta, 0.05)
        diag[f"{prec}_obj"] = ls.regularized_objective(C, mu, nu, plan, 0.05)
    diag["crb"] = np.array([ls.contraction_rate_bound(R, e) for R, e in ((1.0, 0.1), (0.5, 0.01), (0.0, 1.0))])
    np.savez_compressed(os.path.join(HERE, "diagnostics.npz"), **diag)
    print("reduction cases", len(res), "diagnostics", {k: v for k, v in diag.items() if k.endswith(("kkt", "obj"))})


if __name__ == "__main__":
    main()
