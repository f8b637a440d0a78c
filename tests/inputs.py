"""Regenerate the exact inputs of every golden fixture from its recipe.

Uses only the oracle's seeded generators (the same numpy PCG64 streams the
reference generators use); each regenerated input is checked against the
sha256 prefix stored in the fixture by tests/golden/make_golden.py.
"""

import numpy as np

import lsk_oracle as O
from conftest import golden, sha


def fixture_problem(name):
    """-> (z, C64, mu_w, nu_w) for a solve fixture."""
    z = golden(name)
    keys = set(z.files)
    if "grid" in keys:
        n, m, seed = (int(v) for v in z["grid"])
        mu_w, nu_w, C64 = O.grid_problem(n, m, seed)
    elif "shape" in keys:
        n, m = (int(v) for v in z["shape"])
        C64, mu_w, nu_w, _, _ = O.random_problem(n, m, int(z["seed"]))
    elif "C" in keys:
        C64 = z["C"]
        mu_w, nu_w = z["mu"], z["nu"]
    elif "perm" in keys:  # rigid pair, max-normalised
        n = z["alpha"].shape[0]
        X, Y, perm = O.rigid_pair(n, 3, 0.1, [0.1, 0.0, 0.0], 0.01, 0)
        assert sha(X) == str(z["X_sha"]) and sha(Y) == str(z["Y_sha"])
        C64 = O.max_normalized(O.sq_euclidean_cost(X, Y))
        mu_w = nu_w = np.full(n, 1.0 / n)
        mu_w = z["mu"]
        nu_w = z["nu"]
    else:  # uniform points
        n, d, seed = int(z["n"]), int(z["d"]), int(z["seed"])
        X, Y = O.uniform_points(n, d, seed)
        assert sha(X) == str(z["X_sha"]) and sha(Y) == str(z["Y_sha"])
        C64 = O.sq_euclidean_cost(X, Y)
        if bool(z["normalize"]):
            C64 = O.max_normalized(C64)
        mu_w, nu_w = z["mu"], z["nu"]
    assert sha(C64.astype(np.float32)) == str(z["C32_sha"]), name
    return z, C64, mu_w, nu_w


def fixture_points(name):
    """-> (z, X, Y, normalize) for the point-cloud fixtures."""
    z = golden(name)
    if "perm" in z.files:
        n = z["alpha"].shape[0]
        X, Y, _ = O.rigid_pair(n, 3, 0.1, [0.1, 0.0, 0.0], 0.01, 0)
        return z, X, Y, "max"
    n, d, seed = int(z["n"]), int(z["d"]), int(z["seed"])
    X, Y = O.uniform_points(n, d, seed)
    return z, X, Y, ("max" if bool(z["normalize"]) else "none")
