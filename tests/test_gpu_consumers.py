"""Plan consumers without the plan vs numpy on the plan.

The reference computes P = materialize_plan(...) then barycentric_map(P, Y)
(applications.py:75-97) or P.argmax(axis=1) (195-204). Here the same
quantities come from the potentials on the fly; the check recomputes the plan
in fp64 from the same potentials and compares.
"""

import numpy as np
import pytest

import lsk_oracle as O
import paper_2605_00837_b200 as lsk
from paper_2605_00837_b200 import applications as A
from paper_2605_00837_b200 import points as PT

pytestmark = pytest.mark.gpu


def plan64(C64, f, g, eps, n, m):
    z = (f.astype(np.float64)[:, None] + g.astype(np.float64)[None, :] - C64) / np.float32(eps)
    return np.exp(z + np.log(1.0 / n) + np.log(1.0 / m))


def test_barycentric_map_points(cuda_ok):
    n, m, d, eps = 300, 517, 3, 0.02
    X, _ = O.uniform_points(n, d, 1)
    _, Y = O.uniform_points(m, d, 2)
    cfg = lsk.SinkhornConfig(epsilon=eps, tolerance=1e-30, max_iterations=50)
    rep, pot = PT.solve_points_otf(X, Y, None, None, cfg)
    mapped = A.barycentric_map_points(X, Y, pot, eps)
    P = plan64(O.sq_euclidean_cost(X, Y), pot.alpha, pot.beta, eps, n, m)
    want = (P @ Y) / P.sum(axis=1)[:, None]
    np.testing.assert_allclose(mapped, want, rtol=2e-5, atol=2e-6)


def test_barycentric_map_dense_plan(cuda_ok):
    n, m, eps = 64, 80, 0.05
    X, Y = O.uniform_points(n, 2, 3)
    Y = Y[:m] if m <= n else np.vstack([Y, Y])[:m]
    C64 = O.sq_euclidean_cost(X, Y)
    cfg = lsk.SinkhornConfig(epsilon=eps)
    w_n, w_m = lsk.make_distribution(np.ones(n)), lsk.make_distribution(np.ones(m))
    rep, pot = lsk.solve(lsk.CostMatrix(values=C64), w_n, w_m, cfg)
    plan = lsk.materialize_plan(lsk.CostMatrix(values=C64), w_n, w_m, pot.alpha, pot.beta, eps)
    got = A.barycentric_map(plan, Y)
    P = plan.values.astype(np.float64)
    np.testing.assert_allclose(got, (P @ Y) / P.sum(1)[:, None], rtol=1e-12)


def test_match_point_clouds_rigid(cuda_ok):
    n = 2048
    X, Y, perm = O.rigid_pair(n, 3, 0.1, [0.1, 0.0, 0.0], 0.01, 0)
    pairs, rep = A.match_point_clouds_with_report(X, Y, 1e-3, lsk.SinkhornConfig(epsilon=1e-3, max_iterations=300))
    assert [p.source_index for p in pairs] == list(range(n))
    idx = np.array([p.target_index for p in pairs])
    # the argmax of the fp64 plan built from the same potentials (ties/near-ties aside)
    C = O.max_normalized(O.sq_euclidean_cost(X, Y))
    _, pot = PT.solve_points_otf(X, Y, None, None, lsk.SinkhornConfig(epsilon=1e-3, max_iterations=300),
                                 normalize="max")
    P = plan64(C, pot.alpha, pot.beta, 1e-3, n, n)
    agree = np.mean(idx == P.argmax(axis=1))
    assert agree > 0.995, agree
    w = np.array([p.weight for p in pairs])
    np.testing.assert_allclose(w, P[np.arange(n), idx], rtol=1e-3)
    assert np.mean(idx == perm) > 0.5  # the matching problem itself is solved (sanity)
