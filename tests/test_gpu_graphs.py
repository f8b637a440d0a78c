"""CUDA-graph replay of the points solve's iteration blocks (include/lsk.h
LSK_FLAG_NO_GRAPH): replaying captured blocks of check_interval iterations
must give exactly the results of enqueueing every iteration -- status,
iteration count, checkpoint trace, potentials, cost -- for even and odd check
intervals (one or two captured shapes), caps that end mid-block, early stops
inside a replay, per-problem stops in a batch and the emulated P-rank
decompositions (their collectives captured as device copies)."""

import numpy as np
import pytest

import paper_2605_00837_b200 as lsk
from paper_2605_00837_b200 import points as PT

pytestmark = pytest.mark.gpu


def same(a, b):
    (ra, pa), (rb, pb) = a, b
    assert (ra.status, ra.iterations) == (rb.status, rb.iterations)
    assert ra.error_trace == rb.error_trace
    np.testing.assert_array_equal(pa.alpha, pb.alpha)
    np.testing.assert_array_equal(pa.beta, pb.beta)
    assert ra.transport_cost == rb.transport_cost or (np.isnan(ra.transport_cost) and np.isnan(rb.transport_cost))


@pytest.mark.parametrize("K,c,tol", [(80, 10, 1e-30), (61, 7, 1e-30), (95, 10, 1e-30), (400, 10, 1e-5),
                                     (300, 3, 1e-4)])
def test_graph_replay_matches_enqueue(cuda_ok, K, c, tol):
    rng = np.random.default_rng(K + c)
    X, Y = rng.uniform(0, 1, (3000, 3)), rng.uniform(0, 1, (2500, 3))
    cfg = lsk.SinkhornConfig(epsilon=2e-3, tolerance=tol, max_iterations=K, check_interval=c)
    a = PT.solve_points_otf(X, Y, None, None, cfg, normalize="max", graphs=True)
    b = PT.solve_points_otf(X, Y, None, None, cfg, normalize="max", graphs=False)
    same(a, b)
    if tol > 1e-20:
        assert a[0].status == "converged" and a[0].iterations < K


def test_graph_replay_batched(cuda_ok):
    """Per-problem stops inside replays: problems converge at different checkpoints."""
    rng = np.random.default_rng(2)
    X = rng.uniform(0, 1, (6, 700, 3))
    Y = rng.uniform(0, 1, (6, 800, 3)) * np.linspace(0.5, 1.5, 6)[:, None, None]
    cfg = lsk.SinkhornConfig(epsilon=1e-2, tolerance=1e-6, max_iterations=300, check_interval=5)
    outs_g = PT.solve_points_batched(X, Y, cfg, graphs=True)
    outs_e = PT.solve_points_batched(X, Y, cfg, graphs=False)
    for a, b in zip(outs_g, outs_e):
        same(a, b)
    assert len({r.iterations for r, _ in outs_g}) > 1


@pytest.mark.parametrize("shard", ["partials", "owner", "allreduce"])
def test_graph_replay_emulated_ranks(cuda_ok, shard):
    rng = np.random.default_rng(4)
    X, Y = rng.uniform(0, 1, (8192, 3)), rng.uniform(0, 1, (3000, 3))
    cfg = lsk.SinkhornConfig(epsilon=2e-3, tolerance=1e-30, max_iterations=45, check_interval=5)
    ra, pa, ma = PT.solve_points_emulated(X, Y, None, None, cfg, 4, "max", shard=shard, graphs=True)
    rb, pb, mb = PT.solve_points_emulated(X, Y, None, None, cfg, 4, "max", shard=shard, graphs=False)
    assert ma == 0 and mb == 0
    same((ra, pa), (rb, pb))
