"""The multi-GPU data plane on one B200: P virtual ranks.

``solve_points_emulated`` runs the exact P-rank decomposition of the sharded
points solve -- each rank's slab, its own workspace, the exchanges of
partials / potential slabs -- with the collectives replaced by device copies.
The reference contract is that results do not depend on the worker count
(tests/test_solver.py:247-257 bit-identical repeats):

* owner computes and column partials: bit-identical to the unsharded solve
  for every P, and every virtual rank ends with the same bits;
* allreduce (stale sums combined by a SUM collective): within float rounding.

Only NCCL itself (the transport of the same bytes) is left to a multi-GPU run.
"""

import numpy as np
import pytest

import lsk_oracle as O
import paper_2605_00837_b200 as lsk

from conftest import rel_max
from paper_2605_00837_b200 import points as PT

pytestmark = pytest.mark.gpu


def cfg(eps, K, tol=1e-30, check=10):
    return lsk.SinkhornConfig(epsilon=eps, tolerance=tol, max_iterations=K, check_interval=check)


def same(a, b):
    (ra, pa), (rb, pb) = a, b
    assert ra.status == rb.status and ra.iterations == rb.iterations
    assert ra.error_trace == rb.error_trace
    np.testing.assert_array_equal(pa.alpha, pb.alpha)
    np.testing.assert_array_equal(pa.beta, pb.beta)
    assert ra.transport_cost == rb.transport_cost or (np.isnan(ra.transport_cost) and np.isnan(rb.transport_cost))


def emu(X, Y, c, P, shard, **kw):
    rep, pot, mism = PT.solve_points_emulated(X, Y, None, None, c, P, kw.pop("normalize", "max"), shard=shard, **kw)
    assert mism == 0, f"{mism} virtual ranks disagree with rank 0 ({shard}, P={P})"
    return rep, pot


@pytest.mark.parametrize("shard,Ps", [("owner", [1, 2, 3, 4, 8]), ("partials", [1, 2, 4, 8])])
def test_sharded_bitwise_equals_one_gpu(cuda_ok, shard, Ps):
    """C4-shaped (rigid pair, C/max, eps=1e-3) with a ragged target count."""
    X, Y, _ = O.rigid_pair(16384, 3, 0.1, [0.1, 0.0, 0.0], 0.01, 0)
    Y = Y[:12001]
    c = cfg(1e-3, 23)
    ref = PT.solve_points_otf(X, Y, None, None, c, normalize="max")
    for P in Ps:
        same(emu(X, Y, c, P, shard), ref)


def test_sharded_allreduce_close(cuda_ok):
    X, Y, _ = O.rigid_pair(16384, 3, 0.1, [0.1, 0.0, 0.0], 0.01, 1)
    c = cfg(1e-3, 30)
    rr, pr = PT.solve_points_otf(X, Y, None, None, c, normalize="max")
    for P in (1, 2, 4, 8):
        r, p = emu(X, Y, c, P, "allreduce")
        assert r.iterations == rr.iterations
        assert rel_max(p.alpha, pr.alpha) <= 1e-6 and rel_max(p.beta, pr.beta) <= 1e-6, P
        assert abs(r.transport_cost - rr.transport_cost) <= 1e-6 * abs(rr.transport_cost)
        if P == 1:
            same((r, p), (rr, pr))


@pytest.mark.parametrize("n,m,d", [(5000, 777, 2), (2049, 4096, 3), (300, 5000, 1)])
def test_sharded_ragged_and_empty_slabs(cuda_ok, n, m, d):
    """Slabs that do not divide evenly; partials ranks with no source chunk."""
    X, _ = O.uniform_points(n, d, n)
    _, Y = O.uniform_points(m, d, m + 7)
    c = cfg(0.01, 31, check=7)
    ref = PT.solve_points_otf(X, Y, None, None, c, normalize="none")
    for P in (2, 3, 5):
        same(emu(X, Y, c, P, "owner", normalize="none"), ref)
    L2 = 1
    while L2 < -(-n // 2048):
        L2 *= 2
    for P in (1, 2, 4):
        if P <= L2:
            same(emu(X, Y, c, P, "partials", normalize="none"), ref)
    if 2 * L2 <= 16:
        with pytest.raises(ValueError):
            emu(X, Y, c, 2 * L2, "partials", normalize="none")


def test_sharded_exact_variant_and_guard(cuda_ok):
    """The online (max, sumexp) pair exchange on every iteration (stale shift
    off) and the stale guard's exact fallback under sharding: both bitwise."""
    X, Y = O.uniform_points(6000, 2, 11)
    c = cfg(3e-4, 15)
    for stale in (False, True):
        ref = PT.solve_points_otf(X * 3, Y * 3, None, None, c, normalize="none", stale_shift=stale)
        for P in (2, 4):
            same(emu(X * 3, Y * 3, c, P, "partials", normalize="none", stale_shift=stale), ref)
            same(emu(X * 3, Y * 3, c, P, "owner", normalize="none", stale_shift=stale), ref)


def test_sharded_convergence_stop(cuda_ok):
    """A solve that converges stops at the same check on every rank."""
    X, Y = O.uniform_points(4500, 2, 3)
    c = cfg(0.05, 2000, tol=1e-6)
    ref = PT.solve_points_otf(X, Y, None, None, c, normalize="none")
    assert ref[0].status == "converged" and ref[0].iterations < 2000
    for shard, P in (("partials", 2), ("owner", 3), ("allreduce", 2)):
        r, p = emu(X, Y, c, P, shard, normalize="none")
        assert r.status == "converged"
        if shard != "allreduce":
            same((r, p), ref)
