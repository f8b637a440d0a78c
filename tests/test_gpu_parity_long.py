"""Parity at the benchmarked configurations (BASELINE configs C2, C3, C4).

Fixtures come from the reference itself (C2/C3 at n = m = 8192:
tests/golden/make_golden.py long_*) or, for C4 at n = m = 65536 where the
reference cannot run (~290 GB of temporaries), from the blocked
bit-exact oracle pinned against the reference at n = 2048
(tests/golden/make_golden_c4.py). The bar is the north star's:
max|f - f_ref| / max|f_ref| <= 1e-5 per potential (and for g) and
|cost - cost_ref| / |cost_ref| <= 1e-5, at the same eps and iteration count.

Set LSK_PARITY_LOG=<file> to append the measured errors as JSON lines
(profiles/r2_parity_errors.jsonl is such a log from a B200 run).
"""

import json
import os

import numpy as np
import pytest

import lsk_oracle as O
import paper_2605_00837_b200 as lsk
from paper_2605_00837_b200.solver import to_device_cost
from conftest import GOLDEN, golden, rel_max, sha
from inputs import fixture_points
from paper_2605_00837_b200 import points as PT

pytestmark = pytest.mark.gpu
RTOL = 1e-5


def have(name):
    return os.path.exists(os.path.join(GOLDEN, name + ".npz"))


def dist(w):
    w = np.asarray(w, np.float64)
    return lsk.DiscreteDistribution(weights=w, log_weights=np.log(w))


def config_of(z):
    return lsk.SinkhornConfig(epsilon=float(z["eps"]), tolerance=float(z["tol"]),
                              max_iterations=int(z["K"]), check_interval=int(z["check"]))


def record(name, variant, rep, pot, z):
    ef, eg = rel_max(pot.alpha, z["alpha"]), rel_max(pot.beta, z["beta"])
    ec = abs(rep.transport_cost - float(z["cost"])) / abs(float(z["cost"]))
    row = dict(fixture=name, variant=variant, K=int(z["K"]), eps=float(z["eps"]), f_rel=ef, g_rel=eg, cost_rel=ec,
               err=rep.final_marginal_error, err_ref=float(z["err"]), status=rep.status)
    log = os.environ.get("LSK_PARITY_LOG")
    if log:
        with open(log, "a") as fh:
            fh.write(json.dumps(row) + "\n")
    return ef, eg, ec


def check(name, variant, rep, pot, z):
    ef, eg, ec = record(name, variant, rep, pot, z)
    assert rep.status == str(z["status"]) and rep.iterations == int(z["iterations"])
    assert [k for k, _ in rep.error_trace] == [int(k) for k in z["trace"][:, 0]]
    assert ef <= RTOL, (name, variant, "f", ef)
    assert eg <= RTOL, (name, variant, "g", eg)
    assert ec <= RTOL, (name, variant, "cost", ec)


DENSE = ["g2_c2_n8192_k200", "g2_c2_n8192_k1000", "g2_c2_n8192_k2000", "g3_c3_n8192_k200", "g3_c3_n8192_k1000"]


@pytest.mark.parametrize("mult", [True, False], ids=["mult", "direct"])
@pytest.mark.parametrize("name", DENSE)
def test_dense_benchmarked_configs(cuda_ok, name, mult):
    """C2 (eps=1e-3) at n = m = 8192, K = 200, 1000 and 2000, and C3 (eps=1e-4) at
    K = 200 and 1000: the headline kernel (multiplicative column update where it
    applies -- C2, its first 1000 iterations) and the direct g-side arithmetic,
    both against the reference."""
    if not have(name):
        pytest.skip(f"fixture {name} not generated")
    z, X, Y, norm = fixture_points(name)
    C = lsk.squared_euclidean_cost(X, Y)
    assert sha(to_device_cost(C).values.cpu().numpy()) == str(z["C32_sha"])
    rep, pot = lsk.solve(C, dist(z["mu"]), dist(z["nu"]), config_of(z), multiplicative=mult)
    check(name, "mult" if mult else "direct", rep, pot, z)


def test_dense_c2_mult_vs_direct_k1000(cuda_ok):
    """The multiplicative update's own drift against the direct update at the
    benchmarked iteration count (both must sit inside the bar above; this
    bounds their difference)."""
    X, Y = O.uniform_points(8192, 2, 0)
    C = lsk.squared_euclidean_cost(X, Y)
    w = lsk.make_distribution(np.ones(8192))
    cfg = lsk.SinkhornConfig(epsilon=1e-3, tolerance=1e-30, max_iterations=1000)
    r1, p1 = lsk.solve(C, w, w, cfg, multiplicative=True)
    r0, p0 = lsk.solve(C, w, w, cfg, multiplicative=False)
    assert rel_max(p1.alpha, p0.alpha) <= RTOL and rel_max(p1.beta, p0.beta) <= RTOL


C4 = "g4_c4_n65536_k20"


@pytest.mark.parametrize("how", ["one_gpu", "partials_P8", "owner_P8", "allreduce_P8"])
def test_c4_full_size(cuda_ok, how):
    """C4 at its full size: generate_rigid_pair(65536, 3, 0.1, [0.1,0,0], 0.01, 0),
    C / C.max(), eps = 1e-3, on the fly, K = 20 -- on one GPU and as the
    8-rank decompositions (emulated: every virtual rank's result must agree
    bit for bit, and partials / owner must equal the one-GPU solve)."""
    if not have(C4):
        pytest.skip("C4 fixture not generated")
    z = golden(C4)
    X, Y, perm = O.rigid_pair(65536, 3, 0.1, [0.1, 0.0, 0.0], 0.01, 0)
    assert sha(X) == str(z["X_sha"]) and sha(Y) == str(z["Y_sha"])
    cfg = config_of(z)
    if how == "one_gpu":
        rep, pot = PT.solve_points_otf(X, Y, None, None, cfg, normalize="max")
    else:
        shard = how.split("_")[0]
        rep, pot, mism = PT.solve_points_emulated(X, Y, None, None, cfg, 8, "max", shard=shard)
        assert mism == 0
        if shard != "allreduce":
            r1, p1 = PT.solve_points_otf(X, Y, None, None, cfg, normalize="max")
            np.testing.assert_array_equal(pot.alpha, p1.alpha)
            np.testing.assert_array_equal(pot.beta, p1.beta)
            assert rep.transport_cost == r1.transport_cost
    check(C4, how, rep, pot, z)
