"""Parity of the CUDA path (through the C ABI) against the reference.

Targets are the golden fixtures the reference itself produced
(tests/golden/make_golden.py) plus, at sizes the CPU finishes in seconds,
the oracle run live on the same inputs. Bars (north star):
potentials and transport cost within 1e-5 relative (max-norm) in fp32;
status, iteration count and checkpoint iterations identical; marginal errors
within their fp32 rounding noise.
"""

import numpy as np
import pytest

import lsk_oracle as O
import paper_2605_00837_b200 as lsk
from paper_2605_00837_b200.solver import to_device_cost
from conftest import golden, golden_names, rel_max, sha
from inputs import fixture_points, fixture_problem

pytestmark = pytest.mark.gpu

SMALL = [n for n in golden_names() if n.startswith(("grid", "rand_", "antidiag", "constant", "failure"))]
BIG = ["g1_c1_n1024", "g2_c2_n8192_k10", "g3_c3_n8192_k10", "n1024_eps1e-4_k1000", "n2048_eps1e-3_k200",
       "g5_c5_n4096_rgb_k200", "rigid2048_eps1e-3_k200"]
RTOL = 1e-5  # north-star parity bar, fp32 vs the reference's single precision


def dist(w):
    w = np.asarray(w, np.float64)
    return lsk.DiscreteDistribution(weights=w, log_weights=np.log(w))


def config_of(z):
    return lsk.SinkhornConfig(epsilon=float(z["eps"]), tolerance=float(z["tol"]),
                              max_iterations=int(z["K"]), check_interval=int(z["check"]))


def assert_potentials(pot, z):
    fa, fb = np.asarray(pot.alpha), np.asarray(pot.beta)
    ra, rb = z["alpha"], z["beta"]
    if not np.isfinite(ra).all():
        assert not (np.isfinite(fa).all() and np.isfinite(fb).all())
        return
    scale = max(np.abs(ra).max(), np.abs(rb).max())
    for x, ref in ((fa, ra), (fb, rb)):
        den = max(np.abs(ref).max(), 1e-2 * scale)
        assert np.abs(x.astype(np.float64) - ref).max() <= RTOL * den, (np.abs(x - ref).max(), den)


def err_tol(ref_err, mu):
    # |r_i - mu_i| terms carry fp32 rounding of r_i ~ mu_i: a few ulps each
    return 1e-4 * abs(ref_err) + len(mu) * float(np.max(mu)) * 2.0 ** -21


def _assert_semantics(rep, z):
    """The reference's own status/trace contract (tests/test_solver.py:210-238)."""
    c, K, tol = int(z["check"]), int(z["K"]), float(z["tol"])
    ks = [k for k, _ in rep.error_trace]
    want = list(range(c, rep.iterations + 1, c))
    if rep.iterations % c and rep.iterations == K:
        want.append(K)  # the extra check at a cap that is not a checkpoint (solver.py:301-316)
    if rep.status != "numerical_failure":
        assert ks == want
        assert rep.error_trace[-1][1] == pytest.approx(rep.final_marginal_error, rel=1e-6)
        assert (rep.status == "converged") == (rep.final_marginal_error < tol)
        assert rep.status == "converged" or rep.iterations == K


def assert_report(rep, z, mu):
    tr = z["trace"]
    tol = float(z["tol"])
    # A checkpoint whose reference error is within fp32 noise of the tolerance
    # is a coin flip for any implementation whose exp/log/summation order differ
    # from numpy's (near the floor the error IS rounding noise).
    # There the stop iteration may differ; the traces must agree up to it and
    # the reference's status/trace semantics must hold.
    amb = [int(k) for k, e in tr if abs(e - tol) <= err_tol(e, mu)]
    if amb:
        n_common = sum(1 for k, _ in tr if int(k) < amb[0])
        assert [k for k, _ in rep.error_trace[:n_common]] == [int(k) for k in tr[:n_common, 0]]
        for (_, e), (_, er) in zip(rep.error_trace[:n_common], tr[:n_common]):
            assert abs(e - er) <= err_tol(er, mu), (e, er)
        assert rep.iterations >= amb[0]
        _assert_semantics(rep, z)
        return True
    assert rep.status == str(z["status"])
    assert rep.iterations == int(z["iterations"])
    assert [k for k, _ in rep.error_trace] == [int(k) for k in tr[:, 0]]
    for (_, e), (_, er) in zip(rep.error_trace, tr):
        assert abs(e - er) <= err_tol(er, mu), (e, er)
    ref_err = float(z["err"])
    if np.isnan(ref_err):
        assert np.isnan(rep.final_marginal_error)
    else:
        assert abs(rep.final_marginal_error - ref_err) <= err_tol(ref_err, mu)
    ref_cost = float(z["cost"])
    if np.isnan(ref_cost):
        assert np.isnan(rep.transport_cost)
    else:
        assert abs(rep.transport_cost - ref_cost) <= RTOL * abs(ref_cost) + 1e-12
    return False


@pytest.mark.parametrize("variant", ["stale", "exact"])
@pytest.mark.parametrize("name", SMALL)
def test_solve_small(cuda_ok, name, variant):
    z, C64, mu_w, nu_w = fixture_problem(name)
    stale = variant == "stale"
    with np.errstate(all="ignore"):
        rep, pot = lsk.solve(lsk.CostMatrix(values=C64), dist(mu_w), dist(nu_w), config_of(z), stale_shift=stale)
    if assert_report(rep, z, mu_w) and rep.iterations != int(z["iterations"]):
        # stopped at a different (noise-decided) checkpoint: compare with the
        # oracle run to the same iteration count instead
        r = O.solve(C64, mu_w, nu_w, float(z["eps"]), tol=1e-30, max_iter=rep.iterations, check=int(z["check"]))
        assert rel_max(pot.alpha, r["alpha"]) <= RTOL and rel_max(pot.beta, r["beta"]) <= RTOL
    else:
        assert_potentials(pot, z)


@pytest.mark.parametrize("mult", [True, False], ids=["mult", "direct"])
@pytest.mark.parametrize("name", BIG)
def test_solve_golden_points(cuda_ok, name, mult):
    """C1/C2/C3/C5-shaped fixtures; the cost is built on the device (fp64-exact)."""
    z, X, Y, norm = fixture_points(name)
    C = lsk.squared_euclidean_cost(X, Y, normalize=norm)
    assert sha(to_device_cost(C).values.cpu().numpy()) == str(z["C32_sha"])  # fp32(C64) bit for bit
    rep, pot = lsk.solve(C, dist(z["mu"]), dist(z["nu"]), config_of(z), multiplicative=mult)
    assert_report(rep, z, z["mu"])
    assert_potentials(pot, z)


def test_half_steps(cuda_ok):
    z = golden("half_steps")
    eps = float(z["eps"])
    for n, m in z["shapes"]:
        n, m = int(n), int(m)
        key = f"{n}x{m}"
        C64, mu_w, nu_w, a_in, b_in = O.random_problem(n, m, 100 + n + m)
        cost = lsk.CostMatrix(values=C64)
        mu, nu = dist(mu_w), dist(nu_w)
        a = lsk.update_alpha(cost, nu, b_in, eps)
        assert a.dtype == np.float32 and rel_max(a, z[key + "_alpha"]) <= RTOL
        b = lsk.update_beta(cost, mu, a_in, eps)
        assert rel_max(b, z[key + "_beta_out"]) <= RTOL
        bt = lsk.update_beta(cost, mu, a_in, eps, transposed_cost=np.ascontiguousarray(C64.T))
        np.testing.assert_array_equal(b, bt)  # strided == transposed, bitwise (test_solver.py:101-111)
        e = lsk.marginal_error(cost, mu, nu, a_in, b_in, eps)
        assert abs(e - float(z[key + "_merr"])) <= err_tol(float(z[key + "_merr"]), mu_w)
        c = lsk.transport_cost(cost, mu, nu, a_in, b_in, eps)
        assert abs(c - float(z[key + "_tcost"])) <= RTOL * abs(float(z[key + "_tcost"]))
        P = lsk.materialize_plan(cost, mu, nu, a_in, b_in, eps).values
        assert P.dtype == np.float32 and P.shape == (n, m)
        np.testing.assert_allclose(P[:4, :4], z[key + "_plan_corner"], rtol=1e-5)
        np.testing.assert_allclose(P.sum(axis=1, dtype=np.float64), z[key + "_plan_rows"], rtol=1e-5)


def test_known_answers(cuda_ok):
    """Reference known answers (tests/test_solver.py:38-49, 163-178)."""
    cost = lsk.make_cost_matrix(1, 1, [0.5])
    nu = lsk.make_distribution([1.0])
    assert lsk.update_alpha(cost, nu, np.zeros(1, np.float32), 0.1)[0] == pytest.approx(0.5, rel=1e-6)
    c = lsk.make_cost_matrix(3, 4, [0.7] * 12)
    np.testing.assert_allclose(lsk.update_alpha(c, lsk.make_distribution([1.0] * 4), np.zeros(4, np.float32), 0.3),
                               0.7, rtol=1e-6)
    w4 = lsk.make_distribution([1.0] * 4)
    c4 = lsk.make_cost_matrix(4, 4, [0.3] * 16)
    v = lsk.transport_cost(c4, w4, w4, np.full(4, 0.3, np.float32), np.zeros(4, np.float32), 0.1)
    assert v == pytest.approx(0.3, rel=1e-6)


def test_bit_identical_repeats(cuda_ok):
    """Determinism contract (reference tests/test_solver.py:247-257)."""
    mu_w, nu_w, C64 = O.grid_problem(128, 128, 3)
    cfg = lsk.SinkhornConfig(epsilon=0.01)
    r1, p1 = lsk.solve(lsk.CostMatrix(values=C64), dist(mu_w), dist(nu_w), cfg)
    r2, p2 = lsk.solve(lsk.CostMatrix(values=C64), dist(mu_w), dist(nu_w), cfg)
    assert r1.iterations == r2.iterations and r1.error_trace == r2.error_trace
    assert r1.transport_cost == r2.transport_cost
    np.testing.assert_array_equal(p1.alpha, p2.alpha)
    np.testing.assert_array_equal(p1.beta, p2.beta)


def test_transpose_flag_is_bit_neutral(cuda_ok):
    mu_w, nu_w, C64 = O.grid_problem(96, 96, 4)
    r1, p1 = lsk.solve(lsk.CostMatrix(values=C64), dist(mu_w), dist(nu_w), lsk.SinkhornConfig(epsilon=0.01))
    r2, p2 = lsk.solve(lsk.CostMatrix(values=C64), dist(mu_w), dist(nu_w),
                       lsk.SinkhornConfig(epsilon=0.01, transpose_for_beta=True))
    assert r1.transport_cost == r2.transport_cost
    np.testing.assert_array_equal(p1.alpha, p2.alpha)


def test_live_oracle_ragged(cuda_ok):
    """Fresh ragged shapes (n < #SMs, m % 4 != 0, m > n) vs the oracle run now."""
    for (n, m, eps, seed) in [(7, 3, 0.2, 1), (150, 9, 0.05, 2), (149, 2047, 0.02, 3), (513, 4095, 0.01, 4)]:
        C64, mu_w, nu_w, _, _ = O.random_problem(n, m, seed)
        K = 43
        r = O.solve(C64, mu_w, nu_w, eps, tol=1e-30, max_iter=K, check=10)
        rep, pot = lsk.solve(lsk.CostMatrix(values=C64), dist(mu_w), dist(nu_w),
                             lsk.SinkhornConfig(epsilon=eps, tolerance=1e-30, max_iterations=K))
        assert rep.iterations == K and [k for k, _ in rep.error_trace] == [10, 20, 30, 40, 43]
        assert rel_max(pot.alpha, r["alpha"]) <= RTOL and rel_max(pot.beta, r["beta"]) <= RTOL
        assert abs(rep.transport_cost - r["cost"]) <= RTOL * abs(r["cost"])


def test_device_tensor_cost_and_outputs(cuda_ok):
    import torch

    mu_w, nu_w, C64 = O.grid_problem(200, 300, 1)
    Ct = torch.from_numpy(C64).to("cuda", torch.float32)
    cfg = lsk.SinkhornConfig(epsilon=0.02, max_iterations=50, tolerance=1e-30)
    r1, p1 = lsk.solve(lsk.CostMatrix(values=Ct), dist(mu_w), dist(nu_w), cfg, return_device=True)
    r2, p2 = lsk.solve(lsk.CostMatrix(values=C64), dist(mu_w), dist(nu_w), cfg)
    assert p1.alpha.is_cuda
    np.testing.assert_array_equal(p1.alpha.cpu().numpy(), p2.alpha)


def test_dense_wide_loop_path(cuda_ok):
    """m > 8192: the multi-kernel dense loop, same semantics (trace, extra check
    at a cap off the checkpoints, early stop) against the oracle."""
    for (n, m, eps, K, tol, seed) in [(300, 9000, 0.02, 25, 1e-30, 7), (129, 8200, 0.2, 500, 1e-4, 8)]:
        C64, mu_w, nu_w, _, _ = O.random_problem(n, m, seed)
        r = O.solve(C64, mu_w, nu_w, eps, tol=tol, max_iter=K, check=10)
        rep, pot = lsk.solve(lsk.CostMatrix(values=C64), dist(mu_w), dist(nu_w),
                             lsk.SinkhornConfig(epsilon=eps, tolerance=tol, max_iterations=K))
        assert rep.status == r["status"] and rep.iterations == r["iterations"]
        assert [k for k, _ in rep.error_trace] == [int(k) for k, _ in r["trace"]]
        assert rel_max(pot.alpha, r["alpha"]) <= RTOL and rel_max(pot.beta, r["beta"]) <= RTOL
        assert abs(rep.transport_cost - r["cost"]) <= RTOL * abs(r["cost"])


def test_dense_wide_loop_uniform(cuda_ok):
    """m > 8192 with uniform targets: the loop's uniform row kernels (log nu read
    once) and the checkpoint terms fused into the stale row pass, against the
    oracle; and the uniform-flag contract there (a non-uniform log nu ends the
    solve as numerical_failure after 0 iterations)."""
    import torch

    from paper_2605_00837_b200 import solver as S

    rng = np.random.default_rng(11)
    n, m = 200, 9000
    X, Y = rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (m, 2))
    C64 = O.sq_euclidean_cost(X, Y)
    mu_w = rng.uniform(0.5, 1.5, n)
    mu_w /= mu_w.sum()
    nu_w = np.full(m, 1.0 / m)
    for K, tol in ((43, 1e-30), (400, 1e-4)):
        r = O.solve(C64, mu_w, nu_w, 0.02, tol=tol, max_iter=K, check=10)
        rep, pot = lsk.solve(lsk.CostMatrix(values=C64), dist(mu_w), lsk.make_distribution(np.ones(m)),
                             lsk.SinkhornConfig(epsilon=0.02, tolerance=tol, max_iterations=K))
        assert rep.status == r["status"] and rep.iterations == r["iterations"]
        assert [k for k, _ in rep.error_trace] == [int(k) for k, _ in r["trace"]]
        assert rel_max(pot.alpha, r["alpha"]) <= RTOL and rel_max(pot.beta, r["beta"]) <= RTOL
        assert abs(rep.transport_cost - r["cost"]) <= RTOL * abs(r["cost"])
    C = lsk.squared_euclidean_cost(X, Y)
    cfg = lsk.SinkhornConfig(epsilon=0.02, tolerance=1e-30, max_iterations=20)
    mu = lsk.make_distribution(mu_w)
    bad_nu = lsk.make_distribution(rng.uniform(0.5, 1.5, m))
    r, _ = S._launch_solve(torch, C, S._dev_f32(torch, mu.log_weights), S._dev_f32(torch, bad_nu.log_weights),
                           S._dev_f32(torch, mu.weights), cfg, uniform_nu=True)
    res = r.res.cpu().numpy()
    assert res[0] == 2 and res[1] == 0


def test_argument_build_bitwise(cuda_ok):
    """The packed argument builder reproduces numpy's separately rounded fp32
    ops bit for bit (solver.py:77-79; an FMA here breaks eps=1e-4)."""
    import torch

    from paper_2605_00837_b200 import _lib

    rng = np.random.default_rng(0)
    k = 1 << 20
    for eps in (1e-2, 1e-3, 1e-4):
        a = (rng.uniform(-1, 1, k) * 1e-3).astype(np.float32)
        c = rng.uniform(0, 2, k).astype(np.float32)
        l = np.full(k, -np.log(8192.0), dtype=np.float32) + rng.uniform(-1, 1, k).astype(np.float32)
        inv = np.float32(1.0) / np.float32(eps)
        want = ((a - c) * inv) + l  # numpy fp32: three separately rounded ops
        dev = [torch.from_numpy(x).cuda() for x in (a, c, l)]
        out = torch.empty(k, dtype=torch.float32, device="cuda")
        _lib.call("lsk_debug_arg3_f32", dev[0].data_ptr(), dev[1].data_ptr(), eps, dev[2].data_ptr(),
                  out.data_ptr(), k, torch.cuda.current_stream().cuda_stream)
        np.testing.assert_array_equal(out.cpu().numpy(), want)


def test_uniform_nu_flag_bitwise_and_contract(cuda_ok):
    """LSK_FLAG_UNIFORM_NU (broadcast log nu) is bit-identical to the general
    kernel on uniform targets (both run 8 warps per CTA with the same column
    ownership), including padded columns (m % 4 != 0).
    A caller that sets the flag for non-uniform targets gets status 2 after 0
    iterations."""
    import torch

    from paper_2605_00837_b200 import solver as S

    rng = np.random.default_rng(12)
    for n, m in ((300, 1021), (200, 8190), (64, 3000), (500, 777)):
        X, Y = rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (m, 2))
        C = lsk.squared_euclidean_cost(X, Y)
        mu = lsk.make_distribution(rng.uniform(0.5, 1.5, n))
        nu = lsk.make_distribution(np.ones(m))
        cfg = lsk.SinkhornConfig(epsilon=0.01, tolerance=1e-30, max_iterations=60, check_interval=7)
        lm, ln, w = S._dev_f32(torch, mu.log_weights), S._dev_f32(torch, nu.log_weights), S._dev_f32(torch, mu.weights)
        out = []
        for uni in (False, True):  # the grid kernels (the single-cluster one: tests/test_gpu_cluster.py)
            r, _ = S._launch_solve(torch, C, lm, ln, w, cfg, uniform_nu=uni, mult=False, cluster=False)
            torch.cuda.synchronize()
            out.append((r.f.cpu().numpy(), r.g.cpu().numpy(), r.res.cpu().numpy(), r.resf.cpu().numpy()))
        for a, b in zip(out[0], out[1]):
            np.testing.assert_array_equal(a, b)
    nu_bad = lsk.make_distribution(rng.uniform(0.5, 1.5, m))
    r, _ = S._launch_solve(torch, C, lm, S._dev_f32(torch, nu_bad.log_weights), w, cfg, uniform_nu=True)
    res = r.res.cpu().numpy()
    assert res[0] == 2 and res[1] == 0


@pytest.mark.parametrize("n,m,eps", [(8192, 8192, 1e-3), (1024, 1024, 1.5e-3), (4096, 2048, 2e-3)])
def test_multiplicative_column_update_close_to_direct(cuda_ok, n, m, eps):
    """The multiplicative column update (uniform nu, n*m >= 2^20, 1e-3 <= eps <= 2e-3) against the
    direct g-side arithmetic on the same problem: potentials within the fp32 parity
    tolerance, same status and iteration count, cost to 1e-6."""
    import torch

    from paper_2605_00837_b200 import solver as S

    rng = np.random.default_rng(5)
    X, Y = rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (m, 2))
    C = lsk.squared_euclidean_cost(X, Y)
    mu, nu = lsk.make_distribution(np.ones(n)), lsk.make_distribution(np.ones(m))
    cfg = lsk.SinkhornConfig(epsilon=eps, tolerance=1e-30, max_iterations=300)
    lm, ln, w = S._dev_f32(torch, mu.log_weights), S._dev_f32(torch, nu.log_weights), S._dev_f32(torch, mu.weights)
    out = []
    for mult in (False, True):  # grid kernels; the single-cluster kernel: tests/test_gpu_cluster.py
        r, _ = S._launch_solve(torch, C, lm, ln, w, cfg, uniform_nu=True, mult=mult, cluster=False)
        torch.cuda.synchronize()
        out.append((r.f.cpu().numpy(), r.g.cpu().numpy(), r.res.cpu().numpy(), r.resf.cpu().numpy()))
    (f0, g0, r0, c0), (f1, g1, r1, c1) = out
    assert r0[0] == r1[0] and r0[1] == r1[1]
    assert rel_max(f1, f0) <= 1e-5 and rel_max(g1, g0) <= 1e-5, (rel_max(f1, f0), rel_max(g1, g0))
    assert abs(c1[1] - c0[1]) <= 1e-6 * abs(c0[1])


@pytest.mark.parametrize("n,m,eps", [(1, 8192, 1e-3), (149, 4097, 2e-3), (5000, 8191, 1e-3), (20000, 6000, 5e-3),
                                     (300, 8192, 1e-4)])
def test_uniform_kernel_shapes_vs_general(cuda_ok, n, m, eps):
    """The uniform-target kernel (8 warps x 32 columns beyond m = 4096, multiplicative column
    update where it applies) against the general kernel on awkward shapes: one row, one or two
    rows per CTA, heavy column padding, hundreds of rows per CTA, and eps below the
    multiplicative gate."""
    import torch

    from paper_2605_00837_b200 import solver as S

    rng = np.random.default_rng(n + m)
    X, Y = rng.uniform(0, 1, (n, 2)), rng.uniform(0, 1, (m, 2))
    C = lsk.squared_euclidean_cost(X, Y)
    mu, nu = lsk.make_distribution(rng.uniform(0.5, 1.5, n)), lsk.make_distribution(np.ones(m))
    cfg = lsk.SinkhornConfig(epsilon=eps, tolerance=1e-30, max_iterations=40, check_interval=10)
    lm, ln, w = S._dev_f32(torch, mu.log_weights), S._dev_f32(torch, nu.log_weights), S._dev_f32(torch, mu.weights)
    out = []
    for uni in (False, True):
        r, _ = S._launch_solve(torch, C, lm, ln, w, cfg, uniform_nu=uni)
        torch.cuda.synchronize()
        out.append((r.f.cpu().numpy(), r.g.cpu().numpy(), r.res.cpu().numpy(), r.resf.cpu().numpy()))
    (f0, g0, r0, c0), (f1, g1, r1, c1) = out
    assert r0[0] == r1[0] and r0[1] == r1[1]
    assert np.isfinite(f1).all() and np.isfinite(g1).all()
    assert rel_max(f1, f0) <= 1e-5 and rel_max(g1, g0) <= 1e-5, (rel_max(f1, f0), rel_max(g1, g0))
    assert abs(c1[1] - c0[1]) <= 1e-5 * abs(c0[1])
