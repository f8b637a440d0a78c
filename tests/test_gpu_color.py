"""Colour-transfer pipeline against the reference.

Golden fixtures (tests/golden/make_golden_color.py) hold the reference
``color_transfer_with_report`` outputs for the same images, sample counts,
eps and seeds; the properties below are the reference's own
``tests/test_applications.py::TestColorTransfer`` checks run on this path.
"""

import numpy as np
import pytest
from conftest import golden, golden_names

import paper_2605_00837_b200 as lsk
from paper_2605_00837_b200 import _lib
from paper_2605_00837_b200 import color as CT

pytestmark = pytest.mark.gpu


def checker(side, seed):
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:side, 0:side]
    base = np.stack([0.25 + 0.5 * (x / max(side - 1, 1)), 0.25 + 0.5 * (y / max(side - 1, 1)),
                     0.5 + 0.3 * np.sin(2 * np.pi * x / max(side, 1))], axis=-1).reshape(-1, 3)
    base += rng.normal(0.0, 0.02, base.shape)
    return CT.make_rgb_image(side, side, base)


@pytest.mark.parametrize("name", golden_names("color_"))
def test_color_transfer_matches_reference(cuda_ok, name):
    G = golden(name)
    w, h = int(G["width"]), int(G["height"])
    src = CT.make_rgb_image(w, h, G["src"])
    tside = int(np.sqrt(G["tgt"].shape[0]))
    tgt = CT.make_rgb_image(tside, tside, G["tgt"])
    out, rep = CT.color_transfer_with_report(src, tgt, int(G["sample_count"]), float(G["eps"]), int(G["seed"]))
    assert rep.status == str(G["status"])
    assert rep.iterations == int(G["iterations"])
    assert abs(rep.final_marginal_error - float(G["err"])) <= 1e-9 + 1e-6 * abs(float(G["err"]))
    assert abs(rep.transport_cost - float(G["cost"])) <= 1e-12 + 1e-9 * abs(float(G["cost"]))
    assert out.pixels.shape == G["out"].shape
    np.testing.assert_allclose(out.pixels, G["out"], rtol=0, atol=1e-10)


def test_recolor_nearest_is_exact(cuda_ok):
    """Bit-exact argmin (ties to the lowest index) against the reference loop's arithmetic."""
    import torch

    rng = np.random.default_rng(5)
    S, N = 300, 5000
    smp = rng.uniform(0, 1, (S, 3))
    smp[17] = smp[3]  # duplicate sample: ties must resolve to index 3
    pix = np.vstack([rng.uniform(0, 1, (N - 10, 3)), np.repeat(smp[3:4], 10, axis=0)])
    mapped = rng.uniform(-0.2, 1.2, (S, 3))
    d = pix[:, None, :] - smp[None, :, :]
    want = np.argmin((d * d).sum(axis=2), axis=1)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda")
    P, Sm, M = dev(pix), dev(smp), dev(mapped)
    out = torch.empty_like(P)
    near = torch.empty(N, dtype=torch.int32, device="cuda")
    _lib.call("lsk_recolor_nearest_f64", P.data_ptr(), N, Sm.data_ptr(), S, M.data_ptr(), out.data_ptr(),
              near.data_ptr(), None)
    got = near.cpu().numpy()
    np.testing.assert_array_equal(got, want)
    assert (got[-10:] == 3).all()
    np.testing.assert_array_equal(out.cpu().numpy(), np.clip(mapped[want], 0.0, 1.0))


def test_barycentric_points_vs_plan(cuda_ok):
    """On-the-fly fp64 barycentric map == materialize_plan + barycentric_map in fp64."""
    import torch

    rng = np.random.default_rng(8)
    n, m, eps = 200, 333, 0.03
    X, Y = rng.uniform(0, 1, (n, 3)), rng.uniform(0, 1, (m, 3))
    f, g = rng.normal(0, 0.01, n), rng.normal(0, 0.01, m)
    lmu, lnu = np.full(n, -np.log(n)), np.full(m, -np.log(m))
    C = ((X[:, None, :] - Y[None, :, :]) ** 2).sum(axis=2)
    Z = f[:, None] + g[None, :]
    Z -= C
    Z *= 1.0 / eps
    Z += lmu[:, None]
    Z += lnu[None, :]
    P = np.exp(Z)
    want = (P[:, :, None] * Y[None, :, :]).sum(axis=1) / P.sum(axis=1)[:, None]
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")
    out = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    Xd, Yd, LM, LN, F, Gd = dev(X), dev(Y), dev(lmu), dev(lnu), dev(f), dev(g)  # keep alive over the call
    _lib.call("lsk_barycentric_points_f64", Xd.data_ptr(), Yd.data_ptr(), Yd.data_ptr(), n, m, 3, 3, 0.0,
              LM.data_ptr(), LN.data_ptr(), F.data_ptr(), Gd.data_ptr(), eps, out.data_ptr(), flags.data_ptr(), None)
    torch.cuda.synchronize()
    assert flags.cpu().numpy().tolist() == [0, 0]
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=1e-12, atol=1e-14)


def test_build_cost_f64_bit_exact(cuda_ok):
    import torch

    rng = np.random.default_rng(2)
    X, Y = rng.uniform(-3, 3, (70, 3)), rng.uniform(-3, 3, (91, 3))
    want = ((X[:, None, :] - Y[None, :, :]) ** 2).sum(axis=2)
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    C = torch.empty((70, 91), dtype=torch.float64, device="cuda")
    _lib.call("lsk_build_cost_f64", Xd.data_ptr(), Yd.data_ptr(), 70, 91, 3, 0, C.data_ptr(), 91, None, None, 0, None)
    np.testing.assert_array_equal(C.cpu().numpy(), want)
    ws = torch.empty(_lib.load().lsk_build_cost_workspace_bytes(), dtype=torch.uint8, device="cuda")
    cmax = torch.zeros(1, dtype=torch.float64, device="cuda")
    _lib.call("lsk_build_cost_f64", Xd.data_ptr(), Yd.data_ptr(), 70, 91, 3, 1, C.data_ptr(), 91, cmax.data_ptr(),
              ws.data_ptr(), ws.numel(), None)
    assert float(cmax.item()) == want.max()
    np.testing.assert_array_equal(C.cpu().numpy(), want / want.max())


# ---- the reference's TestColorTransfer properties, on this path
def test_self_transfer_close_to_identity(cuda_ok):
    image = checker(32, seed=0)
    out = lsk.color_transfer(image, image, sample_count=256, eps=0.01, seed=0)
    close = (np.abs(out.pixels - image.pixels) <= 0.1).all(axis=1)
    assert close.mean() >= 0.95


def test_output_within_target_sample_range(cuda_ok):
    source, target = checker(16, seed=1), checker(16, seed=2)
    out = lsk.color_transfer(source, target, sample_count=64, eps=0.05, seed=3)
    assert (out.pixels >= target.pixels.min(axis=0) - 1e-9).all()
    assert (out.pixels <= target.pixels.max(axis=0) + 1e-9).all()


def test_gray_source_gives_constant_output(cuda_ok):
    gray = CT.make_rgb_image(8, 8, np.full((64, 3), 0.5))
    out = lsk.color_transfer(gray, checker(8, seed=4), sample_count=16, eps=0.05, seed=5)
    assert np.abs(out.pixels - out.pixels[0]).max() <= 1e-9


def test_seeded_determinism(cuda_ok):
    source, target = checker(12, seed=9), checker(12, seed=10)
    a = lsk.color_transfer(source, target, sample_count=48, eps=0.05, seed=11)
    b = lsk.color_transfer(source, target, sample_count=48, eps=0.05, seed=11)
    np.testing.assert_array_equal(a.pixels, b.pixels)


def test_large_image(cuda_ok):
    """A 512x512 image with 2048 samples: the recolour is the dominant kernel."""
    src, tgt = checker(512, seed=31), checker(256, seed=32)
    out, rep = CT.color_transfer_with_report(src, tgt, 2048, 0.02, 1)
    assert rep.status == "converged"
    assert out.pixels.shape == src.pixels.shape
    assert (out.pixels >= 0).all() and (out.pixels <= 1).all()
