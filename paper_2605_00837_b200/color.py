"""Colour transfer on the B200 path.

Mirrors the reference pipeline ``color_transfer[_with_report]``
(``applications.py:110-161``) and its value types (``RgbImage``,
``make_rgb_image``, ``applications.py:37-72``):

1. seeded uniform sampling of ``sample_count`` pixels from each image
   without replacement -- the same ``numpy`` PCG64 draws as the reference,
   so the samples are identical;
2. fp64 squared-Euclidean cost of the samples (``lsk_build_cost_f64``) and a
   double-precision solve (``solver64``; the reference pipeline always solves
   in double, ``applications.py:100-107``);
3. the barycentric map of the source samples onto the target samples with
   the plan weights recomputed on the fly (``lsk_barycentric_points_f64``:
   materialize_plan + barycentric_map without the plan);
4. every source pixel recoloured by the mapped colour of its nearest source
   sample (``lsk_recolor_nearest_f64``; bit-exact argmin, ties to the lowest
   sample index, channels clamped to [0, 1]).

All arithmetic after the sampling is in CUDA kernels; there is no CPU path.
"""

from dataclasses import dataclass

import numpy as np

from . import _lib
from . import solver64
from .errors import DimensionMismatch, NonFiniteResult, ZeroRowMass
from .solver import _ptr, _stream_ptr, _torch
from .types import STATUS_NUMERICAL_FAILURE, SinkhornConfig, make_distribution

__all__ = ["RgbImage", "make_rgb_image", "color_transfer", "color_transfer_with_report", "generate_rigid_pair"]


@dataclass(frozen=True, eq=False)
class RgbImage:
    """Row-major RGB pixels (height * width, 3) in [0, 1] (``applications.py:37-50``)."""

    width: int
    height: int
    pixels: np.ndarray


def make_rgb_image(width, height, pixels):
    """An RgbImage with channels clamped into [0, 1]; a pixel array that does
    not hold ``width * height`` RGB triples raises ValueError."""
    p = np.asarray(pixels, dtype=np.float64).reshape(height * width, 3)
    return RgbImage(width=width, height=height, pixels=np.clip(p, 0.0, 1.0))


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")


def color_transfer_with_report(source, target, sample_count, eps, seed):
    """Recoloured source image and the SolveReport of the sample solve."""
    n_src = source.pixels.shape[0]
    n_tgt = target.pixels.shape[0]
    if not (1 <= sample_count <= min(n_src, n_tgt)):
        raise ValueError("sample_count must be >= 1 and <= both images' pixel counts")
    rng = np.random.Generator(np.random.PCG64(seed))
    src_idx = rng.choice(n_src, size=sample_count, replace=False)
    tgt_idx = rng.choice(n_tgt, size=sample_count, replace=False)
    src_samples = np.ascontiguousarray(source.pixels[src_idx], dtype=np.float64)
    tgt_samples = np.ascontiguousarray(target.pixels[tgt_idx], dtype=np.float64)

    torch = _torch()
    st = _stream_ptr(torch)
    S = sample_count
    Xs, Ys = _dev(torch, src_samples), _dev(torch, tgt_samples)
    C = torch.empty((S, S), dtype=torch.float64, device="cuda")
    _lib.call("lsk_build_cost_f64", _ptr(Xs), _ptr(Ys), S, S, 3, 0, _ptr(C), S, None, None, 0, st)

    uniform = make_distribution(np.ones(S))
    report, pot = solver64.solve(C, uniform, uniform, SinkhornConfig(epsilon=eps, precision="double"),
                                 return_device=True)
    if report.status == STATUS_NUMERICAL_FAILURE:
        raise NonFiniteResult(f"solver reported numerical_failure at eps={eps}")

    lw = _dev(torch, uniform.log_weights)
    mapped = torch.empty((S, 3), dtype=torch.float64, device="cuda")
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    _lib.call("lsk_barycentric_points_f64", _ptr(Xs), _ptr(Ys), _ptr(Ys), S, S, 3, 3, 0.0, _ptr(lw), _ptr(lw),
              _ptr(pot.alpha), _ptr(pot.beta), float(eps), _ptr(mapped), _ptr(flags), st)
    fl = flags.cpu().numpy()
    if fl[0]:
        raise NonFiniteResult("transport plan contains non-finite entries")
    if fl[1]:
        raise ZeroRowMass("a transport plan row has zero total mass")

    px = _dev(torch, source.pixels)
    out = torch.empty_like(px)
    _lib.call("lsk_recolor_nearest_f64", _ptr(px), n_src, _ptr(Xs), S, _ptr(mapped), _ptr(out), None, st)
    image = RgbImage(width=source.width, height=source.height, pixels=out.cpu().numpy())
    return image, report


def color_transfer(source, target, sample_count, eps, seed):
    """Transfer the target's palette onto the source (``applications.py:110-124``)."""
    return color_transfer_with_report(source, target, sample_count, eps, seed)[0]


def _rotation(dimension, angle):
    c, s = np.cos(angle), np.sin(angle)
    if dimension == 2:
        return np.array([[c, -s], [s, c]])
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def generate_rigid_pair(n, dimension, rotation_angle, translation, noise_sigma, seed):
    """Seeded test-data generator of the matching pipeline (``applications.py:217-251``):
    X uniform in the unit cube, Y = rotate(X) + t + N(0, sigma^2), shuffled by a
    seeded permutation; returns (X, shuffled Y, perm) with X[i] <-> Y[perm[i]].
    Host-side data generation (the same PCG64 draws as the reference)."""
    if dimension not in (2, 3):
        raise ValueError("dimension must be 2 or 3")
    if noise_sigma < 0:
        raise ValueError("noise_sigma must be >= 0")
    t = np.asarray(translation, dtype=np.float64).reshape(-1)
    if t.shape[0] != dimension:
        raise DimensionMismatch(f"translation has {t.shape[0]} components, expected {dimension}")
    rng = np.random.Generator(np.random.PCG64(seed))
    X = rng.uniform(0.0, 1.0, (n, dimension))
    Y = X @ _rotation(dimension, rotation_angle).T + t
    Y = Y + rng.normal(0.0, noise_sigma, (n, dimension))
    perm = rng.permutation(n)
    out = np.empty_like(Y)
    out[perm] = Y
    return X, out, perm
