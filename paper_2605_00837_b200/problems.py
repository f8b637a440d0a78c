"""Seeded benchmark problems and cost rescaling of the reference
(``costs.py:53-116``), used by the CLI harness. Host-side data preparation:
the same PCG64 draw order as the reference, so a seed gives bit-identical
problems on both sides.
"""

import warnings

import numpy as np

from .errors import DegenerateRange
from .types import CostMatrix, make_distribution

__all__ = ["generate_grid_problem", "normalize_cost"]


def normalize_cost(cost, target_max):
    """Affine rescale to [0, target_max]; a constant matrix becomes zeros
    with a DegenerateRange warning."""
    if not (target_max > 0):
        raise ValueError("target_max must be > 0")
    v = np.asarray(cost.values)
    if cost.value_range == 0:
        warnings.warn("constant cost matrix rescaled to all zeros", DegenerateRange, stacklevel=2)
        return CostMatrix(values=np.zeros_like(v), value_range=0.0)
    return CostMatrix(values=np.ascontiguousarray((v - v.min()) * (target_max / cost.value_range)))


def generate_grid_problem(n, m, seed):
    """(mu, nu, C) on the 1-D grids i/(n-1), j/(m-1): C = squared distance
    divided by its max; weights = seeded Gaussian bump (center U(0.2, 0.8),
    width U(0.05, 0.1), 1e-4 floor) times per-point jitter U(0.5, 1.5), bump
    geometry drawn before the jitter."""
    if n < 1 or m < 1:
        raise ValueError("n and m must be >= 1")
    rng = np.random.Generator(np.random.PCG64(seed))
    c = rng.uniform(0.2, 0.8, 2)
    w = rng.uniform(0.05, 0.1, 2)
    x = np.arange(n) / (n - 1) if n > 1 else np.zeros(1)
    y = np.arange(m) / (m - 1) if m > 1 else np.zeros(1)
    a = np.exp(-0.5 * ((x - c[0]) / w[0]) ** 2) + 1e-4
    a *= rng.uniform(0.5, 1.5, n)
    b = np.exp(-0.5 * ((y - c[1]) / w[1]) ** 2) + 1e-4
    b *= rng.uniform(0.5, 1.5, m)
    C = (x[:, None] - y[None, :]) ** 2
    top = C.max()
    if top > 0:
        C /= top
    return make_distribution(a), make_distribution(b), CostMatrix(values=np.ascontiguousarray(C))
