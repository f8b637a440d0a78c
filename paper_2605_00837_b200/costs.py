"""Cost construction on the device.

``squared_euclidean_cost`` stands in for the reference's
``costs.squared_euclidean_cost`` (``costs.py:36-50``): the same fp64 direct
sum over coordinates in coordinate order, computed by ``lsk_build_cost_f32``
on the GPU and rounded once to the fp32 the solver consumes (solver.py:253),
so the device matrix equals ``fp32(C64)`` bit for bit. With
``normalize="max"`` it applies the point-cloud pipeline's ``C / C.max()``
(``applications.py:186-188``) in fp64 before that rounding.
"""

import numpy as np

from . import _lib
from .errors import DimensionMismatch, EmptyInput, NonFiniteInput
from .solver import _ptr, _stream_ptr, _torch, solve
from .types import DeviceCostMatrix

__all__ = ["as_points", "squared_euclidean_cost", "solve_points"]


def as_points(coords):
    """Validate a point cloud as an (n, d) float64 array (costs.py:18-33)."""
    X = np.asarray(coords, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    if X.ndim != 2:
        raise DimensionMismatch(f"point cloud must be 2-D, got shape {X.shape}")
    if X.size == 0:
        raise EmptyInput("point cloud is empty")
    if not np.isfinite(X).all():
        raise NonFiniteInput("point coordinates must be finite")
    return np.ascontiguousarray(X)


def squared_euclidean_cost(X, Y, normalize="none"):
    """fp32(sum_k (x_ik - y_jk)^2) as a DeviceCostMatrix (see module doc).

    ``normalize``: "none" (reference costs.py) or "max" (divide by the
    maximum when the range is non-zero, as applications.py:186-188).
    ``.cmax`` holds the maximum of the un-normalised fp64 cost.
    """
    if normalize not in ("none", "max"):
        raise ValueError("normalize must be 'none' or 'max'")
    X = as_points(X)
    Y = as_points(Y)
    if X.shape[1] != Y.shape[1]:
        raise DimensionMismatch(f"point dimensions differ: {X.shape[1]} vs {Y.shape[1]}")
    torch = _torch()
    n, m, d = X.shape[0], Y.shape[0], X.shape[1]
    Xd = torch.from_numpy(X).to("cuda")
    Yd = torch.from_numpy(Y).to("cuda")
    ldc = (m + 3) // 4 * 4
    C = torch.zeros((n, ldc), dtype=torch.float32, device="cuda")
    wsb = _lib.load().lsk_build_cost_workspace_bytes()
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    cmax = torch.zeros(1, dtype=torch.float64, device="cuda")
    _lib.call("lsk_build_cost_f32", _ptr(Xd), _ptr(Yd), n, m, d, int(normalize == "max"), _ptr(C), ldc,
              _ptr(cmax), _ptr(ws), wsb, _stream_ptr(torch))
    return DeviceCostMatrix(data=C, rows=n, cols=m, cmax=float(cmax.item()))


def solve_points(X, Y, mu, nu, config, normalize="none", **kw):
    """``solve(squared_euclidean_cost(X, Y) [/ max], mu, nu, config)`` with the
    cost built on the device (fp64-exact, rounded once to fp32)."""
    C = squared_euclidean_cost(X, Y, normalize=normalize)
    return solve(C, mu, nu, config, **kw)
