"""Cost construction on the device.

``squared_euclidean_cost`` is the reference's ``costs.squared_euclidean_cost``
(``costs.py:36-50``) with the same return type: a ``CostMatrix`` whose
``values`` behave as the (n, m) float64 matrix ``sum_k (x_ik - y_jk)^2`` --
``values.max()`` / ``.min()`` exact, ``value_range`` cached, ``values / s``
the exact fp64 quotient, ``np.asarray(values)`` the host fp64 matrix -- but
held as the two point clouds on the device (``SquaredEuclideanValues``). So the
reference's own composition runs unchanged::

    cost = squared_euclidean_cost(X, Y)
    if cost.value_range > 0:                                   # applications.py:186-188
        cost = CostMatrix(values=np.ascontiguousarray(cost.values / cost.values.max()))
    report, pot = solve(cost, mu, nu, config)

``solve`` on the un-materialised form builds ``fp32(C64 / s)`` directly on the
device (``lsk_build_cost_div_f32``: the same fp64 direct sum in coordinate
order, one fp64 division, one fp32 rounding, so bit-identical to the
reference's cast). ``np.ascontiguousarray`` (as the reference
pipelines call it) materialises the host fp64 matrix, exactly but at host
speed; ``normalize="max"`` (or passing ``cost.values / cost.values.max()``
straight to ``CostMatrix``) keeps it on the device.
"""

import ctypes

import numpy as np

from . import _lib
from .errors import DimensionMismatch, EmptyInput, NonFiniteInput
from .solver import _ptr, _stream_ptr, _torch, solve
from .types import CostMatrix, DeviceCostMatrix

__all__ = ["as_points", "squared_euclidean_cost", "solve_points", "SquaredEuclideanValues"]


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


class SquaredEuclideanValues:
    """fp64-semantics view of ``sum_k (x_ik - y_jk)^2 / s1 / s2 ...`` (never
    materialised unless converted to a numpy array)."""

    __array_priority__ = 1000
    dtype = np.dtype(np.float64)
    ndim = 2

    def __init__(self, Xd, Yd, n, m, d, cmax, cmin, divisors=()):
        self._X, self._Y = Xd, Yd
        self._n, self._m, self._d = n, m, d
        self._cmax, self._cmin = float(cmax), float(cmin)
        self._div = tuple(divisors)
        self._dev32 = None

    @property
    def shape(self):
        return (self._n, self._m)

    @property
    def size(self):
        return self._n * self._m

    def _scaled(self, v):
        for s in self._div:  # Python floats: IEEE fp64 division, as numpy's
            v = v / s
        return np.float64(v)

    def max(self):
        return self._scaled(self._cmax)

    def min(self):
        return self._scaled(self._cmin)

    def __truediv__(self, s):
        s = float(s)
        return SquaredEuclideanValues(self._X, self._Y, self._n, self._m, self._d, self._cmax, self._cmin,
                                      self._div + (s,))

    def device_f64(self):
        """The fp64 matrix on the device (n, m), exactly the reference's values."""
        torch = _torch()
        C = torch.empty((self._n, self._m), dtype=torch.float64, device="cuda")
        wsb = _lib.load().lsk_build_cost_workspace_bytes()
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        _lib.call("lsk_build_cost_f64", _ptr(self._X), _ptr(self._Y), self._n, self._m, self._d, 0, _ptr(C),
                  self._m, None, _ptr(ws), wsb, _stream_ptr(torch))
        for s in self._div:
            # a device tensor divisor: an IEEE division per element (torch turns a
            # Python-scalar divisor into a multiplication by its reciprocal)
            C = torch.div(C, torch.full((1, 1), s, dtype=torch.float64, device="cuda"))
        return C

    def __array__(self, dtype=None, copy=None):
        a = self.device_f64().cpu().numpy()
        return a if dtype is None else a.astype(dtype)

    def device_fp32(self):
        """The kernels' padded fp32 layout (cached): fp32(C64 / s) bit for bit."""
        if self._dev32 is None:
            torch = _torch()
            ldc = (self._m + 3) // 4 * 4
            if len(self._div) <= 1:
                C = torch.zeros((self._n, ldc), dtype=torch.float32, device="cuda")
                _lib.call("lsk_build_cost_div_f32", _ptr(self._X), _ptr(self._Y), self._n, self._m, self._d,
                          self._div[0] if self._div else 0.0, _ptr(C), ldc, _stream_ptr(torch))
            else:
                src = self.device_f64()
                C = torch.empty((self._n, ldc), dtype=torch.float32, device="cuda")
                _lib.call("lsk_cast_cost_f32", _ptr(src), 1, self._m, self._n, self._m, _ptr(C), ldc,
                          _stream_ptr(torch))
            self._dev32 = DeviceCostMatrix(data=C, rows=self._n, cols=self._m, cmax=self._cmax)
        return self._dev32


def squared_euclidean_cost(X, Y, normalize="none"):
    """``costs.squared_euclidean_cost`` (``costs.py:36-50``) -> ``CostMatrix``
    with device-held fp64-semantics values (see module doc).

    ``normalize``: "none" (the reference) or "max": divide by the maximum
    when the range is non-zero, as ``applications.py:186-188``.
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
    wsb = _lib.load().lsk_build_cost_workspace_bytes()
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    rng = (ctypes.c_double * 2)()
    _lib.call("lsk_cost_range_f64", _ptr(Xd), _ptr(Yd), n, m, d, rng, _ptr(ws), wsb, _stream_ptr(torch))
    vals = SquaredEuclideanValues(Xd, Yd, n, m, d, rng[0], rng[1])
    if normalize == "max" and rng[0] - rng[1] > 0:
        vals = vals / vals.max()
    return CostMatrix(values=vals, value_range=float(vals.max() - vals.min()))


def solve_points(X, Y, mu, nu, config, normalize="none", **kw):
    """``solve(squared_euclidean_cost(X, Y) [/ max], mu, nu, config)`` with the
    cost built on the device (fp64-exact, rounded once to fp32)."""
    C = squared_euclidean_cost(X, Y, normalize=normalize)
    return solve(C, mu, nu, config, **kw)
