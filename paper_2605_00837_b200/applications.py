"""Plan consumers on the B200 path.

Mirrors of the reference's ``applications.py`` consumers of a solve:

* ``barycentric_map(plan, targets)`` (``applications.py:75-97``) on a given
  (materialised) plan;
* ``barycentric_map_points`` / ``match_point_clouds[_with_report]``
  (``applications.py:164-205``) that never materialise the (n, m) plan: the
  weights pi_ij are recomputed on the fly from the potentials inside
  ``lsk_points_consume_f32`` (the only way at n = m = 65536, where the plan
  would be 17 GB).

Precision: the reference pipelines solve in double (``_solve_double``,
``applications.py:100-107``); the B200 path is fp32, so the
mapped points and correspondences follow the fp32 potentials. Ties in the
argmax go to the lowest target index, as ``np.argmax``.
"""

from dataclasses import dataclass

import numpy as np

from . import _lib
from .costs import as_points
from .errors import DimensionMismatch, NonFiniteResult, ZeroRowMass
from .points import _batch_points, _weights, points_scale, solve_points_otf
from .solver import _ptr, _stream_ptr, _torch
from .types import STATUS_NUMERICAL_FAILURE, SinkhornConfig

__all__ = ["Correspondence", "barycentric_map", "barycentric_map_points", "match_point_clouds",
           "match_point_clouds_with_report"]


@dataclass(frozen=True)
class Correspondence:
    """One source-to-target match (reference ``applications.py:53-66``)."""

    source_index: int
    target_index: int
    weight: float


def barycentric_map(plan, targets):
    """``mapped_i = sum_j pi_ij t_j / sum_j pi_ij`` for a materialised plan
    (``applications.py:75-97``) in fp64 (``lsk_barycentric_plan_f64``, target
    coordinates in chunks of up to 4); raises ZeroRowMass for an empty row."""
    torch = _torch()
    T = as_points(targets)
    P = plan.values
    Pt = P if isinstance(P, torch.Tensor) else torch.from_numpy(np.asarray(P))
    Pt = Pt.to("cuda", torch.float64).contiguous()
    if Pt.dim() != 2 or Pt.shape[1] != T.shape[0]:
        raise DimensionMismatch(f"plan has {Pt.shape[1]} columns but {T.shape[0]} targets given")
    n, m, d = Pt.shape[0], Pt.shape[1], T.shape[1]
    out = np.empty((n, d), dtype=np.float64)
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    for k0 in range(0, d, 4):
        dt = min(4, d - k0)
        Td = torch.from_numpy(np.ascontiguousarray(T[:, k0:k0 + dt])).to("cuda")
        mapped = torch.empty((n, dt), dtype=torch.float64, device="cuda")
        _lib.call("lsk_barycentric_plan_f64", _ptr(Pt), Pt.stride(0), n, m, _ptr(Td), dt, _ptr(mapped), _ptr(flags),
                  _stream_ptr(torch))
        out[:, k0:k0 + dt] = mapped.cpu().numpy()
    if int(flags[1].item()):
        raise ZeroRowMass("a transport plan row has zero total mass")
    return out


def _consume(X, Y, pot, eps, normalize, mu=None, nu=None):
    torch = _torch()
    Xb, Yb = _batch_points(X), _batch_points(Y)
    B, n, d = Xb.shape
    m = Yb.shape[1]
    _, lmu = _weights(mu, B, n, "mu")
    _, lnu = _weights(nu, B, m, "nu")
    Xd = torch.from_numpy(Xb).to("cuda")
    Yd = torch.from_numpy(Yb).to("cuda")
    scale = points_scale(Xd, Yd, normalize)  # value_range rule of applications.py:186-188
    f = torch.as_tensor(np.asarray(pot.alpha, np.float32) if not isinstance(pot.alpha, torch.Tensor) else pot.alpha)
    g = torch.as_tensor(np.asarray(pot.beta, np.float32) if not isinstance(pot.beta, torch.Tensor) else pot.beta)
    f = f.to("cuda", torch.float32).reshape(B, n).contiguous()
    g = g.to("cuda", torch.float32).reshape(B, m).contiguous()
    lmu_d = torch.from_numpy(lmu.astype(np.float32)).to("cuda")
    lnu_d = torch.from_numpy(lnu.astype(np.float32)).to("cuda")
    mapped = torch.empty((B, n, d), dtype=torch.float32, device="cuda")
    idx = torch.empty((B, n), dtype=torch.int32, device="cuda")
    wt = torch.empty((B, n), dtype=torch.float32, device="cuda")
    zero = torch.zeros(1, dtype=torch.int32, device="cuda")
    wsb = _lib.load().lsk_points_consume_workspace_bytes(B, n, m)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.call("lsk_points_consume_f32", _ptr(Xd), _ptr(Yd), B, n, m, d, _ptr(scale), _ptr(f), _ptr(g), _ptr(lmu_d),
              _ptr(lnu_d), float(eps), _ptr(mapped), _ptr(idx), _ptr(wt), _ptr(zero), _ptr(ws), wsb,
              _stream_ptr(torch))
    if int(zero.item()):
        raise ZeroRowMass("a transport plan row has zero total mass")
    return mapped.cpu().numpy()[0], idx.cpu().numpy()[0], wt.cpu().numpy()[0]


def barycentric_map_points(X, Y, potentials, eps, normalize="none", mu=None, nu=None):
    """Barycentric map of X onto Y under the plan of ``potentials`` (from
    ``solve_points_otf`` / ``solve`` on the same cost), without the plan."""
    return _consume(X, Y, potentials, eps, normalize, mu, nu)[0]


def match_point_clouds_with_report(X, Y, eps, config=None):
    """``applications.match_point_clouds_with_report`` (``applications.py:177-205``):
    uniform weights, cost rescaled by its max, one solve, then per source row
    the argmax plan entry (lowest target index on ties) with its mass --
    computed on the fly, never materialising the plan."""
    X = as_points(X)
    Y = as_points(Y)
    if X.shape[1] != Y.shape[1]:
        raise DimensionMismatch(f"point dimensions differ: {X.shape[1]} vs {Y.shape[1]}")
    cfg = config or SinkhornConfig(epsilon=eps)
    if X.shape[1] > 3:  # beyond the on-the-fly kernels (d <= 3): the dense path and its plan
        from .costs import squared_euclidean_cost
        from .solver import materialize_plan, solve
        from .types import make_distribution

        cost = squared_euclidean_cost(X, Y, normalize="max")
        mu, nu = make_distribution(np.ones(X.shape[0])), make_distribution(np.ones(Y.shape[0]))
        report, pot = solve(cost, mu, nu, cfg)
        if report.status == STATUS_NUMERICAL_FAILURE:
            raise NonFiniteResult(f"solver reported numerical_failure at eps={eps}")
        P = np.asarray(materialize_plan(cost, mu, nu, pot.alpha, pot.beta, cfg.epsilon).values)
        idx = P.argmax(axis=1)
        wt = P[np.arange(P.shape[0]), idx]
    else:
        report, pot = solve_points_otf(X, Y, None, None, cfg, normalize="max")
        if report.status == STATUS_NUMERICAL_FAILURE:
            raise NonFiniteResult(f"solver reported numerical_failure at eps={eps}")
        _, idx, wt = _consume(X, Y, pot, cfg.epsilon, "max")
    pairs = [Correspondence(source_index=i, target_index=int(j), weight=float(w))
             for i, (j, w) in enumerate(zip(idx, wt))]
    return pairs, report


def match_point_clouds(X, Y, eps, config=None):
    """Correspondences only (``applications.py:164-174``)."""
    return match_point_clouds_with_report(X, Y, eps, config)[0]
