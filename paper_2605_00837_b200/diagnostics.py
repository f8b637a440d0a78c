"""Plan diagnostics of the reference (``solver.py:461-519``) on the GPU:
``kkt_residual`` (``lsk_kkt_residual``), ``regularized_objective``
(``lsk_regularized_objective_f64``) and the scalar ``contraction_rate_bound``.
Dtype rules as the reference: the KKT residual runs in the plan's precision
(float32 / float64, else float64); the objective always in float64.
"""

import numpy as np

from . import _lib
from .solver import _ptr, _stream_ptr, _torch

__all__ = ["kkt_residual", "regularized_objective", "contraction_rate_bound"]


def _dev(torch, a, dt):
    if hasattr(a, "device_f64"):  # costs.SquaredEuclideanValues
        return a.device_f64().to(dt)
    if isinstance(a, torch.Tensor):
        return a.to("cuda", dt).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a))).to("cuda", dt)


def kkt_residual(cost, mu, nu, plan, alpha, beta, eps):
    """max over P_ij >= tiny of |C_ij + eps ln(P_ij / (mu_i nu_j)) - alpha_i - beta_j|."""
    torch = _torch()
    P = plan.values
    pdt = P.dtype if not isinstance(P, torch.Tensor) else np.dtype(str(P.dtype).replace("torch.", ""))
    dt = np.dtype(pdt) if np.dtype(pdt) in (np.float32, np.float64) else np.dtype(np.float64)
    tdt = torch.float32 if dt == np.float32 else torch.float64
    Pd = _dev(torch, P, tdt)
    n, m = Pd.shape
    Cd = _dev(torch, cost.values, tdt)[:, :m].contiguous()
    a, b = _dev(torch, alpha, tdt), _dev(torch, beta, tdt)
    w_mu, w_nu = _dev(torch, mu.weights, tdt), _dev(torch, nu.weights, tdt)
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    cnt = torch.zeros(2, dtype=torch.int32, device="cuda")
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    _lib.call("lsk_kkt_residual", _ptr(Cd), _ptr(Pd), m, n, m, _ptr(w_mu), _ptr(w_nu), _ptr(a), _ptr(b),
              float(dt.type(eps)), int(dt == np.float64), _ptr(out), _ptr(cnt), _ptr(ws), 16, _stream_ptr(torch))
    c = cnt.cpu().numpy()
    if c[0] == 0:
        return 0.0
    if c[1]:
        return float("nan")
    return float(dt.type(out.item()))


def regularized_objective(cost, mu, nu, plan, eps):
    """<C, P> + eps * KL(P | mu x nu), KL = sum P (ln(P / (mu nu)) - 1) + 1, in float64."""
    torch = _torch()
    Pd = _dev(torch, plan.values, torch.float64)
    n, m = Pd.shape
    Cd = _dev(torch, cost.values, torch.float64)[:, :m].contiguous()
    w_mu, w_nu = _dev(torch, mu.weights, torch.float64), _dev(torch, nu.weights, torch.float64)
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws = torch.empty(16 * n, dtype=torch.uint8, device="cuda")
    _lib.call("lsk_regularized_objective_f64", _ptr(Cd), _ptr(Pd), m, n, m, _ptr(w_mu), _ptr(w_nu), float(eps),
              _ptr(out), _ptr(ws), 16 * n, _stream_ptr(torch))
    return float(out.item())


def contraction_rate_bound(R, eps):
    """(exp(-2R/eps), tanh(R/(4 eps))^2): the published per-iteration contraction
    factors for cost radius R (scalar host arithmetic)."""
    if R < 0:
        raise ValueError("R must be >= 0")
    if not (eps > 0):
        raise ValueError("eps must be > 0")
    return float(np.exp(-2.0 * R / eps)), float(np.tanh(R / (4.0 * eps)) ** 2)
