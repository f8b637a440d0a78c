"""fp64 host side: ``precision="double"`` solves and the half-steps called with
float64 potentials (the dtype rule of reference ``solver.py:60-65``).

Same functions and return types as ``solver.py``; every call is one fp64 C-ABI
entry point (``lsk_*_f64``, ``csrc/lsk_f64.cu``) over an fp64 device copy of C.
"""

import time

import numpy as np

from . import _lib
from .errors import DimensionMismatch, NonFiniteResult
from .types import _STATUS_BY_CODE, STATUS_NUMERICAL_FAILURE, CostMatrix, DualPotentials, SolveReport, TransportPlan


def float_dtype(*arrays):
    """The reference's ``_float_dtype``: the first float32/float64 array decides,
    otherwise float64 (numpy arrays, sequences or torch tensors)."""
    try:
        import torch

        tensor = torch.Tensor
    except Exception:  # pragma: no cover
        torch, tensor = None, ()
    for a in arrays:
        if torch is not None and isinstance(a, tensor):
            if a.dtype == torch.float32:
                return np.dtype(np.float32)
            if a.dtype == torch.float64:
                return np.dtype(np.float64)
            continue
        dt = np.asarray(a).dtype
        if dt in (np.float32, np.float64):
            return np.dtype(dt)
    return np.dtype(np.float64)


def _cost64(torch, cost):
    vals = cost.values if isinstance(cost, CostMatrix) else getattr(cost, "data", cost)
    if hasattr(vals, "device_f64"):  # costs.SquaredEuclideanValues
        return vals.device_f64()
    if isinstance(vals, torch.Tensor):
        t = vals.to("cuda", torch.float64)
        if hasattr(cost, "cols") and t.shape[1] != cost.cols:  # DeviceCostMatrix padding
            t = t[:, : cost.cols]
        return t.contiguous()
    A = np.asarray(vals)
    if A.ndim != 2:
        raise DimensionMismatch("cost matrix must be 2-D")
    return torch.from_numpy(np.ascontiguousarray(A, dtype=np.float64)).to("cuda")


def _v64(torch, x):
    if isinstance(x, torch.Tensor):
        return x.to("cuda", torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x), dtype=np.float64)).to("cuda")


def _s(torch):
    return torch.cuda.current_stream().cuda_stream or None


def solve(cost, mu, nu, config, return_device=False):
    """``solver.solve`` in double precision (reference dt = float64)."""
    import torch

    t0 = time.perf_counter()
    C = _cost64(torch, cost)
    n, m = C.shape
    lmu, lnu, w = _v64(torch, mu.log_weights), _v64(torch, nu.log_weights), _v64(torch, mu.weights)
    K, c = int(config.max_iterations), int(config.check_interval)
    cap = _lib.load().lsk_trace_capacity(K, c)
    wsb = _lib.load().lsk_solve_dense_f64_workspace_bytes(n, m)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    f = torch.empty(n, dtype=torch.float64, device="cuda")
    g = torch.empty(m, dtype=torch.float64, device="cuda")
    ti = torch.zeros(cap, dtype=torch.int32, device="cuda")
    te = torch.zeros(cap, dtype=torch.float64, device="cuda")
    res = torch.zeros(8, dtype=torch.int32, device="cuda")
    resf = torch.zeros(2, dtype=torch.float64, device="cuda")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    _lib.call("lsk_solve_dense_f64", C.data_ptr(), C.stride(0), n, m, lmu.data_ptr(), lnu.data_ptr(), w.data_ptr(),
              float(config.epsilon), float(config.tolerance), K, c, _lib.LSK_FLAG_COST, f.data_ptr(), g.data_ptr(),
              ti.data_ptr(), te.data_ptr(), res.data_ptr(), resf.data_ptr(), ws.data_ptr(), wsb, _s(torch))
    ev1.record()
    r, rf = res.cpu().numpy(), resf.cpu().numpy()
    nt = int(r[2])
    status = _STATUS_BY_CODE[int(r[0])]
    trace = tuple((int(k), float(e)) for k, e in zip(ti[:nt].cpu().numpy(), te[:nt].cpu().numpy()))
    report = SolveReport(status=status, iterations=int(r[1]), final_marginal_error=float(rf[0]),
                         transport_cost=float(rf[1]) if status != STATUS_NUMERICAL_FAILURE else float("nan"),
                         error_trace=trace, elapsed_seconds=time.perf_counter() - t0,
                         device_seconds=ev0.elapsed_time(ev1) * 1e-3)
    if return_device:
        return report, DualPotentials(alpha=f, beta=g)
    return report, DualPotentials(alpha=f.cpu().numpy(), beta=g.cpu().numpy())


def update_alpha(cost, nu, beta, eps):
    import torch

    C = _cost64(torch, cost)
    n, m = C.shape
    b, lnu = _v64(torch, beta), _v64(torch, nu.log_weights)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.call("lsk_update_alpha_f64", C.data_ptr(), C.stride(0), n, m, b.data_ptr(), lnu.data_ptr(), float(eps),
              out.data_ptr(), _s(torch))
    return out.cpu().numpy()


def update_beta(cost, mu, alpha, eps):
    import torch

    C = _cost64(torch, cost)
    n, m = C.shape
    a, lmu = _v64(torch, alpha), _v64(torch, mu.log_weights)
    out = torch.empty(m, dtype=torch.float64, device="cuda")
    wsb = _lib.load().lsk_update_beta_f64_workspace_bytes(n, m)
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
    _lib.call("lsk_update_beta_f64", C.data_ptr(), C.stride(0), n, m, a.data_ptr(), lmu.data_ptr(), float(eps),
              out.data_ptr(), ws.data_ptr(), ws.numel(), _s(torch))
    return out.cpu().numpy()


def marginal_error(cost, mu, nu, alpha, beta, eps):
    import torch

    C = _cost64(torch, cost)
    n, m = C.shape
    w, lmu, lnu = _v64(torch, mu.weights), _v64(torch, mu.log_weights), _v64(torch, nu.log_weights)
    a, b = _v64(torch, alpha), _v64(torch, beta)
    ws = torch.empty(n, dtype=torch.float64, device="cuda")
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.call("lsk_marginal_error_f64", C.data_ptr(), C.stride(0), n, m, w.data_ptr(), lmu.data_ptr(),
              lnu.data_ptr(), a.data_ptr(), b.data_ptr(), float(eps), out.data_ptr(), ws.data_ptr(), n * 8, _s(torch))
    return float(out.item())


def transport_cost(cost, mu, nu, alpha, beta, eps):
    import torch

    C = _cost64(torch, cost)
    n, m = C.shape
    lmu, lnu, a, b = (_v64(torch, x) for x in (mu.log_weights, nu.log_weights, alpha, beta))
    ws = torch.empty(n, dtype=torch.float64, device="cuda")
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.call("lsk_transport_cost_f64", C.data_ptr(), C.stride(0), n, m, lmu.data_ptr(), lnu.data_ptr(),
              a.data_ptr(), b.data_ptr(), float(eps), out.data_ptr(), ws.data_ptr(), n * 8, _s(torch))
    return float(out.item())


def materialize_plan(cost, mu, nu, alpha, beta, eps, return_device=False):
    import torch

    C = _cost64(torch, cost)
    n, m = C.shape
    lmu, lnu, a, b = (_v64(torch, x) for x in (mu.log_weights, nu.log_weights, alpha, beta))
    P = torch.empty((n, m), dtype=torch.float64, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("lsk_materialize_plan_f64", C.data_ptr(), C.stride(0), n, m, lmu.data_ptr(), lnu.data_ptr(),
              a.data_ptr(), b.data_ptr(), float(eps), P.data_ptr(), m, bad.data_ptr(), _s(torch))
    if int(bad.item()) != 0:
        raise NonFiniteResult("transport plan contains non-finite entries")
    return TransportPlan(values=P if return_device else P.cpu().numpy())
