"""Standard-domain Sinkhorn on the GPU.

``solve_standard_domain(cost, mu, nu, config) -> (SolveReport, u, v)`` mirrors
the reference's deliberately unguarded twin of the log-domain solve
(``solver.py:340-431``): K = exp(-C / eps) materialised once, then
``u = mu / (K v)``, ``v = nu / (K^T u)`` from u = v = 1, with the same
checkpoint logic, trace, final extra check and cost (fp32 with m <= 8192: one
persistent kernel reading K once per iteration, ``csrc/lsk_stdfused.cuh``).
Overflow, underflow and
division by zero propagate and surface as numerical_failure at the next
checkpoint, as in the reference. One C-ABI call (``lsk_solve_standard_f32`` /
``_f64``, ``csrc/lsk_standard.cu``) per solve; precision follows
``config.precision``.
"""

import time

import numpy as np

from . import _lib
from . import solver64 as _s64
from .solver import _check_dims, _ptr, _stream_ptr, _torch, to_device_cost
from .types import _STATUS_BY_CODE, STATUS_NUMERICAL_FAILURE, SolveReport

__all__ = ["solve_standard_domain"]


def solve_standard_domain(cost, mu, nu, config, *, fused=True):
    """(SolveReport, u, v) of the standard-domain iteration (see module doc).

    fp32 problems with m <= 8192 run the one-pass persistent kernel (one read of
    K per iteration); ``fused=False`` forces the two-pass multi-kernel loop."""
    _check_dims(cost, mu, nu)
    torch = _torch()
    t0 = time.perf_counter()
    double = config.precision == "double"
    tdt = torch.float64 if double else torch.float32
    if double:
        C = _s64._cost64(torch, cost)
        Cp, ldc = C, C.stride(0)
    else:
        Cd = to_device_cost(cost)
        Cp, ldc = Cd.data, Cd.ldc
    n, m = mu.size, nu.size
    npdt = np.float64 if double else np.float32
    w_mu = torch.from_numpy(np.ascontiguousarray(mu.weights.astype(npdt))).to("cuda")
    w_nu = torch.from_numpy(np.ascontiguousarray(nu.weights.astype(npdt))).to("cuda")
    K, c = int(config.max_iterations), int(config.check_interval)
    cap = _lib.load().lsk_trace_capacity(K, c)
    wsb = _lib.load().lsk_solve_standard_workspace_bytes(n, m, int(double))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    u = torch.empty(n, dtype=tdt, device="cuda")
    v = torch.empty(m, dtype=tdt, device="cuda")
    ti = torch.zeros(cap, dtype=torch.int32, device="cuda")
    te = torch.zeros(cap, dtype=tdt, device="cuda")
    res = torch.zeros(8, dtype=torch.int32, device="cuda")
    resf = torch.zeros(2, dtype=tdt, device="cuda")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    _lib.call("lsk_solve_standard_f64" if double else "lsk_solve_standard_f32", _ptr(Cp), ldc, n, m, _ptr(w_mu),
              _ptr(w_nu), float(config.epsilon), float(config.tolerance), K, c,
              _lib.LSK_FLAG_COST | (0 if fused else _lib.LSK_FLAG_STD_MULTIKERNEL), _ptr(u), _ptr(v),
              _ptr(ti), _ptr(te), _ptr(res), _ptr(resf), _ptr(ws), wsb, _stream_ptr(torch))
    ev1.record()
    r, rf = res.cpu().numpy(), resf.cpu().numpy()
    nt = int(r[2])
    status = _STATUS_BY_CODE[int(r[0])]
    trace = tuple((int(k), float(e)) for k, e in zip(ti[:nt].cpu().numpy(), te[:nt].cpu().numpy()))
    report = SolveReport(status=status, iterations=int(r[1]), final_marginal_error=float(rf[0]),
                         transport_cost=float(rf[1]) if status != STATUS_NUMERICAL_FAILURE else float("nan"),
                         error_trace=trace, elapsed_seconds=time.perf_counter() - t0,
                         device_seconds=ev0.elapsed_time(ev1) * 1e-3)
    return report, u.cpu().numpy(), v.cpu().numpy()
