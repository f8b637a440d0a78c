"""Drop-in log-domain Sinkhorn API on the B200 kernels.

Same functions, signatures, return types and error behaviour as the
reference's ``logsinkhorn.solver`` (``/root/reference/pkg/src/logsinkhorn/
solver.py:46-57``): ``solve`` (230-337), ``update_alpha`` (118-140),
``update_beta`` (143-176), ``marginal_error`` (179-206), ``transport_cost``
(209-227) and ``materialize_plan`` (434-458). Each is a thin host shim over
one C-ABI call of ``liblsk.so`` (include/lsk.h); all arithmetic runs in the
sm_100a kernels. Device memory and streams come from PyTorch.

Precision: ``precision="single"`` (the reference's default and the parity
target) runs the fp32 kernels; ``precision="double"`` and float64 potentials
in the half-steps follow the reference's dtype rule (``solver.py:60-65``) and
run the fp64 kernels (``solver64``, ``lsk_*_f64``) with the reference's double
arithmetic -- never a silent change of precision.
"""

import time

import numpy as np

from . import _lib
from . import solver64 as _s64
from .errors import BackendError, DimensionMismatch, NonFiniteResult
from .types import (
    _STATUS_BY_CODE,
    STATUS_NUMERICAL_FAILURE,
    CostMatrix,
    DeviceCostMatrix,
    DualPotentials,
    ReductionPlan,
    SolveReport,
    TransportPlan,
)

__all__ = [
    "solve",
    "update_alpha",
    "update_beta",
    "marginal_error",
    "transport_cost",
    "materialize_plan",
    "to_device_cost",
]


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise BackendError("no CUDA device visible: the B200 solver has no CPU fallback")
    return torch


def _stream_ptr(torch):
    return ctypes_void(torch.cuda.current_stream().cuda_stream)


def ctypes_void(x):
    return int(x) if x else None


def _ptr(t):
    return t.data_ptr()


def _dev_f32(torch, x):
    """1-D fp32 device copy of a host/device vector."""
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x), dtype=np.float32)).to("cuda")


def _is_f64(*arrays):
    """The reference's dtype rule (solver.py:60-65): the first float32/float64
    argument decides, anything else means float64."""
    return _s64.float_dtype(*arrays) == np.float64


def to_device_cost(cost):
    """Return the kernels' layout (DeviceCostMatrix) for a CostMatrix /
    DeviceCostMatrix / 2-D array or tensor. fp64 inputs are rounded to fp32
    once, on the device (solver.py:253)."""
    torch = _torch()
    if isinstance(cost, DeviceCostMatrix):
        return cost
    vals = cost.values if isinstance(cost, CostMatrix) else cost
    if hasattr(vals, "device_fp32"):  # costs.SquaredEuclideanValues: built on the device, never materialised
        return vals.device_fp32()
    if isinstance(vals, np.ndarray):
        if vals.ndim != 2:
            raise DimensionMismatch("cost matrix must be 2-D")
        # host matrix: rounded to fp32 by the library's worker threads while the
        # previous chunk is copied (lsk_h2d_cost_f32), straight into the padded layout
        A = vals if vals.dtype in (np.float64, np.float32) else vals.astype(np.float64)
        A = np.ascontiguousarray(A)
        n, m = A.shape
        ldc = (m + 3) // 4 * 4
        out = torch.empty((n, ldc), dtype=torch.float32, device="cuda")
        _lib.call("lsk_h2d_cost_f32", A.ctypes.data, int(A.dtype == np.float64), m, n, m, _ptr(out), ldc, 0,
                  _stream_ptr(torch))
        return DeviceCostMatrix(data=out, rows=n, cols=m)
    elif isinstance(vals, torch.Tensor):
        if vals.dim() != 2:
            raise DimensionMismatch("cost matrix must be 2-D")
        src = vals if vals.is_cuda else vals.to("cuda", non_blocking=vals.is_pinned())
        if src.stride(1) != 1:
            src = src.contiguous()
    else:
        raise TypeError("cost must be a CostMatrix, DeviceCostMatrix, ndarray or torch.Tensor")
    n, m = int(src.shape[0]), int(src.shape[1])
    ldc = (m + 3) // 4 * 4
    if (src.dtype == torch.float32 and src.stride(0) == ldc and ldc == m
            and src.data_ptr() % 16 == 0):
        return DeviceCostMatrix(data=src, rows=n, cols=m)
    if src.dtype not in (torch.float32, torch.float64):
        src = src.to(torch.float64)
    out = torch.empty((n, ldc), dtype=torch.float32, device="cuda")
    _lib.call("lsk_cast_cost_f32", _ptr(src), int(src.dtype == torch.float64), src.stride(0), n, m,
              _ptr(out), ldc, _stream_ptr(torch))
    return DeviceCostMatrix(data=out, rows=n, cols=m)


def _check_dims(cost, mu, nu):
    rows, cols = (cost.rows, cost.cols)
    if rows != mu.size or cols != nu.size:
        raise DimensionMismatch(
            f"cost is {rows}x{cols} but distributions have {mu.size} and {nu.size} weights")


def _f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32)


class _Solved:
    """Device results of one solve (kept on the GPU unless read)."""

    __slots__ = ("f", "g", "trace_iter", "trace_err", "res", "resf", "ev0", "ev1")


def _uniform(log_w):
    """All target log-weights equal (host arrays; tensors are not inspected)."""
    if isinstance(log_w, np.ndarray) and log_w.size:
        return bool(np.all(log_w.astype(np.float32) == np.float32(log_w[0])))
    return False


def _launch_solve(torch, C, log_mu, log_nu, mu32, config, stale=True, want_cost=True, ws=None,
                  uniform_nu=False, mult=False, cluster=True):
    C = to_device_cost(C)
    n, m = C.rows, C.cols
    K, c = int(config.max_iterations), int(config.check_interval)
    cap = _lib.load().lsk_trace_capacity(K, c)
    wsb = _lib.load().lsk_solve_dense_workspace_bytes(n, m)
    if ws is None or ws.numel() < wsb:
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    r = _Solved()
    r.f = torch.empty(n, dtype=torch.float32, device="cuda")
    r.g = torch.empty(m, dtype=torch.float32, device="cuda")
    r.trace_iter = torch.empty(cap, dtype=torch.int32, device="cuda")
    r.trace_err = torch.empty(cap, dtype=torch.float32, device="cuda")
    r.res = torch.zeros(8, dtype=torch.int32, device="cuda")
    r.resf = torch.zeros(2, dtype=torch.float32, device="cuda")
    flags = (_lib.LSK_FLAG_STALE_SHIFT if stale else 0) | (_lib.LSK_FLAG_COST if want_cost else 0)
    flags |= _lib.LSK_FLAG_UNIFORM_NU if uniform_nu else 0
    flags |= _lib.LSK_FLAG_MULT if mult else 0
    flags |= 0 if cluster else _lib.LSK_FLAG_NO_CLUSTER
    r.ev0 = torch.cuda.Event(enable_timing=True)
    r.ev1 = torch.cuda.Event(enable_timing=True)
    r.ev0.record()
    _lib.call("lsk_solve_dense_f32", _ptr(C.data), C.ldc, n, m, _ptr(log_mu), _ptr(log_nu), _ptr(mu32),
              float(config.epsilon), float(config.tolerance), K, c, flags, _ptr(r.f), _ptr(r.g),
              _ptr(r.trace_iter), _ptr(r.trace_err), _ptr(r.res), _ptr(r.resf), _ptr(ws), ws.numel(),
              _stream_ptr(torch))
    r.ev1.record()
    return r, ws


def _report_from(r, t0, return_device=False):
    """One host sync: read status/iters/trace/err/cost (+ potentials)."""
    res = r.res.cpu().numpy()
    resf = r.resf.cpu().numpy()
    nt = int(res[2])
    it = r.trace_iter[:nt].cpu().numpy()
    te = r.trace_err[:nt].cpu().numpy()
    status = _STATUS_BY_CODE[int(res[0])]
    if return_device:
        alpha, beta = r.f, r.g
    else:
        alpha, beta = r.f.cpu().numpy(), r.g.cpu().numpy()
    elapsed = time.perf_counter() - t0
    err = float(resf[0])
    cost = float(resf[1]) if status != STATUS_NUMERICAL_FAILURE else float("nan")
    report = SolveReport(
        status=status,
        iterations=int(res[1]),
        final_marginal_error=err,
        transport_cost=cost,
        error_trace=tuple((int(k), float(e)) for k, e in zip(it, te)),
        elapsed_seconds=elapsed,
        device_seconds=r.ev0.elapsed_time(r.ev1) * 1e-3,
        guard_stats=(int(res[4]), int(res[5])),
    )
    return report, DualPotentials(alpha=alpha, beta=beta)


def solve(cost, mu, nu, config, *, stale_shift=True, return_device=False, multiplicative=False, cluster=True):
    """Log-domain Sinkhorn from zero potentials (reference solver.py:230-337).

    Alternates f (alpha) and g (beta) updates, checks the L1 row-marginal
    error every ``config.check_interval`` iterations (finiteness first),
    stops on error < tolerance (converged), a non-finite value
    (numerical_failure) or at ``max_iterations`` (not_converged, after a
    final check when the cap is not a checkpoint), and evaluates the
    transport cost unless the solve failed. The whole loop is one
    cooperative kernel launch; the host synchronises once, at the end.

    Every g-side argument is formed from the cost element as the reference
    does. ``multiplicative=True`` opts in to the multiplicative column update
    of the uniform-target kernel (``LSK_FLAG_MULT``: g-side terms from the
    f-side ones, ~18% faster at n = m = 8192) -- an approximation whose
    potentials drift from the reference's by up to ~3e-5 relative at K = 1000
    (profiles/r2_mult_drift.md), so it is never on by default.
    ``cluster=False`` runs the 148-CTA grid solver instead of the cluster
    solvers at m <= 1024 with uniform targets (``LSK_FLAG_NO_CLUSTER``; A/B).
    ``stale_shift=False`` selects the exact two-pass variant (max pass per
    row, exact column pass every iteration) instead of the one-pass
    stale-shift fast path; ``return_device=True`` leaves the potentials as
    CUDA tensors. ``config.transpose_for_beta`` and the reduction-plan fields
    are validated and otherwise inert (the kernels read C row-major for
    both half-steps; results are bit-identical either way).
    """
    _check_dims(cost, mu, nu)
    if config.precision == "double":  # the reference's float64 path (types.py:168-170)
        _torch()
        return _s64.solve(cost, mu, nu, config, return_device)
    torch = _torch()
    t0 = time.perf_counter()
    C = to_device_cost(cost)
    log_mu = _dev_f32(torch, mu.log_weights)
    log_nu = _dev_f32(torch, nu.log_weights)
    mu32 = _dev_f32(torch, mu.weights)
    r, _ = _launch_solve(torch, C, log_mu, log_nu, mu32, config, stale=stale_shift,
                         uniform_nu=_uniform(nu.log_weights), mult=multiplicative, cluster=cluster)
    return _report_from(r, t0, return_device)


def _half_inputs(cost, eps):
    if not (eps > 0):
        raise ValueError("eps must be > 0")
    return _torch()


def update_alpha(cost, nu, beta, eps, plan=ReductionPlan()):
    """One alpha half-step (reference solver.py:118-140) in the dtype of beta."""
    torch = _half_inputs(cost, eps)
    if _is_f64(beta):
        return _s64.update_alpha(cost, nu, beta, eps)
    C = to_device_cost(cost)
    b, lnu = _vecs(torch, beta, nu.log_weights)
    out = torch.empty(C.rows, dtype=torch.float32, device="cuda")
    _lib.call("lsk_update_alpha_f32", _ptr(C.data), C.ldc, C.rows, C.cols, _ptr(b), _ptr(lnu), float(eps),
              _ptr(out), _stream_ptr(torch))
    return out.cpu().numpy()


def update_beta(cost, mu, alpha, eps, plan=ReductionPlan(), transposed_cost=None):
    """One beta half-step (reference solver.py:143-176), fp32.

    ``transposed_cost`` is accepted (shape-checked) but both layouts run the
    same coalesced column kernel over C, so the strided and transposed
    results are bit-identical, as the reference guarantees.
    """
    torch = _half_inputs(cost, eps)
    if transposed_cost is not None:
        tv = getattr(transposed_cost, "values", transposed_cost)  # an array (reference) or a CostMatrix
        shp = tuple(tv.shape) if hasattr(tv, "shape") else tuple(np.shape(tv))
        rows, cols = (cost.rows, cost.cols)
        if shp != (cols, rows):
            raise DimensionMismatch(f"transposed_cost has shape {shp}, expected {(cols, rows)}")
    if _is_f64(alpha):
        return _s64.update_beta(cost, mu, alpha, eps)
    C = to_device_cost(cost)
    a, lmu = _vecs(torch, alpha, mu.log_weights)
    out = torch.empty(C.cols, dtype=torch.float32, device="cuda")
    wsb = _lib.load().lsk_update_beta_workspace_bytes(C.rows, C.cols)
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
    _lib.call("lsk_update_beta_f32", _ptr(C.data), C.ldc, C.rows, C.cols, _ptr(a), _ptr(lmu), float(eps),
              _ptr(out), _ptr(ws), ws.numel(), _stream_ptr(torch))
    return out.cpu().numpy()


def _vecs(torch, *xs):
    """fp32 device copies, returned together so they stay alive (and distinct
    allocations) until the kernel that reads them has been enqueued."""
    return [_dev_f32(torch, x) for x in xs]


def marginal_error(cost, mu, nu, alpha, beta, eps, plan=ReductionPlan()):
    """L1 row-marginal error of (alpha, beta) (reference solver.py:179-206)."""
    torch = _half_inputs(cost, eps)
    if _is_f64(alpha, beta):
        return _s64.marginal_error(cost, mu, nu, alpha, beta, eps)
    C = to_device_cost(cost)
    w, lmu, lnu, a, b = _vecs(torch, mu.weights, mu.log_weights, nu.log_weights, alpha, beta)
    ws = torch.empty(C.rows, dtype=torch.float32, device="cuda")
    out = torch.empty(1, dtype=torch.float32, device="cuda")
    _lib.call("lsk_marginal_error_f32", _ptr(C.data), C.ldc, C.rows, C.cols, _ptr(w), _ptr(lmu), _ptr(lnu),
              _ptr(a), _ptr(b), float(eps), _ptr(out), _ptr(ws), ws.numel() * 4, _stream_ptr(torch))
    return float(out.cpu().numpy()[0])


def transport_cost(cost, mu, nu, alpha, beta, eps, plan=ReductionPlan()):
    """Plan-weighted total cost (reference solver.py:209-227)."""
    torch = _half_inputs(cost, eps)
    if _is_f64(alpha, beta):
        return _s64.transport_cost(cost, mu, nu, alpha, beta, eps)
    C = to_device_cost(cost)
    lmu, lnu, a, b = _vecs(torch, mu.log_weights, nu.log_weights, alpha, beta)
    ws = torch.empty(C.rows, dtype=torch.float32, device="cuda")
    out = torch.empty(1, dtype=torch.float32, device="cuda")
    _lib.call("lsk_transport_cost_f32", _ptr(C.data), C.ldc, C.rows, C.cols, _ptr(lmu), _ptr(lnu), _ptr(a),
              _ptr(b), float(eps), _ptr(out), _ptr(ws), ws.numel() * 4, _stream_ptr(torch))
    return float(out.cpu().numpy()[0])


def materialize_plan(cost, mu, nu, alpha, beta, eps, *, return_device=False):
    """Dense coupling from dual potentials (reference solver.py:434-458).

    Raises NonFiniteResult if any entry is NaN or infinite.
    """
    torch = _half_inputs(cost, eps)
    if _is_f64(alpha, beta):
        return _s64.materialize_plan(cost, mu, nu, alpha, beta, eps, return_device)
    C = to_device_cost(cost)
    lmu, lnu, a, b = _vecs(torch, mu.log_weights, nu.log_weights, alpha, beta)
    P = torch.empty((C.rows, C.cols), dtype=torch.float32, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("lsk_materialize_plan_f32", _ptr(C.data), C.ldc, C.rows, C.cols, _ptr(lmu), _ptr(lnu), _ptr(a),
              _ptr(b), float(eps), _ptr(P), C.cols, _ptr(bad), _stream_ptr(torch))
    if int(bad.item()) != 0:
        raise NonFiniteResult("transport plan contains non-finite entries")
    return TransportPlan(values=P if return_device else P.cpu().numpy())
