"""The reference's deterministic reductions (``reduction.py``) on the GPU.

Same names, signatures and tree shape: max / sum / log-sum-exp over rows,
columns or a 1-D view with a ``ReductionPlan(chunk_width, group_size)``
(lane fold, ceil-halving within chunks, then across chunks). One C-ABI call
per reduction (``lsk_reduce_rows`` / ``lsk_reduce_cols``, ``csrc/lsk_reduce.cu``):
max and sum are bit-identical to the reference for every plan, log-sum-exp
matches to the exponential's ulps. float32 and float64 inputs keep their dtype;
other dtypes are reduced in float64.
"""

import numpy as np

from . import _lib
from .errors import EmptyView
from .solver import _ptr, _stream_ptr, _torch
from .types import ReductionPlan

__all__ = ["SUM_FLOOR", "reduce_max", "reduce_sum", "log_sum_exp", "reduce_max_rows", "reduce_sum_rows",
           "log_sum_exp_rows", "reduce_max_cols", "reduce_sum_cols", "log_sum_exp_cols"]

SUM_FLOOR = 1e-30
_OPS = {"max": 0, "sum": 1, "lse": 2}


def _run(A, plan, op, cols):
    torch = _torch()
    A = np.asarray(A)
    if A.ndim != 2:
        raise ValueError("expected a 2-D array")
    if A.dtype not in (np.float32, np.float64):
        A = A.astype(np.float64)
    L, R = (A.shape[0], A.shape[1]) if cols else (A.shape[1], A.shape[0])
    if A.size == 0:
        raise EmptyView("reduction over an empty view")
    dt = 1 if A.dtype == np.float64 else 0
    Ad = torch.from_numpy(np.ascontiguousarray(A)).to("cuda")
    out = torch.empty(R, dtype=Ad.dtype, device="cuda")
    wsb = _lib.load().lsk_reduce_workspace_bytes(R, dt) if op == 2 else 0
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
    fn = "lsk_reduce_cols" if cols else "lsk_reduce_rows"
    # dense row-major copy: the row stride is the row length (a size-1 leading
    # dimension may carry stride 0 in numpy/torch)
    lda = R if cols else L
    _lib.call(fn, _ptr(Ad), lda, (L if cols else R), (R if cols else L), dt, op, plan.chunk_width,
              plan.group_size, _ptr(out), _ptr(ws), wsb, _stream_ptr(torch))
    return out.cpu().numpy()


def reduce_max_rows(A, plan):
    """Per-row maximum over the deterministic tree (NaN propagates)."""
    return _run(A, plan, 0, False)


def reduce_sum_rows(A, plan):
    """Per-row sum over the deterministic tree."""
    return _run(A, plan, 1, False)


def reduce_max_cols(A, plan):
    """Per-column maximum, reading along the strided axis."""
    return _run(A, plan, 0, True)


def reduce_sum_cols(A, plan):
    """Per-column sum, reading along the strided axis."""
    return _run(A, plan, 1, True)


def log_sum_exp_rows(A, plan, workspace=None):
    """Per-row max-shifted log-sum-exp (sum floored at 1e-30; rows whose max is
    not finite give -inf). ``workspace`` is accepted for signature parity and unused."""
    return _run(A, plan, 2, False)


def log_sum_exp_cols(A, plan, workspace=None):
    """Per-column mirror of :func:`log_sum_exp_rows`."""
    return _run(A, plan, 2, True)


def _view(view):
    v = np.asarray(view)
    if v.ndim != 1:
        v = v.reshape(-1)
    if v.size == 0:
        raise EmptyView("reduction over an empty view")
    return v


def reduce_max(view, plan=ReductionPlan()):
    """Maximum of a 1-D view (equals a sequential scan exactly)."""
    return reduce_max_rows(_view(view)[None, :], plan)[0]


def reduce_sum(view, plan=ReductionPlan()):
    """Fixed-tree sum of a 1-D view."""
    return reduce_sum_rows(_view(view)[None, :], plan)[0]


def log_sum_exp(view, plan=ReductionPlan()):
    """Stable log(sum(exp(view))) of a 1-D view; -inf if every entry is -inf."""
    return log_sum_exp_rows(np.ascontiguousarray(_view(view))[None, :], plan)[0]
