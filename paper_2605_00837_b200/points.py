"""Point-cloud solves with the cost recomputed on the fly (configs C4/C5).

Drop-in for the reference composition ``squared_euclidean_cost(X, Y)``
(``costs.py:36-50``), optionally ``C / C.max()`` (``applications.py:186-188``,
``estimator.py:87-89``), then ``solve`` (``solver.py:230-337``) -- without ever
materialising the (n, m) cost: one ``lsk_solve_points_f32`` call runs the whole
solve for a batch of problems, recomputing ``sum_k (x_ik - y_jk)^2`` in
registers. Returns the reference's ``(SolveReport, DualPotentials)``.

* ``solve_points_otf``: one problem; with ``comm`` (``dist.Communicator``) it
  is sharded over the ranks: ``shard="partials"`` (default: row
  slabs of the source cloud, per-column partials exchanged and merged by a
  fixed tree), ``"allreduce"`` (stale sums by ncclAllReduce) or ``"owner"``
  (owner computes, potential slabs allgathered).
* ``solve_points_emulated``: the same P-rank decomposition on one GPU
  (collectives as device copies); reports whether every virtual rank ended
  bit-identical.
* ``solve_points_batched``: B independent problems of one shape in a single
  launch sequence; each problem stops on its own (per-problem status / trace).

Numerics: fp32 cost from fp32-rounded points in the direct form (SURVEY F5:
~2-3e-6 on the potentials at eps=1e-3). Callers choose the path:
``costs.solve_points`` always builds the fp64-exact dense matrix (bit-identical
to the reference's cast); this module is the on-the-fly path for clouds whose
(n, m) matrix should not be stored (C4: 17 GB) and for batches (C5).
"""

import time

import numpy as np

from . import _lib
from .costs import as_points
from .errors import DimensionMismatch
from .solver import _STATUS_BY_CODE, _ptr, _stream_ptr, _torch
from .types import DualPotentials, SolveReport

__all__ = ["solve_points_otf", "solve_points_batched", "solve_points_emulated", "points_cost_max"]


def _batch_points(P):
    """(B, k, d) float64 contiguous from a (k, d) / (B, k, d) array."""
    A = np.asarray(P, dtype=np.float64)
    if A.ndim == 2:
        A = A[None]
    if A.ndim != 3:
        raise DimensionMismatch(f"point batch must be (B, k, d), got {A.shape}")
    for b in range(A.shape[0]):
        as_points(A[b])  # validation (EmptyInput / NonFiniteInput)
    return np.ascontiguousarray(A)


def _weights(dist, B, k, name):
    """(B, k) fp64 weights and log-weights from None (uniform) / a
    DiscreteDistribution / a sequence of them."""
    if dist is None:
        w = np.full((B, k), 1.0 / k)
        return w, np.log(w)
    if hasattr(dist, "weights"):
        dist = [dist] * B
    if len(dist) != B:
        raise DimensionMismatch(f"{name}: expected {B} distributions, got {len(dist)}")
    w = np.stack([np.asarray(d.weights, np.float64) for d in dist])
    lw = np.stack([np.asarray(d.log_weights, np.float64) for d in dist])
    if w.shape != (B, k):
        raise DimensionMismatch(f"{name}: weights of shape {w.shape}, expected {(B, k)}")
    return w, lw


def points_cost_range(Xd, Yd):
    """(B, 2) device doubles: the exact fp64 max and min of the cost per problem."""
    torch = _torch()
    B, n, d = Xd.shape
    m = Yd.shape[1]
    out = torch.empty((B, 2), dtype=torch.float64, device="cuda")
    wsb = _lib.load().lsk_points_cost_range_workspace_bytes(B, n, m)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.call("lsk_points_cost_range", _ptr(Xd), _ptr(Yd), B, n, m, d, _ptr(out), _ptr(ws), wsb, _stream_ptr(torch))
    return out


def points_scale(Xd, Yd, normalize):
    """(B,) fp32 cost scale: 1/C.max() where value_range > 0 (applications.py:186-188), else 1."""
    torch = _torch()
    B = Xd.shape[0]
    if normalize != "max":
        return torch.ones(B, dtype=torch.float32, device="cuda")
    r = points_cost_range(Xd, Yd)
    cmax, cmin = r[:, 0], r[:, 1]
    return torch.where(cmax > cmin, 1.0 / cmax, torch.ones_like(cmax)).to(torch.float32)


def points_cost_max(Xd, Yd):
    """Exact fp64 max of the squared-Euclidean cost per problem (device)."""
    torch = _torch()
    B, n, d = Xd.shape
    m = Yd.shape[1]
    out = torch.empty(B, dtype=torch.float64, device="cuda")
    wsb = _lib.load().lsk_points_cost_max_workspace_bytes(B, n, m)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.call("lsk_points_cost_max", _ptr(Xd), _ptr(Yd), B, n, m, d, _ptr(out), _ptr(ws), wsb, _stream_ptr(torch))
    return out  # ws is freed to the caching allocator in stream order: safe


class _PointsRun:
    __slots__ = ("B", "n", "m", "f", "g", "ti", "te", "res", "resf", "ev0", "ev1", "t0", "keep", "mismatch")


_SHARD = {"owner": (_lib.LSK_SHARD_OWNER, 0), "partials": (_lib.LSK_SHARD_PARTIALS, _lib.LSK_FLAG_SHARD_PARTIALS),
          "allreduce": (_lib.LSK_SHARD_ALLREDUCE, _lib.LSK_FLAG_SHARD_ALLREDUCE)}


# The expansion form c = |x|^2 + |y|^2 - 2 x.y (kernels translate every problem to
# the centre c of its bounding box) carries an absolute rounding error of about
# (|x - c|^2 + |y - c|^2) 2^-24 in c, i.e. that over eps (and the cost
# normaliser) in every exponent. It is requested only when that bound stays
# below 1e-5 -- the C5 RGB unit-cube problems at eps = 1e-2 sit at 9e-6 and are
# parity-tested per potential; wider clouds or smaller eps use the direct
# (x - y)^2 form.
_EXPANSION_BOUND = 1e-5


def _expansion_ok(Xb, Yb, eps, normalize):
    lo = np.minimum(Xb.min(axis=1), Yb.min(axis=1))[:, None, :]
    hi = np.maximum(Xb.max(axis=1), Yb.max(axis=1))[:, None, :]
    c = 0.5 * (lo + hi)  # the kernels' translation (k_pts_center)
    rx = ((Xb - c) ** 2).sum(axis=2).max(axis=1)
    ry = ((Yb - c) ** 2).sum(axis=2).max(axis=1)
    # C.max() >= max_j |y_j - x_0|^2 (x_0 a source point): a lower bound of the normaliser
    ry0 = ((Yb - Xb[:, :1, :]) ** 2).sum(axis=2).max(axis=1)
    div = np.where((normalize == "max") & (ry0 > 0), ry0, 1.0)
    bound = (rx + ry) * 2.0 ** -24 / (float(eps) * div)
    return bool(np.all(bound <= _EXPANSION_BOUND))


def _launch(X, Y, mu, nu, config, normalize, stale, want_cost, comm, expansion=False, shard="partials",
            emulate_ranks=None, graphs=True):
    torch = _torch()
    if config.precision != "single":
        raise NotImplementedError("the on-the-fly points solver computes in fp32; use precision='single', or "
                                  "solve(squared_euclidean_cost(X, Y), ...) for precision='double'")
    if normalize not in ("none", "max"):
        raise ValueError("normalize must be 'none' or 'max'")
    Xb, Yb = _batch_points(X), _batch_points(Y)
    if Xb.shape[0] != Yb.shape[0] or Xb.shape[2] != Yb.shape[2]:
        raise DimensionMismatch(f"point batches {Xb.shape} and {Yb.shape} do not match")
    B, n, d = Xb.shape
    m = Yb.shape[1]
    wmu, lmu = _weights(mu, B, n, "mu")
    _, lnu = _weights(nu, B, m, "nu")
    r = _PointsRun()
    r.t0 = time.perf_counter()
    r.B, r.n, r.m = B, n, m
    Xd = torch.from_numpy(Xb).to("cuda")
    Yd = torch.from_numpy(Yb).to("cuda")
    # reference: C / C.max() only when the cost has a non-zero range (applications.py:186-188)
    scale = points_scale(Xd, Yd, normalize)
    lmu_d = torch.from_numpy(lmu.astype(np.float32)).to("cuda")
    lnu_d = torch.from_numpy(lnu.astype(np.float32)).to("cuda")
    mu_d = torch.from_numpy(wmu.astype(np.float32)).to("cuda")
    K, c = int(config.max_iterations), int(config.check_interval)
    cap = _lib.load().lsk_trace_capacity(K, c)
    if shard not in _SHARD:
        raise ValueError("shard must be 'partials', 'allreduce' or 'owner'")
    mode, shard_flag = _SHARD[shard]
    lib = _lib.load()
    if emulate_ranks is not None:
        if B != 1 or comm is not None:
            raise ValueError("emulate_ranks: one problem, no communicator")
        P = int(emulate_ranks)
        wsb = P * lib.lsk_solve_points_sharded_workspace_bytes(n, m, P, mode)
    elif comm is not None:
        if B != 1:
            raise ValueError("a sharded solve takes one problem (split batches over ranks instead)")
        wsb = lib.lsk_solve_points_sharded_workspace_bytes(n, m, comm.world, mode)
    else:
        shard_flag = 0
        wsb = lib.lsk_solve_points_workspace_bytes(B, n, m)
    if wsb == 0:
        _lib.call("lsk_solve_points_sharded_workspace_bytes", n, m, emulate_ranks or comm.world, mode)
        raise ValueError(f"shard={shard!r} does not support this rank count / shape")
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    r.f = torch.empty((B, n), dtype=torch.float32, device="cuda")
    r.g = torch.empty((B, m), dtype=torch.float32, device="cuda")
    r.ti = torch.zeros((B, cap), dtype=torch.int32, device="cuda")
    r.te = torch.zeros((B, cap), dtype=torch.float32, device="cuda")
    r.res = torch.zeros((B, 8), dtype=torch.int32, device="cuda")
    r.resf = torch.zeros((B, 2), dtype=torch.float32, device="cuda")
    flags = (_lib.LSK_FLAG_STALE_SHIFT if stale else 0) | (_lib.LSK_FLAG_COST if want_cost else 0)
    if expansion and not _expansion_ok(Xb, Yb, config.epsilon, normalize):
        expansion = False
    flags |= _lib.LSK_FLAG_EXPANSION if expansion else 0
    flags |= shard_flag
    # CUDA-graph replay of the iteration blocks (include/lsk.h): the library's default,
    # off with graphs=False, NCCL collectives captured too with graphs="nccl"
    flags |= _lib.LSK_FLAG_NO_GRAPH if graphs is False else 0
    flags |= _lib.LSK_FLAG_GRAPH_NCCL if graphs == "nccl" else 0
    r.ev0 = torch.cuda.Event(enable_timing=True)
    r.ev1 = torch.cuda.Event(enable_timing=True)
    r.mismatch = None
    r.ev0.record()
    if emulate_ranks is not None:
        r.mismatch = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.call("lsk_solve_points_emulated_f32", _ptr(Xd), _ptr(Yd), n, m, d, _ptr(scale), _ptr(lmu_d),
                  _ptr(lnu_d), _ptr(mu_d), float(config.epsilon), float(config.tolerance), K, c, flags,
                  int(emulate_ranks), mode, _ptr(r.f), _ptr(r.g), _ptr(r.ti), _ptr(r.te), _ptr(r.res),
                  _ptr(r.resf), _ptr(r.mismatch), _ptr(ws), wsb, _stream_ptr(torch))
    else:
        _lib.call("lsk_solve_points_f32", _ptr(Xd), _ptr(Yd), B, n, m, d, _ptr(scale), _ptr(lmu_d), _ptr(lnu_d),
                  _ptr(mu_d), float(config.epsilon), float(config.tolerance), K, c, flags, _ptr(r.f), _ptr(r.g),
                  _ptr(r.ti), _ptr(r.te), _ptr(r.res), _ptr(r.resf), _ptr(ws), wsb,
                  comm.handle if comm is not None else None, _stream_ptr(torch))
    r.ev1.record()
    r.keep = (Xd, Yd, scale, lmu_d, lnu_d, mu_d, ws)  # alive until the results are read
    return r


def _reports(r, return_device=False):
    res = r.res.cpu().numpy()
    resf = r.resf.cpu().numpy()
    ti = r.ti.cpu().numpy()
    te = r.te.cpu().numpy()
    dev = r.ev0.elapsed_time(r.ev1) * 1e-3
    f = r.f if return_device else r.f.cpu().numpy()
    g = r.g if return_device else r.g.cpu().numpy()
    elapsed = time.perf_counter() - r.t0
    out = []
    for b in range(r.B):
        nt = int(res[b, 2])
        status = _STATUS_BY_CODE[int(res[b, 0])]
        rep = SolveReport(status=status, iterations=int(res[b, 1]), final_marginal_error=float(resf[b, 0]),
                          transport_cost=float(resf[b, 1]) if status != "numerical_failure" else float("nan"),
                          error_trace=tuple((int(k), float(e)) for k, e in zip(ti[b, :nt], te[b, :nt])),
                          elapsed_seconds=elapsed, device_seconds=dev)
        out.append((rep, DualPotentials(alpha=f[b], beta=g[b])))
    return out


def solve_points_otf(X, Y, mu, nu, config, normalize="none", *, stale_shift=True, comm=None, return_device=False,
                     expansion=False, shard="partials", graphs=True):
    """One on-the-fly solve of points X (n, d) vs Y (m, d); see module doc.
    ``expansion=True`` (opt-in speed mode) evaluates the cost as
    |x|^2+|y|^2-2x.y in the stale sweeps when eps >= 5e-3 and the rounding
    bound of that form is small against eps (``_expansion_ok``; 3 instead of 6
    FP32 ops per pair). Its cancellation moves the potentials by up to ~3e-5
    (per potential) on the C5 shape -- outside the 1e-5 parity bar -- so the
    default is the direct form.
    ``comm`` / ``shard``: see the module doc. ``graphs``: CUDA-graph replay of the
    iteration blocks (True: the library default; False: off; "nccl": also capture
    the collectives of a sharded solve)."""
    r = _launch(X, Y, mu, nu, config, normalize, stale_shift, True, comm, expansion, shard, graphs=graphs)
    return _reports(r, return_device)[0]


def solve_points_emulated(X, Y, mu, nu, config, ranks, normalize="none", *, shard="partials", stale_shift=True,
                          expansion=False, graphs=True):
    """The P-rank decomposition of ``solve_points_otf(..., comm=<P ranks>,
    shard=shard)`` run on this one GPU: every virtual rank has its own
    workspace, its kernels run rank after rank, and the collectives are device
    copies (``lsk_solve_points_emulated_f32``). Returns ``(report, potentials,
    rank_mismatch)`` -- rank 0's results and the number of ranks whose returned
    potentials / status / error / cost differ from rank 0's in any bit."""
    r = _launch(X, Y, mu, nu, config, normalize, stale_shift, True, None, expansion, shard, ranks, graphs=graphs)
    rep, pot = _reports(r)[0]
    return rep, pot, int(r.mismatch.item())


def solve_points_batched(X, Y, config, mu=None, nu=None, normalize="none", *, stale_shift=True,
                         return_device=False, expansion=False, graphs=True):
    """B independent solves, X (B, n, d) vs Y (B, m, d), uniform marginals by
    default (``mu``/``nu``: a DiscreteDistribution for all, or one per problem).
    Returns a list of (SolveReport, DualPotentials)."""
    r = _launch(X, Y, mu, nu, config, normalize, stale_shift, True, None, expansion, graphs=graphs)
    return _reports(r, return_device)
