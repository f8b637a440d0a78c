"""CPU oracle for the log-domain Sinkhorn hot path -- TEST INFRASTRUCTURE ONLY.

This module is the *checker*, never the product. Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it. The shipped package
(``paper_2605_00837_b200``) never imports anything from ``oracle/``; it fails
loudly when its CUDA library is missing instead of falling back here.

What it restates (reference = ``/root/reference/pkg/src/logsinkhorn``):

* the fixed-shape reduction tree of ``reduction.py:72-113`` (lane fold over
  ``group_size`` lanes, ceil-halving inside ``chunk_width`` chunks, then
  across chunks; ``ReductionPlan(1, 1)`` is a flat scan) and the two-pass
  log-sum-exp of ``reduction.py:179-208`` with ``SUM_FLOOR`` (44);
* the half-steps ``_alpha_step`` / ``_beta_step_*`` (``solver.py:76-94``),
  ``_marginal_error`` (97-104), ``_transport_cost`` (107-115), the ``solve``
  loop with its status / trace / final-check semantics (230-337) and
  ``materialize_plan`` (434-458);
* the fp64 direct-broadcast cost ``squared_euclidean_cost``
  (``costs.py:36-50``; the coordinate sum runs ``(d0^2 + d1^2) + d2^2``),
  the pipeline max-normalisation (``applications.py:186-188``) and the
  seeded generators ``generate_grid_problem`` (``costs.py:73-116``) and
  ``generate_rigid_pair`` (``applications.py:215-247``).

Every elementwise op is the same numpy ufunc in the same dtype and order as
the reference, and the tree is the same tree, so results are bit-identical to
the reference (pinned by ``tests/test_oracle.py`` against the fixtures in
``tests/golden/`` that ``tests/golden/make_golden.py`` produced by running the
reference itself). Rows (and, through the transpose, columns) are independent,
so the row blocking and the thread pool used here do not change a single bit;
they only bound memory and let the CPU baseline use every host core.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

SUM_FLOOR = 1e-30  # reduction.py:44

STATUS_CONVERGED = "converged"  # types.py:35-37
STATUS_NOT_CONVERGED = "not_converged"
STATUS_NUMERICAL_FAILURE = "numerical_failure"

_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1))
    return _POOL


def host_threads():
    return max(1, os.cpu_count() or 1)


# ---------------------------------------------------------------------------
# fixed-shape reduction tree (reduction.py:72-113)


def _ceil_halve(a, op):
    """Fold the last axis of ``a`` in place: pair k with k+ceil(w/2)."""
    w = a.shape[-1]
    while w > 1:
        h = (w + 1) // 2
        op(a[..., : w - h], a[..., h:w], out=a[..., : w - h])
        w = h
    return a[..., 0]


def tree_reduce_rows(A, op, identity, chunk_width=32, group_size=256):
    """Per-row reduction of a 2-D array on the reference's frozen tree."""
    A = np.ascontiguousarray(A)
    R, L = A.shape
    B = group_size
    k = -(-L // B)
    if k * B != L:
        A = np.concatenate([A, np.full((R, k * B - L), identity, A.dtype)], axis=1)
    blocks = A.reshape(R, k, B)
    lanes = blocks[:, 0, :].copy()
    for s in range(1, k):
        op(lanes, blocks[:, s, :], out=lanes)
    if B == 1:
        return lanes[:, 0].copy()
    chunks = lanes.reshape(R, B // chunk_width, chunk_width)
    heads = np.ascontiguousarray(_ceil_halve(chunks, op))
    return _ceil_halve(heads, op).copy()


def tree_max_rows(A, cw=32, gs=256):
    return tree_reduce_rows(A, np.maximum, -np.inf, cw, gs)


def tree_sum_rows(A, cw=32, gs=256):
    return tree_reduce_rows(A, np.add, 0.0, cw, gs)


def lse_rows(T, cw=32, gs=256):
    """Two-pass row log-sum-exp (reduction.py:179-208)."""
    dt = T.dtype.type
    M = tree_max_rows(T, cw, gs)
    empty = ~np.isfinite(M)
    if empty.any():
        M = np.where(empty, dt(0.0), M)
    D = np.exp(T - M[:, None])
    S = tree_sum_rows(D, cw, gs)
    np.maximum(S, dt(SUM_FLOOR), out=S)
    out = M + np.log(S)
    if empty.any():
        out[empty] = -np.inf
    return out


# ---------------------------------------------------------------------------
# half-steps, blocked over rows (bit-neutral: rows are independent)


def _row_blocks(R, L, budget=1 << 22):
    step = max(1, min(R, budget // max(L, 1)))
    return [(r, min(R, r + step)) for r in range(0, R, step)]


def _map_rows(fn, R, L, threads=True):
    blocks = _row_blocks(R, L)
    if threads and len(blocks) > 1 and host_threads() > 1:
        parts = list(_pool().map(fn, blocks))
    else:
        parts = [fn(b) for b in blocks]
    return np.concatenate(parts)


def row_update(C, other, log_w, inv_eps, neg_eps, cw=32, gs=256, threads=True):
    """``neg_eps * LSE_j((other_j - C_ij) * inv_eps + log_w_j)``.

    alpha-step on C (solver.py:76-80); the beta-step is the same call on
    C^T with (alpha, log_mu) (solver.py:83-94: strided == transposed, bitwise).
    """
    R, L = C.shape

    def blk(b):
        r0, r1 = b
        T = np.subtract(other[None, :], C[r0:r1])
        np.multiply(T, inv_eps, out=T)
        np.add(T, log_w[None, :], out=T)
        return neg_eps * lse_rows(T, cw, gs)

    return _map_rows(blk, R, L, threads)


def check_rows(C, alpha, beta, log_nu, inv_eps, cw=32, gs=256, threads=True):
    """Row LSE of the marginal-error argument (solver.py:98-102)."""
    R, L = C.shape

    def blk(b):
        r0, r1 = b
        T = np.add(alpha[r0:r1, None], beta[None, :])
        np.subtract(T, C[r0:r1], out=T)
        np.multiply(T, inv_eps, out=T)
        np.add(T, log_nu[None, :], out=T)
        return lse_rows(T, cw, gs)

    return _map_rows(blk, R, L, threads)


def marginal_err(C, mu_d, log_mu, log_nu, alpha, beta, inv_eps, cw=32, gs=256, threads=True):
    """solver.py:97-104."""
    L = check_rows(C, alpha, beta, log_nu, inv_eps, cw, gs, threads)
    r = np.exp(log_mu + L)
    return tree_sum_rows(np.abs(r - mu_d)[None, :], cw, gs)[0]


def transport_cost_rows(C, log_mu, log_nu, alpha, beta, inv_eps, cw=32, gs=256, threads=True):
    """solver.py:107-115: per-row tree sums of C*P, then a tree sum."""
    R, L = C.shape

    def blk(b):
        r0, r1 = b
        Cb = C[r0:r1]
        Z = alpha[r0:r1, None] + beta[None, :]
        Z -= Cb
        Z *= inv_eps
        Z += log_mu[r0:r1, None]
        Z += log_nu[None, :]
        P = np.exp(Z)
        return tree_sum_rows(Cb * P, cw, gs)

    rows = _map_rows(blk, R, L, threads)
    return float(tree_sum_rows(rows[None, :], cw, gs)[0])


def plan_values(C, log_mu, log_nu, alpha, beta, inv_eps):
    """solver.py:434-458 (without the NonFiniteResult raise)."""
    Z = alpha[:, None] + beta[None, :]
    Z -= C
    Z *= inv_eps
    Z += log_mu[:, None]
    Z += log_nu[None, :]
    return np.exp(Z)


# ---------------------------------------------------------------------------
# the solve loop (solver.py:230-337)


def solve(C, mu_w, nu_w, eps, tol=1e-6, max_iter=10000, check=10, dtype=np.float32,
          cw=32, gs=256, threads=True, CT=None):
    """Restated ``solve``. ``C`` (n, m) fp64 or already-cast; ``mu_w``/``nu_w``
    are normalised fp64 weights. Returns a dict with status, iterations,
    err, cost, trace, alpha, beta."""
    dt = np.dtype(dtype)
    C = np.ascontiguousarray(C, dtype=dt)
    if CT is None:
        CT = np.ascontiguousarray(C.T)
    else:
        CT = np.ascontiguousarray(CT, dtype=dt)
    mu_w = np.asarray(mu_w, np.float64)
    nu_w = np.asarray(nu_w, np.float64)
    log_mu = np.log(mu_w).astype(dt)
    log_nu = np.log(nu_w).astype(dt)
    mu_d = mu_w.astype(dt)
    inv_eps = dt.type(1.0) / dt.type(eps)
    neg_eps = -dt.type(eps)
    n, m = C.shape
    alpha = np.zeros(n, dt)
    beta = np.zeros(m, dt)
    trace = []
    status = STATUS_NOT_CONVERGED
    err = np.inf
    it = 0

    def finite():
        return bool(np.isfinite(alpha).all() and np.isfinite(beta).all())

    def merr():
        return marginal_err(C, mu_d, log_mu, log_nu, alpha, beta, inv_eps, cw, gs, threads)

    for k in range(1, max_iter + 1):
        alpha = row_update(C, beta, log_nu, inv_eps, neg_eps, cw, gs, threads)
        beta = row_update(CT, alpha, log_mu, inv_eps, neg_eps, cw, gs, threads)
        it = k
        if k % check == 0:
            if not finite():
                status, err = STATUS_NUMERICAL_FAILURE, np.nan
                break
            err = merr()
            trace.append((k, float(err)))
            if not np.isfinite(err):
                status = STATUS_NUMERICAL_FAILURE
                break
            if err < tol:
                status = STATUS_CONVERGED
                break
    else:
        if it % check != 0:
            if finite():
                err = merr()
                trace.append((it, float(err)))
                if not np.isfinite(err):
                    status = STATUS_NUMERICAL_FAILURE
                elif err < tol:
                    status = STATUS_CONVERGED
            else:
                status, err = STATUS_NUMERICAL_FAILURE, np.nan
    if status == STATUS_NUMERICAL_FAILURE:
        cost = np.nan
    else:
        cost = transport_cost_rows(C, log_mu, log_nu, alpha, beta, inv_eps, cw, gs, threads)
        if not np.isfinite(cost):
            status, cost = STATUS_NUMERICAL_FAILURE, np.nan
    return dict(status=status, iterations=it, err=float(err), cost=float(cost),
                trace=tuple(trace), alpha=alpha, beta=beta)


# ---------------------------------------------------------------------------
# inputs: distributions, costs, generators


def normalized_weights(raw):
    """types.py:208-240 without the validation: (weights, log_weights)."""
    w = np.asarray(raw, dtype=np.float64).reshape(-1)
    weights = w / w.sum()
    return weights, np.log(weights)


def sq_euclidean_cost(X, Y, block=1024):
    """costs.py:36-50: fp64 ``sum_k (x_k - y_k)^2``, coordinate order fixed."""
    X = np.asarray(X, np.float64)
    Y = np.asarray(Y, np.float64)
    if X.ndim == 1:
        X = X[:, None]
    if Y.ndim == 1:
        Y = Y[:, None]
    out = np.empty((X.shape[0], Y.shape[0]), np.float64)
    for r in range(0, X.shape[0], block):
        d = X[r:r + block, None, :] - Y[None, :, :]
        out[r:r + block] = (d * d).sum(axis=2)
    return out


def max_normalized(C64):
    """applications.py:186-188 (only when the range is non-zero)."""
    if float(C64.max() - C64.min()) > 0:
        return C64 / C64.max()
    return C64


def uniform_points(n, d, seed, count=2):
    """``count`` successive U[0,1]^(n x d) draws of one PCG64(seed) stream."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return [rng.uniform(0.0, 1.0, (n, d)) for _ in range(count)]


def grid_problem(n, m, seed):
    """costs.py:73-116 -> (mu_w, nu_w, C64)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    centers = rng.uniform(0.2, 0.8, 2)
    widths = rng.uniform(0.05, 0.1, 2)
    x = np.arange(n) / (n - 1) if n > 1 else np.zeros(1)
    y = np.arange(m) / (m - 1) if m > 1 else np.zeros(1)
    mu = np.exp(-0.5 * ((x - centers[0]) / widths[0]) ** 2) + 1e-4
    mu *= rng.uniform(0.5, 1.5, n)
    nu = np.exp(-0.5 * ((y - centers[1]) / widths[1]) ** 2) + 1e-4
    nu *= rng.uniform(0.5, 1.5, m)
    C = (x[:, None] - y[None, :]) ** 2
    cmax = C.max()
    if cmax > 0:
        C /= cmax
    return normalized_weights(mu)[0], normalized_weights(nu)[0], np.ascontiguousarray(C)


def rigid_pair(n, dimension, angle, translation, sigma, seed):
    """applications.py:215-247 -> (X, Y_shuffled, perm)."""
    c, s = np.cos(angle), np.sin(angle)
    if dimension == 2:
        Rm = np.array([[c, -s], [s, c]])
    else:
        Rm = np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])
    t = np.asarray(translation, dtype=np.float64).reshape(-1)
    rng = np.random.Generator(np.random.PCG64(seed))
    X = rng.uniform(0.0, 1.0, (n, dimension))
    Y = X @ Rm.T + t
    Y = Y + rng.normal(0.0, sigma, (n, dimension))
    perm = rng.permutation(n)
    out = np.empty_like(Y)
    out[perm] = Y
    return X, out, perm


def random_problem(n, m, seed):
    """Seeded ragged test problem: (C64 uniform[0,1), mu_w, nu_w, alpha, beta).

    Used by tests/golden/make_golden.py to feed the reference and by the
    tests to regenerate the very same inputs without storing them.
    """
    rng = np.random.default_rng(seed)
    C = rng.uniform(0, 1, (n, m))
    mu_w, _ = normalized_weights(rng.uniform(0.2, 1.0, n))
    nu_w, _ = normalized_weights(rng.uniform(0.2, 1.0, m))
    alpha = rng.uniform(-0.5, 0.5, n).astype(np.float32)
    beta = rng.uniform(-0.5, 0.5, m).astype(np.float32)
    return C, mu_w, nu_w, alpha, beta
