"""Scikit-learn style estimator on the B200 path.

``SinkhornTransport`` mirrors the reference estimator (``estimator.py:21-132``):
same hyperparameters, fitted attributes and transform rule. ``fit`` builds the
fp64 squared-Euclidean cost on the device (optionally divided by its maximum
when the range is non-zero), solves in double precision (``solver64``),
materialises ``plan_`` and maps the fitted sources barycentrically
(``lsk_barycentric_plan_f64``); ``transform`` moves every point with its
nearest fitted source point, ties to the lowest index
(``lsk_nearest_map_f64``). Validation goes through scikit-learn's
``check_array`` / ``check_is_fitted`` as in the reference.
"""

import numpy as np
from sklearn.base import BaseEstimator, TransformerMixin
from sklearn.utils.validation import check_array, check_is_fitted

from . import _lib
from . import solver64
from .errors import NonFiniteResult, ZeroRowMass
from .solver import _ptr, _stream_ptr, _torch
from .types import STATUS_NUMERICAL_FAILURE, SinkhornConfig, make_distribution

__all__ = ["SinkhornTransport"]


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")


class SinkhornTransport(TransformerMixin, BaseEstimator):
    """Entropic OT from a source sample to a target sample as a transformer
    (uniform weights, squared Euclidean cost, double-precision solve).

    Parameters: ``epsilon`` (0.01), ``tolerance`` (1e-6), ``max_iterations``
    (10000), ``check_interval`` (10), ``normalize_cost`` (True: divide the
    cost by its maximum when the range is non-zero).

    Fitted attributes: ``source_``, ``target_``, ``plan_`` (n, m),
    ``report_``, ``alpha_``, ``beta_``, ``n_features_in_``.
    """

    def __init__(self, epsilon=0.01, tolerance=1e-6, max_iterations=10000, check_interval=10,
                 normalize_cost=True):
        self.epsilon = epsilon
        self.tolerance = tolerance
        self.max_iterations = max_iterations
        self.check_interval = check_interval
        self.normalize_cost = normalize_cost

    def fit(self, X, y):
        """Solve transport from source sample X to target sample y."""
        X = check_array(X, dtype=np.float64)
        y = check_array(y, dtype=np.float64)
        if X.shape[1] != y.shape[1]:
            raise ValueError(f"source and target dimensions differ: {X.shape[1]} vs {y.shape[1]}")
        torch = _torch()
        st = _stream_ptr(torch)
        n, m, d = X.shape[0], y.shape[0], X.shape[1]
        Xd, Yd = _dev(torch, X), _dev(torch, y)
        C = torch.empty((n, m), dtype=torch.float64, device="cuda")
        ws = torch.empty(_lib.load().lsk_build_cost_workspace_bytes(), dtype=torch.uint8, device="cuda")
        cmax = torch.zeros(1, dtype=torch.float64, device="cuda")
        norm = 1 if self.normalize_cost else 0
        _lib.call("lsk_build_cost_f64", _ptr(Xd), _ptr(Yd), n, m, d, norm, _ptr(C), m, _ptr(cmax), _ptr(ws),
                  ws.numel(), st)
        mu = make_distribution(np.ones(n))
        nu = make_distribution(np.ones(m))
        config = SinkhornConfig(epsilon=self.epsilon, tolerance=self.tolerance, max_iterations=self.max_iterations,
                                check_interval=self.check_interval, precision="double")
        report, pot = solver64.solve(C, mu, nu, config, return_device=True)
        if report.status == STATUS_NUMERICAL_FAILURE:
            raise NonFiniteResult(f"transport solve failed numerically at epsilon={self.epsilon}")
        plan = solver64.materialize_plan(C, mu, nu, pot.alpha, pot.beta, self.epsilon, return_device=True)
        mapped = torch.empty((n, d), dtype=torch.float64, device="cuda")
        flags = torch.zeros(2, dtype=torch.int32, device="cuda")
        for k0 in range(0, d, 4):  # the barycentric kernel maps up to 4 coordinates per pass
            dt = min(4, d - k0)
            Yk = Yd[:, k0:k0 + dt].contiguous()
            mk = torch.empty((n, dt), dtype=torch.float64, device="cuda")
            _lib.call("lsk_barycentric_plan_f64", _ptr(plan.values), m, n, m, _ptr(Yk), dt, _ptr(mk), _ptr(flags), st)
            mapped[:, k0:k0 + dt] = mk
        if int(flags[1].item()):
            raise ZeroRowMass("a transport plan row has zero total mass")
        self.source_ = X
        self.target_ = y
        self.plan_ = plan.values.cpu().numpy()
        self.alpha_ = pot.alpha.cpu().numpy()
        self.beta_ = pot.beta.cpu().numpy()
        self.report_ = report
        self.n_features_in_ = d
        self._source_dev = Xd
        self._mapped_sources = mapped
        return self

    def transform(self, X):
        """Map points into the target domain through the fitted plan."""
        check_is_fitted(self, "plan_")
        X = check_array(X, dtype=np.float64)
        if X.shape[1] != self.n_features_in_:
            raise ValueError(f"expected {self.n_features_in_} features, got {X.shape[1]}")
        torch = _torch()
        Q = _dev(torch, X)
        out = torch.empty_like(Q)
        _lib.call("lsk_nearest_map_f64", _ptr(Q), X.shape[0], X.shape[1], _ptr(self._source_dev),
                  self.source_.shape[0], _ptr(self._mapped_sources), X.shape[1], 0, _ptr(out), None,
                  _stream_ptr(torch))
        return out.cpu().numpy()
