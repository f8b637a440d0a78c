"""B200-native log-domain Sinkhorn (sm_100a CUDA behind a C ABI).

Drop-in for the solver path of the reference package ``logsinkhorn``:
``solve``, ``update_alpha``, ``update_beta``, ``marginal_error``,
``transport_cost``, ``materialize_plan`` and the value / error types, with
the same names, signatures and error behaviour. Kernels live in
``liblsk.so`` (``include/lsk.h``); there is no CPU fallback.
"""

from .applications import Correspondence, barycentric_map, match_point_clouds, match_point_clouds_with_report
from .color import RgbImage, color_transfer, color_transfer_with_report, generate_rigid_pair, make_rgb_image
from .costs import as_points, solve_points, squared_euclidean_cost
from .points import solve_points_batched, solve_points_otf
from .errors import (
    BackendError,
    DegenerateRange,
    DimensionMismatch,
    EmptyInput,
    EmptyView,
    FileFormatError,
    LogSinkhornError,
    NegativeOrNonFiniteEntry,
    NonFiniteInput,
    NonFiniteResult,
    ZeroRowMass,
    ZeroWeight,
)
from .solver import (
    marginal_error,
    materialize_plan,
    solve,
    to_device_cost,
    transport_cost,
    update_alpha,
    update_beta,
)
from .diagnostics import contraction_rate_bound, kkt_residual, regularized_objective
from .estimator import SinkhornTransport
from .fileio import read_correspondences, read_point_cloud, read_ppm, write_correspondences, write_point_cloud, write_ppm
from .problems import generate_grid_problem, normalize_cost
from .reduction import (
    log_sum_exp,
    log_sum_exp_cols,
    log_sum_exp_rows,
    reduce_max,
    reduce_max_cols,
    reduce_max_rows,
    reduce_sum,
    reduce_sum_cols,
    reduce_sum_rows,
)
from .standard import solve_standard_domain
from .types import (
    STATUS_CONVERGED,
    STATUS_NOT_CONVERGED,
    STATUS_NUMERICAL_FAILURE,
    CostMatrix,
    DeviceCostMatrix,
    DiscreteDistribution,
    DualPotentials,
    ReductionPlan,
    SinkhornConfig,
    SolveReport,
    TransportPlan,
    make_cost_matrix,
    make_distribution,
)

__version__ = "0.1.0"
