"""Host-side behaviour of the drop-in API that needs no GPU: validation and
error types mirror the reference (types.py:154-166, 230-262,
solver.py:68-73), and compute entry points fail loudly without a device."""

import numpy as np
import pytest
import torch

import paper_2605_00837_b200 as lsk


def test_config_defaults_and_validation():
    c = lsk.SinkhornConfig(epsilon=0.1)
    assert (c.tolerance, c.max_iterations, c.check_interval, c.chunk_width, c.group_size) == (1e-6, 10000, 10, 32, 256)
    assert c.precision == "single" and c.dtype == np.float32 and not c.transpose_for_beta
    for bad in [dict(epsilon=0), dict(epsilon=0.1, tolerance=0), dict(epsilon=0.1, max_iterations=0),
                dict(epsilon=0.1, check_interval=0), dict(epsilon=0.1, precision="half"),
                dict(epsilon=0.1, chunk_width=3, group_size=256), dict(epsilon=0.1, chunk_width=0)]:
        with pytest.raises(ValueError):
            lsk.SinkhornConfig(**bad)


def test_distribution_validation():
    d = lsk.make_distribution([1, 3])
    np.testing.assert_allclose(d.weights, [0.25, 0.75])
    np.testing.assert_allclose(d.log_weights, np.log([0.25, 0.75]))
    with pytest.raises(lsk.EmptyInput):
        lsk.make_distribution([])
    with pytest.raises(lsk.NonFiniteInput):
        lsk.make_distribution([1, np.nan])
    with pytest.raises(lsk.ZeroWeight):
        lsk.make_distribution([1, 0])


def test_cost_matrix_validation():
    c = lsk.make_cost_matrix(2, 2, [0, 1, 1, 0])
    assert c.rows == 2 and c.cols == 2 and c.value_range == 1.0
    with pytest.raises(lsk.DimensionMismatch):
        lsk.make_cost_matrix(2, 2, [0, 1, 1])
    with pytest.raises(lsk.NegativeOrNonFiniteEntry):
        lsk.make_cost_matrix(1, 2, [0, -1])


def test_dimension_mismatch_before_any_device_work():
    mu = lsk.make_distribution([1.0, 1.0])
    nu = lsk.make_distribution([1.0, 1.0, 1.0])
    cost = lsk.make_cost_matrix(2, 2, [0.1] * 4)
    with pytest.raises(ValueError):
        lsk.solve(cost, mu, nu, lsk.SinkhornConfig(epsilon=0.1))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    mu = lsk.make_distribution([1.0, 1.0])
    cost = lsk.make_cost_matrix(2, 2, [0.0, 1.0, 1.0, 0.0])
    with pytest.raises(lsk.BackendError):
        lsk.solve(cost, mu, mu, lsk.SinkhornConfig(epsilon=0.1))
    with pytest.raises(lsk.BackendError):
        lsk.update_alpha(cost, mu, np.zeros(2, np.float32), 0.1)


def test_product_never_imports_oracle():
    import pathlib

    pkg = pathlib.Path(lsk.__file__).parent
    for p in pkg.rglob("*.py"):
        assert "oracle" not in p.read_text().replace("oracle/`", ""), p
