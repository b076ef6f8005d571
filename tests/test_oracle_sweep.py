"""Oracle pinning: the sweep layer. Ports proj/tests/test_sweep.cpp:22-109 and
acceptance c09 (proj/tests/acceptance.cpp:308-319)."""
import numpy as np
import pytest

import fields


def opts(oracle, threads, method="sp4", dz=0.02):
    o = oracle.SweepOptions()
    o.method = method
    o.dz = dz
    o.threads = threads
    return o


def test_angle_grid_validation(oracle):  # :22-31
    AG = oracle.AngleGrid
    for t0, t1 in (([], [0.0]), ([1.0], []), ([1.0, 1.0], [0.0]), ([3.0, 2.0], [0.0]), ([0.0, 2.0], [0.0]),
                   ([89.0, 90.0], [0.0])):
        with pytest.raises(oracle.ConfigError):
            AG.validated(t0, t1)
    assert AG.validated([1.0, 2.0, 3.0], [0.0, 45.0]).rows() == 6


def test_row_order(oracle):  # :33-46
    grid = oracle.AngleGrid.validated([4.0, 8.0, 12.0], [0.0, 30.0])
    c = oracle.rocking_curve(fields.layered_field(oracle), fields.rods11(oracle), fields.K_GAMMA11, grid,
                             opts(oracle, 1))
    assert c.theta0 == [4.0, 8.0, 12.0] * 2
    assert c.theta1 == [0.0] * 3 + [30.0] * 3
    assert c.method == "sp4" and c.solve_seconds > 0


def test_thread_count_bitwise(oracle):  # :48-61
    grid = oracle.AngleGrid.validated([2.0, 5.0, 8.0, 11.0, 14.0, 17.0, 20.0], [0.0])
    args = (fields.layered_field(oracle), fields.rods11(oracle), fields.K_GAMMA11, grid)
    one = oracle.rocking_curve(*args, opts(oracle, 1)).eta
    for t in (4, 8, 0):
        assert np.array_equal(one, oracle.rocking_curve(*args, opts(oracle, t)).eta)


def test_table_budget_bitwise(oracle):  # :63-73
    grid = oracle.AngleGrid.validated([3.0, 6.0, 9.0], [0.0])
    args = (fields.layered_field(oracle), fields.rods11(oracle), fields.K_GAMMA11, grid)
    without = opts(oracle, 2)
    without.table_budget_bytes = 0
    assert np.array_equal(oracle.rocking_curve(*args, opts(oracle, 2)).eta, oracle.rocking_curve(*args, without).eta)


def test_worker_failure_surfaces(oracle):  # :90-105
    o = opts(oracle, 4, "sp6", 0.02)
    o.rhst_threshold = float("inf")
    layers = [(-1.0 - 2.0 * i, -0.22, 2.2, 0.7, 0.08) for i in range(75)]
    field = oracle.PotentialField.gaussian_layers(-150.0, layers)
    grid = oracle.AngleGrid.validated([3.0, 5.0, 7.0, 9.0], [0.0])
    with pytest.raises(oracle.SolverError):
        oracle.rocking_curve(field, fields.rods11(oracle), fields.K_GAMMA11, grid, o)


def test_unknown_method(oracle):  # :107-114
    with pytest.raises(oracle.ConfigError):
        oracle.rocking_curve(fields.layered_field(oracle), fields.rods11(oracle), fields.K_GAMMA11,
                             oracle.AngleGrid.validated([5.0], [0.0]), opts(oracle, 1, "sp8"))


def test_acceptance_c09_flux_bound(oracle):  # acceptance.cpp:308-319
    grid = oracle.AngleGrid.validated([float(t) for t in range(1, 70)], [0.0])
    c = oracle.rocking_curve(fields.layered_field(oracle), fields.rods11(oracle), fields.K_GAMMA11, grid,
                             opts(oracle, 4))
    assert c.eta.sum(axis=1).max() <= 1.0 + 1e-8


def test_curve_error_semantics(oracle):  # curve.cpp:22-41 via test_curve_csv.cpp:53-83
    grid = oracle.AngleGrid.validated([3.0, 6.0], [0.0])
    args = (fields.layered_field(oracle), fields.rods11(oracle), fields.K_GAMMA11, grid)
    a = oracle.rocking_curve(*args, opts(oracle, 1))
    assert oracle.curve_error(a, a) == 0.0
    b = oracle.rocking_curve(*args, opts(oracle, 1, "sp6"))
    e = oracle.curve_error(b, a)
    assert 0 < e < 1e-3
    other = oracle.rocking_curve(fields.layered_field(oracle), fields.rods11(oracle), fields.K_GAMMA11,
                                 oracle.AngleGrid.validated([3.0, 7.0], [0.0]), opts(oracle, 1))
    with pytest.raises(oracle.CompareError):
        oracle.curve_error(other, a)
