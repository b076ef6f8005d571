"""Oracle pinning: dense kernels. Ports proj/tests/test_kernels.cpp:68-120 and
acceptance c08 (proj/tests/acceptance.cpp:276-303)."""
import math

import numpy as np
import pytest


def rand_c(rng, n, m=None, scale=1.0):
    m = n if m is None else m
    return scale * (rng.uniform(-1, 1, (n, m)) + 1j * rng.uniform(-1, 1, (n, m)))


def test_solve_right_computes_B_Ainv(oracle):  # test_kernels.cpp:68-76
    rng = np.random.default_rng(19)
    for _ in range(10):
        A = rand_c(rng, 7) + 3.0 * np.eye(7)
        B = rand_c(rng, 7)
        X = oracle.solve_right(B, A)
        assert np.linalg.norm(X @ A - B) <= 1e-12 * np.linalg.norm(B)


def test_solve_right_rectangular_rhs(oracle):
    rng = np.random.default_rng(3)
    A = rand_c(rng, 9) + 3.0 * np.eye(9)
    B = rand_c(rng, 4, 9)
    X = oracle.solve_right(B, A)
    assert X.shape == (4, 9)
    assert np.linalg.norm(X - B @ np.linalg.inv(A)) <= 1e-12 * np.linalg.norm(X)


def test_solve_right_rejects_singular(oracle):  # test_kernels.cpp:78-84
    A = np.zeros((3, 3), complex)
    A[0, 0] = 1.0
    A[1, 1] = 1.0
    with pytest.raises(oracle.SingularMatrixError):
        oracle.solve_right(np.eye(3, dtype=complex), A)


def test_gershgorin_exact_on_diagonal(oracle):  # test_kernels.cpp:86-92
    Q = np.diag([4j, -2.0, -0.5j])
    assert oracle.gershgorin_cond(Q) == pytest.approx(8.0, rel=1e-14)


def test_gershgorin_overestimates_eigen_spread(oracle):  # test_kernels.cpp:94-114
    rng = np.random.default_rng(23)
    for _ in range(200):
        n = int(rng.integers(4, 17))
        Q = rand_c(rng, n)
        for i in range(n):
            r = np.abs(Q[i]).sum() - abs(Q[i, i])
            Q[i, i] = complex(r + 0.1 + abs(rng.uniform(-1, 1)), rng.uniform(-1, 1))
        xi = oracle.gershgorin_cond(Q)
        ev = np.abs(np.linalg.eigvals(Q))
        assert math.isfinite(xi)
        assert xi + 1e-12 >= ev.max() / ev.min()


def test_gershgorin_infinite_without_dominance(oracle):  # test_kernels.cpp:116-120
    Q = np.eye(2, dtype=complex)
    Q[0, 1] = 2.0
    assert math.isinf(oracle.gershgorin_cond(Q))


def test_acceptance_c08_gershgorin_1000(oracle):  # acceptance.cpp:276-303
    rng = np.random.default_rng(20260818)
    violations = 0
    for _ in range(1000):
        n = int(rng.integers(4, 33))
        Q = rand_c(rng, n)
        for r in range(n):
            radius = np.abs(Q[r]).sum() - abs(Q[r, r])
            Q[r, r] = (radius + 0.2 + 1.5 * rng.uniform()) * np.exp(1j * math.pi * rng.uniform(-1, 1))
        ev = np.abs(np.linalg.eigvals(Q))
        if not oracle.gershgorin_cond(Q) >= ev.max() / ev.min():
            violations += 1
    assert violations == 0
