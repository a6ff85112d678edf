"""Pins for oracle.sylvester2d (no GPU): special cases with closed-form answers,
Kronecker brute force vs Bartels–Stewart, and the x<->y symmetry of the scheme."""
import numpy as np
import pytest

from oracle.sylvester2d import operators_2d, BartelsStewart, solve_kron, step_2d_dense


def _ops(n, a1, a2, dt):
    h = 1.0 / (n + 1)
    x = h * np.arange(1, n + 1)
    return operators_2d(a1, a2, n, n, h, h, dt, 1 + x, 2 - x, 1 + x ** 2, 2 - x ** 2), x


def test_half_identity_gives_rhs():
    """dt = 0 => A1 = A2 = I/2 => X = C."""
    (A1, A2), _ = _ops(32, 1.3, 1.7, 0.0)
    C = np.random.default_rng(0).standard_normal((32, 32))
    np.testing.assert_allclose(BartelsStewart(A1, A2).solve(C), C, rtol=1e-13, atol=1e-13)


def test_zero_rhs():
    (A1, A2), _ = _ops(24, 1.3, 1.7, 0.1)
    assert np.all(BartelsStewart(A1, A2).solve(np.zeros((24, 24))) == 0)


@pytest.mark.parametrize("a1,a2", [(1.3, 1.7), (1.7, 1.9), (2.0, 2.0)])
def test_kron_vs_bartels_stewart(a1, a2):
    (A1, A2), x = _ops(32, a1, a2, 1.0 / 16)
    C = np.outer(np.sin(np.pi * x), x * (1 - x)) + np.outer(x, np.cos(x))
    Xk = solve_kron(A1, A2, C)
    Xb = BartelsStewart(A1, A2).solve(C)
    assert np.linalg.norm(Xk - Xb) <= 1e-10 * np.linalg.norm(Xk)
    # the residual of Eq. (4.3) itself
    assert np.linalg.norm(A1 @ Xk + Xk @ A2.T - C) <= 1e-11 * np.linalg.norm(C)


def test_symmetry():
    """alpha1 = alpha2, same coefficients, symmetric C => X = X^T."""
    n = 40
    h = 1.0 / (n + 1)
    x = h * np.arange(1, n + 1)
    A1, A2 = operators_2d(1.5, 1.5, n, n, h, h, 0.1, 1 + x, 2 - x, 1 + x, 2 - x)
    C = np.outer(np.sin(np.pi * x), np.sin(np.pi * x)) + np.outer(x, x)
    X = step_2d_dense(BartelsStewart(A1, A2), np.zeros((n, n)), C, 1.0)
    assert np.linalg.norm(X - X.T) <= 1e-12 * np.linalg.norm(X)


def test_split_independence():
    """The 1/2 split of I does not change X: (I + dt F1) X + X (dt F2)^T = C."""
    (A1, A2), x = _ops(20, 1.4, 1.6, 0.2)
    C = np.outer(x, 1 - x)
    X = solve_kron(A1, A2, C)
    X2 = solve_kron(A1 + 0.5 * np.eye(20), A2 - 0.5 * np.eye(20), C)
    assert np.linalg.norm(X - X2) <= 1e-11 * np.linalg.norm(X)
