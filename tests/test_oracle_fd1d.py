"""Pins for oracle.fd1d (no GPU): worked matrices, FFT vs dense, closed forms,
M-matrix / diagonal-dominance invariants, the alpha = 2 limit against a
LAPACK banded solver, and trajectory special cases."""
import os

import numpy as np
import pytest
import scipy.linalg as sla

from oracle.gl import gl_weights
from oracle.fd1d import (toeplitz_T, assemble_A, step_dense, trajectory_dense,
                         toeplitz_matvec_fft, apply_A_fft, backward_error)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_small_T_golden():
    with open(os.path.join(GOLDEN, "toeplitz_small.txt")) as fh:
        rows = [l.split("#")[0].split() for l in fh if l.split("#")[0].strip()]
    for r in rows:
        alpha, n = float(r[0]), int(r[1])
        want = np.array([float(v) for v in r[2:]]).reshape(n, n)
        np.testing.assert_allclose(toeplitz_T(alpha, n), want, rtol=1e-15, atol=0)
    np.testing.assert_array_equal(toeplitz_T(2.0, 3) @ np.ones(3), [1, 0, 1])


@pytest.mark.parametrize("alpha", [1.3, 1.7, 2.0])
def test_T_structure(alpha):
    """Eq. (2.6): diagonal alpha, superdiagonal -1, zero above, -g_k below."""
    n = 40
    T = toeplitz_T(alpha, n)
    g = gl_weights(alpha, n + 1)
    assert np.all(np.diag(T) == alpha)
    assert np.all(np.diag(T, 1) == -1.0)
    assert np.all(np.triu(T, 2) == 0)
    for k in range(1, n):
        assert np.all(np.diag(T, -k) == -g[k + 1])


@pytest.mark.parametrize("alpha", [1.2, 1.5, 1.8])
def test_T_times_ones_closed_form(alpha):
    """(T 1)_i = -g^(a-1)_{i+1} (i < n-1), last = 1 - g^(a-1)_n (binomial partial sums)."""
    n = 300
    g1 = gl_weights(alpha - 1.0, n + 1)
    want = -g1[1:n + 1].copy()
    want[-1] += 1.0
    np.testing.assert_allclose(toeplitz_T(alpha, n) @ np.ones(n), want, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("n", [1, 2, 100, 257])
def test_fft_matvec_matches_dense(n):
    rng = np.random.default_rng(0)
    x = rng.standard_normal(n)
    T = toeplitz_T(1.6, n)
    for tr, M in ((False, T), (True, T.T)):
        y = toeplitz_matvec_fft(1.6, x, transpose=tr)
        assert np.linalg.norm(y - M @ x) <= 1e-12 * max(np.linalg.norm(M @ x), 1e-300)


@pytest.mark.parametrize("alpha", [1.2, 1.8])
def test_A_sdd_m_matrix(alpha):
    """A_m strictly diagonally dominant (margin >= 1), off-diagonal <= 0 => A^{-1} >= 0."""
    n = 256
    rng = np.random.default_rng(1)
    dp, dm = rng.uniform(0.0, 2.0, n), rng.uniform(0.0, 2.0, n)
    h, dt = 1.0 / (n + 1), 0.1
    A = assemble_A(alpha, n, h, dt, dp, dm)
    off = A - np.diag(np.diag(A))
    assert np.all(off <= 0)
    margin = np.diag(A) - np.abs(off).sum(1)
    assert margin.min() >= 1.0 - 1e-9
    Ai = np.linalg.inv(A)
    assert Ai.min() >= -1e-14 * np.abs(Ai).max()
    assert np.abs(Ai).sum(1).max() <= 1.0 + 1e-12


def test_alpha2_matches_banded_heat_equation():
    """alpha = 2: A = I + (dt/h^2) diag(d+ + d-) tridiag(-1,2,-1); LAPACK gbsv solve."""
    n, K = 128, 6
    h, dt = 1.0 / (n + 1), 1.0 / K
    x = h * np.arange(1, n + 1)
    rng = np.random.default_rng(3)
    u = x * (1 - x)
    for m in range(K):
        dp, dm = 1 + x * rng.uniform(), 1 + x ** 2 * rng.uniform()
        f = np.sin(np.pi * x) * (m + 1)
        A = assemble_A(2.0, n, h, dt, dp, dm)
        u_or, _ = step_dense(A, u, f, dt)
        s = dt / h ** 2 * (dp + dm)
        ab = np.zeros((3, n))
        ab[0, 1:] = -s[:-1]       # superdiagonal: row i, col i+1 -> -s[i]
        ab[1, :] = 1 + 2 * s
        ab[2, :-1] = -s[1:]       # subdiagonal: row i+1, col i -> -s[i+1]
        u_ref = sla.solve_banded((1, 1), ab, u + dt * f)
        assert np.linalg.norm(u_or - u_ref) <= 1e-12 * np.linalg.norm(u_ref)
        u = u_ref


def test_step_special_cases():
    n = 64
    h = 1.0 / (n + 1)
    rng = np.random.default_rng(4)
    u, f = rng.standard_normal(n), rng.standard_normal(n)
    dp, dm = rng.uniform(0.5, 2, n), rng.uniform(0.5, 2, n)
    # dt = 0 => A = I, u = u_prev
    got, _ = step_dense(assemble_A(1.5, n, h, 0.0, dp, dm), u, f, 0.0)
    np.testing.assert_array_equal(got, u)
    # d+- = 0 => u = u_prev + dt f
    got, _ = step_dense(assemble_A(1.5, n, h, 0.1, 0 * dp, 0 * dm), u, f, 0.1)
    np.testing.assert_allclose(got, u + 0.1 * f, rtol=1e-15)
    # f = 0, u0 = 0 => zero trajectory
    tr = trajectory_dense(1.5, n, h, 0.1, [dp] * 3, [dm] * 3, [0 * f] * 3, 0 * u)
    assert all(np.all(v == 0) for v in tr)


def test_maximum_principle_and_lu_reuse():
    n, K = 200, 5
    h, dt = 1.0 / (n + 1), 0.05
    x = h * np.arange(1, n + 1)
    dp, dm = 1 + x, 2 - x
    f = np.abs(np.sin(3 * np.pi * x))
    u0 = x * (1 - x)
    a = trajectory_dense(1.7, n, h, dt, [dp] * K, [dm] * K, [f] * K, u0, time_invariant=True)
    b = trajectory_dense(1.7, n, h, dt, [dp] * K, [dm] * K, [f] * K, u0, time_invariant=False)
    for ua, ub in zip(a, b):
        np.testing.assert_array_equal(ua, ub)          # LU reuse bitwise
        assert ua.min() >= -1e-8 * np.abs(ua).max()


@pytest.mark.parametrize("alpha", [1.3, 1.8])
def test_backward_error_of_dense_solve(alpha):
    n = 512
    h, dt = 1.0 / (n + 1), 1.0 / 32
    rng = np.random.default_rng(5)
    dp, dm = rng.uniform(0.5, 1.5, n), rng.uniform(0.5, 1.5, n)
    A = assemble_A(alpha, n, h, dt, dp, dm)
    b = rng.standard_normal(n)
    u = np.linalg.solve(A, b)
    np.testing.assert_allclose(apply_A_fft(alpha, h, dt, dp, dm, u), A @ u,
                               rtol=0, atol=1e-9 * np.abs(A @ u).max())
    be = backward_error(alpha, h, dt, dp, dm, u, b)
    assert be["eta"] < 1e-14
    # perturbing u by 1e-6 relative must be visible in eta
    be2 = backward_error(alpha, h, dt, dp, dm, u * (1 + 1e-6 * rng.standard_normal(n)), b)
    assert be2["eta"] > 1e-9
