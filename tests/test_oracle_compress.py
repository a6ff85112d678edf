"""Pins for oracle.compress (no GPU): the partition, the exact block structure of
T used by every compression, the special case
alpha = 2 (ranks <= 1), the paper's rank bounds (Lemma 3.6/3.7, Cor. 3.8) and
the truncation-error bound of the compressed matrix."""
import os

import numpy as np
import pytest

from oracle.gl import gl_weights
from oracle.fd1d import toeplitz_T, assemble_A
from oracle.compress import (hodlr_levels, hodlr_leaves, level_ranks, compressed_T,
                             compressed_A, bound_B, qsrank_bound_T, qsrank_bound_A,
                             truncate_svd)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("n,leaf", [(256, 32), (1000, 64), (1001, 125), (7, 2), (5, 8), (3, 2), (4096, 64)])
def test_partition(n, leaf):
    levels = hodlr_levels(n, leaf)
    leaves = hodlr_leaves(n, leaf)
    assert len(leaves) == 2 ** len(levels)
    pos = 0
    for r0, s in leaves:
        assert r0 == pos and 1 <= s <= leaf or (n <= leaf and s == n)
        pos += s
    assert pos == n
    for lvl in levels:
        for r0, n1, n2 in lvl:
            assert n2 - n1 in (0, 1)          # N1 = floor, N2 = ceil
    if (n // leaf) & (n // leaf - 1) == 0 and n % leaf == 0:
        assert all(s == leaf for _, s in leaves)


@pytest.mark.parametrize("alpha", [1.3, 1.8])
def test_block_structure(alpha):
    """Lower node block = -H J with H = [g_{2+i+j}]; upper = single -g_0."""
    n = 256
    T = toeplitz_T(alpha, n)
    g = gl_weights(alpha, 2 * n + 2)
    for lvl in hodlr_levels(n, 16):
        for r0, n1, n2 in lvl:
            Y = T[r0 + n1:r0 + n1 + n2, r0:r0 + n1]
            i = np.arange(n2)[:, None]
            j = np.arange(n1)[None, :]
            H = g[2 + i + j]
            np.testing.assert_array_equal(Y, -H[:, ::-1])
            Up = T[r0:r0 + n1, r0 + n1:r0 + n1 + n2]
            assert np.count_nonzero(Up) == 1 and Up[n1 - 1, 0] == -1.0


def test_alpha2_ranks_at_most_one():
    assert max(level_ranks(2.0, 512, 32, 1e-12)) <= 1


def test_bound_golden():
    with open(os.path.join(GOLDEN, "rank_bounds.txt")) as fh:
        rows = [l.split("#")[0].split() for l in fh if l.split("#")[0].strip()]
    for kind, N, eps, val in rows:
        f = {"B": bound_B, "QT": qsrank_bound_T, "QA": qsrank_bound_A}[kind]
        assert f(int(N), float(eps)) == int(val)


@pytest.mark.parametrize("alpha", [1.3, 1.7])
@pytest.mark.parametrize("n", [512, 1024])
def test_measured_qsrank_within_bound(alpha, n):
    """Measured eps-qsrank of T (largest maximal lower block) <= B(N, eps/2) (Lemma 3.7)."""
    T = toeplitz_T(alpha, n)
    nrm = np.linalg.norm(T, 2)
    eps = 1e-8
    worst = 0
    for s in range(1, n):
        if s % 37 and s not in (n // 2, 1, n - 1):
            continue
        sv = np.linalg.svd(T[s:, :s], compute_uv=False)
        worst = max(worst, int(np.sum(sv > eps * nrm)))
    assert worst <= qsrank_bound_T(n, eps)
    assert abs(nrm - 2 ** alpha) <= 1e-3 * 2 ** alpha      # reading R7 (||T|| ~ 2^alpha)


def test_A_qsrank_bound():
    n, alpha = 512, 1.5
    h, dt = 1.0 / (n + 1), 0.1
    x = h * np.arange(1, n + 1)
    A = assemble_A(alpha, n, h, dt, 1 + x, 2 - x)
    nA = np.linalg.norm(A, 2)
    eps = 1e-8
    T = toeplitz_T(alpha, n)
    c = dt / h ** alpha
    eps_hat = nA / (np.linalg.norm(T, 2) * 2.0 * c) * eps
    s = n // 2
    sv = np.linalg.svd(A[s:, :s], compute_uv=False)
    assert int(np.sum(sv > eps * nA)) <= qsrank_bound_A(n, eps_hat)


@pytest.mark.parametrize("alpha,tol", [(1.5, 1e-12), (1.3, 1e-10), (1.9, 1e-8)])
def test_truncation_error_bound(alpha, tol):
    """Per level the truncated blocks are disjoint, each error < tau, so ||T - T~|| <= L tau."""
    n, leaf = 512, 32
    tau = tol * 2 ** alpha
    T = toeplitz_T(alpha, n)
    Tt = compressed_T(alpha, n, leaf, tol)
    L = len(hodlr_levels(n, leaf))
    assert np.linalg.norm(T - Tt, 2) <= L * tau
    # ranks are far below the bound and monotone non-increasing toward the leaves
    r = level_ranks(alpha, n, leaf, tol)
    assert all(a >= b for a, b in zip(r, r[1:]))
    assert max(r) <= qsrank_bound_T(n, tol)


def test_truncate_svd_special_cases():
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal((50, 1)), rng.standard_normal((40, 1))
    US, V, r = truncate_svd(a @ b.T + 0 * rng.standard_normal((50, 40)), 1e-10)
    assert r == 1
    Y = rng.standard_normal((60, 7)) @ rng.standard_normal((7, 45))
    US, V, r = truncate_svd(Y, 1e-9 * np.linalg.norm(Y, 2))
    assert r == 7 and np.linalg.norm(US @ V.T - Y) <= 1e-10 * np.linalg.norm(Y)


def test_compressed_solve_close_to_exact():
    n, alpha = 256, 1.5
    h, dt = 1.0 / (n + 1), 1.0 / 8
    x = h * np.arange(1, n + 1)
    dp, dm = np.ones(n), np.ones(n)
    A = assemble_A(alpha, n, h, dt, dp, dm)
    At = compressed_A(alpha, n, h, dt, dp, dm, 32, 1e-12)
    b = np.sin(np.pi * x)
    u, ut = np.linalg.solve(A, b), np.linalg.solve(At, b)
    assert np.linalg.norm(u - ut) <= 1e-10 * np.linalg.norm(u)
