"""Pins for oracle.gl (no GPU).  Each test fixes g by something other than the
recursion itself: worked values, exact rational arithmetic of the product
formula, the Gamma form, the paper's stated
properties and a binomial identity."""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle.gl import gl_weights

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_rows(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.split("#")[0].strip()
            if line:
                rows.append(line.split())
    return rows


def test_worked_values():
    for row in _golden_rows("gl_weights.txt"):
        alpha = float(row[0])
        want = np.array([float(v) for v in row[1:]])
        got = gl_weights(alpha, len(want) - 1)
        np.testing.assert_allclose(got, want, rtol=1e-15, atol=0)


@pytest.mark.parametrize("alpha", [1.1, 1.3, 1.5, 1.8, 1.9, 2.0])
def test_g0_g1_exact(alpha):
    g = gl_weights(alpha, 5)
    assert g[0] == 1.0 and g[1] == -alpha


@pytest.mark.parametrize("num,den", [(3, 2), (13, 10), (9, 5), (11, 10)])
def test_product_formula_exact_rational(num, den):
    """g_k = (-1)^k/k! * a(a-1)...(a-k+1) in exact rational arithmetic."""
    a = Fraction(num, den)
    g = gl_weights(num / den, 80)
    prod = Fraction(1)
    for k in range(81):
        exact = (-1) ** k * prod / math.factorial(k)
        assert abs(g[k] - float(exact)) <= 1e-14 * abs(float(exact)) + 1e-300
        prod *= (a - k)


@pytest.mark.parametrize("alpha", [1.2, 1.5, 1.8])
def test_gamma_form(alpha):
    """g_k = a(a-1) Gamma(k-a) / (Gamma(k+1) Gamma(2-a)), k >= 2."""
    g = gl_weights(alpha, 400)
    for k in range(2, 401):
        lg = (math.lgamma(k - alpha) - math.lgamma(k + 1) - math.lgamma(2 - alpha))
        want = alpha * (alpha - 1) * math.exp(lg)
        assert abs(g[k] - want) <= 1e-12 * want


@pytest.mark.parametrize("alpha", [1.1, 1.5, 1.9])
def test_positive_decreasing_and_decay(alpha):
    """g_0 > g_2 > g_3 > ... > 0 and g_k = O(k^{-alpha-1})."""
    g = gl_weights(alpha, 100000)
    assert g[0] > g[2]
    assert np.all(g[2:] > 0)
    assert np.all(np.diff(g[2:]) < 0)
    k = np.arange(100, 1001)
    slope = np.polyfit(np.log(k), np.log(g[k]), 1)[0]
    assert abs(slope + alpha + 1) < 0.1


@pytest.mark.parametrize("alpha", [1.2, 1.5, 1.8])
def test_partial_sum_identity(alpha):
    """sum_{k<=n} g_k^(a) = g_n^(a-1)  (Pascal: binom(a,k) = binom(a-1,k) + binom(a-1,k-1)).

    Makes "sum g_k = 0" (the (1-1)^a limit, BASELINE north_star) quantitative:
    the partial sums are negative and vanish like n^{-a} (reading R3)."""
    g = gl_weights(alpha, 3000)
    g1 = gl_weights(alpha - 1.0, 3000)
    s = np.cumsum(g)
    np.testing.assert_allclose(s, g1, rtol=1e-11, atol=1e-16)
    assert np.all(s[2:] < 0) and abs(s[-1]) < 3000.0 ** (-alpha + 0.9)


@pytest.mark.parametrize("alpha", [1.1, 1.5, 1.9])
def test_hankel_psd(alpha):
    """Lemma 3.4: H = [g_{i+j}]_{i,j>=1} is positive semidefinite."""
    n = 200
    g = gl_weights(alpha, 2 * n + 2)
    i = np.arange(1, n + 1)
    H = g[i[:, None] + i[None, :]]
    ev = np.linalg.eigvalsh(H)
    assert ev.min() >= -1e-10 * np.abs(ev).max()
