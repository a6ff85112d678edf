"""Pin of the oracle's operator against the paper's shifted Grunwald-Letnikov scheme, written
out row by row (no GPU).

PAPER.md P:205-211 (Sec. 2.1.1) states the scheme before its matrix form (Eq. 2.5):

    (u_i^(m) - u_i^(m-1)) / dt = d+_i / h^a  sum_{k=0}^{i+1}   g_k u_{i-k+1}^(m)
                               + d-_i / h^a  sum_{k=0}^{N-i+2} g_k u_{i+k-1}^(m) + f_i^(m),

i = 1..N, with u_0 = u_{N+1} = 0 (absorbing boundary: u vanishes outside (L, R)).
So (A u)_i = u_i - (dt/h^a) (d+_i S+_i + d-_i S-_i).  Here S+- are evaluated with explicit loops
and the g_k come from the product formula g_k = prod_{j=1..k} (1 - (a+1)/j), not from
the oracle's recursion or its Toeplitz matrix, so a swapped D+/D- placement, a transposed T, a
wrong power of h or an off-by-one shift of the stencil in oracle.fd1d fails here.  alpha != 2 and
d+ != d- are essential: at alpha = 2 T is symmetric and h^alpha = h^2.
"""
import numpy as np
import pytest

from oracle.fd1d import assemble_A, apply_A_fft


def _g_product(alpha, K):
    """g_0..g_K by the product formula g_k = prod_{j=1}^{k} (1 - (alpha + 1)/j)."""
    g = [1.0]
    for k in range(1, K + 1):
        g.append(g[-1] * (1.0 - (alpha + 1.0) / k))
    return g


def _scheme_apply(alpha, h, dt, dp, dm, u):
    """(A u)_i from the scheme of P:205-211 with explicit loops (u_0 = u_{N+1} = 0)."""
    N = len(u)
    g = _g_product(alpha, N + 2)
    ue = [0.0] + list(u) + [0.0]                 # ue[i] = u_i, i = 0..N+1
    out = np.empty(N)
    for i in range(1, N + 1):
        sp = 0.0
        for k in range(0, i + 2):                # sum_{k=0}^{i+1} g_k u_{i-k+1}
            sp += g[k] * ue[i - k + 1]
        sm = 0.0
        for k in range(0, N - i + 3):            # sum_{k=0}^{N-i+2} g_k u_{i+k-1}
            sm += g[k] * ue[i + k - 1]
        out[i - 1] = u[i - 1] - dt / h ** alpha * (dp[i - 1] * sp + dm[i - 1] * sm)
    return out


@pytest.mark.parametrize("alpha", [1.3, 1.8])
@pytest.mark.parametrize("n", [7, 64])
def test_assemble_A_matches_scheme_rows(alpha, n):
    rng = np.random.default_rng(11 + n)
    h, dt = 1.0 / (n + 1), 0.37
    dp = rng.uniform(0.2, 1.0, n)                # d+ and d- clearly different
    dm = rng.uniform(1.5, 3.0, n)
    u = rng.standard_normal(n)
    want = _scheme_apply(alpha, h, dt, dp, dm, u)
    A = assemble_A(alpha, n, h, dt, dp, dm)
    scale = np.abs(want).max()
    np.testing.assert_allclose(A @ u, want, rtol=0, atol=1e-13 * scale)
    np.testing.assert_allclose(apply_A_fft(alpha, h, dt, dp, dm, u), want, rtol=0, atol=1e-12 * scale)


@pytest.mark.parametrize("alpha", [1.3, 1.8])
def test_scheme_pin_detects_plausible_mistakes(alpha):
    """The pin itself separates the mistakes it is meant to catch (a D+/D- swap, h^2 for h^alpha)."""
    n = 16
    rng = np.random.default_rng(5)
    h, dt = 1.0 / (n + 1), 0.37
    dp, dm = rng.uniform(0.2, 1.0, n), rng.uniform(1.5, 3.0, n)
    u = rng.standard_normal(n)
    want = _scheme_apply(alpha, h, dt, dp, dm, u)
    swapped = assemble_A(alpha, n, h, dt, dm, dp) @ u
    wrong_h = assemble_A(alpha, n, h, dt * h ** alpha / h ** 2, dp, dm) @ u
    for bad in (swapped, wrong_h):
        assert np.abs(bad - want).max() > 1e-3 * np.abs(want).max()


def test_scheme_columns_are_T_entries():
    """Single columns: A e_j has entries -c d+_i g_{i-j+1} - c d-_i g_{j-i+1} off the identity
    (the two sums of P:205-211 pick exactly one k each)."""
    n, alpha = 9, 1.55
    h, dt = 1.0 / (n + 1), 0.5
    rng = np.random.default_rng(2)
    dp, dm = rng.uniform(0.1, 1, n), rng.uniform(2, 3, n)
    A = assemble_A(alpha, n, h, dt, dp, dm)
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        np.testing.assert_allclose(A[:, j], _scheme_apply(alpha, h, dt, dp, dm, e), rtol=1e-14, atol=1e-14)
