"""Dense 1D finite-difference operator and implicit-Euler step -- oracle
(test infrastructure only, see oracle/__init__.py).

Definitions followed:
  * T_{alpha,N} = -[g_{i-j+1}]  (lower Hessenberg Toeplitz, Eq. 2.6):
        T[i, j] = -g[i - j + 1]  if i - j + 1 >= 0, else 0.
  * A_m = I + (dt / h^alpha) (D_+ T + D_- T^T)            (Eq. 2.5)
    generalised to  shift * I + ...  so the 2D operators 1/2 I + ... (Eq. 4.3,
    P:1497-1500) use the same routine.
  * one implicit-Euler step  A_m u^(m) = u^(m-1) + dt f^(m)
    solved by LAPACK LU (scipy lu_factor / lu_solve), the LU reused when A_m
    does not change.
  * large-n residuals by circulant embedding of size 2N (
    SPEC S:103): the 2N circulant whose first column is
        [t_0, t_1, ..., t_{N-1}, 0, r_{N-1}, ..., r_1]
    with t = first column of T, r = first row of T, has T as its leading block.
  * backward error  eta = ||A u - b|| / (||A|| ||u|| + ||b||)  with the bound
    ||A_m||_2 <= |shift| + c 2^alpha (max d_+ + max d_-)  (reading R7:
    ||T||_2 <= sup |1 - e^{i theta}|^alpha = 2^alpha).
"""
import numpy as np
import scipy.linalg as sla

from .gl import gl_weights


def toeplitz_T(alpha: float, n: int) -> np.ndarray:
    """Dense T_{alpha,n} of Eq. (2.6), entry by entry."""
    g = gl_weights(alpha, n + 1)
    i = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    k = i - j + 1                                  # T[i, j] = -g[i - j + 1]
    return np.where(k >= 0, -g[np.clip(k, 0, n)], 0.0)


def assemble_A(alpha, n, h, dt, d_plus, d_minus, shift=1.0):
    """Dense A = shift*I + (dt/h^alpha)(D_+ T + D_- T^T)  (Eq. 2.5)."""
    d_plus = np.asarray(d_plus, dtype=np.float64)
    d_minus = np.asarray(d_minus, dtype=np.float64)
    T = toeplitz_T(alpha, n)
    c = dt / h ** alpha
    return shift * np.eye(n) + c * (d_plus[:, None] * T + d_minus[:, None] * T.T)


def step_dense(A, u_prev, f, dt, lu=None):
    """u^(m) = A_m^{-1}(u^(m-1) + dt f^(m)) by LAPACK LU.

    Returns (u, lu) so a caller with time-invariant A_m reuses the LU.
    """
    if lu is None:
        lu = sla.lu_factor(A)
    b = np.asarray(u_prev, dtype=np.float64) + dt * np.asarray(f, dtype=np.float64)
    return sla.lu_solve(lu, b), lu


def trajectory_dense(alpha, n, h, dt, d_plus_steps, d_minus_steps, f_steps, u0,
                     time_invariant=False, shift=1.0):
    """Run K implicit-Euler steps densely.  *_steps[m-1] are samples at t_m."""
    u = np.asarray(u0, dtype=np.float64).copy()
    out = []
    lu = None
    for m in range(len(f_steps)):
        if lu is None or not time_invariant:
            A = assemble_A(alpha, n, h, dt, d_plus_steps[m], d_minus_steps[m], shift)
            lu = None
        u, lu = step_dense(A, u, f_steps[m], dt, lu)
        out.append(u.copy())
    return out


def _first_col_row(alpha, n):
    g = gl_weights(alpha, n + 1)
    col = -g[1:n + 1].copy()                 # T[i,0] = -g[i+1]
    row = np.zeros(n, dtype=np.float64)      # T[0,j] = -g[1-j]
    row[0] = -g[1]
    if n > 1:
        row[1] = -g[0]
    return col, row


def toeplitz_matvec_fft(alpha, x, transpose=False):
    """T x (or T^T x) by 2N circulant embedding and the FFT."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[0]
    col, row = _first_col_row(alpha, n)
    if transpose:
        col, row = row, col
    emb = np.concatenate([col, [0.0], row[1:][::-1]])
    y = np.fft.ifft(np.fft.fft(emb) * np.fft.fft(np.concatenate([x, np.zeros(n)])))
    return y[:n].real


def apply_A_fft(alpha, h, dt, d_plus, d_minus, u, shift=1.0):
    """A_m u without forming A_m (P:215 with FFT matvecs)."""
    c = dt / h ** alpha
    return shift * u + c * (np.asarray(d_plus) * toeplitz_matvec_fft(alpha, u)
                            + np.asarray(d_minus) * toeplitz_matvec_fft(alpha, u, True))


def norm_A_bound(alpha, h, dt, d_plus, d_minus, shift=1.0):
    """Upper bound |shift| + c 2^alpha (max|d+| + max|d-|) on ||A_m||_2 (reading R7)."""
    c = dt / h ** alpha
    return abs(shift) + c * 2.0 ** alpha * (np.max(np.abs(d_plus)) + np.max(np.abs(d_minus)))


def backward_error(alpha, h, dt, d_plus, d_minus, u, b, shift=1.0):
    """Return dict with eta, ||r||/||b|| and the paper's ||r||/||u||."""
    r = apply_A_fft(alpha, h, dt, d_plus, d_minus, u, shift) - b
    nr, nu, nb = np.linalg.norm(r), np.linalg.norm(u), np.linalg.norm(b)
    nA = norm_A_bound(alpha, h, dt, d_plus, d_minus, shift)
    return {"eta": nr / (nA * nu + nb) if (nA * nu + nb) > 0 else 0.0,
            "res_b": nr / nb if nb > 0 else nr,
            "res_u": nr / nu if nu > 0 else nr}
