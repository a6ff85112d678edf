"""2D FDE time step as a Sylvester equation -- oracle
(test infrastructure only, see oracle/__init__.py).

Eq. (4.3), with the 1D operators of Eq. (2.5) split as 1/2 I:
    A_1 U^(m+1) + U^(m+1) A_2^T = U^(m) + dt F^(m+1),
    A_i = 1/2 I + (dt/h_i^alpha_i)(D_{i,+} T_{alpha_i} + D_{i,-} T_{alpha_i}^T).
Reading R11: the right-hand side carries dt (consistent with Eq. 2.5;
the paper's runs have dt = 1).  Reading R12: the 1/2 split is as written.

Solved densely by Bartels–Stewart (real Schur of A_1 and A_2^T once, LAPACK
trsyl per step) and, for n <= 64, by the Kronecker system
    (I kron A_1 + A_2 kron I) vec(X) = vec(C)     (vec(AXB) = (B^T kron A) vec X).
"""
import numpy as np
import scipy.linalg as sla

from .fd1d import assemble_A


def operators_2d(alpha1, alpha2, nx, ny, hx, hy, dt, d1p, d1m, d2p, d2m):
    A1 = assemble_A(alpha1, nx, hx, dt, d1p, d1m, shift=0.5)
    A2 = assemble_A(alpha2, ny, hy, dt, d2p, d2m, shift=0.5)
    return A1, A2


class BartelsStewart:
    """Solve A1 X + X A2^T = C for many C with one pair of real Schur forms."""

    def __init__(self, A1, A2):
        self.T1, self.Q1 = sla.schur(A1, output="real")
        self.T2, self.Q2 = sla.schur(A2.T, output="real")
        self.trsyl = sla.get_lapack_funcs("trsyl", (self.T1,))

    def solve(self, C):
        Ct = self.Q1.T @ C @ self.Q2
        Y, scale, info = self.trsyl(self.T1, self.T2, Ct)
        if info < 0:
            raise RuntimeError("trsyl failed: info=%d" % info)
        return self.Q1 @ (Y / scale) @ self.Q2.T


def solve_kron(A1, A2, C):
    """Kronecker-system solve (n <= 64) of A1 X + X A2^T = C."""
    nx, ny = C.shape
    K = np.kron(np.eye(ny), A1) + np.kron(A2, np.eye(nx))
    x = np.linalg.solve(K, C.reshape(-1, order="F"))
    return x.reshape((nx, ny), order="F")


def step_2d_dense(bs: BartelsStewart, U_prev, F_next, dt):
    """One step of Eq. (4.3): returns U^(m+1)."""
    return bs.solve(np.asarray(U_prev) + dt * np.asarray(F_next))
