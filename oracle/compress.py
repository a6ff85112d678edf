"""HODLR partition, per-level truncated-SVD compression and rank bounds -- oracle
(test infrastructure only, see oracle/__init__.py).

* Partition: a node of size s splits into N1 = floor(s/2) (first)
  and N2 = ceil(s/2).  Reading R10: every node of a level is split
  while the largest node of that level exceeds the leaf size, so all leaves sit
  at the same depth L (identical to "split while s > leaf" whenever n/leaf is a
  power of two, i.e. every BASELINE config).
* "Compressed": drop the SVD components of an off-diagonal block whose
  singular value is below eps*||A||_2.  Reading R7: the threshold is applied to
  the blocks of T_{alpha,N} with tau = tol * 2^alpha (||T||_2 <= 2^alpha), so the
  diagonally scaled blocks of A_m carry an error <= tol * c * max(d) * 2^alpha.
* Only the lower block of T is dense at each node; the upper block holds the
  single entry -g_0, so T-tilde = T with every node's lower block
  replaced by its truncated SVD, and A-tilde = shift I + c (D+ T~ + D- T~^T).
* Bounds: Lemma 3.6  B(N, eps) = 2 + 2 ceil(2/pi^2 log(4N/pi) log(16/eps));
  Lemma 3.7 qsrank_eps(T) <= B(N, eps/2);  Cor. 3.8.
  "log" is the natural logarithm (reading R14).
"""
import math

import numpy as np

from .fd1d import toeplitz_T


def hodlr_levels(n: int, leaf: int):
    """Return [[(r0, n1, n2), ...] per level 0..L-1] for the uniform-depth partition."""
    if n < 1 or leaf < 2:
        # leaf >= 2 guarantees no empty node: ceil(n/2^(L-1)) >= 3 => floor(n/2^L) >= 1
        raise ValueError("need n >= 1 and leaf >= 2")
    levels = []
    nodes = [(0, n)]
    while max(s for _, s in nodes) > leaf:
        lvl, nxt = [], []
        for r0, s in nodes:
            n1 = s // 2
            n2 = s - n1
            lvl.append((r0, n1, n2))
            nxt.append((r0, n1))
            nxt.append((r0 + n1, n2))
        levels.append(lvl)
        nodes = nxt
    return levels


def hodlr_leaves(n: int, leaf: int):
    """Leaves (r0, size) of the uniform-depth partition."""
    nodes = [(0, n)]
    for lvl in hodlr_levels(n, leaf):
        nodes = []
        for r0, n1, n2 in lvl:
            nodes.append((r0, n1))
            nodes.append((r0 + n1, n2))
    return nodes


def truncate_svd(Y: np.ndarray, tau: float):
    """Truncated SVD keeping sigma >= tau.  Returns (U*S, V, rank)."""
    if Y.size == 0:
        return np.zeros((Y.shape[0], 0)), np.zeros((Y.shape[1], 0)), 0
    U, s, Vt = np.linalg.svd(Y, full_matrices=False)
    r = int(np.sum(s >= tau))
    return U[:, :r] * s[:r], Vt[:r].T, r


def level_ranks(alpha: float, n: int, leaf: int, tol: float):
    """Per-level max rank of the truncated lower T-blocks (tau = tol*2^alpha)."""
    T = toeplitz_T(alpha, n)
    tau = tol * 2.0 ** alpha
    ranks = []
    for lvl in hodlr_levels(n, leaf):
        rmax = 0
        for r0, n1, n2 in lvl:
            Y = T[r0 + n1:r0 + n1 + n2, r0:r0 + n1]
            rmax = max(rmax, truncate_svd(Y, tau)[2])
        ranks.append(rmax)
    return ranks


def compressed_T(alpha: float, n: int, leaf: int, tol: float) -> np.ndarray:
    """T-tilde: every node's lower block replaced by its truncated SVD."""
    T = toeplitz_T(alpha, n)
    Tt = T.copy()
    tau = tol * 2.0 ** alpha
    for lvl in hodlr_levels(n, leaf):
        for r0, n1, n2 in lvl:
            Y = T[r0 + n1:r0 + n1 + n2, r0:r0 + n1]
            US, V, _ = truncate_svd(Y, tau)
            Tt[r0 + n1:r0 + n1 + n2, r0:r0 + n1] = US @ V.T
    return Tt


def compressed_A(alpha, n, h, dt, d_plus, d_minus, leaf, tol, shift=1.0):
    """A-tilde = shift I + c (D+ T~ + D- T~^T): the matrix a HODLR solver inverts."""
    Tt = compressed_T(alpha, n, leaf, tol)
    c = dt / h ** alpha
    return shift * np.eye(n) + c * (np.asarray(d_plus)[:, None] * Tt
                                    + np.asarray(d_minus)[:, None] * Tt.T)


def bound_B(N: int, eps: float) -> int:
    """Beckermann–Townsend bound B(N, eps) of Lemma 3.6."""
    return 2 + 2 * math.ceil(2.0 / math.pi ** 2 * math.log(4.0 * N / math.pi)
                             * math.log(16.0 / eps))


def qsrank_bound_T(N: int, eps: float) -> int:
    """Lemma 3.7: qsrank_eps(T_{alpha,N}) <= B(N, eps/2)."""
    return bound_B(N, eps / 2.0)


def qsrank_bound_A(N: int, eps_hat: float) -> int:
    """Corollary 3.8: qsrank_eps(A_m) <= 1 + B(N, eps_hat/2)."""
    return 3 + 2 * math.ceil(2.0 / math.pi ** 2 * math.log(4.0 * N / math.pi)
                             * math.log(32.0 / eps_hat))
