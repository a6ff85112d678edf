"""Grünwald–Letnikov weights -- oracle (test infrastructure only, see oracle/__init__.py).

g_k^(alpha) = (-1)^k binom(alpha, k)
computed by the paper's recursion
    g_0 = 1,  g_1 = -alpha,  g_{k+1} = g_k (k - alpha)/(k + 1).

Pinned in tests/test_oracle_gl.py against: the worked values of SPEC S:60-62
(golden file), the product formula, the Gamma form,
positivity/monotonicity/decay, and the binomial partial-sum identity
sum_{k<=n} g_k^(a) = g_n^(a-1).
"""
import numpy as np


def gl_weights(alpha: float, n: int) -> np.ndarray:
    """Return g_0..g_n (length n+1) by the sequential recursion of P:1190-1193.

    Any real alpha is accepted here (the identity pins use alpha-1 in (0,1));
    the domain alpha in (1,2] is enforced at the C-ABI boundary.
    """
    if n < 0:
        raise ValueError("n must be >= 0")
    g = np.empty(n + 1, dtype=np.float64)
    g[0] = 1.0
    for k in range(n):
        # g_{k+1} = g_k * (k - alpha) / (k + 1); k=0 gives g_1 = -alpha
        g[k + 1] = g[k] * ((k - alpha) / (k + 1))
    return g
