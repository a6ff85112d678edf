"""Seeded synthetic inputs for the BASELINE.json configs.

This module holds NO arithmetic of the method: it only samples coefficient and
source functions on the grid x_i = i h (i = 1..n), t_m = m dt (m = 1..K)
(reading R4/R5/R6 in DESIGN.md) with numpy's PCG64 ``default_rng(seed)`` in a
fixed draw order.  Both the oracle tests and the CUDA path consume exactly
these arrays, so both sides see the same bits.

The paper's own workloads are formulas, not datasets: 1D §3.6 and 2D
§5.1.  The configs below are BASELINE.json's synthetic stand-ins
with the paper's shapes (alpha in (1,2), smooth power-law / sinusoidal
diffusion coefficients, smooth sine-series sources, N a power of two).
"""
from dataclasses import dataclass, field
import math

import numpy as np


@dataclass
class Workload1D:
    name: str
    batch: int
    n: int
    h: float
    alpha: np.ndarray          # (batch,)
    K: int                     # number of implicit-Euler steps
    dt: float
    leaf: int
    tol: float
    time_invariant: bool
    u0: np.ndarray             # (batch, n)
    d_plus: np.ndarray         # (K or 1, batch, n): samples at t_m, m = 1..K
    d_minus: np.ndarray        # (K or 1, batch, n)
    f: np.ndarray              # (K or 1, batch, n)
    x: np.ndarray = field(default=None)

    def coeffs(self, m):
        """(d_plus, d_minus) at t_m, m = 1..K, shape (batch, n)."""
        i = 0 if self.d_plus.shape[0] == 1 else m - 1
        return self.d_plus[i], self.d_minus[i]

    def source(self, m):
        i = 0 if self.f.shape[0] == 1 else m - 1
        return self.f[i]


def _sine_series(x, coef):
    """sum_j coef[j-1] sin(j pi x) for j = 1..len(coef); x (n,), coef (..., J)."""
    j = np.arange(1, coef.shape[-1] + 1)
    return np.asarray(coef) @ np.sin(np.pi * j[:, None] * x[None, :])


def cfg1():
    """n=256, alpha=1.5, 8 steps, d+-=1, u0=x^2(1-x)^2, f=(1+t) sum_8 c_j sin(j pi x)."""
    n, K = 256, 8
    h, dt = 1.0 / (n + 1), 1.0 / K
    x = h * np.arange(1, n + 1)
    c = np.random.default_rng(1).standard_normal(8)
    base = _sine_series(x, c)
    t = dt * np.arange(1, K + 1)
    f = np.stack([(1.0 + tm) * base for tm in t])[:, None, :]
    ones = np.ones((1, 1, n))
    return Workload1D("cfg1", 1, n, h, np.array([1.5]), K, dt, 32, 1e-12, True,
                      (x ** 2 * (1 - x) ** 2)[None, :], ones, ones.copy(), f, x)


def cfg2(K=64):
    """n=4096, alpha=1.3, 64 steps, d+ = G(3-a)(1+x)^a(1+t/2), d- = G(3-a)(2-x)^a(1+t/2)."""
    n, alpha = 4096, 1.3
    h, dt = 1.0 / (n + 1), 1.0 / 64
    x = h * np.arange(1, n + 1)
    c = np.random.default_rng(2).standard_normal(16)
    base = _sine_series(x, c)
    t = dt * np.arange(1, K + 1)
    g = math.gamma(3.0 - alpha)
    dp = np.stack([g * (1 + x) ** alpha * (1 + 0.5 * tm) for tm in t])[:, None, :]
    dm = np.stack([g * (2 - x) ** alpha * (1 + 0.5 * tm) for tm in t])[:, None, :]
    f = np.stack([math.exp(-tm) * base for tm in t])[:, None, :]
    return Workload1D("cfg2", 1, n, h, np.array([alpha]), K, dt, 64, 1e-12, False,
                      np.zeros((1, n)), dp, dm, f, x)


def cfg3(K=32, n=65536):
    """n=65536, alpha=1.8, 32 steps, d+ = 1+sin(2 pi x)cos(t)/2, d- = 1+cos(2 pi x)sin(t)/2."""
    alpha = 1.8
    h, dt = 1.0 / (n + 1), 1.0 / 32
    x = h * np.arange(1, n + 1)
    c = np.random.default_rng(3).standard_normal(32)
    base = _sine_series(x, c)
    t = dt * np.arange(1, K + 1)
    dp = np.stack([1 + 0.5 * np.sin(2 * np.pi * x) * math.cos(tm) for tm in t])[:, None, :]
    dm = np.stack([1 + 0.5 * np.cos(2 * np.pi * x) * math.sin(tm) for tm in t])[:, None, :]
    return Workload1D("cfg3", 1, n, h, np.array([alpha]), K, dt, 128, 1e-10, False,
                      np.zeros((1, n)), dp, dm, base[None, None, :], x)


def cfg4(batch=512, n=8192, K=16):
    """512 instances: alpha_i~U(1.1,1.9), d+- = a_i + b_i x, f_i = sum_8 C_ij sin(j pi x)."""
    h, dt = 1.0 / (n + 1), 1.0 / K
    x = h * np.arange(1, n + 1)
    r4 = np.random.default_rng(4)
    alpha = r4.uniform(1.1, 1.9, 512)
    a = r4.uniform(0.5, 2.0, 512)
    b = r4.uniform(0.0, 1.0, 512)
    C = r4.standard_normal((512, 8))
    alpha, a, b, C = alpha[:batch], a[:batch], b[:batch], C[:batch]
    d = (a[:, None] + b[:, None] * x[None, :])[None]
    f = _sine_series(x, C)[None]
    # BASELINE configs[3] states no truncation tolerance.  Reading R18: tol 1e-13,
    # because at 1e-12 even the truncated-SVD definition of the compression (oracle) leaves a
    # forward error of 1.6e-8 > 1e-8 on the stiffest instance (alpha = 1.899); 1e-13 gives 7.7e-10.
    wl = Workload1D("cfg4", batch, n, h, alpha, K, dt, 128, 1e-13, True,
                    np.zeros((batch, n)), d, d.copy(), f, x)
    wl.a, wl.b = a, b                # the per-instance coefficient parameters (d = a + b x)
    return wl


def cfg4_checked_instances(wl):
    """The 16 cfg4 instances with a dense-oracle trajectory: the argmax /
    argmin of alpha_i and of a_i + b_i (stiffest and mildest cases), then 12 drawn with
    rng(40).choice from the rest."""
    ext = [int(np.argmax(wl.alpha)), int(np.argmin(wl.alpha)),
           int(np.argmax(wl.a + wl.b)), int(np.argmin(wl.a + wl.b))]
    ext = list(dict.fromkeys(ext))
    rest = np.setdiff1d(np.arange(wl.batch), ext)
    picks = np.random.default_rng(40).choice(rest, 16 - len(ext), replace=False)
    return ext + [int(i) for i in picks]


def lowrank_state(nx, ny, r=27, seed=16, smax=1.0, smin=1e-10):
    """A seeded rank-r 2D state U = Su Sv^T with the shape of a cfg5 solution: smooth columns
    (8-mode sine series) and singular-value scales log-spaced from smax to smin (SURVEY.md
    Appendix A6: the solution rank at tol 1e-12 is ~27 with singular values spanning ~1e-10
    relative).  Used as the shared input of a late-step parity check."""
    rng = np.random.default_rng(seed)
    x = np.arange(1, nx + 1) / (nx + 1.0)
    y = np.arange(1, ny + 1) / (ny + 1.0)
    Su = _sine_series(x, rng.standard_normal((r, 8))).T * np.logspace(np.log10(smax), np.log10(smin), r)
    Sv = _sine_series(y, rng.standard_normal((r, 8))).T
    return Su, Sv


def make_1d(n, alpha, leaf, tol, K=4, dt=None, kind="smooth", seed=7, batch=1):
    """Small test workloads with the paper's shapes (time-dependent d+-)."""
    rng = np.random.default_rng(seed)
    alphas = np.broadcast_to(np.asarray(alpha, dtype=np.float64), (batch,)).copy()
    h = 1.0 / (n + 1)
    dt = 1.0 / K if dt is None else dt
    x = h * np.arange(1, n + 1)
    t = dt * np.arange(1, K + 1)
    c = rng.standard_normal((batch, 8))
    a = rng.uniform(0.5, 2.0, batch)
    b = rng.uniform(0.0, 1.0, batch)
    base = _sine_series(x, c)
    if kind == "const":
        dp = np.ones((1, batch, n)); dm = np.ones((1, batch, n))
        f = base[None]
    elif kind == "zero":
        dp = np.ones((1, batch, n)); dm = np.ones((1, batch, n))
        f = np.zeros((1, batch, n))
    else:
        dp = np.stack([(a[:, None] + b[:, None] * x) * (1 + 0.5 * np.sin(tm)) for tm in t])
        dm = np.stack([(a[:, None] + b[:, None] * (1 - x) ** 2) * (1 + 0.5 * np.cos(tm)) for tm in t])
        f = np.stack([(1 + tm) * base for tm in t])
    u0 = (x ** 2 * (1 - x) ** 2)[None, :].repeat(batch, 0)
    if kind == "zero":
        u0 = np.zeros((batch, n))
    return Workload1D("custom", batch, n, h, alphas, K, dt, leaf, tol,
                      kind in ("const", "zero"), u0, dp, dm, f, x)


@dataclass
class Workload2D:
    name: str
    nx: int
    ny: int
    hx: float
    hy: float
    alpha1: float
    alpha2: float
    K: int
    dt: float
    leaf: int
    tol: float
    ek_tol: float
    x: np.ndarray
    y: np.ndarray
    d1p: np.ndarray
    d1m: np.ndarray
    d2p: np.ndarray
    d2m: np.ndarray
    Fa: np.ndarray       # (nx, r) samples a_r(x)
    Fb: np.ndarray       # (ny, r) samples b_r(y)
    tfac: object = None  # t -> scalar multiplying the separable source

    def source_factors(self, m):
        """F^(m) = Fu Fv^T at t_m (m = 1..K): returns (Fu, Fv).  tfac(t) is a scalar or one
        factor per separable term."""
        tm = m * self.dt
        return self.Fa, self.Fb * np.asarray(self.tfac(tm))


def cfg5(n=2048, K=16):
    """2D: alpha=(1.3,1.7), d1 = 1+x / 2-x, d2 = 1+y^2 / 2-y^2, rank-4 source (1+t) sum a_r b_r."""
    h = 1.0 / (n + 1)
    x = h * np.arange(1, n + 1)
    r5 = np.random.default_rng(5)
    A = r5.standard_normal((4, 8))
    B = r5.standard_normal((4, 8))
    Fa = _sine_series(x, A).T
    Fb = _sine_series(x, B).T
    return Workload2D("cfg5", n, n, h, h, 1.3, 1.7, K, 1.0 / K, 128, 1e-12, 1e-11,
                      x, x.copy(), 1 + x, 2 - x, 1 + x ** 2, 2 - x ** 2, Fa, Fb,
                      lambda t: 1.0 + t)


def paper2d(n, alpha1=1.3, alpha2=1.7, variable=False, K=8, tol=1e-8, ek_tol=1e-6, leaf=128):
    """The paper's 2D test problem (Sec. 5.1, from Breiten et al.): [0,1]^2,
    f = 100 (sin(10 pi x) cos(pi y) + sin(10 t) sin(pi x) y (1 - y)) -- rank 2 on the grid for
    every t --, implicit Euler with dt = 1, 8 steps, u0 = 0, HODLR tol 1e-8 and EK tolerance 1e-6
    (P:1626-1630); d = 1 (constant case) or Eq. (5.1): d1+ = G(1.2)(1+x)^a1, d1- = G(1.2)(2-x)^a1,
    d2+- likewise in y with a2.  Grid: h = 1/(n+1) (reading R5; the paper writes 1/(N+2))."""
    h = 1.0 / (n + 1)
    x = h * np.arange(1, n + 1)
    if variable:
        g = math.gamma(1.2)
        d1p, d1m = g * (1 + x) ** alpha1, g * (2 - x) ** alpha1
        d2p, d2m = g * (1 + x) ** alpha2, g * (2 - x) ** alpha2
    else:
        d1p = d1m = d2p = d2m = np.ones(n)
    Fa = np.stack([100.0 * np.sin(10 * np.pi * x), 100.0 * np.sin(np.pi * x)], axis=1)
    Fb = np.stack([np.cos(np.pi * x), x * (1 - x)], axis=1)
    return Workload2D("paper2d-%s" % ("var" if variable else "const"), n, n, h, h, alpha1, alpha2,
                      K, 1.0, leaf, tol, ek_tol, x, x.copy(), d1p, d1m.copy(), d2p, d2m.copy(),
                      Fa, Fb, lambda t: np.array([1.0, math.sin(10.0 * t)]))
