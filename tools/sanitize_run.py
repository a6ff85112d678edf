"""Small invocations of every kernel path for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): cfg1-sized 1D problems through the pipelined run (k_run), the fused step
(k_step), the kept factor (k_leaf + k_levels), its solve (k_leaf_apply + k_solve_level), the
HODLR matvec, the compression (k_pchol / k_eig / k_ltransform), a batched instance set, and one
2D Sylvester step (n = 64).  Usage: compute-sanitizer --tool <t> python tools/sanitize_run.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200 import workloads as W  # noqa: E402
from paper_1804_05522_b200.hodlr import Fde1dStepper, Fde2dStepper, Hodlr, FDE_NO_KEEP, FDE_SYNC  # noqa: E402

t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def main():
    for (n, alpha, leaf, batch) in ((256, 1.5, 32, 1), (300, 1.3, 40, 2)):
        wl = W.make_1d(n, np.linspace(alpha, alpha + 0.2, batch), leaf, 1e-12, K=3, batch=batch)
        dp, dm = wl.coeffs(1)
        st = Fde1dStepper(n, wl.alpha, wl.h, wl.tol, leaf, batch=batch)
        DP = torch.stack([t(wl.coeffs(m)[0]) for m in range(1, 4)])
        DM = torch.stack([t(wl.coeffs(m)[1]) for m in range(1, 4)])
        F = torch.stack([t(wl.source(m)) for m in range(1, 4)])
        st.run(wl.dt, DP, DM, F, t(wl.u0), flags=FDE_SYNC)                       # k_run
        u = st.step(wl.dt, t(dp), t(dm), t(wl.source(1)), t(wl.u0), flags=FDE_NO_KEEP | FDE_SYNC)   # k_step
        u = st.step(wl.dt, t(dp), t(dm), t(wl.source(1)), u, flags=FDE_SYNC)     # k_leaf + k_levels
        u = st.step(wl.dt, t(dp), t(dm), t(wl.source(2)), u, coeffs_changed=False, flags=FDE_SYNC)  # solve
        st.close()
        H = Hodlr(n, wl.alpha, wl.h, wl.dt, t(dp), t(dm), wl.tol, leaf, batch=batch)
        H.factor(flags=FDE_SYNC)
        X = t(np.random.default_rng(0).standard_normal((batch, 5, n)))
        Y = H.matvec(X, flags=FDE_SYNC)
        H.solve(Y, flags=FDE_SYNC)
        H.close()
    w2 = W.cfg5(n=64)
    s2 = Fde2dStepper(w2.nx, w2.ny, w2.alpha1, w2.alpha2, w2.hx, w2.hy, w2.dt, t(w2.d1p), t(w2.d1m),
                      t(w2.d2p), t(w2.d2m), w2.tol, ek_tol=w2.ek_tol, leaf=w2.leaf)
    Fa, Fb = w2.source_factors(1)
    Xu, Xv, _, _ = s2.step(t(Fa.T), t(Fb.T))
    Fa, Fb = w2.source_factors(2)
    s2.step(t(Fa.T), t(Fb.T), Xu, Xv)
    s2.close()
    torch.cuda.synchronize()
    print("sanitize_run: done")


if __name__ == "__main__":
    main()
