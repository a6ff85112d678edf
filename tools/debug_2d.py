"""2D step diagnostics: FDE_DEBUG2D=1 python tools/debug_2d.py [n] [K]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200 import workloads as W  # noqa: E402
from paper_1804_05522_b200.hodlr import Fde2dStepper  # noqa: E402
from oracle.sylvester2d import operators_2d, BartelsStewart  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = W.cfg5(n=n)
t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
st = Fde2dStepper(wl.nx, wl.ny, wl.alpha1, wl.alpha2, wl.hx, wl.hy, wl.dt, t(wl.d1p), t(wl.d1m),
                  t(wl.d2p), t(wl.d2m), wl.tol, ek_tol=1e-11, leaf=wl.leaf)
A1, A2 = operators_2d(wl.alpha1, wl.alpha2, wl.nx, wl.ny, wl.hx, wl.hy, wl.dt, wl.d1p, wl.d1m, wl.d2p, wl.d2m)
bs = BartelsStewart(A1, A2)
Uo = np.zeros((n, n))
Xu = Xv = None
for m in range(1, K + 1):
    Fa, Fb = wl.source_factors(m)
    try:
        if Xu is None:
            Xu, Xv, res, its = st.step(t(Fa.T), t(Fb.T))
        else:
            Xu, Xv, res, its = st.step(t(Fa.T), t(Fb.T), Xu, Xv)
    except Exception as e:
        print("step", m, "failed:", e)
        break
    Xg = Xu.cpu().numpy().T @ Xv.cpu().numpy()
    Uo = bs.solve(Uo + wl.dt * Fa @ Fb.T)
    print("step %d rank %d res %.3e its %d relerr %.3e" % (m, Xu.shape[0], res, its,
          np.linalg.norm(Xg - Uo) / np.linalg.norm(Uo)))
