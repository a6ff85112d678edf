"""Wall time of the first 4 cfg5 steps (as bench.py measure_cfg5), 3 repetitions."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200 import workloads as W  # noqa: E402
from paper_1804_05522_b200.hodlr import Fde2dStepper  # noqa: E402

wl = W.cfg5()
t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
for rep in range(3):
    st = Fde2dStepper(wl.nx, wl.ny, wl.alpha1, wl.alpha2, wl.hx, wl.hy, wl.dt, t(wl.d1p), t(wl.d1m), t(wl.d2p),
                      t(wl.d2m), wl.tol, ek_tol=wl.ek_tol, leaf=wl.leaf)
    Fs = [tuple(t(f.T) for f in wl.source_factors(m)) for m in range(1, 5)]
    st.step(*Fs[0])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Xu = Xv = None
    for m in range(4):
        Xu, Xv, res, it = st.step(*Fs[m]) if Xu is None else st.step(*Fs[m], Xu, Xv)
    torch.cuda.synchronize()
    print("cfg5 4 steps: %.1f ms/step" % (1e3 * (time.perf_counter() - t0) / 4))
    st.close()
