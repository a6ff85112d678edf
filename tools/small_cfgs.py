"""cfg1 / cfg2 / cfg3 time per step through fde1d_run (CUDA events, best of 3), as bench.py's
measure_small; for A/B comparisons of run-time switches of the diagnostics library."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200 import workloads as W  # noqa: E402
from paper_1804_05522_b200.hodlr import Fde1dStepper  # noqa: E402

dev = torch.device("cuda")
for name in sys.argv[1:] or ["cfg1", "cfg2", "cfg3"]:
    if name.startswith("n="):                          # n=<size>: cfg3-like (alpha 1.8, leaf 128, tol 1e-10)
        wl = W.make_1d(int(name[2:]), 1.8, 128, 1e-10, K=32)
    else:
        wl = W.cfg3(K=64) if name == "cfg3" else getattr(W, name)()
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)
    DP, DM, F, U0 = t(wl.d_plus), t(wl.d_minus), t(wl.f), t(wl.u0)
    st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf, batch=wl.batch)
    st.run(wl.dt, DP, DM, F, U0)
    torch.cuda.synchronize()
    best = None
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st.run(wl.dt, DP, DM, F, U0)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
    print("%s split=%s  %.1f us/step" % (name, os.environ.get("FDE_RUN_SPLIT", "-"), 1e3 * best / wl.K))
    st.close()
