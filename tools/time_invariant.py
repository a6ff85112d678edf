"""Time-invariant coefficients, K = 16 steps: the factor-once pipelined launch (fde1d_run with
stride-0 coefficients, k_run inv mode) against the kept-factor per-step path (fde1d_step: factor
with step 1, then 15 solves with the kept factor), over problem sizes.  CUDA events, best of 3."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
from paper_1804_05522_b200 import workloads as W            # noqa: E402
from paper_1804_05522_b200.hodlr import Fde1dStepper         # noqa: E402

dev = torch.device("cuda:0")
K = 16
CASES = [(65536, 128, 1), (8192, 128, 8),
         (8192, 128, 32), (8192, 128, 128), (8192, 128, 512)]
for n, leaf, batch in CASES:
    wl = W.make_1d(n, np.linspace(1.5, 1.8, batch), leaf, 1e-12, K=K, batch=batch)
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)
    dp, dm = wl.coeffs(1)
    DP, DM, F, U0 = t(dp), t(dm), t(wl.source(1)), t(wl.u0)
    st = Fde1dStepper(n, wl.alpha, wl.h, wl.tol, leaf, batch=batch)
    u = [U0.clone(), torch.empty_like(U0)]

    def best(fn):
        fn()
        torch.cuda.synchronize()
        b = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            b = e0.elapsed_time(e1) if b is None else min(b, e0.elapsed_time(e1))
        return b

    def kept():
        for k in range(K):
            st.step(wl.dt, DP, DM, F, u[k % 2], u_next=u[(k + 1) % 2], coeffs_changed=(k == 0))
    ms_run = best(lambda: st.run(wl.dt, DP[None], DM[None], F[None], U0, K=K))
    ms_kept = best(kept)
    print(json.dumps({"n": n, "leaf": leaf, "batch": batch, "leaves": batch * (-(-n // leaf)),
                      "ms_run_inv": ms_run, "ms_kept_steps": ms_kept}), flush=True)
    st.close()
