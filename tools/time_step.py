"""Device time of the per-step path (one fde1d_step = one k_step launch) on cfg3."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200 import workloads as W  # noqa: E402
from paper_1804_05522_b200.hodlr import Fde1dStepper, FDE_NO_KEEP  # noqa: E402

wl = W.cfg3(K=32)
dev = torch.device("cuda")
DP = torch.as_tensor(wl.d_plus[:, 0, :], device=dev).contiguous()
DM = torch.as_tensor(wl.d_minus[:, 0, :], device=dev).contiguous()
F = torch.as_tensor(wl.f[0, 0, :], device=dev).contiguous()
u = [torch.zeros(wl.n, dtype=torch.float64, device=dev) for _ in range(2)]
st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for rep in range(2):
    tot = 0.0
    for k in range(16):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st.step(wl.dt, DP[k], DM[k], F, u[k % 2], u_next=u[(k + 1) % 2], flags=FDE_NO_KEEP)
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    print("k_step per-step: %.1f us/step" % (1e3 * tot / 16))
