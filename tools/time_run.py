"""Device time of fde1d_run on cfg3 for several K (CUDA events, L2 flushed before each run)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200 import workloads as W  # noqa: E402
from paper_1804_05522_b200.hodlr import Fde1dStepper  # noqa: E402

Ks = [int(x) for x in sys.argv[1:]] or [4, 8, 16, 32, 64]
wl = W.cfg3(K=max(Ks))
dev = torch.device("cuda")
DP = torch.as_tensor(wl.d_plus, device=dev).contiguous()
DM = torch.as_tensor(wl.d_minus, device=dev).contiguous()
F = torch.as_tensor(wl.f[0:1], device=dev).contiguous()
U0 = torch.as_tensor(wl.u0, device=dev).contiguous()
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
st.run(wl.dt, DP[:2], DM[:2], F, U0)
for K in Ks:
    for rep in range(2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        st.run(wl.dt, DP[:K], DM[:K], F, U0)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        print("K=%3d  %.3f ms  %.1f us/step" % (K, ms, 1e3 * ms / K))
