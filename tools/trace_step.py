"""cfg3 phase trace: FDE_TRACE_LEVELS=1 python tools/trace_step.py  (prints per-phase timings)."""
import os
import sys

os.environ["FDE_TRACE_LEVELS"] = "1"
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200 import workloads as W  # noqa: E402
from paper_1804_05522_b200.hodlr import Fde1dStepper, FDE_NO_KEEP  # noqa: E402

wl = W.cfg3(K=4)
dev = torch.device("cuda")
DP = torch.as_tensor(wl.d_plus[:, 0, :], device=dev).contiguous()
DM = torch.as_tensor(wl.d_minus[:, 0, :], device=dev).contiguous()
F = torch.as_tensor(wl.f[0, 0, :], device=dev).contiguous()
u = [torch.zeros(wl.n, dtype=torch.float64, device=dev) for _ in range(2)]
st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
for i in range(3):
    st.step(wl.dt, DP[i], DM[i], F, u[i % 2], u_next=u[(i + 1) % 2], flags=FDE_NO_KEEP)
    torch.cuda.synchronize()
