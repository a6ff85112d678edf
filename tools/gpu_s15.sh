#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FDE_LIB_DEBUG=1 FDE_COMP_TRACE=1 timeout 300 python -c "
import torch, sys
sys.path.insert(0,'.')
from paper_1804_05522_b200 import workloads as W
from paper_1804_05522_b200.hodlr import Fde1dStepper, FDE_NO_KEEP
wl=W.cfg3(K=2)
t=lambda a: torch.as_tensor(a, device='cuda').contiguous()
st=Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
u0=t(wl.u0); u1=torch.empty_like(u0)
st.step(wl.dt, t(wl.d_plus[1,0]), t(wl.d_minus[1,0]), t(wl.f[0,0]), u0, u_next=u1, flags=FDE_NO_KEEP)
torch.cuda.synchronize()
print('ok')
" > gpurun_out/s15.log 2>&1
cat gpurun_out/s15.log | sort | head -40
