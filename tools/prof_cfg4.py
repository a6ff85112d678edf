"""cfg4 (512 x n=8192) per-kernel times: factor once, then solve steps (LU reuse)."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200 import workloads as W  # noqa: E402
from paper_1804_05522_b200 import _lib  # noqa: E402
from paper_1804_05522_b200.hodlr import Fde1dStepper  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 512
wl = W.cfg4(batch=batch)
t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
dp, dm = wl.coeffs(1)
DP, DM, F = t(dp), t(dm), t(wl.source(1))
u = [t(wl.u0), torch.empty_like(t(wl.u0))]
st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf, batch=batch)
st.step(wl.dt, DP, DM, F, u[0], u_next=u[1], coeffs_changed=True)
torch.cuda.synchronize()
lib = _lib.load()
for label, refac in (("solve", False), ("refactor", True)):
    lib.fde_profile_enable(1)
    for k in range(4):
        st.step(wl.dt, DP, DM, F, u[k % 2], u_next=u[(k + 1) % 2], coeffs_changed=refac)
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16)
    lib.fde_profile_dump(buf, 1 << 16)
    lib.fde_profile_enable(0)
    d = json.loads(buf.value.decode())
    print(label, {k: (v[0] / 4, round(v[1] / 4, 3)) for k, v in d.items()}, "ranks", st.ranks(0))
