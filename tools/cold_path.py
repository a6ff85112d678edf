"""Cold path (S1 + S2 inside every step: fde1d_step with FDE_RECOMPRESS) per-kernel device times
on cfg3 and cfg4 (first 64 instances), via the library's launch profiler (CUDA events)."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200 import workloads as W, _lib  # noqa: E402
from paper_1804_05522_b200.hodlr import Fde1dStepper, FDE_NO_KEEP, FDE_RECOMPRESS  # noqa: E402

t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
lib = _lib.load()
out = {}
for name in ("cfg3", "cfg4"):
    wl = W.cfg3(K=4) if name == "cfg3" else W.cfg4(batch=64)
    if name == "cfg3":
        DP, DM, F = t(wl.d_plus[1, 0]), t(wl.d_minus[1, 0]), t(wl.f[0, 0])
        u = [t(wl.u0[0] if wl.u0.ndim > 1 else wl.u0), None]
    else:
        dp, dm = wl.coeffs(1)
        DP, DM, F = t(dp), t(dm), t(wl.source(1))
        u = [t(wl.u0), None]
    u[1] = torch.empty_like(u[0])
    st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf, batch=wl.batch)
    fl = FDE_RECOMPRESS | (FDE_NO_KEEP if name == "cfg3" else 0)
    for k in range(3):
        st.step(wl.dt, DP, DM, F, u[k % 2], u_next=u[(k + 1) % 2], flags=fl)
    torch.cuda.synchronize()
    R = 8
    lib.fde_profile_enable(1)
    for k in range(R):
        st.step(wl.dt, DP, DM, F, u[k % 2], u_next=u[(k + 1) % 2], flags=fl)
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16)
    lib.fde_profile_dump(buf, 1 << 16)
    lib.fde_profile_enable(0)
    d = json.loads(buf.value.decode())
    per = {k: round(1e3 * v[1] / R, 1) for k, v in d.items()}
    cold = sum(v for k, v in per.items() if k in ("k_gl_seg", "k_gl_expand", "k_pchol", "k_eig", "k_ltransform", "k_colofs"))
    out[name] = {"us_per_step": per, "s1_s2_us": round(cold, 1), "ranks": st.ranks(0)}
    print(name, json.dumps(out[name]))
    st.close()
