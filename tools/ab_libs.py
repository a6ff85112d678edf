"""A/B timing of library builds: python tools/ab_libs.py <lib.so> ...  -- per library: cfg4
refactor every step (fused k_step per step and the pipelined run, 16 steps x 512 instances) and
cfg1 / cfg2 / cfg3 (pipelined runs), CUDA events, best of 3.  Each library runs in its own process."""
import os
import subprocess
import sys

if len(sys.argv) > 2:                                  # one process per library
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, __file__, lib], check=False)
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.abspath(sys.argv[1])
from paper_1804_05522_b200 import workloads as W  # noqa: E402
from paper_1804_05522_b200.hodlr import Fde1dStepper, FDE_NO_KEEP, FDE_REFACTOR  # noqa: E402

dev = torch.device("cuda")
tag = os.path.basename(sys.argv[1])
t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)


def best(fn):
    fn()
    torch.cuda.synchronize()
    r = None
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        r = ms if r is None else min(r, ms)
    return r


wl = W.cfg4()
dp, dm = wl.coeffs(1)
DP, DM, F = t(dp), t(dm), t(wl.source(1))
u = [t(wl.u0), torch.empty_like(t(wl.u0))]
st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf, batch=wl.batch)
st.step(wl.dt, DP, DM, F, u[0], u_next=u[1], coeffs_changed=True)


def refactor():
    for k in range(16):
        st.step(wl.dt, DP, DM, F, u[k % 2], u_next=u[(k + 1) % 2], coeffs_changed=True, flags=FDE_NO_KEEP)


print("%s cfg4 refactor k_step  %.1f ms" % (tag, best(refactor)), flush=True)
print("%s cfg4 refactor run     %.1f ms" % (tag, best(lambda: st.run(wl.dt, DP[None], DM[None], F[None], u[0], K=16, flags=FDE_REFACTOR))), flush=True)
st.close()
for name in ("cfg1", "cfg2", "cfg3"):
    wl = W.cfg3(K=64) if name == "cfg3" else getattr(W, name)()
    DP, DM, F, U0 = t(wl.d_plus), t(wl.d_minus), t(wl.f), t(wl.u0)
    st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
    # (refactor every step: cfg1's time-invariant d+- would otherwise factor once)
    print("%s %s run  %.1f us/step" % (tag, name, 1e3 * best(lambda: st.run(wl.dt, DP, DM, F, U0, flags=FDE_REFACTOR)) / wl.K), flush=True)
    st.close()
