"""cfg5 per-kernel time breakdown of fde2d_step (steps 1..K)."""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200 import workloads as W  # noqa: E402
from paper_1804_05522_b200 import _lib  # noqa: E402
from paper_1804_05522_b200.hodlr import Fde2dStepper  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = W.cfg5()
t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
st = Fde2dStepper(wl.nx, wl.ny, wl.alpha1, wl.alpha2, wl.hx, wl.hy, wl.dt, t(wl.d1p), t(wl.d1m),
                  t(wl.d2p), t(wl.d2m), wl.tol, ek_tol=wl.ek_tol, leaf=wl.leaf)
Fs = [tuple(t(f.T) for f in wl.source_factors(m)) for m in range(1, K + 1)]
st.step(*Fs[0])
torch.cuda.synchronize()
lib = _lib.load()
lib.fde_profile_enable(1)
Xu = Xv = None
t0 = time.perf_counter()
for m in range(K):
    Xu, Xv, res, it = st.step(*Fs[m]) if Xu is None else st.step(*Fs[m], Xu, Xv)
    print("step", m + 1, "rank", Xu.shape[0], "its", it, "res %.2e" % res)
torch.cuda.synchronize()
el = time.perf_counter() - t0
buf = ctypes.create_string_buffer(1 << 16)
lib.fde_profile_dump(buf, 1 << 16)
d = json.loads(buf.value.decode())
tot = sum(v[1] for v in d.values())
print("wall %.1f ms/step, kernel sum %.1f ms/step" % (el / K * 1e3, tot / K))
for k, v in sorted(d.items(), key=lambda kv: -kv[1][1]):
    print("  %-16s launches/step %7.1f  ms/step %8.3f" % (k, v[0] / K, v[1] / K))
