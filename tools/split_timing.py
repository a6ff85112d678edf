"""cfg3 top-level split (fde1d_step_split) timed on ONE GPU.  All parts of a world-G split run in
this process one after the other (rank = -1); CUDA events around every launch (fde_profile) give
the subtree launches ("k_step_part", G per step, equal work) and the top-levels + finals launch
("k_step_top").  A rank of a real G-GPU split runs one part + the top launch with only its own
leaves' finals, so  part_total / G + top  bounds its device time per step from above (the top
launch here runs the finals of ALL leaves), to which the two all-gathers ((xc_p - 1) x xc_p and
n / G doubles per rank) add NVLink latency.  Printed as JSON next to the unsplit fused step."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200 import workloads as W, _lib  # noqa: E402
from paper_1804_05522_b200.split1d import Split1dStepper  # noqa: E402
from paper_1804_05522_b200.hodlr import Fde1dStepper, FDE_NO_KEEP  # noqa: E402


def prof(lib, fn, reps):
    lib.fde_profile_enable(1)
    for k in range(reps):
        fn(k)
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16)
    lib.fde_profile_dump(buf, 1 << 16)
    lib.fde_profile_enable(0)
    return {k: v[1] / reps for k, v in json.loads(buf.value.decode()).items()}


def main():
    wl = W.cfg3(K=8)
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
    lib = _lib.load()
    DP = [t(wl.coeffs(m)[0][0]) for m in range(1, 9)]
    DM = [t(wl.coeffs(m)[1][0]) for m in range(1, 9)]
    F = t(wl.source(1)[0])
    v = [t(wl.u0[0]), torch.empty_like(t(wl.u0[0]))]
    res = {}
    ref = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
    step = lambda k: ref.step(wl.dt, DP[k][None], DM[k][None], F[None], v[k % 2][None], u_next=v[(k + 1) % 2][None],
                              flags=FDE_NO_KEEP)
    for k in range(2):
        step(k)
    res["unsplit_k_step_ms"] = prof(lib, step, 8).get("k_step")
    ref.close()
    for world in (2, 4, 8):
        sp = Split1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf, world=world, rank=-1)
        st = lambda k: sp.step(wl.dt, DP[k], DM[k], F, v[k % 2], v[(k + 1) % 2], use_callback=False)
        for k in range(2):
            st(k)
        d = prof(lib, st, 8)
        part, top = d.get("k_step_part", 0.0), d.get("k_step_top", 0.0)
        res["world_%d" % world] = {"parts_total_ms": part, "top_ms": top,
                                   "per_rank_bound_ms": part / world + top}
        sp.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
