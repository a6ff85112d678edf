"""Per-task durations inside k_run (cfg3), printed as one JSON object.

Runs against the diagnostics library (FDE_LIB_DEBUG=1 -> libfdehodlr_dbg.so, whose k_run
records per-task globaltimer stamps when FDE_TRACE_RUN names a file).  bench.py calls this in a
subprocess after its timed runs: the numbers are a diagnostic, never the bench value.
Usage: FDE_LIB_DEBUG=1 python tools/task_profile.py [K]
"""
import collections
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    if os.environ.get("FDE_LIB_DEBUG") != "1":
        raise SystemExit("run with FDE_LIB_DEBUG=1 (the trace switches exist only in the diagnostics build)")
    import torch
    from paper_1804_05522_b200 import workloads as W
    from paper_1804_05522_b200.hodlr import Fde1dStepper
    wl = W.cfg3(K=K)
    dev = torch.device("cuda")
    DP = torch.as_tensor(wl.d_plus, device=dev).contiguous()
    DM = torch.as_tensor(wl.d_minus, device=dev).contiguous()
    F = torch.as_tensor(wl.f[0:1], device=dev).contiguous()
    U0 = torch.as_tensor(wl.u0, device=dev).contiguous()
    st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
    st.run(wl.dt, DP, DM, F, U0)                     # warm-up (untraced)
    torch.cuda.synchronize()
    path = os.path.join(tempfile.gettempdir(), "fde_run_trace_%d.txt" % os.getpid())
    os.environ["FDE_TRACE_RUN"] = path
    st.run(wl.dt, DP, DM, F, U0)
    torch.cuda.synchronize()
    del os.environ["FDE_TRACE_RUN"]
    st.close()
    rows = [tuple(int(x) for x in ln.split()) for ln in open(path)]
    os.remove(path)
    names = {100: "A", 101: "B", 102: "B'", 103: "final"}
    names.update({50 + m: "R%d" % m for m in range(24)})   # split run: right-hand-side units
    by = collections.defaultdict(list)
    t0, t1 = min(r[0] for r in rows), max(r[1] for r in rows)
    nsm = len(set(r[3] for r in rows))
    for s_, e_, code, sm in rows:
        kind = code % 1000
        by[names.get(kind, "L%d" % kind)].append((e_ - s_) / 1e3)
    busy = sum(sum(v) for v in by.values())
    print(json.dumps({
        "steps": K, "us_per_step": (t1 - t0) / 1e3 / K, "sm_busy": busy / ((t1 - t0) / 1e3 * nsm),
        "tasks": {k: {"n": len(v), "mean_us": sum(v) / len(v), "sm_us_per_step_per_sm": sum(v) / nsm / K}
                  for k, v in sorted(by.items())},
        "note": "diagnostics library (libfdehodlr_dbg.so), per-task globaltimer stamps; not the timed run"}))


if __name__ == "__main__":
    main()
