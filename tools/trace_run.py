"""Timeline of the pipelined run (k_run): FDE_TRACE_RUN=<file> python tools/trace_run.py [K]
prints per-kind task counts / mean durations, SM busy fraction, and per-step completion times."""
import collections
import os
import sys

out = os.environ.setdefault("FDE_TRACE_RUN", "gpurun_out/run_trace.txt")
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200 import workloads as W  # noqa: E402
from paper_1804_05522_b200.hodlr import Fde1dStepper  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
wl = W.cfg3(K=K)
dev = torch.device("cuda")
DP = torch.as_tensor(wl.d_plus, device=dev).contiguous()
DM = torch.as_tensor(wl.d_minus, device=dev).contiguous()
F = torch.as_tensor(wl.f[0:1], device=dev).contiguous()
U0 = torch.as_tensor(wl.u0, device=dev).contiguous()
st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
for _ in range(2):
    st.run(wl.dt, DP, DM, F, U0)
    torch.cuda.synchronize()
rows = [tuple(int(x) for x in ln.split()) for ln in open(out)]
t0 = min(r[0] for r in rows)
t1 = max(r[1] for r in rows)
span = (t1 - t0) / 1e3
names = {100: "A leaf", 101: "B proj", 102: "B' rhs", 103: "final"}
names.update({50 + m: "R%d" % m for m in range(24)})   # split run: right-hand-side units
by = collections.defaultdict(list)
step_end = collections.defaultdict(int)
busy = 0
for s, e, code, sm in rows:
    step, kind = divmod(code, 1000)
    by[names.get(kind, "L%d" % kind)].append((e - s) / 1e3)
    busy += e - s
    if kind == 200:
        step_end[step] = max(step_end[step], e)
nsm = len(set(r[3] for r in rows))
print("K=%d span %.1f us  (%.1f us/step)  SMs %d  busy %.1f%%" % (K, span, span / K, nsm,
                                                                 100.0 * busy / 1e3 / (span * nsm)))
for k in sorted(by):
    v = by[k]
    print("  %-8s n=%5d  mean %7.2f us  total %8.1f us*SM  (%.1f us/step of 148 SMs)"
          % (k, len(v), sum(v) / len(v), sum(v), sum(v) / nsm / K))
prev = t0
for s in sorted(step_end):
    print("  step %d done at %8.1f us (+%.1f)" % (s, (step_end[s] - t0) / 1e3, (step_end[s] - prev) / 1e3))
    prev = step_end[s]
