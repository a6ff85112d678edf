"""Per-(step, kind) first-start / last-end table of a k_run trace (FDE_TRACE_RUN output)."""
import collections
import sys

rows = [tuple(int(x) for x in ln.split()) for ln in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/run_trace.txt")]
t0 = min(r[0] for r in rows)
ph = collections.defaultdict(lambda: [float("inf"), 0, 0, 0.0])
for s, e, c, sm in rows:
    st, k = divmod(c, 1000)
    p = ph[(st, k)]
    p[0] = min(p[0], s); p[1] = max(p[1], e); p[2] += 1; p[3] += (e - s) / 1e3
steps = sorted(set(k[0] for k in ph))
pick = [int(x) for x in sys.argv[2:]] or steps[1:3]
for key in sorted(ph, key=lambda k: ph[k][0]):
    if key[0] in pick:
        p = ph[key]
        print("step %d kind %3d  %8.1f - %8.1f us  n=%4d  mean %.1f" % (key[0], key[1], (p[0] - t0) / 1e3, (p[1] - t0) / 1e3, p[2], p[3] / p[2]))
# busy SMs over time (10 us bins)
T = max(r[1] for r in rows) - t0
nb = int(T / 1e4) + 1
busy = [0.0] * nb
for s, e, c, sm in rows:
    a, b = (s - t0) / 1e4, (e - t0) / 1e4
    i = int(a)
    while i < b and i < nb:
        busy[i] += min(b, i + 1) - max(a, i)
        i += 1
print("busy SMs per 10us bin (first 200 bins):")
print(" ".join("%d" % round(x) for x in busy[:200]))
