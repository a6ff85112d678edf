"""Per-source-line stall breakdown of a ncu report (source page, cuda+sass correlation).
usage: python tools/ncu_stalls.py <rep> [reason=stall_long_sb] [top=25]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
reason = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr = None, None
agg, allv, text = collections.Counter(), collections.Counter(), {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        i_r, i_a = hdr.index(reason), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or r[0] in ("Function Name",) or not r[0] or len(r) <= max(i_r, i_a):
        continue
    try:
        v, va = float(r[i_r] or 0), float(r[i_a] or 0)
    except ValueError:
        continue
    key = (fname, int(r[0]))
    agg[key] += v
    allv[key] += va
    text[key] = r[1][:90]
tot, tota = sum(agg.values()), sum(allv.values())
print("%s: %.1f%% of all samples" % (reason, 100 * tot / max(tota, 1)))
for (f, l), v in agg.most_common(top):
    print("%5.2f%% (%5.2f%% all) %s:%d %s" % (100 * v / tota, 100 * allv[(f, l)] / tota, f, l, text[(f, l)].strip()))
