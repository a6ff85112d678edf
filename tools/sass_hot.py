"""Summarise an ncu --page source --csv dump: top stall SASS lines with context."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
si, wi, ie = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
body = rows[2:]
half = len(body) // 2
if body[:half] == body[half:]:
    body = body[:half]
tot = sum(int(r[wi]) for r in body if r[wi].isdigit())
print("total samples", tot)
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 6
top = sorted([(int(r[wi]), i) for i, r in enumerate(body) if r[wi].isdigit()], reverse=True)[: int(sys.argv[3]) if len(sys.argv) > 3 else 8]
for v, i in top:
    print("=== %d samples (%.1f%%) at %d" % (v, 100.0 * v / tot, i))
    for r in body[max(0, i - ctx): i + 2]:
        print("%7s %9s  %s" % (r[wi], r[ie], r[si][:100]))
