"""Summarise gpurun_out/ ncu artefacts into profiles/ (run here, no GPU needed).

usage: python tools/ncu_summary.py <tag> [rep=gpurun_out/prof.ncu-rep] [launches=gpurun_out/launches.csv]
Writes profiles/<tag>_ncu.md (per-kernel key counters + stall mix + launch-list shares) and
updates profiles/ncu_traffic.json (dram read+write bytes per launch, read by bench.py)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def to_bytes(v, u):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return float(v.replace(",", "")) * f


def to_us(v, u):
    f = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(u, 1e-3)
    return float(v.replace(",", "")) * f


def main():
    tag = sys.argv[1]
    rep = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "prof.ncu-rep")
    lcsv = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", "launches.csv")
    out = ["# ncu summary %s" % tag, ""]
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        traffic = json.load(open(traffic_path))
    except Exception:
        traffic = {}
    if os.path.exists(rep):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        ix = {h: i for i, h in enumerate(hdr)}
        per = collections.OrderedDict()
        for r in rows[2:]:
            name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").split("<")[0]
            per.setdefault(name, []).append(r)
        out.append("## `ncu --set full` (%s)" % os.path.basename(rep))
        for name, rs in per.items():
            out.append("")
            out.append("### %s (%d captured launches; values of the last)" % (name, len(rs)))
            r = rs[-1]
            for k in KEYS:
                if k in ix:
                    out.append("- %s = %s %s" % (k, r[ix[k]], units[ix[k]]))
            rb = to_bytes(r[ix["dram__bytes_read.sum"]], units[ix["dram__bytes_read.sum"]])
            wb = to_bytes(r[ix["dram__bytes_write.sum"]], units[ix["dram__bytes_write.sum"]])
            traffic[name] = rb + wb
            out.append("- dram read+write per launch = %.1f MB" % ((rb + wb) / 1e6))
            st = []
            for i, h in enumerate(hdr):
                if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                    try:
                        st.append((float(r[i].replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
                    except ValueError:
                        pass
            tot = sum(v for v, _ in st) or 1.0
            out.append("- stall mix (pc samples): " + ", ".join(
                "%s %.1f%%" % (h, 100 * v / tot) for v, h in sorted(st, reverse=True)[:8]))
        json.dump(traffic, open(traffic_path, "w"), indent=1)
    if os.path.exists(lcsv):
        rows = list(csv.reader(open(lcsv)))
        hdr = None
        agg = collections.OrderedDict()
        for r in rows:
            if "Kernel Name" in r:
                hdr = r
                continue
            if hdr is None or len(r) != len(hdr):
                continue
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = d["Kernel Name"].split("(")[0].replace("void ", "")
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += to_us(d["Metric Value"], d["Metric Unit"])
        tot = sum(t for _, t in agg.values()) or 1.0
        out.append("")
        out.append("## launch list (`--metrics gpu__time_duration.sum --clock-control none`, cold, serialised)")
        out.append("")
        out.append("| kernel | launches | total us | us/launch | share |")
        out.append("|---|---|---|---|---|")
        for k, (c, t) in agg.items():
            out.append("| %s | %d | %.1f | %.1f | %.1f%% |" % (k, c, t, t / c, 100 * t / tot))
    path = os.path.join(ROOT, "profiles", "%s_ncu.md" % tag)
    open(path, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
