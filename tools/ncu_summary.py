#!/usr/bin/env python3
"""Summarise ncu evidence into profiles/*.md (run here, on the CPU box).

  tools/ncu_summary.py --launches gpurun_out/launches.csv --rep gpurun_out/prof.ncu-rep \
      --bytes-per-launch 3.0e9 --out profiles/r01_pcg.md --title "..."
"""
import argparse
import csv
import io
import subprocess
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def launches_table(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    tot = 0.0
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    out = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {c} | {t / 1e3:.3f} | {100 * t / tot:.1f}% |")
    return "\n".join(out), agg, tot


def rep_metrics(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    h, u = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"Kernel Name": row[h.index("Kernel Name")] if "Kernel Name" in h else "?"}
        for k in KEYS:
            if k in h:
                d[k] = (row[h.index(k)], u[h.index(k)])
        res.append(d)
    return res


def stall_table(path, top=10):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return ""
    h = rows[1]
    data = rows[2:]
    si = h.index("Warp Stall Sampling (All Samples)")
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(float(r[si] or 0) for r in data) or 1.0
    agg = {c: sum(float(r[h.index(c)] or 0) for r in data) for c in cols}
    out = ["| stall reason | share of samples |", "|---|---|"]
    for c, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        out.append(f"| {c} | {100 * v / tot:.1f}% |")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--bytes-per-launch", type=float, default=None)
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--notes", default="")
    a = ap.parse_args()
    md = [f"# {a.title}", ""]
    if a.notes:
        md += [a.notes, ""]
    if a.launches:
        t, _, tot = launches_table(a.launches)
        md += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`)", "",
               "Cold-cache, serialised per-launch times: compare shares, not absolutes.", "",
               f"Total device time of the listed launches: {tot / 1e3:.3f} ms", "", t, ""]
    if a.rep:
        for d in rep_metrics(a.rep):
            md += [f"## `ncu --set full` capture: `{d['Kernel Name'][:80]}`", "", "| metric | value |", "|---|---|"]
            for k in KEYS:
                if k in d:
                    md.append(f"| {k} | {d[k][0]} {d[k][1]} |")
            if "gpu__time_duration.sum" in d and "dram__bytes_read.sum" in d:
                t = float(d["gpu__time_duration.sum"][0].replace(",", ""))
                tu = d["gpu__time_duration.sum"][1]
                t_s = t * {"ns": 1e-9, "nsecond": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3,
                           "ms": 1e-3}.get(tu, 1.0)
                def gb(x):
                    v = float(x[0].replace(",", ""))
                    return v * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}.get(x[1], 1.0)
                traffic = gb(d["dram__bytes_read.sum"]) + gb(d["dram__bytes_write.sum"])
                md.append(f"| DRAM traffic (read+write) | {traffic:.3f} GB |")
                md.append(f"| DRAM bandwidth (traffic / duration) | {traffic / t_s:.1f} GB/s |")
                if a.bytes_per_launch:
                    md.append(f"| algorithmic bytes of this launch | {a.bytes_per_launch / 1e9:.3f} GB |")
                    md.append(f"| traffic / algorithmic | {traffic / (a.bytes_per_launch / 1e9):.3f} |")
            md.append("")
        st = stall_table(a.rep)
        if st:
            md += ["### Warp stall sampling (source page)", "", st, ""]
    open(a.out, "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
