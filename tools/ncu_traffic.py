#!/usr/bin/env python3
"""Measure the DRAM traffic of the bench's dominant kernel with ncu and store it, stamped with the source hash of
the build, as gpurun_out/ncu_traffic/ncu_traffic.json; committed as profiles/ncu_traffic.json, bench.py reports
it as roofline.traffic only while the hash matches the build it runs.

Runs on the GPU box: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--clock-control none -k regex:k_pcg (k_gmres for config 4) over tools/one_solve.py CONFIG (two global solves of
system s = 3; the second launch is taken), and divides the DRAM bytes by the solve's iterations (summed over the
groups of a batched solve; Arnoldi steps for GMRES).  usage: ncu_traffic.py [CONFIG ...]   (default 5)"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2001_01158_b200 import build  # noqa: E402

out_dir = os.path.join(ROOT, "gpurun_out", "ncu_traffic")
os.makedirs(out_dir, exist_ok=True)
build.build()
cfgs = [int(c) for c in sys.argv[1:]] or [5]
db = {}
for cfg in cfgs:
    kname = "k_gmres" if cfg == 4 else "k_pcg"          # regex:k_pcg also matches the batched k_pcg_dyn (config 3)
    log = os.path.join(out_dir, f"{kname}_c{cfg}.csv")
    js = os.path.join(out_dir, f"one_solve_c{cfg}.json")
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "--csv", "--print-units", "base", "-k", f"regex:{kname}", "--log-file", log,
           sys.executable, os.path.join(ROOT, "tools", "one_solve.py"), str(cfg), "--json", js]
    subprocess.check_call(cmd, cwd=ROOT)
    rows = [r for r in csv.DictReader(l for l in open(log) if l.startswith('"'))]
    ids = sorted({int(r["ID"]) for r in rows})
    last = [r for r in rows if int(r["ID"]) == ids[-1]]
    val = {r["Metric Name"]: float(r["Metric Value"].replace(",", "")) for r in last}
    meta = json.load(open(js))
    its = sum(i["iterations"] for i in meta["info"])     # batched: summed over the groups, like the bench's count
    rd, wr = val["dram__bytes_read.sum"], val["dram__bytes_write.sum"]
    unit = "Arnoldi steps" if cfg == 4 else "iterations" + (" summed over the groups" if len(meta["info"]) > 1 else "")
    entry = {"dram_bytes_per_iteration": int((rd + wr) / its), "config": cfg, "layout": meta["layout"],
             "source_sha256": build.source_sha256(),
             "source": (f"tools/ncu_traffic.py: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                        f"--clock-control none, the global {'GMRES' if cfg == 4 else 'PCG'} of config {cfg} s=3 "
                        f"({its} {unit}, kernel {last[0]['Kernel Name'][:40]}): {rd / 1e9:.2f} + {wr / 1e9:.2f} GB in "
                        f"{val['gpu__time_duration.sum'] / 1e6:.2f} ms")}
    if cfg != 4:
        entry["lazy_x_depths"] = sorted({i["lazy_x_depth"] for i in meta["info"]})
    db[f"{kname}@c{cfg}"] = entry
    if cfg == 5:
        db["k_pcg"] = entry                               # the key the first version of this file used
# written under gpurun_out/ (what a gpurun call brings back); copy it to profiles/ncu_traffic.json to commit it
with open(os.path.join(out_dir, "ncu_traffic.json"), "w") as f:
    json.dump(db, f, indent=2)
print(json.dumps(db, indent=2))
