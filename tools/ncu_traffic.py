#!/usr/bin/env python3
"""Measure the DRAM traffic of the bench's dominant kernel with ncu and store it, stamped with the source hash of
the build, as gpurun_out/ncu_traffic/ncu_traffic.json; committed as profiles/ncu_traffic.json, bench.py reports
it as roofline.traffic only while the hash matches the build it runs.

Runs on the GPU box: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--clock-control none -k regex:k_pcg over tools/one_solve.py 5 (two global solves of config 5, s = 3; the second
launch is taken), and divides the DRAM bytes by the solve's iterations."""
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
log = os.path.join(out_dir, "k_pcg_c5.csv")
js = os.path.join(out_dir, "one_solve_c5.json")
build.build()
cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum", "--clock-control",
       "none", "--csv", "--print-units", "base", "-k", "regex:k_pcg", "--log-file", log, sys.executable,
       os.path.join(ROOT, "tools", "one_solve.py"), "5", "--json", js]
subprocess.check_call(cmd, cwd=ROOT)
rows = [r for r in csv.DictReader(l for l in open(log) if l.startswith('"'))]
ids = sorted({int(r["ID"]) for r in rows})
last = [r for r in rows if int(r["ID"]) == ids[-1]]
val = {r["Metric Name"]: float(r["Metric Value"].replace(",", "")) for r in last}
meta = json.load(open(js))
its = meta["info"][0]["iterations"]
rd, wr = val["dram__bytes_read.sum"], val["dram__bytes_write.sum"]
entry = {"dram_bytes_per_iteration": int((rd + wr) / its), "config": 5, "layout": meta["layout"],
         "lazy_x_depths": [meta["info"][0]["lazy_x_depth"]], "source_sha256": build.source_sha256(),
         "source": (f"tools/ncu_traffic.py: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control "
                    f"none, the global PCG of config 5 s=3 ({its} iterations, lazy x depth "
                    f"{meta['info'][0]['lazy_x_depth']}): {rd / 1e9:.2f} + {wr / 1e9:.2f} GB in "
                    f"{val['gpu__time_duration.sum'] / 1e6:.2f} ms")}
db = {"k_pcg": entry}
# written under gpurun_out/ (what a gpurun call brings back); copy it to profiles/ncu_traffic.json to commit it
with open(os.path.join(out_dir, "ncu_traffic.json"), "w") as f:
    json.dump(db, f, indent=2)
print(json.dumps(db, indent=2))
