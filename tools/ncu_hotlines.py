#!/usr/bin/env python3
"""Warp-stall samples of an ncu --set full --import-source on capture, per SOURCE line.

ncu's CSV source page lists SASS instructions with their stall counters but no line numbers; nvdisasm -g on the
cubin of the same build lists the same instructions with `//## File ... line N` markers.  This tool joins the two
by instruction offset and prints the hottest lines with their dominant stall reasons and the headline metrics.

  tools/ncu_hotlines.py REP.ncu-rep build/pcg.cu.o [--top 30]
"""
import argparse
import csv
import io
import os
import re
import subprocess
import tempfile
from collections import defaultdict

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("obj")
ap.add_argument("--top", type=int, default=30)
a = ap.parse_args()

sass = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
kernel = rows[0][1]
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
body = rows[2:]
mangled = None
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(a.obj)], cwd=td, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(td, cub)], capture_output=True, text=True).stdout
    names = subprocess.run(["cuobjdump", "-elf", os.path.join(td, cub)], capture_output=True, text=True).stdout
# sections of the disassembly, demangled to find the captured kernel
secs = {}
cur = None
for l in dis.split("\n"):
    m = re.match(r"\s*\.section\s+\.text\.(\S+?),", l)
    if m:
        cur = m.group(1)
        secs[cur] = []
        continue
    if cur is not None:
        secs[cur].append(l)
dem = subprocess.run(["c++filt"], input="\n".join(secs), capture_output=True, text=True).stdout.split("\n")
want = re.sub(r"\(int\)|\(bool\)|\s", "", kernel.replace("void ", "")).split("(")[0]
pick = None
for mang, d in zip(secs, dem):
    if re.sub(r"\s", "", d).split("(")[0].replace("void", "") == want.replace("lc::", "lc::"):
        pick = mang
if pick is None:        # fall back: the section with as many instructions as the capture
    for mang, ls in secs.items():
        n = sum(1 for l in ls if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l))
        if n == len(body):
            pick = mang
ins = []
src = None
for l in secs[pick]:
    m = re.search(r'//## File ".*?([^/"]+)", line (\d+)', l)
    if m:
        src = (m.group(1), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), src))
assert len(ins) == len(body), (len(ins), len(body), pick)
base = int(body[0][0], 16)
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
agg = defaultdict(lambda: defaultdict(int))
tot = 0
for (off, s), r in zip(ins, body):
    assert int(r[0], 16) - base == off
    n = int(r[ci["# Samples"]])
    tot += n
    agg[s]["n"] += n
    for c in cols:
        agg[s][c] += int(r[ci[c]] or 0)
texts = {}
print(f"kernel: {kernel}\nsamples: {tot}\n")
print("| line | share | main stalls | source |\n|---|---|---|---|")
root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2001_01158_b200", "csrc")
for s, d in sorted(agg.items(), key=lambda x: -x[1]["n"])[:a.top]:
    txt = ""
    if s:
        f = os.path.join(root, s[0])
        if os.path.exists(f):
            texts.setdefault(f, open(f).read().split("\n"))
            txt = texts[f][s[1] - 1].strip()[:70].replace("|", "\\|")
    main = ", ".join(f"{c[6:]} {100 * v / max(d['n'], 1):.0f}%" for c, v in sorted(d.items(), key=lambda x: -x[1])
                     if c != "n" and v > 0.15 * d["n"])
    print(f"| {s[0] + ':' + str(s[1]) if s else '?'} | {100 * d['n'] / tot:.1f}% | {main} | `{txt}` |")
