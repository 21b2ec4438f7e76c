#!/usr/bin/env python3
"""Summarise bench JSON lines: value, e2e, roofline frac, breakdown (ms local / global per method)."""
import json
import sys

for f in sys.argv[1:]:
    lines = [x for x in open(f) if x.startswith("{")]
    if not lines:
        print(f, "NO JSON")
        continue
    d = json.loads(lines[-1])
    bd = d.get("config", {}).get("breakdown", {})
    parts = [f"{k}: {v['ms_local']:.2f}/{v['ms_global']:.2f}" for k, v in bd.items()]
    print(f, d["value"], (d.get("e2e") or {}).get("value"), d.get("roofline", {}).get("frac"),
          d.get("clocks", {}).get("sm_mhz"), "; ".join(parts))
