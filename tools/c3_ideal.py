#!/usr/bin/env python3
"""Config 3 (batched multi-group PCG): measured device time of a global solve vs the bandwidth-ideal time
sum_g it_g * rows_g * bytes_per_row / peak (each group pays only for its own iterations)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

PEAK = 6542e9
s = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sy = synth.system(3, s)
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, batch=sy.batch)
inf = A.info()
b = torch.from_numpy(sy.b).cuda()
x0 = torch.from_numpy(sy.x0).cuda()
best = None
for _ in range(3):
    x = x0.clone()
    info = lc.solve_global(A, b, x)
    t = info[0]["seconds"]
    best = t if best is None else min(best, t)
its = [i["iterations"] for i in info]
rows = sy.nrows // sy.batch
bpr = (8 * inf["max_row"] if inf["layout"] != "sell" else 12 * inf["max_row"]) + 96
ideal = sum(its) * rows * bpr / PEAK
print(json.dumps(dict(layout=inf["layout"], its=its, max_it=max(its), sum_it=sum(its), measured_ms=best * 1e3,
                      ideal_ms=ideal * 1e3, frac=ideal / best, us_per_max_it=best / max(its) * 1e6)))
