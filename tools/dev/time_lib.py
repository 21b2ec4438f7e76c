#!/usr/bin/env python3
"""Global-solve device time per iteration with a given liblc build (A/B of compile-time variants).
usage: time_lib.py LIB CONFIG [CONFIG ...]"""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

lc.load_library(sys.argv[1])
for cfg in [int(c) for c in sys.argv[2:]]:
    sy = synth.system(cfg, 3)
    A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=sy.block, batch=sy.batch)
    b = torch.from_numpy(sy.b).cuda()
    x0 = torch.from_numpy(sy.x0).cuda()
    best = 1e9
    for _ in range(4):
        x = x0.clone()
        info = lc.solve_global(A, b, x, method=lc.GMRES if sy.block == 3 else lc.PCG)
        best = min(best, info[0]["seconds"])
    its = max(i["iterations"] for i in info)
    print(f"{sys.argv[1]} config {cfg}: its {its} {best * 1e3:.3f} ms {best / its * 1e6:.2f} us/it", flush=True)
