#!/usr/bin/env python3
"""One row-partitioned global PCG solve on config 5 with p emulated ranks (for ncu captures).
usage: python tools/dist_one.py [p] [config] [n]"""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import dist as ldist  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n = int(sys.argv[3]) if len(sys.argv) > 3 else None
sy = synth.system(cfg, 10, n=n)
R = ldist.split_rows(sy.nrows, P, 256)
ranks = []
for l in range(P):
    rp, ci, va = ldist.slab_csr(sy.rp, sy.ci, sy.val, R[l], R[l + 1])
    ranks.append(lc.DistRank(sy.nrows, R[l], R[l + 1] - R[l], l, P, rp, ci, va))
lc.dist_connect_local(ranks)
b = torch.from_numpy(sy.b).cuda()
x0 = torch.from_numpy(sy.x0).cuda()
bs = [b[R[l]:R[l + 1]].contiguous() for l in range(P)]
xs = [x0[R[l]:R[l + 1]].clone() for l in range(P)]
info = lc.dist_solve_global(ranks, bs, xs)
print(info)
