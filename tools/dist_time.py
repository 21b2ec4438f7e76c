#!/usr/bin/env python3
"""NEXT-4 on one GPU: device time per PCG iteration of the row-partitioned solve (p emulated ranks, one
cooperative launch; halo rows read from the neighbour slabs' workspaces, every dot product through the
ranks' exchange blocks) against the single-GPU k_pcg, on config 5 (256^3) by default.

The emulated p-rank run does the same total work on the same SMs as p = 1, so the difference to p = 1 is
the cost of the partition itself (halo branches, the exchange round trip per reduction).
usage: python tools/dist_time.py [config] [n]
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import dist as ldist  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
sy = synth.system(cfg, 10, n=n)
dev = torch.device("cuda")
out = {"config": cfg, "N": sy.nrows}
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val)
b, x0 = torch.from_numpy(sy.b).to(dev), torch.from_numpy(sy.x0).to(dev)
best = 1e9
for _ in range(3):
    x = x0.clone()
    info = lc.solve_global(A, b, x)[0]
    best = min(best, info["seconds"] / max(info["iterations"], 1))
out["single_gpu_us_per_it"] = best * 1e6
out["iterations"] = info["iterations"]
del A
for P in (1, 2, 4, 8):
    R = ldist.split_rows(sy.nrows, P, 256)
    ranks = []
    for l in range(P):
        rp, ci, va = ldist.slab_csr(sy.rp, sy.ci, sy.val, R[l], R[l + 1])
        ranks.append(lc.DistRank(sy.nrows, R[l], R[l + 1] - R[l], l, P, rp, ci, va))
    lc.dist_connect_local(ranks)
    bs = [b[R[l]:R[l + 1]].contiguous() for l in range(P)]
    best = 1e9
    for _ in range(3):
        xs = [x0[R[l]:R[l + 1]].clone() for l in range(P)]
        info = lc.dist_solve_global(ranks, bs, xs)
        best = min(best, info["seconds"] / max(info["iterations"], 1))
    out[f"emulated_p{P}_us_per_it"] = best * 1e6
    out[f"emulated_p{P}_iterations"] = info["iterations"]
    del ranks
print(json.dumps(out))
