"""One residual-criterion domain selection (a1-a5) on config 5 at 256^3, repeated (for ncu captures of the
SpMV-shaped kernels).  usage: python tools/select_one.py [reps]"""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sy = synth.system(5, 3)
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val)
b = torch.from_numpy(sy.b).cuda()
x0 = torch.from_numpy(sy.x0).cuda()
for _ in range(reps):
    d = lc.select_domain(A, b, x0, criterion=0, threshold=0, param=1e-10, expand_rounds=1)
    g = lc.select_domain(A, b, x0, criterion=1, threshold=1, param=1e-4)
print(d.K, g.K)
