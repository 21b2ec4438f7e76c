"""GMRES timeline (debug build) of config 4's LOCAL solve (explicit subsystem, ~26k unknowns): CTA 0's phases."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

lc.load_library(sys.argv[1])
sy = synth.system(4, 3)
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=3)
b = torch.from_numpy(sy.b).cuda()
x0 = torch.from_numpy(sy.x0).cuda()
dom = lc.select_domain(A, b, x0, criterion=0, threshold=0, param=1e-10, expand_rounds=1)
sub = lc.extract_sub(A, dom, b, x0)
for i in range(2):
    x = x0.clone()
    info = lc.solve_local(sub, x, method=lc.GMRES)
print(info, dom.K)
K = 7
buf = (ctypes.c_ulonglong * 16384)()
lc._lib.lc_debug_timeline_gmres(buf, 16384)
t = np.array(buf[:K * 30], dtype=np.int64).reshape(-1, K)
d = np.diff(t, axis=1)
print("per step (ns): 1a | sync1a | 1b | sync+red1b | hstore+update | sync+red")
for j in (1, 5, 15, 25, 29):
    print(j, d[j], "step", t[j + 1, 0] - t[j, 0] if j + 1 < len(t) else None)
print("median", np.median(d[1:29], axis=0), "step total", np.median(np.diff(t[1:29, 0])))
