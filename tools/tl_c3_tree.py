"""Config 3 timeline (debug build -DLC_DEBUG_TIMELINE): per reduction of the batched PCG, CTA 0's pass end,
the last CTA's arrival (the tree's top arriver starts summing), the release, and CTA 0's exit from the
reduction.  usage: python tools/tl_c3_tree.py paper_2001_01158_b200/liblc_tl.so"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

lc.load_library(sys.argv[1])
sy = synth.system(3, 3)
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, batch=20)
b = torch.from_numpy(sy.b).cuda()
x = torch.from_numpy(sy.x0).cuda()
buf = (ctypes.c_ulonglong * 8192)()
lc._lib.lc_debug_timeline_tree(buf, 8192)          # reset the tree counter
info = lc.solve_global(A, b, x.clone())
nit = max(i["iterations"] for i in info)
tl = (ctypes.c_ulonglong * 8192)()
lc._lib.lc_debug_timeline(tl, 8192)
lc._lib.lc_debug_timeline_tree(buf, 8192)
t = np.array(tl[:6 * (nit + 3)], dtype=np.int64).reshape(-1, 6)
tx = np.array(buf[:], dtype=np.int64).reshape(-1, 2)
print("iterations", nit, "ms", info[0]["seconds"] * 1e3)
print("k | passA  cta0_end->last_arrival  last_arrival->release  release->cta0_out | passB  ... (ns)")
for k in (5, 50, 200, 400, 600, 800, 900):
    if k >= len(t) or 2 * k + 1 >= len(tx):
        continue
    a = t[k]
    ra, rb = tx[2 * k], tx[2 * k + 1]
    print(k, "|", a[1] - a[0], ra[0] - a[1], ra[1] - ra[0], a[2] - ra[1], "|", a[4] - a[3], rb[0] - a[4], rb[1] - rb[0],
          a[5] - rb[1])
