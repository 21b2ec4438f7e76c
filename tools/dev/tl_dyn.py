"""Block-0 timeline of the dynamic-teams batched PCG (debug build): per pass of CTA 0's team: chunk work, barrier +
reduction, team size.  python tools/dev/tl_dyn.py build_dbg/liblc_dbg.so [s]"""
import ctypes
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

lc.load_library(sys.argv[1])
s = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lc.set_tuning(batched_schedule=2)
sy = synth.system(3, s)
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, batch=20)
b = torch.from_numpy(sy.b).cuda()
x = torch.from_numpy(sy.x0).cuda()
for i in range(2):
    xx = x.clone()
    info = lc.solve_global(A, b, xx)
print("iters", [i["iterations"] for i in info], "ms", info[0]["seconds"] * 1e3, info[0]["kernel"])
buf = (ctypes.c_ulonglong * 8192)()
lc._lib.lc_debug_timeline(buf, 8192)
t = np.array(buf[:8192], dtype=np.int64).reshape(-1, 4)
t = t[t[:, 0] > 0]
work = (t[:, 1] - t[:, 0]) / 1e3
red = (t[:, 2] - t[:, 1]) / 1e3
gap = np.r_[(t[1:, 0] - t[:-1, 2]) / 1e3, 0]
tn = t[:, 3]
print("passes recorded", len(t), "(CTA 0's team; the next pass start - this pass end = scalars or a re-team)")
for k in list(range(0, len(t), max(1, len(t) // 40))) + [len(t) - 1]:
    print(f"pass {k:5d} team {tn[k]:4d} work {work[k]:7.2f} us  barrier+sum {red[k]:6.2f} us  gap {gap[k]:7.2f} us")
for lo, hi in ((0, 200), (200, 1000), (1000, 1400), (1400, len(t))):
    sl = slice(lo, min(hi, len(t)))
    if lo < len(t):
        print(f"passes {lo}-{min(hi, len(t))}: work {work[sl].mean():.2f} barrier+sum {red[sl].mean():.2f} gap {gap[sl].mean():.2f}")
