"""Time lc_smooth_gs (one sweep) on the heat model's 2-D Picard system and on config 5 (3-D).
usage: python tools/gs_time.py [lib]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

if len(sys.argv) > 1:
    lc.load_library(sys.argv[1])
    lc._lib.lc_matrix_info.argtypes = None
for n in (99, 1024):
    T = torch.from_numpy(synth.heat_initial(n, n)).cuda()
    rp, ci, va, b = lc.heat_assemble(n, n, 1e-2, T, T)
    A = lc.Matrix(n * n, rp, ci, va)
    best = 1e9
    for _ in range(5):
        x = T.clone()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lc.smooth_gs(A, b, x, 1)
        best = min(best, time.perf_counter() - t0)
    print(f"heat {n}^2: {best * 1e3:.3f} ms per sweep", flush=True)
sy = synth.system(5, 3)
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val)
b = torch.from_numpy(sy.b).cuda()
best = 1e9
for _ in range(3):
    x = torch.from_numpy(sy.x0).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lc.smooth_gs(A, b, x, 1)
    best = min(best, time.perf_counter() - t0)
print(f"config 5 (256^3): {best * 1e3:.3f} ms per sweep", flush=True)
