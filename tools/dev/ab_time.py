"""A/B: time the global PCG (device time per iteration) with two liblc builds."""
import os
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

lib = sys.argv[1]
cfgs = [int(c) for c in sys.argv[2:]]
lc.load_library(lib)
lc._lib.lc_matrix_info.argtypes = None
for cfg in cfgs:
    sy = synth.system(cfg, 3)
    A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=sy.block, batch=sy.batch)
    b = torch.from_numpy(sy.b).cuda()
    x0 = torch.from_numpy(sy.x0).cuda()
    best = 1e9
    for rep in range(4):
        x = x0.clone()
        info = lc.solve_global(A, b, x, method=lc.GMRES if cfg == 4 else lc.PCG)
        best = min(best, info[0]["seconds"])
        its = max(i["iterations"] for i in info)
    print(f"{os.path.basename(lib)} stencil_off={os.environ.get('LC_DISABLE_STENCIL','0')} config {cfg}: its {its} "
          f"{best*1e3:.3f} ms {best/its*1e6:.2f} us/it", flush=True)
