"""A/B timing of the global PCG on configs (device time per iteration from lc_solve_info)."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

cfgs = [int(c) for c in sys.argv[1:]] or [1, 5, 3, 2]
for cfg in cfgs:
    sy = synth.system(cfg, 3)
    dev = torch.device("cuda")
    A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=sy.block, batch=sy.batch)
    b = torch.from_numpy(sy.b).to(dev)
    x0 = torch.from_numpy(sy.x0).to(dev)
    best = 1e9
    for rep in range(4):
        x = x0.clone()
        info = lc.solve_global(A, b, x, method=lc.GMRES if cfg == 4 else lc.PCG)
        best = min(best, info[0]["seconds"])
        its = max(i["iterations"] for i in info)
    print(f"config {cfg}: {A.info()['layout']} its {its} best {best*1e3:.3f} ms  {best/its*1e6:.2f} us/it", flush=True)
