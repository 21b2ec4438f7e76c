"""A/B of liblc builds: device time of the global solves (configs from argv) and the config 3 / 5 local solves,
best of 3, one line per measurement.  python tools/dev/ab_solves.py LIB CFG..."""
import os
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

lib = sys.argv[1]
lc.load_library(lib)
tag = os.path.basename(os.path.dirname(lib)) or "main"
args = sys.argv[2:]
if "--tune" in args:
    i = args.index("--tune")
    kv = dict(x.split("=") for x in args[i + 1].split(","))
    lc.set_tuning(**{k: int(v) for k, v in kv.items()})
    tag += " " + args[i + 1]
    args = args[:i] + args[i + 2:]
for cfg in (int(c) for c in args):
    sy = synth.system(cfg, 3)
    A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=sy.block, batch=sy.batch)
    b = torch.from_numpy(sy.b).cuda()
    x0 = torch.from_numpy(sy.x0).cuda()
    m = lc.GMRES if cfg == 4 else lc.PCG
    best, its = 1e9, 0
    for _ in range(3):
        x = x0.clone()
        info = lc.solve_global(A, b, x, method=m)
        best = min(best, info[0]["seconds"]); its = max(i["iterations"] for i in info)
    print(f"{tag} config {cfg} global: its {its} {best*1e3:.3f} ms {best/its*1e6:.2f} us/it", flush=True)
    if cfg in (2, 3, 4, 5):
        rule = {2: dict(criterion=1, threshold=2, param=0.9, dilate_hops=2),
                3: dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1),
                4: dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1),
                5: dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1)}[cfg]
        bl = 1e9
        for _ in range(3):
            x, rep = lc.local_method(A, b, x0, rule, method=m)
            bl = min(bl, max(i["seconds"] for i in rep["local"]))
        print(f"{tag} config {cfg} local: its {max(i['iterations'] for i in rep['local'])} {bl*1e3:.3f} ms", flush=True)
