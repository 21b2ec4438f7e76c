#!/usr/bin/env python3
"""Device time of the method2 local solve (residual domain, E_max = 1) with a given liblc build.
usage: time_local.py LIB CONFIG [CONFIG ...] [field=value ...]   (lc_tuning fields for an A/B)"""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

lc.load_library(sys.argv[1])
tune = dict(a.split("=") for a in sys.argv[2:] if "=" in a)
if tune:
    lc.set_tuning(**{k: int(v) for k, v in tune.items()})
for cfg in [int(c) for c in sys.argv[2:] if "=" not in c]:
    sy = synth.system(cfg, 3)
    A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=sy.block, batch=sy.batch)
    b = torch.from_numpy(sy.b).cuda()
    x0 = torch.from_numpy(sy.x0).cuda()
    rule = dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1)
    if cfg == 2:
        rule = dict(criterion=1, threshold=2, param=0.9, expand_rounds=0, dilate_hops=2)
    best = 1e9
    for _ in range(4):
        dom = lc.select_domain(A, b, x0, **rule)
        sub = lc.extract_sub(A, dom, b, x0)
        x = x0.clone()
        info = lc.solve_local(sub, x)
        best = min(best, max(i["seconds"] for i in info))
    its = max(i["iterations"] for i in info)
    print(f"{sys.argv[1]} {tune or ''} config {cfg} local: K {sum(dom.K)} its {its} {best * 1e3:.3f} ms "
          f"kernel {info[0]['kernel']} lazy {info[0]['lazy_x_depth']}", flush=True)
