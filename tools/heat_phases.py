#!/usr/bin/env python3
"""Per-phase times of one Alg. 1 pass on a heat Picard system (the paper's model) at n x n:
wall time of each C-ABI call (host-synchronous) and the device time the solves report.
usage: python tools/heat_phases.py [n] [steps_before]"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
pre = int(sys.argv[2]) if len(sys.argv) > 2 else 3
T0 = torch.from_numpy(synth.heat_initial(n, n)).cuda()
T, _, _, _ = lc.heat_run(n, n, T0, pre, method=0)          # advance a few steps (a front has formed)
rp, ci, va, b = lc.heat_assemble(n, n, 1e-2, T, T)
A = lc.Matrix(n * n, rp, ci, va)
out = {"n": n, "N": n * n, "layout": A.info()["layout"]}


def wall(f):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t) * 1e3


for name, rule in (("method1", dict(criterion=1, threshold=1, param=1e-4)),
                   ("method2", dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1))):
    for rep in range(2):
        x = T.clone()
        dom, t_dom = wall(lambda: lc.select_domain(A, b, T, **rule))
        sub, t_ext = wall(lambda: lc.extract_sub(A, dom, b, T))
        inf, t_loc = wall(lambda: lc.solve_local(sub, x))
        _, t_gs = wall(lambda: lc.smooth_gs(A, b, x, 1))
        glb, t_glb = wall(lambda: lc.solve_global(A, b, x))
    out[name] = dict(eta=sum(dom.K) / (n * n), ms_select=t_dom, ms_extract=t_ext, ms_local_wall=t_loc,
                     ms_local_dev=inf[0]["seconds"] * 1e3, it_local=inf[0]["iterations"], ms_gs=t_gs,
                     ms_global_wall=t_glb, ms_global_dev=glb[0]["seconds"] * 1e3, it_global=glb[0]["iterations"])
x = T.clone()
glb, t0 = wall(lambda: lc.solve_global(A, b, x))
out["method0"] = dict(ms_wall=t0, ms_dev=glb[0]["seconds"] * 1e3, it=glb[0]["iterations"])
print(json.dumps(out))
