#!/usr/bin/env python3
"""Host wall time against device time of one bench step through the one-call path: lc_create_csr, then per rule
lc_local_method.  Each call is bracketed by a stream synchronise, so wall - device = launch, allocation and host
round-trip time of that call.  usage: step_wall.py [CONFIG] [REPS]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
dev = torch.device("cuda")
rules, solver = bench.CFG_RULES[cfg]
method = lc.GMRES if solver == "gmres" else lc.PCG
systems = []
for s in range(3, 3 + reps):
    sy = synth.system(cfg, s)
    systems.append((sy, {k: torch.from_numpy(getattr(sy, k)).to(dev) for k in ("rp", "ci", "val", "b", "x0")}))


def t(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


for sy, inp in systems:
    A, tc = t(lambda: lc.Matrix(sy.nrows, inp["rp"], inp["ci"], inp["val"], block=sy.block, batch=sy.batch))
    out = [f"create wall {tc:.3f}"]
    tot = tc
    for name, rule in rules:
        (x, rep), tw = t(lambda: lc.local_method(A, inp["b"], inp["x0"], rule, method=method))
        ms = rep["ms"]
        devt = sum(ms.values())
        tot += tw
        out.append(f"{name}: wall {tw:.3f} dev {devt:.3f} (" + " ".join(f"{k} {v:.3f}" for k, v in ms.items()) + ")")
    _, td = t(lambda: A.__del__() if hasattr(A, "__del__") else None)
    print(f"config {cfg} s={sy.s} step wall {tot:.3f} ms; " + "; ".join(out) + f"; destroy {td:.3f}", flush=True)
# the same steps back to back, one synchronise at the end (what the bench times)
torch.cuda.synchronize()
t0 = time.perf_counter()
for sy, inp in systems:
    A = lc.Matrix(sy.nrows, inp["rp"], inp["ci"], inp["val"], block=sy.block, batch=sy.batch)
    for name, rule in rules:
        lc.local_method(A, inp["b"], inp["x0"], rule, method=method)
torch.cuda.synchronize()
print(f"back to back: {(time.perf_counter() - t0) * 1e3 / len(systems):.3f} ms per step", flush=True)
