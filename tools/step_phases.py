#!/usr/bin/env python3
"""Wall time (host, synchronised around each call) of the phases of one bench step: lc_create_csr from device
CSR, then per rule of the config lc_select_domain, lc_extract_sub, lc_solve_local, lc_solve_global (and method0's
lc_solve_global), next to the device time the solves report.  usage: step_phases.py [CONFIG]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
sy = synth.system(cfg, 3)
dev = torch.device("cuda")
inp = {k: torch.from_numpy(getattr(sy, k)).to(dev) for k in ("rp", "ci", "val", "b", "x0")}
rules, solver = bench.CFG_RULES[cfg]
method = lc.GMRES if solver == "gmres" else lc.PCG


def t(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


for rep in range(4):
    A, tc = t(lambda: lc.Matrix(sy.nrows, inp["rp"], inp["ci"], inp["val"], block=sy.block, batch=sy.batch))
    out = [f"create {tc:.3f}"]
    tot = tc
    for name, rule in rules:
        x, tx = t(lambda: inp["x0"].clone())
        tot += tx
        parts = [f"clone {tx:.3f}"]
        if rule is not None:
            dom, ts = t(lambda: lc.select_domain(A, inp["b"], inp["x0"], **rule))
            sub, te = t(lambda: lc.extract_sub(A, dom, inp["b"], inp["x0"]))
            il, tl = t(lambda: lc.solve_local(sub, x, method))
            parts += [f"select {ts:.3f}", f"extract {te:.3f}",
                      f"local {tl:.3f} (dev {1e3 * max(i['seconds'] for i in il):.3f}, K {sum(dom.K)})"]
            tot += ts + te + tl
            del sub, dom
        ig, tg = t(lambda: lc.solve_global(A, inp["b"], x, method))
        tot += tg
        parts.append(f"global {tg:.3f} (dev {1e3 * max(i['seconds'] for i in ig):.3f})")
        out.append(f"{name}: " + " ".join(parts))
    del A
    print(f"config {cfg} ms: total {tot:.3f}; " + "; ".join(out), flush=True)
