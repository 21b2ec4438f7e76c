#!/usr/bin/env python3
"""Wall time (synchronised) of the non-solve phases of one bench step on config 5: lc_create_csr from device CSR,
lc_select_domain and lc_extract_sub per rule, and the x0 copy of local_method.  usage: step_phases.py [CONFIG]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
sy = synth.system(cfg, 3)
dev = torch.device("cuda")
inp = {k: torch.from_numpy(getattr(sy, k)).to(dev) for k in ("rp", "ci", "val", "b", "x0")}
rules = [dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1), dict(criterion=1, threshold=1, param=1e-4)]


def t(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


for rep in range(3):
    A, tc = t(lambda: lc.Matrix(sy.nrows, inp["rp"], inp["ci"], inp["val"], block=sy.block, batch=sy.batch))
    out = [f"create {tc:.2f}"]
    for i, rule in enumerate(rules):
        _, tx = t(lambda: inp["x0"].clone())
        dom, ts = t(lambda: lc.select_domain(A, inp["b"], inp["x0"], **rule))
        sub, te = t(lambda: lc.extract_sub(A, dom, inp["b"], inp["x0"]))
        out.append(f"rule{i}: clone {tx:.2f} select {ts:.2f} extract {te:.2f} (K {sum(dom.K)})")
        del sub, dom
    del A
    print("ms:", "; ".join(out), flush=True)
