#!/usr/bin/env python3
"""CSR row-slab SpMV (lc_spmv_csr) vs the handle layouts (lc_spmv: stencil / SELL-32) on configs 2 and 5:
device time per call (CUDA events, 20 calls after 3 warm-up) and the algorithmic GB/s of each format."""
import json
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402


def timed(f, reps=20):
    for _ in range(3):
        f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


out = []
for cfg in (int(c) for c in (sys.argv[1:] or ["2", "5"])):
    sy = synth.system(cfg, 3)
    n, nnz = sy.nrows, len(sy.ci)
    dev = torch.device("cuda")
    rp = torch.from_numpy(sy.rp).to(dev)
    ci = torch.from_numpy(sy.ci).to(dev)
    va = torch.from_numpy(sy.val).to(dev)
    x = torch.from_numpy(sy.x0).to(dev)
    y1, y2 = torch.empty_like(x), torch.empty_like(x)
    t_csr = timed(lambda: lc.spmv_csr(rp, ci, va, x, y1))
    row = dict(config=cfg, n=n, nnz=nnz, csr_us=t_csr * 1e6, csr_gbs=(12 * nnz + 8 * (n + 1) + 16 * n) / t_csr / 1e9)
    for layout, stencil in (("stencil", 1), ("sell", 0)):
        prev = lc.set_tuning(stencil_layout=stencil)
        A = lc.Matrix(n, sy.rp, sy.ci, sy.val)
        lc.set_tuning(**prev)
        inf = A.info()
        t = timed(lambda: lc.spmv(A, x, y2))
        assert torch.equal(y1, y2)
        mb = inf["matrix_bytes"]
        row[f"{inf['layout']}_us"] = t * 1e6
        row[f"{inf['layout']}_gbs"] = (mb + 16 * n) / t / 1e9
        del A
    out.append(row)
    print(json.dumps(row), flush=True)
