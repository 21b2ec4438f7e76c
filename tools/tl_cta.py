#!/usr/bin/env python3
"""Per-CTA pass timeline of k_pcg (debug build, tools/build_debug.sh): for 64 consecutive passes from pass0,
every CTA's pass start / pass end / reduction-out times.  Prints, per pass, the pass-end spread (first to last
CTA arrival), the barrier exit spread, and how late CTAs correlate with their index.
usage: tl_cta.py build_dbg/liblc_dbg.so CONFIG PASS0 [n|0] [local]"""
import ctypes
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

lc.load_library(sys.argv[1])
cfg, pass0 = int(sys.argv[2]), int(sys.argv[3])
n = int(sys.argv[4]) if len(sys.argv) > 4 and int(sys.argv[4]) > 0 else None
sy = synth.system(cfg, 3, n=n) if n else synth.system(cfg, 3)
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=sy.block, batch=sy.batch)
b = torch.from_numpy(sy.b).cuda()
x = torch.from_numpy(sy.x0).cuda()
lib = lc._lib
local = len(sys.argv) > 5 and sys.argv[5] == "local"      # the method2 local solve (residual domain, E_max = 1)
if local:
    dom = lc.select_domain(A, b, x, criterion=0, threshold=0, param=1e-10, expand_rounds=1)
    sub = lc.extract_sub(A, dom, b, x)
    print(json.dumps(dict(K=dom.K)))


def run():
    xx = x.clone()
    return lc.solve_local(sub, xx) if local else lc.solve_global(A, b, xx)


lib.lc_debug_cta_window(ctypes.c_int(1 << 30))
run()
lib.lc_debug_cta_window(ctypes.c_int(pass0))
info = run()
buf = np.zeros(64 * 1024 * 3, dtype=np.uint64)
lib.lc_debug_cta(ctypes.c_void_p(buf.ctypes.data))
t = buf.reshape(64, 1024, 3).astype(np.int64)
ncta = int((t[0, :, 0] > 0).sum())
t = t[:, :ncta, :]
ok = (t[:, :, 0] > 0).all(axis=1)
res = []
for k in range(64):
    if not ok[k]:
        continue
    st, en, out = t[k, :, 0], t[k, :, 1], t[k, :, 2]
    t0 = st.min()
    dur = en - st
    late = np.argsort(en)[-8:]
    res.append(dict(pass_=pass0 + k, start_spread=int(st.max() - st.min()), end_spread=int(en.max() - en.min()),
                    first_end=int(en.min() - t0), last_end=int(en.max() - t0), out_first=int(out.min() - t0),
                    out_last=int(out.max() - t0), dur_med=int(np.median(dur)), dur_max=int(dur.max()),
                    late_ctas=[int(c) for c in late], corr_start_bid=float(np.corrcoef(st, np.arange(ncta))[0, 1])))
print(json.dumps(dict(config=cfg, nCTA=ncta, iters=[i["iterations"] for i in info], ms=info[0]["seconds"] * 1e3)))
for r in res:
    print(json.dumps(r))
