import ctypes, sys
sys.path.insert(0, ".")
import numpy as np, torch, synth
from paper_2001_01158_b200 import lc
lc.load_library(sys.argv[1])
if len(sys.argv) > 2:
    lc.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in sys.argv[2].split(","))})
    print("tuning", sys.argv[2])
sy = synth.system(3, 3)
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, batch=20)
b = torch.from_numpy(sy.b).cuda(); x = torch.from_numpy(sy.x0).cuda()
for i in range(2):
    xx = x.clone(); info = lc.solve_global(A, b, xx)
print("iters per group", [i["iterations"] for i in info], "ms", info[0]["seconds"] * 1e3)
buf = (ctypes.c_ulonglong * 8192)()
lc._lib.lc_debug_timeline(buf, 8192)
t = np.array(buf[:6 * 900], dtype=np.int64).reshape(-1, 6)
t = t[t[:, 0] > 0]
d = np.diff(t, axis=1)
print("phases: passA | syncA+red | scalarsA | passB | syncB+red")
for k in (5, 20, 50, 100, 200, 300, 400, 500, 600, 700, 800, 900):
    if k < len(d): print(k, d[k])
