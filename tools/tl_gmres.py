import ctypes, sys
sys.path.insert(0, ".")
import numpy as np, torch, synth
from paper_2001_01158_b200 import lc
lc.load_library(sys.argv[1])
sy = synth.system(4, 3)
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=3)
b = torch.from_numpy(sy.b).cuda(); x = torch.from_numpy(sy.x0).cuda()
for i in range(2):
    xx = x.clone(); info = lc.solve_global(A, b, xx, method=lc.GMRES)
print(info)
buf = (ctypes.c_ulonglong * 16384)()
lc._lib.lc_debug_timeline_gmres(buf, 16384)
t = np.array(buf[:9 * 40], dtype=np.int64).reshape(-1, 9)
d = np.diff(t, axis=1)
print("per step (ns): 1a | sync1a | 1b | sync+red1b | hstore+2 | sync+red2 | 3 | sync+red3")
for j in (1, 5, 15, 25):
    print(j, d[j])
print("median", np.median(d[1:30], axis=0), "step total", np.median(np.diff(t[1:30, 0])))
