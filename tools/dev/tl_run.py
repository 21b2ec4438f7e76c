import ctypes, sys
sys.path.insert(0, ".")
import numpy as np, torch, synth
from paper_2001_01158_b200 import lc
lc.load_library(sys.argv[1]); lc._lib.lc_matrix_info.argtypes = None
sy = synth.system(int(sys.argv[2]), 3)
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=sy.block, batch=sy.batch)
b = torch.from_numpy(sy.b).cuda(); x = torch.from_numpy(sy.x0).cuda()
for i in range(2):
    xx = x.clone(); info = lc.solve_global(A, b, xx)
buf = (ctypes.c_ulonglong * 8192)()
lc._lib.lc_debug_timeline(buf, 8192)
t = np.array(buf[:6 * 100], dtype=np.int64).reshape(-1, 6)
d = np.diff(t, axis=1)
nxt = t[1:, 0] - t[:-1, 5]
print("phases (ns): passA | syncA+red | scalarsA | passB | syncB+red  ; then scalarsB+loop")
print("median", np.median(d[5:90], axis=0), np.median(nxt[5:90]))
print("iter total median", np.median(np.diff(t[5:90, 0])))
