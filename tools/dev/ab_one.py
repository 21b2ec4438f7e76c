import sys
sys.path.insert(0, ".")
import torch, synth
from paper_2001_01158_b200 import lc
lc.load_library(sys.argv[1]); lc._lib.lc_matrix_info.argtypes = None
sy = synth.system(int(sys.argv[2]), 3)
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=sy.block, batch=sy.batch)
b = torch.from_numpy(sy.b).cuda(); x = torch.from_numpy(sy.x0).cuda()
for i in range(2):
    xx = x.clone(); info = lc.solve_global(A, b, xx)
print(info[0])
