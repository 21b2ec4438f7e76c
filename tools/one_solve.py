import sys
sys.path.insert(0, ".")
import torch, synth
from paper_2001_01158_b200 import lc
cfg = int(sys.argv[1])
sy = synth.system(cfg, 3)
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=sy.block, batch=sy.batch)
b = torch.from_numpy(sy.b).cuda(); x = torch.from_numpy(sy.x0).cuda()
for i in range(2):
    xx = x.clone(); info = lc.solve_global(A, b, xx, method=lc.GMRES if sy.block == 3 else lc.PCG)
print(info[0])
