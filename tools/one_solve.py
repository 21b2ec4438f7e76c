"""One global solve (method0 from x0) of system s = 3 of a config, twice (the second is the measured one); prints
the solve info and, with --json FILE, writes it (iterations, lazy-x depth, layout) for tools/ncu_traffic.py."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

cfg = int(sys.argv[1])
sy = synth.system(cfg, 3)
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=sy.block, batch=sy.batch)
b = torch.from_numpy(sy.b).cuda()
x = torch.from_numpy(sy.x0).cuda()
for i in range(2):
    xx = x.clone()
    info = lc.solve_global(A, b, xx, method=lc.GMRES if sy.block == 3 else lc.PCG)
print(info[0])
if "--json" in sys.argv:
    with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
        json.dump(dict(config=cfg, layout=A.info()["layout"], info=info), f)
