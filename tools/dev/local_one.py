"""One masked local solve on config 5 (method1's gradient domain, eta ~ 1: the full-sweep masked path) and the
method0 global solve of the same system, device time per iteration of each (for A/B and ncu captures)."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

sy = synth.system(5, 3)
A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val)
b = torch.from_numpy(sy.b).cuda()
x0 = torch.from_numpy(sy.x0).cuda()
dom = lc.select_domain(A, b, x0, criterion=1, threshold=1, param=1e-4)
sub = lc.extract_sub(A, dom, b, x0)
x = x0.clone()
li = lc.solve_local(sub, x)[0]
xg = x0.clone()
gi = lc.solve_global(A, b, xg)[0]
print(f"K/N {sum(dom.K) / sy.nrows:.4f} local {li['iterations']} its {li['seconds'] / li['iterations'] * 1e6:.1f} us/it;"
      f" global {gi['iterations']} its {gi['seconds'] / gi['iterations'] * 1e6:.1f} us/it")
# method2's residual domain (eta ~ 0.1: the slice-list masked path)
dom = lc.select_domain(A, b, x0, criterion=0, threshold=0, param=1e-10, expand_rounds=1)
sub = lc.extract_sub(A, dom, b, x0)
x = x0.clone()
li = lc.solve_local(sub, x)[0]
print(f"K/N {sum(dom.K) / sy.nrows:.4f} local (slice list) {li['iterations']} its "
      f"{li['seconds'] / li['iterations'] * 1e6:.1f} us/it")
