#!/usr/bin/env python3
"""NEXT-2: the paper's 2-D heat experiment (Table in) on the device.

99 x 99, dt = 1e-2, 100 steps, Picard (||dT|| < 1e-8), linear eps = 1e-10; method0 (global Jacobi-PCG),
method1 (Alg. 2, alpha = 1e-4) and method2 (Alg. 3, E_max = 1), one GS sweep for the local methods.
Reports total time per method (device driver wall time), S = t0 / t_m, eta per step, Picard counts and the
Fig. 2 differences max_n ||T_m - T_0|| / ||T_0||.  (The device driver against the CPU oracle's driver is a
GPU test, tests/test_gpu_parity.py::test_heat_run_vs_oracle; tools never run the oracle.)
The paper's numbers (E5-2620, BoomerAMG-GMRES): 39.19 / 28.09 / 29.76 s, S 1.40 / 1.32, e 7.6e-9 / 7.0e-9.
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

nx = ny = int(dict(a.split("=") for a in sys.argv[1:] if "=" in a).get("n", 99))
steps = int(dict(a.split("=") for a in sys.argv[1:] if "=" in a).get("steps", 100))
T0 = torch.from_numpy(synth.heat_initial(nx, ny)).cuda()
res = {"grid": f"{nx}x{ny}", "steps": steps, "methods": {}}
fields = {}
for m in (0, 1, 2):
    T = T0.clone()
    diffs, per_all, eta_all, tot = [], [], [], 0.0
    its_l = its_g = 0
    for step in range(steps):      # step by step so that the Fig. 2 difference can be tracked
        T, per, eta, rep = lc.heat_run(nx, ny, T, 1, method=m, gs_sweeps=1 if m else 0)
        tot += rep.seconds
        its_l += rep.it_local; its_g += rep.it_global
        per_all.append(int(per[0])); eta_all.append(float(eta[0]))
        fields.setdefault(m, []).append(T.clone())
    res["methods"][f"method{m}"] = dict(seconds=tot, picard_total=sum(per_all), picard_per_step=per_all,
                                        eta_mean=float(np.mean(eta_all)) if m else 0.0,
                                        eta_first=eta_all[0], eta_last=eta_all[-1], it_local=its_l,
                                        it_global=its_g)
for m in (1, 2):
    d = [(torch.linalg.norm(a - b) / torch.linalg.norm(b)).item() for a, b in zip(fields[m], fields[0])]
    res["methods"][f"method{m}"]["fig2_max_rel_diff"] = max(d)
    res["methods"][f"method{m}"]["speedup"] = res["methods"]["method0"]["seconds"] / res["methods"][f"method{m}"]["seconds"]
print(json.dumps(res))
