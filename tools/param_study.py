#!/usr/bin/env python3
"""NEXT-3: parameter studies of the local character-based method on the GPU path
(PAPER.md s3.5).

  alpha study  (method1, Alg. 2): alpha in {1, 1e-1, ..., 1e-11} on two multi-group systems
               (config 3 groups g = 0 and g = 15, stand-ins for T1000N1S0G0 / G55);
  E_max study  (method2, Alg. 3): E_max in {0, ..., 6} on two 3T systems (config 4, s = 0 and s = 20,
               stand-ins for t20000 / t80000).

For each parameter value: eta = K/N, local / global iterations and device times, whether x~ (after the
local solve, before any global iteration) already satisfies Eq. 6, and S = t_method0 / t_local_method.
alpha_opt follows the reading R37 of P:1582-1587: the LARGEST alpha of the grid whose x~ satisfies Eq. 6.
Prints one JSON object per study (the committed copy lives in profiles/).
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

EPS = 1e-10
ALPHAS = [10.0 ** -k for k in range(0, 12)]
EMAXS = list(range(0, 7))


def group_system(sy, g):
    """Segment g of a block-diagonal config-3 system as its own CSR system."""
    n = sy.nrows // sy.batch
    r0, r1 = g * n, (g + 1) * n
    k0, k1 = sy.rp[r0], sy.rp[r1]
    return dict(n=n, rp=sy.rp[r0:r1 + 1] - k0, ci=sy.ci[k0:k1] - r0, val=sy.val[k0:k1], b=sy.b[r0:r1],
                x0=sy.x0[r0:r1], block=1)


def run_case(A, b, x0, rule, method, it_m0, t_m0):
    """One local-method solve with the device time of each phase (CUDA events around the calls)."""
    t0 = time.perf_counter()
    x, rep = lc.local_method(A, b, x0, rule, method=method, rel_tol=EPS)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    t_loc = sum(i["seconds"] for i in rep.get("local", [])[:1])
    t_glb = rep["global"][0]["seconds"]
    # does x~ (local solve only) satisfy Eq. 6?  -> a global solve with max_iters = 0 reports it
    xt = x0.clone()
    if rule is not None and sum(rep["K"]) > 0:
        dom = lc.select_domain(A, b, x0, **rule)
        sub = lc.extract_sub(A, dom, b, x0)
        lc.solve_local(sub, xt, method=method, rel_tol=EPS)
    chk = lc.solve_global(A, b, xt, method=method, rel_tol=EPS, max_iters=0)
    return dict(eta=sum(rep["K"]) / A.N, it_local=rep.get("local", [{"iterations": 0}])[0]["iterations"],
                it_global=rep["global"][0]["iterations"], ms_local=1e3 * t_loc, ms_global=1e3 * t_glb,
                xtilde_converged=chk[0]["status"] == 0, xtilde_relres=chk[0]["rel_residual"],
                speedup=t_m0 / max(t_loc + t_glb, 1e-12), wall_s=wall)


def study_alpha():
    out = []
    sy = synth.system(3, 10)
    for g in (0, 15):
        gs = group_system(sy, g)
        A = lc.Matrix(gs["n"], gs["rp"], gs["ci"], gs["val"])
        b = torch.from_numpy(gs["b"]).cuda()
        x0 = torch.from_numpy(gs["x0"]).cuda()
        x, r0 = lc.local_method(A, b, x0, None, rel_tol=EPS)
        t_m0, it_m0 = r0["global"][0]["seconds"], r0["global"][0]["iterations"]
        rows = []
        for a in ALPHAS:
            res = run_case(A, b, x0, dict(criterion=1, threshold=1, param=a), lc.PCG, it_m0, t_m0)
            res["alpha"] = a
            rows.append(res)
        conv = [r["alpha"] for r in rows if r["xtilde_converged"]]
        best = max(rows, key=lambda r: r["speedup"])
        out.append(dict(study="alpha", system=f"config3 s=10 group {g}", method0_it=it_m0,
                        method0_ms=1e3 * t_m0, rows=rows, alpha_opt_R37=max(conv) if conv else None,
                        alpha_best_speedup=best["alpha"], best_speedup=best["speedup"]))
    return out


def study_emax():
    out = []
    for s in (0, 20):
        sy = synth.system(4, s)
        A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=3)
        b = torch.from_numpy(sy.b).cuda()
        x0 = torch.from_numpy(sy.x0).cuda()
        x, r0 = lc.local_method(A, b, x0, None, method=lc.GMRES, rel_tol=EPS)
        t_m0, it_m0 = r0["global"][0]["seconds"], r0["global"][0]["iterations"]
        rows = []
        for em in EMAXS:
            res = run_case(A, b, x0, dict(criterion=0, threshold=0, param=EPS, expand_rounds=em), lc.GMRES,
                           it_m0, t_m0)
            res["E_max"] = em
            rows.append(res)
        best = max(rows, key=lambda r: r["speedup"])
        out.append(dict(study="E_max", system=f"config4 s={s}", method0_it=it_m0, method0_ms=1e3 * t_m0,
                        rows=rows, E_max_best_speedup=best["E_max"], best_speedup=best["speedup"]))
    return out


if __name__ == "__main__":
    which = sys.argv[1:] or ["alpha", "emax"]
    res = []
    if "alpha" in which:
        res += study_alpha()
    if "emax" in which:
        res += study_emax()
    for r in res:
        print(json.dumps(r))
