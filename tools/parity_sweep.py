#!/usr/bin/env python3
"""Full-size parity sweep: EVERY system of the five BASELINE configs, at BASELINE size, through the C-ABI
path and through the CPU oracle, compared per system, per rule and per segment (group) with the bars of
BASELINE.json's north_star / SURVEY 8(c) C-P:

  - Omega bit-exact, except units whose criterion / admission value lies within 1e-12 relative of tau
    ("near") and differences inherited from those through growth ("cascade"): both counted and reported;
  - tau within 1e-14 relative (double-double rounding, R23), criterion values bit-exact;
  - b_sub and x_B0 of Eq. 3 bit-exact (same fma chains, R22) where the sets agree;
  - x~ of Eq. 4 within 1e-9 relative of the oracle's x~, its complement bitwise x0;
  - local and global iteration counts within +-1 (R30);
  - the final x within 1e-9 relative, Eq. 6 re-checked with the oracle's residual, plus method0.

Each worker process pins itself to one host core, generates its system (single-threaded), runs the GPU path
(the GPU is time-sliced between the workers; nothing here is timed on it), then the oracle (Alg. 1 as
or_local_method, one thread), and compares.  The oracle's per-phase times (P:995-1001's CPU_loc-constr /
local / global split) are recorded too.

python tools/parity_sweep.py [--configs 1,2,3,4,5] [--systems 0,1,...] [--workers 15] [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

EPS = 1e-10
# domain rules per config (readings R13-R16); every system also runs method0
RULES = {
    1: [("method2", dict(criterion=0, threshold=1, param=1e-3, expand_rounds=0, dilate_hops=0))],
    2: [("method1", dict(criterion=1, threshold=2, param=0.9, expand_rounds=0, dilate_hops=2))],
    3: [("method2", dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1, dilate_hops=0))],
    4: [("method2", dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1, dilate_hops=0))],
    5: [("method2", dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1, dilate_hops=0)),
        ("method1", dict(criterion=1, threshold=1, param=1e-4, expand_rounds=0, dilate_hops=0))],
}
COST = {5: 200.0, 3: 170.0, 2: 50.0, 4: 10.0, 1: 0.1}     # rough oracle seconds per system (ordering only)

_core = None


def _init(counter, lock, ncores):
    global _core
    with lock:
        _core = counter.value % ncores
        counter.value += 1
    try:
        os.sched_setaffinity(0, {_core})
    except (AttributeError, OSError):
        pass


def _neighbours(A, u, cell):
    out = set()
    for a in range(cell):
        i = u * cell + a
        for k in range(A.rp[i], A.rp[i + 1]):
            v = int(A.ci[k]) // cell
            if v != u:
                out.add(v)
    return out


def _compare_sets(A, gpu_units, d, cell, tol=1e-12):
    import numpy as np
    ora = np.flatnonzero(d.flag.reshape(-1, cell)[:, 0])
    diff = sorted(set(map(int, gpu_units)) ^ set(map(int, ora)))
    near = set()
    for u in diff:
        c, a = d.crit[u], d.adm[u]
        if abs(c - d.tau) <= tol * abs(d.tau) or (np.isfinite(a) and abs(a - d.tau) <= tol * abs(d.tau)):
            near.add(u)
    cascade, frontier = set(), set(near)
    for _ in range(8):
        nxt = set()
        for u in frontier:
            for v in _neighbours(A, u, cell):
                if v in diff and v not in near and v not in cascade:
                    cascade.add(v); nxt.add(v)
        frontier = nxt
    bad = [u for u in diff if u not in near and u not in cascade]
    return len(near), len(cascade), bad


def run_system(task):
    cfg, s = task
    import numpy as np
    import torch

    import oracle as orc
    import synth
    from paper_2001_01158_b200 import lc

    t0 = time.time()
    sy = synth.system(cfg, s)
    cell, N, G = sy.block, sy.N, sy.batch
    method = lc.GMRES if cfg == 4 else lc.PCG
    dev = torch.device("cuda")
    # ---------------- GPU path (C-ABI), everything kept on the host afterwards
    A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=sy.block, batch=sy.batch)
    b, x0 = torch.from_numpy(sy.b).to(dev), torch.from_numpy(sy.x0).to(dev)
    gpu = {}
    for name, rule in RULES[cfg]:
        # tau, the criterion and Eq. 3 from the step-by-step calls; x, x~, Omega and the iterations from Alg. 1 in
        # one call (lc_local_method)
        dom = lc.select_domain(A, b, x0, **rule)
        _, tau, crit, _ = dom.export(want_crit=True)
        crit = crit.cpu().numpy()
        bsub = xb0 = None
        if sum(dom.K) > 0:
            sub = lc.extract_sub(A, dom, b, x0)
            bsub, xb0 = (t.cpu().numpy() for t in sub.export())
            del sub
        del dom
        x, rep = lc.local_method(A, b, x0, rule, method=method, rel_tol=EPS, keep=True)
        gpu[name] = dict(x=x.cpu().numpy(), xt=rep["xt"].cpu().numpy(), idx=rep["idx"].cpu().numpy(),
                         tau=list(tau), K=list(rep["K"]), crit=crit, bsub=bsub, xB0=xb0,
                         it_local=[i["iterations"] for i in rep.get("local", [])] or [0] * G,
                         it_global=[i["iterations"] for i in rep["global"]],
                         st_global=[i["status"] for i in rep["global"]])
        del x, rep
    x, rep = lc.local_method(A, b, x0, None, method=method, rel_tol=EPS)
    gpu["method0"] = dict(x=x.cpu().numpy(), it_global=[i["iterations"] for i in rep["global"]],
                          st_global=[i["status"] for i in rep["global"]])
    del x, rep, A, b, x0
    torch.cuda.synchronize()
    t_gpu = time.time() - t0
    # ---------------- oracle, segment by segment, and the comparison
    Ao = orc.Csr.from_bsr(sy.rp, sy.ci, sy.val) if cell == 3 else orc.Csr(sy.rp, sy.ci, sy.val)
    sp = orc.SolverParams(1 if cfg == 4 else 0, 3, 30, EPS, 3000 if cfg == 4 else 20000, 0)
    recs = []
    for name in [r[0] for r in RULES[cfg]] + ["method0"]:
        rule = dict(RULES[cfg])[name] if name != "method0" else None
        gr = gpu[name]
        off = 0
        for g in range(G):
            r0, r1 = g * N // G, (g + 1) * N // G
            As = Ao.segment(r0, r1) if G > 1 else Ao
            bs_, x0s = sy.b[r0:r1], sy.x0[r0:r1]
            rec = dict(config=cfg, s=s, rule=name, segment=g, rows=r1 - r0, fail=[])
            if rule is not None:
                dp = orc.DomainParams(rule["criterion"], rule["threshold"], rule["param"], rule["expand_rounds"],
                                      rule["dilate_hops"], cell)
                d = orc.select_domain(As, bs_, x0s, rule["criterion"], rule["threshold"], rule["param"],
                                      rule["expand_rounds"], rule["dilate_hops"], cell)
                Kg = gr["K"][g]
                gi = gr["idx"][off:off + Kg]
                units = (gi[::cell] - r0) // cell
                rec.update(K_gpu=int(Kg), K_oracle=int(d.K), eta=round(Kg / (r1 - r0), 6), tau=d.tau)
                rec["tau_rel_diff"] = abs(gr["tau"][g] - d.tau) / abs(d.tau) if d.tau else abs(gr["tau"][g])
                if rec["tau_rel_diff"] > 1e-14:
                    rec["fail"].append("tau")
                if not np.array_equal(gr["crit"][r0 // cell:r1 // cell], d.crit):
                    rec["fail"].append("criterion values")
                if len(gi) > 1 and not np.all(np.diff(gi) > 0):
                    rec["fail"].append("Omega not ascending")
                near, casc, bad = _compare_sets(As, units, d, cell)
                rec.update(near=near, cascade=casc, set_diff_outside_window=len(bad))
                if bad:
                    rec["fail"].append(f"{len(bad)} Omega differences outside the 1e-12 window")
                same = np.array_equal(gi - r0, np.flatnonzero(d.flag))
                rec["omega_bit_exact"] = bool(same)
                xt = gr["xt"][r0:r1]
                comp = np.ones(r1 - r0, bool)
                comp[gi - r0] = False
                rec["complement_bitwise_x0"] = bool(np.array_equal(xt[comp], x0s[comp]))
                if not rec["complement_bitwise_x0"]:
                    rec["fail"].append("x~ complement != x0")
                if same and Kg > 0:
                    so = orc.extract(As, bs_, x0s, d.flag)
                    rec["bsub_bit_exact"] = bool(np.array_equal(gr["bsub"][off:off + Kg], so.bsub))
                    rec["xB0_bit_exact"] = bool(np.array_equal(gr["xB0"][off:off + Kg], so.xB0))
                    if not rec["bsub_bit_exact"]:
                        rec["fail"].append("b_sub")
                    if not rec["xB0_bit_exact"]:
                        rec["fail"].append("x_B0")
                    del so
                off += Kg
                xo, _, ro, xto = orc.local_method(As, bs_, x0s, dp, sp, want_xt=True)
                if same:
                    rec["xt_rel_err"] = float(np.linalg.norm(xt - xto) / np.linalg.norm(xto))
                    if rec["xt_rel_err"] > 1e-9:
                        rec["fail"].append("x~")
                rec.update(it_local_gpu=gr["it_local"][g], it_local_oracle=ro.it_local)
                if Kg > 0 and d.K > 0 and abs(gr["it_local"][g] - ro.it_local) > 1:
                    rec["fail"].append("local iterations")
            else:
                xo, _, ro = orc.local_method(As, bs_, x0s, None, sp)
            rec.update(it_global_gpu=gr["it_global"][g], it_global_oracle=ro.it_global,
                       oracle_seconds={"select": ro.t_select, "extract": ro.t_extract, "local": ro.t_local,
                                       "global": ro.t_global})
            if abs(gr["it_global"][g] - ro.it_global) > 1:
                rec["fail"].append("global iterations")
            xs = gr["x"][r0:r1]
            rec["x_rel_err"] = float(np.linalg.norm(xs - xo) / np.linalg.norm(xo))
            if rec["x_rel_err"] > 1e-9:
                rec["fail"].append("x")
            res = float(np.linalg.norm(orc.residual(As, bs_, xs)))
            rec["eq6_rel_residual"] = res / float(np.linalg.norm(bs_))
            if res > EPS * np.linalg.norm(bs_) * (1 + 1e-6) or gr["st_global"][g] != 0:
                rec["fail"].append("Eq. 6")
            recs.append(rec)
    return dict(config=cfg, s=s, core=_core, t_gpu=round(t_gpu, 2), t_total=round(time.time() - t0, 2),
                records=recs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--systems", default=None, help="comma list of system indices (default: all)")
    ap.add_argument("--workers", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity_sweep.json"))
    args = ap.parse_args()
    os.environ["OMP_NUM_THREADS"] = "1"            # single-threaded generator in every pinned worker
    import synth
    tasks = []
    for c in [int(v) for v in args.configs.split(",")]:
        ss = [int(v) for v in args.systems.split(",")] if args.systems else range(synth.default_systems(c))
        tasks += [(c, s) for s in ss if s < synth.default_systems(c)]
    tasks.sort(key=lambda t: -COST[t[0]])
    ctx = mp.get_context("spawn")
    counter, lock = ctx.Value("i", 0), ctx.Lock()
    ncores = os.cpu_count() or 1
    t0 = time.time()
    results = []
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with ctx.Pool(args.workers, initializer=_init, initargs=(counter, lock, ncores), maxtasksperchild=4) as pool:
        for r in pool.imap_unordered(run_system, tasks):
            results.append(r)
            nf = sum(1 for rec in r["records"] if rec["fail"])
            print(f"[{time.time() - t0:7.1f}s] config {r['config']} s={r['s']}: {len(r['records'])} records, "
                  f"{nf} failing, gpu {r['t_gpu']} s, total {r['t_total']} s", flush=True)
    recs = [rec for r in results for rec in r["records"]]
    summary = {}
    for c in sorted({r["config"] for r in recs}):
        rc = [r for r in recs if r["config"] == c]
        summary[c] = dict(
            systems=len({r["s"] for r in rc}), records=len(rc), failures=sum(1 for r in rc if r["fail"]),
            near=sum(r.get("near", 0) for r in rc), cascade=sum(r.get("cascade", 0) for r in rc),
            omega_bit_exact=sum(1 for r in rc if r.get("omega_bit_exact")),
            omega_records=sum(1 for r in rc if "omega_bit_exact" in r),
            max_x_rel_err=max(r["x_rel_err"] for r in rc),
            max_xt_rel_err=max([r["xt_rel_err"] for r in rc if "xt_rel_err" in r] or [0.0]),
            max_it_global_diff=max(abs(r["it_global_gpu"] - r["it_global_oracle"]) for r in rc),
            max_it_local_diff=max([abs(r["it_local_gpu"] - r["it_local_oracle"]) for r in rc
                                   if "it_local_gpu" in r and r["K_gpu"] > 0] or [0]),
            oracle_seconds=round(sum(sum(r["oracle_seconds"].values()) for r in rc), 1))
    try:
        cpu_model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except (OSError, IndexError):
        cpu_model = platform.processor()
    out = dict(tool="tools/parity_sweep.py", host=dict(cpu=cpu_model, nproc=os.cpu_count(), workers=args.workers,
                                                       oracle_threads_per_worker=1),
               wall_seconds=round(time.time() - t0, 1), bars=dict(omega="bit-exact outside 1e-12 of tau",
                                                                  tau_rel=1e-14, xt_rel=1e-9, x_rel=1e-9,
                                                                  iterations=1, bsub="bit-exact"),
               summary=summary, failures=[r for r in recs if r["fail"]], records=recs)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1, default=float)
    print(json.dumps(dict(summary=summary, failures=len(out["failures"]), wall=out["wall_seconds"])))
    return 1 if out["failures"] else 0


if __name__ == "__main__":
    sys.exit(main())
