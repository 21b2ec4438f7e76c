#!/usr/bin/env python3
"""Benchmark of the local character-based method's hot path on B200.

Workload: BASELINE.json configs[4], 3-D heat conduction 256^3
(16,777,216 unknowns, 117,047,296 stored nonzeros, FP64), systems s of the
seeded 20-step sequence (x0_s = x*_{s-1}).  One step = one system through
  - lc_create_csr   (CSR in HBM -> SELL-32)
  - method2: residual domain (tau = 1e-10 ||b||/sqrt(N), E_max = 1), extraction,
             local Jacobi-PCG, global Jacobi-PCG from x~       (rows a1,a3-a9)
  - method1: gradient domain (Eq. 5, alpha = 1e-4), same rest  (rows a2-a9)
  - method0: global Jacobi-PCG from x0                          (row a10)
each to ||b - A x|| <= 1e-10 ||b||.  value = linear solves per second (3 per step)
summed over ranks.  Inputs (1.8 GB per system) are far larger than L2 (126 MB).

python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config C]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

EPS = 1e-10
CFG_RULES = {
    # config: [(name, domain rule or None)], solver
    1: ([("method2", dict(criterion=0, threshold=1, param=1e-3)), ("method0", None)], "pcg"),
    2: ([("method1", dict(criterion=1, threshold=2, param=0.9, dilate_hops=2)), ("method0", None)], "pcg"),
    3: ([("method2", dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1)), ("method0", None)], "pcg"),
    4: ([("method2", dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1)), ("method0", None)], "gmres"),
    5: ([("method2", dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1)),
         ("method1", dict(criterion=1, threshold=1, param=1e-4)), ("method0", None)], "pcg"),
}
WORKLOAD = {1: "heat2d-64x64", 2: "heat2d-1024x1024", 3: "multigroup2d-512x512-G20", 4: "3T-512x512-bsr3",
            5: "heat3d-256^3"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lc", choices=["lc", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--n", type=int, default=None, help="grid override (testing only)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gs", type=int, default=0, help="Gauss-Seidel sweeps of Alg. 1 l.7 (paper: 1; parity path: 0)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def systems_for_rank(rank, count, nsys):
    """Weak scaling: rank r works on its own systems of the sequence (independent problems)."""
    return [(rank * 7 + i) % nsys for i in range(count)]


def aggregate(ms, solves, world, dist=None, device=None):
    """Whole-job throughput: max elapsed over ranks, sum of solves over ranks -> (ms_max, solves/s)."""
    import torch
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    n = torch.tensor([float(solves)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(n, op=dist.ReduceOp.SUM)
    return float(t.item()), float(n.item()) / (float(t.item()) * 1e-3)


# ----------------------------------------------------------------- clocks ---
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        try:
            p = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                  "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                                 stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        while not self._stop.is_set():
            line = p.stdout.readline()
            if not line:
                break
            self.rows.append([v.strip() for v in line.split(",")])
        p.terminate()

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(timeout=3)

    def summary(self):
        sm = []
        smax = None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1])); smax = float(r[2])
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- LC (GPU) -----
def run_lc(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world > 1:   # share the host cores between the ranks' OpenMP input generators (set before libgomp loads)
        os.environ.setdefault("OMP_NUM_THREADS", str(max(1, (os.cpu_count() or 8) // world)))
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2001_01158_b200 import build as lcbuild
    lcbuild.build()
    from paper_2001_01158_b200 import lc

    cfg = args.config
    n = args.n or synth.default_n(cfg)
    rules, solver = CFG_RULES[cfg]
    method = lc.GMRES if solver == "gmres" else lc.PCG
    nsys = synth.default_systems(cfg)
    ids = systems_for_rank(rank, args.warmup + args.steps, nsys)

    # ---- inputs resident in HBM before the timed region; host copies kept only for the e2e / cpu legs
    t0 = time.time()
    host = {}
    dev_in = []
    # host copies: the first system (cpu baseline, shapes) and the first two TIMED systems (the e2e loop feeds
    # those, so its iteration counts match the device-timed steps')
    e2e_ids = ids[args.warmup:args.warmup + 2] or ids[:2]
    keep = set(ids[:1]) | set(e2e_ids)
    for s in ids:
        sy = host[s] if s in host else synth.system(cfg, s, n=n)
        dev_in.append(dict(s=s, rp=torch.from_numpy(sy.rp).to(dev), ci=torch.from_numpy(sy.ci).to(dev),
                           val=torch.from_numpy(sy.val).to(dev), b=torch.from_numpy(sy.b).to(dev),
                           x0=torch.from_numpy(sy.x0).to(dev)))
        if s in keep:
            host[s] = sy
        del sy
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    sy0 = host[ids[0]]
    N = sy0.N
    nnz = len(sy0.ci) * sy0.block * sy0.block

    stream = torch.cuda.current_stream()

    def one_step(inp, out_x=None, rec=None):
        A = lc.Matrix(sy0.nrows, inp["rp"], inp["ci"], inp["val"], block=sy0.block, batch=sy0.batch)
        nsolves = 0
        for name, rule in rules:
            x, rep = lc.local_method(A, inp["b"], inp["x0"], rule, method=method, rel_tol=EPS,
                                     gs_sweeps=args.gs if rule is not None else 0)
            nsolves += sy0.batch
            if out_x is not None:
                out_x.append(x)
            if rec is not None:
                rec.append((name, rep))
        return nsolves

    # ---- warm-up
    for i in range(args.warmup):
        one_step(dev_in[i])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---- timed region (device events on the launching stream, inputs > L2)
    reps = []
    l0 = lc.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        solves = 0
        for i in range(args.steps):
            solves += one_step(dev_in[args.warmup + i], rec=reps)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = lc.kernel_launches() - l0
    ms = ev0.elapsed_time(ev1)
    ms_max, value = aggregate(ms, solves, world, dist, dev)

    # ---- per-method breakdown and roofline of the dominant kernel (global PCG launches on A)
    Ainfo = lc.Matrix(sy0.nrows, dev_in[0]["rp"], dev_in[0]["ci"], dev_in[0]["val"], block=sy0.block,
                      batch=sy0.batch).info()
    if Ainfo["layout"] == "symstencil":      # diagonal + upper values only: (nnz + N) / 2 stored values
        mat_bytes, rule = 8.0 * (nnz + N) / 2.0, "8 B x (nnz + N)/2 symmetric-stencil values"
    elif Ainfo["layout"] == "stencil":
        mat_bytes, rule = 8.0 * nnz, "8 B/nnz stencil values"
    else:
        mat_bytes, rule = 12.0 * nnz, "12 B/nnz SELL values + columns"
    # matrix once + pass A 32 B/row + pass B 64 B/row; single-segment solves update x every L-th
    # iteration (lazy x of depth L = 3: pass B 40, 40, 80 B/row, i.e. (40 (L - 1) + 56 + 8 L) / L on average)
    L = int(os.environ.get("LC_LAZY_X_DEPTH", "3"))
    lazy = solver == "pcg" and sy0.batch == 1 and not os.environ.get("LC_NO_LAZY_X") and L > 1
    vec_bytes = 32.0 + (40.0 * (L - 1) + 56.0 + 8.0 * L) / L if lazy else 96.0
    it_bytes = mat_bytes + vec_bytes * N
    try:
        trafficdb = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except OSError:
        trafficdb = {}
    # GMRES(m), low-sync CGS2 (R39): per Arnoldi step j: 8 nnz + 80 N + 16 (j+1) N bytes
    # (M^-1 apply 48 N; SpMV + w write + one V read for h and the Gram column; one merged update pass)
    m_restart = 30

    def gmres_bytes(steps):
        tot, left = 0.0, steps
        while left > 0:
            L = min(m_restart, left)
            tot += L * (8.0 * nnz + 80.0 * N) + 16.0 * N * L * (L + 1) / 2
            tot += 8.0 * nnz + 24.0 * N + (8.0 * L + 48.0) * N        # true residual + x update per cycle
            left -= L
        return tot
    by = {}
    pcg_bytes = 0.0
    pcg_sec = 0.0
    pcg_its = 0
    for name, rep in reps:
        d = by.setdefault(name, dict(K=0, it_local=0, it_global=0, t_local=0.0, t_global=0.0, n=0))
        d["n"] += 1
        d["K"] += sum(rep["K"])
        # a batched (config 3) solve is ONE launch for all groups: every group reports that launch's device
        # time, so the time is taken once (max), the iterations summed over the groups
        if rep.get("local"):
            d["t_local"] += max(inf["seconds"] for inf in rep["local"])
        for inf in rep.get("local", []):
            d["it_local"] += inf["iterations"]
        d["t_global"] += max(inf["seconds"] for inf in rep["global"])
        for inf in rep["global"]:
            d["it_global"] += inf["iterations"]
            if solver == "pcg":
                pcg_bytes += inf["iterations"] * it_bytes / sy0.batch
            else:
                pcg_bytes += gmres_bytes(inf["iterations"])
            pcg_its += inf["iterations"]
        pcg_sec += max(inf["seconds"] for inf in rep["global"])
    breakdown = {k: dict(eta=round(v["K"] / (v["n"] * N), 5), it_local=v["it_local"] / v["n"],
                         it_global=v["it_global"] / v["n"], ms_local=1e3 * v["t_local"] / v["n"],
                         ms_global=1e3 * v["t_global"] / v["n"]) for k, v in by.items()}
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    roof = None
    if pcg_sec > 0 and pcg_bytes > 0:
        ach = pcg_bytes / pcg_sec / 1e9
        nlaunch = len(reps)
        kname = "k_pcg" if solver == "pcg" else "k_gmres"
        tr = None
        if kname in trafficdb and cfg == 5 and Ainfo["layout"] == trafficdb[kname].get("layout"):
            # measured DRAM bytes per iteration (ncu) x the mean iterations per launch, like `achieved`
            tr = int(trafficdb[kname]["dram_bytes_per_iteration"] * pcg_its / max(nlaunch, 1))
        roof = {"kernel": f"{kname} (global solves, one cooperative launch per solve)", "bound": "hbm",
                "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s", "frac": round(ach / hbm_peak, 4),
                "traffic": tr, "algorithmic_bytes_per_launch": int(pcg_bytes / max(nlaunch, 1)),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if peaks else "fallback 6650",
                "layout": Ainfo["layout"],
                "bytes_rule": (f"{rule} + {vec_bytes:.2f} B/row vectors per PCG iteration" if solver == "pcg"
                               else "8 B/nnz + 80 B/unknown + 16 (j+1) B/unknown per Arnoldi step j")}

    # ---- the FP64 SpMV alone (BASELINE metric "SpMV HBM GB/s"): lc_spmv y = A x on the last system,
    # 20 calls timed with events on the launching stream (A, x, y = 0.9 GB + 0.27 GB at 256^3, > L2)
    spmv = None
    if sy0.batch >= 1:
        Asp = lc.Matrix(sy0.nrows, dev_in[-1]["rp"], dev_in[-1]["ci"], dev_in[-1]["val"], block=sy0.block,
                        batch=sy0.batch)
        xs_, ys_ = dev_in[-1]["x0"], torch.empty_like(dev_in[-1]["x0"])
        for _ in range(3):
            lc.spmv(Asp, xs_, ys_)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s0.record(stream)
        for _ in range(20):
            lc.spmv(Asp, xs_, ys_)
        s1.record(stream)
        torch.cuda.synchronize()
        t_sp = s0.elapsed_time(s1) / 1e3 / 20
        sp_bytes = mat_bytes + 16.0 * N
        spmv = {"kernel": "lc_spmv (k_spmv_stencil / k_spmv)", "bound": "hbm", "achieved": round(sp_bytes / t_sp / 1e9, 1),
                "peak": hbm_peak, "unit": "GB/s", "frac": round(sp_bytes / t_sp / 1e9 / hbm_peak, 4),
                "us_per_call": round(t_sp * 1e6, 2), "bytes_per_call": int(sp_bytes),
                "bytes_rule": f"{rule} + 16 B/row (x, y)"}
        del Asp

    # ---- e2e: host buffers through the C-ABI, H2D + D2H inside the timed region
    e2e = None
    if args.e2e_steps > 0:
        pins = []
        for i in range(len(e2e_ids)):
            sy = host[e2e_ids[i]]
            pins.append({k: torch.from_numpy(getattr(sy, k)).pin_memory() for k in ("rp", "ci", "val", "b", "x0")})
        h2d = sum(t.numel() * t.element_size() for t in pins[0].values())
        d2h = len(rules) * N * 8
        outs_host = [torch.empty(N, dtype=torch.float64).pin_memory() for _ in rules]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # H2D of step i+1 runs on a copy stream into one of two preallocated device input sets while step i
        # computes (the copies stay inside the timed region; the first one is not hidden), results go back
        # D2H on another stream behind each step; no allocation inside the timed loop
        h2d_stream, d2h_stream = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        bufs = [{k: torch.empty_like(v, device=dev) for k, v in pins[j % len(pins)].items()} for j in range(2)]
        freed = [None, None]                       # event: step using bufs[k] finished

        def prefetch(i):
            p, buf = pins[i % len(pins)], bufs[i % 2]
            with torch.cuda.stream(h2d_stream):
                if freed[i % 2] is not None:
                    h2d_stream.wait_event(freed[i % 2])
                for k, v in p.items():
                    buf[k].copy_(v, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d_stream)
            return buf, ev

        # this box's pinned H2D bandwidth (one copy of a step's inputs, outside the timed region): the e2e number
        # hides all but the first step's copy only while it is shorter than a step
        hb0, hb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        hb0.record(stream)
        for k, v in pins[0].items():
            bufs[0][k].copy_(v, non_blocking=True)
        hb1.record(stream)
        torch.cuda.synchronize()
        h2d_gbs = h2d / (hb0.elapsed_time(hb1) * 1e-3) / 1e9
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h2d_stream.wait_event(e0)
        sol = 0
        nxt = prefetch(0)
        for i in range(args.e2e_steps):
            inp, ev = nxt
            stream.wait_event(ev)
            if i + 1 < args.e2e_steps:
                nxt = prefetch(i + 1)
            xs = []
            sol += one_step(inp, out_x=xs)
            done = torch.cuda.Event()
            done.record(stream)
            freed[i % 2] = done
            d2h_stream.wait_event(done)
            with torch.cuda.stream(d2h_stream):
                for xo, xh in zip(xs, outs_host):
                    xh.copy_(xo, non_blocking=True)
                    xo.record_stream(d2h_stream)
        stream.wait_stream(d2h_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        _, evalue = aggregate(e0.elapsed_time(e1), sol, world, dist, dev)
        e2e = {"value": round(evalue, 4), "unit": "solves/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "h2d_gbs_measured": round(h2d_gbs, 1)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, n, host[ids[0]], breakdown, rules, solver)

    if rank == 0:
        line = {
            "metric": "linear solves/s (local character-based method + method0, FP64, rel. residual 1e-10)",
            "value": round(value, 4), "unit": "solves/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY 8(d))",
            "config": {"workload": WORKLOAD[cfg], "config_index": cfg, "n": n, "unknowns": N, "nnz": nnz,
                       "solves_per_step": len(rules) * sy0.batch, "methods": [r[0] for r in rules],
                       "systems": ids[args.warmup:], "rel_tol": EPS, "l2": "inputs > L2 (1.8 GB/system)",
                       "breakdown": breakdown, "gen_seconds": round(gen_s, 1)},
            "roofline": roof, "spmv": spmv, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------- CPU oracle -----
def oracle_sample(cfg, n, sy, rules, solver, pcg_iters=3):
    """Time the oracle (as it stands, 1 thread) on a bounded sample of one system and scale it to
    solves/s: full-size domain selection + extraction per rule, plus `pcg_iters` Krylov iterations
    whose per-iteration cost is multiplied by the iteration counts the solves need."""
    import oracle as orc
    A = orc.Csr.from_bsr(sy.rp, sy.ci, sy.val) if sy.block == 3 else orc.Csr(sy.rp, sy.ci, sy.val)
    t = {}
    for name, rule in rules:
        if rule is None:
            continue
        t0 = time.perf_counter()
        d = orc.select_domain(A, sy.b, sy.x0, rule.get("criterion", 0), rule.get("threshold", 0), rule["param"],
                              rule.get("expand_rounds", 0), rule.get("dilate_hops", 0), sy.block)
        t1 = time.perf_counter()
        orc.extract(A, sy.b, sy.x0, d.flag)
        t2 = time.perf_counter()
        t[name] = (t1 - t0, t2 - t1, d.K / A.n)
    t0 = time.perf_counter()
    if solver == "pcg":
        orc.pcg(A, sy.b, sy.x0, eps=EPS, max_iters=pcg_iters)
    else:
        orc.gmres_bj(A, sy.b, sy.x0, bs=3, eps=EPS, max_iters=pcg_iters)
    t_it = (time.perf_counter() - t0) / pcg_iters
    return t, t_it


def cpu_baseline(cfg, n, sy, breakdown, rules, solver):
    t, t_it = oracle_sample(cfg, n, sy, rules, solver)
    t_it /= sy.batch          # the sample iterates over all G groups; the counts below are per group, summed
    total = 0.0
    for name, rule in rules:
        bd = breakdown.get(name, {})
        it_l, it_g = bd.get("it_local", 0.0), bd.get("it_global", 0.0)
        eta = t.get(name, (0, 0, 0))[2]
        sel = t.get(name, (0, 0, 0))[0] + t.get(name, (0, 0, 0))[1]
        total += sel + t_it * (eta * it_l + it_g)
    nsol = len(rules) * sy.batch
    return {"value": round(nsol / total, 6), "unit": "solves/s", "cores": 1, "kind": "oracle",
            "sample": (f"oracle (C, 1 thread) on system s={sy.s} of {WORKLOAD[cfg]}: full-size domain selection + "
                       f"extraction per rule timed, plus 3 Krylov iterations timed ({t_it:.3f} s/iteration) and "
                       f"scaled by the iteration counts of this run (local iterations weighted by eta; per group for G > 1)")}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    cfg = args.config
    n = args.n or synth.default_n(cfg)
    rules, solver = CFG_RULES[cfg]
    sy = synth.system(cfg, 10 % synth.default_systems(cfg), n=n)
    # the oracle's own full-size iteration counts are too slow to run every step; take the
    # per-iteration cost from each sample and the iteration counts from one oracle-complete run
    # on a system of the same sequence at the reduced grid n/8 scaled by sqrt(N) growth is NOT used:
    # counts come from the GPU-free estimate of Jacobi-PCG below (documented in DESIGN.md s8).
    it_est = {"pcg": 120, "gmres": 200}[solver]
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        t, t_it = oracle_sample(cfg, n, sy, rules, solver, pcg_iters=2)
        el = time.perf_counter() - t0
        total = sum(v[0] + v[1] for v in t.values()) + t_it * it_est * len(rules)
        if i >= args.warmup:
            times.append(total)
        _ = el
    mean = float(np.mean(times))
    nsol = len(rules) * sy.batch
    val = nsol / mean
    line = {"impl": "reference", "metric": "linear solves/s (local character-based method + method0, FP64, "
            "rel. residual 1e-10)", "value": round(val, 6), "unit": "solves/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(mean * 1e3, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, SURVEY 8(d))",
            "config": {"workload": WORKLOAD[cfg], "config_index": cfg, "n": n},
            "cpu_baseline": {"value": round(val, 6), "unit": "solves/s", "cores": 1, "kind": "oracle",
                             "sample": f"per step: full-size domain selection + extraction per rule and 2 timed "
                                       f"Krylov iterations of the oracle, scaled to {it_est} iterations per solve"},
            "e2e": {"value": round(val, 6), "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_lc(a)
