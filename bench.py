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
    ap.add_argument("--tune", default="", help="lc_tuning fields for A/B runs, e.g. lazy_x_depth=2,pcg_tma=0")
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
    if world > 1:       # a stale liblc.so is rebuilt by rank 0 alone (the ranks share the tree)
        if rank == 0:
            lcbuild.build()
        dist.barrier()
    lcbuild.build()
    from paper_2001_01158_b200 import lc
    if args.tune:
        lc.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in args.tune.split(","))})

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

    def one_step(inp, out_x=None, rec=None, keep=False):
        A = lc.Matrix(sy0.nrows, inp["rp"], inp["ci"], inp["val"], block=sy0.block, batch=sy0.batch)
        nsolves = 0
        for name, rule in rules:
            x, rep = lc.local_method(A, inp["b"], inp["x0"], rule, method=method, rel_tol=EPS,
                                     gs_sweeps=args.gs if rule is not None else 0, keep=keep,
                                     timing=rec is not None)
            nsolves += sy0.batch
            if out_x is not None:
                out_x.append(x)
            if rec is not None:
                rec.append((name, rep))
        return nsolves

    # ---- the oracle baseline (rank 0, N = 1): complete oracle solves of the first system, one pinned process per
    # rule, started after the e2e leg (their host-memory traffic slows the pinned H2D copies the e2e leg times) and
    # running while the SpMV leg and the report run; they also check that system's GPU results
    cpu = None
    cpu_runs = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        runs, xs_ = {}, []
        one_step(dev_in[0], out_x=xs_, rec=(recs0 := []), keep=True)
        for (name, rep), x in zip(recs0, xs_):
            its = {"local": [i["iterations"] for i in rep.get("local", [])] or [0] * sy0.batch,
                   "global": [i["iterations"] for i in rep["global"]]}
            runs[name] = (x.cpu().numpy(), rep["idx"].cpu().numpy() if "idx" in rep else None, its)
        del xs_, recs0
        cpu_runs = runs

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

    # matrix once + pass A 32 B/row + pass B 64 B/row; a solve that updates x every L-th iteration
    # (lazy x of depth L, reported by lc_solve_info) moves (40 (L - 1) + 56 + 8 L) / L B/row in pass B on average
    def vec_bytes_of(L):
        return 32.0 + (40.0 * (L - 1) + 56.0 + 8.0 * L) / L if L > 1 else 96.0
    try:
        trafficdb = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except OSError:
        trafficdb = {}
    src_sha = lcbuild.source_sha256()
    # GMRES(m), low-sync CGS2 (R39): per Arnoldi step j: 8 nnz + 80 N + 16 (j+1) N bytes
    # (M^-1 apply 48 N; SpMV + w write + one V read for h and the Gram column; one merged update pass)
    m_restart = 30

    # the matrix term: the bytes one SpMV streams (lc_matrix_info; the 3T matrices' compact coupling copy: 21 of
    # the 45 stored values per cell are nonzero)
    gm_mat = float(Ainfo["matrix_bytes"]) if Ainfo["matrix_bytes"] > 0 else 8.0 * nnz

    def gmres_bytes(steps):
        tot, left = 0.0, steps
        while left > 0:
            L = min(m_restart, left)
            tot += L * (gm_mat + 80.0 * N) + 16.0 * N * L * (L + 1) / 2
            tot += gm_mat + 24.0 * N + (8.0 * L + 48.0) * N        # true residual + x update per cycle
            left -= L
        return tot
    by = {}
    pcg_bytes = 0.0
    pcg_sec = 0.0
    pcg_its = 0
    depths = set()
    for name, rep in reps:
        d = by.setdefault(name, dict(K=0, it_local=0, it_global=0, t_local=0.0, t_global=0.0, n=0,
                                     ms={"select": 0.0, "extract": 0.0, "local": 0.0, "gs": 0.0, "global": 0.0}))
        d["n"] += 1
        d["K"] += sum(rep["K"])
        for k, v in rep.get("ms", {}).items():
            d["ms"][k] += v
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
                depths.add(inf["lazy_x_depth"])
                pcg_bytes += inf["iterations"] * (mat_bytes + vec_bytes_of(inf["lazy_x_depth"]) * N) / sy0.batch
            else:
                pcg_bytes += gmres_bytes(inf["iterations"])
            pcg_its += inf["iterations"]
        pcg_sec += max(inf["seconds"] for inf in rep["global"])
    # per method: device-time breakdown (lc_solve_info kernel seconds), phase times on the stream (CUDA events:
    # select = Alg. 1 l.2, extract = l.3-4, local = l.5-6, global = l.8-11, launches and info reads included),
    # that method's own solves/s and the paper's speedup S = t_method0 / t_method
    t_m0 = sum(by["method0"]["ms"].values()) / by["method0"]["n"] if "method0" in by else None
    breakdown = {}
    for k, v in by.items():
        t_m = sum(v["ms"].values()) / v["n"]
        breakdown[k] = dict(eta=round(v["K"] / (v["n"] * N), 5), it_local=v["it_local"] / v["n"],
                            it_global=v["it_global"] / v["n"], ms_local=1e3 * v["t_local"] / v["n"],
                            ms_global=1e3 * v["t_global"] / v["n"],
                            phase_ms={p: round(t / v["n"], 3) for p, t in v["ms"].items()},
                            ms_total=round(t_m, 3), solves_per_s=round(sy0.batch * 1e3 / t_m, 3),
                            S=round(t_m0 / t_m, 3) if t_m0 else None)
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
        tr, tr_note = None, "no ncu capture for this config"
        tdb = trafficdb.get(f"{kname}@c{cfg}") or trafficdb.get(kname, {})
        if tdb and cfg == tdb.get("config") and Ainfo["layout"] == tdb.get("layout"):
            if tdb.get("source_sha256") == src_sha and sorted(depths) == tdb.get("lazy_x_depths", sorted(depths)):
                # measured DRAM bytes per iteration (ncu, this build) x the mean iterations per launch, like `achieved`
                tr = int(tdb["dram_bytes_per_iteration"] * pcg_its / max(nlaunch, 1))
                tr_note = tdb.get("source", "")
            else:
                tr_note = "profiles/ncu_traffic.json was measured on another build (source sha256 differs): dropped"
        roof = {"kernel": f"{kname} (global solves, one cooperative launch per solve)", "bound": "hbm",
                "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s", "frac": round(ach / hbm_peak, 4),
                "traffic": tr, "traffic_note": tr_note, "algorithmic_bytes_per_launch": int(pcg_bytes / max(nlaunch, 1)),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if peaks else "fallback 6650",
                "layout": Ainfo["layout"],
                "lazy_x_depths": sorted(depths),
                "bytes_rule": (f"{rule} + " + " / ".join(f"{vec_bytes_of(L):.2f}" for L in sorted(depths))
                               + " B/row vectors per PCG iteration (lazy-x depth " + "/".join(map(str, sorted(depths)))
                               + " as reported by lc_solve_info)" if solver == "pcg"
                               else f"{gm_mat / 1e6:.1f} MB matrix (lc_matrix_info: the compact 3T coupling copy when present) "
                               "+ 80 B/unknown + 16 (j+1) B/unknown per Arnoldi step j")}

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

    if cpu_runs is not None:
        cpu = CpuBaseline(cfg, sy0, rules, solver, args.gs, cpu_runs)
        cpu_runs = None
    parity = None
    if cpu is not None:
        cpu, parity = cpu.result()

    if rank == 0:
        line = {
            "metric": "linear solves/s (local character-based method + method0, FP64, rel. residual 1e-10)",
            "value": round(value, 4), "unit": "solves/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY 8(d))",
            "config": {"workload": WORKLOAD[cfg], "config_index": cfg, "n": n, "unknowns": N, "nnz": nnz,
                       "solves_per_step": len(rules) * sy0.batch, "methods": [r[0] for r in rules],
                       "systems": ids[args.warmup:], "rel_tol": EPS, "l2": "inputs > L2 (1.8 GB/system)",
                       "breakdown": breakdown, "gen_seconds": round(gen_s, 1),
                       "tuning": {k: v for k, v in lc.get_tuning().items() if lc.tuning_defaults()[k] != v}
                       or "library defaults"},
            "roofline": roof, "spmv": spmv, "cpu_baseline": cpu, "parity": parity, "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------- CPU oracle -----
# bench.py is the only product-side file that may execute oracle/ (its cpu_baseline leg and --impl reference).

def host_info():
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except (OSError, IndexError):
        model = "unknown"
    return {"cpu": model, "nproc": os.cpu_count()}


def sample_segments(G):
    """config 3: 4 of the G groups (first, last and two between: group sigma_g spans 4 decades, so iteration
    counts differ), else the whole system"""
    return sorted({0, G // 3, (2 * G) // 3, G - 1}) if G > 4 else list(range(G))


def _neighbours(A, u, cell):
    out = set()
    for a in range(cell):
        i = u * cell + a
        for k in range(A.rp[i], A.rp[i + 1]):
            v = int(A.ci[k]) // cell
            if v != u:
                out.add(v)
    return out


def cpu_worker(spec):
    """One complete oracle Alg. 1 (or method0) of one rule on the sampled segments of one system, pinned to one
    core (1 thread); compares the result with the GPU's run of the same system (Omega incl. near-threshold /
    cascade counts, iterations, x).  Prints one JSON line."""
    import oracle as orc
    try:
        os.sched_setaffinity(0, {spec["core"]})
    except (AttributeError, OSError):
        pass
    d = spec["dir"]
    ld = lambda k: np.load(os.path.join(d, k + ".npy"), mmap_mode="r")
    rp, ci, val, b, x0 = ld("rp"), ld("ci"), ld("val"), ld("b"), ld("x0")
    block, G, N = spec["block"], spec["batch"], len(b)
    Ao = orc.Csr.from_bsr(rp, ci, val) if block == 3 else orc.Csr(rp, ci, val)
    rule = spec["rule"]
    sp = orc.SolverParams(1 if spec["solver"] == "gmres" else 0, 3, 30, EPS, 3000 if spec["solver"] == "gmres" else 20000,
                          spec["gs"])
    xg = np.load(os.path.join(d, f"x_{spec['name']}.npy"), mmap_mode="r")
    gi_all = np.load(os.path.join(d, f"idx_{spec['name']}.npy")) if rule is not None else None
    its = json.load(open(os.path.join(d, f"its_{spec['name']}.json")))
    out = {"name": spec["name"], "core": spec["core"], "segments": spec["segments"], "seconds": 0.0,
           "phases": {"select": 0.0, "extract": 0.0, "local": 0.0, "global": 0.0}, "near": 0, "cascade": 0,
           "omega_bit_exact": True, "max_x_rel_err": 0.0, "max_it_local_diff": 0, "max_it_global_diff": 0}
    for g in spec["segments"]:
        r0, r1 = g * N // G, (g + 1) * N // G
        As = Ao.segment(r0, r1) if G > 1 else Ao
        bs_, x0s = np.ascontiguousarray(b[r0:r1]), np.ascontiguousarray(x0[r0:r1])
        dp = None
        if rule is not None:
            dp = orc.DomainParams(rule.get("criterion", 0), rule.get("threshold", 0), rule["param"],
                                  rule.get("expand_rounds", 0), rule.get("dilate_hops", 0), block)
        t0 = time.perf_counter()
        xo, flag, rep = orc.local_method(As, bs_, x0s, dp, sp)
        out["seconds"] += time.perf_counter() - t0
        for k, v in (("select", rep.t_select), ("extract", rep.t_extract), ("local", rep.t_local),
                     ("global", rep.t_global)):
            out["phases"][k] += v
        out["max_x_rel_err"] = max(out["max_x_rel_err"],
                                   float(np.linalg.norm(xg[r0:r1] - xo) / np.linalg.norm(xo)))
        out["max_it_global_diff"] = max(out["max_it_global_diff"], abs(its["global"][g] - rep.it_global))
        if rule is not None:
            gi = gi_all[(gi_all >= r0) & (gi_all < r1)] - r0
            ora = np.flatnonzero(flag)
            if its["local"][g] or rep.it_local:
                out["max_it_local_diff"] = max(out["max_it_local_diff"], abs(its["local"][g] - rep.it_local))
            if not np.array_equal(gi, ora):
                out["omega_bit_exact"] = False
                dd = orc.select_domain(As, bs_, x0s, rule.get("criterion", 0), rule.get("threshold", 0),
                                       rule["param"], rule.get("expand_rounds", 0), rule.get("dilate_hops", 0), block)
                gu, ou = set((gi[::block] // block).tolist()), set((ora[::block] // block).tolist())
                diff = gu ^ ou
                near = {u for u in diff if abs(dd.crit[u] - dd.tau) <= 1e-12 * dd.tau or
                        (np.isfinite(dd.adm[u]) and abs(dd.adm[u] - dd.tau) <= 1e-12 * dd.tau)}
                casc, fr = set(), set(near)
                for _ in range(8):
                    fr = {v for u in fr for v in _neighbours(As, u, block) if v in diff and v not in near | casc}
                    casc |= fr
                out["near"] += len(near)
                out["cascade"] += len(casc)
                out["outside_window"] = out.get("outside_window", 0) + len(diff - near - casc)
    print(json.dumps(out), flush=True)


class CpuBaseline:
    """The oracle (as it stands, single-threaded C) on one complete system of the workload: one process per
    rule, each pinned to its own host core, started while the GPU arm runs."""

    def __init__(self, cfg, sy, rules, solver, gs, gpu_runs):
        import tempfile
        self.dir = tempfile.mkdtemp(prefix="lc_cpu_")
        for k in ("rp", "ci", "val", "b", "x0"):
            np.save(os.path.join(self.dir, k + ".npy"), getattr(sy, k))
        self.segs = sample_segments(sy.batch)
        self.sy, self.cfg, self.rules = sy, cfg, rules
        ncores = os.cpu_count() or 1
        self.procs = []
        for j, (name, rule) in enumerate(rules):
            x, idx, its = gpu_runs[name]
            np.save(os.path.join(self.dir, f"x_{name}.npy"), x)
            if idx is not None:
                np.save(os.path.join(self.dir, f"idx_{name}.npy"), idx)
            json.dump(its, open(os.path.join(self.dir, f"its_{name}.json"), "w"))
            core = ncores - 1 - j if ncores > j + 1 else j % ncores
            spec = dict(dir=self.dir, name=name, rule=rule, solver=solver, gs=gs if rule is not None else 0,
                        block=sy.block, batch=sy.batch, segments=self.segs, core=core)
            self.procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), "--cpu-worker",
                                                json.dumps(spec)], stdout=subprocess.PIPE, text=True,
                                               env=dict(os.environ, OMP_NUM_THREADS="1")))

    def result(self):
        import shutil
        outs = []
        for p in self.procs:
            so, _ = p.communicate()
            if p.returncode != 0 or not so.strip():
                raise RuntimeError("oracle cpu worker failed")
            outs.append(json.loads(so.strip().splitlines()[-1]))
        shutil.rmtree(self.dir, ignore_errors=True)
        nsol = len(outs) * len(self.segs)
        tot = sum(o["seconds"] for o in outs)
        cb = {"value": round(nsol / tot, 6), "unit": "solves/s", "cores": 1, "kind": "oracle",
              "sample": (f"oracle (C, 1 thread per process) running COMPLETE Alg. 1 / method0 solves of system "
                         f"s={self.sy.s} of {WORKLOAD[self.cfg]}: {', '.join(n for n, _ in self.rules)}"
                         + (f" on groups {self.segs} of {self.sy.batch}" if self.sy.batch > 1 else "")
                         + f"; one process per rule, each pinned to its own core, concurrently with the GPU arm; "
                           f"value = solves / summed single-core seconds"),
              "measured_seconds": round(tot, 2), "host": host_info(),
              "processes": [{"rule": o["name"], "core": o["core"], "seconds": round(o["seconds"], 3),
                             "phases": {k: round(v, 3) for k, v in o["phases"].items()}} for o in outs]}
        parity = {o["name"]: {k: o[k] for k in ("omega_bit_exact", "near", "cascade", "max_x_rel_err",
                                                "max_it_local_diff", "max_it_global_diff") if k in o}
                  for o in outs}
        for o in outs:
            if "outside_window" in o:
                parity[o["name"]]["outside_window"] = o["outside_window"]
        return cb, {"system": self.sy.s, "segments": self.segs, "by_rule": parity}


def run_reference(args):
    """The reference arm: the oracle itself (no reference implementation exists; the reference is a paper).  Each
    step is ONE complete oracle Alg. 1 solve of the workload's cheapest rule (method2, or method1 for config 2) on
    system s_i (on 4 of the 20 groups for config 3), timed whole; every printed time was spent."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    import oracle as orc
    cfg = args.config
    n = args.n or synth.default_n(cfg)
    rules, solver = CFG_RULES[cfg]
    name, rule = rules[0]
    nsys = synth.default_systems(cfg)
    sp = orc.SolverParams(1 if solver == "gmres" else 0, 3, 30, EPS, 3000 if solver == "gmres" else 20000, 0)
    times, nsol = [], 0
    sys_done = []
    wall0 = time.perf_counter()
    for i in range(args.warmup + args.steps):
        sy = synth.system(cfg, (10 + i) % nsys, n=n)
        Ao = orc.Csr.from_bsr(sy.rp, sy.ci, sy.val) if sy.block == 3 else orc.Csr(sy.rp, sy.ci, sy.val)
        dp = orc.DomainParams(rule.get("criterion", 0), rule.get("threshold", 0), rule["param"],
                              rule.get("expand_rounds", 0), rule.get("dilate_hops", 0), sy.block)
        segs = sample_segments(sy.batch)
        t = 0.0
        for g in segs:
            r0, r1 = g * sy.N // sy.batch, (g + 1) * sy.N // sy.batch
            As = Ao.segment(r0, r1) if sy.batch > 1 else Ao
            t0 = time.perf_counter()
            orc.local_method(As, sy.b[r0:r1], sy.x0[r0:r1], dp, sp)
            t += time.perf_counter() - t0
        if i >= args.warmup:
            times.append(t)
            nsol += len(segs)
            sys_done.append(sy.s)
    total = float(sum(times))
    val = nsol / total
    line = {"impl": "reference", "metric": "linear solves/s (local character-based method + method0, FP64, "
            "rel. residual 1e-10)", "value": round(val, 6), "unit": "solves/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, SURVEY 8(d))",
            "config": {"workload": WORKLOAD[cfg], "config_index": cfg, "n": n, "systems": sys_done},
            "cpu_baseline": {"value": round(val, 6), "unit": "solves/s", "cores": 1, "kind": "oracle",
                             "host": host_info(),
                             "sample": f"per step one complete oracle Alg. 1 ({name}: domain, extraction, local "
                                       f"and global solve) of system s_i"
                                       + (f", groups {sample_segments(20)} of 20" if cfg == 3 else "")
                                       + "; every timed second was spent (no extrapolation)"},
            "wall_seconds": round(time.perf_counter() - wall0, 1),
            "e2e": {"value": round(val, 6), "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


if __name__ == "__main__":
    if len(sys.argv) == 3 and sys.argv[1] == "--cpu-worker":
        cpu_worker(json.loads(sys.argv[2]))
        sys.exit(0)
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_lc(a)
