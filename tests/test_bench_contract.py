"""bench.py's JSON contract on CPU: the reference arm (the oracle, `--impl reference`) on the small config 1,
and the rank-0-only rule under a multi-rank launch (other ranks print nothing and exit 0)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = dict(os.environ, **(env_extra or {}))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    return out


def test_reference_arm_json_line():
    out = _run(["--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "1"])
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["steps"] == 2 and line["warmup"] == 1 and line["n_gpus"] == 1
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    e2e = line["e2e"]
    assert e2e["value"] == line["value"] and e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0
    assert line["config"]["workload"]


def test_reference_arm_other_ranks_silent():
    out = _run(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "1"],
               {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip() == ""


def test_cpu_baseline_workers():
    """The cpu_baseline leg's pinned oracle processes (host logic only): fed the oracle's own results as the
    'GPU' side, they time complete solves and report exact parity (no near / cascade differences)."""
    sys.path.insert(0, ROOT)
    import numpy as np

    import bench
    import oracle as orc
    import synth
    sy = synth.system(1, 4)
    rules, solver = bench.CFG_RULES[1]
    A = orc.Csr(sy.rp, sy.ci, sy.val)
    runs = {}
    for name, rule in rules:
        sp = orc.SolverParams(0, 1, 30, 1e-10, 20000, 0)
        if rule is None:
            x, _, rep = orc.local_method(A, sy.b, sy.x0, None, sp)
            runs[name] = (x, None, {"local": [0], "global": [rep.it_global]})
        else:
            dp = orc.DomainParams(rule["criterion"], rule["threshold"], rule["param"], 0, 0, 1)
            x, flag, rep = orc.local_method(A, sy.b, sy.x0, dp, sp)
            runs[name] = (x, np.flatnonzero(flag).astype(np.int32), {"local": [rep.it_local], "global": [rep.it_global]})
    cb, parity = bench.CpuBaseline(1, sy, rules, solver, 0, runs).result()
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["value"] > 0
    assert len(cb["processes"]) == len(rules) and cb["host"]["nproc"] >= 1
    for name, _ in rules:
        p = parity["by_rule"][name]
        assert p["max_x_rel_err"] == 0.0 and p["max_it_global_diff"] == 0
    assert parity["by_rule"]["method2"]["omega_bit_exact"] and parity["by_rule"]["method2"]["near"] == 0


def test_traffic_stamp_file():
    """profiles/ncu_traffic.json (roofline.traffic's source): one entry per measured config under the key bench.py
    looks up (kernel@cCONFIG), each stamped with the source hash of the build it measured and positive bytes."""
    db = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    assert "k_pcg@c5" in db                                     # the default bench's config
    for key, e in db.items():
        assert e["dram_bytes_per_iteration"] > 0 and len(e["source_sha256"]) == 64 and e["source"]
        if "@c" in key:
            kname, c = key.split("@c")
            assert int(c) == e["config"] and kname in ("k_pcg", "k_gmres")
            assert (kname == "k_gmres") == (e["config"] == 4)
