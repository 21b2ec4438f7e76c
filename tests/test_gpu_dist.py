"""GPU parity of the row-partitioned form (NEXT-4, Sec. 2.4 / Alg. 4-5) against the CPU oracle.

p ranks are emulated on the one GPU (lc_dist_connect_local: one cooperative launch runs every rank's CTAs,
halo rows are read from the neighbour slab's workspace and every reduction goes through the ranks'
exchange blocks, exactly the code a one-GPU-per-rank run executes).  Bars as tests/test_gpu_parity.py:
index sets bit-exact outside the 1e-12 window of tau, iterations +-1, solutions within 1e-9 relative, plus
Eq. 6 re-checked.  The distributed Omega must equal the one Alg. 3 / Alg. 2 finds on the whole matrix
(R40: the expansion stops on the GLOBAL admission count).
"""
import numpy as np
import pytest

import oracle as orc
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2001_01158_b200 import build as lcbuild
    from paper_2001_01158_b200 import dist as ldist
    from paper_2001_01158_b200 import lc
    lcbuild.build()

from test_gpu_parity import compare_sets  # noqa: E402

EPS = 1e-10
DEV = "cuda"

R_RES = dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1, dilate_hops=0)
R_GRAD = dict(criterion=1, threshold=1, param=1e-4, expand_rounds=0, dilate_hops=0)
R_C1 = dict(criterion=0, threshold=1, param=1e-3, expand_rounds=0, dilate_hops=0)
R_C2 = dict(criterion=1, threshold=1, param=1e-2, expand_rounds=0, dilate_hops=2)


def make_ranks(sy, P, align=32, R=None):
    R = R or ldist.split_rows(sy.nrows, P, align)
    ranks = []
    for l in range(P):
        rp, ci, va = ldist.slab_csr(sy.rp, sy.ci, sy.val, R[l], R[l + 1])
        ranks.append(lc.DistRank(sy.nrows, R[l], R[l + 1] - R[l], l, P, rp, ci, va))
    lc.dist_connect_local(ranks)
    return ranks, R


def slabs(v, R):
    return [torch.from_numpy(np.ascontiguousarray(v[R[l]:R[l + 1]])).to(DEV) for l in range(len(R) - 1)]


def gather(ts):
    return np.concatenate([t.cpu().numpy() for t in ts])


def run_and_check(sy, rule, P, align=32, R=None):
    Ao = orc.Csr(sy.rp, sy.ci, sy.val)
    ranks, R = make_ranks(sy, P, align, R)
    b, x0 = slabs(sy.b, R), slabs(sy.x0, R)
    x, rep = lc.dist_local_method(ranks, b, x0, rule, rel_tol=EPS)
    xg = gather(x)
    sp = orc.SolverParams(0, 3, 30, EPS, 20000)
    if rule is None:
        xo, _, ro = orc.local_method(Ao, sy.b, sy.x0, None, sp)
    else:
        d = orc.select_domain(Ao, sy.b, sy.x0, rule["criterion"], rule["threshold"], rule["param"],
                              rule["expand_rounds"], rule["dilate_hops"], 1)
        fl = [r.domain_flags() for r in ranks]
        idx = np.concatenate([ldist.omega_from_flags(f.cpu().numpy(), r.row0) for (f, _), r in zip(fl, ranks)])
        assert rep["K"] == idx.size
        for _, tau in fl:
            assert tau == pytest.approx(d.tau, rel=1e-14, abs=0)
        compare_sets(Ao, idx, d, 1)
        xo, _, ro = orc.local_method(Ao, sy.b, sy.x0, orc.DomainParams(rule["criterion"], rule["threshold"],
                                                                        rule["param"], rule["expand_rounds"],
                                                                        rule["dilate_hops"], 1), sp)
        if d.K > 0 and rep["K"] > 0:
            assert abs(rep["local"]["iterations"] - ro.it_local) <= 1, (rep["local"], ro.it_local)
    assert abs(rep["global"]["iterations"] - ro.it_global) <= 1, (rep["global"], ro.it_global)
    err = np.linalg.norm(xg - xo) / np.linalg.norm(xo)
    assert err <= 1e-9, err
    res = np.linalg.norm(orc.residual(Ao, sy.b, xg))
    assert res <= EPS * np.linalg.norm(sy.b) * (1 + 1e-6)
    return rep


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("s", [0, 5])
def test_dist_config1(P, s):
    run_and_check(synth.system(1, s), R_C1, P)


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("rule", ["res", "grad", "method0"])
def test_dist_config5_reduced(P, rule):
    sy = synth.system(5, 10, n=24)
    run_and_check(sy, {"res": R_RES, "grad": R_GRAD, "method0": None}[rule], P)


@pytest.mark.parametrize("P", [2, 5])
def test_dist_config2_reduced_dilation(P):
    """2-D 5-point operator with 1e4 contrast; gradient criterion + 2 dilation hops across slab boundaries."""
    run_and_check(synth.system(2, 3, n=96), R_C2, P)


@pytest.mark.parametrize("P,n,s", [(1, 96, 3), (2, 96, 3), (5, 96, 3), (3, 128, 30), (8, 160, 11)])
def test_dist_config2_percentile_rule(P, n, s):
    """Config 2's own rule on the partition: gradient criterion, nearest-rank P90 threshold over ALL ranks' rows
    (radix select whose digit counts go through the rank exchange), 2 dilation hops: tau and Omega equal the
    oracle's on the whole matrix for every p."""
    rule = dict(criterion=1, threshold=2, param=0.9, expand_rounds=0, dilate_hops=2)
    rep = run_and_check(synth.system(2, s, n=n), rule, P)
    assert rep["K"] > 0


@pytest.mark.parametrize("p", [0.5, 0.999])
def test_dist_percentile_of_residual(p):
    """The percentile threshold with the residual criterion (ties at c = 0 included: x0 is exact on most rows)."""
    sy = synth.system(5, 6, n=20)
    run_and_check(sy, dict(criterion=0, threshold=2, param=p, expand_rounds=0, dilate_hops=0), 3)


def test_dist_ragged_slabs():
    """Slab boundaries off the 32-row slices (ragged first and last slices in every rank)."""
    sy = synth.system(5, 4, n=20)
    N = sy.nrows
    R = [0, 2011, 4013, 6007, N]
    run_and_check(sy, R_RES, 4, R=R)


def test_dist_expansion_rounds():
    """E_max = 3 expansion rounds: admissions read neighbour slabs' flags of the previous round."""
    sy = synth.system(5, 7, n=24)
    run_and_check(sy, dict(criterion=0, threshold=0, param=1e-10, expand_rounds=3, dilate_hops=0), 3)


def test_dist_empty_domain():
    """x0 = the exact solution: Omega = {} (K = 0), the local solve is a no-op, 0 global iterations."""
    sy = synth.system(1, 2)
    ranks, R = make_ranks(sy, 2)
    xs = orc.pcg(orc.Csr(sy.rp, sy.ci, sy.val), sy.b, sy.x0, 1e-15)[0]
    b = slabs(sy.b, R)
    x0 = slabs(xs, R)
    K = lc.dist_select_domain(ranks, b, x0, **R_RES)
    assert K == 0
    x = [t.clone() for t in x0]
    info = lc.dist_solve_local(ranks, x)
    assert info["iterations"] == 0
    g = lc.dist_solve_global(ranks, b, x)
    assert g["iterations"] == 0


def test_dist_full_domain_theta0():
    """theta = 0 => Omega = everything (R11): the local solve is method0, the global solve takes 0 iterations."""
    sy = synth.system(1, 3)
    ranks, R = make_ranks(sy, 3)
    b, x0 = slabs(sy.b, R), slabs(sy.x0, R)
    x, rep = lc.dist_local_method(ranks, b, x0, dict(criterion=1, threshold=1, param=0.0), rel_tol=EPS)
    assert rep["K"] == sy.nrows
    assert rep["global"]["iterations"] == 0
    _, it0, _, _ = orc.pcg(orc.Csr(sy.rp, sy.ci, sy.val), sy.b, sy.x0, EPS)
    assert abs(rep["local"]["iterations"] - it0) <= 1


def test_dist_matches_single_gpu_path_config5_full():
    """Config 5 at its BASELINE size (256^3) on 4 emulated ranks: Omega bit-equal to the single-GPU
    lc_select_domain (itself parity-tested against the oracle), iterations +-1, solutions within 1e-9."""
    sy = synth.system(5, 10)
    A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val)
    bd, x0d = torch.from_numpy(sy.b).to(DEV), torch.from_numpy(sy.x0).to(DEV)
    dom = lc.select_domain(A, bd, x0d, **R_RES)
    idx1 = dom.export()[0].cpu().numpy()
    x1, rep1 = lc.local_method(A, bd, x0d, R_RES)
    del A
    ranks, R = make_ranks(sy, 4, align=256)
    b, x0 = slabs(sy.b, R), slabs(sy.x0, R)
    x, rep = lc.dist_local_method(ranks, b, x0, R_RES, rel_tol=EPS)
    idx = np.concatenate([ldist.omega_from_flags(r.domain_flags()[0].cpu().numpy(), r.row0) for r in ranks])
    np.testing.assert_array_equal(idx, idx1)
    assert abs(rep["local"]["iterations"] - rep1["local"][0]["iterations"]) <= 1
    assert abs(rep["global"]["iterations"] - rep1["global"][0]["iterations"]) <= 1
    xg = gather(x)
    x1 = x1.cpu().numpy()
    assert np.linalg.norm(xg - x1) / np.linalg.norm(x1) <= 1e-9


@pytest.mark.parametrize("P", [1, 3])
def test_dist_lazy_x_bitwise(P, tune):
    """Lazy x in the row-partitioned PCG (x updated every second iteration with the same fma roundings, the
    CONFIRM pass gathering x plus its pending update from the neighbour slabs) gives bitwise the solution
    of the every-pass update, local and global solves."""
    sy = synth.system(5, 7, n=28)
    outs = []
    for lazy in (True, False):
        if lazy:
            tune(lazy_x_depth=3)
        else:
            tune(lazy_x_depth=1)
        ranks, R = make_ranks(sy, P)
        b, x0 = slabs(sy.b, R), slabs(sy.x0, R)
        x, rep = lc.dist_local_method(ranks, b, x0, R_RES, rel_tol=EPS)
        outs.append((gather(x), rep["local"]["iterations"], rep["global"]["iterations"]))
        del ranks
    assert outs[0][1:] == outs[1][1:]
    np.testing.assert_array_equal(outs[0][0], outs[1][0])


class _Sys:
    pass


def test_dist_1d_three_point_generic_width():
    """A 1-D three-point operator (generic-width kernels) on 3 emulated ranks through Alg. 5 + the solves."""
    n = 3000
    xg = np.arange(n) / n
    xs = 0.1 + 0.9 * 0.5 * (1 - np.tanh((xg - 0.5) / 0.01))
    x0 = 0.1 + 0.9 * 0.5 * (1 - np.tanh((xg - 0.49) / 0.01))
    k = (0.5 * (x0[:-1] + x0[1:])) ** 2.5
    lam = 50.0
    rp, ci, va = [0], [], []
    for i in range(n):
        d = 1.0
        if i > 0:
            ci.append(i - 1); va.append(-lam * k[i - 1]); d += lam * k[i - 1]
        ci.append(i); va.append(0.0); di = len(va) - 1
        if i < n - 1:
            ci.append(i + 1); va.append(-lam * k[i]); d += lam * k[i]
        va[di] = d
        rp.append(len(ci))
    sy = _Sys()
    sy.nrows = n
    sy.rp, sy.ci, sy.val = np.array(rp), np.array(ci, np.int32), np.array(va)
    sy.b = orc.spmv(orc.Csr(sy.rp, sy.ci, sy.val), xs)
    sy.x0 = x0
    run_and_check(sy, dict(criterion=0, threshold=0, param=1e-10, expand_rounds=2, dilate_hops=0), 3, align=1,
                  R=[0, 1001, 1999, n])


def test_dist_rejects_non_stencil_and_short_slabs():
    sy = synth.random_system(300, 7, True, 5)   # random band: no constant offset set
    rp, ci, va = ldist.slab_csr(sy.rp, sy.ci, sy.val, 0, 150)
    with pytest.raises(lc.LcError, match="LC_ERR_PATTERN"):
        lc.DistRank(sy.nrows, 0, 150, 0, 2, rp, ci, va)
    # tridiagonal plus the couplings (0, 5), (5, 0): rows with different offset sets
    n = 64
    M = np.eye(n) * 4.0
    for i in range(n - 1):
        M[i, i + 1] = M[i + 1, i] = -1.0
    M[0, 5] = M[5, 0] = -0.5
    Ao = orc.Csr.from_dense(M)
    with pytest.raises(lc.LcError, match="LC_ERR_PATTERN"):
        lc.DistRank(n, 0, n, 0, 1, Ao.rp, Ao.ci, Ao.val)
    sy = synth.system(5, 0, n=12)               # reach 144 rows; a 100-row slab is too short
    N = sy.nrows
    R = [0, N - 100, N]
    ranks = []
    for l in range(2):
        rp, ci, va = ldist.slab_csr(sy.rp, sy.ci, sy.val, R[l], R[l + 1])
        ranks.append(lc.DistRank(N, R[l], R[l + 1] - R[l], l, 2, rp, ci, va))
    with pytest.raises(lc.LcError, match="LC_ERR_DIMENSION"):
        lc.dist_connect_local(ranks)


# ---------------------------------------------------------------- one process per rank (IPC plumbing) ----

def test_dist_multiprocess_api_world1():
    """tools/dist_mp.py through the one-process-per-GPU API (export / all-gather / lc_dist_connect, nr = 1)
    at world size 1 (the only size one GPU can run without ranks waiting on each other across launches)."""
    import json
    import os
    import subprocess
    import sys
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", WORLD_SIZE="1",
               LOCAL_RANK="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "dist_mp.py"), "--config", "1", "--align", "32"],
                         env=env, capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    sy = synth.system(1, 10)
    Ao = orc.Csr(sy.rp, sy.ci, sy.val)
    d = orc.select_domain(Ao, sy.b, sy.x0, 0, 0, 1e-10, 1, 0, 1)
    assert r["K"] == r["K_gathered"] == d.K
    assert r["rel_residual"] <= 1e-10 * (1 + 1e-6)


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, port, q):
    import os
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2")
    tdist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2001_01158_b200 import dist as ld
        from paper_2001_01158_b200 import lc as llc
        sy = synth.system(1, 0)
        R = ld.split_rows(sy.nrows, 2, 32)
        rp, ci, va = ld.slab_csr(sy.rp, sy.ci, sy.val, R[rank], R[rank + 1])
        me = llc.DistRank(sy.nrows, R[rank], R[rank + 1] - R[rank], rank, 2, rp, ci, va)
        hs = ld.exchange_handles(me.export_handle())
        me.connect(hs, ld.exchange_sizes(R[rank + 1] - R[rank]))   # opens the other process's workspace
        tdist.barrier()                                                # both mapped before either unmaps
        del me
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    tdist.destroy_process_group()


def test_dist_ipc_connect_two_processes():
    """Two processes (one device): each exports its workspace and opens the other's through CUDA IPC.  No
    kernel runs (cross-process waits need one GPU per rank)."""
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
