"""lc_local_method: Alg. 1 in one C-ABI call.

The one-call path runs the same kernels with the same launch configurations as the step-by-step sequence
lc_select_domain -> lc_extract_sub -> lc_solve_local -> lc_smooth_gs -> lc_solve_global, so every output is
compared with that sequence BITWISE, and against the oracle's Alg. 1 (iterations +-1, x within 1e-9); the
element-by-element parity of every config runs through it in test_gpu_parity.check_system.  Edge cases: method0
(no domain), an empty Omega (R12), Omega = everything (alpha = 0), Gauss-Seidel sweeps (l.7), GMRES,
batched groups, argument errors.
"""
import ctypes

import numpy as np
import pytest

import oracle as orc
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2001_01158_b200 import build as lcbuild
    from paper_2001_01158_b200 import lc
    lcbuild.build()

EPS = 1e-10
RES = dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1)
GRAD = dict(criterion=1, threshold=1, param=1e-4)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def matrix(sy):
    return lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=sy.block, batch=sy.batch)


def oracle_csr(sy):
    return orc.Csr.from_bsr(sy.rp, sy.ci, sy.val) if sy.block == 3 else orc.Csr(sy.rp, sy.ci, sy.val)


def same_as_steps(A, b, x0, rule, method=0, gs=0):
    x1, r1 = lc.local_method(A, b, x0, rule, method=method, gs_sweeps=gs, keep=True)
    x2, r2 = lc.local_method_steps(A, b, x0, rule, method=method, gs_sweeps=gs, keep=True)
    assert torch.equal(x1, x2)
    assert r1["K"] == r2["K"]
    if rule is not None:
        assert torch.equal(r1["xt"], r2["xt"])
        assert torch.equal(r1["idx"], r2["idx"])
    else:                                   # method0: x~ = x0
        assert torch.equal(r1["xt"], x0)
    for k in ("local", "global"):
        a, c = r1.get(k, []), r2.get(k, [])
        assert [(i["iterations"], i["status"], i["kernel"]) for i in a] == \
               [(i["iterations"], i["status"], i["kernel"]) for i in c], k
        assert [i["rel_residual"] for i in a] == [i["rel_residual"] for i in c], k
    return x1, r1


@pytest.mark.parametrize("cfg,n,rule", [(1, 64, dict(criterion=0, threshold=1, param=1e-3)), (5, 40, RES),
                                        (5, 40, GRAD), (5, 40, None), (2, 96, dict(criterion=1, threshold=2,
                                                                                    param=0.9, dilate_hops=2))])
def test_one_call_equals_steps_and_oracle(cfg, n, rule):
    sy = synth.system(cfg, 3, n=n)
    A = matrix(sy)
    x, rep = same_as_steps(A, dev(sy.b), dev(sy.x0), rule)
    dp = None
    if rule is not None:
        dp = orc.DomainParams(rule.get("criterion", 0), rule.get("threshold", 0), rule["param"],
                              rule.get("expand_rounds", 0), rule.get("dilate_hops", 0), 1)
    xo, flag, ro = orc.local_method(oracle_csr(sy), sy.b, sy.x0, dp, orc.SolverParams(0, 1, 30, EPS, 20000))
    assert rep["K"][0] == int(np.count_nonzero(flag)) if rule is not None else rep["K"] == [0]
    assert abs(rep["global"][0]["iterations"] - ro.it_global) <= 1
    if rule is not None and rep["K"][0] > 0:
        assert abs(rep["local"][0]["iterations"] - ro.it_local) <= 1
    err = np.linalg.norm(x.cpu().numpy() - xo) / np.linalg.norm(xo)
    assert err <= 1e-9
    assert all(v >= 0 for v in rep["ms"].values())


def test_one_call_gmres_3t():
    sy = synth.system(4, 2, n=24)
    A = matrix(sy)
    x, rep = same_as_steps(A, dev(sy.b), dev(sy.x0), RES, method=lc.GMRES)
    assert rep["global"][0]["kernel"] == "gmres"
    xo, _, ro = orc.local_method(oracle_csr(sy), sy.b, sy.x0, orc.DomainParams(0, 0, 1e-10, 1, 0, 3),
                                 orc.SolverParams(1, 3, 30, EPS, 3000))
    assert np.linalg.norm(x.cpu().numpy() - xo) / np.linalg.norm(xo) <= 1e-9
    assert abs(rep["global"][0]["iterations"] - ro.it_global) <= 1


def test_one_call_batched_groups():
    sy = synth.system(3, 4, n=30, G=5)
    A = matrix(sy)
    x, rep = same_as_steps(A, dev(sy.b), dev(sy.x0), RES)
    assert len(rep["K"]) == 5 and len(rep["global"]) == 5


def test_one_call_gauss_seidel_sweep():
    sy = synth.system(5, 2, n=32)
    same_as_steps(matrix(sy), dev(sy.b), dev(sy.x0), RES, gs=1)


def test_one_call_empty_and_full_domain():
    sy = synth.system(5, 1, n=32)
    A = matrix(sy)
    b, x0 = dev(sy.b), dev(sy.x0)
    x_m0, r0 = lc.local_method(A, b, x0, None)
    # theta = 1 with the strict '>' (R10): nothing exceeds max c -> Omega empty, x~ = x0 and the global solve is
    # method0 (R12)
    x_e, re = same_as_steps(A, b, x0, dict(criterion=0, threshold=1, param=1.0))
    assert re["K"] == [0] and "local" not in re
    assert torch.equal(re["xt"], x0)
    assert torch.equal(x_e, x_m0) and re["global"][0]["iterations"] == r0["global"][0]["iterations"]
    # theta = 0: Omega = everything, the local solve is the global solve and Eq. 6 holds at x~
    x_f, rf = same_as_steps(A, b, x0, dict(criterion=0, threshold=1, param=0.0))
    assert rf["K"] == [sy.N] and rf["global"][0]["iterations"] == 0
    assert torch.allclose(x_f, x_m0, rtol=0, atol=1e-9 * float(x_m0.abs().max()))


def test_one_call_argument_errors():
    sy = synth.system(1, 0, n=16)
    A = matrix(sy)
    b, x0 = dev(sy.b), dev(sy.x0)
    lib = lc.load_library()
    sp = lc.SolverParams(lc.PCG, lc.JACOBI, 30, EPS, 20000)
    P = ctypes.c_void_p
    st = lib.lc_local_method(A.h, P(b.data_ptr()), P(x0.data_ptr()), None, ctypes.byref(sp), 0, P(x0.data_ptr()),
                             None, None, lc._stream(), None, None, None, None)
    assert st == -1 and b"alias" in lib.lc_last_error()
    x = torch.empty_like(x0)
    st = lib.lc_local_method(A.h, P(b.data_ptr()), P(x0.data_ptr()), None, None, 0, P(x.data_ptr()), None, None,
                             lc._stream(), None, None, None, None)
    assert st == -1
    bad = lc.SolverParams(lc.PCG, lc.BLOCK_JACOBI, 30, EPS, 20000)
    st = lib.lc_local_method(A.h, P(b.data_ptr()), P(x0.data_ptr()), None, ctypes.byref(bad), 0, P(x.data_ptr()),
                             None, None, lc._stream(), None, None, None, None)
    assert st == -1
    # and a good call afterwards still works (no state left behind)
    st = lib.lc_local_method(A.h, P(b.data_ptr()), P(x0.data_ptr()), None, ctypes.byref(sp), 0, P(x.data_ptr()),
                             None, None, lc._stream(), None, None, None, None)
    assert st == 0


def test_one_call_side_stream():
    """On a non-default stream: the call enqueues on it and returns after its own synchronisation."""
    sy = synth.system(5, 3, n=32)
    A = matrix(sy)
    b, x0 = dev(sy.b), dev(sy.x0)
    x_ref, _ = lc.local_method(A, b, x0, RES)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        x_s, _ = lc.local_method(A, b, x0, RES)
    assert torch.equal(x_s, x_ref)
