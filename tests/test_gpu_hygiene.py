"""GPU tests of the library's handle, stream, thread and error hygiene (VERDICT r1 "multi-device and thread
hygiene"): per-thread tuning, two host threads driving the library on two streams at once,
handle lifetime across streams, the structural-symmetry check of the GS sweep, a failed lc_update_values,
and the kernel / lazy-x report of lc_solve_info."""
import threading

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

DEV = "cuda"
RES = dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1, dilate_hops=0)


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def test_two_host_threads_two_streams_bitwise():
    """Two host threads, each on its own stream, run the local method concurrently on different systems
    (grid kernel, cluster-resident kernel, GMRES): each result is bitwise the one a single thread gets."""
    cases = [(synth.system(5, 4, n=40), lc.PCG), (synth.system(1, 6), lc.PCG), (synth.system(4, 3, n=24), lc.GMRES)]
    ref = []
    for sy, m in cases:
        A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=sy.block)
        x, rep = lc.local_method(A, to_dev(sy.b), to_dev(sy.x0), RES, method=m)
        ref.append((x.cpu(), [i["iterations"] for i in rep["global"]]))
    out = {}
    errors = []

    def worker(t):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for rep_i in range(3):
                    for k, (sy, m) in enumerate(cases):
                        if (k + t) % 2:
                            continue
                        A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val, block=sy.block)
                        x, rep = lc.local_method(A, to_dev(sy.b), to_dev(sy.x0), RES, method=m)
                        st.synchronize()
                        out[(t, rep_i, k)] = (x.cpu(), [i["iterations"] for i in rep["global"]])
        except Exception as e:          # pragma: no cover - reported below
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    assert len(out) == 3 * len(cases)
    for (t, r, k), (x, its) in out.items():
        assert torch.equal(x, ref[k][0]), (t, r, k)
        assert its == ref[k][1]


def test_tuning_is_per_thread():
    """lc_set_tuning affects only the calling thread: another thread still sees (and uses) the defaults."""
    defaults = lc.tuning_defaults()
    prev = lc.set_tuning(stencil_layout=0)
    try:
        seen = {}

        def other():
            seen["t"] = lc.get_tuning()
            sy = synth.system(5, 2, n=12)
            seen["layout"] = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val).info()["layout"]

        th = threading.Thread(target=other)
        th.start()
        th.join()
        assert seen["t"] == defaults
        assert seen["layout"] == "stencil"
        sy = synth.system(5, 2, n=12)
        assert lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val).info()["layout"] == "sell"
    finally:
        lc.set_tuning(**prev)


def test_destroy_right_after_side_stream_work():
    """A matrix destroyed while lc_spmv calls it enqueued on a side stream may still run keeps its memory until
    they finish (the destroy is ordered after the handle's last stream): the products stay exact although
    the freed memory is immediately reused by new allocations."""
    sy = synth.system(5, 3, n=64)
    Ao = orc.Csr(sy.rp, sy.ci, sy.val)
    ref = orc.spmv(Ao, sy.x0)
    st = torch.cuda.Stream()
    x = to_dev(sy.x0)
    ys = []
    for trial in range(4):
        A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val)
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            y = torch.empty_like(x)
            for _ in range(20):
                lc.spmv(A, x, y)
            ys.append(y)
        del A                                          # destroyed while the side stream still works
        B = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val * 2.0)   # reuses the pool
        del B
    torch.cuda.synchronize()
    for y in ys:
        np.testing.assert_array_equal(y.cpu().numpy(), ref)


def test_gs_rejects_structurally_nonsymmetric_general_pattern(tune):
    """The sync-free GS sweep needs a structurally symmetric pattern (gs.cu): a general-layout matrix with a
    one-sided coupling is refused with LC_ERR_PATTERN, a symmetric one is swept bit-exactly."""
    tune(stencil_layout=0)
    n = 200
    M = np.eye(n) * 4.0
    for i in range(n - 1):
        M[i, i + 1] = M[i + 1, i] = -1.0
    M[5, 150] = -0.5                                   # one-sided coupling: (5, 150) stored, (150, 5) not
    Ao = orc.Csr.from_dense(M)
    A = lc.Matrix(n, Ao.rp, Ao.ci, Ao.val)
    b = np.ones(n)
    with pytest.raises(lc.LcError) as e:
        lc.smooth_gs(A, to_dev(b), to_dev(np.zeros(n)), 1)
    assert e.value.status == -3
    M[150, 5] = -0.25                                  # structurally symmetric, values nonsymmetric: allowed
    Ao = orc.Csr.from_dense(M)
    A = lc.Matrix(n, Ao.rp, Ao.ci, Ao.val)
    x = to_dev(np.zeros(n))
    lc.smooth_gs(A, to_dev(b), x, 2)
    np.testing.assert_array_equal(x.cpu().numpy(), orc.gauss_seidel(Ao, b, np.zeros(n), 2))


def test_failed_update_values_invalidates_the_handle():
    """lc_update_values with a zero diagonal fails and leaves the handle refusing calls (its values are half
    written); a later successful update makes it usable again, equal to a fresh matrix."""
    s1, s2 = synth.system(5, 3, n=20), synth.system(5, 4, n=20)
    A = lc.Matrix(s1.nrows, s1.rp, s1.ci, s1.val)
    diag = [k for k in range(s2.rp[7], s2.rp[8]) if s2.ci[k] == 7][0]      # the diagonal of row 7
    bad = s2.val.copy()
    bad[diag] = 0.0
    with pytest.raises(lc.LcError) as e:
        A.update_values(s2.rp, s2.ci, bad)
    assert e.value.status == -4
    b, x0 = to_dev(s2.b), to_dev(s2.x0)
    with pytest.raises(lc.LcError) as e:
        lc.solve_global(A, b, x0.clone())
    assert e.value.status == -1 and "update_values" in str(e.value)
    A.update_values(s2.rp, s2.ci, s2.val)
    B = lc.Matrix(s2.nrows, s2.rp, s2.ci, s2.val)
    xa, xb = x0.clone(), x0.clone()
    lc.solve_global(A, b, xa)
    lc.solve_global(B, b, xb)
    assert torch.equal(xa, xb)


def test_solve_info_reports_kernel_and_lazy_x(tune):
    """lc_solve_info names the kernel that ran and the lazy-x depth it used (the bench's byte model reads
    them instead of mirroring the library's dispatch)."""
    sy = synth.system(5, 3, n=40)
    A = lc.Matrix(sy.nrows, sy.rp, sy.ci, sy.val)
    x = to_dev(sy.x0)
    i = lc.solve_global(A, to_dev(sy.b), x)[0]
    assert i["kernel"] == "pcg_grid" and i["lazy_x_depth"] == 3
    tune(lazy_x_depth=2)
    i = lc.solve_global(A, to_dev(sy.b), to_dev(sy.x0))[0]
    assert i["lazy_x_depth"] == 2
    tune(lazy_x_depth=0)
    i = lc.solve_global(A, to_dev(sy.b), to_dev(sy.x0))[0]
    assert i["lazy_x_depth"] == 1
    sy1 = synth.system(1, 3)
    A1 = lc.Matrix(sy1.nrows, sy1.rp, sy1.ci, sy1.val)
    i = lc.solve_global(A1, to_dev(sy1.b), to_dev(sy1.x0))[0]
    assert i["kernel"] == "pcg_resident" and i["lazy_x_depth"] == 1
    sy3 = synth.system(3, 3, n=32, G=4)
    A3 = lc.Matrix(sy3.nrows, sy3.rp, sy3.ci, sy3.val, batch=4)
    infos = lc.solve_global(A3, to_dev(sy3.b), to_dev(sy3.x0))
    assert all(i["kernel"] in ("pcg_lockstep", "pcg_teams", "pcg_dynteams") for i in infos)
    sy4 = synth.system(4, 3, n=16)
    A4 = lc.Matrix(sy4.nrows, sy4.rp, sy4.ci, sy4.val, block=3)
    assert lc.solve_global(A4, to_dev(sy4.b), to_dev(sy4.x0), method=lc.GMRES)[0]["kernel"] == "gmres"
