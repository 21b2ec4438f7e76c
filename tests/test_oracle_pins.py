"""Pins of the CPU oracle against what the paper and the mathematics fix
(never against the oracle itself).  CPU only (-m "not gpu").

Each test names the passage / closed form it pins.  A plausible mistake in
the oracle (dropped term, wrong sign or index, transposed operand, non-strict
comparison, wrong threshold normalisation) fails at least one of them.
"""
import math

import numpy as np
import pytest

import oracle as orc
import synth
from conftest import read_golden


# ---------------------------------------------------------------- Example 1 ---

def example1():
    g = read_golden("example1.txt")
    n = 9
    A = np.eye(n)
    for i in range(n - 1):                      # a_{i,i+1} = a_{i+1,i} = -1/(i+2) with 0-based i
        A[i, i + 1] = A[i + 1, i] = -1.0 / (i + 2)
    x = np.array([float(v) for v in g["x"]])
    x0 = np.array([float(v) for v in g["x0"]])
    b = A @ x                                    # "The right hand side is set to b = Ax"
    return g, A, x, x0, b


def sig3(v):
    return float(f"{v:.2e}")


def test_example1_residual_printed_values():
    """r0 = b - A x0 matches the printed vector to 3 significant digits;
    component 2 uses the reading 3.60e-1 (R1: the printed 3.66e-1 is garbled)."""
    g, A, x, x0, b = example1()
    r = orc.residual(orc.Csr.from_dense(A), b, x0)
    printed = [float(v) for v in g["r0"]]
    printed[1] = float(g["r0_2_reading"][0])
    for i, (ri, pi) in enumerate(zip(r, printed)):
        assert sig3(ri) == pytest.approx(pi, rel=1e-12), (i, ri, pi)
    # the garbled printed value is NOT reproduced (documented reading R1)
    assert sig3(r[1]) != float(g["r0"][1])


def test_example1_tau_and_bad_points():
    """tau = eps ||b||_2 / sqrt(N) = 3.44e-7 and bad points {1,2,3}."""
    g, A, x, x0, b = example1()
    Ac = orc.Csr.from_dense(A)
    assert orc.norm2(b) == pytest.approx(math.sqrt(math.fsum(v * v for v in b)), rel=1e-15)
    d = orc.select_domain(Ac, b, x0, orc.CRIT_RESIDUAL, orc.THR_PAPER, 1e-5, expand_rounds=0)
    assert sig3(d.tau) == float(g["tau"][0])
    assert list(d.idx + 1) == [int(v) for v in g["bad"]]


def test_example1_table1_expansion():
    """Alg. 3 with E_max = 6 reproduces Table 1: admits {4},{5},{6}, rejects 7 at
    1.430e-7 < tau and breaks at m = 4 with K = 6; admission values to 4 significant digits."""
    g, A, x, x0, b = example1()
    d = orc.select_domain(orc.Csr.from_dense(A), b, x0, orc.CRIT_RESIDUAL, orc.THR_PAPER, 1e-5,
                          expand_rounds=int(g["emax"][0]))
    assert d.trace["rounds"] == 4
    assert d.trace["front"] == [1, 1, 1, 1]
    assert d.trace["admitted"] == [1, 1, 1, 0]
    assert d.trace["K_after"] == [4, 5, 6, 6]
    assert d.K == 6 and list(d.idx + 1) == [1, 2, 3, 4, 5, 6]
    for m, j in zip(range(1, 5), [4, 5, 6, 7]):
        row = g[f"table1_m{m}"]
        assert int(row[0]) == j
        assert float(f"{d.adm[j - 1]:.3e}") == float(row[3]), (m, d.adm[j - 1])


def test_example1_emax_one_and_zero():
    """E_max = 1 => {1,2,3,4} (Table 1 row m=1); E_max = 0 => the bad points only."""
    g, A, x, x0, b = example1()
    Ac = orc.Csr.from_dense(A)
    d1 = orc.select_domain(Ac, b, x0, orc.CRIT_RESIDUAL, orc.THR_PAPER, 1e-5, expand_rounds=1)
    assert list(d1.idx + 1) == [1, 2, 3, 4]
    d0 = orc.select_domain(Ac, b, x0, orc.CRIT_RESIDUAL, orc.THR_PAPER, 1e-5, expand_rounds=0)
    assert list(d0.idx + 1) == [1, 2, 3]


def test_example1_gradient_hand_values():
    """Eq. 5 evaluated by hand on Example 1's x0 (SPEC S:215-217 derived values)."""
    g, A, x, x0, b = example1()
    gr = orc.gradient(orc.Csr.from_dense(A), x0)
    expect = [0.9, 0.998999, 0.0998999, 9.9099e-4, 9.9099e-5, 9.9099e-6, 9.9099e-7, 9.9099e-8, 9.009e-9]
    np.testing.assert_allclose(gr, expect, rtol=1e-12)


@pytest.mark.parametrize("alpha,expect", [(0.5, [1, 2]), (1e-2, [1, 2, 3]), (1e-4, [1, 2, 3, 4]),
                                          (1.0, []), (0.0, list(range(1, 10)))])
def test_example1_gradient_domain(alpha, expect):
    """Alg. 2: g_i > alpha g_max; alpha = 1 => empty, alpha = 0 => Omega (R11)."""
    g, A, x, x0, b = example1()
    d = orc.select_domain(orc.Csr.from_dense(A), b, x0, orc.CRIT_GRADIENT, orc.THR_REL_MAX, alpha)
    assert list(d.idx + 1) == expect


def test_example1_extraction_values():
    """Eq. 3 with Omega = {1,2,3}: B = leading 3x3 block, E has the single entry -1/4, so
    b_sub = b_B - E x_C^(0) = (9.5e-2, -4.033333e-2, -2.333308e-3) (hand evaluation)."""
    g, A, x, x0, b = example1()
    flag = np.zeros(9, np.uint8); flag[:3] = 1
    sub = orc.extract(orc.Csr.from_dense(A), b, x0, flag)
    np.testing.assert_array_equal(sub.idx, [0, 1, 2])
    np.testing.assert_array_equal(sub.B.to_dense(), A[:3, :3])
    np.testing.assert_allclose(sub.bsub, [9.5e-2, -4.0333333333e-2, -2.3333083333e-3], rtol=1e-9)
    np.testing.assert_array_equal(sub.xB0, x0[:3])


def test_example1_local_solve_annihilates_and_skips_global():
    """Alg. 1 on Example 1 (eps = 1e-5, E_max = 6 -> Omega = {1..6}): the local subsystem solve makes
    x~ satisfy Eq. 6 with no global iteration (the paper's 'x~ is a final solution'),
    the Omega rows' residual is annihilated to the subsystem tolerance and the complement is kept."""
    g, A, x, x0, b = example1()
    Ac = orc.Csr.from_dense(A)
    dp = orc.DomainParams(orc.CRIT_RESIDUAL, orc.THR_PAPER, 1e-5, 6, 0, 1)
    sp = orc.SolverParams(0, 1, 30, 1e-5, 20000, 0)
    xs, flag, rep = orc.local_method(Ac, b, x0, dp, sp)
    assert rep.K == 6 and rep.it_global == 0 and rep.st_global == 0
    assert rep.it_local <= 6                      # CG: at most K distinct eigenvalues
    r = b - A @ xs
    assert np.linalg.norm(r) <= 1e-5 * np.linalg.norm(b)
    np.testing.assert_array_equal(xs[6:], x0[6:])
    # local annihilation: B x_B = b_sub holds to the subsystem tolerance
    sub = orc.extract(Ac, b, x0, flag)
    rB = sub.bsub - sub.B.to_dense() @ xs[:6]
    assert np.linalg.norm(rB) <= 1e-5 * np.linalg.norm(sub.bsub) * (1 + 1e-12)


def test_xt_output_is_eq4_assembly():
    """x~ returned by or_local_method (Eq. 4, Alg. 1 l.6): on Omega the solution of B x_B = b_sub
    (dense solve of the hand-checked Example 1 subsystem, to the subsystem tolerance times ||B^-1||), on the
    complement x0 bitwise; one GS sweep (l.7) happens after it, so x~ does not depend on gs_sweeps."""
    g, A, x, x0, b = example1()
    Ac = orc.Csr.from_dense(A)
    dp = orc.DomainParams(orc.CRIT_RESIDUAL, orc.THR_PAPER, 1e-5, 0, 0, 1)     # Omega = {1,2,3}
    for gs in (0, 1):
        sp = orc.SolverParams(0, 1, 30, 1e-10, 20000, gs)
        _, flag, rep, xt = orc.local_method(Ac, b, x0, dp, sp, want_xt=True)
        assert rep.K == 3
        np.testing.assert_array_equal(xt[3:], x0[3:])
        B = A[:3, :3]
        bsub = b[:3] - A[:3, 3:] @ x0[3:]
        xB = np.linalg.solve(B, bsub)
        bound = 1e-10 * np.linalg.norm(bsub) * np.linalg.norm(np.linalg.inv(B), 2) * (1 + 1e-6) + 1e-16
        assert np.linalg.norm(xt[:3] - xB) <= bound
        if gs == 0:
            xt0 = xt
        else:
            np.testing.assert_array_equal(xt, xt0)


# ------------------------------------------------------------ brute force ----

@pytest.mark.parametrize("seed", range(6))
def test_spmv_residual_vs_dense(seed):
    """spmv / residual agree with a dense matrix-vector product for n <= 20."""
    s = synth.random_system(12 + seed, bw=2 + seed % 3, spd=seed % 2 == 0, seed=seed + 11)
    A = orc.Csr(s.rp, s.ci, s.val)
    D = A.to_dense()
    np.testing.assert_allclose(orc.spmv(A, s.x0), D @ s.x0, rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(orc.residual(A, s.b, s.x0), s.b - D @ s.x0, rtol=1e-12, atol=1e-14)


def test_residual_of_manufactured_solution_is_zero():
    """residual(A, A x*, x*) == 0 bitwise when b uses the same ascending fma chain."""
    for cfg, n in [(1, 16), (3, 8), (5, 8)]:
        s = synth.system(cfg, 0, n=n, G=3)
        r = orc.residual(orc.Csr(s.rp, s.ci, s.val), s.b, s.xs)
        assert np.all(r == 0.0), cfg


@pytest.mark.parametrize("seed", range(8))
def test_bad_points_brute_force(seed):
    """Eq. 7 bad-point set = support of |r_i| > eps ||b|| / sqrt(N), by brute force, n <= 12."""
    rng = np.random.default_rng(seed)
    n = 12
    M = np.diag(rng.uniform(2, 3, n)) + np.diag(rng.uniform(-0.5, 0, n - 1), 1)
    M = M + np.triu(M, 1).T
    xs = rng.uniform(-1, 1, n)
    x0 = xs.copy(); x0[rng.integers(0, n, 3)] += rng.uniform(-1e-3, 1e-3, 3)
    b = M @ xs
    eps = 10.0 ** rng.uniform(-8, -3)
    r = b - M @ x0
    tau = eps * math.sqrt(math.fsum(v * v for v in b)) / math.sqrt(n)
    d = orc.select_domain(orc.Csr.from_dense(M), b, x0, orc.CRIT_RESIDUAL, orc.THR_PAPER, eps)
    brute = [i for i in range(n) if abs(r[i]) > tau and abs(abs(r[i]) - tau) > 1e-9 * tau]
    near = [i for i in range(n) if abs(abs(r[i]) - tau) <= 1e-9 * tau]
    got = [i for i in d.idx if i not in near]
    assert got == brute


def test_rel_max_threshold_closed_form():
    """rel-max: {i : |r_i| > theta max|r|} (config 1 rule); theta = 0 -> Omega; x0 exact -> empty."""
    s = synth.system(1, 3, n=16)
    A = orc.Csr(s.rp, s.ci, s.val)
    r = np.abs(s.b - A.to_dense() @ s.x0)
    d = orc.select_domain(A, s.b, s.x0, orc.CRIT_RESIDUAL, orc.THR_REL_MAX, 1e-3)
    expect = np.flatnonzero(r > 1e-3 * r.max())
    np.testing.assert_array_equal(d.idx, expect)
    assert orc.select_domain(A, s.b, s.x0, orc.CRIT_RESIDUAL, orc.THR_REL_MAX, 0.0).K == A.n
    assert orc.select_domain(A, s.b, s.xs, orc.CRIT_RESIDUAL, orc.THR_REL_MAX, 1e-3).K == 0


def test_percentile_threshold_vs_np_partition():
    """R14: tau = nearest-rank P90 of g = np.partition(g, k)[k], k = ceil(0.9 N) - 1; select g > tau."""
    s = synth.system(2, 0, n=32)
    A = orc.Csr(s.rp, s.ci, s.val)
    g = orc.gradient(A, s.x0)
    k = math.ceil(0.9 * A.n) - 1
    tau = np.partition(g, k)[k]
    d = orc.select_domain(A, s.b, s.x0, orc.CRIT_GRADIENT, orc.THR_PERCENTILE, 0.9)
    assert d.tau == tau
    np.testing.assert_array_equal(d.idx, np.flatnonzero(g > tau))
    assert d.K <= A.n - k - 1 + 1


def test_gradient_five_point_formula():
    """Eq. 5 on a 5-point matrix equals the displayed four-term formula, evaluated with
    array shifts on the grid (closed form), including boundary cells with fewer neighbours."""
    n = 9
    s = synth.system(1, 0, n=n)
    A = orc.Csr(s.rp, s.ci, s.val)
    X = s.x0.reshape(n, n)          # [iy, ix]
    G = np.zeros_like(X)
    G[:, 1:] += np.abs(X[:, :-1] - X[:, 1:]); G[:, :-1] += np.abs(X[:, 1:] - X[:, :-1])
    G[1:, :] += np.abs(X[:-1, :] - X[1:, :]); G[:-1, :] += np.abs(X[1:, :] - X[:-1, :])
    np.testing.assert_allclose(orc.gradient(A, s.x0), G.ravel(), rtol=1e-14, atol=0)


def test_gradient_shift_scale_invariance():
    """g(x0 + c) = g(x0), g(c x0) = c g(x0) -- exact for c a power of 2."""
    s = synth.system(2, 1, n=16)
    A = orc.Csr(s.rp, s.ci, s.val)
    g = orc.gradient(A, s.x0)
    np.testing.assert_allclose(orc.gradient(A, s.x0 + 3.0), g, rtol=1e-12, atol=1e-14)
    np.testing.assert_array_equal(orc.gradient(A, 4.0 * s.x0), 4.0 * g)


@pytest.mark.parametrize("hops", [1, 2, 3])
def test_dilation_is_l1_ball(hops):
    """R15: d hops of unconditional dilation on a 5-pt (7-pt) grid = the L1 ball of radius d."""
    for cfg, n, dims in [(1, 11, 2), (5, 7, 3)]:
        s = synth.system(cfg, 0, n=n)
        A = orc.Csr(s.rp, s.ci, s.val)
        N = A.n
        c = N // 2
        # criterion: x0 with one spike -> gradient is largest at the spike's neighbours; use rel-max on
        # a residual that is nonzero at one cell only: b = A x0 + e_c
        b = orc.spmv(A, s.x0); b[c] += 1.0
        d = orc.select_domain(A, b, s.x0, orc.CRIT_RESIDUAL, orc.THR_REL_MAX, 0.5, dilate_hops=hops)
        coords = np.array(np.unravel_index(np.arange(N), (n,) * dims))
        cc = np.array(np.unravel_index(c, (n,) * dims))[:, None]
        ball = np.flatnonzero(np.abs(coords - cc).sum(axis=0) <= hops)
        np.testing.assert_array_equal(d.idx, ball)


def test_expansion_invariants():
    """Alg. 3: K non-decreasing in E_max and nested; every admitted index is a neighbour of the
    pre-round domain; admission uses r0 without recomputation."""
    s = synth.system(5, 4, n=12)
    A = orc.Csr(s.rp, s.ci, s.val)
    D = A.to_dense() != 0
    prev = None
    for em in range(0, 5):
        d = orc.select_domain(A, s.b, s.x0, orc.CRIT_RESIDUAL, orc.THR_PAPER, 1e-10, expand_rounds=em)
        if prev is not None:
            assert set(prev.idx) <= set(d.idx)
            new = sorted(set(d.idx) - set(prev.idx))
            for j in new:
                assert any(D[j, l] and l != j for l in prev.idx)
        prev = d


def test_alpha_nesting():
    """alpha1 <= alpha2 => domain(alpha2) subset of domain(alpha1); eta monotone."""
    s = synth.system(5, 2, n=10)
    A = orc.Csr(s.rp, s.ci, s.val)
    prev = None
    for alpha in [1e-1, 1e-2, 1e-3, 1e-4, 1e-6]:
        d = orc.select_domain(A, s.b, s.x0, orc.CRIT_GRADIENT, orc.THR_REL_MAX, alpha)
        if prev is not None:
            assert set(prev.idx) <= set(d.idx)
        prev = d


def test_extraction_vs_dense_and_roundtrip():
    """Eq. 2/3: B = A[Omega, Omega], b_sub = b_B - A[Omega, C] x0_C (dense, independent); full Omega gives
    B = A and b_sub = b bitwise; assembly keeps the complement bitwise (Eq. 4)."""
    s = synth.random_system(30, bw=3, spd=False, seed=5)
    A = orc.Csr(s.rp, s.ci, s.val); D = A.to_dense()
    rng = np.random.default_rng(3)
    flag = (rng.uniform(size=30) < 0.4).astype(np.uint8)
    sub = orc.extract(A, s.b, s.x0, flag)
    idx = np.flatnonzero(flag); comp = np.flatnonzero(flag == 0)
    np.testing.assert_array_equal(sub.idx, idx)
    np.testing.assert_array_equal(sub.B.to_dense(), D[np.ix_(idx, idx)])
    np.testing.assert_allclose(sub.bsub, s.b[idx] - D[np.ix_(idx, comp)] @ s.x0[comp], rtol=1e-12, atol=1e-13)
    full = orc.extract(A, s.b, s.x0, np.ones(30, np.uint8))
    np.testing.assert_array_equal(full.B.val, A.val); np.testing.assert_array_equal(full.bsub, s.b)
    xt = orc.assemble(sub, np.arange(len(idx), dtype=float), s.x0)
    np.testing.assert_array_equal(xt[comp], s.x0[comp])
    np.testing.assert_array_equal(xt[idx], np.arange(len(idx), dtype=float))


# ------------------------------------------------------------------ solvers ---

@pytest.mark.parametrize("seed", range(5))
def test_pcg_vs_dense_lu(seed):
    """Jacobi-PCG to eps = 1e-10 matches a dense LU solve to 1e-8 relative, n <= 50, and
    satisfies Eq. 6 when re-checked."""
    s = synth.random_system(40 + seed, bw=3, spd=True, seed=100 + seed)
    A = orc.Csr(s.rp, s.ci, s.val); D = A.to_dense()
    xlu = np.linalg.solve(D, s.b)
    x, it, st, rr = orc.pcg(A, s.b, s.x0, eps=1e-10)
    assert st == orc.OK and it > 0
    assert np.linalg.norm(x - xlu) / np.linalg.norm(xlu) <= 1e-8
    assert np.linalg.norm(s.b - D @ x) <= 1e-10 * np.linalg.norm(s.b) * (1 + 1e-6)


def test_pcg_identity_and_exact():
    """A = I converges in <= 1 iteration to x = b; x0 exact -> 0 iterations."""
    n = 10
    A = orc.Csr.from_dense(np.eye(n))
    b = np.arange(1.0, n + 1)
    x, it, st, _ = orc.pcg(A, b, np.zeros(n))
    assert st == orc.OK and it <= 1 and np.allclose(x, b, rtol=1e-15)
    x, it, st, _ = orc.pcg(A, b, b)
    assert st == orc.OK and it == 0


def test_pcg_finite_termination():
    """CG terminates in at most d steps when the (Jacobi-scaled) matrix has d distinct eigenvalues:
    A = I + 3 u u^T with |u_i| = 1/sqrt(n) has a constant diagonal (Jacobi = scalar) and 2 distinct
    eigenvalues -> 2 iterations."""
    n = 20
    rng = np.random.default_rng(0)
    u = rng.choice([-1.0, 1.0], n) / math.sqrt(n)
    M = np.eye(n) + 3.0 * np.outer(u, u)
    A = orc.Csr.from_dense(M)
    b = M @ rng.uniform(-1, 1, n)
    x, it, st, _ = orc.pcg(A, b, np.zeros(n), eps=1e-12)
    assert st == orc.OK and it == 2
    np.testing.assert_allclose(x, np.linalg.solve(M, b), rtol=1e-10)


@pytest.mark.parametrize("seed", range(4))
def test_gmres_vs_dense_lu(seed):
    """Right-preconditioned block-Jacobi GMRES(30)/CGS2 matches dense LU to 1e-8 relative at eps 1e-10
    on nonsymmetric diagonally dominant systems, with restarts exercised (n > 30)."""
    s = synth.random_system(45, bw=4, spd=False, seed=200 + seed)
    A = orc.Csr(s.rp, s.ci, s.val); D = A.to_dense()
    xlu = np.linalg.solve(D, s.b)
    for bs in (1, 3):
        x, it, st, rr = orc.gmres_bj(A, s.b, s.x0, bs=bs, eps=1e-10, restart=30)
        assert st == orc.OK
        assert np.linalg.norm(x - xlu) / np.linalg.norm(xlu) <= 1e-8
        assert np.linalg.norm(s.b - D @ x) <= 1e-10 * np.linalg.norm(s.b) * (1 + 1e-6)


def test_gmres_exact_in_n_steps():
    """Unrestarted GMRES is exact in at most n Arnoldi steps; with M = the exact block inverse of a
    block-diagonal A, one step suffices (happy breakdown)."""
    rng = np.random.default_rng(7)
    nb = 5
    D = np.zeros((3 * nb, 3 * nb))
    for c in range(nb):
        blk = rng.uniform(-1, 1, (3, 3)) + 4 * np.eye(3)
        D[3 * c:3 * c + 3, 3 * c:3 * c + 3] = blk
    A = orc.Csr.from_dense(D)
    b = rng.uniform(-1, 1, 3 * nb)
    x, it, st, _ = orc.gmres_bj(A, b, np.zeros(3 * nb), bs=3, eps=1e-12, restart=30)
    assert st == orc.OK and it == 1
    np.testing.assert_allclose(x, np.linalg.solve(D, b), rtol=1e-12)


def test_bsr_expansion_vs_dense():
    """or_bsr_to_csr: scalar (3c+a, 3c'+b) = block (c,c')[a][b] (config 4 layout)."""
    s = synth.system(4, 0, n=4)
    A = orc.Csr.from_bsr(s.rp, s.ci, s.val)
    D = A.to_dense()
    for c in range(s.nrows):
        for k in range(s.rp[c], s.rp[c + 1]):
            cc = s.ci[k]
            blk = s.val[9 * k:9 * k + 9].reshape(3, 3)
            np.testing.assert_array_equal(D[3 * c:3 * c + 3, 3 * cc:3 * cc + 3], blk)
    assert np.all(orc.residual(A, s.b, s.xs) == 0.0)


# ----------------------------------------------------- Alg. 1 invariants ----

def _heat(cfg=1, n=24, s=3):
    sy = synth.system(cfg, s, n=n)
    return sy, orc.Csr(sy.rp, sy.ci, sy.val)


def test_full_domain_reduces_to_global_solve():
    """BASELINE.json invariant: Omega_local = Omega => the local method returns method0's result
    bitwise, with 0 global iterations."""
    sy, A = _heat()
    sp = orc.SolverParams(0, 1, 30, 1e-10, 20000, 0)
    x0m, _, rep0 = orc.local_method(A, sy.b, sy.x0, None, sp)
    full = orc.DomainParams(orc.CRIT_RESIDUAL, orc.THR_REL_MAX, 0.0, 0, 0, 1)
    x1, flag, rep1 = orc.local_method(A, sy.b, sy.x0, full, sp)
    assert rep1.K == A.n and rep1.it_global == 0
    np.testing.assert_array_equal(x1, x0m)
    assert rep1.it_local == rep0.it_global


def test_empty_domain_is_method0():
    """Omega = {} (x0 exact in the criterion's eyes) => x~ = x0 and the result is method0's bitwise (R12)."""
    sy, A = _heat()
    sp = orc.SolverParams(0, 1, 30, 1e-10, 20000, 0)
    x0m, _, _ = orc.local_method(A, sy.b, sy.x0, None, sp)
    empty = orc.DomainParams(orc.CRIT_GRADIENT, orc.THR_REL_MAX, 1.0, 0, 0, 1)
    x1, flag, rep = orc.local_method(A, sy.b, sy.x0, empty, sp)
    assert rep.K == 0
    np.testing.assert_array_equal(x1, x0m)


@pytest.mark.parametrize("cfg,n", [(1, 32), (2, 32), (3, 8), (5, 10)])
def test_manufactured_solution_bound(cfg, n):
    """Manufactured solution (b = A x*): for A = D + lambda0 L with D >= I, ||A^-1|| <= 1, so
    ||x - x*|| <= ||b - A x|| <= 1e-10 ||b|| (R31) -- for method0 and for the local method."""
    sy = synth.system(cfg, 2, n=n, G=3)
    A = orc.Csr(sy.rp, sy.ci, sy.val)
    sp = orc.SolverParams(0, 1, 30, 1e-10, 20000, 0)
    segs = [(0, A.n)] if cfg != 3 else [(g * n * n, (g + 1) * n * n) for g in range(3)]
    for r0, r1 in segs:
        As = A.segment(r0, r1)
        b = sy.b[r0:r1]; x0 = sy.x0[r0:r1]; xs = sy.xs[r0:r1]
        for dp in (None, orc.DomainParams(orc.CRIT_RESIDUAL, orc.THR_PAPER, 1e-10, 1, 0, 1)):
            x, _, rep = orc.local_method(As, b, x0, dp, sp)
            assert rep.st_global == orc.OK
            res = np.linalg.norm(orc.residual(As, b, x))
            assert res <= 1e-10 * np.linalg.norm(b) * (1 + 1e-6)
            assert np.linalg.norm(x - xs) <= res * (1 + 1e-6) + 1e-300


def test_3t_gmres_manufactured():
    """Config 4 (3T, BSR, nonsymmetric, row-diagonally dominant with margin 1): block-Jacobi GMRES(30)
    reaches Eq. 6 at 1e-10 and ||x - x*||_inf <= ||r||_inf (margin-1 dominance => ||A^-1||_inf <= 1)."""
    sy = synth.system(4, 3, n=12)
    A = orc.Csr.from_bsr(sy.rp, sy.ci, sy.val)
    D = A.to_dense()
    assert not np.allclose(D, D.T)
    x, it, st, rr = orc.gmres_bj(A, sy.b, sy.x0, bs=3, eps=1e-10)
    assert st == orc.OK
    r = sy.b - D @ x
    assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(sy.b) * (1 + 1e-6)
    assert np.max(np.abs(x - sy.xs)) <= np.max(np.abs(r)) * (1 + 1e-6)


def test_cell_granular_domain():
    """R16: on the 3T system a cell is in Omega iff any of its 3 components has |r| > tau; the
    expansion admits whole cells; flags come in whole-cell triples."""
    sy = synth.system(4, 1, n=10)
    A = orc.Csr.from_bsr(sy.rp, sy.ci, sy.val)
    r = np.abs(sy.b - A.to_dense() @ sy.x0)
    tau = 1e-10 * np.linalg.norm(sy.b) / math.sqrt(A.n)
    d = orc.select_domain(A, sy.b, sy.x0, orc.CRIT_RESIDUAL, orc.THR_PAPER, 1e-10, expand_rounds=0, cell=3)
    cells = r.reshape(-1, 3).max(axis=1)
    near = np.abs(cells - tau) <= 1e-9 * tau
    mark = d.flag.reshape(-1, 3)
    assert np.all(mark.min(axis=1) == mark.max(axis=1))
    np.testing.assert_array_equal(mark[~near, 0], (cells > tau)[~near])


# ------------------------------------------------ NEXT-1: Gauss-Seidel (Alg. 1 l.7) --

def test_gs_spec_2x2_hand_value():
    """[[2,1],[1,2]], b = (3,3), x = 0, one sweep -> (1.5, 0.75) (hand recurrence)."""
    A = orc.Csr.from_dense(np.array([[2.0, 1.0], [1.0, 2.0]]))
    np.testing.assert_array_equal(orc.gauss_seidel(A, [3.0, 3.0], [0.0, 0.0], 1), [1.5, 0.75])


def test_gs_identity_and_fixed_point():
    """A = I -> x = b after one sweep; the exact solution of a tiny diagonal system is a fixed point."""
    n = 7
    A = orc.Csr.from_dense(np.eye(n))
    b = np.arange(1.0, n + 1)
    np.testing.assert_array_equal(orc.gauss_seidel(A, b, np.zeros(n)), b)
    D = orc.Csr.from_dense(np.diag([2.0, 4.0, 8.0]))
    np.testing.assert_array_equal(orc.gauss_seidel(D, [2.0, 4.0, 8.0], [1.0, 1.0, 1.0], 3), [1.0, 1.0, 1.0])


@pytest.mark.parametrize("seed", range(4))
def test_gs_vs_triangular_solve(seed):
    """One forward sweep = (D + L)^{-1} (b - U x_old) (dense triangular solve, library routine)."""
    import scipy.linalg
    s = synth.random_system(25, bw=3, spd=seed % 2 == 0, seed=300 + seed)
    A = orc.Csr(s.rp, s.ci, s.val); M = A.to_dense()
    L = np.tril(M); U = np.triu(M, 1)
    expect = scipy.linalg.solve_triangular(L, s.b - U @ s.x0, lower=True)
    np.testing.assert_allclose(orc.gauss_seidel(A, s.b, s.x0, 1), expect, rtol=1e-12, atol=1e-14)


def test_gs_decreases_energy_error():
    """For SPD A one GS sweep does not increase the A-norm of the error (invariant)."""
    sy = synth.system(1, 4, n=20)
    A = orc.Csr(sy.rp, sy.ci, sy.val); M = A.to_dense()
    e0 = sy.x0 - sy.xs
    x1 = orc.gauss_seidel(A, sy.b, sy.x0, 1)
    e1 = x1 - sy.xs
    assert e1 @ M @ e1 <= e0 @ M @ e0


def test_local_method_with_gs_sweep():
    """Alg. 1 with the paper's one GS sweep: the smoothed x~ still converges to Eq. 6 and the sweep
    never needs more global iterations than without it on the heat sequence."""
    sy = synth.system(5, 6, n=12)
    A = orc.Csr(sy.rp, sy.ci, sy.val)
    dp = orc.DomainParams(orc.CRIT_RESIDUAL, orc.THR_PAPER, 1e-10, 1, 0, 1)
    x0s, _, r0 = orc.local_method(A, sy.b, sy.x0, dp, orc.SolverParams(0, 1, 30, 1e-10, 20000, 0))
    x1s, _, r1 = orc.local_method(A, sy.b, sy.x0, dp, orc.SolverParams(0, 1, 30, 1e-10, 20000, 1))
    assert r1.st_global == 0 and r0.st_global == 0
    assert np.linalg.norm(orc.residual(A, sy.b, x1s)) <= 1e-10 * np.linalg.norm(sy.b) * (1 + 1e-6)


# ------------------------------------------------ NEXT-2: the paper's heat model --

def test_heat_assembly_constant_kappa_is_textbook_stencil():
    """T = 1 everywhere -> kappa = 1 on every face: the textbook implicit 5-point stencil, diag 1 + lam*(number of
    faces incl. the Dirichlet x faces), off-diagonals -lam, Neumann y faces dropped; b = T_old + lam*kf*T_bnd with
    kf = (1 + kappa(T_bnd))/2 on the boundary faces (SPEC heat-model, hand derivation)."""
    nx, ny, dt = 4, 3, 1e-2
    h = 1.0 / (nx + 1); lam = dt / h ** 2
    Ts = np.ones(nx * ny); Told = np.full(nx * ny, 0.5)
    A, b = orc.heat_assemble(nx, ny, dt, Ts, Told, khalf=3, Tl=1.0, Tr=1e-4)
    M = A.to_dense()
    kr = (1.0 + (1e-4) ** 3.5) / 2
    for q in range(ny):
        for p in range(nx):
            i = p + nx * q
            faces = 4 - (q == 0) - (q == ny - 1)
            extra = (kr - 1.0) if p == nx - 1 else 0.0      # the right Dirichlet face has kf = kr, not 1
            assert M[i, i] == pytest.approx(1 + lam * (faces + extra), rel=1e-14)
            for j in range(nx * ny):
                if j != i:
                    adj = abs(j - i) == nx or (abs(j - i) == 1 and j // nx == i // nx)
                    assert M[i, j] == (-lam if adj else 0.0)
            rhs = 0.5 + (lam * 1.0 * 1.0 if p == 0 else 0.0) + (lam * kr * 1e-4 if p == nx - 1 else 0.0)
            assert b[i] == pytest.approx(rhs, rel=1e-14)
    np.testing.assert_array_equal(M, M.T)


def test_heat_uniform_steady_state():
    """T_l = T_r = T0 = c: the uniform field is the solution; Picard stops after one iteration."""
    nx = ny = 6
    T0 = np.full(nx * ny, 0.7)
    T, per, rep = orc.heat_run(nx, ny, T0, 3, None, orc.SolverParams(0, 1, 30, 1e-12, 20000, 0), Tl=0.7, Tr=0.7)
    np.testing.assert_allclose(T, 0.7, rtol=1e-12)
    assert list(per) == [1, 1, 1]


def test_heat_run_maximum_principle_and_y_symmetry():
    """The discrete maximum principle holds and y-independent data stays y-independent (SPEC heat-model
    invariants) over a short run of Alg. 6; every Picard loop converges.  The exact discrete solution is
    y-uniform; each solve is only accurate to ||x - x*|| <= ||r|| <= 1e-10 ||b|| (R31, lambda_min >= 1), so
    rows may differ by up to 2e-10 ||b|| (||b|| <= ||T|| + lam kf T_l sqrt(ny) bounded by 2 ||T|| + 1e3 here)."""
    nx, ny = 15, 7
    T0 = synth.heat_initial(nx, ny)
    T, per, rep = orc.heat_run(nx, ny, T0, 5, None, orc.SolverParams(0, 1, 30, 1e-10, 20000, 0))
    lo, hi = min(1e-4, T0.min()), max(1.0, T0.max())
    assert T.min() >= lo - 1e-12 and T.max() <= hi + 1e-12
    G = T.reshape(ny, nx)
    assert np.max(np.abs(G - G[0])) <= 2e-10 * (2 * np.linalg.norm(T) + 1e3)
    assert rep.picard_max_hit == 0 and all(p >= 2 for p in per)


def test_heat_methods_agree_like_fig2():
    """Fig. 2 / P:1106-1107: the local methods' fields agree with method0's (the paper reports <= 7.6e-9
    relative); here after 4 steps of the 99x99 problem, methods 1 and 2 with one GS sweep."""
    nx = ny = 99
    T0 = synth.heat_initial(nx, ny)
    sp = orc.SolverParams(0, 1, 30, 1e-10, 20000, 1)
    T0m, _, _ = orc.heat_run(nx, ny, T0, 4, None, orc.SolverParams(0, 1, 30, 1e-10, 20000, 0))
    T1m, _, r1 = orc.heat_run(nx, ny, T0, 4, orc.DomainParams(1, 1, 1e-4, 0, 0, 1), sp)
    T2m, _, r2 = orc.heat_run(nx, ny, T0, 4, orc.DomainParams(0, 0, 1e-10, 1, 0, 1), sp)
    for Tm in (T1m, T2m):
        assert np.linalg.norm(Tm - T0m) / np.linalg.norm(T0m) <= 7.6e-9
