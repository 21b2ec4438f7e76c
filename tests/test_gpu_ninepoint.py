"""Nine-point stencils (the paper's own discretisation of the multi-group and 3T problems is a 9-point scheme on a
deforming mesh) in the value-only stencil layout (up to 16 offsets per row), against the
oracle: the layout is detected, the SpMV and the Gauss-Seidel sweep are bitwise the oracle's, Alg. 1 with the
residual (Alg. 3, E_max = 1) and gradient (Alg. 2) domains gives the oracle's Omega bit-exactly, iterations +-1 and
solutions within 1e-9, on a grid with a ragged last slice and with a 3-D 15-point stencil (19 points: SELL-32)."""
import numpy as np
import pytest

import oracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2001_01158_b200 import build as lcbuild
    from paper_2001_01158_b200 import lc
    lcbuild.build()

EPS = 1e-10


def stencil_system(dims, offsets_nd, seed):
    """SPD system I + L on a regular grid with the given neighbour offsets (a symmetric set without 0): edge weight
    w_uv = (k_u + k_v) / 2, k seeded in [0.1, 1] with a hot blob; rows sorted by column.  Returns CSR + b, x0."""
    rng = np.random.default_rng(seed)
    shape = tuple(dims)
    N = int(np.prod(shape))
    idx = np.arange(N).reshape(shape)
    coords = np.stack(np.unravel_index(np.arange(N), shape), axis=1)
    k = rng.uniform(0.1, 1.0, N)
    c = np.array(shape) / 2.0
    k += 20.0 * np.exp(-((coords - c) ** 2).sum(axis=1) / (0.02 * max(shape) ** 2))
    rows = [[] for _ in range(N)]
    for d in offsets_nd:
        d = np.array(d)
        nb = coords + d
        ok = np.all((nb >= 0) & (nb < np.array(shape)), axis=1)
        u = np.flatnonzero(ok)
        v = idx[tuple(nb[ok].T)]
        w = 0.5 * (k[u] + k[v]) * 40.0
        for a, bb, ww in zip(u, v, w):
            rows[a].append((int(bb), -ww))
    rp, ci, val = [0], [], []
    for u in range(N):
        diag = 1.0 - sum(w for _, w in rows[u])
        ent = sorted(rows[u] + [(u, diag)])
        ci += [e[0] for e in ent]
        val += [e[1] for e in ent]
        rp.append(len(ci))
    xs = np.sin(0.05 * np.arange(N)) + 0.5
    A = orc.Csr(np.array(rp, np.int64), np.array(ci, np.int32), np.array(val))
    b = orc.spmv(A, xs)
    x0 = xs + 0.3 * np.exp(-((coords - c * 0.8) ** 2).sum(axis=1) / (0.01 * max(shape) ** 2))
    return A, b, x0


NINE = [(dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1) if (dy, dx) != (0, 0)]
FIFTEEN = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)
           if (a, b, c) != (0, 0, 0) and (abs(a) + abs(b) + abs(c) == 1 or abs(a) * abs(b) * abs(c) == 1)]
NINETEEN = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)
            if (a, b, c) != (0, 0, 0) and abs(a) + abs(b) + abs(c) <= 2]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("dims,offs", [((45, 47), NINE), ((61, 64), NINE), ((14, 15, 16), FIFTEEN),
                                       ((14, 15, 16), NINETEEN)])
def test_stencil_layout_spmv_gs(dims, offs):
    A, b, x0 = stencil_system(dims, offs, 3)
    M = lc.Matrix(A.n, A.rp, A.ci, A.val)
    info = M.info()
    # <= 16 offsets: the value-only stencil layout; 19 offsets: SELL-32 with explicit columns
    assert info["layout"] == ("stencil" if len(offs) + 1 <= 16 else "sell") and info["max_row"] == len(offs) + 1
    y = torch.empty(A.n, dtype=torch.float64, device="cuda")
    lc.spmv(M, dev(x0), y)
    np.testing.assert_array_equal(y.cpu().numpy(), orc.spmv(A, x0))
    x = dev(x0)
    if len(offs) + 1 > 16:                     # lc_smooth_gs takes rows of at most 16 entries (include/lc.h)
        with pytest.raises(lc.LcError, match="LC_ERR_PATTERN"):
            lc.smooth_gs(M, dev(b), x, 1)
        return
    lc.smooth_gs(M, dev(b), x, 1)
    np.testing.assert_array_equal(x.cpu().numpy(), orc.gauss_seidel(A, b, x0, 1))


@pytest.mark.parametrize("rule", [dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1),
                                  dict(criterion=1, threshold=1, param=1e-2), None])
@pytest.mark.parametrize("dims,offs", [((61, 64), NINE), ((14, 15, 16), FIFTEEN)])
def test_local_method_vs_oracle(dims, offs, rule):
    A, b, x0 = stencil_system(dims, offs, 5)
    M = lc.Matrix(A.n, A.rp, A.ci, A.val)
    assert M.info()["layout"] == "stencil"
    x, rep = lc.local_method(M, dev(b), dev(x0), rule, keep=rule is not None)
    dp = None
    if rule is not None:
        dp = orc.DomainParams(rule["criterion"], rule["threshold"], rule["param"], rule.get("expand_rounds", 0), 0, 1)
    xo, flag, ro = orc.local_method(A, b, x0, dp, orc.SolverParams(0, 1, 30, EPS, 20000))
    if rule is not None:
        np.testing.assert_array_equal(rep["idx"].cpu().numpy(), np.flatnonzero(flag))
        if rep["K"][0] > 0:
            assert abs(rep["local"][0]["iterations"] - ro.it_local) <= 1
    assert abs(rep["global"][0]["iterations"] - ro.it_global) <= 1
    assert np.linalg.norm(x.cpu().numpy() - xo) / np.linalg.norm(xo) <= 1e-9


def three_t_system(dims, offsets_nd, seed, diagonal_couplings=True):
    """A nonsymmetric 3T-like block system on a regular grid: per cell a full 3x3 diagonal block (identity +
    exchange terms + the cell's share of the diffusion), per stored neighbour a coupling block -w diag(kappa_a)
    (diagonal, as the 3T couplings P:1477-1482) or, with diagonal_couplings=False, one coupling block with an
    off-diagonal entry.  Returns BSR arrays (row-major 3x3 blocks) + b, x0 for the 3 N unknowns."""
    A1, _, _ = stencil_system(dims, offsets_nd, seed)
    rng = np.random.default_rng(seed + 100)
    n = A1.n
    rp, ci, v1 = np.asarray(A1.rp), np.asarray(A1.ci), np.asarray(A1.val)
    kap = np.array([1.0, 0.35, 2.5])
    val = np.zeros((ci.size, 9))
    for u in range(n):
        off = 0.0
        for p in range(rp[u], rp[u + 1]):
            if ci[p] != u:
                val[p, [0, 4, 8]] = v1[p] * kap
                off += -v1[p]
        p = rp[u] + int(np.flatnonzero(ci[rp[u]:rp[u + 1]] == u)[0])
        W = rng.uniform(0.01, 30.0, (3, 3))
        np.fill_diagonal(W, 0.0)
        D = np.diag(1.0 + off * kap + W.sum(axis=1)) - W          # rows sum to 1 + diffusion: nonsymmetric, dominant
        val[p] = D.reshape(9)
    if not diagonal_couplings:
        u = n // 2
        p = rp[u] + (0 if ci[rp[u]] != u else 1)
        val[p, 1] = 0.25 * val[p, 0]
    xs = np.sin(0.03 * np.arange(3 * n)) + 0.7
    Ao = orc.Csr.from_bsr(rp, ci, val.reshape(-1))
    b = orc.spmv(Ao, xs)
    x0 = xs.copy()
    hot = slice(3 * (n // 3), 3 * (n // 3) + 3 * max(8, n // 40))
    x0[hot] += 0.4 * np.cos(0.11 * np.arange(hot.stop - hot.start))
    return rp, ci, val.reshape(-1), Ao, b, x0


@pytest.mark.parametrize("dims,offs,diag", [((33, 35), NINE, True), ((33, 35), NINE, False),
                                            ((40, 37), [(-1, 0), (0, -1), (0, 1), (1, 0)], True)])
@pytest.mark.parametrize("rule", [dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1), None])
def test_three_t_block_stencils_gmres(dims, offs, diag, rule):
    """Block 3 (3T) systems on the nine-point scheme and on a five-point grid with a ragged last slice:
    the GMRES kernel's rows -- the branch-free five-point row, the slot loop for other widths, the full-block path
    when a coupling block is not diagonal, the uniform-width explicit subsystem -- against the oracle's
    right-preconditioned block-Jacobi GMRES(30): cell-granular Omega equal, Arnoldi steps +-1, x within 1e-9."""
    rp, ci, val, Ao, b, x0 = three_t_system(dims, offs, 11, diag)
    n = rp.size - 1
    M = lc.Matrix(n, rp, ci, val, block=3)
    assert M.info()["layout"] == "stencil" and M.info()["max_row"] == len(offs) + 1
    x, rep = lc.local_method(M, dev(b), dev(x0), rule, method=lc.GMRES, keep=rule is not None)
    dp = None
    if rule is not None:
        dp = orc.DomainParams(rule["criterion"], rule["threshold"], rule["param"], rule["expand_rounds"], 0, 3)
    xo, flag, ro = orc.local_method(Ao, b, x0, dp, orc.SolverParams(1, 3, 30, EPS, 3000))
    if rule is not None:
        np.testing.assert_array_equal(rep["idx"].cpu().numpy(), np.flatnonzero(flag))
        assert rep["K"][0] > 0
        assert abs(rep["local"][0]["iterations"] - ro.it_local) <= 1
    assert abs(rep["global"][0]["iterations"] - ro.it_global) <= 1
    assert np.linalg.norm(x.cpu().numpy() - xo) / np.linalg.norm(xo) <= 1e-9
