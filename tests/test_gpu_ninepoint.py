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
