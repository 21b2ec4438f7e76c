"""ctypes wrapper of the plain C oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs.  The product package
``paper_2001_01158_b200`` never imports this module.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

CRIT_RESIDUAL, CRIT_GRADIENT = 0, 1
THR_PAPER, THR_REL_MAX, THR_PERCENTILE = 0, 1, 2
OK, NOT_CONVERGED = 0, 1


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-std=c99", "-D_POSIX_C_SOURCE=199309L",
                               "-shared", "-fPIC", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


class DomainParams(ctypes.Structure):
    _fields_ = [("criterion", ctypes.c_int32), ("threshold", ctypes.c_int32), ("param", ctypes.c_double),
                ("expand_rounds", ctypes.c_int32), ("dilate_hops", ctypes.c_int32), ("cell", ctypes.c_int32)]


class Trace(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int32), ("front", ctypes.c_int64 * 64), ("admitted", ctypes.c_int64 * 64),
                ("K_after", ctypes.c_int64 * 64), ("K_base", ctypes.c_int64)]


class SolverParams(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int32), ("bs", ctypes.c_int32), ("restart", ctypes.c_int32),
                ("eps", ctypes.c_double), ("max_iters", ctypes.c_int32), ("gs_sweeps", ctypes.c_int32)]


class Report(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int64), ("tau", ctypes.c_double), ("it_local", ctypes.c_int32),
                ("it_global", ctypes.c_int32), ("st_local", ctypes.c_int32), ("st_global", ctypes.c_int32),
                ("relres_local", ctypes.c_double), ("relres_global", ctypes.c_double),
                ("t_select", ctypes.c_double), ("t_extract", ctypes.c_double), ("t_local", ctypes.c_double),
                ("t_global", ctypes.c_double)]


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.or_spmv.argtypes = [I64, P, P, P, P, P]
        lib.or_residual.argtypes = [I64, P, P, P, P, P, P]
        lib.or_norm2.argtypes = [I64, P]
        lib.or_norm2.restype = D
        lib.or_gradient.argtypes = [I64, P, P, P, P]
        lib.or_bsr_to_csr.argtypes = [I64, P, P, P, P, P, P]
        lib.or_select_domain.argtypes = [I64, P, P, P, P, P, ctypes.POINTER(DomainParams), P, P, P, P, P,
                                         ctypes.POINTER(Trace)]
        lib.or_extract.argtypes = [I64, P, P, P, P, P, P, P, P, P, P, P, P, P, P]
        lib.or_assemble.argtypes = [I64, P, P, P]
        lib.or_pcg.argtypes = [I64, P, P, P, P, P, D, I32, P, P]
        lib.or_gmres_bj.argtypes = [I64, P, P, P, I32, P, P, D, I32, I32, P, P]
        lib.or_gauss_seidel.argtypes = [I64, P, P, P, P, P, I32]
        lib.or_gauss_seidel.restype = I32
        lib.or_heat_assemble.argtypes = [I32, I32, D, I32, D, D, P, P, P, P, P, P]
        lib.or_heat_run.argtypes = [I32, I32, D, I32, D, D, I32, D, I32, ctypes.POINTER(DomainParams),
                                    ctypes.POINTER(SolverParams), P, P, ctypes.c_void_p]
        lib.or_heat_run.restype = I32
        lib.or_local_method.argtypes = [I64, P, P, P, P, P, ctypes.POINTER(DomainParams),
                                        ctypes.POINTER(SolverParams), P, ctypes.POINTER(Report), P]
        for f in ("or_select_domain", "or_extract", "or_pcg", "or_gmres_bj", "or_local_method"):
            getattr(lib, f).restype = I32
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class Csr:
    """Scalar CSR on the host (int64 row_ptr, int32 col, f64 val)."""

    def __init__(self, rp, ci, val):
        self.rp = _c(rp, np.int64); self.ci = _c(ci, np.int32); self.val = _c(val, np.float64)
        self.n = len(self.rp) - 1

    @staticmethod
    def from_bsr(brp, bci, bval) -> "Csr":
        nb = len(brp) - 1
        nnzb = len(bci)
        rp = np.empty(3 * nb + 1, np.int64); ci = np.empty(9 * nnzb, np.int32); a = np.empty(9 * nnzb)
        _load().or_bsr_to_csr(nb, _p(_c(brp, np.int64)), _p(_c(bci, np.int32)), _p(_c(bval, np.float64)),
                              _p(rp), _p(ci), _p(a))
        return Csr(rp, ci, a)

    @staticmethod
    def from_dense(M) -> "Csr":
        M = np.asarray(M, dtype=np.float64)
        n = M.shape[0]
        rp = [0]; ci = []; val = []
        for i in range(n):
            for j in range(n):
                if M[i, j] != 0.0 or i == j:
                    ci.append(j); val.append(M[i, j])
            rp.append(len(ci))
        return Csr(np.array(rp), np.array(ci), np.array(val))

    def segment(self, r0: int, r1: int) -> "Csr":
        """Rows [r0, r1) of a block-diagonal matrix, columns shifted by -r0."""
        k0, k1 = self.rp[r0], self.rp[r1]
        return Csr(self.rp[r0:r1 + 1] - k0, self.ci[k0:k1] - r0, self.val[k0:k1])

    def to_dense(self):
        M = np.zeros((self.n, self.n))
        for i in range(self.n):
            for k in range(self.rp[i], self.rp[i + 1]):
                M[i, self.ci[k]] = self.val[k]
        return M


def spmv(A: Csr, x):
    x = _c(x, np.float64); y = np.empty(A.n)
    _load().or_spmv(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(x), _p(y))
    return y


def residual(A: Csr, b, x):
    b = _c(b, np.float64); x = _c(x, np.float64); r = np.empty(A.n)
    _load().or_residual(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(b), _p(x), _p(r))
    return r


def norm2(v):
    v = _c(v, np.float64)
    return _load().or_norm2(len(v), _p(v))


def gradient(A: Csr, x):
    x = _c(x, np.float64); g = np.empty(A.n)
    _load().or_gradient(A.n, _p(A.rp), _p(A.ci), _p(x), _p(g))
    return g


@dataclass
class Domain:
    flag: np.ndarray      # uint8[n] per scalar row
    K: int
    tau: float
    crit: np.ndarray      # per unit (cell)
    adm: np.ndarray       # per unit, NaN if never a neighbour
    trace: dict

    @property
    def idx(self):
        return np.flatnonzero(self.flag)


def select_domain(A: Csr, b, x0, criterion=CRIT_RESIDUAL, threshold=THR_PAPER, param=1e-10, expand_rounds=0,
                  dilate_hops=0, cell=1) -> Domain:
    lib = _load()
    b = _c(b, np.float64); x0 = _c(x0, np.float64)
    m = A.n // cell
    flag = np.zeros(A.n, np.uint8); crit = np.zeros(max(m, 1)); adm = np.zeros(max(m, 1))
    tau = np.zeros(1); K = np.zeros(1, np.int64); tr = Trace()
    p = DomainParams(criterion, threshold, param, expand_rounds, dilate_hops, cell)
    st = lib.or_select_domain(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(b), _p(x0), ctypes.byref(p), _p(flag),
                              _p(crit), _p(adm), _p(tau), _p(K), ctypes.byref(tr))
    if st != 0:
        raise ValueError(f"or_select_domain status {st}")
    trace = {"rounds": tr.rounds, "front": list(tr.front[:tr.rounds]), "admitted": list(tr.admitted[:tr.rounds]),
             "K_after": list(tr.K_after[:tr.rounds]), "K_base": tr.K_base}
    return Domain(flag, int(K[0]), float(tau[0]), crit[:m], adm[:m], trace)


@dataclass
class Sub:
    idx: np.ndarray
    B: Csr
    bsub: np.ndarray
    xB0: np.ndarray


def extract(A: Csr, b, x0, flag) -> Sub:
    lib = _load()
    b = _c(b, np.float64); x0 = _c(x0, np.float64); flag = _c(flag, np.uint8)
    K0 = int(flag.sum()); nnz = int(A.rp[-1])
    idx = np.empty(max(K0, 1), np.int64); Brp = np.empty(K0 + 1, np.int64)
    Bci = np.empty(max(nnz, 1), np.int32); Ba = np.empty(max(nnz, 1)); bsub = np.empty(max(K0, 1))
    xB0 = np.empty(max(K0, 1)); K = np.zeros(1, np.int64); Bn = np.zeros(1, np.int64)
    lib.or_extract(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(b), _p(x0), _p(flag), _p(idx), _p(Brp), _p(Bci), _p(Ba),
                   _p(bsub), _p(xB0), _p(K), _p(Bn))
    K = int(K[0]); Bn = int(Bn[0])
    return Sub(idx[:K], Csr(Brp, Bci[:Bn], Ba[:Bn]), bsub[:K], xB0[:K])


def assemble(sub: Sub, xB, x):
    x = np.array(x, dtype=np.float64, copy=True)
    x[sub.idx] = xB
    return x


def pcg(A: Csr, b, x0, eps=1e-10, max_iters=20000):
    b = _c(b, np.float64); x = np.array(x0, dtype=np.float64, copy=True)
    it = np.zeros(1, np.int32); rr = np.zeros(1)
    st = _load().or_pcg(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(b), _p(x), eps, max_iters, _p(it), _p(rr))
    return x, int(it[0]), st, float(rr[0])


def gmres_bj(A: Csr, b, x0, bs=3, eps=1e-10, restart=30, max_iters=3000):
    b = _c(b, np.float64); x = np.array(x0, dtype=np.float64, copy=True)
    it = np.zeros(1, np.int32); rr = np.zeros(1)
    st = _load().or_gmres_bj(A.n, _p(A.rp), _p(A.ci), _p(A.val), bs, _p(b), _p(x), eps, restart, max_iters,
                             _p(it), _p(rr))
    return x, int(it[0]), st, float(rr[0])


def gauss_seidel(A: Csr, b, x, sweeps=1):
    """Alg. 1 l.7: forward natural-order Gauss-Seidel sweeps (returns a new vector)."""
    b = _c(b, np.float64); y = np.array(x, dtype=np.float64, copy=True)
    st = _load().or_gauss_seidel(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(b), _p(y), sweeps)
    if st != 0:
        raise ValueError(f"or_gauss_seidel status {st}")
    return y


class HeatReport(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_int32), ("picard_total", ctypes.c_int32), ("picard_max_hit", ctypes.c_int32),
                ("it_local", ctypes.c_int64), ("it_global", ctypes.c_int64), ("eta_sum", ctypes.c_double),
                ("seconds", ctypes.c_double)]


def heat_assemble(nx, ny, dt, Ts, Told, khalf=3, Tl=1.0, Tr=1e-4):
    """The paper's 2-D heat Picard system at the iterate Ts: (Csr, b)."""
    n = nx * ny
    rp = np.empty(n + 1, np.int64); ci = np.empty(5 * n, np.int32); a = np.empty(5 * n); b = np.empty(n)
    _load().or_heat_assemble(nx, ny, dt, khalf, Tl, Tr, _p(_c(Ts, np.float64)), _p(_c(Told, np.float64)), _p(rp),
                             _p(ci), _p(a), _p(b))
    z = int(rp[-1])
    return Csr(rp, ci[:z], a[:z]), b


def heat_run(nx, ny, T0, steps, domain: DomainParams | None, solver: SolverParams, dt=1e-2, khalf=3, Tl=1.0,
             Tr=1e-4, picard_tol=1e-8, picard_max=100):
    """Alg. 6 on the CPU oracle.  Returns (T_final, picard counts per step, HeatReport)."""
    T = np.array(T0, dtype=np.float64, copy=True)
    per = np.zeros(max(steps, 1), np.int32); rep = HeatReport()
    st = _load().or_heat_run(nx, ny, dt, khalf, Tl, Tr, steps, picard_tol, picard_max,
                             ctypes.byref(domain) if domain is not None else None, ctypes.byref(solver), _p(T),
                             _p(per), ctypes.byref(rep))
    if st < 0:
        raise RuntimeError(f"or_heat_run status {st}")
    return T, per[:steps], rep


def local_method(A: Csr, b, x0, domain: DomainParams | None, solver: SolverParams, want_xt=False):
    """Alg. 1 (domain given) or method0 (domain None).  Returns (x, flag, Report), plus x~ (Eq. 4, after
    Alg. 1 l.6, before any GS sweep) when want_xt."""
    b = _c(b, np.float64); x = np.array(x0, dtype=np.float64, copy=True)
    flag = np.zeros(A.n, np.uint8); rep = Report()
    xt = np.array(x0, dtype=np.float64, copy=True) if want_xt else None
    st = _load().or_local_method(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(b), _p(x),
                                 ctypes.byref(domain) if domain is not None else None, ctypes.byref(solver),
                                 _p(flag), ctypes.byref(rep), _p(xt))
    if st < 0:
        raise RuntimeError(f"or_local_method status {st}")
    return (x, flag, rep, xt) if want_xt else (x, flag, rep)


def tau_paper(b, eps):
    """Eq. 7 threshold as the oracle evaluates it: eps * ||b||_2 / sqrt(N)."""
    return eps * norm2(b) / math.sqrt(len(b))
