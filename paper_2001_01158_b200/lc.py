"""Thin ctypes binding of liblc.so (include/lc.h).  Argument marshalling only:
every step of the path runs in the library's sm_100a kernels.  PyTorch supplies
device memory and the current CUDA stream.

There is NO CPU fallback: if liblc.so is missing or CUDA is unavailable, every
call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblc.so")

LC_OK, LC_NOT_CONVERGED = 0, 1
FMT_SELL32 = 0
CRIT_RESIDUAL, CRIT_GRADIENT = 0, 1
THR_PAPER, THR_REL_MAX, THR_PERCENTILE = 0, 1, 2
PCG, GMRES = 0, 1
JACOBI, BLOCK_JACOBI = 0, 1

_STATUS = {0: "LC_OK", 1: "LC_NOT_CONVERGED", -1: "LC_ERR_INVALID_ARG", -2: "LC_ERR_DIMENSION",
           -3: "LC_ERR_PATTERN", -4: "LC_ERR_ZERO_DIAGONAL", -5: "LC_ERR_BREAKDOWN", -6: "LC_ERR_NONFINITE",
           -7: "LC_ERR_CUDA", -8: "LC_ERR_OOM"}

EXPORTED = ["lc_create_csr", "lc_update_values", "lc_select_domain", "lc_domain_export", "lc_extract_sub", "lc_solve_local",
            "lc_solve_global", "lc_smooth_gs", "lc_heat_assemble", "lc_heat_run", "lc_matrix_info", "lc_destroy_matrix", "lc_destroy_domain",
            "lc_destroy_sub", "lc_spmv", "lc_spmv_csr", "lc_dist_create", "lc_dist_export_handle", "lc_dist_connect", "lc_dist_connect_local",
            "lc_dist_select_domain", "lc_dist_domain_export", "lc_dist_solve_local", "lc_dist_solve_global",
            "lc_dist_destroy", "lc_last_error", "lc_kernel_launches", "lc_tuning_defaults", "lc_set_tuning",
            "lc_get_tuning", "lc_sub_export", "lc_local_method"]
DIST_HANDLE_BYTES = 64


class LcError(RuntimeError):
    def __init__(self, status, where, msg):
        super().__init__(f"{where}: {_STATUS.get(status, status)}: {msg}")
        self.status = status


class DomainParams(ctypes.Structure):
    _fields_ = [("criterion", ctypes.c_int32), ("threshold", ctypes.c_int32), ("param", ctypes.c_double),
                ("expand_rounds", ctypes.c_int32), ("dilate_hops", ctypes.c_int32)]


class SolverParams(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int32), ("precond", ctypes.c_int32), ("restart", ctypes.c_int32),
                ("rel_tol", ctypes.c_double), ("max_iters", ctypes.c_int32)]


class HeatParams(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("dt", ctypes.c_double), ("khalf", ctypes.c_int32),
                ("t_left", ctypes.c_double), ("t_right", ctypes.c_double), ("steps", ctypes.c_int32),
                ("picard_tol", ctypes.c_double), ("picard_max", ctypes.c_int32), ("method", ctypes.c_int32),
                ("alpha", ctypes.c_double), ("e_max", ctypes.c_int32), ("gs_sweeps", ctypes.c_int32),
                ("rel_tol", ctypes.c_double)]


class HeatReport(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_int32), ("picard_total", ctypes.c_int32), ("picard_max_hit", ctypes.c_int32),
                ("it_local", ctypes.c_int64), ("it_global", ctypes.c_int64), ("eta_sum", ctypes.c_double),
                ("seconds", ctypes.c_double), ("local_not_converged", ctypes.c_int32),
                ("global_not_converged", ctypes.c_int32)]


class SolveInfo(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("status", ctypes.c_int32), ("rel_residual", ctypes.c_double),
                ("seconds", ctypes.c_double), ("kernel", ctypes.c_int32), ("lazy_x_depth", ctypes.c_int32)]


class MethodTimes(ctypes.Structure):
    _fields_ = [("select", ctypes.c_double), ("extract", ctypes.c_double), ("local", ctypes.c_double),
                ("gs", ctypes.c_double), ("global_", ctypes.c_double)]


KERNELS = {0: "none", 1: "pcg_grid", 2: "pcg_cluster", 3: "pcg_resident", 4: "pcg_lockstep", 5: "pcg_teams",
           6: "gmres", 7: "pcg_dynteams"}


class Tuning(ctypes.Structure):
    """lc_tuning (include/lc.h): implementation choices of the calling thread, all parity-tested."""
    _fields_ = [("stencil_layout", ctypes.c_int32), ("symmetric_layout", ctypes.c_int32),
                ("pcg_cluster_resident", ctypes.c_int32), ("pcg_cluster", ctypes.c_int32),
                ("pcg_tma", ctypes.c_int32), ("lazy_x_depth", ctypes.c_int32), ("batched_schedule", ctypes.c_int32),
                ("pcg_max_ctas", ctypes.c_int32), ("sub_repr", ctypes.c_int32), ("gmres_exact_cgs2", ctypes.c_int32),
                ("gs_lines", ctypes.c_int32), ("spmv_csr_tma", ctypes.c_int32),
                ("spmv_tma", ctypes.c_int32), ("batched_cluster", ctypes.c_int32),
                ("block_dcoup", ctypes.c_int32), ("l2_stream_hint", ctypes.c_int32)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load liblc.so and declare the C signatures (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built (run __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    lib.lc_create_csr.argtypes = [I64, I32, I32, P, P, P, I32, I32, P, ctypes.POINTER(P)]
    lib.lc_select_domain.argtypes = [P, P, P, ctypes.POINTER(DomainParams), P, ctypes.POINTER(P), P]
    lib.lc_domain_export.argtypes = [P, P, P, P, P, P]
    lib.lc_extract_sub.argtypes = [P, P, P, P, P, ctypes.POINTER(P)]
    lib.lc_sub_export.argtypes = [P, P, P, P]
    lib.lc_sub_export.restype = ctypes.c_int
    lib.lc_solve_local.argtypes = [P, ctypes.POINTER(SolverParams), P, P, P]
    lib.lc_solve_global.argtypes = [P, P, P, ctypes.POINTER(SolverParams), P, P]
    lib.lc_matrix_info.argtypes = [P, P, P, P, P, P, P, P]
    lib.lc_smooth_gs.argtypes = [P, P, P, I32, P]
    lib.lc_spmv.argtypes = [P, P, P, P]
    lib.lc_spmv.restype = ctypes.c_int
    lib.lc_spmv_csr.argtypes = [I64, P, P, P, P, P, P]
    lib.lc_spmv_csr.restype = ctypes.c_int
    lib.lc_update_values.argtypes = [P, P, P, P, I32, P]
    lib.lc_local_method.argtypes = [P, P, P, ctypes.POINTER(DomainParams), ctypes.POINTER(SolverParams), I32, P, P, P,
                                    P, P, ctypes.POINTER(SolveInfo), ctypes.POINTER(SolveInfo),
                                    ctypes.POINTER(MethodTimes)]
    lib.lc_heat_assemble.argtypes = [I32, I32, D, I32, D, D, P, P, P, P, P, P, P]
    lib.lc_heat_run.argtypes = [ctypes.POINTER(HeatParams), P, P, P, P, ctypes.POINTER(HeatReport)]
    for f in ("lc_create_csr", "lc_select_domain", "lc_domain_export", "lc_extract_sub", "lc_solve_local",
              "lc_solve_global", "lc_matrix_info", "lc_smooth_gs", "lc_heat_assemble", "lc_heat_run",
              "lc_update_values", "lc_local_method"):
        getattr(lib, f).restype = ctypes.c_int
    PP = ctypes.POINTER(P)
    lib.lc_dist_create.argtypes = [I64, I64, I64, I32, I32, P, P, P, I32, P, PP]
    lib.lc_dist_export_handle.argtypes = [P, P]
    lib.lc_dist_connect.argtypes = [P, P, P]
    lib.lc_dist_connect_local.argtypes = [PP, I32]
    lib.lc_dist_select_domain.argtypes = [PP, I32, PP, PP, ctypes.POINTER(DomainParams), P, P]
    lib.lc_dist_domain_export.argtypes = [P, P, P, P]
    lib.lc_dist_solve_local.argtypes = [PP, I32, ctypes.POINTER(SolverParams), PP, P, ctypes.POINTER(SolveInfo)]
    lib.lc_dist_solve_global.argtypes = [PP, I32, PP, PP, ctypes.POINTER(SolverParams), P, ctypes.POINTER(SolveInfo)]
    for f in ("lc_dist_create", "lc_dist_export_handle", "lc_dist_connect", "lc_dist_connect_local",
              "lc_dist_select_domain", "lc_dist_domain_export", "lc_dist_solve_local", "lc_dist_solve_global"):
        getattr(lib, f).restype = ctypes.c_int
    lib.lc_dist_destroy.argtypes = [P]
    lib.lc_dist_destroy.restype = None
    for f in ("lc_destroy_matrix", "lc_destroy_domain", "lc_destroy_sub"):
        getattr(lib, f).argtypes = [P]
        getattr(lib, f).restype = None
    lib.lc_tuning_defaults.argtypes = [ctypes.POINTER(Tuning)]
    lib.lc_tuning_defaults.restype = None
    lib.lc_set_tuning.argtypes = [ctypes.POINTER(Tuning)]
    lib.lc_set_tuning.restype = ctypes.c_int
    lib.lc_get_tuning.argtypes = [ctypes.POINTER(Tuning)]
    lib.lc_get_tuning.restype = ctypes.c_int
    lib.lc_last_error.restype = ctypes.c_char_p
    lib.lc_kernel_launches.restype = ctypes.c_int64
    _lib = lib
    return lib


def _check(st, where, ok=(LC_OK, LC_NOT_CONVERGED)):
    if st not in ok:
        raise LcError(st, where, load_library().lc_last_error().decode())
    return st


def _stream():
    if not torch.cuda.is_available():
        raise RuntimeError("CUDA device required: liblc has no CPU path")
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dptr(t: torch.Tensor, dtype, n=None):
    if not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise TypeError(f"expected a contiguous CUDA {dtype} tensor, got {t.dtype} on {t.device}")
    if n is not None and t.numel() < n:
        raise ValueError(f"tensor has {t.numel()} elements, need {n}")
    return ctypes.c_void_p(t.data_ptr())


def kernel_launches() -> int:
    return int(load_library().lc_kernel_launches())


def tuning_defaults() -> dict:
    t = Tuning()
    load_library().lc_tuning_defaults(ctypes.byref(t))
    return {f: getattr(t, f) for f, _ in Tuning._fields_}


def get_tuning() -> dict:
    t = Tuning()
    _check(load_library().lc_get_tuning(ctypes.byref(t)), "lc_get_tuning", ok=(LC_OK,))
    return {f: getattr(t, f) for f, _ in Tuning._fields_}


def set_tuning(**fields) -> dict:
    """Set the calling thread's lc_tuning: the library defaults updated by `fields` (no argument = defaults).
    Returns the previous setting (pass it back as set_tuning(**prev) to restore)."""
    prev = get_tuning()
    t = Tuning()
    load_library().lc_tuning_defaults(ctypes.byref(t))
    for k, v in fields.items():
        if k not in prev:
            raise KeyError(f"unknown lc_tuning field {k!r}")
        setattr(t, k, int(v))
    _check(load_library().lc_set_tuning(ctypes.byref(t)), "lc_set_tuning", ok=(LC_OK,))
    return prev


class Matrix:
    """A (Eq. 1) in the library's SELL-32 layout.  row_ptr/col_idx/values may be host numpy arrays or CUDA
    tensors (copied either way).  block = 3: BSR with 9 f64 per block; batch = G equal diagonal segments."""

    def __init__(self, n, row_ptr, col_idx, values, block=1, batch=1):
        lib = load_library()
        s = _stream()
        self.n_units, self.block, self.batch = int(n), int(block), int(batch)
        h = ctypes.c_void_p()
        if isinstance(row_ptr, torch.Tensor) and row_ptr.is_cuda:
            st = lib.lc_create_csr(n, block, batch, _dptr(row_ptr, torch.int64), _dptr(col_idx, torch.int32),
                                   _dptr(values, torch.float64), 1, FMT_SELL32, s, ctypes.byref(h))
        else:
            import numpy as np
            rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
            ci = np.ascontiguousarray(col_idx, dtype=np.int32)
            va = np.ascontiguousarray(values, dtype=np.float64)
            st = lib.lc_create_csr(n, block, batch, rp.ctypes.data, ci.ctypes.data, va.ctypes.data, 0, FMT_SELL32,
                                   s, ctypes.byref(h))
        _check(st, "lc_create_csr", ok=(LC_OK,))
        self.h = h

    def update_values(self, row_ptr, col_idx, values):
        """New values for the pattern the matrix was created with (lc_update_values)."""
        s = _stream()
        if isinstance(row_ptr, torch.Tensor) and row_ptr.is_cuda:
            st = load_library().lc_update_values(self.h, _dptr(row_ptr, torch.int64), _dptr(col_idx, torch.int32),
                                                 _dptr(values, torch.float64), 1, s)
        else:
            import numpy as np
            rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
            ci = np.ascontiguousarray(col_idx, dtype=np.int32)
            va = np.ascontiguousarray(values, dtype=np.float64)
            st = load_library().lc_update_values(self.h, rp.ctypes.data, ci.ctypes.data, va.ctypes.data, 0, s)
        _check(st, "lc_update_values", ok=(LC_OK,))

    @property
    def N(self):
        return self.n_units * self.block

    def info(self):
        vals = [ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32(),
                ctypes.c_int32(), ctypes.c_int64()]
        _check(load_library().lc_matrix_info(self.h, *[ctypes.byref(v) for v in vals]), "lc_matrix_info")
        return dict(N=vals[0].value, nnz=vals[1].value, batch=vals[2].value, nslices=vals[3].value,
                    max_row=vals[4].value, layout={0: "sell", 1: "stencil", 2: "symstencil"}[vals[5].value],
                    matrix_bytes=vals[6].value)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.lc_destroy_matrix(self.h)
            self.h = None


@dataclass
class DomainResult:
    dom: "Domain"
    K: list


class Domain:
    def __init__(self, A: Matrix, h, K):
        self.A, self.h, self.K = A, h, K

    def export(self, want_crit=False, want_adm=False):
        """-> (idx int32 CUDA tensor [sum K], tau list [batch], crit [n_units] or None, adm or None)"""
        s = _stream()
        dev = torch.device("cuda")
        total = int(sum(self.K))
        idx = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        tau = (ctypes.c_double * self.A.batch)()
        crit = torch.empty(self.A.n_units, dtype=torch.float64, device=dev) if want_crit else None
        adm = torch.empty(self.A.n_units, dtype=torch.float64, device=dev) if want_adm else None
        _check(load_library().lc_domain_export(self.h, ctypes.c_void_p(idx.data_ptr()), tau,
                                     ctypes.c_void_p(crit.data_ptr()) if crit is not None else None,
                                     ctypes.c_void_p(adm.data_ptr()) if adm is not None else None, s),
               "lc_domain_export")
        return idx[:total], list(tau), crit, adm

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.lc_destroy_domain(self.h)
            self.h = None


def select_domain(A: Matrix, b: torch.Tensor, x0: torch.Tensor, criterion=CRIT_RESIDUAL, threshold=THR_PAPER,
                  param=1e-10, expand_rounds=0, dilate_hops=0) -> Domain:
    s = _stream()
    p = DomainParams(criterion, threshold, param, expand_rounds, dilate_hops)
    h = ctypes.c_void_p()
    K = (ctypes.c_int64 * A.batch)()
    _check(load_library().lc_select_domain(A.h, _dptr(b, torch.float64, A.N), _dptr(x0, torch.float64, A.N), ctypes.byref(p),
                                 s, ctypes.byref(h), K), "lc_select_domain", ok=(LC_OK,))
    return Domain(A, h, list(K))


class Sub:
    def __init__(self, A: Matrix, dom: Domain, b, x0):
        s = _stream()
        h = ctypes.c_void_p()
        _check(load_library().lc_extract_sub(A.h, dom.h, _dptr(b, torch.float64, A.N), _dptr(x0, torch.float64, A.N), s,
                                   ctypes.byref(h)), "lc_extract_sub", ok=(LC_OK,))
        self.h, self.A, self.K = h, A, list(dom.K)

    def export(self):
        """-> (b_sub, x_B0): CUDA f64 tensors [sum K] in Omega order (lc_sub_export, Eq. 3)."""
        tot = int(sum(self.K))
        bsub = torch.empty(max(tot, 1), dtype=torch.float64, device="cuda")
        xb0 = torch.empty(max(tot, 1), dtype=torch.float64, device="cuda")
        _check(load_library().lc_sub_export(self.h, ctypes.c_void_p(bsub.data_ptr()), ctypes.c_void_p(xb0.data_ptr()),
                                            _stream()), "lc_sub_export", ok=(LC_OK,))
        return bsub[:tot], xb0[:tot]

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.lc_destroy_sub(self.h)
            self.h = None


def extract_sub(A: Matrix, dom: Domain, b, x0) -> Sub:
    return Sub(A, dom, b, x0)


def _solver(method, rel_tol, max_iters, restart):
    if method == PCG:
        return SolverParams(PCG, JACOBI, restart, rel_tol, max_iters)
    return SolverParams(GMRES, BLOCK_JACOBI, restart, rel_tol, max_iters)


def _infos(arr):
    return [dict(iterations=i.iterations, status=i.status, rel_residual=i.rel_residual, seconds=i.seconds,
                 kernel=KERNELS.get(i.kernel, i.kernel), lazy_x_depth=i.lazy_x_depth) for i in arr]


def solve_local(sub: Sub, x: torch.Tensor, method=PCG, rel_tol=1e-10, max_iters=20000, restart=30):
    """Alg. 1 l.5-6: x (in = x0) becomes x~ (Omega entries replaced by the subsystem solution)."""
    s = _stream()
    p = _solver(method, rel_tol, max_iters, restart)
    info = (SolveInfo * sub.A.batch)()
    st = load_library().lc_solve_local(sub.h, ctypes.byref(p), _dptr(x, torch.float64, sub.A.N), s, info)
    _check(st, "lc_solve_local")
    return _infos(info)


def solve_global(A: Matrix, b: torch.Tensor, x: torch.Tensor, method=PCG, rel_tol=1e-10, max_iters=20000,
                 restart=30):
    """Alg. 1 l.8-11 (or method0 when x = x0): in-place solve of A x = b from the warm start x."""
    s = _stream()
    p = _solver(method, rel_tol, max_iters, restart)
    info = (SolveInfo * A.batch)()
    st = load_library().lc_solve_global(A.h, _dptr(b, torch.float64, A.N), _dptr(x, torch.float64, A.N), ctypes.byref(p), s,
                              info)
    _check(st, "lc_solve_global")
    return _infos(info)


def spmv(A: Matrix, x: torch.Tensor, y: torch.Tensor):
    """y = A x on the current stream (lc_spmv)."""
    _check(load_library().lc_spmv(A.h, _dptr(x, torch.float64, A.N), _dptr(y, torch.float64, A.N), _stream()),
           "lc_spmv", ok=(LC_OK,))
    return y


def spmv_csr(row_ptr: torch.Tensor, col_idx: torch.Tensor, values: torch.Tensor, x: torch.Tensor, y: torch.Tensor):
    """y = A x from CSR device tensors (lc_spmv_csr, the row-slab CSR kernel)."""
    n = row_ptr.numel() - 1
    _check(load_library().lc_spmv_csr(n, _dptr(row_ptr, torch.int64), _dptr(col_idx, torch.int32),
                                      _dptr(values, torch.float64), _dptr(x, torch.float64, n),
                                      _dptr(y, torch.float64, n), _stream()), "lc_spmv_csr", ok=(LC_OK,))
    return y


def smooth_gs(A: Matrix, b: torch.Tensor, x: torch.Tensor, sweeps=1):
    """Alg. 1 l.7: forward natural-order Gauss-Seidel sweeps on x, in place."""
    _check(load_library().lc_smooth_gs(A.h, _dptr(b, torch.float64, A.N), _dptr(x, torch.float64, A.N), sweeps, _stream()),
           "lc_smooth_gs", ok=(LC_OK,))


def local_method(A: Matrix, b, x0, domain: dict | None, method=PCG, rel_tol=1e-10, max_iters=20000, restart=30,
                 gs_sweeps=0, keep=False, timing=False):
    """Alg. 1 in one C-ABI call (lc_local_method; domain=None: method0): domain (l.2), extraction (l.3-4), local
    solve + assembly (l.5-6), gs_sweeps Gauss-Seidel sweeps (l.7), global solve (l.8-11), two host syncs.
    Returns (x, report dict): K per segment, "local" / "global" solve infos per segment, "ms" = device time of
    each phase on the current stream (select, extract, local, gs, global).  keep=True also returns rep["idx"]
    (Omega, ascending rows) and rep["xt"] (x~ of Eq. 4, before any GS sweep).  `timing` is accepted for the
    composed form's signature (the phase times are always reported)."""
    s = _stream()
    N = A.N
    bp, x0p = _dptr(b, torch.float64, N), _dptr(x0, torch.float64, N)
    x = torch.empty_like(x0)
    xt = torch.empty_like(x0) if keep else None
    idx = torch.empty(max(N, 1), dtype=torch.int32, device=x0.device) if keep and domain is not None else None
    dp = DomainParams(domain.get("criterion", CRIT_RESIDUAL), domain.get("threshold", THR_PAPER),
                      domain.get("param", 1e-10), domain.get("expand_rounds", 0),
                      domain.get("dilate_hops", 0)) if domain is not None else None
    sp = _solver(method, rel_tol, max_iters, restart)
    K = (ctypes.c_int64 * A.batch)()
    li, gi = (SolveInfo * A.batch)(), (SolveInfo * A.batch)()
    tm = MethodTimes()
    st = load_library().lc_local_method(A.h, bp, x0p, ctypes.byref(dp) if dp is not None else None, ctypes.byref(sp),
                                        int(gs_sweeps), ctypes.c_void_p(x.data_ptr()),
                                        ctypes.c_void_p(xt.data_ptr()) if xt is not None else None,
                                        ctypes.c_void_p(idx.data_ptr()) if idx is not None else None, s, K, li, gi,
                                        ctypes.byref(tm))
    _check(st, "lc_local_method")
    rep = {"K": list(K), "global": _infos(gi),
           "ms": {"select": tm.select, "extract": tm.extract, "local": tm.local, "gs": tm.gs, "global": tm.global_}}
    if domain is not None and sum(rep["K"]) > 0:
        rep["local"] = _infos(li)
    if keep:
        rep["xt"] = xt
        if idx is not None:
            rep["idx"] = idx[:sum(rep["K"])]
    return x, rep


def local_method_steps(A: Matrix, b, x0, domain: dict | None, method=PCG, rel_tol=1e-10, max_iters=20000, restart=30,
                 gs_sweeps=0, keep=False, timing=False):
    """Alg. 1 composed from the step-by-step C-ABI calls (domain=None: method0): domain (l.2), extraction (l.3-4),
    local solve + assembly (l.5-6), gs_sweeps Gauss-Seidel sweeps (l.7), global solve (l.8-11).
    Returns (x, report dict).  keep=True also returns the intermediate results for parity checks:
    rep["idx"] (Omega, ascending rows), rep["tau"], rep["bsub"], rep["xB0"] (Eq. 3, Omega order) and
    rep["xt"] (x~ of Eq. 4, before any GS sweep).  timing=True: rep["ms"] = CUDA-event times of the phases on
    the current stream (select = l.2, extract = l.3-4, local = l.5-6, gs = l.7, global = l.8-11)."""
    ev = {}

    def mark(k):
        if timing:
            ev[k] = torch.cuda.Event(enable_timing=True)
            ev[k].record()
    mark("start")
    x = x0.clone()
    rep = {"K": [0] * A.batch}
    if domain is not None:
        dom = select_domain(A, b, x0, **domain)
        mark("select")
        rep["K"] = dom.K
        if keep:
            idx, tau, _, _ = dom.export()
            rep["idx"], rep["tau"] = idx, tau
        if sum(dom.K) > 0:
            sub = extract_sub(A, dom, b, x0)
            mark("extract")
            if keep:
                rep["bsub"], rep["xB0"] = sub.export()
            rep["local"] = solve_local(sub, x, method, rel_tol, max_iters, restart)
        mark("local")
        if keep:
            rep["xt"] = x.clone()
        if gs_sweeps > 0:
            smooth_gs(A, b, x, gs_sweeps)
        mark("gs")
    rep["global"] = solve_global(A, b, x, method, rel_tol, max_iters, restart)
    mark("global")
    if timing:
        ev["global"].synchronize()
        order = [k for k in ("start", "select", "extract", "local", "gs", "global") if k in ev]
        rep["ms"] = {k: ev[p].elapsed_time(ev[k]) for p, k in zip(order, order[1:])}
    return x, rep


def heat_assemble(nx, ny, dt, Ts: torch.Tensor, Told: torch.Tensor, khalf=3, t_left=1.0, t_right=1e-4):
    """The paper's heat Picard system on the device -> (row_ptr, col_idx, values, b) CUDA tensors."""
    n = nx * ny
    nnz = 5 * n - 2 * nx - 2 * ny
    dev = Ts.device
    rp = torch.empty(n + 1, dtype=torch.int64, device=dev)
    ci = torch.empty(nnz, dtype=torch.int32, device=dev)
    va = torch.empty(nnz, dtype=torch.float64, device=dev)
    b = torch.empty(n, dtype=torch.float64, device=dev)
    _check(load_library().lc_heat_assemble(nx, ny, dt, khalf, t_left, t_right, _dptr(Ts, torch.float64, n),
                                 _dptr(Told, torch.float64, n), _dptr(rp, torch.int64), _dptr(ci, torch.int32),
                                 _dptr(va, torch.float64), _dptr(b, torch.float64), _stream()), "lc_heat_assemble",
           ok=(LC_OK,))
    return rp, ci, va, b


def heat_run(nx, ny, T0: torch.Tensor, steps, method=0, alpha=1e-4, e_max=1, gs_sweeps=1, dt=1e-2, khalf=3,
             t_left=1.0, t_right=1e-4, picard_tol=1e-8, picard_max=100, rel_tol=1e-10):
    """Alg. 6 on the device (lc_heat_run).  Returns (T, picard counts per step, mean eta per step, report);
    report.global_not_converged counts global solves that hit their cap (LC_NOT_CONVERGED, non-fatal)."""
    import numpy as np
    p = HeatParams(nx, ny, dt, khalf, t_left, t_right, steps, picard_tol, picard_max, method, alpha, e_max,
                   gs_sweeps, rel_tol)
    T = T0.clone()
    per = np.zeros(max(steps, 1), np.int32)
    eta = np.zeros(max(steps, 1), np.float64)
    rep = HeatReport()
    _check(load_library().lc_heat_run(ctypes.byref(p), _dptr(T, torch.float64, nx * ny), per.ctypes.data, eta.ctypes.data,
                            _stream(), ctypes.byref(rep)), "lc_heat_run")
    return T, per[:steps], eta[:steps], rep


# ---- NEXT-4: row-partitioned multi-GPU form (include/lc.h "lc_dist_*", Alg. 4/5) ----

class DistRank:
    """One rank's row slab [row0, row0 + n_local) of an n_global-row stencil system (lc_dist_create).
    row_ptr (0-based, n_local + 1), col_idx (GLOBAL columns) and values: host numpy arrays or CUDA tensors."""

    def __init__(self, n_global, row0, n_local, rank, nranks, row_ptr, col_idx, values):
        lib = load_library()
        s = _stream()
        self.n_global, self.row0, self.n_local = int(n_global), int(row0), int(n_local)
        self.rank, self.nranks = int(rank), int(nranks)
        h = ctypes.c_void_p()
        if isinstance(row_ptr, torch.Tensor) and row_ptr.is_cuda:
            st = lib.lc_dist_create(n_global, row0, n_local, rank, nranks, _dptr(row_ptr, torch.int64),
                                    _dptr(col_idx, torch.int32), _dptr(values, torch.float64), 1, s, ctypes.byref(h))
        else:
            import numpy as np
            rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
            ci = np.ascontiguousarray(col_idx, dtype=np.int32)
            va = np.ascontiguousarray(values, dtype=np.float64)
            st = lib.lc_dist_create(n_global, row0, n_local, rank, nranks, rp.ctypes.data, ci.ctypes.data,
                                    va.ctypes.data, 0, s, ctypes.byref(h))
        _check(st, "lc_dist_create", ok=(LC_OK,))
        self.h = h

    def export_handle(self) -> bytes:
        buf = (ctypes.c_char * DIST_HANDLE_BYTES)()
        _check(load_library().lc_dist_export_handle(self.h, buf), "lc_dist_export_handle", ok=(LC_OK,))
        return bytes(buf)

    def connect(self, handles, n_local_all):
        """One process per rank: handles = every rank's export_handle() bytes in rank order."""
        import numpy as np
        blob = b"".join(handles)
        nl = np.ascontiguousarray(n_local_all, dtype=np.int64)
        _check(load_library().lc_dist_connect(self.h, blob, nl.ctypes.data), "lc_dist_connect", ok=(LC_OK,))

    def domain_flags(self):
        """-> (uint8 CUDA tensor [n_local]: stage or 255, tau)"""
        f = torch.empty(self.n_local, dtype=torch.uint8, device="cuda")
        tau = ctypes.c_double()
        _check(load_library().lc_dist_domain_export(self.h, _dptr(f, torch.uint8), ctypes.byref(tau), _stream()),
               "lc_dist_domain_export", ok=(LC_OK,))
        return f, tau.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.lc_dist_destroy(self.h)
            self.h = None


def _handles(ranks):
    return (ctypes.c_void_p * len(ranks))(*[r.h.value for r in ranks])


def _ptrs(ts, ranks):
    return (ctypes.c_void_p * len(ts))(*[_dptr(t, torch.float64, r.n_local).value for t, r in zip(ts, ranks)])


def dist_connect_local(ranks):
    """Emulation: all ranks of the partition in this process (one device)."""
    _check(load_library().lc_dist_connect_local(_handles(ranks), len(ranks)), "lc_dist_connect_local", ok=(LC_OK,))


def dist_select_domain(ranks, b, x0, criterion=CRIT_RESIDUAL, threshold=THR_PAPER, param=1e-10, expand_rounds=0,
                       dilate_hops=0) -> int:
    """Alg. 4 / 5 on the partition (+ the masked extraction); returns the global K."""
    p = DomainParams(criterion, threshold, param, expand_rounds, dilate_hops)
    K = ctypes.c_int64()
    _check(load_library().lc_dist_select_domain(_handles(ranks), len(ranks), _ptrs(b, ranks), _ptrs(x0, ranks),
                                                ctypes.byref(p), _stream(), ctypes.byref(K)),
           "lc_dist_select_domain", ok=(LC_OK,))
    return K.value


def dist_solve_local(ranks, x, rel_tol=1e-10, max_iters=20000):
    p = _solver(PCG, rel_tol, max_iters, 30)
    info = SolveInfo()
    _check(load_library().lc_dist_solve_local(_handles(ranks), len(ranks), ctypes.byref(p), _ptrs(x, ranks),
                                              _stream(), ctypes.byref(info)), "lc_dist_solve_local")
    return _infos([info])[0]


def dist_solve_global(ranks, b, x, rel_tol=1e-10, max_iters=20000):
    p = _solver(PCG, rel_tol, max_iters, 30)
    info = SolveInfo()
    _check(load_library().lc_dist_solve_global(_handles(ranks), len(ranks), _ptrs(b, ranks), _ptrs(x, ranks),
                                               ctypes.byref(p), _stream(), ctypes.byref(info)), "lc_dist_solve_global")
    return _infos([info])[0]


def dist_local_method(ranks, b, x0, domain: dict | None, rel_tol=1e-10, max_iters=20000):
    """Alg. 1 on the partition: domain (Alg. 4/5) + masked extraction, local solve + assembly, global solve.
    b, x0: per-rank slab tensors.  Returns (x slabs, report)."""
    x = [t.clone() for t in x0]
    rep = {"K": 0}
    if domain is not None:
        rep["K"] = dist_select_domain(ranks, b, x0, **domain)
        rep["local"] = dist_solve_local(ranks, x, rel_tol, max_iters)
    rep["global"] = dist_solve_global(ranks, b, x, rel_tol, max_iters)
    return x, rep
