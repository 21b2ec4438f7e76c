"""Seeded synthetic inputs for the five BASELINE.json configs (shared by the
oracle tests, the CUDA parity tests and bench.py).

This module holds no arithmetic of the local character-based method: it only
builds A_s, b_s = A_s x*_s and x0_s = x*_{s-1}.
The heavy lifting is in ``synth.c`` (OpenMP C, built into ``libsynth.so``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsynth.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        lib.synth_dims.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P]
        lib.synth_dims.restype = ctypes.c_int
        lib.synth_system.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                     P, P, P, P, P, P]
        lib.synth_system.restype = ctypes.c_int
        lib.synth_random_nnz.argtypes = [ctypes.c_int, ctypes.c_int]
        lib.synth_random_nnz.restype = ctypes.c_int64
        lib.synth_random.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, P, P, P, P, P, P]
        lib.synth_random.restype = ctypes.c_int
        lib.synth_default_n.argtypes = [ctypes.c_int]
        lib.synth_default_systems.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


@dataclass
class System:
    """One linear system A x = b with warm start x0 and manufactured solution xs.

    ``block`` = 1: CSR with scalar rows.  ``block`` = 3: BSR, ``nrows`` block rows,
    ``val`` holds 9 f64 per block (row-major).  ``batch`` = G equal independent
    diagonal segments (config 3)."""
    config: int
    n: int
    s: int
    nrows: int
    block: int
    batch: int
    rp: np.ndarray   # int64[nrows+1]
    ci: np.ndarray   # int32[nnz]
    val: np.ndarray  # f64[nnz*block*block]
    b: np.ndarray
    x0: np.ndarray
    xs: np.ndarray

    @property
    def N(self) -> int:
        return self.nrows * self.block


def default_n(config: int) -> int:
    return _load().synth_default_n(config)


def default_systems(config: int) -> int:
    return _load().synth_default_systems(config)


def system(config: int, s: int, n: int | None = None, G: int = 20, seed_offset: int = 0) -> System:
    lib = _load()
    n = default_n(config) if n is None else n
    nrows = np.zeros(1, np.int64); nnz = np.zeros(1, np.int64); blk = np.zeros(1, np.int32)
    if lib.synth_dims(config, n, G, _p(nrows), _p(nnz), _p(blk)) != 0:
        raise ValueError(f"bad config {config} / n {n}")
    nr, nz, bs = int(nrows[0]), int(nnz[0]), int(blk[0])
    rp = np.empty(nr + 1, np.int64); ci = np.empty(nz, np.int32); val = np.empty(nz * bs * bs, np.float64)
    b = np.empty(nr * bs); x0 = np.empty(nr * bs); xs = np.empty(nr * bs)
    if lib.synth_system(config, n, G, s, seed_offset, _p(rp), _p(ci), _p(val), _p(b), _p(x0), _p(xs)) != 0:
        raise RuntimeError("synth_system failed")
    return System(config, n, s, nr, bs, G if config == 3 else 1, rp, ci, val, b, x0, xs)


def random_system(n: int, bw: int = 2, spd: bool = True, seed: int = 1) -> System:
    """Row-diagonally-dominant (margin 1) banded system for oracle self-tests."""
    lib = _load()
    nz = lib.synth_random_nnz(n, bw)
    rp = np.empty(n + 1, np.int64); ci = np.empty(nz, np.int32); val = np.empty(nz)
    b = np.empty(n); x0 = np.empty(n); xs = np.empty(n)
    lib.synth_random(n, bw, 1 if spd else 0, seed, _p(rp), _p(ci), _p(val), _p(b), _p(x0), _p(xs))
    return System(0, n, 0, n, 1, 1, rp, ci, val, b, x0, xs)


def heat_initial(nx: int, ny: int, Tl: float = 1.0, Tr: float = 1e-4) -> np.ndarray:
    """The paper's heat-model initial field T_0(x, y) = e^{-100 x} T_l + T_r at the interior nodes
    x_p = (p+1)/(nx+1), row i = p + nx q (an input of Alg. 6, shared by the oracle and the device driver)."""
    x = (np.arange(nx) + 1.0) / (nx + 1)
    return np.tile(np.exp(-100.0 * x) * Tl + Tr, ny)
