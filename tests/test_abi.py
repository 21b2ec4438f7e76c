"""CPU-side checks of the boundary: liblc.so loads without a GPU, exports every
entry point include/lc.h declares, and the binding's structs match the header."""
import ctypes
import os
import re

import pytest

from paper_2001_01158_b200 import build as lcbuild
from paper_2001_01158_b200 import lc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "lc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lc_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    lcbuild.build()
    return lc.load_library()


def test_header_declares_the_five_calls():
    fns = header_functions()
    for f in ("lc_create_csr", "lc_select_domain", "lc_extract_sub", "lc_solve_local", "lc_solve_global"):
        assert f in fns


def test_every_declared_symbol_is_exported(lib):
    for f in header_functions():
        assert hasattr(lib, f), f
    assert set(lc.EXPORTED) == set(header_functions())


def test_struct_layouts_match_header():
    # lc_domain_params: int32, int32, double, int32, int32 -> 24 bytes with natural alignment
    assert ctypes.sizeof(lc.DomainParams) == 24
    assert lc.DomainParams.param.offset == 8
    # lc_solver_params: int32 x3, double, int32 -> 32 bytes
    assert ctypes.sizeof(lc.SolverParams) == 32
    assert lc.SolverParams.rel_tol.offset == 16
    # lc_solve_info: int32, int32, double, double -> 24 bytes
    assert ctypes.sizeof(lc.SolveInfo) == 24


def test_no_cpu_fallback_without_device(lib):
    """Without a CUDA device the binding refuses to run (no silent CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        lc.Matrix(2, [0, 1, 2], [0, 1], [1.0, 1.0])


def test_invalid_args_rejected_before_device_work(lib):
    """Argument validation happens on the host side of the ABI (no GPU needed)."""
    h = ctypes.c_void_p()
    st = lib.lc_create_csr(4, 2, 1, None, None, None, 0, 0, None, ctypes.byref(h))
    assert st == -1 and h.value is None
    assert b"null" in lib.lc_last_error()
    st = lib.lc_select_domain(None, None, None, None, None, ctypes.byref(h), None)
    assert st == -1
    assert lib.lc_kernel_launches() == 0


def test_sass_is_sm100a():
    """The built library carries sm_100a SASS (cuobjdump), i.e. nvcc really targeted B200."""
    import shutil
    import subprocess
    lcbuild.build()
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump missing")
    out = subprocess.run([exe, "--list-elf", lc.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
