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


STRUCTS = {"lc_domain_params": "DomainParams", "lc_solver_params": "SolverParams", "lc_solve_info": "SolveInfo",
           "lc_heat_params": "HeatParams", "lc_heat_report": "HeatReport", "lc_tuning": "Tuning"}


def test_struct_layouts_match_header(tmp_path):
    """Every struct of include/lc.h has the binding's size and field offsets: a C program compiled against the
    header prints sizeof / offsetof, compared with the ctypes layouts."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc missing")
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "lc.h"', 'int main(void) {']
    for cname, pyname in STRUCTS.items():
        st = getattr(lc, pyname)
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in st._fields_:
            lines.append(f'  printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ['  return 0;', '}']
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = {}
    for line in subprocess.check_output([str(exe)], text=True).splitlines():
        c, f, v = line.split()
        got[(c, f)] = int(v)
    for cname, pyname in STRUCTS.items():
        st = getattr(lc, pyname)
        assert got[(cname, "size")] == ctypes.sizeof(st), cname
        for f, _ in st._fields_:
            assert got[(cname, f)] == getattr(st, f).offset, (cname, f)


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


def test_tuning_host_only_roundtrip(lib):
    """lc_tuning lives on the host (no device needed): defaults, range checks, thread-local set / get."""
    import threading
    d = lc.tuning_defaults()
    assert d == dict(stencil_layout=1, symmetric_layout=0, pcg_cluster_resident=2, pcg_cluster=1, pcg_tma=1,
                     lazy_x_depth=3, batched_schedule=-1, pcg_max_ctas=0, sub_repr=-1, gmres_exact_cgs2=0,
                     gs_lines=1, spmv_csr_tma=1, spmv_tma=1, batched_cluster=0, block_dcoup=1, l2_stream_hint=-1)
    assert lc.get_tuning() == d
    prev = lc.set_tuning(lazy_x_depth=2, batched_schedule=1)
    try:
        assert lc.get_tuning()["lazy_x_depth"] == 2 and lc.get_tuning()["batched_schedule"] == 1
        seen = {}
        th = threading.Thread(target=lambda: seen.update(lc.get_tuning()))
        th.start(); th.join()
        assert seen == d                                   # other threads keep the defaults
        for bad in (dict(lazy_x_depth=4), dict(batched_schedule=3), dict(stencil_layout=2), dict(sub_repr=-2),
                    dict(pcg_max_ctas=-1), dict(l2_stream_hint=2)):
            with pytest.raises(lc.LcError):
                lc.set_tuning(**bad)
    finally:
        lc.set_tuning(**prev)
    assert lc.get_tuning() == d


def test_library_reads_no_environment():
    """No getenv in the product library (every implementation choice is an explicit lc_tuning field)."""
    import glob
    for f in glob.glob(os.path.join(ROOT, "paper_2001_01158_b200", "csrc", "*")):
        assert "getenv" not in open(f).read(), f
