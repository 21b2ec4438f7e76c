import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def read_golden(name):
    """key = values fixture under tests/golden (comments start with #)."""
    out = {}
    with open(os.path.join(ROOT, "tests", "golden", name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            k, v = line.split("=", 1)
            out[k.strip()] = v.split()
    return out


@pytest.fixture
def tune():
    """tune(**fields): set lc_tuning fields for this test (include/lc.h; accumulates); defaults restored after."""
    from paper_2001_01158_b200 import lc

    def set_(**fields):
        cur = lc.get_tuning()
        cur.update(fields)
        lc.set_tuning(**cur)
    yield set_
    lc.set_tuning()


def pytest_terminal_summary(terminalreporter):
    """Near-threshold / cascaded index-set differences counted by the parity tests (BASELINE north_star: cells
    whose criterion lies within 1e-12 relative of tau are counted and reported)."""
    mod = sys.modules.get("test_gpu_parity") or sys.modules.get("tests.test_gpu_parity")
    log = getattr(mod, "NEAR_LOG", None)
    if log is None:
        return
    tr = terminalreporter
    tr.write_sep("-", f"index-set parity: {len(log)} segment(s) with near-threshold / cascaded differences")
    for r in log:
        tr.write_line(str(r))
