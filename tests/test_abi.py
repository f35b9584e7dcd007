"""The C ABI library loads and exports every function include/qm1b_b200.h declares (no GPU needed)."""
import ctypes
import os
import re

from paper_2311_01135_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "qm1b_b200.h")).read()
    return set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(dftb_\w+)\s*\(", text, re.M))


def test_header_symbols_exported():
    assert os.path.exists(_lib.LIB_PATH), "build with `python __graft_entry__.py`"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = _declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert set(_lib.SIGNATURES) == names


def test_load_without_device_reports_cleanly():
    lib = _lib.load(require_device=False)
    assert lib.dftb_version().decode().startswith("qm1b_b200")
    # no compute is attempted here; on a CPU-only box the device query must fail loudly
    n = ctypes.c_int32(0)
    rc = lib.dftb_device_count(ctypes.byref(n))
    assert rc == 0 or lib.dftb_last_error()
