"""ctypes binding of libqm1b_b200.so (the C ABI in include/qm1b_b200.h).

The library is built in-tree (`python __graft_entry__.py` / `make -C
paper_2311_01135_b200/csrc`).  There is no CPU fallback: if the shared library
or a CUDA device is missing, every compute entry point raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import DeskDFTError, DeviceError, DimensionError, ResourceLimitError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqm1b_b200.so")
# Development override for same-box A/B timing of two builds (tools/); it must name a file
# inside this repository and is reported on stderr, so it cannot silently swap the product.
_DEV_LIB = os.environ.get("QM1B_B200_DEV_LIB")
if _DEV_LIB:
    _repo = os.path.dirname(_HERE)
    if not os.path.realpath(_DEV_LIB).startswith(os.path.realpath(_repo) + os.sep):
        raise RuntimeError(f"QM1B_B200_DEV_LIB={_DEV_LIB} is outside the repository")
    import sys as _sys

    print(f"[qm1b_b200] development library override: {_DEV_LIB}", file=_sys.stderr)
    LIB_PATH = _DEV_LIB
NMAX = 96

c_i32p = ctypes.POINTER(ctypes.c_int32)
c_f64p = ctypes.POINTER(ctypes.c_double)


class BatchIn(ctypes.Structure):
    _fields_ = [
        ("n_mol", ctypes.c_int32), ("n_atom", ctypes.c_int32), ("n_shell", ctypes.c_int32),
        ("mol_natom", c_i32p), ("mol_nshell", c_i32p), ("mol_nocc", c_i32p),
        ("atom_z", c_i32p), ("atom_xyz", c_f64p),
        ("shell_kind", c_i32p), ("shell_atom", c_i32p),
        ("shell_exp", c_f64p), ("shell_cs", c_f64p), ("shell_cp", c_f64p),
        ("n_tmpl", ctypes.c_int32), ("tmpl_xyzw", c_f64p),
        ("atom_tmpl0", c_i32p), ("atom_tmpln", c_i32p),
    ]


class Opts(ctypes.Structure):
    _fields_ = [
        ("precision", ctypes.c_int32), ("max_iterations", ctypes.c_int32),
        ("convergence_std", ctypes.c_double), ("diis_history", ctypes.c_int32),
        ("diis_start", ctypes.c_int32), ("damping_factor", ctypes.c_double),
        ("screen_eps", ctypes.c_double),
    ]


class Results(ctypes.Structure):
    _fields_ = [
        ("E_total", c_f64p), ("E_comp", c_f64p), ("history", c_f64p),
        ("iterations", c_i32p), ("converged", c_i32p), ("n_mo", c_i32p),
        ("epsilon", c_f64p), ("C", c_f64p), ("status", c_i32p),
    ]


class ResultsDev(ctypes.Structure):
    """dftb_results_dev: caller-owned DEVICE pointers (same layouts as Results)."""
    _fields_ = [(name, ctypes.c_void_p) for name, _ in Results._fields_]


ST_OVERLAP_NOT_PD, ST_NEG_WEIGHT, ST_XC_NONFINITE, ST_NO_ORBITALS, ST_SINGULAR = 1, 2, 4, 8, 16

_lib = None

# exported symbols (checked by tests/test_abi.py against include/qm1b_b200.h)
SIGNATURES = {
    "dftb_last_error": (ctypes.c_char_p, []),
    "dftb_version": (ctypes.c_char_p, []),
    "dftb_device_count": (ctypes.c_int, [c_i32p]),
    "dftb_scf_batch": (ctypes.c_int, [ctypes.POINTER(BatchIn), ctypes.POINTER(Opts), ctypes.POINTER(Results), ctypes.c_void_p]),
    "dftb_plan_create": (ctypes.c_int, [ctypes.POINTER(BatchIn), ctypes.POINTER(Opts), ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "dftb_plan_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "dftb_plan_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "dftb_plan_begin": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "dftb_plan_iterate": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]),
    "dftb_plan_fetch": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Results), ctypes.c_void_p]),
    "dftb_plan_fetch_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ResultsDev), ctypes.c_void_p]),
    "dftb_plan_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]),
    "dftb_plan_one_electron": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "dftb_plan_eri": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    "dftb_plan_grid": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "dftb_plan_jk": (ctypes.c_int, [ctypes.c_void_p, c_f64p, c_f64p, c_f64p, ctypes.c_void_p]),
    "dftb_plan_xc": (ctypes.c_int, [ctypes.c_void_p, c_f64p, c_f64p, c_f64p, ctypes.c_void_p]),
    "dftb_plan_eval_ao": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, c_f64p, c_f64p, ctypes.c_void_p]),
    "dftb_plan_roothaan": (ctypes.c_int, [ctypes.c_void_p, c_f64p, c_f64p, c_f64p, c_i32p, ctypes.c_void_p]),
    "dftb_plan_eri_compact": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_double, c_f64p,
                                             ctypes.POINTER(ctypes.c_int64)] + [ctypes.c_void_p] * 5 + [ctypes.c_void_p]),
    "dftb_plan_eri_load": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64] + [ctypes.c_void_p] * 5 + [ctypes.c_void_p]),
    "dftb_plan_load_grid": (ctypes.c_int, [ctypes.c_void_p, c_f64p, c_f64p, ctypes.c_int64, ctypes.c_void_p]),
    "dftb_plan_set": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int32, c_f64p, ctypes.c_int64, ctypes.c_void_p]),
    "dftb_plan_get": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int32, c_f64p, ctypes.c_int64, ctypes.c_void_p]),
    "dftb_b3lyp": (ctypes.c_int, [c_f64p, c_f64p, ctypes.c_int64, c_f64p, c_f64p, c_f64p, ctypes.c_void_p]),
    "dftb_diis": (ctypes.c_int, [c_f64p, c_f64p, ctypes.c_int32, ctypes.c_int32, c_f64p, ctypes.c_void_p]),
    "dftb_plan_stage_times": (ctypes.c_int, [ctypes.c_void_p, c_f64p, ctypes.c_int]),
    "dftb_plan_launch_count": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]),
    "dftb_plan_set_timing": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "dftb_plan_set_full_eig": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "dftb_fma_peak": (ctypes.c_int, [ctypes.c_int, c_f64p, ctypes.c_void_p]),
    "dftb_plan_kernel_times": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, c_f64p, c_f64p, ctypes.c_void_p]),
    "dftb_plan_post_time": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, c_f64p, ctypes.c_void_p]),
}


def load(require_device: bool = True):
    """Load the shared library (once).  Raises DeviceError when it is missing, or when
    `require_device` and no CUDA device is visible — never falls back to the CPU."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build` "
                              "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if _DEV_LIB and not hasattr(lib, name):
                continue   # an older build under A/B: entry points it lacks stay unbound
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_device:
        n = ctypes.c_int32(0)
        rc = _lib.dftb_device_count(ctypes.byref(n))
        if rc != 0 or n.value < 1:
            raise DeviceError("no CUDA device visible to libqm1b_b200 (there is no CPU fallback): "
                              + _lib.dftb_last_error().decode())
    return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = _lib.dftb_last_error().decode() if _lib is not None else "library not loaded"
    if rc == 1:
        raise DimensionError(msg) if "shape" in msg or "size" in msg else DeskDFTError(msg)
    if rc == 2:
        raise ResourceLimitError(msg)
    if rc == 4:
        raise DeskDFTError(msg)
    raise DeviceError(msg)


def ptr(a: np.ndarray, ctype=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def vptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def current_stream():
    """The current torch CUDA stream handle if torch is imported and CUDA is up, else NULL."""
    import sys

    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized():
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    return ctypes.c_void_p(0)
