"""Batch engine: one device plan per batch of molecules.

`Plan` owns a `dftb_plan` (C ABI): creation packs the molecules on the host
(batch.pack + native planning in plan.cu) and uploads them; `run()` enqueues the
whole SCF (setup kernels, core guess, every iteration) on one CUDA stream with no
host synchronisation; `fetch()` copies the per-molecule results back.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .batch import NMAX, PackedBatch, pack
from .basis import BasisSet
from .errors import DeskDFTError, DimensionError
from .molio import Molecule


@dataclass
class EngineOptions:
    precision: str = "f64"
    max_iterations: int = 50
    convergence_std: float = 0.01
    diis_history: int = 8
    diis_start: int = 3
    damping_factor: float = 0.5
    screen_eps: float = 1e-12
    grid_level: int | None = 1

    def c_struct(self) -> _lib.Opts:
        return _lib.Opts(1 if self.precision == "f32" else 0, int(self.max_iterations),
                         float(self.convergence_std), int(self.diis_history), int(self.diis_start),
                         float(self.damping_factor), float(self.screen_eps))


@dataclass
class BatchResults:
    E_total: np.ndarray
    E_comp: np.ndarray
    history: np.ndarray
    iterations: np.ndarray
    converged: np.ndarray
    n_mo: np.ndarray
    epsilon: np.ndarray
    C: list
    status: np.ndarray


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Plan:
    """A batch resident on the current CUDA device."""

    def __init__(self, mols: list[Molecule] | PackedBatch, basis: BasisSet | None,
                 opts: EngineOptions, stream=None):
        self.lib = _lib.load()
        self.opts = opts
        self.pk = mols if isinstance(mols, PackedBatch) else pack(mols, basis, opts.grid_level)
        self.stream = stream if stream is not None else _lib.current_stream()
        pk = self.pk
        self._keep = [_i32(pk.mol_natom), _i32(pk.mol_nshell), _i32(pk.mol_nocc), _i32(pk.atom_z),
                      _f64(pk.atom_xyz), _i32(pk.shell_kind), _i32(pk.shell_atom), _f64(pk.shell_exp),
                      _f64(pk.shell_cs), _f64(pk.shell_cp), _f64(pk.tmpl_xyzw), _i32(pk.atom_tmpl0),
                      _i32(pk.atom_tmpln)]
        k = self._keep
        P, D = _lib.c_i32p, _lib.c_f64p
        self.c_in = _lib.BatchIn(
            pk.n_mol, pk.n_atom, pk.n_shell,
            _lib.ptr(k[0], ctypes.c_int32), _lib.ptr(k[1], ctypes.c_int32), _lib.ptr(k[2], ctypes.c_int32),
            _lib.ptr(k[3], ctypes.c_int32), _lib.ptr(k[4]),
            _lib.ptr(k[5], ctypes.c_int32), _lib.ptr(k[6], ctypes.c_int32),
            _lib.ptr(k[7]), _lib.ptr(k[8]), _lib.ptr(k[9]),
            int(len(k[10])), _lib.ptr(k[10]), _lib.ptr(k[11], ctypes.c_int32), _lib.ptr(k[12], ctypes.c_int32))
        del P, D
        self.c_opts = opts.c_struct()
        h = ctypes.c_void_p()
        _lib.check(self.lib.dftb_plan_create(ctypes.byref(self.c_in), ctypes.byref(self.c_opts),
                                             self.stream, ctypes.byref(h)))
        self.h = h

    # -- lifecycle
    def close(self):
        if getattr(self, "h", None):
            self.lib.dftb_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- stages
    def run(self):
        _lib.check(self.lib.dftb_plan_run(self.h, self.stream))

    def begin(self):
        _lib.check(self.lib.dftb_plan_begin(self.h, self.stream))

    def iterate(self, it: int):
        _lib.check(self.lib.dftb_plan_iterate(self.h, int(it), self.stream))

    def kernel_times(self, reps: int = 5, xc: bool = True) -> tuple[float, float | None]:
        """(ms per J/K launch set, ms per XC launch set or None) re-run on the resident density."""
        jk, x = ctypes.c_double(0.0), ctypes.c_double(0.0)
        _lib.check(self.lib.dftb_plan_kernel_times(self.h, int(reps), ctypes.byref(jk),
                                                   ctypes.byref(x) if xc else None, self.stream))
        return jk.value, (x.value if xc else None)

    def post_time(self, reps: int = 5) -> float:
        """ms per launch of the post kernel re-run as a non-final iteration (dftb_plan_post_time;
        advances the SCF state - after fetch only)."""
        ms = ctypes.c_double(0.0)
        _lib.check(self.lib.dftb_plan_post_time(self.h, int(reps), ctypes.byref(ms), self.stream))
        return ms.value

    def eri(self, screened: bool = True):
        """Operator stage: pair tables, Schwarz bounds and the dense ERI store (dftb_plan_eri)."""
        _lib.check(self.lib.dftb_plan_eri(self.h, 1 if screened else 0, self.stream))

    def jk(self, rho: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """Operator stage: J, K of the whole batch for host densities (dftb_plan_jk)."""
        n = int(np.sum(np.asarray(self.pk.mol_nao, dtype=np.int64) ** 2))
        r = np.ascontiguousarray(rho, np.float64).reshape(-1)
        if r.size != n:
            raise DimensionError(f"rho has {r.size} elements, the batch needs {n}")
        J, K = np.empty(n), np.empty(n)
        _lib.check(self.lib.dftb_plan_jk(self.h, _lib.ptr(r), _lib.ptr(J), _lib.ptr(K), self.stream))
        return J, K

    def set_full_eig(self, on: bool = True):
        """Diagonalise every iteration (C available per iteration) instead of purifying."""
        _lib.check(self.lib.dftb_plan_set_full_eig(self.h, 1 if on else 0))

    def set_timing(self, on: bool = True):
        _lib.check(self.lib.dftb_plan_set_timing(self.h, 1 if on else 0))

    def stage_times(self) -> list[float]:
        ms = np.zeros(3)
        _lib.check(self.lib.dftb_plan_stage_times(self.h, _lib.ptr(ms), 3))
        return ms.tolist()

    def launch_count(self) -> int:
        c = ctypes.c_int64(0)
        _lib.check(self.lib.dftb_plan_launch_count(self.h, ctypes.byref(c)))
        return int(c.value)

    def info(self) -> dict:
        v = np.zeros(20, np.int64)
        _lib.check(self.lib.dftb_plan_info(self.h, v.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 20))
        keys = ["n_mol", "n_pair", "n_pts", "mem_bytes", "eri_bytes", "q_llll", "q_llls", "q_llss",
                "q_lsls", "q_lsss", "q_ssss", "n_jk_cta", "n_xc_cta", "nmax", "mat_elems", "launches",
                "h2d_bytes", "pairs_ll", "pairs_ls", "pairs_ss"]
        return dict(zip(keys, (int(x) for x in v)))

    def get(self, which: str, mol: int = 0) -> np.ndarray:
        n = int(self.pk.mol_nao[mol])
        sizes = {"qao": n * (n + 1) // 2, "points": 3 * int(self.pk.mol_npts[mol]),
                 "weights": int(self.pk.mol_npts[mol]), "enn": 1, "dbg": 16}
        npp = n * (n + 1) // 2
        sizes["eri"] = npp * (npp + 1) // 2
        cnt = sizes.get(which, n * n)
        out = np.empty(cnt)
        _lib.check(self.lib.dftb_plan_get(self.h, which.encode(), int(mol), _lib.ptr(out), cnt, self.stream))
        if which == "points":
            return out.reshape(-1, 3)
        if which == "dbg":
            return out.view(np.int64)
        if cnt == n * n and which not in sizes:
            return out.reshape(n, n)
        return out

    def fetch_device(self, out: dict):
        """Enqueue the results into caller-owned device tensors (torch, on this plan's device)
        on the plan's stream; no host synchronisation.  Keys: the dftb_results_dev members."""
        ptrs = {k: ctypes.c_void_p(int(v.data_ptr())) for k, v in out.items()}
        r = _lib.ResultsDev(**ptrs)
        _lib.check(self.lib.dftb_plan_fetch_device(self.h, ctypes.byref(r), self.stream))

    def fetch(self, want_C: bool = True) -> BatchResults:
        pk = self.pk
        nm, mi = pk.n_mol, int(self.opts.max_iterations)
        E = np.empty(nm)
        comp = np.empty((nm, 5))
        hist = np.empty((nm, mi))
        it = np.empty(nm, np.int32)
        conv = np.empty(nm, np.int32)
        nmo = np.empty(nm, np.int32)
        eps = np.empty((nm, NMAX))
        st = np.empty(nm, np.int32)
        nao = pk.mol_nao.astype(np.int64)
        Cflat = np.empty(int((nao * nao).sum())) if want_C else None
        r = _lib.Results(_lib.ptr(E), _lib.ptr(comp), _lib.ptr(hist), _lib.ptr(it, ctypes.c_int32),
                         _lib.ptr(conv, ctypes.c_int32), _lib.ptr(nmo, ctypes.c_int32), _lib.ptr(eps),
                         _lib.ptr(Cflat) if want_C else None, _lib.ptr(st, ctypes.c_int32))
        _lib.check(self.lib.dftb_plan_fetch(self.h, ctypes.byref(r), self.stream))
        Cs = []
        if want_C:
            off = 0
            for m in range(nm):
                n = int(nao[m])
                Cs.append(Cflat[off:off + n * n].reshape(n, n)[:, :nmo[m]])
                off += n * n
        return BatchResults(E, comp, hist, it, conv.astype(bool), nmo, eps, Cs, st)


def status_error(code: int) -> DeskDFTError | None:
    """Map a per-molecule status word to the reference's exception (None if clean)."""
    if code & _lib.ST_OVERLAP_NOT_PD:
        return DeskDFTError("overlap matrix not positive definite")
    if code & _lib.ST_SINGULAR:
        return DeskDFTError("overlap matrix singular after linear-dependence drop")
    if code & _lib.ST_NO_ORBITALS:
        return DimensionError("n_occ exceeds the orbital count (basis too small)")
    if code & _lib.ST_NEG_WEIGHT:
        return DeskDFTError("negative quadrature weight beyond numerical noise")
    if code & _lib.ST_XC_NONFINITE:
        return DeskDFTError("non-finite functional output (density underflow mishandled)")
    return None
