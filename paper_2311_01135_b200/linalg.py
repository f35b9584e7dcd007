"""Device mirrors of the reference's small dense linear algebra on arbitrary inputs.

`roothaan_device(F, S)` mirrors deskdft.scf.solve_roothaan (scf.py:86-98) for any
symmetric F and SPD S: a one-molecule plan with N single-AO shells is created only
to size the device buffers, S is loaded, and the device orthogonaliser (parallel
Jacobi, s > 1e-7 kept) plus the device eigensolver produce C and epsilon.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .batch import PackedBatch
from .engine import EngineOptions, Plan
from .errors import DeskDFTError, DimensionError


def bare_batch(n_ao: int, n_occ: int = 0) -> PackedBatch:
    """A single 'molecule' of n_ao S shells (geometry irrelevant) for operator-level calls."""
    if not 1 <= n_ao <= _lib.NMAX:
        raise DimensionError(f"n_ao={n_ao} outside the device range 1..{_lib.NMAX}")
    z = np.zeros(n_ao, np.int32)
    e = np.tile(np.array([3.0, 1.0, 0.3]), (n_ao, 1))
    c = np.tile(np.array([0.1, 0.5, 0.5]), (n_ao, 1))
    return PackedBatch(
        n_mol=1, n_atom=1, n_shell=n_ao, mol_natom=np.array([1], np.int32),
        mol_nshell=np.array([n_ao], np.int32), mol_nocc=np.array([n_occ], np.int32),
        mol_nao=np.array([n_ao], np.int32), atom_z=np.array([1], np.int32),
        atom_xyz=np.zeros((1, 3)), shell_kind=z.copy(), shell_atom=z.copy(),
        shell_ao=np.arange(n_ao, dtype=np.int32), shell_exp=e, shell_cs=c, shell_cp=np.zeros_like(c),
        tmpl_xyzw=np.zeros((0, 4)), atom_tmpl0=np.zeros(1, np.int32), atom_tmpln=np.zeros(1, np.int32),
        mol_npts=np.zeros(1, np.int64))


def roothaan_device(F: np.ndarray, S: np.ndarray, n_occ: int = 0):
    from .scf import OrbitalSolution

    F = np.asarray(F)
    S = np.asarray(S)
    n = S.shape[0]
    if S.shape != (n, n) or F.shape != (n, n):
        raise DimensionError(f"F {F.shape} / S {S.shape} must be square and equal")
    dtype = F.dtype if F.dtype in (np.float32, np.float64) else np.float64
    with Plan(bare_batch(n, n_occ), None, EngineOptions(grid_level=None, max_iterations=1)) as p:
        lib = p.lib
        S64 = np.ascontiguousarray(S, np.float64)
        _lib.check(lib.dftb_plan_set(p.h, b"S", 0, _lib.ptr(S64), n * n, p.stream))
        F64 = np.ascontiguousarray(F, np.float64)
        C = np.empty((n, n))
        eps = np.empty(_lib.NMAX)
        nmo = np.zeros(1, np.int32)
        import ctypes
        _lib.check(lib.dftb_plan_roothaan(p.h, _lib.ptr(F64), _lib.ptr(C), _lib.ptr(eps),
                                          _lib.ptr(nmo, ctypes.c_int32), p.stream))
        status = int(p.fetch(want_C=False).status[0])
    m = int(nmo[0])
    if status & _lib.ST_OVERLAP_NOT_PD:
        raise DeskDFTError("overlap matrix not positive definite")
    if m == 0 or status & _lib.ST_SINGULAR:
        raise DeskDFTError("overlap matrix singular after linear-dependence drop")
    return OrbitalSolution(C=C[:, :m].astype(dtype), epsilon=eps[:m].astype(dtype), n_occ=n_occ)
