"""Integral operators — drop-in for deskdft.integrals (integrals.py:27-291).

`one_electron`, `eri_packed` and `build_jk` run on the GPU:
  * one_electron  -> k_onee (S, T, V per fused shell pair);
  * eri_packed    -> k_schwarz + class-specialised k_eri into the dense 8-fold store,
                     then k_compact applies the reference's three screens (split-shell
                     pair bound, AO-level bound, |v| >= eps) and emits the canonical
                     list in composite order;
  * build_jk      -> the packed list is scattered into the dense (ket-tiled) store and
                     digested by the tile J/K kernel (deterministic, no atomics).
Values are computed without the reference's primitive-pair screen, i.e. they equal
the exact (screen_eps = 0) integrals; the *selection* follows eps exactly.
Dense unpacking and the binary dump formats are host-side formatting, as in the
reference.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .basis import AOBasis, BasisSet
from .engine import EngineOptions, Plan
from .errors import DimensionError, ResourceLimitError
from .linalg import bare_batch
from .molio import Molecule

DEFAULT_SCREEN_EPS = 1e-12
DEFAULT_MAX_N_AO = 128
DEFAULT_BUDGET_BYTES = 4 << 30


@dataclass(frozen=True)
class IntegralSet:
    S: np.ndarray
    T: np.ndarray
    V: np.ndarray
    n_ao: int

    def __post_init__(self):
        for name in ("S", "T", "V"):
            m = getattr(self, name)
            if m.shape != (self.n_ao, self.n_ao):
                raise DimensionError(f"{name} has shape {m.shape}, expected ({self.n_ao}, {self.n_ao})")


@dataclass(frozen=True)
class PackedERI:
    i: np.ndarray
    j: np.ndarray
    k: np.ndarray
    l: np.ndarray
    values: np.ndarray
    degeneracy: np.ndarray
    n_ao: int
    screen_eps: float

    @property
    def quads(self) -> np.ndarray:
        return np.stack([self.i, self.j, self.k, self.l], axis=1)

    @property
    def n_entries(self) -> int:
        return int(self.values.shape[0])

    def nbytes(self) -> int:
        return self.i.nbytes * 4 + self.values.nbytes + self.degeneracy.nbytes


def molecule_from_ao(ao: AOBasis) -> tuple[Molecule, BasisSet]:
    """Rebuild (Molecule, BasisSet) from an AOBasis: atoms from the shell centres, the
    element basis from the shells placed on the first atom of each element."""
    natom = max(ia for ia, _ in ao.shells) + 1
    Z = [0] * natom
    pos = np.zeros((natom, 3))
    per_el: dict[int, list] = {}
    first_atom: dict[int, int] = {}
    for s, (ia, sh) in enumerate(ao.shells):
        Z[ia] = sh.element
        pos[ia] = ao.shell_center[s]
        if sh.element not in first_atom:
            first_atom[sh.element] = ia
        if first_atom[sh.element] == ia:
            per_el.setdefault(sh.element, []).append(sh)
    b = BasisSet(name="from-aobasis", shells={z: tuple(v) for z, v in per_el.items()})
    return Molecule(tuple(Z), pos), b


def _plan(ao: AOBasis, m: Molecule | None = None) -> Plan:
    mol, b = molecule_from_ao(ao)
    if m is not None:
        mol = m
    return Plan([mol], b, EngineOptions(grid_level=None, max_iterations=1))


def one_electron(ao: AOBasis, m: Molecule, dtype=np.float64) -> IntegralSet:
    """S, T, V on the device (integrals.py:115-132)."""
    with _plan(ao, m) as p:
        _lib.check(p.lib.dftb_plan_one_electron(p.h, p.stream))
        S, T, V = p.get("S"), p.get("T"), p.get("V")
    dtype = np.dtype(dtype)
    return IntegralSet(S=S.astype(dtype), T=T.astype(dtype), V=V.astype(dtype), n_ao=ao.n_ao)


def _split_pair_bounds(ao: AOBasis, qao: np.ndarray) -> np.ndarray:
    """Per AO pair, the reference's split-shell pair bound q_pair = max sqrt((ab|ab)) over
    the split-shell pair block containing it (integrals.py:99-112, _kernels.py:450-488)."""
    n = ao.n_ao
    shell_of = np.empty(n, np.int64)
    for s in range(ao.n_shells):
        nc = (int(ao.shell_l[s]) + 1) * (int(ao.shell_l[s]) + 2) // 2
        shell_of[ao.ao_offsets[s]:ao.ao_offsets[s] + nc] = s
    i, j = np.tril_indices(n)
    P = i * (i + 1) // 2 + j
    si, sj = shell_of[i], shell_of[j]
    a, b = np.maximum(si, sj), np.minimum(si, sj)
    key = a * (a + 1) // 2 + b
    qpair = np.zeros(ao.n_shells * (ao.n_shells + 1) // 2)
    np.maximum.at(qpair, key, qao[P])
    out = np.empty(len(P))
    out[P] = qpair[key]
    return out


def eri_packed(ao: AOBasis, screen_eps: float = DEFAULT_SCREEN_EPS, dtype=np.float64,
               max_n_ao: int = DEFAULT_MAX_N_AO, budget_bytes: int = DEFAULT_BUDGET_BYTES,
               _pairs=None) -> PackedERI:
    """Canonical quadruples with Schwarz screening at screen_eps (integrals.py:135-196)."""
    if ao.n_ao > max_n_ao:
        raise ResourceLimitError(f"N={ao.n_ao} exceeds configured maximum {max_n_ao}")
    dtype = np.dtype(dtype)
    with _plan(ao) as p:
        _lib.check(p.lib.dftb_plan_eri(p.h, 0, p.stream))
        qao = p.get("qao")
        qsp = np.ascontiguousarray(_split_pair_bounds(ao, qao))
        cnt = ctypes.c_int64(0)
        _lib.check(p.lib.dftb_plan_eri_compact(p.h, 0, float(screen_eps), _lib.ptr(qsp), ctypes.byref(cnt),
                                               None, None, None, None, None, p.stream))
        total = int(cnt.value)
        entry_bytes = 4 * 2 + dtype.itemsize + 1
        if total * entry_bytes > budget_bytes:
            raise ResourceLimitError(f"packed ERI would need {total * entry_bytes / 1e6:.0f} MB "
                                     f"(> budget {budget_bytes / 1e6:.0f} MB)")
        i, j, k, l = (np.empty(total, np.uint16) for _ in range(4))
        v = np.empty(total)
        if total:
            _lib.check(p.lib.dftb_plan_eri_compact(p.h, 0, float(screen_eps), _lib.ptr(qsp), ctypes.byref(cnt),
                                                   _lib.vptr(i), _lib.vptr(j), _lib.vptr(k), _lib.vptr(l),
                                                   _lib.vptr(v), p.stream))
    deg = (np.where(i != j, 2, 1) * np.where(k != l, 2, 1) * np.where((i != k) | (j != l), 2, 1)).astype(np.uint8)
    return PackedERI(i=i, j=j, k=k, l=l, values=v.astype(dtype), degeneracy=deg, n_ao=ao.n_ao,
                     screen_eps=float(screen_eps))


def build_jk(eri: PackedERI, rho: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """J and K (with -1/2) from a packed tensor, on the device (integrals.py:199-218)."""
    n = eri.n_ao
    if rho.shape != (n, n):
        raise DimensionError(f"rho shape {rho.shape} does not match n_ao={n}")
    if n > _lib.NMAX:
        raise ResourceLimitError(f"N={n} exceeds the device path maximum {_lib.NMAX}")
    prec = "f32" if eri.values.dtype == np.float32 else "f64"
    with Plan(bare_batch(n), None, EngineOptions(precision=prec, grid_level=None, max_iterations=1)) as p:
        ii, jj, kk, ll = (np.ascontiguousarray(x, np.uint16) for x in (eri.i, eri.j, eri.k, eri.l))
        vv = np.ascontiguousarray(eri.values, np.float64)
        _lib.check(p.lib.dftb_plan_eri_load(p.h, 0, eri.n_entries, _lib.vptr(ii), _lib.vptr(jj), _lib.vptr(kk),
                                            _lib.vptr(ll), _lib.vptr(vv), p.stream))
        r = np.ascontiguousarray(rho, np.float64)
        J = np.empty((n, n))
        K = np.empty((n, n))
        _lib.check(p.lib.dftb_plan_jk(p.h, _lib.ptr(r), _lib.ptr(J), _lib.ptr(K), p.stream))
    return J.astype(rho.dtype), K.astype(rho.dtype)


def unpack_eri(eri: PackedERI) -> np.ndarray:
    """Dense N^4 tensor with all 8 images (host formatting, integrals.py:221-238)."""
    n = eri.n_ao
    d = np.zeros((n, n, n, n))
    i, j, k, l = (x.astype(np.intp) for x in (eri.i, eri.j, eri.k, eri.l))
    v = eri.values.astype(np.float64)
    for a, b, c, e in ((i, j, k, l), (j, i, k, l), (i, j, l, k), (j, i, l, k),
                       (k, l, i, j), (l, k, i, j), (k, l, j, i), (l, k, j, i)):
        d[a, b, c, e] = v
    return d


def dense_eri(ao: AOBasis, max_n_ao: int = 32) -> np.ndarray:
    if ao.n_ao > max_n_ao:
        raise ResourceLimitError(f"dense_eri limited to N <= {max_n_ao}, got {ao.n_ao}")
    return unpack_eri(eri_packed(ao, screen_eps=0.0))


_DUMP_MAGIC = 0x45524931
_SET_MAGIC = 0x53545631


def dump_packed(eri: PackedERI, path: str) -> None:
    """Same little-endian layout as the reference (integrals.py:252-260)."""
    with open(path, "wb") as fh:
        fh.write(struct.pack("<IIQB", _DUMP_MAGIC, eri.n_ao, eri.n_entries, eri.values.dtype.itemsize))
        fh.write(np.ascontiguousarray(eri.quads.astype("<u2")).tobytes())
        fh.write(np.ascontiguousarray(eri.values.astype(f"<f{eri.values.dtype.itemsize}")).tobytes())


def load_packed(path: str) -> PackedERI:
    with open(path, "rb") as fh:
        magic, n_ao, count, itemsize = struct.unpack("<IIQB", fh.read(17))
        if magic != _DUMP_MAGIC:
            raise ValueError(f"{path}: not a packed-ERI dump")
        q = np.frombuffer(fh.read(count * 8), dtype="<u2").reshape(count, 4)
        v = np.frombuffer(fh.read(count * itemsize), dtype=f"<f{itemsize}")
    i, j, k, l = (np.ascontiguousarray(q[:, c]) for c in range(4))
    deg = np.where(i != j, 2, 1) * np.where(k != l, 2, 1) * np.where((i != k) | (j != l), 2, 1)
    return PackedERI(i=i, j=j, k=k, l=l, values=v.copy(), degeneracy=deg.astype(np.uint8),
                     n_ao=int(n_ao), screen_eps=float("nan"))


def dump_integral_set(ints: IntegralSet, path: str) -> None:
    with open(path, "wb") as fh:
        fh.write(struct.pack("<II", _SET_MAGIC, ints.n_ao))
        for mat in (ints.S, ints.T, ints.V):
            fh.write(np.ascontiguousarray(mat, dtype="<f8").tobytes())


def load_integral_set(path: str) -> IntegralSet:
    with open(path, "rb") as fh:
        magic, n = struct.unpack("<II", fh.read(8))
        if magic != _SET_MAGIC:
            raise ValueError(f"{path}: not an integral-set dump")
        mats = [np.frombuffer(fh.read(8 * n * n), dtype="<f8").reshape(n, n).copy() for _ in range(3)]
    return IntegralSet(S=mats[0], T=mats[1], V=mats[2], n_ao=int(n))
