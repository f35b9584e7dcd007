"""Host-side batch packing: molecules -> the flat arrays of `dftb_batch_in`.

Everything here is vectorised over the batch with per-element caches, because at
10^3+ molecules/s per GPU the host setup is on the critical path (SURVEY.md
§8(f) #2).  The per-element work (fused-shell normalisation, atom-centred grid
templates) is computed once per (element, grid level) and reused.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from .basis import BasisSet, fused_element
from .errors import BasisError, MoleculeError, ResourceLimitError
from .grids import atom_template
from .molio import Molecule, electron_count

NMAX = 96  # DFTB_NMAX in include/qm1b_b200.h


@dataclass
class PackedBatch:
    n_mol: int
    n_atom: int
    n_shell: int
    mol_natom: np.ndarray
    mol_nshell: np.ndarray
    mol_nocc: np.ndarray
    mol_nao: np.ndarray
    atom_z: np.ndarray
    atom_xyz: np.ndarray
    shell_kind: np.ndarray
    shell_atom: np.ndarray
    shell_ao: np.ndarray
    shell_exp: np.ndarray
    shell_cs: np.ndarray
    shell_cp: np.ndarray
    tmpl_xyzw: np.ndarray
    atom_tmpl0: np.ndarray
    atom_tmpln: np.ndarray
    mol_npts: np.ndarray


class _TemplateCache:
    """Concatenated atom-centred grid templates for the (Z, level) keys seen so far.

    Shared by the labeling pipeline's worker threads (one plan per thread): a key's
    (offset, count) and the chunk it points to are published together under the lock, and
    array() returns a snapshot that contains every template whose key a caller already got
    (templates are only ever appended)."""

    def __init__(self):
        self.index: dict[tuple[int, int], tuple[int, int]] = {}
        self.chunks: list[np.ndarray] = []
        self.total = 0
        self._cat: np.ndarray | None = None
        self._lock = threading.Lock()

    def get(self, z: int, level: int) -> tuple[int, int]:
        key = (z, level)
        hit = self.index.get(key)
        if hit is not None:
            return hit
        t = atom_template(z, level)          # outside the lock: pure function of (z, level)
        with self._lock:
            if key not in self.index:
                self.chunks.append(t)
                self.index[key] = (self.total, len(t))
                self.total += len(t)
                self._cat = None
            return self.index[key]

    def array(self) -> np.ndarray:
        with self._lock:
            if self._cat is None:
                self._cat = (np.ascontiguousarray(np.concatenate(self.chunks))
                             if self.chunks else np.zeros((0, 4)))
            return self._cat


_TEMPLATES = _TemplateCache()


class _ElementTable:
    """Per-basis lookup tables indexed by Z (fused shells), built once."""

    def __init__(self, basis: BasisSet):
        zs = sorted(basis.shells)
        self.zmax = max(zs)
        self.nsh = np.zeros(self.zmax + 1, np.int64)
        self.nao = np.zeros(self.zmax + 1, np.int64)
        self.sh0 = np.zeros(self.zmax + 1, np.int64)
        self.ok = np.zeros(self.zmax + 1, bool)
        kinds, exps, cs, cp, sao = [], [], [], [], []
        for z in zs:
            try:
                el = fused_element(basis, z)
            except BasisError:
                continue
            self.ok[z] = True
            self.sh0[z] = len(kinds)
            self.nsh[z] = len(el.kinds)
            self.nao[z] = el.n_ao
            off = 0
            for k in el.kinds:
                sao.append(off)
                off += 4 if k else 1
            kinds.extend(el.kinds)
            exps.append(el.exps)
            cs.append(el.cs)
            cp.append(el.cp)
        self.kind = np.asarray(kinds, np.int32)
        self.sao = np.asarray(sao, np.int64)        # AO offset of the shell within its atom
        self.exp = np.vstack(exps)
        self.cs = np.vstack(cs)
        self.cp = np.vstack(cp)


_TABLES: dict[int, _ElementTable] = {}


def _table(basis: BasisSet) -> _ElementTable:
    t = _TABLES.get(id(basis))
    if t is None or t.basis_ref is not basis:
        t = _ElementTable(basis)
        t.basis_ref = basis
        _TABLES[id(basis)] = t
    return t


def _segment_exclusive_cumsum(vals: np.ndarray, seg_len: np.ndarray) -> np.ndarray:
    """Exclusive cumsum of vals restarting at every segment boundary."""
    cs = np.cumsum(vals) - vals
    starts = np.repeat(np.cumsum(seg_len) - seg_len, seg_len)
    return cs - cs[starts] if len(vals) else cs


def pack(mols: list[Molecule], basis: BasisSet, grid_level: int | None,
         max_n_ao: int = 128) -> PackedBatch:
    """Validate and pack a batch (vectorised over atoms and shells).  Raises the reference's
    error classes: MoleculeError (electron count / basis too small), BasisError,
    ResourceLimitError."""
    n_mol = len(mols)
    tab = _table(basis)
    natom = np.fromiter((m.n_atoms for m in mols), np.int64, n_mol)
    z_all = np.fromiter((z for m in mols for z in m.atomic_numbers), np.int64, int(natom.sum()))
    charge = np.fromiter((m.charge for m in mols), np.int64, n_mol)
    xyz = np.concatenate([m.positions for m in mols]) if n_mol else np.zeros((0, 3))
    if len(z_all) and (z_all.max() > tab.zmax or not tab.ok[z_all].all()):
        bad = sorted({int(z) for z in z_all if z > tab.zmax or not tab.ok[z]})
        missing = [z for z in bad if z not in basis.shells]
        if missing:
            raise BasisError(f"basis {basis.name!r} missing element(s) Z={missing}")
        fused_element(basis, bad[0])  # raises the specific BasisError
    mol_of_atom = np.repeat(np.arange(n_mol), natom)
    nelec = np.bincount(mol_of_atom, weights=z_all, minlength=n_mol).astype(np.int64) - charge
    for im in np.nonzero((nelec <= 0) | (nelec % 2 != 0))[0]:
        raise MoleculeError(f"electron count {int(nelec[im])}: restricted-closed-shell violation")
    nao = np.bincount(mol_of_atom, weights=tab.nao[z_all], minlength=n_mol).astype(np.int64)
    nocc = nelec // 2
    for im in np.nonzero(nocc > nao)[0]:
        raise MoleculeError(f"{int(nelec[im])} electrons need {int(nocc[im])} orbitals but basis has {int(nao[im])}")
    for im in np.nonzero(nao > max_n_ao)[0]:
        raise ResourceLimitError(f"N={int(nao[im])} exceeds configured maximum {max_n_ao}")
    for im in np.nonzero(nao > NMAX)[0]:
        raise ResourceLimitError(f"N={int(nao[im])} exceeds the device path maximum {NMAX}")
    # shells: atom-major, element shell order
    nsh_atom = tab.nsh[z_all]
    atom_of_shell = np.repeat(np.arange(len(z_all)), nsh_atom)
    local_sh = _segment_exclusive_cumsum(np.ones(len(atom_of_shell), np.int64), nsh_atom)
    esh = tab.sh0[z_all[atom_of_shell]] + local_sh
    atom0 = np.cumsum(natom) - natom
    # AO offset of each atom within its molecule, then of each shell
    ao_atom = _segment_exclusive_cumsum(tab.nao[z_all], natom)
    shell_ao = ao_atom[atom_of_shell] + tab.sao[esh]
    shell_atom = atom_of_shell - atom0[mol_of_atom[atom_of_shell]]
    nsh_mol = np.bincount(mol_of_atom, weights=nsh_atom, minlength=n_mol).astype(np.int64)
    t0 = np.zeros(len(z_all), np.int32)
    tn = np.zeros(len(z_all), np.int32)
    npts = np.zeros(n_mol, np.int64)
    if grid_level is not None:
        uz = np.unique(z_all)
        lut0 = np.zeros(tab.zmax + 1, np.int32)
        lutn = np.zeros(tab.zmax + 1, np.int32)
        for z in uz:
            lut0[z], lutn[z] = _TEMPLATES.get(int(z), grid_level)
        t0, tn = lut0[z_all], lutn[z_all]
        npts = np.bincount(mol_of_atom, weights=tn, minlength=n_mol).astype(np.int64)
        tmpl = _TEMPLATES.array()
    else:
        tmpl = np.zeros((0, 4))
    return PackedBatch(
        n_mol=n_mol, n_atom=int(len(z_all)), n_shell=int(len(esh)),
        mol_natom=natom.astype(np.int32), mol_nshell=nsh_mol.astype(np.int32),
        mol_nocc=nocc.astype(np.int32), mol_nao=nao.astype(np.int32),
        atom_z=z_all.astype(np.int32), atom_xyz=np.ascontiguousarray(xyz, np.float64),
        shell_kind=np.ascontiguousarray(tab.kind[esh]), shell_atom=shell_atom.astype(np.int32),
        shell_ao=shell_ao.astype(np.int32),
        shell_exp=np.ascontiguousarray(tab.exp[esh]), shell_cs=np.ascontiguousarray(tab.cs[esh]),
        shell_cp=np.ascontiguousarray(tab.cp[esh]),
        tmpl_xyzw=np.ascontiguousarray(tmpl, np.float64), atom_tmpl0=np.asarray(t0, np.int32),
        atom_tmpln=np.asarray(tn, np.int32), mol_npts=npts)


def check_basis_supported(basis: BasisSet, zs) -> None:
    for z in set(zs):
        try:
            fused_element(basis, z)
        except BasisError:
            raise


def check(mols: list[Molecule], basis: BasisSet, max_n_ao: int = 128) -> list:
    """Per-molecule validation with pack()'s rules and error classes: returns, for each
    molecule, None or the exception pack() would raise for it alone.  Lets a caller drop
    bad entries from a batch instead of failing the whole batch (pipeline.run)."""
    tab = _table(basis)
    out = []
    for m in mols:
        try:
            zs = np.asarray(m.atomic_numbers, np.int64)
            if zs.max() > tab.zmax or not tab.ok[zs].all():
                bad = sorted({int(z) for z in zs if z > tab.zmax or not tab.ok[z]})
                missing = [z for z in bad if z not in basis.shells]
                if missing:
                    raise BasisError(f"basis {basis.name!r} missing element(s) Z={missing}")
                fused_element(basis, bad[0])
            nelec = int(zs.sum()) - int(m.charge)
            if nelec <= 0 or nelec % 2:
                raise MoleculeError(f"electron count {nelec}: restricted-closed-shell violation")
            nao = int(tab.nao[zs].sum())
            if nelec // 2 > nao:
                raise MoleculeError(f"{nelec} electrons need {nelec // 2} orbitals but basis has {nao}")
            if nao > max_n_ao:
                raise ResourceLimitError(f"N={nao} exceeds configured maximum {max_n_ao}")
            if nao > NMAX:
                raise ResourceLimitError(f"N={nao} exceeds the device path maximum {NMAX}")
            out.append(None)
        except (BasisError, MoleculeError, ResourceLimitError) as exc:
            out.append(exc)
    return out
