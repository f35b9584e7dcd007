"""Host-side batch packing: molecules -> the flat arrays of `dftb_batch_in`.

Everything here is vectorised over the batch with per-element caches, because at
10^3+ molecules/s per GPU the host setup is on the critical path (SURVEY.md
§8(f) #2).  The per-element work (fused-shell normalisation, atom-centred grid
templates) is computed once per (element, grid level) and reused.
"""

from __future__ import annotations

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
    """Concatenated atom-centred grid templates for the (Z, level) keys seen so far."""

    def __init__(self):
        self.index: dict[tuple[int, int], tuple[int, int]] = {}
        self.chunks: list[np.ndarray] = []
        self.total = 0
        self._cat: np.ndarray | None = None

    def get(self, z: int, level: int) -> tuple[int, int]:
        key = (z, level)
        if key not in self.index:
            t = atom_template(z, level)
            self.index[key] = (self.total, len(t))
            self.chunks.append(t)
            self.total += len(t)
            self._cat = None
        return self.index[key]

    def array(self) -> np.ndarray:
        if self._cat is None:
            self._cat = (np.ascontiguousarray(np.concatenate(self.chunks))
                         if self.chunks else np.zeros((0, 4)))
        return self._cat


_TEMPLATES = _TemplateCache()


def pack(mols: list[Molecule], basis: BasisSet, grid_level: int | None,
         max_n_ao: int = 128) -> PackedBatch:
    """Validate and pack a batch.  Raises the reference's error classes:
    MoleculeError (electron count / basis too small), BasisError, ResourceLimitError."""
    n_mol = len(mols)
    natom = np.fromiter((m.n_atoms for m in mols), np.int32, n_mol)
    z_all = np.fromiter((z for m in mols for z in m.atomic_numbers), np.int32, int(natom.sum()))
    xyz = (np.concatenate([m.positions for m in mols]) if n_mol else np.zeros((0, 3)))
    nocc = np.empty(n_mol, np.int32)
    nao = np.empty(n_mol, np.int32)
    nsh = np.empty(n_mol, np.int32)
    kinds, satom, sao, sexp, scs, scp = [], [], [], [], [], []
    for im, m in enumerate(mols):
        ne = electron_count(m)
        n = 0
        ns = 0
        for ia, z in enumerate(m.atomic_numbers):
            el = fused_element(basis, z)
            k = len(el.kinds)
            kinds.append(np.asarray(el.kinds, np.int32))
            satom.append(np.full(k, ia, np.int32))
            off = np.empty(k, np.int32)
            for s, kd in enumerate(el.kinds):
                off[s] = n
                n += 4 if kd else 1
            sao.append(off)
            sexp.append(el.exps)
            scs.append(el.cs)
            scp.append(el.cp)
            ns += k
        if ne // 2 > n:
            raise MoleculeError(f"{ne} electrons need {ne // 2} orbitals but basis has {n}")
        if n > max_n_ao:
            raise ResourceLimitError(f"N={n} exceeds configured maximum {max_n_ao}")
        if n > NMAX:
            raise ResourceLimitError(f"N={n} exceeds the device path maximum {NMAX}")
        nocc[im] = ne // 2
        nao[im] = n
        nsh[im] = ns
    cat = (lambda L, dt, shape: np.ascontiguousarray(np.concatenate(L).astype(dt))
           if L else np.zeros(shape, dt))
    t0 = np.zeros(len(z_all), np.int32)
    tn = np.zeros(len(z_all), np.int32)
    npts = np.zeros(n_mol, np.int64)
    if grid_level is not None:
        a = 0
        for im, m in enumerate(mols):
            for z in m.atomic_numbers:
                t0[a], tn[a] = _TEMPLATES.get(int(z), grid_level)
                npts[im] += tn[a]
                a += 1
        tmpl = _TEMPLATES.array()
    else:
        tmpl = np.zeros((0, 4))
    return PackedBatch(
        n_mol=n_mol, n_atom=int(len(z_all)), n_shell=int(nsh.sum()),
        mol_natom=natom, mol_nshell=nsh, mol_nocc=nocc, mol_nao=nao,
        atom_z=z_all, atom_xyz=np.ascontiguousarray(xyz, np.float64),
        shell_kind=cat(kinds, np.int32, (0,)), shell_atom=cat(satom, np.int32, (0,)),
        shell_ao=cat(sao, np.int32, (0,)),
        shell_exp=cat(sexp, np.float64, (0, 3)), shell_cs=cat(scs, np.float64, (0, 3)),
        shell_cp=cat(scp, np.float64, (0, 3)),
        tmpl_xyzw=np.ascontiguousarray(tmpl, np.float64), atom_tmpl0=t0, atom_tmpln=tn,
        mol_npts=npts)


def check_basis_supported(basis: BasisSet, zs) -> None:
    for z in set(zs):
        try:
            fused_element(basis, z)
        except BasisError:
            raise
