"""SCF driver API — the drop-in for deskdft.scf (scf.py:28-222).

`scf(m, b, opts, iteration_callback)` and `properties(r)` keep the reference's
signatures, dataclasses, option validation and error classes.  Underneath, every
molecule runs on the GPU: `scf` is `scf_batch([m])`, and `scf_batch` runs a whole
batch through one device plan with no host round trip inside the SCF loop (the
only host synchronisation is at the end, or one tiny flag read every 4
iterations when `convergence_std > 0`).  `iteration_callback` is honoured on a
slow path that copies rho and C to the host once per iteration.

Numerics: the f64 build reproduces the reference f64 path to
~1e-10 Ha; the f32 build stores ERIs in f32 and runs the XC grid contractions in
f32 (the reference's f32 BLAS path), everything else in f64.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .basis import BasisSet, expand
from .constants import HARTREE_TO_EV
from .engine import EngineOptions, Plan, status_error
from .errors import DeskDFTError, DimensionError, MoleculeError, ResourceLimitError
from .grids import check_level
from .molio import Molecule, electron_count

EXACT_EXCHANGE_FRACTION = 0.20
LINDEP_THRESHOLD = 1e-7
DIIS_COND_MAX = 1e12
DIIS_RING_MAX = 64        # device DIIS ring (csrc/common.cuh DIIS_MAX)


@dataclass(frozen=True)
class OrbitalSolution:
    C: np.ndarray
    epsilon: np.ndarray
    n_occ: int


@dataclass(frozen=True)
class SCFResult:
    solution: OrbitalSolution
    E_total: float
    E_components: dict
    energy_history: list
    converged: bool
    iterations: int
    n_ao: int


@dataclass
class SCFOptions:
    max_iterations: int = 50
    convergence_std: float = 0.01
    diis_history: int = 8
    precision: str = "f64"
    damping_factor: float = 0.5
    grid_level: int = 1
    screen_eps: float = 1e-12
    diis_start: int = 3

    def __post_init__(self):
        if self.max_iterations < 5:
            raise DeskDFTError("max_iterations must be >= 5 (convergence window needs 5 energies)")
        if self.precision not in ("f32", "f64"):
            raise DeskDFTError(f"precision must be 'f32' or 'f64', got {self.precision!r}")

    @property
    def dtype(self):
        return np.float32 if self.precision == "f32" else np.float64

    def ring(self) -> int:
        """DIIS ring slots: the reference keeps the last diis_history (F, error) pairs, so
        never more than max_iterations of them (scf.py:191-195).  diis_history <= 0 leaves
        the buffer empty, which the reference's diis_step rejects once DIIS is reached."""
        h = min(int(self.diis_history), int(self.max_iterations))
        if h < 1:
            if self.diis_start <= self.max_iterations:
                raise DeskDFTError("diis_step requires at least one (F, error) pair")
            return 1                      # DIIS never runs
        if h > DIIS_RING_MAX:
            raise ResourceLimitError(f"diis_history={h} exceeds the device DIIS ring ({DIIS_RING_MAX})")
        return h

    def engine(self) -> EngineOptions:
        check_level(self.grid_level)
        return EngineOptions(self.precision, self.max_iterations, self.convergence_std,
                             self.ring(), self.diis_start, self.damping_factor,
                             self.screen_eps, self.grid_level)


COMPONENT_KEYS = ("E_nn", "E_core", "E_coulomb", "E_exx", "E_xc")


def _result(res, m: int, nocc: int, n_ao: int, dtype) -> SCFResult:
    nit = int(res.iterations[m])
    comps = {k: float(v) for k, v in zip(COMPONENT_KEYS, res.E_comp[m])}
    nmo = int(res.n_mo[m])
    sol = OrbitalSolution(C=res.C[m].astype(dtype), epsilon=res.epsilon[m, :nmo].astype(dtype),
                          n_occ=nocc)
    return SCFResult(solution=sol, E_total=float(res.history[m, nit - 1]), E_components=comps,
                     energy_history=[float(x) for x in res.history[m, :nit]],
                     converged=bool(res.converged[m]), iterations=nit, n_ao=n_ao)


def scf_batch(mols: list[Molecule], b: BasisSet, opts: SCFOptions | None = None,
              errors: str = "raise", stream=None) -> list:
    """Run the SCF for every molecule of `mols` in one device batch.

    errors="raise" raises the first per-molecule failure (the reference's exception
    class); errors="return" puts the exception object in that molecule's slot.
    `stream`: CUDA stream handle (int / c_void_p) to run on; default the current torch
    stream.  The call returns when the batch's results are on the host."""
    opts = opts or SCFOptions()
    if not mols:
        return []
    return finish_batch(start_batch(mols, b, opts, stream), opts, errors)


class DeviceLabels(dict):
    """The tensors of scf_batch_device, plus the device plan they were computed by: the
    plan is released (stream-ordered) by close() / garbage collection, so the call itself
    never waits for the device."""

    def __init__(self, tensors: dict, plan: Plan):
        super().__init__(tensors)
        self._plan = plan

    def close(self):
        if self._plan is not None:
            self._plan.close()
            self._plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def scf_batch_device(mols: list[Molecule], b: BasisSet, opts: SCFOptions | None = None,
                     with_orbitals: bool = False) -> DeviceLabels:
    """scf_batch for device consumers: the labels land in torch tensors on the current CUDA
    device, written on the current torch stream with no host synchronisation (the caller
    owns the tensors; dftb_plan_fetch_device).  Keys: E_total [n] f64, E_comp [n, 5],
    history [n, max_iterations] (NaN past `iterations`), iterations / converged / n_mo /
    status [n] i32, epsilon [n, NMAX] (ascending, first n_mo valid) and, with
    with_orbitals, C (concatenated row-major n_ao x n_ao blocks).  Per-molecule failures
    are reported through `status` (DFTB_ST_* bits), not raised."""
    import torch

    opts = opts or SCFOptions()
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    plan = start_batch(mols, b, opts, stream)
    try:
        n, mi = int(plan.pk.n_mol), int(opts.max_iterations)
        f64 = dict(dtype=torch.float64, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        out = {"E_total": torch.empty(n, **f64), "E_comp": torch.empty((n, 5), **f64),
               "history": torch.empty((n, mi), **f64), "iterations": torch.empty(n, **i32),
               "converged": torch.empty(n, **i32), "n_mo": torch.empty(n, **i32),
               "epsilon": torch.empty((n, _lib.NMAX), **f64), "status": torch.empty(n, **i32)}
        if with_orbitals:
            nao = np.asarray(plan.pk.mol_nao, dtype=np.int64)
            out["C"] = torch.empty(int((nao * nao).sum()), **f64)
        plan.fetch_device(out)
    except BaseException:
        plan.close()
        raise
    return DeviceLabels(out, plan)


def start_batch(mols: list[Molecule], b: BasisSet, opts: SCFOptions, stream=None) -> Plan:
    """First half of scf_batch: pack, create the device plan and enqueue the whole SCF on
    `stream` without waiting (the labeling pipeline prepares the next batch meanwhile)."""
    plan = Plan(list(mols), b, opts.engine(), stream=stream)
    try:
        plan.run()
    except BaseException:
        plan.close()
        raise
    return plan


def finish_batch(plan: Plan, opts: SCFOptions, errors: str = "raise") -> list:
    """Second half of scf_batch: wait for the plan, copy the results back, release it."""
    try:
        res = plan.fetch()
    finally:
        plan.close()
    out = []
    for m in range(int(plan.pk.n_mol)):
        err = status_error(int(res.status[m]))
        if err is not None:
            if errors == "raise":
                raise err
            out.append(err)
            continue
        out.append(_result(res, m, int(plan.pk.mol_nocc[m]), int(plan.pk.mol_nao[m]), opts.dtype))
    return out


def scf(m: Molecule, b: BasisSet, opts: SCFOptions | None = None,
        iteration_callback=None) -> SCFResult:
    """Drop-in for deskdft.scf.scf (scf.py:139-210)."""
    opts = opts or SCFOptions()
    nelec = electron_count(m)
    ao = expand(m, b)
    if nelec // 2 > ao.n_ao:
        raise MoleculeError(f"{nelec} electrons need {nelec // 2} orbitals but basis has {ao.n_ao}")
    if iteration_callback is None:
        return scf_batch([m], b, opts)[0]
    return _scf_with_callback(m, b, opts, iteration_callback)


def _scf_with_callback(m, b, opts, cb) -> SCFResult:
    """Slow path: one device iteration at a time, rho / C copied to the host for the callback."""
    with Plan([m], b, opts.engine()) as plan:
        plan.set_full_eig(True)          # the callback observes C every iteration
        plan.begin()
        S = plan.get("S").astype(opts.dtype)
        n = int(plan.pk.mol_nao[0])
        for it in range(opts.max_iterations):
            rho = plan.get("rho").astype(opts.dtype)
            C = plan.get("C")
            plan.iterate(it)
            res = plan.fetch(want_C=False)
            nmo = int(res.n_mo[0])
            cb(it, rho, S, C[:, :nmo].astype(opts.dtype), float(res.history[0, it]))
            if res.converged[0]:
                break
        res = plan.fetch()
    err = status_error(int(res.status[0]))
    if err is not None:
        raise err
    del n
    return _result(res, 0, int(plan.pk.mol_nocc[0]), int(plan.pk.mol_nao[0]), opts.dtype)


def properties(r: SCFResult) -> dict[str, float]:
    """HOMO and LUMO (Hartree) and the gap (eV) (scf.py:213-222)."""
    sol = r.solution
    if sol.n_occ >= sol.epsilon.shape[0]:
        raise DeskDFTError("no virtual orbital: n_occ equals the orbital count")
    if sol.n_occ < 1:
        raise DeskDFTError("no occupied orbital")
    homo = float(sol.epsilon[sol.n_occ - 1])
    lumo = float(sol.epsilon[sol.n_occ])
    return {"homo": homo, "lumo": lumo, "gap": (lumo - homo) * HARTREE_TO_EV}


# ---------------------------------------------------------------------------- operator mirrors

def density(sol: OrbitalSolution) -> np.ndarray:
    """rho = 2 C_occ C_occ^T (scf.py:68-74).  Host helper: the device loop fuses it."""
    if sol.n_occ > sol.C.shape[1]:
        raise DimensionError(f"n_occ={sol.n_occ} exceeds {sol.C.shape[1]} orbitals (basis too small)")
    c = sol.C[:, :sol.n_occ]
    return 2.0 * c @ c.T


def fock(ints, J: np.ndarray, K: np.ndarray, Vxc: np.ndarray) -> np.ndarray:
    """F = V + T + J + a_x K + V_xc (scf.py:77-83).  Host helper: the device loop fuses it."""
    n = ints.n_ao
    for name, mat in (("J", J), ("K", K), ("Vxc", Vxc)):
        if mat.shape != (n, n):
            raise DimensionError(f"{name} shape {mat.shape} != ({n}, {n})")
    return ints.V + ints.T + J + EXACT_EXCHANGE_FRACTION * K + Vxc


def solve_roothaan(F: np.ndarray, S: np.ndarray, n_occ: int = 0) -> OrbitalSolution:
    """Canonical orthogonalisation + eigensolve on the device (scf.py:86-98).

    The device solver needs the overlap as produced by a basis, so this mirror runs
    on a synthetic plan whose S is overwritten... see integrals.solve_roothaan_device."""
    from .linalg import roothaan_device

    return roothaan_device(F, S, n_occ)


def diis_step(history: list) -> np.ndarray:
    """Pulay extrapolation with the cond(B) > 1e12 fallback, on the device (scf.py:101-132)."""
    if not history:
        raise DeskDFTError("diis_step requires at least one (F, error) pair")
    if len(history) == 1:
        return history[0][0]
    if len(history) > DIIS_RING_MAX:
        raise ResourceLimitError(f"{len(history)} DIIS entries exceed the device limit {DIIS_RING_MAX}")
    lib = _lib.load()
    F = np.ascontiguousarray(np.stack([h[0] for h in history]), dtype=np.float64)
    E = np.ascontiguousarray(np.stack([h[1] for h in history]), dtype=np.float64)
    n = F.shape[1]
    out = np.empty((n, n))
    _lib.check(lib.dftb_diis(_lib.ptr(F), _lib.ptr(E), len(history), n, _lib.ptr(out), _lib.current_stream()))
    return out.astype(history[-1][0].dtype)
