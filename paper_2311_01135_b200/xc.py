"""Grid, AO values and B3LYP — drop-in for deskdft.xc (xc.py:60-350).

`build_grid` (atom-centred templates + device Becke partition), `eval_ao`
(device AO values and gradients), `b3lyp` (device pointwise functional) and
`xc_matrix` (the fused device kernel: AO recompute, density, functional, V_xc)
keep the reference's names, dataclasses, options and errors.  The fused kernel
recomputes AO values from the basis, so `xc_matrix` needs an `AOGridValues`
produced by this module's `eval_ao` (it carries its basis); the device never
stores phi for the SCF.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .basis import AOBasis
from .batch import pack
from .engine import EngineOptions, Plan, status_error
from .errors import DeskDFTError, DimensionError
from .grids import check_level
from .integrals import molecule_from_ao
from .molio import Molecule

DENSITY_FLOOR = 1e-12
XC_BATCH = 8192
W_LSDA_X, W_B88_X, W_VWN_C, W_LYP_C = 0.08, 0.72, 0.19, 0.81


@dataclass(frozen=True)
class Grid:
    points: np.ndarray
    weights: np.ndarray
    level: int

    @property
    def n_points(self) -> int:
        return int(self.points.shape[0])


@dataclass(frozen=True)
class AOGridValues:
    phi: np.ndarray
    grad_phi: np.ndarray
    ao: AOBasis | None = field(default=None, compare=False, repr=False)
    grid: Grid | None = field(default=None, compare=False, repr=False)


@dataclass(frozen=True)
class XCResult:
    E_xc: float
    V_xc: np.ndarray


def build_grid(m: Molecule, level: int = 1) -> Grid:
    """Per-atom TA-radial x pruned-Lebedev grids with Becke weights (xc.py:123-162)."""
    check_level(level)
    from .basis import load_basis

    b = load_basis("sto-3g") if all(z <= 10 for z in m.atomic_numbers) else None
    if b is None:
        raise DeskDFTError("the device grid path covers H-Ne")
    # the electron count is irrelevant for a grid: pack with a neutral dummy occupation
    pk = pack([_neutral(m)], b, level)
    with Plan(pk, None, EngineOptions(grid_level=level, max_iterations=1)) as p:
        _lib.check(p.lib.dftb_plan_grid(p.h, p.stream))
        pts = p.get("points")
        w = p.get("weights")
        st = _status(p)
    err = status_error(st)
    if err is not None:
        raise err
    pts.setflags(write=False)
    w.setflags(write=False)
    return Grid(points=pts, weights=w, level=level)


def _neutral(m: Molecule) -> Molecule:
    q = sum(m.atomic_numbers) % 2
    return Molecule(m.atomic_numbers, m.positions, charge=q)


def _status(p: Plan) -> int:
    import ctypes

    res = p.fetch(want_C=False)
    del ctypes
    return int(res.status[0])


def _plan_with_grid(ao: AOBasis, g: Grid, precision: str = "f64") -> Plan:
    mol, b = molecule_from_ao(ao)
    pk = pack([_neutral(mol)], b, None)
    n = g.n_points
    pk.tmpl_xyzw = np.zeros((n, 4))
    pk.atom_tmpl0 = np.zeros(pk.n_atom, np.int32)
    pk.atom_tmpln = np.zeros(pk.n_atom, np.int32)
    pk.atom_tmpln[0] = n
    pk.mol_npts = np.array([n], np.int64)
    p = Plan(pk, None, EngineOptions(precision=precision, grid_level=None, max_iterations=1))
    pts = np.ascontiguousarray(g.points, np.float64)
    w = np.ascontiguousarray(g.weights, np.float64)
    _lib.check(p.lib.dftb_plan_load_grid(p.h, _lib.ptr(pts), _lib.ptr(w), n, p.stream))
    return p


def eval_ao(ao: AOBasis, g: Grid, dtype=np.float64) -> AOGridValues:
    """AO values and Cartesian gradients on the grid, computed on the device (xc.py:165-194)."""
    dtype = np.dtype(dtype)
    n = g.n_points
    with _plan_with_grid(ao, g) as p:
        phi = np.empty((n, ao.n_ao))
        grad = np.empty((3, n, ao.n_ao))
        _lib.check(p.lib.dftb_plan_eval_ao(p.h, 0, _lib.ptr(phi), _lib.ptr(grad), p.stream))
    return AOGridValues(phi=phi.astype(dtype), grad_phi=grad.astype(dtype), ao=ao, grid=g)


def b3lyp(rho_grid, sigma):
    """Semi-local B3LYP (exc per particle, vrho, vsigma) on the device (xc.py:277-306)."""
    n_in = np.asarray(rho_grid)
    s_in = np.asarray(sigma)
    if n_in.shape != s_in.shape:
        raise DimensionError("rho/sigma shape mismatch")
    out_dtype = n_in.dtype if n_in.dtype in (np.float32, np.float64) else np.float64
    n = np.ascontiguousarray(n_in, np.float64).ravel()
    s = np.ascontiguousarray(s_in, np.float64).ravel()
    e, vr, vs = np.empty_like(n), np.empty_like(n), np.empty_like(n)
    lib = _lib.load()
    _lib.check(lib.dftb_b3lyp(_lib.ptr(n), _lib.ptr(s), len(n), _lib.ptr(e), _lib.ptr(vr), _lib.ptr(vs),
                              _lib.current_stream()))
    shp = n_in.shape
    return (e.reshape(shp).astype(out_dtype), vr.reshape(shp).astype(out_dtype),
            vs.reshape(shp).astype(out_dtype))


def density_on_grid(aov: AOGridValues, rho: np.ndarray):
    """n and grad n on the grid from stored AO values (xc.py:309-317; test helper)."""
    t = aov.phi @ rho
    n = np.einsum("pi,pi->p", t, aov.phi)
    gn = np.stack([2.0 * np.einsum("pi,pi->p", aov.grad_phi[d], t) for d in range(3)]).astype(aov.phi.dtype)
    return n, gn


def xc_matrix(g: Grid, aov: AOGridValues, rho: np.ndarray) -> XCResult:
    """E_xc and the symmetric V_xc, on the device fused kernel (xc.py:320-350)."""
    n_ao = aov.phi.shape[1]
    if rho.shape != (n_ao, n_ao):
        raise DimensionError(f"rho shape {rho.shape} does not match n_ao={n_ao}")
    if aov.ao is None:
        raise DeskDFTError("xc_matrix needs AOGridValues from this package's eval_ao (it carries the basis)")
    prec = "f32" if aov.phi.dtype == np.float32 else "f64"
    with _plan_with_grid(aov.ao, g, prec) as p:
        r = np.ascontiguousarray(rho, np.float64)
        V = np.empty((n_ao, n_ao))
        E = np.empty(1)
        _lib.check(p.lib.dftb_plan_xc(p.h, _lib.ptr(r), _lib.ptr(V), _lib.ptr(E), p.stream))
    return XCResult(E_xc=float(E[0]), V_xc=V.astype(aov.phi.dtype))
