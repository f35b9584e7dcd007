"""Atom-centred quadrature templates (constant tables for the device grid kernel).

The molecular grid of the reference (deskdft/xc.py:123-162) is, per atom, a
Treutler-Ahlrichs radial rule times pruned Lebedev shells, multiplied by Becke
partition weights.  Everything except the Becke factor depends only on the
element and the grid level, so it is tabulated here once per (Z, level) and the
device kernel (csrc/grid.cu) adds the atom centre and the Becke weight.

Parity needs the identical point set: the Lebedev points and weights come from
scipy.integrate.lebedev_rule (the reference's own source, xc.py:17,101-104),
unrotated, in scipy's order; radial nodes ascending; the pruning thresholds of
xc.py:33-57.
"""

from __future__ import annotations

import math
from functools import lru_cache

import numpy as np

from .constants import ANGSTROM_TO_BOHR
from .errors import DeskDFTError

LEBEDEV_DEGREE = {6: 3, 14: 5, 26: 7, 38: 9, 50: 11, 86: 15, 110: 17, 146: 19, 194: 23, 302: 29}
TA_XI = (0.8, 0.9, 1.8, 1.4, 1.3, 1.1, 0.9, 0.9, 0.9, 0.9,
         1.4, 1.3, 1.3, 1.2, 1.1, 1.0, 1.0, 1.0)
BRAGG_A = (0.35, 0.31, 1.45, 1.05, 0.85, 0.70, 0.65, 0.60, 0.50, 0.38,
           1.80, 1.50, 1.25, 1.10, 1.00, 1.00, 1.00, 0.71)
LEVELS = {
    0: (18, 20, (14, 26, 26, 14), (14, 26, 38, 14)),
    1: (18, 30, (14, 26, 50, 26), (26, 50, 86, 26)),
    2: (30, 45, (26, 50, 146, 86), (38, 86, 194, 110)),
    3: (50, 65, (38, 110, 302, 302), (50, 146, 302, 302)),
}
PRUNE = (0.30, 0.60, 3.0)
FAR_MIN_BOHR = 4.0


def check_level(level: int) -> None:
    if level not in LEVELS:
        raise DeskDFTError(f"unsupported grid level {level}; choose from {sorted(LEVELS)}")


def radial_nodes(n: int, xi: float) -> tuple[np.ndarray, np.ndarray]:
    """Gauss-Chebyshev (2nd kind) nodes mapped by Treutler-Ahlrichs M4 (alpha = 0.6),
    returned with ascending r; weights include dr/dx."""
    k = np.arange(1, n + 1)
    th = k * np.pi / (n + 1)
    x = np.cos(th)
    wx = np.pi / (n + 1) * np.sin(th)
    scale = xi / math.log(2.0)
    lg = np.log(2.0 / (1.0 - x))
    r = scale * (1.0 + x) ** 0.6 * lg
    dr = scale * (1.0 + x) ** 0.6 * (0.6 * lg / (1.0 + x) + 1.0 / (1.0 - x))
    return r[::-1], (wx * dr)[::-1]


@lru_cache(maxsize=None)
def lebedev(npts: int) -> tuple[np.ndarray, np.ndarray]:
    from scipy.integrate import lebedev_rule

    pts, w = lebedev_rule(LEBEDEV_DEGREE[npts])
    return np.ascontiguousarray(pts.T), np.ascontiguousarray(w)


@lru_cache(maxsize=None)
def atom_template(z: int, level: int) -> np.ndarray:
    """(n, 4) array: r * unit vector (Bohr) and w_r r^2 w_ang, in the reference's point order."""
    check_level(level)
    nr_h, nr_x, sh_h, sh_x = LEVELS[level]
    nr, sched = (nr_h, sh_h) if z <= 2 else (nr_x, sh_x)
    r, wr = radial_nodes(nr, TA_XI[z - 1])
    rb = BRAGG_A[z - 1] * ANGSTROM_TO_BOHR
    rows = []
    for i in range(nr):
        if r[i] < PRUNE[0] * rb:
            na = sched[0]
        elif r[i] < PRUNE[1] * rb:
            na = sched[1]
        elif r[i] < max(PRUNE[2] * rb, FAR_MIN_BOHR):
            na = sched[2]
        else:
            na = sched[3]
        u, wa = lebedev(na)
        blk = np.empty((na, 4))
        blk[:, :3] = r[i] * u
        blk[:, 3] = wr[i] * r[i] ** 2 * wa
        rows.append(blk)
    out = np.ascontiguousarray(np.vstack(rows))
    out.setflags(write=False)
    return out
