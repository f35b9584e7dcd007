"""Seeded synthetic closed-shell molecules (the BASELINE.json workload generator).

QM1B / GDB-11 conformers are not available offline, so the benchmark and the
parity suites use this generator with the shape statistics BASELINE.json names:

* heavy atoms drawn from C/N/O/F with p = 0.70/0.12/0.15/0.03;
* bonded as a random spanning tree plus 0-2 ring-closing bonds (valence
  C 4, N 3, O 2, F 1 never exceeded);
* placed by a seeded 3-D random walk: heavy-atom bonds 1.40-1.54 A, bond angles
  109.5 +- 10 degrees to the parent bond, random dihedral;
* open valences filled with H at 1.09 A, pointing away from the existing bonds;
* every pair of atoms at least 0.9 A apart (otherwise the draw is retried);
* even electron count (automatic for fully saturated valences; checked).

Molecule k of a batch with base seed s uses numpy.random.default_rng((s, k)).
"""

from __future__ import annotations

import math

import numpy as np

from .constants import ANGSTROM_TO_BOHR
from .molio import Molecule

HEAVY_Z = np.array([6, 7, 8, 9])
HEAVY_P = np.array([0.70, 0.12, 0.15, 0.03])
VALENCE = {6: 4, 7: 3, 8: 2, 9: 1}
MIN_SEP_A = 0.9
CH_BOND_A = 1.09


def _unit(v):
    return v / np.linalg.norm(v)


def _perp(v, rng):
    """Random unit vector perpendicular to unit v."""
    while True:
        r = rng.standard_normal(3)
        r -= r.dot(v) * v
        nr = np.linalg.norm(r)
        if nr > 1e-6:
            return r / nr


def _cone_dir(axis, angle, rng):
    """Unit vector at `angle` from unit `axis` with a uniformly random azimuth."""
    p = _perp(axis, rng)
    return math.cos(angle) * axis + math.sin(angle) * p


def _topology(n_heavy, rng):
    """Elements + bond list for a random spanning tree plus 0-2 ring closures."""
    for _ in range(1000):
        zs = rng.choice(HEAVY_Z, size=n_heavy, p=HEAVY_P)
        deg = np.zeros(n_heavy, int)
        bonds = []
        ok = True
        for child in range(1, n_heavy):
            cand = [a for a in range(child) if deg[a] < VALENCE[int(zs[a])]]
            if VALENCE[int(zs[child])] < 1 or not cand:
                ok = False
                break
            parent = int(rng.choice(cand))
            bonds.append((parent, child))
            deg[parent] += 1
            deg[child] += 1
        if not ok:
            continue
        n_ring = int(rng.integers(0, 3))
        for _r in range(n_ring):
            free = [a for a in range(n_heavy) if deg[a] < VALENCE[int(zs[a])]]
            pairs = [(a, b) for i, a in enumerate(free) for b in free[i + 1:]
                     if (a, b) not in bonds and (b, a) not in bonds]
            if not pairs:
                break
            a, b = pairs[int(rng.integers(len(pairs)))]
            bonds.append((a, b))
            deg[a] += 1
            deg[b] += 1
        return zs, bonds, deg
    raise RuntimeError("could not draw a valence-consistent spanning tree")


def _slots(back, rng):
    """Four tetrahedral-ish bond directions: slot 0 = `back`; slots 1-3 at
    109.5 +- 10 degrees from it, azimuths 120 degrees apart from a random start."""
    p = _perp(back, rng)
    q = np.cross(back, p)
    phi0 = rng.uniform(0.0, 2.0 * math.pi)
    out = [back]
    for k in range(3):
        ang = math.radians(rng.uniform(99.5, 119.5))
        phi = phi0 + k * 2.0 * math.pi / 3.0 + math.radians(rng.uniform(-10.0, 10.0))
        out.append(math.cos(ang) * back + math.sin(ang) * (math.cos(phi) * p + math.sin(phi) * q))
    return out


def _place(zs, bonds, deg, rng):
    """Random-walk placement of heavy atoms along tree bonds, then H on open valences.

    Each atom owns four tetrahedral slots (slot 0 points back to its parent);
    tree children take the next free slots, hydrogens fill the open valences
    from the slots that remain."""
    n = len(zs)
    children = {i: [] for i in range(n)}
    parent = {0: -1}
    for a, b in bonds[: n - 1]:  # the first n-1 bonds are the spanning tree, parent < child
        children[a].append(b)
        parent[b] = a
    pos = np.zeros((n, 3))
    slots = {0: _slots(_unit(rng.standard_normal(3)), rng)}
    used = {0: 0}  # root: slot 0 is a free direction too
    order = [0]
    k = 0
    while k < len(order):
        a = order[k]
        k += 1
        for c in children[a]:
            d = slots[a][used[a]] if parent[a] < 0 else slots[a][used[a] + 1]
            used[a] += 1
            pos[c] = pos[a] + rng.uniform(1.40, 1.54) * d
            slots[c] = _slots(-d, rng)
            used[c] = 0
            order.append(c)
    hs = []
    for a in range(n):
        nh = VALENCE[int(zs[a])] - int(deg[a])
        first = used[a] if parent[a] < 0 else used[a] + 1
        free = slots[a][first:]
        for d in free[:nh]:
            hs.append(pos[a] + CH_BOND_A * d)
        if nh > len(free):  # ring-closure bookkeeping never frees slots, so this cannot happen
            raise RuntimeError("valence bookkeeping")
    return pos, np.array(hs).reshape(-1, 3)


def random_molecule(n_heavy: int, rng: np.random.Generator, mol_id: str = "",
                    max_tries: int = 200) -> Molecule:
    """One synthetic molecule (positions in Bohr)."""
    for _ in range(max_tries):
        zs, bonds, deg = _topology(n_heavy, rng)
        heavy, hpos = _place(zs, bonds, deg, rng)
        allpos = np.vstack([heavy, hpos])
        d2 = np.sum((allpos[:, None] - allpos[None]) ** 2, axis=-1)
        np.fill_diagonal(d2, np.inf)
        if d2.min() < MIN_SEP_A ** 2:
            continue
        Z = tuple(int(z) for z in zs) + (1,) * len(hpos)
        if sum(Z) % 2:
            continue
        return Molecule(Z, allpos * ANGSTROM_TO_BOHR, id=mol_id)
    raise RuntimeError(f"no valid geometry after {max_tries} draws")


def batch(n_mol: int, heavy, seed: int = 0) -> list[Molecule]:
    """`n_mol` molecules; `heavy` is an int or a sequence to draw uniformly from."""
    out = []
    for k in range(n_mol):
        rng = np.random.default_rng((seed, k))
        nh = heavy if isinstance(heavy, int) else int(rng.choice(list(heavy)))
        out.append(random_molecule(nh, rng, mol_id=f"syn{seed}-{k}"))
    return out


def water_config1() -> Molecule:
    """BASELINE configs[0]: O at the origin, H at 0.9572 A, 104.5 deg, plane xy, bisector +y."""
    r = 0.9572 * ANGSTROM_TO_BOHR
    h = math.radians(104.5) / 2
    pos = np.array([[0.0, 0.0, 0.0],
                    [r * math.sin(h), r * math.cos(h), 0.0],
                    [-r * math.sin(h), r * math.cos(h), 0.0]])
    return Molecule((8, 1, 1), pos, id="water")
