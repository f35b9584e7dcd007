"""Seeded synthetic closed-shell molecules (the BASELINE.json workload generator).

QM1B / GDB-11 conformers are not available offline, so the benchmark and the
parity suites use this generator with the shape statistics BASELINE.json names:

* heavy atoms drawn from C/N/O/F with p = 0.70/0.12/0.15/0.03;
* bonded as a random spanning tree plus 0-2 ring-closing bonds (valence
  C 4, N 3, O 2, F 1 never exceeded);
* placed by a seeded 3-D random walk: heavy-atom bonds 1.40-1.54 A, bond angles
  109.5 +- 10 degrees to the parent bond, random dihedral;
* ring-closing bonds are real bonds geometrically: a ring closes only where an atom
  can sit at bond distance (1.40-1.54 A) from both partners with sp3-compatible
  angles (round 1 closed rings in the bond graph only, which left two distant
  atoms each one H short - diradical-like molecules whose SCF did not settle);
* open valences filled with H at 1.09 A along the open sp3 directions of the
  final bond geometry;
* every pair of atoms at least 0.9 A apart, non-bonded pairs at least 1.5 A
  (otherwise the draw is retried);
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
NONBONDED_MIN_A = 1.5
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


def _tree(n_heavy, rng):
    """Elements + spanning-tree bonds (parent < child) with valences C 4, N 3, O 2, F 1."""
    for _ in range(1000):
        zs = rng.choice(HEAVY_Z, size=n_heavy, p=HEAVY_P)
        deg = np.zeros(n_heavy, int)
        bonds = []
        ok = True
        for child in range(1, n_heavy):
            cand = [a for a in range(child) if deg[a] < VALENCE[int(zs[a])]]
            if not cand:
                ok = False
                break
            parent = int(rng.choice(cand))
            bonds.append((parent, child))
            deg[parent] += 1
            deg[child] += 1
        if ok:
            return zs, bonds, deg
    raise RuntimeError("could not draw a valence-consistent spanning tree")


def _free_dirs(bond_dirs, rng):
    """The 4 - len(bond_dirs) open sp3 directions of an atom whose existing bonds point along
    the unit vectors `bond_dirs`, with the generator's angular jitter:
    one bond: three directions at 109.5 +- 10 degrees from it, azimuths 120 degrees
    apart (+- 10) from a random start; two bonds: the two tetrahedral directions about their
    negative bisector (+- 5 degrees); three bonds: the negative sum; none: a random tetrahedron."""
    nb = len(bond_dirs)
    if nb == 0:
        back = _unit(rng.standard_normal(3))
        return [back] + _free_dirs([back], rng)
    if nb == 1:
        back = bond_dirs[0]
        p = _perp(back, rng)
        q = np.cross(back, p)
        phi0 = rng.uniform(0.0, 2.0 * math.pi)
        out = []
        for k in range(3):
            ang = math.radians(rng.uniform(99.5, 119.5))
            phi = phi0 + k * 2.0 * math.pi / 3.0 + math.radians(rng.uniform(-10.0, 10.0))
            out.append(math.cos(ang) * back + math.sin(ang) * (math.cos(phi) * p + math.sin(phi) * q))
        return out
    if nb == 2:
        u, v = bond_dirs
        s = u + v
        w = _unit(-s) if np.linalg.norm(s) > 1e-6 else _perp(u, rng)
        nrm = np.cross(u, v)
        n = _unit(nrm) if np.linalg.norm(nrm) > 1e-6 else _perp(w, rng)
        out = []
        for sgn in (1.0, -1.0):
            th = math.radians(54.75 + rng.uniform(-5.0, 5.0))
            out.append(_unit(math.cos(th) * w + sgn * math.sin(th) * n))
        return out
    if nb == 3:
        s = bond_dirs[0] + bond_dirs[1] + bond_dirs[2]
        if np.linalg.norm(s) < 1e-6:
            return [_unit(np.cross(bond_dirs[0], bond_dirs[1]))]
        return [_unit(-s)]
    return []


def _angles_ok(d, dirs, min_deg):
    """Unit direction d makes at least `min_deg` with every unit vector in dirs."""
    c = math.cos(math.radians(min_deg))
    return all(float(d.dot(e)) <= c for e in dirs)


def _ring_site(pa, la, pb, lb, others, dirs_a, dirs_b, rng):
    """A position at distance la from pa and lb from pb (the circle where the two bond spheres
    meet) with sp3-compatible angles: >= 95 degrees to the existing bonds of a and of b, an
    a-c-b angle of 90-125 degrees, and >= 1.8 A from every other placed atom.  Of 24 azimuths
    (random start) the one farthest from the other atoms is taken; None if none qualifies."""
    ab = pb - pa
    d = float(np.linalg.norm(ab))
    e = ab / d
    x = (d * d + la * la - lb * lb) / (2.0 * d)
    h2 = la * la - x * x
    if h2 <= 0.0:
        return None
    h = math.sqrt(h2)
    p = _perp(e, rng)
    q = np.cross(e, p)
    phi0 = rng.uniform(0.0, 2.0 * math.pi)
    best, best_sep = None, 1.8
    for k in range(24):
        phi = phi0 + k * 2.0 * math.pi / 24.0
        c = pa + x * e + h * (math.cos(phi) * p + math.sin(phi) * q)
        ua, ub = _unit(c - pa), _unit(c - pb)
        if not (_angles_ok(ua, dirs_a, 95.0) and _angles_ok(ub, dirs_b, 95.0)):
            continue
        acb = math.degrees(math.acos(max(-1.0, min(1.0, float(_unit(pa - c).dot(_unit(pb - c)))))))
        if not 90.0 <= acb <= 125.0:
            continue
        sep = min((float(np.linalg.norm(c - o)) for o in others), default=10.0)
        if sep > best_sep:
            best, best_sep = c, sep
    return best


def _place(zs, tree, tdeg, n_ring, rng):
    """Random-walk placement along the tree bonds with up to `n_ring` ring-closing bonds made
    where the geometry allows one, then H on the open valences.

    Atoms are placed breadth first; a child c of a goes along one of a's open sp3 directions
    at 1.40-1.54 A.  While rings are still wanted and c has a spare valence, c may instead
    close a ring with an already placed heavy atom b (spare valence, not bonded to a, 2.0-2.9 A
    from a): c then sits at bond distance from both a and b (_ring_site), so every ring bond
    has a bonded length (1.40-1.54 A) and sp3-compatible angles.  Hydrogens go along the open
    directions of the final bond geometry at 1.09 A."""
    n = len(zs)
    children = {i: [] for i in range(n)}
    for a, b in tree:
        children[a].append(b)
    spare = np.array([VALENCE[int(z)] for z in zs]) - tdeg
    nbr = {i: [] for i in range(n)}
    pos = np.zeros((n, 3))
    placed = [0]
    rings = []
    order, k = [0], 0
    while k < len(order):
        a = order[k]
        k += 1
        for c in children[a]:
            la = rng.uniform(1.40, 1.54)
            site = None
            if len(rings) < n_ring and spare[c] > 0:
                dist = {b: float(np.linalg.norm(pos[b] - pos[a])) for b in placed}
                cand = [b for b in placed if b != a and b not in nbr[a] and spare[b] > 0
                        and 2.0 <= dist[b] <= 2.9]
                rng.shuffle(cand)
                for b in cand:
                    lb = rng.uniform(1.40, 1.54)
                    others = [pos[o] for o in placed if o not in (a, b)]
                    site = _ring_site(pos[a], la, pos[b], lb, others,
                                      [_unit(pos[x] - pos[a]) for x in nbr[a]],
                                      [_unit(pos[x] - pos[b]) for x in nbr[b]], rng)
                    if site is not None:
                        rings.append((b, c))
                        spare[b] -= 1
                        spare[c] -= 1
                        nbr[b].append(c)
                        nbr[c].append(b)
                        break
            if site is None:
                d = _free_dirs([_unit(pos[x] - pos[a]) for x in nbr[a]], rng)[0]
                site = pos[a] + la * d
            pos[c] = site
            nbr[a].append(c)
            nbr[c].append(a)
            placed.append(c)
            order.append(c)
    hs = []
    for a in range(n):
        nh = int(spare[a])
        free = _free_dirs([_unit(pos[x] - pos[a]) for x in nbr[a]], rng)
        if nh > len(free):
            raise RuntimeError("valence bookkeeping")
        for d in free[:nh]:
            hs.append(pos[a] + CH_BOND_A * d)
    bonds = list(tree) + rings
    return pos, np.array(hs).reshape(-1, 3), bonds


def random_molecule(n_heavy: int, rng: np.random.Generator, mol_id: str = "",
                    max_tries: int = 200) -> Molecule:
    """One synthetic molecule (positions in Bohr).

    Draw checks: every pair of atoms >= 0.9 A apart (BASELINE), and non-bonded pairs
    >= 1.5 A (no non-bonded contacts at bonding distance: the SCF of such draws does not
    settle, like that of a stretched bond)."""
    for _ in range(max_tries):
        zs, tree, tdeg = _tree(n_heavy, rng)
        n_ring = int(rng.integers(0, 3))
        heavy, hpos, bonds = _place(zs, tree, tdeg, n_ring, rng)
        allpos = np.vstack([heavy, hpos])
        n_all = len(allpos)
        d2 = np.sum((allpos[:, None] - allpos[None]) ** 2, axis=-1)
        np.fill_diagonal(d2, np.inf)
        if d2.min() < MIN_SEP_A ** 2:
            continue
        bonded = np.zeros((n_all, n_all), bool)
        for a, b in bonds:
            bonded[a, b] = bonded[b, a] = True
        # H k (index len(zs) + k) is bonded to the heavy atom it was placed from
        h0 = len(zs)
        hk = 0
        for a in range(len(zs)):
            nh = VALENCE[int(zs[a])] - sum(1 for x, y in bonds if a in (x, y))
            for _h in range(nh):
                bonded[a, h0 + hk] = bonded[h0 + hk, a] = True
                hk += 1
        np.fill_diagonal(bonded, True)
        if np.any(d2[~bonded] < NONBONDED_MIN_A ** 2):
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
