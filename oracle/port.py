"""ORACLE — test infrastructure only; never imported by the product package.

A CPU restatement of the reference's restricted-KS B3LYP/STO-3G path
(`deskdft` under /root/reference/pkg/src/deskdft) used to check the CUDA
product: numpy/scipy for the driver, grid and functional, and the C kernels in
oracle/oracle_kernels.c (built to oracle/_oracle.so) for the integral kernels.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use it.

Each function cites the reference function it restates.  The restatement is
pinned against fixtures produced by running the reference itself
(tests/golden/, made by tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
from scipy.integrate import lebedev_rule
from scipy.special import hyp1f1

_HERE = os.path.dirname(os.path.abspath(__file__))

ANG2BOHR = 1.8897259886          # constants.py:16
HA2EV = 27.211386                 # constants.py:17
SYMBOLS = ("H", "He", "Li", "Be", "B", "C", "N", "O", "F", "Ne")

# STO-3G (H..Ne): per element, list of (l-letters, exponents, coefficient columns).
# Published Hehre-Stewart-Pople values (the same data the reference ships in
# basisdata/sto-3g.dat:5-96).  "SP" blocks carry two coefficient columns.
_STO3G_S = (0.15432897, 0.53532814, 0.44463454)
_STO3G_SP_S = (-0.09996723, 0.39951283, 0.70115470)
_STO3G_SP_P = (0.15591627, 0.60768372, 0.39195739)
_STO3G_EXP = {
    1: ((3.42525091, 0.62391373, 0.16885540),),
    2: ((6.36242139, 1.15892300, 0.31364979),),
    3: ((16.1195750, 2.9362007, 0.7946505), (0.6362897, 0.1478601, 0.0480887)),
    4: ((30.1678710, 5.4951153, 1.4871927), (1.3148331, 0.3055389, 0.0993707)),
    5: ((48.7911130, 8.8873622, 2.4052670), (2.2369561, 0.5198205, 0.1690618)),
    6: ((71.6168370, 13.0450960, 3.5305122), (2.9412494, 0.6834831, 0.2222899)),
    7: ((99.1061690, 18.0523120, 4.8856602), (3.7804559, 0.8784966, 0.2857144)),
    8: ((130.7093200, 23.8088610, 6.4436083), (5.0331513, 1.1695961, 0.3803890)),
    9: ((166.6791300, 30.3608120, 8.2168207), (6.4648032, 1.5022812, 0.4885885)),
    10: ((207.0156100, 37.7081510, 10.2052970), (8.2463151, 1.9162662, 0.6232293)),
}


def sto3g_shells(z: int):
    """Split shells (l, exps, coefs) for element z; SP -> S then P (basis.py:122-123,145-148)."""
    e = _STO3G_EXP[z]
    out = [(0, e[0], _STO3G_S)]
    if len(e) > 1:
        out.append((0, e[1], _STO3G_SP_S))
        out.append((1, e[1], _STO3G_SP_P))
    return out


# ----------------------------------------------------------------------------- molecule


@dataclass
class Mol:
    """Atomic numbers + positions in Bohr (molio.py:24-67)."""

    Z: tuple
    pos: np.ndarray
    charge: int = 0

    @property
    def nelec(self) -> int:                      # molio.py:70-75
        n = sum(self.Z) - self.charge
        if n <= 0 or n % 2:
            raise ValueError(f"electron count {n}: restricted-closed-shell violation")
        return n


def nuclear_repulsion(m: Mol) -> float:
    """sum_{a<b} Za Zb / r_ab  (molio.py:78-87)."""
    e = 0.0
    for a in range(len(m.Z)):
        for b in range(a + 1, len(m.Z)):
            e += m.Z[a] * m.Z[b] / math.dist(m.pos[a], m.pos[b])
    return e


# ----------------------------------------------------------------------------- basis


def _dfact(k: int) -> float:
    out = 1.0
    while k > 1:
        out *= k
        k -= 2
    return out


def _prim_norm(a, lx, ly, lz):                    # basis.py:180-184
    l = lx + ly + lz
    df = _dfact(2 * lx - 1) * _dfact(2 * ly - 1) * _dfact(2 * lz - 1)
    return (2 * a / math.pi) ** 0.75 * (4 * a) ** (0.5 * l) / math.sqrt(df)


COMPS = (((0, 0, 0),), ((1, 0, 0), (0, 1, 0), (0, 0, 1)))


@dataclass
class AO:
    """Kernel-facing split-shell SoA (basis.py:200-216)."""

    n_ao: int
    ao_offsets: np.ndarray
    shell_l: np.ndarray
    shell_center: np.ndarray
    prim_start: np.ndarray
    prim_count: np.ndarray
    prim_exp: np.ndarray
    prim_coef: np.ndarray

    @property
    def n_shells(self):
        return len(self.shell_l)


def expand(m: Mol) -> AO:
    """Shells on atoms in atom order, unit-self-overlap AOs (basis.py:223-276)."""
    offs, ls, cen, ps, pc, exps, coefs = [], [], [], [], [], [], []
    n = 0
    for ia, z in enumerate(m.Z):
        for l, e, c in sto3g_shells(z):
            e = np.asarray(e, float)
            c = np.asarray(c, float)
            row = np.zeros((3, 6))
            for ci, (lx, ly, lz) in enumerate(COMPS[l]):
                nrm = np.array([_prim_norm(a, lx, ly, lz) for a in e])
                df = _dfact(2 * lx - 1) * _dfact(2 * ly - 1) * _dfact(2 * lz - 1)
                s = e[:, None] + e[None, :]
                pair = (np.pi / s) ** 1.5 * df / (2 * s) ** l
                cn = c * nrm
                row[:, ci] = c * nrm / math.sqrt(float(cn @ pair @ cn))
            offs.append(n)
            ls.append(l)
            cen.append(m.pos[ia])
            ps.append(len(exps))
            pc.append(3)
            exps.extend(e)
            coefs.append(row)
            n += len(COMPS[l])
    return AO(n, np.array(offs, np.int32), np.array(ls, np.int32),
              np.ascontiguousarray(np.array(cen, float).reshape(-1, 3)),
              np.array(ps, np.int32), np.array(pc, np.int32), np.array(exps, float),
              np.ascontiguousarray(np.vstack(coefs)))


# ----------------------------------------------------------------------------- C kernels

_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "_oracle.so")
        if not os.path.exists(path):
            raise RuntimeError("oracle/_oracle.so missing: run `make -C oracle`")
        _lib = ctypes.CDLL(path)
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def boys_table():
    """431 x 16 table of F_m(T) from the confluent hypergeometric form (_kernels.py:38-45)."""
    ts = np.arange(0.0, 43.0 + 0.05, 0.1)
    ms = np.arange(0, 16)
    tt, mm = np.meshgrid(ts, ms, indexing="ij")
    return np.ascontiguousarray(hyp1f1(mm + 0.5, mm + 1.5, -tt) / (2 * mm + 1))


_BOYS = None


def _boys():
    global _BOYS
    if _BOYS is None:
        _BOYS = boys_table()
    return _BOYS


class PairTables:
    """Shell-pair primitive tables (integrals.py:72-97)."""

    def __init__(self, ao: AO):
        si, sj = np.tril_indices(ao.n_shells)
        self.si = si.astype(np.int32)
        self.sj = sj.astype(np.int32)
        cnt = (ao.prim_count[self.si] * ao.prim_count[self.sj]).astype(np.int64)
        self.start = np.zeros(len(si), np.int64)
        np.cumsum(cnt[:-1], out=self.start[1:])
        self.count = cnt.astype(np.int32)
        npp = int(cnt.sum())
        self.p = np.zeros(npp)
        self.P = np.zeros((npp, 3))
        self.ia = np.zeros(npp, np.int32)
        self.ib = np.zeros(npp, np.int32)
        self.cmaxK = np.zeros(npp)
        self.E = np.zeros((npp, 3, 45))
        lib().orc_pair_tables(ctypes.c_int(len(si)), _p(self.si), _p(self.sj), _p(ao.shell_l),
                              _p(ao.shell_center), _p(ao.prim_start), _p(ao.prim_count),
                              _p(ao.prim_coef), _p(ao.prim_exp), _p(self.start), _p(self.p),
                              _p(self.P), _p(self.ia), _p(self.ib), _p(self.cmaxK), _p(self.E))
        self.ao = ao
        self._schwarz = None

    def schwarz(self):                             # integrals.py:99-112
        if self._schwarz is None:
            ao = self.ao
            qp = np.zeros(len(self.si))
            qa = np.zeros(ao.n_ao * (ao.n_ao + 1) // 2)
            lib().orc_schwarz(ctypes.c_int(len(self.si)), _p(self.si), _p(self.sj), _p(self.start),
                              _p(self.count), _p(ao.shell_l), _p(ao.ao_offsets), _p(self.p),
                              _p(self.P), _p(self.ia), _p(self.ib), _p(self.cmaxK), _p(self.E),
                              _p(ao.prim_coef), _p(_boys()), _p(qp), _p(qa))
            self._schwarz = (qp, qa)
        return self._schwarz


def one_electron(ao: AO, m: Mol, dtype=np.float64):
    """S, T, V (integrals.py:115-132)."""
    n = ao.n_ao
    S, T, V = np.zeros((n, n)), np.zeros((n, n)), np.zeros((n, n))
    pt = PairTables(ao)
    xyz = np.ascontiguousarray(m.pos, dtype=float)
    zz = np.asarray(m.Z, float)
    lib().orc_one_electron(ctypes.c_int(len(pt.si)), _p(pt.si), _p(pt.sj), _p(ao.shell_l),
                           _p(ao.shell_center), _p(ao.ao_offsets), _p(ao.prim_start),
                           _p(ao.prim_count), _p(ao.prim_exp), _p(ao.prim_coef),
                           ctypes.c_int(len(m.Z)), _p(xyz), _p(zz), ctypes.c_int(n),
                           _p(S), _p(T), _p(V), _p(_boys()))
    return S.astype(dtype), T.astype(dtype), V.astype(dtype)


@dataclass
class Packed:
    """Canonical packed ERIs (integrals.py:43-69)."""

    i: np.ndarray
    j: np.ndarray
    k: np.ndarray
    l: np.ndarray
    values: np.ndarray
    degeneracy: np.ndarray
    n_ao: int


def eri_packed(ao: AO, screen_eps=1e-12, dtype=np.float64, pairs: PairTables | None = None):
    """Screened canonical ERIs in composite-pair order (integrals.py:135-196)."""
    dtype = np.dtype(dtype)
    pt = pairs or PairTables(ao)
    qp, qa = pt.schwarz()
    npair = len(pt.si)
    a, b = np.tril_indices(npair)
    if screen_eps > 0:
        keep = qp[a] * qp[b] >= screen_eps
        a, b = a[keep], b[keep]
    a = a.astype(np.int32)
    b = b.astype(np.int32)
    nq = len(a)
    counts = np.zeros(nq, np.int64)
    lib().orc_count(ctypes.c_int64(nq), _p(a), _p(b), _p(pt.si), _p(pt.sj), _p(ao.shell_l),
                    _p(ao.ao_offsets), _p(qa), ctypes.c_double(screen_eps), _p(counts))
    total = int(counts.sum())
    offs = np.zeros(nq, np.int64)
    np.cumsum(counts[:-1], out=offs[1:])
    oi, oj, ok, ol = (np.zeros(total, np.uint16) for _ in range(4))
    ov = np.zeros(total)
    od = np.zeros(total, np.uint8)
    lib().orc_fill(ctypes.c_int64(nq), _p(a), _p(b), _p(offs), _p(pt.si), _p(pt.sj),
                   _p(pt.start), _p(pt.count), _p(ao.shell_l), _p(ao.ao_offsets), _p(pt.p),
                   _p(pt.P), _p(pt.ia), _p(pt.ib), _p(pt.cmaxK), _p(pt.E), _p(ao.prim_coef),
                   _p(_boys()), _p(qa), ctypes.c_double(screen_eps),
                   ctypes.c_int(1 if dtype == np.float32 else 0),
                   _p(oi), _p(oj), _p(ok), _p(ol), _p(ov), _p(od))
    ov = ov.astype(dtype)
    if screen_eps > 0:
        kv = np.abs(ov) >= screen_eps
        oi, oj, ok, ol, ov, od = oi[kv], oj[kv], ok[kv], ol[kv], ov[kv], od[kv]
    ij = oi.astype(np.int64) * (oi.astype(np.int64) + 1) // 2 + oj
    kl = ok.astype(np.int64) * (ok.astype(np.int64) + 1) // 2 + ol
    npp = ao.n_ao * (ao.n_ao + 1) // 2
    o = np.argsort(ij * npp + kl, kind="stable")
    return Packed(oi[o], oj[o], ok[o], ol[o], ov[o], od[o], ao.n_ao)


def build_jk(eri: Packed, rho: np.ndarray):
    """J and K (with -1/2) from packed ERIs, f64 partials (integrals.py:199-218)."""
    n = eri.n_ao
    m = len(eri.values)
    nchunk = max(1, min((m + 65535) // 65536, 4096))
    Jp = np.zeros((nchunk, n, n))
    Kp = np.zeros((nchunk, n, n))
    if m:
        v = np.ascontiguousarray(eri.values, dtype=np.float64)
        r = np.ascontiguousarray(rho, dtype=np.float64)
        lib().orc_jk(ctypes.c_int64(m), _p(eri.i), _p(eri.j), _p(eri.k), _p(eri.l), _p(v), _p(r),
                     ctypes.c_int(n), ctypes.c_int(nchunk), _p(Jp), _p(Kp))
    J = Jp.sum(axis=0)
    K = -0.5 * Kp.sum(axis=0)
    return J.astype(rho.dtype), K.astype(rho.dtype)


def unpack(eri: Packed) -> np.ndarray:
    """Dense N^4 tensor with all images (integrals.py:221-238)."""
    n = eri.n_ao
    d = np.zeros((n, n, n, n))
    i, j, k, l = (x.astype(np.intp) for x in (eri.i, eri.j, eri.k, eri.l))
    v = eri.values.astype(float)
    for a, b, c, e in ((i, j, k, l), (j, i, k, l), (i, j, l, k), (j, i, l, k),
                       (k, l, i, j), (l, k, i, j), (k, l, j, i), (l, k, j, i)):
        d[a, b, c, e] = v
    return d


# ----------------------------------------------------------------------------- grid

LEB_DEG = {6: 3, 14: 5, 26: 7, 38: 9, 50: 11, 86: 15, 110: 17, 146: 19, 194: 23, 302: 29}
TA_XI = (0.8, 0.9, 1.8, 1.4, 1.3, 1.1, 0.9, 0.9, 0.9, 0.9)         # xc.py:37-39
BRAGG = (0.35, 0.31, 1.45, 1.05, 0.85, 0.70, 0.65, 0.60, 0.50, 0.38)  # xc.py:42-44
LEVELS = {0: (18, 20, (14, 26, 26, 14), (14, 26, 38, 14)),           # xc.py:50-55
          1: (18, 30, (14, 26, 50, 26), (26, 50, 86, 26)),
          2: (30, 45, (26, 50, 146, 86), (38, 86, 194, 110)),
          3: (50, 65, (38, 110, 302, 302), (50, 146, 302, 302))}


def radial(n, xi):
    """Gauss-Chebyshev-2 nodes under the Treutler-Ahlrichs M4 map, ascending r (xc.py:85-98)."""
    k = np.arange(1, n + 1)
    th = k * np.pi / (n + 1)
    x = np.cos(th)
    w = np.pi / (n + 1) * np.sin(th)
    c = xi / math.log(2.0)
    lg = np.log(2.0 / (1.0 - x))
    r = c * (1 + x) ** 0.6 * lg
    dr = c * (1 + x) ** 0.6 * (0.6 * lg / (1 + x) + 1.0 / (1.0 - x))
    return r[::-1], (w * dr)[::-1]


_LEB = {}


def lebedev(npts):
    if npts not in _LEB:
        pts, w = lebedev_rule(LEB_DEG[npts])
        _LEB[npts] = (np.ascontiguousarray(pts.T), w.copy())
    return _LEB[npts]


def build_grid(m: Mol, level=1):
    """Atom-centred pruned product grids with Becke weights (xc.py:123-162)."""
    nrh, nrx, sh, sx = LEVELS[level]
    P, W, O = [], [], []
    for ia, z in enumerate(m.Z):
        nr, sched = (nrh, sh) if z <= 2 else (nrx, sx)
        r, wr = radial(nr, TA_XI[z - 1])
        rb = BRAGG[z - 1] * ANG2BOHR
        for ir in range(nr):
            if r[ir] < 0.30 * rb:
                na = sched[0]
            elif r[ir] < 0.60 * rb:
                na = sched[1]
            elif r[ir] < max(3.0 * rb, 4.0):
                na = sched[2]
            else:
                na = sched[3]
            ap, aw = lebedev(na)
            P.append(m.pos[ia] + r[ir] * ap)
            W.append(wr[ir] * r[ir] ** 2 * aw)
            O.append(np.full(len(aw), ia, np.int32))
    pts = np.ascontiguousarray(np.vstack(P))
    w = np.concatenate(W)
    own = np.concatenate(O)
    nat = len(m.Z)
    if nat > 1:
        cen = np.ascontiguousarray(m.pos, dtype=float)
        d = np.linalg.norm(cen[:, None] - cen[None], axis=2)
        np.fill_diagonal(d, 1.0)
        inv = 1.0 / d
        np.fill_diagonal(inv, 0.0)
        inv = np.ascontiguousarray(inv)
        bw = np.empty(len(w))
        lib().orc_becke(ctypes.c_int64(len(w)), ctypes.c_int(nat), _p(cen), _p(inv), _p(pts),
                        _p(own), _p(bw))
        w = w * bw
    neg = w < 0
    if neg.any():
        if np.abs(w[neg]).max() > 1e-14:
            raise ValueError("negative quadrature weight beyond numerical noise")
        w = np.where(neg, 0.0, w)
    return pts, w


def eval_ao(ao: AO, pts: np.ndarray, dtype=np.float64):
    """phi and grad phi on the grid (xc.py:165-194)."""
    npts = len(pts)
    phi = np.zeros((npts, ao.n_ao), dtype)
    grad = np.zeros((3, npts, ao.n_ao), dtype)
    for s in range(ao.n_shells):
        l = int(ao.shell_l[s])
        o = int(ao.ao_offsets[s])
        p0 = int(ao.prim_start[s])
        ex = ao.prim_exp[p0:p0 + 3]
        rel = pts - ao.shell_center[s]
        r2 = np.einsum("pd,pd->p", rel, rel)
        eg = np.exp(-np.outer(r2, ex))
        for c, (lx, ly, lz) in enumerate(COMPS[l]):
            cf = ao.prim_coef[p0:p0 + 3, c]
            base = eg @ cf
            dbase = eg @ (cf * (-2.0 * ex))
            poly = rel[:, 0] ** lx * rel[:, 1] ** ly * rel[:, 2] ** lz
            phi[:, o + c] = poly * base
            for d, ld in enumerate((lx, ly, lz)):
                dp = 0.0
                if ld > 0:
                    dp = ld * rel[:, 0] ** (lx - (d == 0)) * rel[:, 1] ** (ly - (d == 1)) \
                        * rel[:, 2] ** (lz - (d == 2))
                grad[d, :, o + c] = dp * base + poly * rel[:, d] * dbase
    return phi, grad


# ----------------------------------------------------------------------------- functional

CX = 0.75 * (3.0 / math.pi) ** (1.0 / 3.0)        # xc.py:200-205
CXS = 1.5 * (3.0 / (4.0 * math.pi)) ** (1.0 / 3.0)
BETA = 0.0042
VA, VB, VC, VX0 = 0.0310907, 13.0720, 42.7198, -0.409286
LA, LB, LC, LD = 0.04918, 0.132, 0.2533, 0.349
CF = 0.3 * (3.0 * math.pi ** 2) ** (2.0 / 3.0)


def b3lyp(n_in, s_in):
    """0.08 LSDA + 0.72 B88 + 0.19 VWN-RPA + 0.81 LYP, closed shell, f64 (xc.py:277-306).

    Returns (exc per particle, vrho, vsigma), zero below the 1e-12 density floor.
    """
    n = np.maximum(np.asarray(n_in, float), 0.0)
    s = np.maximum(np.asarray(s_in, float), 0.0)
    live = n >= 1e-12
    exc, vr, vs = np.zeros(n.shape), np.zeros(n.shape), np.zeros(n.shape)
    if live.any():
        n_, s_ = n[live], s[live]
        # Slater (per particle) -- xc.py:208-211
        e_lda = -CX * np.cbrt(n_)
        f0, v0 = e_lda * n_, (4.0 / 3.0) * e_lda
        # Becke 88 on spin densities ns = n/2, sigma_s = sigma/4 -- xc.py:214-234
        ns = 0.5 * n_
        t = np.cbrt(ns)
        t4 = t ** 4
        x = np.sqrt(0.25 * s_) / t4
        ash = np.arcsinh(x)
        den = 1.0 + 6.0 * BETA * x * ash
        dden = 6.0 * BETA * (ash + x / np.sqrt(1.0 + x * x))
        g = CXS + BETA * x * x / den
        dg = BETA * (2.0 * x * den - x * x * dden) / (den * den)
        f1 = -2.0 * t4 * g
        v1 = -(4.0 / 3.0) * t * g + t4 * dg * (4.0 / 3.0) * x / ns
        w1 = 0.5 * (-BETA * (2.0 * den - x * dden) / (2.0 * den * den * t4))
        # VWN (RPA parametrisation, paramagnetic) -- xc.py:237-252
        rs = np.cbrt(3.0 / (4.0 * math.pi * n_))
        y = np.sqrt(rs)
        Xy = rs + VB * y + VC
        X0 = VX0 * VX0 + VB * VX0 + VC
        Q = math.sqrt(4.0 * VC - VB * VB)
        at = np.arctan(Q / (2.0 * y + VB))
        ec = VA * (np.log(y * y / Xy) + (2.0 * VB / Q) * at
                   - (VB * VX0 / X0) * (np.log((y - VX0) ** 2 / Xy) + (2.0 * (VB + 2.0 * VX0) / Q) * at))
        dec = VA * (2.0 / y - 2.0 * (y + VB) / Xy
                    - (VB * VX0 / X0) * (2.0 / (y - VX0) - 2.0 * (y + VB + VX0) / Xy))
        f2 = ec * n_
        v2 = ec - (rs / 3.0) * dec / (2.0 * y)
        # LYP closed-shell -- xc.py:255-274
        tt = n_ ** (-1.0 / 3.0)
        Xd = 1.0 + LD * tt
        om = tt ** 11 * np.exp(-LC * tt) / Xd
        dl = tt * (LC + LD / Xd)
        n143 = n_ ** 4 * np.cbrt(n_ * n_)
        f3 = -LA * n_ / Xd - LA * LB * om * CF * n143 + LA * LB * om * n_ * n_ * s_ * (3.0 + 7.0 * dl) / 72.0
        w3 = LA * LB * om * n_ * n_ * (3.0 + 7.0 * dl) / 72.0
        tp = -tt / (3.0 * n_)
        omp = om * tp * (11.0 / tt - LC - LD / Xd)
        dlp = tp * (LC + LD / Xd - LD * LD * tt / (Xd * Xd))
        v3 = (-LA / Xd + LA * n_ * LD * tp / (Xd * Xd)
              - LA * LB * CF * (omp * n143 + om * (14.0 / 3.0) * n143 / n_)
              + (LA * LB * s_ / 72.0) * (omp * n_ * n_ * (3.0 + 7.0 * dl)
                                         + 2.0 * n_ * om * (3.0 + 7.0 * dl) + 7.0 * om * n_ * n_ * dlp))
        ftot = 0.08 * f0 + 0.72 * f1 + 0.19 * f2 + 0.81 * f3
        exc[live] = ftot / n_
        vr[live] = 0.08 * v0 + 0.72 * v1 + 0.19 * v2 + 0.81 * v3
        vs[live] = 0.72 * w1 + 0.81 * w3
    if not (np.isfinite(exc).all() and np.isfinite(vr).all() and np.isfinite(vs).all()):
        raise ValueError("non-finite functional output")
    return exc, vr, vs


def xc_matrix(w_all, phi_all, grad_all, rho):
    """E_xc and V_xc over 8192-point batches, V accumulated in f64 (xc.py:320-350)."""
    dtype = phi_all.dtype
    n = phi_all.shape[1]
    V = np.zeros((n, n))
    e = 0.0
    npts = phi_all.shape[0]
    for lo in range(0, npts, 8192):
        hi = min(npts, lo + 8192)
        phi = phi_all[lo:hi]
        gp = grad_all[:, lo:hi, :]
        w = w_all[lo:hi].astype(dtype)
        t = phi @ rho
        dens = np.einsum("pi,pi->p", t, phi)
        gn = np.stack([2.0 * np.einsum("pi,pi->p", gp[d], t) for d in range(3)]).astype(dtype)
        sig = gn[0] ** 2 + gn[1] ** 2 + gn[2] ** 2
        exc, vr, vs = b3lyp(dens, sig)
        exc, vr, vs = exc.astype(dtype), vr.astype(dtype), vs.astype(dtype)
        e += float(np.sum(w_all[lo:hi] * dens.astype(float) * exc.astype(float)))
        wv = (0.5 * w * vr)[:, None] * phi
        ge = 2.0 * w * vs
        for d in range(3):
            wv += (ge * gn[d])[:, None] * gp[d]
        V += (phi.T @ wv).astype(float)
    V = V + V.T
    return e, V.astype(dtype)


# ----------------------------------------------------------------------------- SCF


def solve_roothaan(F, S):
    """Canonical orthogonalisation (drop s <= 1e-7) + eigh (scf.py:86-98)."""
    s, U = scipy.linalg.eigh(S)
    keep = s > 1e-7
    X = U[:, keep] / np.sqrt(s[keep])
    eps, Cp = scipy.linalg.eigh(X.T @ F @ X)
    return X @ Cp, eps


def diis_step(hist):
    """Pulay extrapolation with the cond(B) > 1e12 damped fallback (scf.py:101-132)."""
    if len(hist) == 1:
        return hist[0][0]
    m = len(hist)
    B = np.empty((m + 1, m + 1))
    B[-1, :] = 1.0
    B[:, -1] = 1.0
    B[-1, -1] = 0.0
    for a in range(m):
        ea = hist[a][1].astype(float).ravel()
        for b in range(a, m):
            B[a, b] = B[b, a] = ea @ hist[b][1].astype(float).ravel()
    rhs = np.zeros(m + 1)
    rhs[-1] = 1.0
    if np.linalg.cond(B) > 1e12:
        return (0.5 * hist[-1][0] + 0.5 * hist[-2][0]).astype(hist[-1][0].dtype)
    c = np.linalg.solve(B, rhs)[:m]
    out = np.zeros(hist[-1][0].shape)
    for a in range(m):
        out += c[a] * hist[a][0].astype(float)
    return out.astype(hist[-1][0].dtype)


@dataclass
class Result:
    E_total: float
    epsilon: np.ndarray
    C: np.ndarray
    n_occ: int
    components: dict
    history: list = field(default_factory=list)
    converged: bool = False
    iterations: int = 0
    n_ao: int = 0

    @property
    def homo(self):
        return float(self.epsilon[self.n_occ - 1])

    @property
    def lumo(self):
        return float(self.epsilon[self.n_occ])

    @property
    def gap_ev(self):
        return (self.lumo - self.homo) * HA2EV


def scf(m: Mol, precision="f64", max_iterations=50, convergence_std=0.01, grid_level=1,
        screen_eps=1e-12, diis_history=8, diis_start=3, damping=0.5) -> Result:
    """Restricted KS B3LYP SCF from the core guess (scf.py:139-210)."""
    dt = np.float32 if precision == "f32" else np.float64
    nocc = m.nelec // 2
    ao = expand(m)
    if nocc > ao.n_ao:
        raise ValueError("basis too small")
    S, T, V = one_electron(ao, m, dt)
    eri = eri_packed(ao, screen_eps, dt)
    pts, w = build_grid(m, grid_level)
    phi, grad = eval_ao(ao, pts, dt)
    enn = nuclear_repulsion(m)
    H = V + T
    C, eps = solve_roothaan(H, S)
    hist, comps, buf = [], {}, []
    rho_prev = None
    conv = False
    for it in range(max_iterations):
        co = C[:, :nocc]
        rho = (2.0 * co @ co.T).astype(dt)
        if rho_prev is not None and 0 < it < diis_start:
            rho = (damping * rho_prev + (1.0 - damping) * rho).astype(dt)
        rho_prev = rho
        J, K = build_jk(eri, rho)
        exc, Vxc = xc_matrix(w, phi, grad, rho)
        F = V + T + J + 0.20 * K + Vxc
        tr = lambda a, b: float(np.sum(a.astype(float) * b.astype(float)))
        comps = {"E_nn": enn, "E_core": tr(rho, H), "E_coulomb": 0.5 * tr(rho, J),
                 "E_exx": 0.5 * 0.20 * tr(rho, K), "E_xc": exc}
        hist.append(sum(comps.values()))
        err = F @ rho @ S - S @ rho @ F
        buf.append((F, err))
        if len(buf) > diis_history:
            buf.pop(0)
        Fu = diis_step(buf) if it + 1 >= diis_start else F
        C, eps = solve_roothaan(Fu, S)
        if len(hist) >= 5 and float(np.std(hist[-5:])) < convergence_std:
            conv = True
            break
    return Result(hist[-1], eps, C, nocc, comps, hist, conv, len(hist), ao.n_ao)
