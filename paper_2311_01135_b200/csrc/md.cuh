// McMurchie-Davidson integral math on fused S / L(sp) shells.
//
// Everything here is __host__ __device__ so tests/cpu_md_check.cpp can run the
// exact device arithmetic on the CPU against the oracle.  The scheme follows the
// reference's Hermite formulation (_kernels.py:48-141, 350-447): Boys F_m by a
// tabulated 7-term Taylor seed + downward recursion, Hermite Coulomb R_{tuv},
// and E^{ab}_{tuv} expansions — but on fused shells: an L shell's s and p
// components share their primitive Gaussian products, so one R table serves all
// (up to 256) component combinations of a quartet, and contraction coefficients
// (with K_ab) are folded into the primitive-pair records.
#pragma once
#include <math.h>
#include <stdint.h>

#ifndef HD
#define HD __host__ __device__ __forceinline__
#endif

namespace dftb {

#ifdef __CUDA_ARCH__
HD double drsqrt(double x) { return rsqrt(x); }
#else
inline double drsqrt(double x) { return 1.0 / sqrt(x); }
#endif

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi25 = 34.98683665524972;   // 2 * pi^2.5
constexpr double kHalfSqrtPi = 0.88622692545275801;  // sqrt(pi) / 2
constexpr int kBoysNcol = 16;
constexpr double kBoysStep = 0.1;
constexpr int kBoysNT = 431;
constexpr int kBoysLMax = 4;     // highest Hermite order of any integral here: (pp|pp), L = 4
// The device reads a per-order slice of the Boys table: slice L holds, for each T grid point,
// the 7 Taylor coefficients F_L .. F_{L+6} (plus one pad) in one 64-byte row, so a lookup is
// four aligned 16-byte loads of one row and a class of fixed L touches a 27.6 KB table (the
// full 431 x 16 table is 55 KB, and its 56-byte windows straddle 128-byte lines).
inline void boys_slices_host(const double *tab, double *sl) {
    for (int L = 0; L <= kBoysLMax; ++L)
        for (int it = 0; it < kBoysNT; ++it)
            for (int j = 0; j < 8; ++j)
                sl[((size_t)L * kBoysNT + it) * 8 + j] = j < 7 ? tab[it * kBoysNcol + L + j] : 0.0;
}

HD constexpr int nherm(int L) { return (L + 1) * (L + 2) * (L + 3) / 6; }
// flat index of Hermite (t,u,v): grouped by order s = t+u+v, then a = u+v, then v
HD constexpr int hidx(int t, int u, int v) {
    return (t + u + v) * (t + u + v + 1) * (t + u + v + 2) / 6 + (u + v) * (u + v + 1) / 2 + v;
}

// F_0..F_L(T); tab = the per-order slices of the 431 x 16 table of F_m at T = 0.1 k
// (boys_slices_host).  Mirrors _kernels.py:48-68.
// exp(-T) is evaluated once, before the branch: quartets of one warp mix small and large T,
// and with an exp in each branch a divergent warp paid for two (for T >= 700 exp(-T) is
// below 1e-304 and leaves the asymptotic recursion unchanged, as the former explicit zero did)
template <int L>
HD void boys(double T, double *F, const double *tab) {
    const double et = exp(-T);
    if (T > 42.95) {
        // sqrt(pi / T) / 2 and 1 / (2T) from one reciprocal square root
        const double rt = drsqrt(T);
        double f = kHalfSqrtPi * rt;
        double h = 0.5 * rt * rt;
        F[0] = f;
#pragma unroll
        for (int m = 0; m < L; ++m) F[m + 1] = ((2 * m + 1) * F[m] - et) * h;
    } else {
        int it = (int)(T * 10.0 + 0.5);
        double dT = T - it * kBoysStep;
        const double *row = tab + ((size_t)L * kBoysNT + it) * 8;
        double rw[8];
#ifdef __CUDA_ARCH__
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const double2 v = __ldg(reinterpret_cast<const double2 *>(row) + j);
            rw[2 * j] = v.x;
            rw[2 * j + 1] = v.y;
        }
#else
        for (int j = 0; j < 8; ++j) rw[j] = row[j];
#endif
        double acc = 0.0;
#pragma unroll
        for (int j = 6; j > 0; --j) acc = (acc + rw[j]) * (-dT) * (1.0 / j);
        F[L] = acc + rw[0];
#pragma unroll
        for (int m = L - 1; m >= 0; --m) F[m] = (2.0 * T * F[m + 1] + et) * (1.0 / (2 * m + 1));
    }
}

// R_{tuv} (order 0) for t+u+v <= L, scaled by `pref`; X,Y,Z = P - Q (or P - C).
template <int L>
HD void hermite_R(double T, double alpha, double X, double Y, double Z, double pref,
                  const double *tab, double *R) {
    double F[L + 1];
    boys<L>(T, F, tab);
    double Rl[L + 1][nherm(L)];
    double pw = pref, m2a = -2.0 * alpha;
#pragma unroll
    for (int n = 0; n <= L; ++n) {
        Rl[n][0] = pw * F[n];
        pw *= m2a;
    }
#pragma unroll
    for (int n = L - 1; n >= 0; --n) {
#pragma unroll
        for (int s = 1; s <= L - n; ++s) {
#pragma unroll
            for (int t = s; t >= 0; --t) {
#pragma unroll
                for (int u = s - t; u >= 0; --u) {
                    const int v = s - t - u;
                    double val;
                    if (t > 0) {
                        val = X * Rl[n + 1][hidx(t - 1, u, v)];
                        if (t > 1) val += (t - 1) * Rl[n + 1][hidx(t - 2, u, v)];
                    } else if (u > 0) {
                        val = Y * Rl[n + 1][hidx(t, u - 1, v)];
                        if (u > 1) val += (u - 1) * Rl[n + 1][hidx(t, u - 2, v)];
                    } else {
                        val = Z * Rl[n + 1][hidx(t, u, v - 1)];
                        if (v > 1) val += (v - 1) * Rl[n + 1][hidx(t, u, v - 2)];
                    }
                    Rl[n][hidx(t, u, v)] = val;
                }
            }
        }
    }
#pragma unroll
    for (int h = 0; h < nherm(L); ++h) R[h] = Rl[0][h];
}

// ---------------------------------------------------------------------------- pair data
// Primitive-pair record fields ([PP_FIELDS][NPP][n_pair] SoA, pair index fastest):
enum { PF_P = 0, PF_X, PF_Y, PF_Z, PF_H, PF_CSS, PF_CSP, PF_CPS, PF_CPP, PF_BOUND };

struct PPView {
    const double *pp;
    int64_t npair;
    HD double get(int f, int k, int64_t pair) const { return pp[((int64_t)f * 9 + k) * npair + pair]; }
};

// Shell component c: 0 = s, 1..3 = p_x, p_y, p_z.  l of component c along dim d:
HD constexpr int cl(int c, int d) { return c == d + 1 ? 1 : 0; }
HD constexpr int cidx(int ca, int cb) { return (ca > 0 ? 2 : 0) + (cb > 0 ? 1 : 0); }

// 1-D Hermite expansion of x_A^la x_B^lb (la, lb <= 1) around P: e[0..la+lb]
HD void e1d(int la, int lb, double pa, double pb, double h, double *e) {
    if (la == 0 && lb == 0) {
        e[0] = 1.0;
    } else if (la == 1 && lb == 0) {
        e[0] = pa; e[1] = h;
    } else if (la == 0 && lb == 1) {
        e[0] = pb; e[1] = h;
    } else {
        e[0] = pa * pb + h; e[1] = h * (pa + pb); e[2] = h * h;
    }
}

// ---------------------------------------------------------------------------- ERI quartet
// (ab|cd) for all bra components x ket components [KC0, KC0+NKS).  Kinds: 0 = S, 1 = L.
// out[bc][k] accumulates (caller zeroes).  prim_cut > 0 skips primitive quartets with
// pref * bound_ab * bound_cd < prim_cut (the reference's primitive screen, _kernels.py:376-377).
// V: bra primitive-pair records; VK: the ket's (any view with get(field, prim, pair); the
// device ERI kernel passes a per-thread shared-memory copy of its ket's nine records).
template <int KA, int KB, int KC, int KD, int KC0, int NKS, typename KV>
HD void eri_quartet_kv(const PPView &V, const KV &VK, int64_t Pp, int64_t Qp, const double *A,
                       const double *B, const double *C, const double *D, const double *tab,
                       double prim_cut, double (*out)[NKS]) {
    constexpr int NA = KA ? 4 : 1, NB = KB ? 4 : 1, ND = KD ? 4 : 1;
    constexpr int LB = KA + KB, LK = KC + KD, L = LB + LK;
    constexpr int NHB = nherm(LB);
    for (int ib = 0; ib < 9; ++ib) {
        const double p = V.get(PF_P, ib, Pp);
        const double Px = V.get(PF_X, ib, Pp), Py = V.get(PF_Y, ib, Pp), Pz = V.get(PF_Z, ib, Pp);
        const double hp = V.get(PF_H, ib, Pp);
        const double bb = V.get(PF_BOUND, ib, Pp);
        double W[NHB][NKS];
#pragma unroll
        for (int h = 0; h < NHB; ++h)
#pragma unroll
            for (int k = 0; k < NKS; ++k) W[h][k] = 0.0;
        for (int ik = 0; ik < 9; ++ik) {
            const double q = VK.get(PF_P, ik, Qp);
            const double hq = VK.get(PF_H, ik, Qp);
            const double r = drsqrt(p + q);
            const double pref = kTwoPi25 * (4.0 * hp * hq) * r;  // 2 pi^2.5 / (p q sqrt(p+q))
            if (prim_cut > 0.0 && pref * bb * VK.get(PF_BOUND, ik, Qp) < prim_cut) continue;
            const double Qx = VK.get(PF_X, ik, Qp), Qy = VK.get(PF_Y, ik, Qp), Qz = VK.get(PF_Z, ik, Qp);
            const double alpha = p * q * (r * r);
            const double X = Px - Qx, Y = Py - Qy, Z = Pz - Qz;
            double R[nherm(L)];
            hermite_R<L>(alpha * (X * X + Y * Y + Z * Z), alpha, X, Y, Z, pref, tab, R);
            double ck[4];
            ck[0] = VK.get(PF_CSS, ik, Qp);
            if (KC || KD) {
                ck[1] = VK.get(PF_CSP, ik, Qp);
                ck[2] = VK.get(PF_CPS, ik, Qp);
                ck[3] = VK.get(PF_CPP, ik, Qp);
            }
            const double QC[3] = {Qx - C[0], Qy - C[1], Qz - C[2]};
            const double QD[3] = {Qx - D[0], Qy - D[1], Qz - D[2]};
#pragma unroll
            for (int k = 0; k < NKS; ++k) {
                const int kc = KC0 + k;
                const int cc = kc / ND, cd = kc % ND;
                double fx[3], fy[3], fz[3];
                e1d(cl(cc, 0), cl(cd, 0), QC[0], QD[0], hq, fx);
                e1d(cl(cc, 1), cl(cd, 1), QC[1], QD[1], hq, fy);
                e1d(cl(cc, 2), cl(cd, 2), QC[2], QD[2], hq, fz);
                const int lx = cl(cc, 0) + cl(cd, 0), ly = cl(cc, 1) + cl(cd, 1), lz = cl(cc, 2) + cl(cd, 2);
                const double cc_ = ck[cidx(cc, cd)];
#pragma unroll
                for (int t = 0; t <= LB; ++t)
#pragma unroll
                    for (int u = 0; u <= LB - t; ++u)
#pragma unroll
                        for (int v = 0; v <= LB - t - u; ++v) {
                            double acc = 0.0;
#pragma unroll
                            for (int a = 0; a <= 2; ++a) {
                                if (a > lx) continue;
#pragma unroll
                                for (int b = 0; b <= 2; ++b) {
                                    if (b > ly) continue;
#pragma unroll
                                    for (int c = 0; c <= 2; ++c) {
                                        if (c > lz) continue;
                                        const double f = fx[a] * fy[b] * fz[c];
                                        const double rv = R[hidx(t + a, u + b, v + c)];
                                        acc += ((a + b + c) & 1) ? -f * rv : f * rv;
                                    }
                                }
                            }
                            W[hidx(t, u, v)][k] += cc_ * acc;
                        }
            }
        }
        // bra contraction for this bra primitive pair
        const double cb4[4] = {V.get(PF_CSS, ib, Pp), (KA || KB) ? V.get(PF_CSP, ib, Pp) : 0.0,
                               (KA || KB) ? V.get(PF_CPS, ib, Pp) : 0.0,
                               (KA || KB) ? V.get(PF_CPP, ib, Pp) : 0.0};
        const double PA[3] = {Px - A[0], Py - A[1], Pz - A[2]};
        const double PB[3] = {Px - B[0], Py - B[1], Pz - B[2]};
#pragma unroll
        for (int bc = 0; bc < NA * NB; ++bc) {
            const int ca = bc / NB, cb = bc % NB;
            double ex[3], ey[3], ez[3];
            e1d(cl(ca, 0), cl(cb, 0), PA[0], PB[0], hp, ex);
            e1d(cl(ca, 1), cl(cb, 1), PA[1], PB[1], hp, ey);
            e1d(cl(ca, 2), cl(cb, 2), PA[2], PB[2], hp, ez);
            const int lx = cl(ca, 0) + cl(cb, 0), ly = cl(ca, 1) + cl(cb, 1), lz = cl(ca, 2) + cl(cb, 2);
            const double c_ = cb4[cidx(ca, cb)];
#pragma unroll
            for (int k = 0; k < NKS; ++k) {
                double acc = 0.0;
#pragma unroll
                for (int t = 0; t <= 2; ++t) {
                    if (t > lx) continue;
#pragma unroll
                    for (int u = 0; u <= 2; ++u) {
                        if (u > ly) continue;
#pragma unroll
                        for (int v = 0; v <= 2; ++v) {
                            if (v > lz) continue;
                            acc += ex[t] * ey[u] * ez[v] * W[hidx(t, u, v)][k];
                        }
                    }
                }
                out[bc][k] += c_ * acc;
            }
        }
    }
}

template <int KA, int KB, int KC, int KD, int KC0, int NKS>
HD void eri_quartet(const PPView &V, int64_t Pp, int64_t Qp, const double *A, const double *B,
                    const double *C, const double *D, const double *tab, double prim_cut,
                    double (*out)[NKS]) {
    eri_quartet_kv<KA, KB, KC, KD, KC0, NKS>(V, V, Pp, Qp, A, B, C, D, tab, prim_cut, out);
}

// ---------------------------------------------------------------------------- one-electron
// 1-D Hermite tables E[i][j][t], i <= 1, j <= 3 (j up to lb+2 for the kinetic term).
HD void e1d_ext(double pa, double pb, double h, double E[2][4][5]) {
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 4; ++j)
            for (int t = 0; t < 5; ++t) E[i][j][t] = 0.0;
    E[0][0][0] = 1.0;
    for (int j = 1; j < 4; ++j)
        for (int t = 0; t <= j; ++t)
            E[0][j][t] = (t > 0 ? h * E[0][j - 1][t - 1] : 0.0) + pb * E[0][j - 1][t] +
                         (t + 1 <= j - 1 ? (t + 1) * E[0][j - 1][t + 1] : 0.0);
    for (int j = 0; j < 4; ++j)
        for (int t = 0; t <= j + 1; ++t)
            E[1][j][t] = (t > 0 ? h * E[0][j][t - 1] : 0.0) + pa * E[0][j][t] +
                         (t + 1 <= j ? (t + 1) * E[0][j][t + 1] : 0.0);
}

// S, T, V blocks for one fused shell pair (ka, kb kinds), shells with exps/cs/cp,
// centres A, B; nuclei (natom, xyz, Z).  out arrays [4][4].  Mirrors _kernels.py:229-343.
HD void onee_pair(int ka, int kb, const double *ea, const double *csa, const double *cpa,
                  const double *eb, const double *csb, const double *cpb, const double *A,
                  const double *B, int natom, const double *axyz, const int *az,
                  const double *tab, double S[4][4], double T[4][4], double Vm[4][4]) {
    const int na = ka ? 4 : 1, nb = kb ? 4 : 1;
    for (int x = 0; x < 4; ++x)
        for (int y = 0; y < 4; ++y) S[x][y] = T[x][y] = Vm[x][y] = 0.0;
    double rab2 = 0.0;
    for (int d = 0; d < 3; ++d) rab2 += (A[d] - B[d]) * (A[d] - B[d]);
    for (int i = 0; i < 3; ++i) {
        const double a = ea[i];
        for (int j = 0; j < 3; ++j) {
            const double b = eb[j], p = a + b, h = 0.5 / p;
            const double kab = exp(-(a * b / p) * rab2);
            double P[3], E[3][2][4][5];
            for (int d = 0; d < 3; ++d) {
                P[d] = (a * A[d] + b * B[d]) / p;
                e1d_ext(P[d] - A[d], P[d] - B[d], h, E[d]);
            }
            const double sq = sqrt(kPi / p), ov = sq * sq * sq;
            double cof[4][4];
            for (int ca = 0; ca < na; ++ca)
                for (int cb = 0; cb < nb; ++cb)
                    cof[ca][cb] = (ca ? cpa[i] : csa[i]) * (cb ? cpb[j] : csb[j]) * kab;
            for (int ca = 0; ca < na; ++ca)
                for (int cb = 0; cb < nb; ++cb) {
                    double s1[3], t1[3];
                    for (int d = 0; d < 3; ++d) {
                        const int li = cl(ca, d), lj = cl(cb, d);
                        s1[d] = E[d][li][lj][0];
                        double kk = -2.0 * b * b * E[d][li][lj + 2][0] + b * (2 * lj + 1) * s1[d];
                        // lj <= 1, so the (lj-2) term of the reference never contributes
                        t1[d] = kk;
                    }
                    S[ca][cb] += cof[ca][cb] * s1[0] * s1[1] * s1[2] * ov;
                    T[ca][cb] += cof[ca][cb] * (t1[0] * s1[1] * s1[2] + s1[0] * t1[1] * s1[2] +
                                                s1[0] * s1[1] * t1[2]) * ov;
                }
            const double pref0 = 2.0 * kPi / p;
            for (int c = 0; c < natom; ++c) {
                const double X = P[0] - axyz[3 * c], Y = P[1] - axyz[3 * c + 1], Z = P[2] - axyz[3 * c + 2];
                double R[nherm(2)];
                hermite_R<2>(p * (X * X + Y * Y + Z * Z), p, X, Y, Z, -az[c] * pref0, tab, R);
                for (int ca = 0; ca < na; ++ca)
                    for (int cb = 0; cb < nb; ++cb) {
                        const int lx = cl(ca, 0) + cl(cb, 0), ly = cl(ca, 1) + cl(cb, 1), lz = cl(ca, 2) + cl(cb, 2);
                        double acc = 0.0;
                        for (int t = 0; t <= lx; ++t)
                            for (int u = 0; u <= ly; ++u)
                                for (int v = 0; v <= lz; ++v)
                                    acc += E[0][cl(ca, 0)][cl(cb, 0)][t] * E[1][cl(ca, 1)][cl(cb, 1)][u] *
                                           E[2][cl(ca, 2)][cl(cb, 2)][v] * R[hidx(t, u, v)];
                        Vm[ca][cb] += cof[ca][cb] * acc;
                    }
            }
        }
    }
}

// Host-side Boys table (same construction on CPU and GPU): F_m(T) by the convergent series
// e^{-T} sum_k (2T)^k / ((2m+1)(2m+3)...(2m+2k+1)), all terms positive (no cancellation).
inline void boys_table_host(double *tab) {
    for (int it = 0; it < 431; ++it) {
        const double T = it * 0.1;
        for (int m = 0; m < kBoysNcol; ++m) {
            long double term = 1.0L / (2 * m + 1), sum = term;
            for (int k = 1; k < 400; ++k) {
                term *= (2.0L * T) / (2 * m + 2 * k + 1);
                sum += term;
                if (term < sum * 1e-21L) break;
            }
            tab[it * kBoysNcol + m] = (double)(expl(-(long double)T) * sum);
        }
    }
}

}  // namespace dftb
