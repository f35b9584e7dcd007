/*
 * ORACLE — test infrastructure only.  Not part of the product path.
 *
 * Plain-C restatement of the reference's numba kernels
 * (/root/reference/pkg/src/deskdft/_kernels.py) so that the CPU oracle
 * (oracle/port.py) runs at numba-like speed without numba.  Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline leg may load this.
 *
 * Every routine cites the reference function it restates.  The arithmetic is
 * the reference's McMurchie-Davidson scheme on split S/P shells, so values
 * agree with the reference to rounding (checked against tests/golden/).
 *
 * Build: see oracle/Makefile (gcc -O2 -fopenmp -shared).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXL 2
#define BOYS_NCOL 16       /* m = 0 .. 4*MAXL + 7  (_kernels.py:32-45) */
#define BOYS_STEP 0.1
#define BOYS_TMAX 43.0
#define BOYS_TAYLOR 7
#define ELEN 45            /* (i*3+j)*5+t, i,j<=2, t<=4   (_kernels.py:72-74) */
#define OE_SJ 5
#define OE_ST 7
#define OE_LEN (3 * OE_SJ * OE_ST)

static const int NCOMP[3] = {1, 3, 6};
static const int COMP_OFF[3] = {0, 1, 4};
static const int CLX[10] = {0, 1, 0, 0, 2, 1, 1, 0, 0, 0};
static const int CLY[10] = {0, 0, 1, 0, 0, 1, 0, 2, 1, 0};
static const int CLZ[10] = {0, 0, 0, 1, 0, 0, 1, 0, 1, 2};

/* Boys F_0..F_mmax(T): tabulated Taylor seed at the top order, downward
 * recursion; asymptotic form beyond the table.  _kernels.py:48-68 */
static void boys(int mmax, double T, double *F, const double *tab) {
    if (T > BOYS_TMAX - 0.5 * BOYS_STEP) {
        F[0] = 0.5 * sqrt(M_PI / T);
        double et = T < 700.0 ? exp(-T) : 0.0;
        double h = 0.5 / T;
        for (int m = 0; m < mmax; ++m) F[m + 1] = ((2 * m + 1) * F[m] - et) * h;
        return;
    }
    int it = (int)(T / BOYS_STEP + 0.5);
    double dT = T - it * BOYS_STEP;
    const double *row = tab + (size_t)it * BOYS_NCOL;
    double acc = 0.0;
    for (int j = BOYS_TAYLOR - 1; j > 0; --j) acc = (acc + row[mmax + j]) * (-dT) / j;
    F[mmax] = acc + row[mmax];
    double et = exp(-T);
    for (int m = mmax - 1; m >= 0; --m) F[m] = (2.0 * T * F[m + 1] + et) / (2 * m + 1);
}

/* 1-D Hermite expansion table, layout (i*sj+j)*st+t.  _kernels.py:79-105 and
 * the extended-j variant :203-226 (same recurrence, wider j). */
static void hermite_1d(int la, int lb, double p, double pa, double pb, double k0,
                       double *E, int sj, int st, int len) {
    memset(E, 0, sizeof(double) * len);
    E[0] = k0;
    double h = 0.5 / p;
    for (int j = 0; j <= lb; ++j)
        for (int i = 0; i <= la; ++i) {
            if (i == 0 && j == 0) continue;
            int src;
            double x;
            if (i > 0) { src = ((i - 1) * sj + j) * st; x = pa; }
            else       { src = (i * sj + (j - 1)) * st; x = pb; }
            int dst = (i * sj + j) * st;
            int nmax = i + j;
            for (int t = 0; t <= nmax; ++t) {
                double v = x * E[src + t];
                if (t > 0) v += h * E[src + t - 1];
                if (t + 1 <= nmax - 1) v += (t + 1) * E[src + t + 1];
                E[dst + t] = v;
            }
        }
}

/* Hermite Coulomb integrals R_{tuv}, order 0, for t+u+v <= L.  The scratch
 * holds all auxiliary orders n; layout n*s3 + t*nn + u*n1 + v.
 * _kernels.py:108-141 */
static void hermite_R(int L, double alpha, double x, double y, double z, double T,
                      double *F, double *R, const double *tab) {
    boys(L, T, F, tab);
    int n1 = L + 1, nn = n1 * n1, s3 = n1 * nn;
    double pw = 1.0, m2a = -2.0 * alpha;
    for (int n = 0; n < n1; ++n) { R[n * s3] = pw * F[n]; pw *= m2a; }
    for (int v = 1; v < n1; ++v)
        for (int n = 0; n < n1 - v; ++n) {
            double val = z * R[(n + 1) * s3 + (v - 1)];
            if (v > 1) val += (v - 1) * R[(n + 1) * s3 + (v - 2)];
            R[n * s3 + v] = val;
        }
    for (int u = 1; u < n1; ++u)
        for (int v = 0; v < n1 - u; ++v)
            for (int n = 0; n < n1 - u - v; ++n) {
                double val = y * R[(n + 1) * s3 + (u - 1) * n1 + v];
                if (u > 1) val += (u - 1) * R[(n + 1) * s3 + (u - 2) * n1 + v];
                R[n * s3 + u * n1 + v] = val;
            }
    for (int t = 1; t < n1; ++t)
        for (int u = 0; u < n1 - t; ++u)
            for (int v = 0; v < n1 - t - u; ++v)
                for (int n = 0; n < n1 - t - u - v; ++n) {
                    double val = x * R[(n + 1) * s3 + (t - 1) * nn + u * n1 + v];
                    if (t > 1) val += (t - 1) * R[(n + 1) * s3 + (t - 2) * nn + u * n1 + v];
                    R[n * s3 + t * nn + u * n1 + v] = val;
                }
}

static double absmax6(const double *c) {
    double m = 0.0;
    for (int k = 0; k < 6; ++k) if (fabs(c[k]) > m) m = fabs(c[k]);
    return m;
}

/* Primitive-pair tables per shell pair.  _kernels.py:148-190 */
void orc_pair_tables(int npair, const int *pair_si, const int *pair_sj,
                     const int *shell_l, const double *shell_center,
                     const int *prim_start, const int *prim_count,
                     const double *prim_coef, const double *prim_exp,
                     const int64_t *pair_pp_start, double *pp_p, double *pp_P,
                     int *pp_ia, int *pp_ib, double *pp_cmaxK, double *pp_E) {
    for (int ip = 0; ip < npair; ++ip) {
        int si = pair_si[ip], sj = pair_sj[ip];
        const double *A = shell_center + 3 * si, *B = shell_center + 3 * sj;
        double rab2 = 0.0;
        for (int d = 0; d < 3; ++d) rab2 += (A[d] - B[d]) * (A[d] - B[d]);
        int64_t idx = pair_pp_start[ip];
        for (int pa = prim_start[si]; pa < prim_start[si] + prim_count[si]; ++pa) {
            double a = prim_exp[pa], ca = absmax6(prim_coef + 6 * pa);
            for (int pb = prim_start[sj]; pb < prim_start[sj] + prim_count[sj]; ++pb, ++idx) {
                double b = prim_exp[pb], p = a + b;
                double kab = exp(-(a * b / p) * rab2);
                pp_p[idx] = p;
                for (int d = 0; d < 3; ++d) pp_P[3 * idx + d] = (a * A[d] + b * B[d]) / p;
                pp_ia[idx] = pa;
                pp_ib[idx] = pb;
                pp_cmaxK[idx] = ca * absmax6(prim_coef + 6 * pb) * kab;
                for (int d = 0; d < 3; ++d)
                    hermite_1d(shell_l[si], shell_l[sj], p, pp_P[3 * idx + d] - A[d],
                               pp_P[3 * idx + d] - B[d], d > 0 ? 1.0 : kab,
                               pp_E + (idx * 3 + d) * ELEN, 3, 5, ELEN);
            }
        }
    }
}

/* S, T, V over shell pairs.  _kernels.py:229-343 */
void orc_one_electron(int npair, const int *pair_si, const int *pair_sj,
                      const int *shell_l, const double *shell_center, const int *ao_offsets,
                      const int *prim_start, const int *prim_count, const double *prim_exp,
                      const double *prim_coef, int natom, const double *atom_xyz,
                      const double *atom_z, int n_ao, double *S, double *Tm, double *V,
                      const double *tab) {
#pragma omp parallel for schedule(dynamic)
    for (int ip = 0; ip < npair; ++ip) {
        double Ex[OE_LEN], Ey[OE_LEN], Ez[OE_LEN], Fb[2 * MAXL + 1];
        double Rb[(2 * MAXL + 1) * (2 * MAXL + 1) * (2 * MAXL + 1) * (2 * MAXL + 1)];
        double sb[36], tb[36], vb[36];
        int si = pair_si[ip], sj = pair_sj[ip], la = shell_l[si], lb = shell_l[sj];
        int na = NCOMP[la], nb = NCOMP[lb];
        const double *A = shell_center + 3 * si, *B = shell_center + 3 * sj;
        double rab2 = 0.0;
        for (int d = 0; d < 3; ++d) rab2 += (A[d] - B[d]) * (A[d] - B[d]);
        memset(sb, 0, sizeof sb); memset(tb, 0, sizeof tb); memset(vb, 0, sizeof vb);
        int L = la + lb, n1 = L + 1, nn = n1 * n1;
        for (int pa = prim_start[si]; pa < prim_start[si] + prim_count[si]; ++pa) {
            double a = prim_exp[pa];
            for (int pb = prim_start[sj]; pb < prim_start[sj] + prim_count[sj]; ++pb) {
                double b = prim_exp[pb], p = a + b;
                double kab = exp(-(a * b / p) * rab2);
                double P[3];
                for (int d = 0; d < 3; ++d) P[d] = (a * A[d] + b * B[d]) / p;
                hermite_1d(la, lb + 2, p, P[0] - A[0], P[0] - B[0], kab, Ex, OE_SJ, OE_ST, OE_LEN);
                hermite_1d(la, lb + 2, p, P[1] - A[1], P[1] - B[1], 1.0, Ey, OE_SJ, OE_ST, OE_LEN);
                hermite_1d(la, lb + 2, p, P[2] - A[2], P[2] - B[2], 1.0, Ez, OE_SJ, OE_ST, OE_LEN);
                double sqp = sqrt(M_PI / p), ov = sqp * sqp * sqp;
                for (int ca = 0; ca < na; ++ca) {
                    int ax = CLX[COMP_OFF[la] + ca], ay = CLY[COMP_OFF[la] + ca], az = CLZ[COMP_OFF[la] + ca];
                    for (int cb = 0; cb < nb; ++cb) {
                        int bx = CLX[COMP_OFF[lb] + cb], by = CLY[COMP_OFF[lb] + cb], bz = CLZ[COMP_OFF[lb] + cb];
                        double cc = prim_coef[6 * pa + ca] * prim_coef[6 * pb + cb];
                        double ex0 = Ex[(ax * OE_SJ + bx) * OE_ST];
                        double ey0 = Ey[(ay * OE_SJ + by) * OE_ST];
                        double ez0 = Ez[(az * OE_SJ + bz) * OE_ST];
                        sb[ca * 6 + cb] += cc * ex0 * ey0 * ez0 * ov;
                        double kx = -2.0 * b * b * Ex[(ax * OE_SJ + bx + 2) * OE_ST] + b * (2 * bx + 1) * ex0;
                        if (bx >= 2) kx -= 0.5 * bx * (bx - 1) * Ex[(ax * OE_SJ + bx - 2) * OE_ST];
                        double ky = -2.0 * b * b * Ey[(ay * OE_SJ + by + 2) * OE_ST] + b * (2 * by + 1) * ey0;
                        if (by >= 2) ky -= 0.5 * by * (by - 1) * Ey[(ay * OE_SJ + by - 2) * OE_ST];
                        double kz = -2.0 * b * b * Ez[(az * OE_SJ + bz + 2) * OE_ST] + b * (2 * bz + 1) * ez0;
                        if (bz >= 2) kz -= 0.5 * bz * (bz - 1) * Ez[(az * OE_SJ + bz - 2) * OE_ST];
                        tb[ca * 6 + cb] += cc * (kx * ey0 * ez0 + ex0 * ky * ez0 + ex0 * ey0 * kz) * ov;
                    }
                }
                double pref = 2.0 * M_PI / p;
                for (int ia = 0; ia < natom; ++ia) {
                    double xp = P[0] - atom_xyz[3 * ia], yp = P[1] - atom_xyz[3 * ia + 1],
                           zp = P[2] - atom_xyz[3 * ia + 2];
                    hermite_R(L, p, xp, yp, zp, p * (xp * xp + yp * yp + zp * zp), Fb, Rb, tab);
                    double zc = -atom_z[ia] * pref;
                    for (int ca = 0; ca < na; ++ca) {
                        int ax = CLX[COMP_OFF[la] + ca], ay = CLY[COMP_OFF[la] + ca], az = CLZ[COMP_OFF[la] + ca];
                        for (int cb = 0; cb < nb; ++cb) {
                            int bx = CLX[COMP_OFF[lb] + cb], by = CLY[COMP_OFF[lb] + cb], bz = CLZ[COMP_OFF[lb] + cb];
                            double cc = prim_coef[6 * pa + ca] * prim_coef[6 * pb + cb];
                            double s = 0.0;
                            for (int t = 0; t <= ax + bx; ++t) {
                                double e1 = Ex[(ax * OE_SJ + bx) * OE_ST + t];
                                if (e1 == 0.0) continue;
                                for (int u = 0; u <= ay + by; ++u) {
                                    double e2 = Ey[(ay * OE_SJ + by) * OE_ST + u];
                                    if (e2 == 0.0) continue;
                                    for (int v = 0; v <= az + bz; ++v) {
                                        double e3 = Ez[(az * OE_SJ + bz) * OE_ST + v];
                                        if (e3 == 0.0) continue;
                                        s += e1 * e2 * e3 * Rb[t * nn + u * n1 + v];
                                    }
                                }
                            }
                            vb[ca * 6 + cb] += zc * cc * s;
                        }
                    }
                }
            }
        }
        int oa = ao_offsets[si], ob = ao_offsets[sj];
        for (int ca = 0; ca < na; ++ca)
            for (int cb = 0; cb < nb; ++cb) {
                size_t x = (size_t)(oa + ca) * n_ao + ob + cb, y = (size_t)(ob + cb) * n_ao + oa + ca;
                S[x] = S[y] = sb[ca * 6 + cb];
                Tm[x] = Tm[y] = tb[ca * 6 + cb];
                V[x] = V[y] = vb[ca * 6 + cb];
            }
    }
}

/* Contracted (ab|cd) block, block[(ca*nb+cb)*36 + cc*nd+cd].  _kernels.py:350-447 */
static void quartet_block(int la, int lb, int lc, int ld, int64_t sa0, int san, int64_t sb0, int sbn,
                          const double *pp_p, const double *pp_P, const int *pp_ia, const int *pp_ib,
                          const double *pp_cmaxK, const double *pp_E, const double *prim_coef,
                          double *F, double *R, const double *tab, double *block, double prim_cut,
                          int f32acc) {
    int na = NCOMP[la], nb = NCOMP[lb], nc = NCOMP[lc], nd = NCOMP[ld];
    for (int q = 0; q < 36 * 36; ++q) block[q] = 0.0;
    int L = la + lb + lc + ld, n1 = L + 1, nn = n1 * n1;
    for (int64_t ppa = sa0; ppa < sa0 + san; ++ppa) {
        double p = pp_p[ppa];
        for (int64_t ppb = sb0; ppb < sb0 + sbn; ++ppb) {
            double q = pp_p[ppb], pq = p * q, sq = sqrt(p + q);
            double pref = 2.0 * pow(M_PI, 2.5) / (pq * sq);
            if (prim_cut > 0.0 && pref * pp_cmaxK[ppa] * pp_cmaxK[ppb] < prim_cut) continue;
            double alpha = pq / (p + q);
            double x = pp_P[3 * ppa] - pp_P[3 * ppb], y = pp_P[3 * ppa + 1] - pp_P[3 * ppb + 1],
                   z = pp_P[3 * ppa + 2] - pp_P[3 * ppb + 2];
            hermite_R(L, alpha, x, y, z, alpha * (x * x + y * y + z * z), F, R, tab);
            int ia = pp_ia[ppa], ib = pp_ib[ppa], ic = pp_ia[ppb], id = pp_ib[ppb];
            const double *Ea = pp_E + ppa * 3 * ELEN, *Eb = pp_E + ppb * 3 * ELEN;
            for (int ca = 0; ca < na; ++ca) {
                int ax = CLX[COMP_OFF[la] + ca], ay = CLY[COMP_OFF[la] + ca], az = CLZ[COMP_OFF[la] + ca];
                for (int cb = 0; cb < nb; ++cb) {
                    int bx = CLX[COMP_OFF[lb] + cb], by = CLY[COMP_OFF[lb] + cb], bz = CLZ[COMP_OFF[lb] + cb];
                    double cab = prim_coef[6 * ia + ca] * prim_coef[6 * ib + cb];
                    if (cab == 0.0) continue;
                    int exi = (ax * 3 + bx) * 5, eyi = (ay * 3 + by) * 5, ezi = (az * 3 + bz) * 5;
                    for (int cc = 0; cc < nc; ++cc) {
                        int cx = CLX[COMP_OFF[lc] + cc], cy = CLY[COMP_OFF[lc] + cc], cz = CLZ[COMP_OFF[lc] + cc];
                        for (int cd = 0; cd < nd; ++cd) {
                            int dx = CLX[COMP_OFF[ld] + cd], dy = CLY[COMP_OFF[ld] + cd], dz = CLZ[COMP_OFF[ld] + cd];
                            double ccd = prim_coef[6 * ic + cc] * prim_coef[6 * id + cd];
                            if (ccd == 0.0) continue;
                            int fxi = (cx * 3 + dx) * 5, fyi = (cy * 3 + dy) * 5, fzi = (cz * 3 + dz) * 5;
                            double s = 0.0;
                            for (int t = 0; t <= ax + bx; ++t) {
                                double e1 = Ea[exi + t];
                                if (e1 == 0.0) continue;
                                for (int u = 0; u <= ay + by; ++u) {
                                    double e2 = e1 * Ea[ELEN + eyi + u];
                                    if (e2 == 0.0) continue;
                                    for (int v = 0; v <= az + bz; ++v) {
                                        double e3 = e2 * Ea[2 * ELEN + ezi + v];
                                        if (e3 == 0.0) continue;
                                        double inner = 0.0;
                                        for (int tau = 0; tau <= cx + dx; ++tau) {
                                            double f1 = Eb[fxi + tau];
                                            if (f1 == 0.0) continue;
                                            double g1 = (tau & 1) ? -f1 : f1;
                                            for (int nu = 0; nu <= cy + dy; ++nu) {
                                                double f2 = g1 * Eb[ELEN + fyi + nu];
                                                if (f2 == 0.0) continue;
                                                double g2 = (nu & 1) ? -f2 : f2;
                                                for (int ph = 0; ph <= cz + dz; ++ph) {
                                                    double f3 = Eb[2 * ELEN + fzi + ph];
                                                    if (f3 == 0.0) continue;
                                                    double g3 = (ph & 1) ? -f3 : f3;
                                                    inner += g2 * g3 * R[(t + tau) * nn + (u + nu) * n1 + (v + ph)];
                                                }
                                            }
                                        }
                                        s += e3 * inner;
                                    }
                                }
                            }
                            double *dst = block + (ca * nb + cb) * 36 + cc * nd + cd;
                            /* f32 working dtype: the reference's block is a float32 array,
                             * so every primitive contribution is rounded on accumulation */
                            *dst = f32acc ? (double)(float)(*dst + pref * cab * ccd * s)
                                          : *dst + pref * cab * ccd * s;
                        }
                    }
                }
            }
        }
    }
}

#define RSCR ((4 * MAXL + 1) * (4 * MAXL + 1) * (4 * MAXL + 1) * (4 * MAXL + 1))

/* Schwarz diagonals (ab|ab): q_ao (sqrt, AO-pair triangle) and q_pair (max).
 * _kernels.py:450-488 */
void orc_schwarz(int npair, const int *pair_si, const int *pair_sj, const int64_t *pp_start,
                 const int *pp_count, const int *shell_l, const int *ao_offsets, const double *pp_p,
                 const double *pp_P, const int *pp_ia, const int *pp_ib, const double *pp_cmaxK,
                 const double *pp_E, const double *prim_coef, const double *tab, double *q_pair,
                 double *q_ao) {
#pragma omp parallel
    {
        double *block = malloc(sizeof(double) * 36 * 36);
        double *R = malloc(sizeof(double) * RSCR);
        double F[4 * MAXL + 1];
#pragma omp for schedule(dynamic)
        for (int ip = 0; ip < npair; ++ip) {
            int si = pair_si[ip], sj = pair_sj[ip], la = shell_l[si], lb = shell_l[sj];
            quartet_block(la, lb, la, lb, pp_start[ip], pp_count[ip], pp_start[ip], pp_count[ip],
                          pp_p, pp_P, pp_ia, pp_ib, pp_cmaxK, pp_E, prim_coef, F, R, tab, block, 0.0, 0);
            double qmax = 0.0;
            int nb = NCOMP[lb];
            for (int ca = 0; ca < NCOMP[la]; ++ca)
                for (int cb = 0; cb < nb; ++cb) {
                    double v = block[(ca * nb + cb) * 36 + ca * nb + cb];
                    v = v < 0.0 ? 0.0 : sqrt(v);
                    int i = ao_offsets[si] + ca, j = ao_offsets[sj] + cb;
                    if (i < j) { int t = i; i = j; j = t; }
                    q_ao[(int64_t)i * (i + 1) / 2 + j] = v;
                    if (v > qmax) qmax = v;
                }
            q_pair[ip] = qmax;
        }
        free(block);
        free(R);
    }
}

/* Canonical AO quartets surviving the AO-level screen, per shell quartet.
 * _kernels.py:491-533 */
void orc_count(int64_t nq, const int *quart_a, const int *quart_b, const int *pair_si,
               const int *pair_sj, const int *shell_l, const int *ao_offsets, const double *q_ao,
               double eps, int64_t *counts) {
#pragma omp parallel for schedule(static)
    for (int64_t iq = 0; iq < nq; ++iq) {
        int pa = quart_a[iq], pb = quart_b[iq];
        int s1 = pair_si[pa], s2 = pair_sj[pa], s3 = pair_si[pb], s4 = pair_sj[pb];
        int64_t cnt = 0;
        for (int c1 = 0; c1 < NCOMP[shell_l[s1]]; ++c1) {
            int i = ao_offsets[s1] + c1;
            for (int c2 = 0; c2 < NCOMP[shell_l[s2]]; ++c2) {
                int j = ao_offsets[s2] + c2;
                if (j > i) continue;
                int64_t ij = (int64_t)i * (i + 1) / 2 + j;
                for (int c3 = 0; c3 < NCOMP[shell_l[s3]]; ++c3) {
                    int k = ao_offsets[s3] + c3;
                    for (int c4 = 0; c4 < NCOMP[shell_l[s4]]; ++c4) {
                        int l = ao_offsets[s4] + c4;
                        if (l > k) continue;
                        int64_t kl = (int64_t)k * (k + 1) / 2 + l;
                        if (pa == pb && kl > ij) continue;
                        if (eps > 0.0 && q_ao[ij] * q_ao[kl] < eps) continue;
                        ++cnt;
                    }
                }
            }
        }
        counts[iq] = cnt;
    }
}

/* ERI values + canonical indices + degeneracy into preallocated slots.
 * _kernels.py:536-619 (values accumulated in f64 and stored as f64 here; the
 * Python side casts to the working dtype exactly like the reference's f32
 * block store, which rounds the contracted value once). */
void orc_fill(int64_t nq, const int *quart_a, const int *quart_b, const int64_t *offsets,
              const int *pair_si, const int *pair_sj, const int64_t *pp_start, const int *pp_count,
              const int *shell_l, const int *ao_offsets, const double *pp_p, const double *pp_P,
              const int *pp_ia, const int *pp_ib, const double *pp_cmaxK, const double *pp_E,
              const double *prim_coef, const double *tab, const double *q_ao, double eps,
              int f32acc, uint16_t *oi, uint16_t *oj, uint16_t *ok, uint16_t *ol, double *ov,
              uint8_t *odeg) {
    double prim_cut = 0.001 * eps;
#pragma omp parallel
    {
        double *block = malloc(sizeof(double) * 36 * 36);
        double *R = malloc(sizeof(double) * RSCR);
        double F[4 * MAXL + 1];
#pragma omp for schedule(dynamic, 64)
        for (int64_t iq = 0; iq < nq; ++iq) {
            int pa = quart_a[iq], pb = quart_b[iq];
            int s1 = pair_si[pa], s2 = pair_sj[pa], s3 = pair_si[pb], s4 = pair_sj[pb];
            int l1 = shell_l[s1], l2 = shell_l[s2], l3 = shell_l[s3], l4 = shell_l[s4];
            quartet_block(l1, l2, l3, l4, pp_start[pa], pp_count[pa], pp_start[pb], pp_count[pb],
                          pp_p, pp_P, pp_ia, pp_ib, pp_cmaxK, pp_E, prim_coef, F, R, tab, block,
                          prim_cut, f32acc);
            int64_t pos = offsets[iq];
            int n2 = NCOMP[l2], n4 = NCOMP[l4];
            for (int c1 = 0; c1 < NCOMP[l1]; ++c1) {
                int i = ao_offsets[s1] + c1;
                for (int c2 = 0; c2 < n2; ++c2) {
                    int j = ao_offsets[s2] + c2;
                    if (j > i) continue;
                    int64_t ij = (int64_t)i * (i + 1) / 2 + j;
                    for (int c3 = 0; c3 < NCOMP[l3]; ++c3) {
                        int k = ao_offsets[s3] + c3;
                        for (int c4 = 0; c4 < n4; ++c4) {
                            int l = ao_offsets[s4] + c4;
                            if (l > k) continue;
                            int64_t kl = (int64_t)k * (k + 1) / 2 + l;
                            if (pa == pb && kl > ij) continue;
                            if (eps > 0.0 && q_ao[ij] * q_ao[kl] < eps) continue;
                            int a = i, b = j, c = k, d = l;
                            if (kl > ij) { a = k; b = l; c = i; d = j; }
                            oi[pos] = (uint16_t)a; oj[pos] = (uint16_t)b;
                            ok[pos] = (uint16_t)c; ol[pos] = (uint16_t)d;
                            ov[pos] = block[(c1 * n2 + c2) * 36 + c3 * n4 + c4];
                            odeg[pos] = (uint8_t)((a != b ? 2 : 1) * (c != d ? 2 : 1) *
                                                  ((a != c || b != d) ? 2 : 1));
                            ++pos;
                        }
                    }
                }
            }
        }
        free(block);
        free(R);
    }
}

/* Becke cell weight of each point for its owning atom.  _kernels.py:622-647 */
void orc_becke(int64_t npts, int natom, const double *centers, const double *inv_rij,
               const double *points, const int *owner, double *out) {
#pragma omp parallel
    {
        double *d = malloc(sizeof(double) * (natom > 0 ? natom : 1));
#pragma omp for schedule(static)
        for (int64_t p = 0; p < npts; ++p) {
            for (int a = 0; a < natom; ++a) {
                double dx = points[3 * p] - centers[3 * a], dy = points[3 * p + 1] - centers[3 * a + 1],
                       dz = points[3 * p + 2] - centers[3 * a + 2];
                d[a] = sqrt(dx * dx + dy * dy + dz * dz);
            }
            double tot = 0.0, pown = 0.0;
            for (int a = 0; a < natom; ++a) {
                double cell = 1.0;
                for (int b = 0; b < natom; ++b) {
                    if (b == a) continue;
                    double f = (d[a] - d[b]) * inv_rij[a * natom + b];
                    for (int it = 0; it < 3; ++it) f = 1.5 * f - 0.5 * f * f * f;
                    cell *= 0.5 * (1.0 - f);
                }
                tot += cell;
                if (a == owner[p]) pown = cell;
            }
            out[p] = tot > 0.0 ? pown / tot : 0.0;
        }
        free(d);
    }
}

/* Per-chunk J/K partials (f64) from canonical packed entries, every distinct
 * symmetric image visited once.  _kernels.py:650-693 */
void orc_jk(int64_t m, const uint16_t *ei, const uint16_t *ej, const uint16_t *ek,
            const uint16_t *el, const double *ev, const double *rho, int n, int nchunk,
            double *Jp, double *Kp) {
    int64_t per = (m + nchunk - 1) / nchunk;
#pragma omp parallel for schedule(static)
    for (int ic = 0; ic < nchunk; ++ic) {
        double *J = Jp + (size_t)ic * n * n, *K = Kp + (size_t)ic * n * n;
        int64_t lo = ic * per, hi = lo + per < m ? lo + per : m;
        for (int64_t e = lo; e < hi; ++e) {
            int i = ei[e], j = ej[e], k = ek[e], l = el[e];
            double v = ev[e];
            int dij = i == j, dkl = k == l, dp = (i == k) && (j == l);
#define RH(a, b) rho[(size_t)(a) * n + (b)]
#define JJ(a, b) J[(size_t)(a) * n + (b)]
#define KK(a, b) K[(size_t)(a) * n + (b)]
            JJ(k, l) += v * RH(i, j);
            KK(i, l) += v * RH(j, k);
            if (!dij) { JJ(k, l) += v * RH(j, i); KK(j, l) += v * RH(i, k); }
            if (!dkl) { JJ(l, k) += v * RH(i, j); KK(i, k) += v * RH(j, l); }
            if (!dij && !dkl) { JJ(l, k) += v * RH(j, i); KK(j, k) += v * RH(i, l); }
            if (!dp) {
                JJ(i, j) += v * RH(k, l);
                KK(k, j) += v * RH(l, i);
                if (!dkl) { JJ(i, j) += v * RH(l, k); KK(l, j) += v * RH(k, i); }
                if (!dij) { JJ(j, i) += v * RH(k, l); KK(k, i) += v * RH(l, j); }
                if (!dij && !dkl) { JJ(j, i) += v * RH(l, k); KK(l, i) += v * RH(k, j); }
            }
#undef RH
#undef JJ
#undef KK
        }
    }
}
