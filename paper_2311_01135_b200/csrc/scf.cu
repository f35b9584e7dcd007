// Device-resident SCF loop body: one CTA per molecule, everything in f64.
//
// Reference: deskdft.scf (scf.py:68-210): density (:68-74), fock (:77-83),
// solve_roothaan (:86-98), diis_step (:101-132), the loop body (:168-200).
//
// k_orth   : eigh(S) by parallel cyclic Jacobi, keep s > 1e-7, X = U/sqrt(s)  (once)
// k_post   : reduce J/K/Vxc partials -> F -> energies -> DIIS error + B row ->
//            Pulay extrapolation (with the cond(B) > 1e12 damped fallback) ->
//            X^T F X -> Jacobi (warm-started from the previous eigenvectors) ->
//            C = X C' -> rho = 2 C_occ C_occ^T (+ pre-DIIS damping) -> convergence.
// No host round trip: the host enqueues J/K, XC and post for every iteration.
#include "common.cuh"
#include <math_constants.h>

namespace dftb {

constexpr int SCF_THREADS = 256;
constexpr int KP = 32;  // GEMM K-panel
constexpr int GST = (KP * NMAX + 255) / 256;   // staging elements per thread per operand (256 threads)

struct Arena {
    int nm;             // arena dimension (largest N of the batch) and staging leading dim
    double *A, *B;      // nm*nm each (B >= 2*KP*64): Jacobi's matrix and eigenvectors
    double *sa, *sb;    // GEMM staging [KP][64] each, inside B (no GEMM reads or writes B)
    double *cs, *sn;    // rotations of the current step [NPH] (2*NPH allocated)
    int *pp, *qq;       // rotation pairs [2][NPH]
    int *perm;          // [NMAX]
    double *dv;         // [NMAX]
    double *Bs;         // [hs*hs] DIIS system (hs = history + 1)
    double *cf;         // [hs]
    double *red;        // [64]
    double *scal;       // [16] scalars broadcast
    long long *dbgp;    // JAC_PHASES builds: [2] angle / apply cycles (else null)
};

constexpr int NPH = NMAX / 2 + 1;

HD size_t arena_b(int nm) { return (size_t)(nm * nm > 2 * KP * 64 ? nm * nm : 2 * KP * 64); }

// hs: the largest bordered DIIS system (diis_history + 1; 10 for kernels without DIIS)
__device__ __forceinline__ Arena carve(unsigned char *base, int nm, int hs = 10) {
    Arena a;
    a.nm = nm;
    double *p = (double *)base;
    a.A = p; p += nm * nm;
    a.B = p; p += arena_b(nm);
    a.sa = a.B;
    a.sb = a.B + KP * 64;
    a.cs = p; p += 2 * NPH;
    a.sn = p; p += 2 * NPH;
    a.dv = p; p += NMAX;
    a.Bs = p; p += hs * hs > 32 ? hs * hs : 32;     // also the Lanczos coefficients (2 x 16)
    a.cf = p; p += hs;
    a.red = p; p += 64;
    a.scal = p; p += 16;
    a.dbgp = nullptr;
    int *q = (int *)p;
    a.pp = q; q += 2 * NPH;
    a.qq = q; q += 2 * NPH;
    a.perm = q; q += NMAX;
    return a;
}

size_t scf_smem_bytes(int nm, int hs = 10) {
    return sizeof(double) * ((size_t)nm * nm + arena_b(nm) + 4 * NPH + NMAX + (size_t)(hs * hs > 32 ? hs * hs : 32) +
                             hs + 64 + 16) +
           sizeof(int) * (4 * NPH + NMAX);
}

// C (M x N, ldc) = alpha * op(A) op(B) + beta * C ; op(A) is M x K, op(B) is K x N.
// Operands may live in global or shared memory; M, N <= NMAX.  The output is computed in
// 64 x 64 blocks (one for M, N <= 64): 16 x 16 threads with 4 x 4 register tiles, K in
// panels of KP staged zero-padded into ar.sa / ar.sb ([KP][64] each), so the inner loop has
// no bounds tests.  C must not alias A or B (blocks are written as they finish).
__device__ void cta_gemm_ffma(double *C, int ldc, const double *A, int lda, bool tA, const double *B, int ldb,
                              bool tB, int M, int N, int K, double alpha, double beta, const Arena &ar) {
    const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
    double *const sa = ar.sa, *const sb = ar.sb;
    constexpr int SU = KP * 64 / SCF_THREADS;           // staged elements per thread per operand
    for (int i0 = 0; i0 < M; i0 += 64)
        for (int j0 = 0; j0 < N; j0 += 64) {
            double acc[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
            for (int k0 = 0; k0 < K; k0 += KP) {
                const int kn = min(KP, K - k0);
                double v[SU];
#pragma unroll
                for (int u = 0; u < SU; ++u) {
                    const int t = tid + u * SCF_THREADS;
                    int kk, i;
                    if (tA) { kk = t >> 6; i = t & 63; } else { i = t / KP; kk = t - i * KP; }
                    const int gi = i0 + i;
                    v[u] = (kk < kn && gi < M) ? (tA ? A[(int64_t)(k0 + kk) * lda + gi]
                                                     : A[(int64_t)gi * lda + k0 + kk]) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < SU; ++u) {
                    const int t = tid + u * SCF_THREADS;
                    int kk, i;
                    if (tA) { kk = t >> 6; i = t & 63; } else { i = t / KP; kk = t - i * KP; }
                    sa[kk * 64 + i] = v[u];
                }
#pragma unroll
                for (int u = 0; u < SU; ++u) {
                    const int t = tid + u * SCF_THREADS;
                    int kk, j;
                    if (!tB) { kk = t >> 6; j = t & 63; } else { j = t / KP; kk = t - j * KP; }
                    const int gj = j0 + j;
                    v[u] = (kk < kn && gj < N) ? (tB ? B[(int64_t)gj * ldb + k0 + kk]
                                                     : B[(int64_t)(k0 + kk) * ldb + gj]) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < SU; ++u) {
                    const int t = tid + u * SCF_THREADS;
                    int kk, j;
                    if (!tB) { kk = t >> 6; j = t & 63; } else { j = t / KP; kk = t - j * KP; }
                    sb[kk * 64 + j] = v[u];
                }
                __syncthreads();
#pragma unroll 4
                for (int kk = 0; kk < kn; ++kk) {
                    double av[4], bv[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) av[a] = sa[kk * 64 + ty + 16 * a];
#pragma unroll
                    for (int c = 0; c < 4; ++c) bv[c] = sb[kk * 64 + tx + 16 * c];
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc[a][c] = fma(av[a], bv[c], acc[a][c]);
                }
                __syncthreads();
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int i = i0 + ty + 16 * a, j = j0 + tx + 16 * c;
                    if (i < M && j < N) {
                        double x = alpha * acc[a][c];
                        if (beta != 0.0) x += beta * C[(int64_t)i * ldc + j];
                        C[(int64_t)i * ldc + j] = x;
                    }
                }
        }
    __syncthreads();
}

// FP64 tensor cores (mma.sync m8n8k4 .f64, DMMA): 256 FMAs per warp instruction at the FP64
// peak (tools/probe/dmma_probe: 37 TFLOP/s with 4 warps x 4 chains per SM, 26-cycle latency)
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

// The same product on the FP64 tensor cores: warp w owns an RW x CW block of 8 x 8 output tiles
// (rows RW (w / 2).., columns CW (w % 2)..), K in steps of 4; fragments read in place (global or
// shared) with zero padding past M, N, K: A fragment element (i0 + g, k0 + q) of op(A), B
// fragment element (k0 + q, j0 + g) of op(B), accumulator elements (i0 + g, j0 + 2q + e).
template <int RW, int CW>
__device__ void cta_gemm_dmma_t(double *C, int ldc, const double *A, int lda, bool tA, const double *B, int ldb,
                                bool tB, int M, int N, int K, double alpha, double beta) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const int r0 = RW * (warp >> 1), c0 = CW * (warp & 1);
    double acc[RW][CW][2];
#pragma unroll
    for (int a = 0; a < RW; ++a)
#pragma unroll
        for (int c = 0; c < CW; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
    const bool any = 8 * r0 < M && 8 * c0 < N;          // warp-uniform
    if (any) {
#pragma unroll 2
        for (int k0 = 0; k0 < K; k0 += 4) {
            const int kk = k0 + q;
            const bool kv = kk < K;
            double fa[RW], fb[CW];
#pragma unroll
            for (int a = 0; a < RW; ++a) {
                const int i = 8 * (r0 + a) + g;
                fa[a] = (kv && i < M) ? (tA ? A[(int64_t)kk * lda + i] : A[(int64_t)i * lda + kk]) : 0.0;
            }
#pragma unroll
            for (int c = 0; c < CW; ++c) {
                const int j = 8 * (c0 + c) + g;
                fb[c] = (kv && j < N) ? (tB ? B[(int64_t)j * ldb + kk] : B[(int64_t)kk * ldb + j]) : 0.0;
            }
#pragma unroll
            for (int a = 0; a < RW; ++a)
#pragma unroll
                for (int c = 0; c < CW; ++c) dmma884(acc[a][c], fa[a], fb[c]);
        }
    }
    __syncthreads();                                     // every operand read before C is written
#pragma unroll
    for (int a = 0; a < RW; ++a)
#pragma unroll
        for (int c = 0; c < CW; ++c)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = 8 * (r0 + a) + g, j = 8 * (c0 + c) + 2 * q + e;
                if (i < M && j < N) {
                    double x = alpha * acc[a][c][e];
                    if (beta != 0.0) x += beta * C[(int64_t)i * ldc + j];
                    C[(int64_t)i * ldc + j] = x;
                }
            }
    __syncthreads();
}

#ifndef GEMM_DMMA
#define GEMM_DMMA 1    // the post kernel's GEMMs on the FP64 tensor cores
#endif
__device__ __forceinline__ void cta_gemm(double *C, int ldc, const double *A, int lda, bool tA, const double *B,
                                         int ldb, bool tB, int M, int N, int K, double alpha, double beta,
                                         const Arena &ar) {
    if (GEMM_DMMA) {
        static_assert(SCF_THREADS == 256, "eight warps: a 4 x 2 grid of tile blocks");
        __syncthreads();                                 // operands written by the caller
        if (M <= 64 && N <= 64) cta_gemm_dmma_t<2, 4>(C, ldc, A, lda, tA, B, ldb, tB, M, N, K, alpha, beta);
        else cta_gemm_dmma_t<3, 6>(C, ldc, A, lda, tA, B, ldb, tB, M, N, K, alpha, beta);
    } else {
        cta_gemm_ffma(C, ldc, A, lda, tA, B, ldb, tB, M, N, K, alpha, beta, ar);
    }
}

// Cyclic Jacobi, round-robin (circle) pairing: n/2 disjoint rotations per step,
// applied at once as J^T A J on 2x2 blocks (rows of pair k1 x columns of pair k2), in
// place: the blocks partition A, so every element is read and written by exactly one
// thread.  V <- V J in place, V stored transposed (V^T, eigenvector k in row k).  Lane l of every warp owns the column pairs l and l + 32
// (their rotations stay in registers for the whole step); warps walk the row pairs with
// broadcast parameters (measured: the post kernel's Roothaan phase -22% against one task
// list over all threads with per-task parameter loads).  A step is two CTA phases: the pair owners compute the step's
// angles from A, then every thread applies them.  In-place A (instead of a second
// buffer) keeps the arena at two n x n matrices, which fits two post CTAs per SM for the
// benchmark's AO counts (N <= 80) instead of one.
// Returns A (diagonal on exit); *nsweeps = sweeps.
constexpr int JAC_NW = SCF_THREADS / 32;
static_assert(NPH <= 64, "two column pairs per lane");

__device__ __forceinline__ void jac_pair(int k, int r, int n2, int &p, int &q) {
    if (k == 0) { p = r; q = n2 - 1; }
    else { p = (r + k) % (n2 - 1); q = (r - k + n2 - 1) % (n2 - 1); }
    if (p > q) { int t = p; p = q; q = t; }
}

// tan of the annihilating angle, t = sign(y) x / (|y| + sqrt(y^2 + x^2)) with y = aqq - app,
// x = 2 apq (= sign(th) / (|th| + sqrt(th^2 + 1)), th = y / x, with one division instead of
// two: the angle step is a serial f64 chain that the whole CTA waits for)
__device__ __forceinline__ void jac_angle(double app, double aqq, double apq, double &c, double &s) {
    c = 1.0;
    s = 0.0;
    if (fabs(apq) > 1e-300 && fabs(apq) > 1e-17 * (fabs(app) + fabs(aqq))) {
        const double y = aqq - app, x = 2.0 * apq;
        const double t = (y >= 0.0 ? x : -x) / (fabs(y) + sqrt(fma(y, y, x * x)));
        c = rsqrt(fma(t, t, 1.0));
        s = t * c;
    }
}

__device__ double *cta_jacobi(double *A, double *V, int n, const Arena &ar, int *nsweeps,
                              int max_sweeps = 30, double tol = 1e-13) {
    const int tid = threadIdx.x, nt = SCF_THREADS;
    const int n2 = n + (n & 1), np = n2 / 2, R = n2 - 1;
    const int kr = tid, lane = tid & 31, wid = tid >> 5;
    const bool rot_owner = tid < np;
    const double *cs = ar.cs, *sn = ar.sn;
    const int *pp = ar.pp, *qq = ar.qq;
    int sweeps = 0;
    for (int g = 0;; ++g) {
        const int r = g % R;
        if (r == 0) {   // convergence: off-diagonal max (elements above 1e-15 sqrt|a_pp a_qq|) vs diagonal max
            double off = 0.0, dg = 0.0;
            for (int t = tid; t < n * n; t += nt) {
                const int p = t / n, q = t - p * n;
                const double a = A[t];
                if (q > p) {
                    if (a * a > 1e-30 * fabs(A[p * n + p] * A[q * n + q])) off = fmax(off, fabs(a));   // no sqrt
                } else if (q == p) {
                    dg = fmax(dg, fabs(a));
                }
            }
            block_max2(off, dg, ar.red);
            if (off <= tol * dg || off < 1e-300 || sweeps >= max_sweeps) break;
            ++sweeps;
        }
#ifdef JAC_PHASES
        long long jt0 = clock64();
#endif
        if (rot_owner) {   // this step's angles from the current A
            int p, q;
            jac_pair(kr, r, n2, p, q);
            double c = 1.0, s1 = 0.0;
            if (q < n) jac_angle(A[p * n + p], A[q * n + q], A[p * n + q], c, s1);
            ar.cs[kr] = c; ar.sn[kr] = s1; ar.pp[kr] = p; ar.qq[kr] = q;
        }
        __syncthreads();
#ifdef JAC_PHASES
        long long jt1 = clock64();
#endif
        // apply: lane l owns the column pairs v = l, l + 32 (parameters in registers); the
        // warps walk the row pairs u (broadcast parameters) and then the rows of V
        {
            double cvj[2], svj[2];
            int pvj[2], qvj[2];
            bool okj[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int v = lane + 32 * j;
                okj[j] = v < np;
                const int vv = okj[j] ? v : 0;
                cvj[j] = cs[vv]; svj[j] = sn[vv]; pvj[j] = pp[vv]; qvj[j] = qq[vv];
            }
            for (int u = wid; u < np; u += JAC_NW) {
                const double c1 = cs[u], s1 = sn[u];
                const int p1 = pp[u], q1 = qq[u];
                const bool hq1 = q1 < n;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    if (!okj[j]) continue;
                    const double c2 = cvj[j], s2 = svj[j];
                    const int p2 = pvj[j], q2 = qvj[j];
                    const bool hq2 = q2 < n;
                    const double xpp = A[p1 * n + p2];
                    const double xpq = hq2 ? A[p1 * n + q2] : 0.0;
                    const double xqp = hq1 ? A[q1 * n + p2] : 0.0;
                    const double xqq = (hq1 && hq2) ? A[q1 * n + q2] : 0.0;
                    const double ypp = c1 * xpp - s1 * xqp, yqp = s1 * xpp + c1 * xqp;
                    const double ypq = c1 * xpq - s1 * xqq, yqq = s1 * xpq + c1 * xqq;
                    A[p1 * n + p2] = c2 * ypp - s2 * ypq;
                    if (hq2) A[p1 * n + q2] = s2 * ypp + c2 * ypq;
                    if (hq1) A[q1 * n + p2] = c2 * yqp - s2 * yqq;
                    if (hq1 && hq2) A[q1 * n + q2] = s2 * yqp + c2 * yqq;
                }
            }
            // V is stored transposed (row k = eigenvector k): rotating eigenvectors p, q is a
            // contiguous, conflict-free row operation; one warp per pair, lanes over components
            for (int k = wid; k < np; k += JAC_NW) {
                const double sv = sn[k];
                if (sv == 0.0) continue;
                const double cv = cs[k];
                double *vp_row = V + pp[k] * n, *vq_row = V + qq[k] * n;
                for (int row = lane; row < n; row += 32) {
                    const double vp = vp_row[row], vq = vq_row[row];
                    vp_row[row] = cv * vp - sv * vq;
                    vq_row[row] = sv * vp + cv * vq;
                }
            }
        }
        __syncthreads();
#ifdef JAC_PHASES
        if (tid == 0 && ar.dbgp) { ar.dbgp[0] += jt1 - jt0; ar.dbgp[1] += clock64() - jt1; }
#endif
    }
    *nsweeps = sweeps;
    return A;
}

// Eigenvalues of a small symmetric matrix (n <= 9: the bordered DIIS system) by the same
// cyclic Jacobi as cta_jacobi (same pairing, angles and block updates, so A is bitwise the
// same), run by warp 0 alone with warp barriers and without eigenvectors: the CTA-wide
// version paid two CTA barriers per step for 25 block updates.  Callers __syncthreads after.
__device__ void warp_jacobi_eigs(double *A, int n, const Arena &ar, double tol = 1e-13, int max_sweeps = 30) {
    const int lane = threadIdx.x & 31;
    const int n2 = n + (n & 1), np = n2 / 2, R = n2 - 1;
    int sweeps = 0;
    for (int g = 0;; ++g) {
        const int r = g % R;
        if (r == 0) {
            double off = 0.0, dg = 0.0;
            for (int t = lane; t < n * n; t += 32) {
                const int p = t / n, q = t - p * n;
                const double a = fabs(A[t]);
                if (q > p) {
                    if (a > 1e-15 * sqrt(fabs(A[p * n + p] * A[q * n + q]))) off = fmax(off, a);
                } else if (q == p) {
                    dg = fmax(dg, a);
                }
            }
            off = warp_max(off);
            dg = warp_max(dg);
            if (off <= tol * dg || off < 1e-300 || sweeps >= max_sweeps) break;
            ++sweeps;
        }
        for (int kr = lane; kr < np; kr += 32) {
            int p, q;
            jac_pair(kr, r, n2, p, q);
            double c = 1.0, s1 = 0.0;
            if (q < n) jac_angle(A[p * n + p], A[q * n + q], A[p * n + q], c, s1);
            ar.cs[kr] = c; ar.sn[kr] = s1; ar.pp[kr] = p; ar.qq[kr] = q;
        }
        __syncwarp();
        // every 2 x 2 block (u, v) reads and writes only its own four elements
        for (int uv = lane; uv < np * np; uv += 32) {
            const int u = uv / np, v = uv % np;
            const double s1 = ar.sn[u], s2 = ar.sn[v], c1 = ar.cs[u], c2 = ar.cs[v];
            const int p1 = ar.pp[u], q1 = ar.qq[u], p2 = ar.pp[v], q2 = ar.qq[v];
            const bool hq1 = q1 < n, hq2 = q2 < n;
            const double xpp = A[p1 * n + p2];
            const double xpq = hq2 ? A[p1 * n + q2] : 0.0;
            const double xqp = hq1 ? A[q1 * n + p2] : 0.0;
            const double xqq = (hq1 && hq2) ? A[q1 * n + q2] : 0.0;
            const double ypp = c1 * xpp - s1 * xqp, yqp = s1 * xpp + c1 * xqp;
            const double ypq = c1 * xpq - s1 * xqq, yqq = s1 * xpq + c1 * xqq;
            A[p1 * n + p2] = c2 * ypp - s2 * ypq;
            if (hq2) A[p1 * n + q2] = s2 * ypp + c2 * ypq;
            if (hq1) A[q1 * n + p2] = c2 * yqp - s2 * yqq;
            if (hq1 && hq2) A[q1 * n + q2] = s2 * yqp + c2 * yqq;
        }
        __syncwarp();
    }
}

// ascending order of diag(A) -> ar.perm (rank of each original index), stable by index
__device__ void sort_dv(int n, const Arena &ar);
__device__ void sort_eigs(const double *A, int n, const Arena &ar) {
    for (int i = threadIdx.x; i < n; i += SCF_THREADS) ar.dv[i] = A[i * n + i];
    __syncthreads();
    sort_dv(n, ar);
}

// ar.perm = ascending rank of ar.dv (ties by index)
__device__ void sort_dv(int n, const Arena &ar) {
    for (int i = threadIdx.x; i < n; i += SCF_THREADS) {
        const double d = ar.dv[i];
        int r = 0;
        for (int j = 0; j < n; ++j) {
            const double e = ar.dv[j];
            r += (e < d) || (e == d && j < i);
        }
        ar.perm[i] = r;
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------- purification
// Density projector without an eigendecomposition: the SCF needs the orbitals only to form
// rho = 2 C_occ C_occ^T (scf.py:68-74), i.e. the spectral projector of F' = X^T F X onto its
// n_occ lowest eigenvectors, and the eigenvalues only after the last iteration (scf.py:202-210).
// Trace-correcting purification (Niklasson, Phys. Rev. B 66, 155115 (2002)) builds that
// projector from matrix squares alone: X0 = (hi I - F') / (hi - lo) maps the spectrum (inside
// the Gershgorin bounds [lo, hi]) into [0, 1] with the occupied levels on top, and each step
// replaces X by X^2 or 2X - X^2 - whichever trace lands closer to n_occ - which drives the
// n_occ highest eigenvalues of X to 1 and the rest to 0 with the eigenvectors unchanged.  It
// converges quadratically once the HOMO-LUMO gap is resolved; we stop one step after the
// idempotency error tr(X - X^2) = sum l(1 - l) falls below 1e-11, i.e. at round-off
// (|l(1 - l)| < 1e-22).  One symmetric square per step (upper 4 x 4 tiles, Y in B) and two
// CTA barriers: ~20-30 steps against the 3-10 Jacobi sweeps of N - 1 rotation steps each.
// Returns false (the caller then diagonalises) if it has not converged after TC2_MAX steps,
// e.g. for a vanishing gap, where the projector is not defined by the spectrum alone.
constexpr int TC2_MAX = 100;
#ifndef TC2_UNR
#define TC2_UNR 2      // unroll of the squaring's l loop (post 0.663 -> 0.644 ms; 4: 0.649)
#endif
constexpr int kTc2Unr = TC2_UNR;

// Extreme-eigenvalue bounds of the symmetric M x M matrix A (shared memory) from LZ_STEPS
// Lanczos steps (start vector (1, 1.01, 1.02, ...), no reorthogonalisation: lost orthogonality
// only duplicates converged extreme Ritz values): [theta_min - beta_K - m, theta_max + beta_K + m],
// beta_K the last Lanczos coefficient (the norm of the factorisation's residual, the Zhou-Saad
// bound) and m = 1% of the Ritz width.  Multisection instead of a serial bisection: the f64
// divisions of 100 Sturm sequences on one thread cost more than ten purification steps.  The Gershgorin bounds (F' spans about 4x its spectrum
// for these molecules: [-55, 36] vs [-24.4, 0.6] Ha) cost the purification ~40% more steps; if
// a bound were ever too tight the purification's convergence test fails and the caller
// diagonalises.  Ritz values of the K x K tridiagonal by Sturm multisection (warps 0 / 1).
constexpr int LZ_STEPS = 16;

__device__ int sturm_count(const double *al, const double *be, int K, double x) {
    // number of eigenvalues of the tridiagonal (al, be) below x
    int c = 0;
    double d = 1.0;
    for (int k = 0; k < K; ++k) {
        d = al[k] - x - (k ? be[k - 1] * be[k - 1] / d : 0.0);
        if (d == 0.0) d = -1e-300;
        c += d < 0.0;
    }
    return c;
}

// CTA sum with one barrier: warp partials into one of two alternating halves of red (a half is
// rewritten only two reductions later, after every thread has read it), then every thread adds
// the partials itself in the same order
__device__ __forceinline__ double cta_sum1(double v, double *red, int &par) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    double *r = red + (par ? 32 : 0);
    par ^= 1;
    if (lane == 0) r[w] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < SCF_THREADS / 32; ++k) t += r[k];
    return t;
}

__device__ void lanczos_bounds(const double *A, int M, const Arena &ar, double *lo, double *hi) {
    const int tid = threadIdx.x, nt = SCF_THREADS;
    double *al = ar.Bs, *be = ar.Bs + LZ_STEPS;        // alpha, beta (Bs >= 32 doubles)
    double *v = ar.B, *vp = ar.B + NMAX, *w = ar.B + 2 * NMAX;   // B is free here (Y comes later)
    int par = 0;
    double nrm = 0.0;
    for (int i = tid; i < M; i += nt) {
        const double x = 1.0 + 0.01 * i;
        vp[i] = 0.0;
        nrm += x * x;
    }
    nrm = cta_sum1(nrm, ar.red, par);
    const double inv = 1.0 / sqrt(nrm);
    for (int i = tid; i < M; i += nt) v[i] = (1.0 + 0.01 * i) * inv;
    __syncthreads();
    int K = 0;
    double bprev = 0.0;
    const int part = tid & 3;
    for (int k = 0; k < LZ_STEPS && k < M; ++k) {
        // w = A v: four threads per row, interleaved columns, combined by shuffles
        double a = 0.0;
        for (int r = tid >> 2; r < ((M + 63) & ~63); r += nt / 4) {
            double s = 0.0;
            if (r < M)
                for (int j = part; j < M; j += 4) s = fma(A[r * M + j], v[j], s);
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            if (r < M && part == 0) {
                w[r] = s;
                a += s * v[r];
            }
        }
        a = cta_sum1(a, ar.red, par);                  // also orders the w writes
        double b2 = 0.0;
        for (int i = tid; i < M; i += nt) {
            const double x = w[i] - a * v[i] - bprev * vp[i];
            w[i] = x;
            b2 += x * x;
        }
        b2 = cta_sum1(b2, ar.red, par);
        const double bk = sqrt(b2);
        if (tid == 0) { al[k] = a; be[k] = bk; }
        K = k + 1;
        bprev = bk;
        if (bk < 1e-12 * fabs(a) + 1e-300) break;     // invariant subspace: Ritz values exact
        for (int i = tid; i < M; i += nt) {            // each thread rewrites only its own i
            vp[i] = v[i];
            v[i] = w[i] / bk;
        }
        __syncthreads();
    }
    __syncthreads();
    // extreme Ritz values: warp 0 the smallest, warp 1 the largest, by 32-way multisection of
    // the tridiagonal's Gershgorin interval (Sturm counts at 32 points per round, 4 rounds:
    // width / 2^20, far below the margins added below)
    if (tid < 64) {
        const int lane = tid & 31, wk = tid >> 5;
        double g0 = 1e300, g1 = -1e300;
        for (int k = 0; k < K; ++k) {
            const double r = (k ? fabs(be[k - 1]) : 0.0) + (k + 1 < K ? fabs(be[k]) : 0.0);
            g0 = fmin(g0, al[k] - r);
            g1 = fmax(g1, al[k] + r);
        }
        const int target = wk == 0 ? 1 : K;            // count below x reaches 1 / K
        double x0 = g0, x1 = g1;
        for (int round = 0; round < 4; ++round) {
            const double h = (x1 - x0) / 33.0;
            const double x = x0 + h * (lane + 1);
            const unsigned ge = __ballot_sync(0xffffffffu, sturm_count(al, be, K, x) >= target);
            // the count is monotone in x: the first lane reaching the target brackets the root
            const int f = ge ? __ffs(ge) - 1 : 32;
            const double nx0 = f == 0 ? x0 : x0 + h * f, nx1 = f == 32 ? x1 : x0 + h * (f + 1);
            x0 = nx0;
            x1 = nx1;
        }
        if (lane == 0) ar.scal[4 + wk] = wk == 0 ? x0 : x1;
    }
    __syncthreads();
    const double tmin = ar.scal[4], tmax = ar.scal[5], m = 0.01 * (tmax - tmin) + fabs(bprev);
    *lo = tmin - m;
    *hi = tmax + m;
    __syncthreads();
}

#ifndef TC2_DMMA
#define TC2_DMMA 1     // purification squarings on the FP64 tensor cores
#endif
// Y = X X for symmetric X (M x M, shared memory, row stride M) over the full square of 8 x 8
// output tiles: warp w owns an RW x CW block of tiles (rows RW (w / 2).., columns CW (w % 2)..),
// so per K step of 4 it loads RW + CW fragments (the B fragment of column tile t is, X being
// symmetric, the A fragment of row tile t: X[8t + g][k + q]) for RW * CW independent MMA
// chains.  Zero-padded past M.  The diagonal goes to ar.dv.
template <int RW, int CW>
__device__ void cta_square_dmma_t(const double *X, double *Y, int M, const Arena &ar) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const int r0 = RW * (warp >> 1), c0 = CW * (warp & 1);
    double acc[RW][CW][2];
#pragma unroll
    for (int a = 0; a < RW; ++a)
#pragma unroll
        for (int c = 0; c < CW; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
#pragma unroll 2
    for (int k0 = 0; k0 < M; k0 += 4) {
        const int kk = k0 + q;
        const bool kv = kk < M;
        double fa[RW], fb[CW];
#pragma unroll
        for (int a = 0; a < RW; ++a) {
            const int r = 8 * (r0 + a) + g;
            fa[a] = (kv && r < M) ? X[r * M + kk] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < CW; ++c) {
            const int r = 8 * (c0 + c) + g;
            fb[c] = (kv && r < M) ? X[r * M + kk] : 0.0;
        }
#pragma unroll
        for (int a = 0; a < RW; ++a)
#pragma unroll
            for (int c = 0; c < CW; ++c) dmma884(acc[a][c], fa[a], fb[c]);
    }
#pragma unroll
    for (int a = 0; a < RW; ++a)
#pragma unroll
        for (int c = 0; c < CW; ++c)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = 8 * (r0 + a) + g, j = 8 * (c0 + c) + 2 * q + e;
                if (i < M && j < M) {
                    Y[i * M + j] = acc[a][c][e];
                    if (i == j) ar.dv[i] = acc[a][c][e];
                }
            }
}

__device__ __forceinline__ void cta_square_dmma(const double *X, double *Y, int M, const Arena &ar) {
    static_assert(SCF_THREADS == 256, "eight warps: a 4 x 2 grid of tile blocks");
    if (M <= 64) cta_square_dmma_t<2, 4>(X, Y, M, ar);
    else cta_square_dmma_t<3, 6>(X, Y, M, ar);
}

__device__ bool cta_tc2(double *X, double *Y, int M, int nocc, const Arena &ar, int *nsteps,
                        long long *prof = nullptr) {
    const int tid = threadIdx.x, nt = SCF_THREADS;
    const long long c0 = clock64();
    const int T = (M + 3) >> 2;                       // tiles per dimension
    const int ntile = T * (T + 1) / 2;                // upper triangle (ta <= tb)
    // spectral bounds: Gershgorin, tightened by a short Lanczos run and X0
    double lo = -1e300, hi = -1e300;                  // lo holds -min
    for (int i = tid; i < M; i += nt) {
        double r = 0.0;
        for (int j = 0; j < M; ++j)
            if (j != i) r += fabs(X[i * M + j]);
        lo = fmax(lo, -(X[i * M + i] - r));
        hi = fmax(hi, X[i * M + i] + r);
    }
    block_max2(lo, hi, ar.red);
    lo = -lo;
    {
        double llo, lhi;
        lanczos_bounds(X, M, ar, &llo, &lhi);
        lo = fmax(lo, llo);
        hi = fmin(hi, lhi);
    }
    const double sc = 1.0 / (hi - lo);
    for (int t = tid; t < M * M; t += nt) {
        const int r = t / M, c = t - r * M;
        X[t] = ((r == c ? hi : 0.0) - X[t]) * sc;
    }
    __syncthreads();                                  // the diagonal below has other writers
    double tr = 0.0;
    for (int i = tid; i < M; i += nt) tr += X[i * M + i];
    tr = block_sum(tr, ar.red);                       // ends with a barrier: X0 complete
    int extra = -1, k = 0;
    bool ok = false;
    const long long c1 = clock64();
    for (; k < TC2_MAX; ++k) {
        // Y = X X (X symmetric: Y_ij = sum_l X_li X_lj), upper 4 x 4 tiles, mirrored on write.
        // The four values of a tile column are read as two 16-byte loads (rows start on 16-byte
        // boundaries: M even or odd, 8 M l + 32 t is a multiple of 16 only for even M, so odd M
        // takes the scalar loads); the sum is bound by shared-memory wavefronts, and 8-byte
        // loads of 15 distinct tile columns per warp cost ~4x the wavefronts of 16-byte ones.
        // Lanes past M read neighbouring values (inside the arena) into products never stored.
        const bool vec = (M & 1) == 0;
        if (TC2_DMMA) cta_square_dmma(X, Y, M, ar);
        else
        for (int u = tid; u < ntile; u += nt) {
            int ta = 0, rem = u;
            while (rem >= T - ta) { rem -= T - ta; ++ta; }
            const int tb = ta + rem;
            const int i0 = 4 * ta, j0 = 4 * tb;
            double acc[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
            if (vec) {
#pragma unroll kTc2Unr
                for (int l = 0; l < M; ++l) {
                    const double *xr = X + l * M;
                    const double2 p0 = *reinterpret_cast<const double2 *>(xr + i0);
                    const double2 p1 = *reinterpret_cast<const double2 *>(xr + i0 + 2);
                    const double2 q0 = *reinterpret_cast<const double2 *>(xr + j0);
                    const double2 q1 = *reinterpret_cast<const double2 *>(xr + j0 + 2);
                    const double xi[4] = {p0.x, p0.y, p1.x, p1.y}, xj[4] = {q0.x, q0.y, q1.x, q1.y};
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc[a][c] = fma(xi[a], xj[c], acc[a][c]);
                }
            } else {
#pragma unroll kTc2Unr
                for (int l = 0; l < M; ++l) {
                    const double *xr = X + l * M;
                    double xi[4], xj[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        xi[a] = i0 + a < M ? xr[i0 + a] : 0.0;
                        xj[a] = j0 + a < M ? xr[j0 + a] : 0.0;
                    }
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc[a][c] = fma(xi[a], xj[c], acc[a][c]);
                }
            }
            double dsum = 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int i = i0 + a, j = j0 + c;
                    if (i < M && j < M) {
                        Y[i * M + j] = acc[a][c];
                        Y[j * M + i] = acc[a][c];
                        if (i == j) dsum += acc[a][c];
                    }
                }
            if (ta == tb) ar.dv[ta] = dsum;
        }
        __syncthreads();
        double tr2 = 0.0;
        if (TC2_DMMA) {
            // every warp forms the same shuffle-tree sum (fixed order, no extra barrier; a
            // serial 58-term sum in every thread cost ~1.5k cycles of shared-memory latency)
            const int ln = tid & 31;
            double t2 = 0.0;
            for (int e = ln; e < M; e += 32) t2 += ar.dv[e];
            tr2 = __shfl_sync(0xffffffffu, warp_sum(t2), 0);   // lane 0's (butterfly orders differ per lane)
        } else {
            for (int a = 0; a < T; ++a) tr2 += ar.dv[a];
        }
        const bool sq = fabs(tr2 - nocc) <= fabs(2.0 * tr - tr2 - nocc);
        const double idem = tr - tr2;
        for (int t = tid; t < M * M; t += nt) X[t] = sq ? Y[t] : 2.0 * X[t] - Y[t];
        tr = sq ? tr2 : 2.0 * tr - tr2;
        __syncthreads();
        if (extra < 0 && fabs(idem) < 1e-11) extra = 0;
        if (extra >= 0 && ++extra > 1) { ok = true; ++k; break; }
    }
    *nsteps = k;
    if (prof && tid == 0) { prof[0] += c1 - c0; prof[1] += clock64() - c1; }
    return ok && fabs(tr - nocc) < 1e-6;
}

// ---------------------------------------------------------------------------- orthogonaliser
__global__ void __launch_bounds__(SCF_THREADS, 2) k_orth(DevBatch b, int nm) {
    extern __shared__ __align__(16) unsigned char ssm[];
    const Arena ar = carve(ssm, nm);
    const int m = b.mol_order[blockIdx.x], N = b.m_nao[m], tid = threadIdx.x;
    const int64_t o = b.m_mat0[m];
    for (int t = tid; t < N * N; t += SCF_THREADS) {
        ar.A[t] = b.S[o + t];
        ar.B[t] = (t / N == t % N) ? 1.0 : 0.0;
    }
    __syncthreads();
    const long long t0 = clock64();
    int nsw = 0;
    const double *Ad = cta_jacobi(ar.A, ar.B, N, ar, &nsw);
    if (b.dbg && tid == 0) { b.dbg[16 * m + 12] = clock64() - t0; b.dbg[16 * m + 13] = nsw; }
    sort_eigs(Ad, N, ar);
    // kept = s > 1e-7, in ascending order: sorted positions [N - M, N)
    if (tid == 0) {
        int M = 0;
        double smax = -1e300;
        for (int i = 0; i < N; ++i) {
            M += ar.dv[i] > 1e-7;
            smax = fmax(smax, ar.dv[i]);
        }
        // scf.py:89-93: not PD if the largest eigenvalue is <= 0, singular if nothing survives
        if (smax <= 0.0) b.status[m] |= DFTB_ST_OVERLAP_NOT_PD;
        else if (M == 0) b.status[m] |= DFTB_ST_SINGULAR;
        if (M < b.m_nocc[m]) b.status[m] |= DFTB_ST_NO_ORBITALS;
        b.nmo[m] = M;
        ar.scal[0] = M;
    }
    __syncthreads();
    const int M = (int)ar.scal[0];
    for (int t = tid; t < N * N; t += SCF_THREADS) {
        const int row = t / N, i = t % N;  // eigenvector column i
        const int r = ar.perm[i] - (N - M);
        if (r >= 0) b.X[o + (int64_t)row * N + r] = ar.B[i * N + row] / sqrt(ar.dv[i]);   // V^T
    }
    for (int t = tid; t < N * N; t += SCF_THREADS) {
        const int r = t % N;
        if (r >= M) b.X[o + t] = 0.0;
    }
}


#ifndef SEQ_SUM_BATCH
#define SEQ_SUM_BATCH 16
#endif
// sum_{u < n} load(u) accumulated left to right (bitwise the plain loop's result), with
// the loads issued 8 at a time: the partial reductions below read L2/HBM, and a serial
// load-add chain left them latency-bound (~20% of the post kernel).
template <typename F>
__device__ __forceinline__ double seq_sum(int n, F load) {
    constexpr int B = SEQ_SUM_BATCH;
    double v = 0.0;
    int u = 0;
    for (; u + B <= n; u += B) {
        double x[B];
#pragma unroll
        for (int k = 0; k < B; ++k) x[k] = load(u + k);
#pragma unroll
        for (int k = 0; k < B; ++k) v += x[k];
    }
    for (; u < n; ++u) v += load(u);
    return v;
}

// J from owner + scattered partials, K = -(G + G^T)/4 from G rows (fixed-order sums).
// (and V_xc = W + W^T with W the fixed-order sum of the per-XC-CTA partials)
template <bool WITH_V>
__device__ void reduce_jkv(const DevBatch &b, int m, int N, double *J, double *K, double *Vx) {
    const int tid = threadIdx.x;
    const int64_t npp = tri(N);
    const double *Jp = b.Jpart + b.m_Jp0[m];
    const int ncj = b.m_jkcta0[m + 1] - b.m_jkcta0[m];
    for (int64_t q = tid; q < npp; q += SCF_THREADS) {
        const double v = seq_sum(ncj + 1, [&](int c) { return Jp[(int64_t)c * npp + q]; });
        int k = (int)((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
        while (tri(k + 1) <= q) ++k;
        while (tri(k) > q) --k;
        const int l = (int)(q - tri(k));
        J[k * N + l] = v;
        J[l * N + k] = v;
    }
    const double *Gp = b.Gpart + b.m_G0[m];   // [ncj][N][N] per-CTA exchange partials
    const int64_t NN = (int64_t)N * N;
    // the exchange and V_xc partial sums in one loop: both load streams in flight together
    const double *Vp = b.Vpart + b.m_V0[m];
    const int ncx = WITH_V ? b.m_xccta0[m + 1] - b.m_xccta0[m] : 0;
    for (int t = tid; t < N * N; t += SCF_THREADS) {
        const double kv = seq_sum(ncj, [&](int c) { return Gp[c * NN + t]; });
        if constexpr (WITH_V) {
            const double vv = seq_sum(ncx, [&](int c) { return Vp[(int64_t)c * NN + t]; });
            Vx[t] = vv;
        }
        K[t] = kv;
    }
    __syncthreads();
    for (int t = tid; t < N * N; t += SCF_THREADS) {
        const int a = t / N, c = t % N;
        if (a < c) {
            const double g = -(K[a * N + c] + K[c * N + a]) * 0.25;
            K[a * N + c] = g;
            K[c * N + a] = g;
        } else if (a == c) {
            K[t] = -0.5 * K[t];
        }
        if constexpr (WITH_V) {
            if (a < c) {
                const double v = Vx[a * N + c] + Vx[c * N + a];
                Vx[a * N + c] = v;
                Vx[c * N + a] = v;
            } else if (a == c) {
                Vx[t] = 2.0 * Vx[t];
            }
        }
    }
}

// V_xc = W + W^T with W the fixed-order sum of the per-CTA partials.
__device__ void reduce_vxc(const DevBatch &b, int m, int N, double *Vx) {
    const int tid = threadIdx.x;
    const double *Vp = b.Vpart + b.m_V0[m];
    const int ncx = b.m_xccta0[m + 1] - b.m_xccta0[m];
    for (int t = tid; t < N * N; t += SCF_THREADS) {
        Vx[t] = seq_sum(ncx, [&](int c) { return Vp[(int64_t)c * N * N + t]; });
    }
    __syncthreads();
    for (int t = tid; t < N * N; t += SCF_THREADS) {
        const int a = t / N, c = t % N;
        if (a < c) {
            const double v = Vx[a * N + c] + Vx[c * N + a];
            Vx[a * N + c] = v;
            Vx[c * N + a] = v;
        } else if (a == c) {
            Vx[t] = 2.0 * Vx[t];
        }
    }
}

__device__ double reduce_exc(const DevBatch &b, int m) {
    double exc = 0.0;
    const int ncx = b.m_xccta0[m + 1] - b.m_xccta0[m];
    for (int c = 0; c < ncx; ++c) exc += b.Epart[b.m_xccta0[m] + c];
    return exc;
}

// Operator-level reductions (dftb_plan_jk / dftb_plan_xc): which = 1 J/K, 2 Vxc.
__global__ void __launch_bounds__(SCF_THREADS) k_reduce(DevBatch b, int which) {
    const int m = blockIdx.x, N = b.m_nao[m];
    const int64_t o = b.m_mat0[m];
    if (which == 1) reduce_jkv<false>(b, m, N, b.J + o, b.K + o, nullptr);
    else {
        reduce_vxc(b, m, N, b.Vxc + o);
        if (threadIdx.x == 0) b.comp[5 * m + 4] = reduce_exc(b, m);
    }
}

void launch_reduce(const DevBatch &b, int which, cudaStream_t s) {
    k_reduce<<<b.n_mol, SCF_THREADS, 0, s>>>(b, which);
}

// ---------------------------------------------------------------------------- post kernel
struct PostArgs {
    int nm;             // arena dimension
    int it;             // iteration index; -1 = core-Hamiltonian guess
    int diis_start, diis_hist;
    double damping, conv_std;
};

// Solve the bordered DIIS system ar.Bs (n1 x n1, rhs e_{n1-1}) -> ar.cf, by one warp:
// Gaussian elimination with partial pivoting in shared memory (the same operations in the
// same order per element as a serial elimination; a thread-local array cost a local-memory
// round trip per element update).  Mx in ar.A (row stride n1 + 1), multipliers in ar.sn.
__device__ void diis_solve_warp(const Arena &ar, int n1) {
    const int lane = threadIdx.x & 31;
    double *Mx = ar.A, *fr = ar.sn;
    const int W = n1 + 1, nh = n1 - 1;
    __syncwarp();
    for (int t = lane; t < n1 * W; t += 32) {
        const int r = t / W, k = t - r * W;
        Mx[t] = k < n1 ? ar.Bs[r * n1 + k] : (r == nh ? 1.0 : 0.0);
    }
    __syncwarp();
    for (int c = 0; c < n1; ++c) {
        int piv = c;
        for (int r = c + 1; r < n1; ++r)
            if (fabs(Mx[r * W + c]) > fabs(Mx[piv * W + c])) piv = r;
        __syncwarp();
        if (piv != c)
            for (int k = lane; k <= n1; k += 32) {
                const double t = Mx[c * W + k];
                Mx[c * W + k] = Mx[piv * W + k];
                Mx[piv * W + k] = t;
            }
        __syncwarp();
        for (int r = c + 1 + lane; r < n1; r += 32) fr[r] = Mx[r * W + c] / Mx[c * W + c];
        __syncwarp();
        const int wk = n1 + 1 - c;
        for (int t = lane; t < (n1 - c - 1) * wk; t += 32) {
            const int r = c + 1 + t / wk, k = c + t % wk;
            Mx[r * W + k] -= fr[r] * Mx[c * W + k];
        }
        __syncwarp();
    }
    if (lane == 0)
        for (int r = n1 - 1; r >= 0; --r) {
            double s = Mx[r * W + n1];
            for (int k = r + 1; k < n1; ++k) s -= Mx[r * W + k] * ar.cf[k];
            ar.cf[r] = s / Mx[r * W + r];
        }
    __syncwarp();
}

__device__ void diis_extrapolate(const DevBatch &b, int m, int N, const double *F, double *Fuse,
                                 const PostArgs &pa, const Arena &ar) {
    const int tid = threadIdx.x;
    const int h = pa.diis_hist, nh = b.ring_n[m], head = b.ring_head[m];
    const int64_t o = b.m_mat0[m], tot = b.m_mat0[b.n_mol];
    auto slot = [&](int a) { return (head - nh + a + 2 * h) % h; };
    if (nh <= 1) {
        for (int t = tid; t < N * N; t += SCF_THREADS) Fuse[t] = F[t];
        __syncthreads();
        return;
    }
    const int n1 = nh + 1;
    const double *Bm = b.Bmat + (int64_t)m * h * h;
    for (int t = tid; t < n1 * n1; t += SCF_THREADS) {
        const int r = t / n1, c = t % n1;
        double v;
        if (r == nh && c == nh) v = 0.0;
        else if (r == nh || c == nh) v = 1.0;
        else v = Bm[slot(r) * h + slot(c)];
        ar.Bs[t] = v;
        ar.A[t] = v;
        ar.B[t] = (r == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (tid < 32) {
        const int lane = tid;
        warp_jacobi_eigs(ar.A, n1, ar);
        __syncwarp();
        bool fallback = false;
        if (lane == 0) {
            const double *Ad = ar.A;
            double mx = 0.0, mn = 1e308;
            for (int i = 0; i < n1; ++i) {
                const double e = fabs(Ad[i * n1 + i]);
                mx = fmax(mx, e);
                mn = fmin(mn, e);
            }
            fallback = !(mn > 0.0) || (mx / mn > 1e12);
            ar.scal[1] = fallback ? 1.0 : 0.0;
        }
        fallback = __shfl_sync(0xffffffffu, fallback, 0);
        if (!fallback) diis_solve_warp(ar, n1);
    }
    __syncthreads();
    if (ar.scal[1] != 0.0) {
        const double *Fl = b.Fring + (int64_t)slot(nh - 1) * tot + o;
        const double *Fp = b.Fring + (int64_t)slot(nh - 2) * tot + o;
        for (int t = tid; t < N * N; t += SCF_THREADS) Fuse[t] = 0.5 * Fl[t] + 0.5 * Fp[t];
    } else if (nh <= 8) {           // the usual history: loads of all entries in flight at once
        int64_t off[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) off[a] = (int64_t)slot(a < nh ? a : 0) * tot + o;
        for (int t = tid; t < N * N; t += SCF_THREADS) {
            double x[8];
#pragma unroll
            for (int a = 0; a < 8; ++a) x[a] = a < nh ? b.Fring[off[a] + t] : 0.0;
            double v = 0.0;
#pragma unroll
            for (int a = 0; a < 8; ++a)
                if (a < nh) v += ar.cf[a] * x[a];
            Fuse[t] = v;
        }
    } else {
        for (int t = tid; t < N * N; t += SCF_THREADS) {
            double v = 0.0;
            for (int a = 0; a < nh; ++a) v += ar.cf[a] * b.Fring[(int64_t)slot(a) * tot + o + t];
            Fuse[t] = v;
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(SCF_THREADS, 2) k_post(DevBatch b, PostArgs pa) {
    extern __shared__ __align__(16) unsigned char ssm[];
    Arena ar = carve(ssm, pa.nm, pa.diis_hist + 1);
    const int m = b.mol_order[blockIdx.x], tid = threadIdx.x;
    if (b.done[m]) return;
#ifdef JAC_PHASES
    if (b.dbg) ar.dbgp = b.dbg + 16 * m + 14;   // dbg[14], dbg[15]: Jacobi angle / apply cycles
#endif
    const int N = b.m_nao[m], M = b.nmo[m], nocc = b.m_nocc[m];
    if (b.status[m] & (DFTB_ST_OVERLAP_NOT_PD | DFTB_ST_SINGULAR | DFTB_ST_NO_ORBITALS)) {
        if (tid == 0) b.done[m] = 1;
        return;
    }
    const int64_t o = b.m_mat0[m], tot = b.m_mat0[b.n_mol];
    double *S = b.S + o, *H = b.H + o, *X = b.X + o, *C = b.C + o, *Cp = b.Cp + o;
    double *rho = b.rho + o, *F = b.F + o, *J = b.J + o, *K = b.K + o, *Vx = b.Vxc + o;
    double *S1 = b.scratch + o, *S2 = b.scratch + tot + o;
    const int it = pa.it;
    const double *Fuse = H;
    long long t0 = clock64(), tl = t0;
    long long *dbg = b.dbg ? b.dbg + 16 * m : nullptr;
    auto tick = [&](int k) { if (dbg && tid == 0) { long long t = clock64(); dbg[k] += t - tl; tl = t; } };
    if (it >= 0) {
        reduce_jkv<true>(b, m, N, J, K, Vx);
        __syncthreads();
        tick(0);
        // (4) F and (5) energies
        double ec = 0.0, ej = 0.0, ek = 0.0;
        for (int t = tid; t < N * N; t += SCF_THREADS) {
            const double f = H[t] + J[t] + 0.20 * K[t] + Vx[t];
            F[t] = f;
            ec += rho[t] * H[t];
            ej += rho[t] * J[t];
            ek += rho[t] * K[t];
        }
        ec = block_sum(ec, ar.red);
        ej = block_sum(ej, ar.red);
        ek = block_sum(ek, ar.red);
        if (tid == 0) {
            const double exc = reduce_exc(b, m);
            double *cp = b.comp + 5 * m;
            cp[0] = b.enn[m];
            cp[1] = ec;
            cp[2] = 0.5 * ej;
            cp[3] = 0.5 * 0.20 * ek;
            cp[4] = exc;
            b.hist[(int64_t)m * b.max_it + it] = cp[0] + cp[1] + cp[2] + cp[3] + cp[4];
        }
        tick(1);
        // (6) DIIS error e = F rho S - S rho F = A - A^T with A = F rho S
        cta_gemm(S1, N, F, N, false, rho, N, false, N, N, N, 1.0, 0.0, ar);
        cta_gemm(S2, N, S1, N, false, S, N, false, N, N, N, 1.0, 0.0, ar);
        const int h = pa.diis_hist, head = b.ring_head[m];
        double *Fs = b.Fring + (int64_t)head * tot + o, *Es = b.Ering + (int64_t)head * tot + o;
        for (int t = tid; t < N * N; t += SCF_THREADS) {
            const int a = t / N, c = t % N;
            Es[t] = S2[a * N + c] - S2[c * N + a];
            Fs[t] = F[t];
        }
        __syncthreads();
        // (7) B row for the new entry against every stored error (physical slots)
        const int nh_new = min(b.ring_n[m] + 1, h);
        double *Bm = b.Bmat + (int64_t)m * h * h;
        for (int a = 0; a < nh_new; ++a) {
            const int sl = (head - a + h) % h;  // walk back from the newest
            const double *Ea = b.Ering + (int64_t)sl * tot + o;
            double d = 0.0;
            for (int t = tid; t < N * N; t += SCF_THREADS) d += Es[t] * Ea[t];
            d = block_sum(d, ar.red);
            if (tid == 0) {
                Bm[head * h + sl] = d;
                Bm[sl * h + head] = d;
            }
        }
        __syncthreads();
        if (tid == 0) {
            b.ring_head[m] = (head + 1) % h;
            b.ring_n[m] = nh_new;
        }
        __syncthreads();
        tick(2);
        // (8) extrapolation
        if (it + 1 >= pa.diis_start) {
            diis_extrapolate(b, m, N, F, S1, pa, ar);
            Fuse = S1;
        } else {
            Fuse = F;
        }
    }
    tick(3);
    // convergence is decided before the solve: it depends on the energies alone (scf.py:198-200),
    // and the last iteration is the one whose orbitals and eigenvalues are returned
    if (tid == 0) {
        int stop = 0, cv = 0;
        if (it >= 0) {
            stop = it + 1 >= b.max_it;
            if (it + 1 >= 5) {
                const double *hh = b.hist + (int64_t)m * b.max_it + it - 4;
                double mean = 0.0;
                for (int k = 0; k < 5; ++k) mean += hh[k];
                mean /= 5.0;
                double var = 0.0;
                for (int k = 0; k < 5; ++k) var += (hh[k] - mean) * (hh[k] - mean);
                if (sqrt(var / 5.0) < pa.conv_std) {
                    cv = 1;
                    stop = 1;
                }
            }
        }
        ar.scal[2] = stop;
        ar.scal[3] = cv;
    }
    __syncthreads();
    const bool last = ar.scal[2] != 0.0;
    // (9) F' = X^T F X; orbitals (last iteration / callback path) or the density projector
    cta_gemm(S2, N, Fuse, N, false, X, N, false, N, M, N, 1.0, 0.0, ar);     // F X  (N x M, ld N)
    cta_gemm(ar.A, M, X, N, true, S2, N, false, M, M, N, 1.0, 0.0, ar);      // X^T (F X)
    tick(7);
    bool eig = last || b.full_eig;
    if (!eig) {
        int nst = 0;
        if (cta_tc2(ar.A, ar.B, M, nocc, ar, &nst, dbg ? dbg + 14 : nullptr)) {
            // rho_new = 2 X P' X^T
            cta_gemm(S2, N, X, N, false, ar.A, M, false, N, M, M, 1.0, 0.0, ar);   // X P'  (N x M)
            cta_gemm(S1, N, S2, N, false, X, N, true, N, N, M, 2.0, 0.0, ar);       // 2 (X P') X^T
            if (tid == 0) { b.puri[m] = nst; b.cpv[m] = 0; if (dbg) dbg[4] += nst; }
        } else {
            eig = true;                               // no converged projector: diagonalise
            if (tid == 0) b.puri[m] = -nst;
            cta_gemm(ar.A, M, X, N, true, S2, N, false, M, M, N, 1.0, 0.0, ar);   // F' again
        }
        tick(8);
    }
    if (eig) {
        const bool warm = b.cpv[m] != 0;
        if (warm) {
            // warm start: Jacobi on C'^T F' C' with V = C' (previous eigenvectors)
            cta_gemm(S1, M, ar.A, M, false, Cp, M, false, M, M, M, 1.0, 0.0, ar); // F' C'
            cta_gemm(ar.A, M, Cp, M, true, S1, M, false, M, M, M, 1.0, 0.0, ar);  // C'^T F' C'
            for (int t = tid; t < M * M; t += SCF_THREADS) ar.B[(t % M) * M + t / M] = Cp[t];   // V^T = C'^T
        } else {
            for (int t = tid; t < M * M; t += SCF_THREADS) ar.B[t] = (t / M == t % M) ? 1.0 : 0.0;
        }
        __syncthreads();
        // f32 build: eigenvectors to f32 resolution (the reference's f32 path diagonalizes in
        // single precision, scf.py:86-98); f64 build: to 1e-13 of the largest |eigenvalue|
        int nsw = 0;
        const double *Ad = cta_jacobi(ar.A, ar.B, M, ar, &nsw, 40, b.prec ? 1e-8 : 1e-13);
        if (dbg && tid == 0) dbg[10] += nsw;
        tick(9);
        sort_eigs(Ad, M, ar);
        tick(5);
        for (int t = tid; t < M * M; t += SCF_THREADS) {
            const int row = t / M, i = t % M;
            Cp[row * M + ar.perm[i]] = ar.B[i * M + row];
        }
        for (int i = tid; i < M; i += SCF_THREADS) b.eps[(int64_t)m * NMAX + ar.perm[i]] = ar.dv[i];
        __syncthreads();
        cta_gemm(C, N, X, N, false, Cp, M, false, N, M, M, 1.0, 0.0, ar);         // C = X C' (N x M)
        // rho_new = 2 C_occ C_occ^T
        cta_gemm(S1, N, C, N, false, C, N, true, N, N, nocc, 2.0, 0.0, ar);
        if (tid == 0) b.cpv[m] = 1;
    }
    // (+ damping when the next iteration is pre-DIIS)
    const int nxt = it + 1;
    const bool damp = nxt > 0 && nxt < pa.diis_start;
    const double d = pa.damping;
    for (int t = tid; t < N * N; t += SCF_THREADS) {
        double v = S1[t];
        if (damp) v = d * rho[t] + (1.0 - d) * v;
        if (b.prec) v = (double)(float)v;
        rho[t] = v;
    }
    tick(6);
    if (dbg && tid == 0) dbg[11] += 1;
    if (tid == 0 && it >= 0) {
        b.iters[m] = it + 1;
        if (ar.scal[3] != 0.0) b.conv[m] = 1;
        if (last) b.done[m] = 1;
    }
}

static int arena_dim(int nmax, int hs = 10) {
    // the DIIS elimination keeps its hs x (hs + 1) working matrix in A
    int nm = nmax < 16 ? 16 : nmax;
    while ((size_t)nm * nm < (size_t)hs * (hs + 1)) ++nm;
    return nm;
}

void launch_orth(const DevBatch &b, int nmax, cudaStream_t s) {
    const int nm = arena_dim(nmax);
    const size_t sm = scf_smem_bytes(nm);
    smem_optin((const void *)k_orth);
    k_orth<<<b.n_mol, SCF_THREADS, sm, s>>>(b, nm);
}

void launch_post(const DevBatch &b, int nmax, int it, int diis_start, int diis_hist, double damping,
                 double conv_std, cudaStream_t s) {
    const int nm = arena_dim(nmax, diis_hist + 1);
    const size_t sm = scf_smem_bytes(nm, diis_hist + 1);
    smem_optin((const void *)k_post);
    PostArgs pa{nm, it, diis_start, diis_hist, damping, conv_std};
    k_post<<<b.n_mol, SCF_THREADS, sm, s>>>(b, pa);
}

// ---------------------------------------------------------------------------- standalone roothaan
// For the operator-level API: F given per molecule in b.F; writes C, eps (cold Jacobi).
__global__ void __launch_bounds__(SCF_THREADS) k_roothaan(DevBatch b, int nm) {
    extern __shared__ __align__(16) unsigned char ssm[];
    const Arena ar = carve(ssm, nm);
    const int m = b.mol_order[blockIdx.x], tid = threadIdx.x;
    const int N = b.m_nao[m], M = b.nmo[m];
    const int64_t o = b.m_mat0[m], tot = b.m_mat0[b.n_mol];
    double *X = b.X + o, *C = b.C + o, *Cp = b.Cp + o, *S2 = b.scratch + tot + o;
    cta_gemm(S2, N, b.F + o, N, false, X, N, false, N, M, N, 1.0, 0.0, ar);
    cta_gemm(ar.A, M, X, N, true, S2, N, false, M, M, N, 1.0, 0.0, ar);
    for (int t = tid; t < M * M; t += SCF_THREADS) ar.B[t] = (t / M == t % M) ? 1.0 : 0.0;
    __syncthreads();
    int nsw = 0;
    const double *Ad = cta_jacobi(ar.A, ar.B, M, ar, &nsw);
    sort_eigs(Ad, M, ar);
    for (int t = tid; t < M * M; t += SCF_THREADS) Cp[(t / M) * M + ar.perm[t % M]] = ar.B[(t % M) * M + t / M];
    for (int i = tid; i < M; i += SCF_THREADS) b.eps[(int64_t)m * NMAX + ar.perm[i]] = ar.dv[i];
    __syncthreads();
    cta_gemm(C, N, X, N, false, Cp, M, false, N, M, M, 1.0, 0.0, ar);
}

void launch_roothaan(const DevBatch &b, int nmax, cudaStream_t s) {
    const int nm = arena_dim(nmax);
    const size_t sm = scf_smem_bytes(nm);
    smem_optin((const void *)k_roothaan);
    k_roothaan<<<b.n_mol, SCF_THREADS, sm, s>>>(b, nm);
}

// ---------------------------------------------------------------------------- device results
// E_total[m] = the last recorded energy; history copied with the tail past iters[m] set to NaN
__global__ void k_fetch(DevBatch b, double *E, double *hist) {
    const int m = blockIdx.x, nit = b.iters[m];
    const double *h = b.hist + (int64_t)m * b.max_it;
    if (E && threadIdx.x == 0) E[m] = nit > 0 ? h[nit - 1] : CUDART_NAN;
    if (hist)
        for (int t = threadIdx.x; t < b.max_it; t += blockDim.x)
            hist[(int64_t)m * b.max_it + t] = t < nit ? h[t] : CUDART_NAN;
}

void launch_fetch_dev(const DevBatch &b, double *E, double *hist, cudaStream_t s) {
    k_fetch<<<b.n_mol, 64, 0, s>>>(b, E, hist);
}

// ---------------------------------------------------------------------------- standalone DIIS
// One system: F, E given as m x (n x n) arrays; out = diis_step(history) (scf.py:101-132).
__global__ void __launch_bounds__(SCF_THREADS) k_diis_single(const double *F, const double *E, int mh, int n,
                                                            double *out, int nm) {
    extern __shared__ __align__(16) unsigned char ssm[];
    const Arena ar = carve(ssm, nm, mh + 1);
    const int tid = threadIdx.x, nn = n * n;
    if (mh == 1) {
        for (int t = tid; t < nn; t += SCF_THREADS) out[t] = F[t];
        return;
    }
    const int n1 = mh + 1;
    for (int a = 0; a < mh; ++a)
        for (int c = a; c < mh; ++c) {
            double d = 0.0;
            for (int t = tid; t < nn; t += SCF_THREADS) d += E[(int64_t)a * nn + t] * E[(int64_t)c * nn + t];
            d = block_sum(d, ar.red);
            if (tid == 0) { ar.Bs[a * n1 + c] = d; ar.Bs[c * n1 + a] = d; }
        }
    __syncthreads();
    for (int t = tid; t < n1 * n1; t += SCF_THREADS) {
        const int r = t / n1, c = t % n1;
        if (r == mh || c == mh) ar.Bs[t] = (r == mh && c == mh) ? 0.0 : 1.0;
    }
    __syncthreads();
    for (int t = tid; t < n1 * n1; t += SCF_THREADS) {
        ar.A[t] = ar.Bs[t];
        ar.B[t] = (t / n1 == t % n1) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (tid < 32) warp_jacobi_eigs(ar.A, n1, ar);
    const double *Ad = ar.A;
    if (tid < 32) {
        bool fb = false;
        if (tid == 0) {
            double mx = 0.0, mn = 1e308;
            for (int i = 0; i < n1; ++i) { const double e = fabs(Ad[i * n1 + i]); mx = fmax(mx, e); mn = fmin(mn, e); }
            fb = !(mn > 0.0) || (mx / mn > 1e12);
            ar.scal[1] = fb;
        }
        fb = __shfl_sync(0xffffffffu, fb, 0);
        if (!fb) diis_solve_warp(ar, n1);
    }
    __syncthreads();
    for (int t = tid; t < nn; t += SCF_THREADS) {
        double v = 0.0;
        if (ar.scal[1] != 0.0) v = 0.5 * F[(int64_t)(mh - 1) * nn + t] + 0.5 * F[(int64_t)(mh - 2) * nn + t];
        else for (int a = 0; a < mh; ++a) v += ar.cf[a] * F[(int64_t)a * nn + t];
        out[t] = v;
    }
}

void launch_diis_single(const double *F, const double *E, int mh, int n, double *out, cudaStream_t s) {
    const int nm = arena_dim(mh + 1, mh + 1);
    const size_t sm = scf_smem_bytes(nm, mh + 1);
    smem_optin((const void *)k_diis_single);
    k_diis_single<<<1, SCF_THREADS, sm, s>>>(F, E, mh, n, out, nm);
}

}  // namespace dftb
