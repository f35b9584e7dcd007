// Fused AO-on-grid + density + B3LYP + V_xc kernel.
//
// Reference: deskdft.xc.eval_ao (xc.py:165-194), density_on_grid (:309-317),
// b3lyp (:277-306) and xc_matrix (:320-350).  The reference stores phi and
// grad phi for the whole grid and runs two BLAS GEMMs per 8192-point batch.
//
// B200 formulation: one CTA owns a contiguous range of one molecule's grid
// points and walks it in BP-point sub-blocks (64 in the f32 build, 32 in f64).
// Per sub-block the AO values and gradients are evaluated ONCE into shared
// memory (never written to HBM), stored [AO][point] with a 16-byte-group XOR
// swizzle so that every access pattern below is bank-conflict free:
//   t = phi rho and n, grad n   4 points x 4 AOs per thread in registers, 128-bit
//                               smem loads, partial sums reduced over the lanes
//                               sharing the points by a shuffle tree;
//   B3LYP                       f64; its three parts (Slater+B88, VWN, LYP) on three
//                               groups of BP threads, combined by the first group;
//   wv = a phi + b . grad phi   elementwise;
//   V += phi wv^T               4 x 4 register tiles accumulated over the CTA's
//                               whole point range, written once as a partial.
// Each SCF iteration reads only rho and writes one N x N partial per CTA.  CTAs
// are launched per AO-count bucket (NQ = ceil(N/16)*4 quads), so every kernel
// instance has compile-time tile loops and its own shared-memory footprint.
// W is the arithmetic type of the contractions: double in the f64 build, float in
// the f32 build (the reference's f32 BLAS path); the functional is always f64.
#include "common.cuh"
#include "b3lyp.cuh"

namespace dftb {

constexpr int XC_THREADS = 256;
constexpr int XC_SHD = 13;       // doubles per shell record in smem

template <typename W>
struct Vec4;
template <>
struct Vec4<float> {
    __device__ static __forceinline__ void ld(const float *p, float (&o)[4]) {
        const float4 v = *reinterpret_cast<const float4 *>(p);
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    }
};
template <>
struct Vec4<double> {
    __device__ static __forceinline__ void ld(const double *p, double (&o)[4]) {
        const double2 a = *reinterpret_cast<const double2 *>(p);
        const double2 b = *reinterpret_cast<const double2 *>(p + 2);
        o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
    }
};

// physical offset of logical (row, col) in a [rows][BP] tile, col groups of 4 swizzled by row quad
template <int BP>
__device__ __forceinline__ int swz(int row, int col) {
    return row * BP + ((((col >> 2) ^ (row >> 2)) & (BP / 4 - 1)) << 2) + (col & 3);
}

template <typename W, int NQ, int BP>
struct XCL {
    static constexpr int NP = 4 * NQ;
    static constexpr size_t rho = 0;
    static constexpr size_t phi = rho + sizeof(W) * NP * NP;
    static constexpr size_t wv = phi + sizeof(W) * 4 * NP * BP;
    static constexpr size_t pt = wv + sizeof(W) * NP * BP;
    static constexpr size_t dn = pt + sizeof(double) * 4 * BP;
    static constexpr size_t red = dn + sizeof(double) * 4 * BP;
    static constexpr size_t fpt = red + sizeof(double) * 32;      // functional parts [10][BP]
    static constexpr size_t dw = fpt + sizeof(double) * 10 * BP;  // wv coefficients [4][BP] (W)
    static constexpr size_t shd = dw + ((sizeof(W) * 4 * BP + 15) & ~(size_t)15);
    static size_t bytes(int nsh) { return shd + sizeof(double) * XC_SHD * (size_t)nsh; }
};

template <typename W, int NQ, int BP>
__device__ __forceinline__ void xc_eval_phi(W *phi, const double *pt, const double *shd, int nsh, int nb) {
    constexpr int NP = 4 * NQ, PL = NP * BP;
    for (int t = threadIdx.x; t < BP * nsh; t += XC_THREADS) {
        const int p = t % BP, sh = t / BP;
        const double *r = shd + XC_SHD * sh;
        const int kind = (int)r[12] & 1, ao = (int)r[12] >> 1;
        W v[4][4];  // [plane][component]
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) v[a][c] = (W)0;
        if (p < nb) {
            const double *q = pt + 4 * p;
            const W dx = (W)(q[0] - r[0]), dy = (W)(q[1] - r[1]), dz = (W)(q[2] - r[2]);
            const W r2 = dx * dx + dy * dy + dz * dz;
            W bs = 0, ds = 0, bp = 0, dp = 0;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const W a = (W)r[3 + k];
                const W ar = a * r2;
                W e;
                if constexpr (sizeof(W) == 4) e = ar < (W)88 ? expf(-ar) : (W)0;
                else e = ar < (W)745 ? exp(-ar) : (W)0;
                const W m2a = (W)-2 * a;
                bs += (W)r[6 + k] * e;
                ds += (W)r[6 + k] * m2a * e;
                bp += (W)r[9 + k] * e;
                dp += (W)r[9 + k] * m2a * e;
            }
            const W rel[3] = {dx, dy, dz};
            v[0][0] = bs;
#pragma unroll
            for (int d = 0; d < 3; ++d) v[d + 1][0] = rel[d] * ds;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                v[0][1 + c] = rel[c] * bp;
#pragma unroll
                for (int d = 0; d < 3; ++d) v[d + 1][1 + c] = (c == d ? bp : (W)0) + rel[c] * rel[d] * dp;
            }
        }
        const int nc = kind ? 4 : 1;
        for (int c = 0; c < nc; ++c) {
            const int o = swz<BP>(ao + c, p);
#pragma unroll
            for (int a = 0; a < 4; ++a) phi[a * PL + o] = v[a][c];
        }
    }
}

template <typename W, int NQ, int BP>
__global__ void __launch_bounds__(XC_THREADS) k_xc(DevBatch b, const int *ctas) {
    using L = XCL<W, NQ, BP>;
    constexpr int NP = 4 * NQ, PL = NP * BP;
    constexpr int PG = BP / 4;                 // point groups (4 points each)
    constexpr int LG = XC_THREADS / PG;        // lanes sharing a point group
    constexpr int QJ = (NQ + LG - 1) / LG;     // column quads per lane in the t phase
    constexpr int NT = NQ * NQ;                // V tiles (4 x 4)
    constexpr int TJ = (NT + XC_THREADS - 1) / XC_THREADS;
    extern __shared__ __align__(16) unsigned char xsm[];
    const int cta = ctas[blockIdx.x];
    const int m = b.xc_mol[cta];
    if (b.done[m]) return;
    const int N = b.m_nao[m];
    const int nsh = b.m_nshell[m], s0 = b.m_shell0[m];
    W *rho = (W *)(xsm + L::rho);
    W *phi = (W *)(xsm + L::phi);
    W *wv = (W *)(xsm + L::wv);
    double *pt = (double *)(xsm + L::pt);
    double *dn = (double *)(xsm + L::dn);
    double *red = (double *)(xsm + L::red);
    double *fpt = (double *)(xsm + L::fpt);
    W *dw = (W *)(xsm + L::dw);
    double *shd = (double *)(xsm + L::shd);
    const int tid = threadIdx.x;
    const double *rg = b.rho + b.m_mat0[m];
    for (int t = tid; t < NP * NP; t += XC_THREADS) {
        const int r = t / NP, c = t % NP;
        rho[t] = (r < N && c < N) ? (W)rg[r * N + c] : (W)0;
    }
    for (int t = tid; t < 4 * PL; t += XC_THREADS) phi[t] = (W)0;
    for (int sh = tid; sh < nsh; sh += XC_THREADS) {
        const int gsh = s0 + sh;
        double *r = shd + XC_SHD * sh;
        const double *A = b.a_xyz + 3 * b.s_atom[gsh];
        for (int d = 0; d < 3; ++d) {
            r[d] = A[d];
            r[3 + d] = b.s_exp[3 * gsh + d];
            r[6 + d] = b.s_cs[3 * gsh + d];
            r[9 + d] = b.s_cp[3 * gsh + d];
        }
        r[12] = (double)((b.s_ao[gsh] << 1) | (b.s_kind[gsh] & 1));
    }
    W acc[TJ][4][4];
#pragma unroll
    for (int j = 0; j < TJ; ++j)
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[j][a][c] = (W)0;
    double e_acc = 0.0;
    int bad = 0;
    const int pg = tid / LG, lg = tid % LG;
    const int64_t p0 = b.xc_p0[cta], p1 = b.xc_p1[cta];
    for (int64_t sb = p0; sb < p1; sb += BP) {
        const int nb = (int)min((int64_t)BP, p1 - sb);
        __syncthreads();                                   // previous sub-block consumed
        if (tid < BP) {
            const int64_t gi = sb + min(tid, nb - 1);
            pt[4 * tid] = b.g_xyz[3 * gi];
            pt[4 * tid + 1] = b.g_xyz[3 * gi + 1];
            pt[4 * tid + 2] = b.g_xyz[3 * gi + 2];
            pt[4 * tid + 3] = tid < nb ? b.g_w[gi] : 0.0;
        }
        __syncthreads();
        xc_eval_phi<W, NQ, BP>(phi, pt, shd, nsh, nb);
        __syncthreads();
        {   // ---- t = phi^T rho for 4 points x 4 AOs, then n and grad n partials
            W n4[4] = {0, 0, 0, 0}, g4[3][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
            for (int j = 0; j < QJ; ++j) {
                const int q = lg + j * LG;
                if (q < NQ) {
                    W t[4][4];
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int c = 0; c < 4; ++c) t[a][c] = (W)0;
                    // k ascending in groups of 4 rows: the swizzled column of a 4-row group is
                    // one XOR (rows >= N are zero in phi and rho, so the tail adds exact zeros)
                    for (int kq = 0; kq < (N + 3) / 4; ++kq) {
                        const W *pr = phi + 4 * kq * BP + (((pg ^ kq) & (BP / 4 - 1)) << 2);
                        const W *rr = rho + 4 * kq * NP + 4 * q;
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            W f[4], r4[4];
                            Vec4<W>::ld(pr + r * BP, f);
                            Vec4<W>::ld(rr + r * NP, r4);
#pragma unroll
                            for (int a = 0; a < 4; ++a)
#pragma unroll
                                for (int c = 0; c < 4; ++c) t[a][c] += f[a] * r4[c];
                        }
                    }
                    const int qo = 4 * q * BP + (((pg ^ q) & (BP / 4 - 1)) << 2);   // rows 4q..4q+3
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        W f0[4], f1[4], f2[4], f3[4];
                        Vec4<W>::ld(phi + qo + c * BP, f0);
                        Vec4<W>::ld(phi + PL + qo + c * BP, f1);
                        Vec4<W>::ld(phi + 2 * PL + qo + c * BP, f2);
                        Vec4<W>::ld(phi + 3 * PL + qo + c * BP, f3);
#pragma unroll
                        for (int a = 0; a < 4; ++a) {
                            n4[a] += t[a][c] * f0[a];
                            g4[0][a] += t[a][c] * f1[a];
                            g4[1][a] += t[a][c] * f2[a];
                            g4[2][a] += t[a][c] * f3[a];
                        }
                    }
                }
            }
#pragma unroll
            for (int o = 1; o < LG; o <<= 1)
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    n4[a] += __shfl_xor_sync(0xffffffffu, n4[a], o);
                    g4[0][a] += __shfl_xor_sync(0xffffffffu, g4[0][a], o);
                    g4[1][a] += __shfl_xor_sync(0xffffffffu, g4[1][a], o);
                    g4[2][a] += __shfl_xor_sync(0xffffffffu, g4[2][a], o);
                }
            if (lg == 0)
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    double *d = dn + 4 * (4 * pg + a);
                    d[0] = (double)n4[a];
                    d[1] = (double)(W)(2 * g4[0][a]);
                    d[2] = (double)(W)(2 * g4[1][a]);
                    d[3] = (double)(W)(2 * g4[2][a]);
                }
        }
        __syncthreads();
        if (tid < 3 * BP) {   // ---- functional (f64): parts on three thread groups, one point each
            const int pt_i = tid % BP, part = tid / BP;
            const double *dq = dn + 4 * pt_i;
            double n = dq[0], sig = 0.0;
            {
                const double gx = dq[1], gy = dq[2], gz = dq[3];
                sig = (double)((W)gx * (W)gx + (W)gy * (W)gy + (W)gz * (W)gz);
            }
            const bool ok = pt_i < nb && b3lyp_clamp(n, sig);
            if (part == 1) {
                const VPart v = ok ? b3lyp_vwn(n) : VPart{0.0, 0.0};
                fpt[5 * BP + pt_i] = v.f2;
                fpt[6 * BP + pt_i] = v.v2;
            } else if (part == 2) {
                const LPart l = ok ? b3lyp_lyp(n, sig) : LPart{0.0, 0.0, 0.0};
                fpt[7 * BP + pt_i] = l.f3;
                fpt[8 * BP + pt_i] = l.v3;
                fpt[9 * BP + pt_i] = l.w3;
            }
            XPart x{0.0, 0.0, 0.0, 0.0, 0.0};
            if (part == 0 && ok) x = b3lyp_x(n, sig);
            asm volatile("bar.sync 1, %0;" ::"r"(3 * BP) : "memory");
            if (part == 0) {
            double *d = dn + 4 * tid;
            if (ok) {
                const double gx = d[1], gy = d[2], gz = d[3];
                const XCOut o = xc_combine(n, x, VPart{fpt[5 * BP + pt_i], fpt[6 * BP + pt_i]},
                                           LPart{fpt[7 * BP + pt_i], fpt[8 * BP + pt_i], fpt[9 * BP + pt_i]});
                if (!(isfinite(o.exc) && isfinite(o.vrho) && isfinite(o.vsigma))) bad = 1;
                const double w = pt[4 * tid + 3];
                e_acc += w * n * (double)(W)o.exc;
                const double ww = (double)(W)w;
                const double a = (double)(W)(0.5 * ww * (double)(W)o.vrho);
                const double bb = (double)(W)(2.0 * ww * (double)(W)o.vsigma);
                dw[pt_i] = (W)a;
                dw[BP + pt_i] = (W)(bb * gx);
                dw[2 * BP + pt_i] = (W)(bb * gy);
                dw[3 * BP + pt_i] = (W)(bb * gz);
            } else {
                dw[pt_i] = dw[BP + pt_i] = dw[2 * BP + pt_i] = dw[3 * BP + pt_i] = (W)0;
            }
            }
        }
        __syncthreads();
        for (int t = tid; t < PL; t += XC_THREADS) {       // ---- wv = a phi + b . grad phi
            const int row = t / BP, p = t % BP;
            const int o = swz<BP>(row, p);
            wv[o] = dw[p] * phi[o] + dw[BP + p] * phi[PL + o] + dw[2 * BP + p] * phi[2 * PL + o] +
                    dw[3 * BP + p] * phi[3 * PL + o];
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < TJ; ++j) {                     // ---- V += phi wv^T, 4 x 4 tiles
            const int T = tid + j * XC_THREADS;
            if (T < NT) {
                const int qa = T / NQ, qb = T % NQ;
                const W *pa = phi + 4 * qa * BP, *pb = wv + 4 * qb * BP;   // rows 4qa.., 4qb..
                for (int c4 = 0; c4 < BP / 4; ++c4) {
                    const int ca = ((c4 ^ qa) & (BP / 4 - 1)) << 2, cb = ((c4 ^ qb) & (BP / 4 - 1)) << 2;
                    W fa[4][4], fb[4][4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        Vec4<W>::ld(pa + a * BP + ca, fa[a]);
                        Vec4<W>::ld(pb + a * BP + cb, fb[a]);
                    }
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int c = 0; c < 4; ++c)
#pragma unroll
                            for (int pp = 0; pp < 4; ++pp) acc[j][a][c] += fa[a][pp] * fb[c][pp];
                }
            }
        }
    }
    const int local = cta - b.m_xccta0[m];
    double *Vp = b.Vpart + b.m_V0[m] + (int64_t)local * N * N;
#pragma unroll
    for (int j = 0; j < TJ; ++j) {
        const int T = tid + j * XC_THREADS;
        if (T < NT) {
            const int qa = T / NQ, qb = T % NQ;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int mu = 4 * qa + a, nu = 4 * qb + c;
                    if (mu < N && nu < N) Vp[mu * N + nu] = (double)acc[j][a][c];
                }
        }
    }
    const double e = block_sum(e_acc, red);
    if (tid == 0) b.Epart[cta] = e;
    if (bad) atomicOr(b.status + m, DFTB_ST_XC_NONFINITE);
}

template <typename W, int NQ, int BP>
static void launch_bucket(const DevBatch &b, const int *ctas, int n, int nsh_max, cudaStream_t s) {
    const size_t sm = XCL<W, NQ, BP>::bytes(nsh_max);
    cudaFuncSetAttribute(k_xc<W, NQ, BP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_xc<W, NQ, BP><<<n, XC_THREADS, sm, s>>>(b, ctas);
}

template <typename W, int BP, int BPL>
static void launch_xc_t(const DevBatch &b, const int *bucket_ctas, const int *bucket_n, int nsh_max,
                        cudaStream_t s) {
    // BP points per sub-block for N <= 64, BPL for larger N (keeps 2 CTAs/SM in f32)
    // buckets: NQ = 4, 8, 12, 16, 20, 24 (N <= 16, 32, ..., 96)
    const int *c = bucket_ctas;
    if (bucket_n[0]) launch_bucket<W, 4, BP>(b, c, bucket_n[0], nsh_max, s);
    c += bucket_n[0];
    if (bucket_n[1]) launch_bucket<W, 8, BP>(b, c, bucket_n[1], nsh_max, s);
    c += bucket_n[1];
    if (bucket_n[2]) launch_bucket<W, 12, BP>(b, c, bucket_n[2], nsh_max, s);
    c += bucket_n[2];
    if (bucket_n[3]) launch_bucket<W, 16, BP>(b, c, bucket_n[3], nsh_max, s);
    c += bucket_n[3];
    if (bucket_n[4]) launch_bucket<W, 20, BPL>(b, c, bucket_n[4], nsh_max, s);
    c += bucket_n[4];
    if (bucket_n[5]) launch_bucket<W, 24, BPL>(b, c, bucket_n[5], nsh_max, s);
}

// bucket_ctas: device array of CTA indices grouped by bucket; bucket_n: host counts [6]
int launch_xc(const DevBatch &b, const int *bucket_ctas, const int *bucket_n, int nsh_max, cudaStream_t s) {
    if (b.n_xc_cta == 0) return 0;
    if (b.prec == 0) launch_xc_t<double, 32, 32>(b, bucket_ctas, bucket_n, nsh_max, s);
    else launch_xc_t<float, 64, 32>(b, bucket_ctas, bucket_n, nsh_max, s);
    int k = 0;
    for (int i = 0; i < 6; ++i) k += bucket_n[i] > 0;
    return k;
}

}  // namespace dftb
