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
#include "umma.cuh"
#ifdef XC_PHASES
#include <cstdio>
#endif

namespace dftb {

constexpr int XC_THREADS = 256;
#ifndef XC_TUNR
#define XC_TUNR 2      // unroll of the t-phase K loop (4-row groups)
#endif
#ifndef XC_VUNR
#define XC_VUNR 16     // unroll of the V-phase point loop (4-point groups; 1: 1.744 ms, 2: 1.722, 4: 1.713, 16 = full: 1.695)
#endif
#ifndef XC_AOUNR
#define XC_AOUNR 2     // unroll of the AO-value task loop
#endif
#ifndef XC_WVUNR
#define XC_WVUNR 1     // unroll of the wv row loop
#endif
constexpr int kXcTunr = XC_TUNR, kXcVunr = XC_VUNR;   // (pragma arguments are not macro-expanded)
constexpr int kXcAoUnr = XC_AOUNR, kXcWvUnr = XC_WVUNR;
// XC_MMA=1: f32 build runs the N 49..64 bucket on the tcgen05 kernel k_xc_mma below (parity
// tests green on B200; measured 2.49 ms vs 2.27 ms per iteration for the FFMA kernel, so the
// FFMA kernel stays the default - see DESIGN.md section 6, "measured and rejected")
#ifndef XC_MMA
#define XC_MMA 0
#endif
constexpr int XC_SHD = 13;       // doubles per shell record in smem
// f64 part of a shell record in k_xc: centre (x, y, z) and the three exponents in f64
constexpr int XC_SHD_D = 6;
// f32 build, AO exponentials.  The reference evaluates phi in f64 and rounds it to f32
// (xc.py:165-194); XC_AO_EXP=0 (default) forms a r^2 and exp(-a r^2) in f32 (relative error
// up to ~a r^2 * 2^-24 per primitive).  XC_AO_EXP=1 forms a r^2 in f64 and evaluates
// exp(-a r^2) = 2^-n exp(-(a r^2 - n ln 2)) with the reduced argument in f32 (~2 ulp of the
// f64 value).  Measured on B200: V_xc vs the reference's own f32
// xc_matrix 1.19e-6 -> 1.09e-6 of max|V| at N = 63, configs[1] f32 labels vs the reference
// f64 MAE 0.150 -> 0.160 meV (max 0.52 -> 0.43) - the f32 contractions dominate - at
// +0.31 ms (+16%) per XC iteration, so the f32 exponent stays.
#ifndef XC_AO_EXP
#define XC_AO_EXP 0
#endif

__device__ __forceinline__ float expneg_f32acc(double x) {
    const double n = rint(x * 1.4426950408889634);            // x / ln 2
    const float f = (float)fma(-n, 0.69314718055994531, x);    // |f| <= 0.35, error ~1e-16 * n
    return ldexpf(expf(-f), -(int)n);
}

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

// W-typed shell record: exponents, c_s, c_p (3 each); the f32 build adds -a log2(e) and -2a
// (3 each) so the AO loop is one ex2.approx and FMAs per primitive
template <typename W> constexpr int xc_swn() { return sizeof(W) == 4 ? 16 : 9; }   // f32: padded to four 16-byte loads

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// XC_MMAV=1 (default): the f32 build's main bucket (N 49..64, 64-point sub-blocks) runs the
// V += phi wv^T contraction on the tensor cores: mma.sync m16n8k8 TF32 with the 3xTF32 split
// (x = hi + lo, hi rounded to TF32, lo the exact f32 remainder; hi*lo + lo*hi + hi*hi), one
// sub-block accumulated by the MMA from zero and added to the CTA's sums in round-to-nearest
// f32 (the tensor core's own accumulation truncates; over a CTA's 2048 points that bias took
// the V_xc error against the reference's f32 xc_matrix from 1.3e-6 to 3.8e-6 of max|V|; with
// the two levels it is 1.4e-6).  The FFMA2 formulation of that phase is bound by
// shared-memory wavefronts (every 16-byte operand load of a 4 x 4 register tile is four
// wavefronts for 16 FMAs per thread: 64 FMA per wavefront against 128 FMA per clock of the
// FP32 pipe); ldmatrix fragments feed 12 MMAs (12 K FMAs) from 12 wavefronts.  Measured on
// B200: mma.sync TF32 276 TFLOP/s = 4x FFMA (tools/probe/mma_probe.cu), so with three MMAs
// per product the phase gains 27% (4.7k -> 3.5k cycles per sub-block) and the kernel 2%
// (1.638 -> 1.603 ms per iteration); the tcgen05 path (umma.cuh, k_xc_mma) would need the
// AO planes in SWIZZLE_128B K-major tiles, which the FFMA phases cannot read conflict free.
#ifndef XC_MMAV
#define XC_MMAV 1
#endif
#ifndef XC_WV4
#define XC_WV4 1       // f32 build: wv phase with four points per thread (16-byte loads / stores)
#endif
// XC_MMAT=1: the same bucket also runs t = phi^T rho on the tensor cores (see the t phase).
// Measured on B200 and kept off: kernel 1.60 -> 1.55 ms per iteration, but n = sum_nu t phi
// inherits the truncating accumulation of a 24-MMA chain and the truncated lo parts as a bias
// of one sign: E_xc error against the reference's f32 xc_matrix 2.3e-6 -> 2.0e-5 Ha at N = 63
// (test bound 6e-6); flushing the MMA accumulators every K step in round-to-nearest f32 would
// cost the gain.
#ifndef XC_MMAT
#define XC_MMAT 0
#endif
__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
// x = hi + lo: hi = x rounded to TF32, lo = the f32 remainder (the MMA reads its top 19 bits)
__device__ __forceinline__ void tf32_split(uint32_t x, uint32_t &hi, uint32_t &lo) {
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(__uint_as_float(x)));
    lo = __float_as_uint(__uint_as_float(x) - __uint_as_float(hi));
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
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
    // shell records: centres [nsh][3] f64 (for the point - centre difference), exponents and
    // coefficients [nsh][9] in W (no per-use f64 -> f32 conversions), (ao << 1 | kind) [nsh]
    static size_t bytes(int nsh) { return shd + (XC_SHD_D * sizeof(double) + xc_swn<W>() * sizeof(W) + sizeof(int)) * (size_t)nsh; }
};

template <typename W, int NQ, int BP>
__device__ __forceinline__ void xc_eval_phi(W *phi, const double *pt, const double *shd, const W *shw,
                                            const int *shi, int nsh, int nb) {
    constexpr int NP = 4 * NQ, PL = NP * BP;
    static_assert(XC_THREADS % BP == 0, "a thread keeps one point for all its shells");
    const int p = threadIdx.x % BP;                    // this thread's point (fixed), in registers
    const double qx = pt[4 * p], qy = pt[4 * p + 1], qz = pt[4 * p + 2];
#pragma unroll kXcAoUnr
    for (int t = threadIdx.x; t < BP * nsh; t += XC_THREADS) {
        const int sh = t / BP;
        const double *r = shd + XC_SHD_D * sh;
        // the shell's constants (warp-uniform): four 16-byte loads in the f32 build instead of 13 scalar ones
        W f[xc_swn<W>()];
        {
            const W *fp_ = shw + xc_swn<W>() * sh;
            if constexpr (sizeof(W) == 4) {
                float q0[4], q1[4], q2[4], q3[4];
                Vec4<float>::ld((const float *)fp_, q0); Vec4<float>::ld((const float *)fp_ + 4, q1);
                Vec4<float>::ld((const float *)fp_ + 8, q2); Vec4<float>::ld((const float *)fp_ + 12, q3);
#pragma unroll
                for (int k = 0; k < 4; ++k) { f[k] = q0[k]; f[4 + k] = q1[k]; f[8 + k] = q2[k]; f[12 + k] = q3[k]; }
            } else {
#pragma unroll
                for (int k = 0; k < xc_swn<W>(); ++k) f[k] = fp_[k];
            }
        }
        int kao;
        if constexpr (sizeof(W) == 4) kao = __float_as_int(f[15]);     // (ao << 1 | kind) rides in the record's pad slot
        else kao = shi[sh];
        const int kind = kao & 1, ao = kao >> 1;
        W v[4][4];  // [plane][component]
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) v[a][c] = (W)0;
        if (p < nb) {
            const double2 rxy = *reinterpret_cast<const double2 *>(r);     // 48-byte records: 16-byte aligned
            const double dxd = qx - rxy.x, dyd = qy - rxy.y, dzd = qz - r[2];
            const double r2d = dxd * dxd + dyd * dyd + dzd * dzd;
            const W dx = (W)dxd, dy = (W)dyd, dz = (W)dzd;
            const W r2 = (W)r2d;
            constexpr W kCut = sizeof(W) == 4 ? (W)88 : (W)745;
            // unless every primitive underflows (exponents descend, f[2] is the smallest; the
            // AO values and gradients then stay exactly zero, as the loop would give: core
            // shells far from the sub-block's points)
            if (f[2] * r2 < kCut) {
            W bs = 0, ds = 0, bp = 0, dp = 0;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const W a = f[k];
                const W ar = a * r2;
                W e, m2a;
                if constexpr (sizeof(W) == 4) {
                    if (XC_AO_EXP) {
                        const double ard = r[3 + k] * r2d;
                        e = ard < (double)kCut ? expneg_f32acc(ard) : (W)0;
                    } else {
                        // exp(-a r^2) = 2^(-a log2(e) r^2); ex2.approx (~2 ulp) flushes the
                        // underflowing primitives to zero, as the cut-off did
                        e = ex2_approx(f[9 + k] * r2);
                    }
                    m2a = f[12 + k];
                } else {
                    e = ar < kCut ? exp(-ar) : (W)0;
                    m2a = (W)-2 * a;
                }
                bs += f[3 + k] * e;
                ds += f[3 + k] * m2a * e;
                bp += f[6 + k] * e;
                dp += f[6 + k] * m2a * e;
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
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {   // fully unrolled: v stays in registers
            if (c > 0 && !kind) break;
            const int o = swz<BP>(ao + c, p);
#pragma unroll
            for (int a = 0; a < 4; ++a) phi[a * PL + o] = v[a][c];
        }
    }
}

template <typename W, int NQ, int BP>
__global__ void __launch_bounds__(XC_THREADS, 2) k_xc(DevBatch b, const int *ctas) {
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
    W *shw = (W *)(shd + XC_SHD_D * nsh);
    int *shi = (int *)(shw + xc_swn<W>() * nsh);
    const int tid = threadIdx.x;
    const double *rg = b.rho + b.m_mat0[m];
    // tensor-core t phase: rho is kept with its columns grouped by residue mod 4 (column nu at
    // 16 (nu & 3) + (nu >> 2)) and its 16-byte groups swizzled by the row quad like the AO planes,
    // so that the MMA fragments below are conflict-free scalar loads
    constexpr bool MMAT = XC_MMAT && XC_MMAV && sizeof(W) == 4 && NQ == 16 && BP == 64;
    for (int t = tid; t < NP * NP; t += XC_THREADS) {
        const int r = t / NP, c = t % NP;
        const W v = (r < N && c < N) ? (W)rg[r * N + c] : (W)0;
        if constexpr (MMAT) rho[swz<BP>(r, 16 * (c & 3) + (c >> 2))] = v;
        else rho[t] = v;
    }
    for (int t = tid; t < 4 * PL; t += XC_THREADS) phi[t] = (W)0;
    for (int sh = tid; sh < nsh; sh += XC_THREADS) {
        const int gsh = s0 + sh;
        double *r = shd + XC_SHD_D * sh;
        W *f = shw + xc_swn<W>() * sh;
        const double *A = b.a_xyz + 3 * b.s_atom[gsh];
        for (int d = 0; d < 3; ++d) {
            r[d] = A[d];
            r[3 + d] = b.s_exp[3 * gsh + d];
            f[d] = (W)b.s_exp[3 * gsh + d];
            f[3 + d] = (W)b.s_cs[3 * gsh + d];
            f[6 + d] = (W)b.s_cp[3 * gsh + d];
            if constexpr (sizeof(W) == 4) {
                f[9 + d] = (W)(-1.4426950408889634 * b.s_exp[3 * gsh + d]);
                f[12 + d] = (W)(-2.0 * b.s_exp[3 * gsh + d]);
                f[15] = __int_as_float((b.s_ao[gsh] << 1) | (b.s_kind[gsh] & 1));   // pad slot of the 16-float record
            }
        }
        shi[sh] = (b.s_ao[gsh] << 1) | (b.s_kind[gsh] & 1);
    }
    // V accumulators: f32 keeps two partial sums (even / odd points of each 4-point chunk)
    // so every update is one packed FFMA2; f64 one DFMA chain
    using VA = typename std::conditional<sizeof(W) == 4, float2, double>::type;
    // tensor-core V phase (see XC_MMAV): warp w owns the 16 AO rows a = 4 g + (w >> 1) (g = 0..15:
    // rows of one residue mod 4, so that the 8 row addresses of an ldmatrix tile fall in 8
    // different row quads = 8 different swizzle keys = no bank conflict) and the 32 columns
    // c = 4 (8 (w & 1) + g') + j', g' = 0..7, j' = 0..3 (four n8 tiles)
    constexpr bool MMAV = XC_MMAV && sizeof(W) == 4 && NQ == 16 && BP == 64;
    constexpr int TJA = MMAV ? 1 : TJ;
    VA acc[TJA][4][4];
    float vacc[4][4];                        // MMAV: [n tile j'][c0..c3]
#pragma unroll
    for (int j = 0; j < TJA; ++j)
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if constexpr (sizeof(W) == 4) acc[j][a][c] = make_float2(0.f, 0.f);
                else acc[j][a][c] = 0.0;
            }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) vacc[a][c] = 0.f;
    // per-lane ldmatrix row addresses (byte addresses in shared memory) and swizzle terms
    uint32_t mA = 0, mB0 = 0, mB1 = 0;
    int xA = 0, xB = 0;
    if constexpr (MMAV) {
        const int lane = tid & 31, wp = tid >> 5, l7 = lane & 7, id = lane >> 3;
        const int quadA = l7 + 8 * (id & 1);                       // A: matrices (half, kh) = (id & 1, id >> 1)
        mA = (uint32_t)__cvta_generic_to_shared(phi + (4 * quadA + (wp >> 1)) * BP);
        xA = quadA ^ (id >> 1);
        const int quadB = 8 * (wp & 1) + l7;                       // B: matrices (n tile, kh) = (2 x + (id >> 1), id & 1)
        mB0 = (uint32_t)__cvta_generic_to_shared(wv + (4 * quadB + (id >> 1)) * BP);
        mB1 = (uint32_t)__cvta_generic_to_shared(wv + (4 * quadB + 2 + (id >> 1)) * BP);
        xB = quadB ^ (id & 1);
    }
    double e_acc = 0.0;
    int bad = 0;
    const int pg = tid / LG, lg = tid % LG;
    const int64_t p0 = b.xc_p0[cta], p1 = b.xc_p1[cta];
#ifdef XC_PHASES
    long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tck = clock64();
    int nsub = 0;
#define XP(k) do { const long long t_ = clock64(); ph[k] += t_ - tck; tck = t_; } while (0)
#else
#define XP(k) do { } while (0)
#endif
    // the points of a sub-block are loaded into pt[] during the previous sub-block's V phase
    // (pt is not read there), so the global-load latency is off the critical path
    auto load_pts = [&](int64_t sb_) {
        if (tid < BP && sb_ < p1) {
            const int nb_ = (int)min((int64_t)BP, p1 - sb_);
            const int64_t gi = sb_ + min(tid, nb_ - 1);
            pt[4 * tid] = b.g_xyz[3 * gi];
            pt[4 * tid + 1] = b.g_xyz[3 * gi + 1];
            pt[4 * tid + 2] = b.g_xyz[3 * gi + 2];
            pt[4 * tid + 3] = tid < nb_ ? b.g_w[gi] : 0.0;
        }
    };
    load_pts(p0);
    for (int64_t sb = p0; sb < p1; sb += BP) {
        const int nb = (int)min((int64_t)BP, p1 - sb);
#ifdef XC_PHASES
        ++nsub;
#endif
        __syncthreads();                                   // previous sub-block consumed, pt loaded
        XP(5);
        XP(0);
        xc_eval_phi<W, NQ, BP>(phi, pt, shd, shw, shi, nsh, nb);
        __syncthreads();
        XP(1);
        if constexpr (MMAT) {
            // ---- t[p][nu] = sum_mu phi[mu][p] rho[mu][nu] on the tensor cores (3xTF32), then n and
            // grad n from the accumulator fragments.  M = points: warp w owns the 16 points of m tile
            // w & 3 and the 32 columns nu = 4 (8 (w >> 2) + n) + j' (n = 0..7 inside n tile j' = 0..3).
            // K = AOs in a permuted order: step (h, j) covers mu = 4 q + j for the row quads q =
            // 8 h + 2 k (fragment columns k = 0..3) and 8 h + 2 k + 1 (k = 4..7).  The four rows a
            // lane group reads in one load then sit in quads whose swizzle keys differ in bits 1-2,
            // the 8 consecutive columns span two 16-byte groups: 32 different banks (A from the AO
            // plane, B from the residue-grouped rho, and the AO values of the epilogue alike).
            const int lane = tid & 31, wp = tid >> 5, g = lane >> 2, tq = lane & 3;
            const int mt = wp & 3, nh = wp >> 2;
            const int gA = 4 * mt + (g >> 2), gl = g & 3;        // column group / offset of point 16 mt + g
            const int gB = 2 * nh + (g >> 2);                    // + 4 j': column group of rho' column 16 j' + 8 nh + g
            float tacc[4][4];
#pragma unroll
            for (int n = 0; n < 4; ++n)
#pragma unroll
                for (int k = 0; k < 4; ++k) tacc[n][k] = 0.f;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int q0 = 8 * (ks >> 2) + 2 * tq, q1 = q0 + 1, jr = ks & 3;
                const float *pa0 = (const float *)phi + (4 * q0 + jr) * BP, *pa1 = (const float *)phi + (4 * q1 + jr) * BP;
                const float *pb0 = (const float *)rho + (4 * q0 + jr) * NP, *pb1 = (const float *)rho + (4 * q1 + jr) * NP;
                uint32_t a[4], ah[4], al[4];
                a[0] = __float_as_uint(pa0[(((gA ^ q0) & 15) << 2) | gl]);
                a[1] = __float_as_uint(pa0[((((gA + 2) ^ q0) & 15) << 2) | gl]);
                a[2] = __float_as_uint(pa1[(((gA ^ q1) & 15) << 2) | gl]);
                a[3] = __float_as_uint(pa1[((((gA + 2) ^ q1) & 15) << 2) | gl]);
#pragma unroll
                for (int k = 0; k < 4; ++k) tf32_split(a[k], ah[k], al[k]);
#pragma unroll
                for (int n = 0; n < 4; ++n) {
                    uint32_t b0h, b0l, b1h, b1l;
                    tf32_split(__float_as_uint(pb0[((((4 * n + gB) ^ q0) & 15) << 2) | gl]), b0h, b0l);
                    tf32_split(__float_as_uint(pb1[((((4 * n + gB) ^ q1) & 15) << 2) | gl]), b1h, b1l);
                    mma_tf32(tacc[n], ah, b0l, b1l);
                    mma_tf32(tacc[n], al, b0h, b1h);
                    mma_tf32(tacc[n], ah, b0h, b1h);
                }
            }
            // accumulator fragment of n tile j': c0, c1 = (point g, nu(2 tq), nu(2 tq + 1)), c2, c3 = (point g + 8, same)
            float h8[8];                                        // index 2 * component + point half
#pragma unroll
            for (int k = 0; k < 8; ++k) h8[k] = 0.f;
#pragma unroll
            for (int n = 0; n < 4; ++n)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int qe = 8 * nh + 2 * tq + e;
                    const float *pr = (const float *)phi + (4 * qe + n) * BP;
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        const float *pp = pr + (((((gA + 2 * hf) ^ qe) & 15) << 2) | gl);
                        const float tv = tacc[n][2 * hf + e];
                        h8[hf] = fmaf(tv, pp[0], h8[hf]);
                        h8[2 + hf] = fmaf(tv, pp[PL], h8[2 + hf]);
                        h8[4 + hf] = fmaf(tv, pp[2 * PL], h8[4 + hf]);
                        h8[6 + hf] = fmaf(tv, pp[3 * PL], h8[6 + hf]);
                    }
                }
            // sum over the four lanes of a point pair (transposing butterfly): lane tq ends with
            // point half tq & 1 and components (tq >> 1) & 1 and 2 + ((tq >> 1) & 1)
#pragma unroll
            for (int s_ = 0; s_ < 2; ++s_) {
                const int o = 1 << s_;
                const bool up = (tq & o) != 0;
#pragma unroll
                for (int k = 0; k < (4 >> s_); ++k) {
                    const float mine = up ? h8[2 * k + 1] : h8[2 * k], other = up ? h8[2 * k] : h8[2 * k + 1];
                    h8[k] = mine + __shfl_xor_sync(0xffffffffu, other, o);
                }
            }
            // the two warps that share an m tile (nu halves) leave their sums side by side; the
            // functional adds them
            float *part = (float *)dn;                          // [2][BP][4] floats
            const int pp_ = 16 * mt + g + 8 * (tq & 1), cmp = (tq >> 1) & 1;
            part[(nh * BP + pp_) * 4 + cmp] = h8[0];
            part[(nh * BP + pp_) * 4 + 2 + cmp] = h8[1];
        } else
        {   // ---- t = phi^T rho for 4 points x 4 AOs, then n and grad n partials
            W n4[4] = {0, 0, 0, 0}, g4[3][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
            for (int j = 0; j < QJ; ++j) {
                const int q = lg + j * LG;
                if constexpr (sizeof(W) == 4) {
                    // f32: Blackwell packed FFMA2 (two FMAs per instruction; the same per-element
                    // fma and order as the scalar code below): t2[h][c] = (t[2h][c], t[2h+1][c])
                    if (q < NQ) {
                        float2 t2[2][4];
#pragma unroll
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int c = 0; c < 4; ++c) t2[h][c] = make_float2(0.f, 0.f);
#pragma unroll kXcTunr
                        for (int kq = 0; kq < (N + 3) / 4; ++kq) {
                            const W *pr = phi + 4 * kq * BP + (((pg ^ kq) & (BP / 4 - 1)) << 2);
                            const W *rr = rho + 4 * kq * NP + 4 * q;
#pragma unroll
                            for (int r = 0; r < 4; ++r) {
                                const float4 f = *reinterpret_cast<const float4 *>(pr + r * BP);
                                const float4 r4 = *reinterpret_cast<const float4 *>(rr + r * NP);
                                const float2 f01 = make_float2(f.x, f.y), f23 = make_float2(f.z, f.w);
                                const float rc[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
                                for (int c = 0; c < 4; ++c) {
                                    t2[0][c] = __ffma2_rn(f01, make_float2(rc[c], rc[c]), t2[0][c]);
                                    t2[1][c] = __ffma2_rn(f23, make_float2(rc[c], rc[c]), t2[1][c]);
                                }
                            }
                        }
                        const int qo = 4 * q * BP + (((pg ^ q) & (BP / 4 - 1)) << 2);   // rows 4q..4q+3
                        float2 n2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
                        float2 g2[3][2] = {{make_float2(0.f, 0.f), make_float2(0.f, 0.f)},
                                           {make_float2(0.f, 0.f), make_float2(0.f, 0.f)},
                                           {make_float2(0.f, 0.f), make_float2(0.f, 0.f)}};
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            float4 fp[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) fp[k] = *reinterpret_cast<const float4 *>(phi + k * PL + qo + c * BP);
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const float2 f0 = h ? make_float2(fp[0].z, fp[0].w) : make_float2(fp[0].x, fp[0].y);
                                n2[h] = __ffma2_rn(t2[h][c], f0, n2[h]);
#pragma unroll
                                for (int d = 0; d < 3; ++d) {
                                    const float2 fd = h ? make_float2(fp[d + 1].z, fp[d + 1].w)
                                                        : make_float2(fp[d + 1].x, fp[d + 1].y);
                                    g2[d][h] = __ffma2_rn(t2[h][c], fd, g2[d][h]);
                                }
                            }
                        }
                        n4[0] += n2[0].x; n4[1] += n2[0].y; n4[2] += n2[1].x; n4[3] += n2[1].y;
#pragma unroll
                        for (int d = 0; d < 3; ++d) {
                            g4[d][0] += g2[d][0].x; g4[d][1] += g2[d][0].y;
                            g4[d][2] += g2[d][1].x; g4[d][3] += g2[d][1].y;
                        }
                    }
                } else if (q < NQ) {
                    W t[4][4];
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int c = 0; c < 4; ++c) t[a][c] = (W)0;
                    // k ascending in groups of 4 rows: the swizzled column of a 4-row group is
                    // one XOR (rows >= N are zero in phi and rho, so the tail adds exact zeros)
#pragma unroll 2
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
            // Sum over the LG lanes that share the point group: a transposing butterfly.  At each of
            // the first four steps a lane keeps the half of its values whose index bit s matches its
            // lane bit s and hands the other half to its partner, so the 16 values per lane shrink to
            // one (15 shuffles and adds instead of 64): after step s, h[k] is value index
            // (k << (s + 1)) | (lane's low s + 1 bits), summed over the lanes differing in those bits.
            // Lane lg ends with value index lg & 15 = 4 * component + point (LG = 32: one more exchange).
            {
                W h[16];
#pragma unroll
                for (int a = 0; a < 4; ++a) { h[a] = n4[a]; h[4 + a] = g4[0][a]; h[8 + a] = g4[1][a]; h[12 + a] = g4[2][a]; }
#pragma unroll
                for (int s_ = 0; s_ < 4; ++s_) {
                    const int o = 1 << s_;
                    const bool up = (lg & o) != 0;
#pragma unroll
                    for (int k = 0; k < (8 >> s_); ++k) {
                        const W mine = up ? h[2 * k + 1] : h[2 * k], other = up ? h[2 * k] : h[2 * k + 1];
                        h[k] = mine + __shfl_xor_sync(0xffffffffu, other, o);
                    }
                }
                W r = h[0];
                if constexpr (LG == 32) r += __shfl_xor_sync(0xffffffffu, r, 16);
                if (lg < 16) {
                    const int comp = lg >> 2, a = lg & 3;
                    dn[4 * (4 * pg + a) + comp] = comp == 0 ? (double)r : (double)(W)(2 * r);
                }
            }
        }
        __syncthreads();
        XP(2);
        if (tid < 3 * BP) {   // ---- functional (f64): parts on three thread groups, one point each
            const int pt_i = tid % BP, part = tid / BP;
            double n, gxd, gyd, gzd, sig = 0.0;
            if constexpr (MMAT) {
                const float4 pa = reinterpret_cast<const float4 *>(dn)[pt_i], pb = reinterpret_cast<const float4 *>(dn)[BP + pt_i];
                n = (double)(pa.x + pb.x);
                gxd = (double)(2 * (pa.y + pb.y)); gyd = (double)(2 * (pa.z + pb.z)); gzd = (double)(2 * (pa.w + pb.w));
            } else {
                const double *dq = dn + 4 * pt_i;
                n = dq[0]; gxd = dq[1]; gyd = dq[2]; gzd = dq[3];
            }
            {
                const double gx = gxd, gy = gyd, gz = gzd;
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
            if (ok) {
                const double gx = gxd, gy = gyd, gz = gzd;
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
        XP(3);
        if constexpr (XC_WV4 && sizeof(W) == 4) {
            // ---- wv = a phi + b . grad phi, four points per thread: the thread's 4-point column group is
            // fixed (its four coefficient vectors stay in registers), rows in steps of XC_THREADS / (BP / 4);
            // 16-byte loads and stores (a quarter warp covers 128 contiguous bytes of one row)
            constexpr int NG = BP / 4, RS = XC_THREADS / NG;
            const int cg = tid % NG;
            float c0[4], c1[4], c2[4], c3[4];
            Vec4<float>::ld((const float *)dw + 4 * cg, c0);
            Vec4<float>::ld((const float *)dw + BP + 4 * cg, c1);
            Vec4<float>::ld((const float *)dw + 2 * BP + 4 * cg, c2);
            Vec4<float>::ld((const float *)dw + 3 * BP + 4 * cg, c3);
#pragma unroll 2
            for (int row = tid / NG; row < NP; row += RS) {
                const int o = row * BP + (((cg ^ (row >> 2)) & (NG - 1)) << 2);
                float f0[4], f1[4], f2[4], f3[4];
                Vec4<float>::ld((const float *)phi + o, f0);
                Vec4<float>::ld((const float *)phi + PL + o, f1);
                Vec4<float>::ld((const float *)phi + 2 * PL + o, f2);
                Vec4<float>::ld((const float *)phi + 3 * PL + o, f3);
                float4 r;
                r.x = c0[0] * f0[0] + c1[0] * f1[0] + c2[0] * f2[0] + c3[0] * f3[0];
                r.y = c0[1] * f0[1] + c1[1] * f1[1] + c2[1] * f2[1] + c3[1] * f3[1];
                r.z = c0[2] * f0[2] + c1[2] * f1[2] + c2[2] * f2[2] + c3[2] * f3[2];
                r.w = c0[3] * f0[3] + c1[3] * f1[3] + c2[3] * f2[3] + c3[3] * f3[3];
                *reinterpret_cast<float4 *>((float *)wv + o) = r;
            }
        } else
        {   // ---- wv = a phi + b . grad phi; this thread's point is fixed (XC_THREADS % BP == 0)
            static_assert(XC_THREADS % BP == 0, "fixed point per thread");
            const int p = tid % BP;
            const W d0 = dw[p], d1 = dw[BP + p], d2 = dw[2 * BP + p], d3 = dw[3 * BP + p];
#pragma unroll kXcWvUnr
            for (int row = tid / BP; row < NP; row += XC_THREADS / BP) {
                const int o = swz<BP>(row, p);
                wv[o] = d0 * phi[o] + d1 * phi[PL + o] + d2 * phi[2 * PL + o] + d3 * phi[3 * PL + o];
            }
        }
        __syncthreads();
        XP(4);
        load_pts(sb + BP);
        if constexpr (MMAV) {                              // ---- V += phi wv^T on the tensor cores (3xTF32)
            // the MMA accumulates one sub-block (64 points) from zero; the CTA-lifetime sums are
            // round-to-nearest adds (the tensor core's own f32 accumulation truncates: over the
            // CTA's 2048 points that bias tripled the V_xc error)
            float sacc[4][4];
#pragma unroll
            for (int n = 0; n < 4; ++n)
#pragma unroll
                for (int k = 0; k < 4; ++k) sacc[n][k] = 0.f;
#pragma unroll
            for (int ks = 0; ks < BP / 8; ++ks) {          // 8 points per step: column groups 2 ks, 2 ks + 1
                uint32_t a[4], b0[4], b1[4];
                ldsm4(mA + 16u * (uint32_t)(((2 * ks) ^ xA) & (BP / 4 - 1)), a);
                ldsm4(mB0 + 16u * (uint32_t)(((2 * ks) ^ xB) & (BP / 4 - 1)), b0);    // n tiles 0, 1: (b0, b1) each
                ldsm4(mB1 + 16u * (uint32_t)(((2 * ks) ^ xB) & (BP / 4 - 1)), b1);    // n tiles 2, 3
                uint32_t ah[4], al[4], bh[8], bl[8];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    tf32_split(a[k], ah[k], al[k]);
                    tf32_split(b0[k], bh[k], bl[k]);
                    tf32_split(b1[k], bh[4 + k], bl[4 + k]);
                }
#pragma unroll
                for (int n = 0; n < 4; ++n) {
                    mma_tf32(sacc[n], ah, bl[2 * n], bl[2 * n + 1]);
                    mma_tf32(sacc[n], al, bh[2 * n], bh[2 * n + 1]);
                    mma_tf32(sacc[n], ah, bh[2 * n], bh[2 * n + 1]);
                }
            }
#pragma unroll
            for (int n = 0; n < 4; ++n)
#pragma unroll
                for (int k = 0; k < 4; ++k) vacc[n][k] += sacc[n][k];
        } else
#pragma unroll
        for (int j = 0; j < TJ; ++j) {                     // ---- V += phi wv^T, 4 x 4 tiles
            const int T = tid + j * XC_THREADS;
            if (T < NT) {
                const int qa = T / NQ, qb = T % NQ;
                const W *pa = phi + 4 * qa * BP, *pb = wv + 4 * qb * BP;   // rows 4qa.., 4qb..
#pragma unroll kXcVunr
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
                        for (int c = 0; c < 4; ++c) {
                            if constexpr (sizeof(W) == 4) {
                                acc[j][a][c] = __ffma2_rn(make_float2(fa[a][0], fa[a][1]),
                                                          make_float2(fb[c][0], fb[c][1]), acc[j][a][c]);
                                acc[j][a][c] = __ffma2_rn(make_float2(fa[a][2], fa[a][3]),
                                                          make_float2(fb[c][2], fb[c][3]), acc[j][a][c]);
                            } else {
#pragma unroll
                                for (int pp = 0; pp < 4; ++pp) acc[j][a][c] += fa[a][pp] * fb[c][pp];
                            }
                        }
                }
            }
        }
    }
#ifdef XC_PHASES
    if (blockIdx.x % 97 == 0 && tid == 0)
        printf("xcffma NQ %d cta %d sub %d: pts %lld phi %lld t %lld func %lld wv %lld V+loop %lld\n", NQ,
               blockIdx.x, nsub, ph[0], ph[1], ph[2], ph[3], ph[4], ph[5]);
#endif
#undef XP
    const int local = cta - b.m_xccta0[m];
    double *Vp = b.Vpart + b.m_V0[m] + (int64_t)local * N * N;
    if constexpr (MMAV) {
        // accumulator fragment: c0, c1 = (row g, cols 2t, 2t+1), c2, c3 = (row g + 8, same cols)
        const int lane = tid & 31, wp = tid >> 5, g = lane >> 2, t2 = 2 * (lane & 3);
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int mu = 4 * (g + 8 * (k >> 1)) + (wp >> 1);
                const int nu = 4 * (8 * (wp & 1) + t2 + (k & 1)) + n;
                if (mu < N && nu < N) Vp[mu * N + nu] = (double)vacc[n][k];
            }
    } else
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
                    if (mu < N && nu < N) {
                        if constexpr (sizeof(W) == 4) Vp[mu * N + nu] = (double)(acc[j][a][c].x + acc[j][a][c].y);
                        else Vp[mu * N + nu] = acc[j][a][c];
                    }
                }
        }
    }
    const double e = block_sum(e_acc, red);
    if (tid == 0) b.Epart[cta] = e;
    if (bad) atomicOr(b.status + m, DFTB_ST_XC_NONFINITE);
}

// ---------------------------------------------------------------------------- tensor cores
// f32 build: the two N^2-per-point contractions on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM), everything else as in k_xc.
//   t[p][nu]  = sum_mu phi[mu][p] rho[mu][nu]   M = 64 points, N = NP, K = NP AOs
//   V[mu][nu] += sum_p phi[mu][p] wv[nu][p]     M = 64 / 128 AOs, N = NP, K = BP points
// Precision: 3xTF32 (x = hi + lo, hi TF32 by round-to-nearest, lo the exact f32 remainder;
// hi*lo + lo*hi + hi*hi per product, f32 accumulation): measured 5e-7 of the largest
// element on random 64^3 products (tools/probe/umma_probe.cu); the reference's f32 path
// is f32 BLAS.  Operands are K-major SWIZZLE_128B tiles (umma.cuh), so phi is kept in two
// layouts: [mu][p] (V-phase A, and the FFMA consumers) and [p][mu] (t-phase A).
// The CTA runs NG independent pipelines ("groups" of 256 threads, own tiles, own TMEM
// accumulators and mbarriers, named barriers) over interleaved BP-point sub-blocks and
// shares the density tiles: while one group waits on its MMAs or runs its (latency-bound,
// f64) functional, the other computes AO values - the latency hiding of two CTAs per SM
// without the second copy of rho.  One elected thread per group issues the MMAs.
constexpr int XCG = 256;   // threads per group

template <int NQ, int BP, int NG>
struct XCM {
    static constexpr int NP = 4 * NQ;
    static constexpr int NSR = (NP + 31) / 32;     // 32-column segments of an AO-indexed row
    static constexpr int NSP = BP / 32;            // 32-column segments of a point-indexed row
    static constexpr int MV = NP <= 64 ? 64 : 128; // V-phase M
    static constexpr int RHO = (NP / 8) * NSR * 256;       // floats per tile buffer
    static constexpr int PHA = (BP / 8) * NSR * 256;       // [BP p rows][NP]  (M = 64 over-reads)
    static constexpr int PHV = (NP / 8) * NSP * 256;       // [NP rows][BP]
    static constexpr int GF = 2 * PHA + 7 * PHV;           // pha h/l, phv l/h, 3 dphi, wv h/l
    static constexpr int EQ = BP / 16;                     // lane quarters holding points
    static constexpr int NCS = NP / 2;                     // epilogue columns per warp
    static_assert(BP == 32 || BP == 64, "sub-block size");
    static_assert(4 * NP <= 256, "three t accumulators + V per group in 256 TMEM columns");
    static_assert((64 - BP) / 8 * NSR * 256 <= 7 * PHV, "t-phase over-read stays in the group's tiles");
    static_assert(MV == 64 || (128 - NP) / 8 * NSP * 256 <= 3 * PHV, "V-phase over-read stays in bounds");
    static constexpr size_t grp(int g) { return 2 * (size_t)RHO + (size_t)g * GF; }
    static constexpr size_t fend = 2 * (size_t)RHO + (size_t)NG * GF;
    // per-group scalars (bytes): pt [BP][4] f64, dn [BP][4] f64, fpt [10][BP] f64 (the
    // epilogue's [2][BP][4] f32 partials alias it), dw [4][BP] f32
    static constexpr size_t GS = 160 * BP;
    static constexpr size_t sc(int g) { return fend * 4 + (size_t)g * GS; }
    static constexpr size_t red = fend * 4 + NG * GS;      // [32] f64
    static constexpr size_t bars = red + 256;              // 2 NG mbarriers + TMEM base
    static constexpr size_t shd = bars + 64;
    // shell records: centres (f64, for the point - centre difference) and f32 exponents /
    // coefficients (no per-use conversions in the AO loop)
    static size_t bytes(int nsh) { return 1024 + shd + (8 * 3 + 4 * 10) * (size_t)nsh; }
};

__device__ __forceinline__ void gbar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int NQ, int BP, int NG>
__global__ void __launch_bounds__(NG * XCG, 1) k_xc_mma(DevBatch b, const int *ctas) {
    using L = XCM<NQ, BP, NG>;
    constexpr int NP = L::NP, NSR = L::NSR, NSP = L::NSP, MV = L::MV, NCS = L::NCS;
    constexpr int NT = NG * XCG;
    extern __shared__ __align__(16) unsigned char xsm_raw[];
    // 1 KB-aligned base by pointer arithmetic on the shared array (an integer round trip would
    // turn every access into a generic load / store)
    unsigned char *xsm = xsm_raw + ((1024u - (umma::saddr(xsm_raw) & 1023u)) & 1023u);
    float *fs = (float *)xsm;
    float *rho_h = fs, *rho_l = fs + L::RHO;
    double *red = (double *)(xsm + L::red), *shd = (double *)(xsm + L::shd);
    uint64_t *bars = (uint64_t *)(xsm + L::bars);
    uint32_t *tbase = (uint32_t *)(bars + 2 * NG);
    const int cta = ctas[blockIdx.x];
    const int m = b.xc_mol[cta];
    if (b.done[m]) return;
    const int N = b.m_nao[m];
    const int nsh = b.m_nshell[m], s0 = b.m_shell0[m];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // ---- setup: rho (K-major rows nu, cols mu) split, zeroed tiles, shell records
    const double *rg = b.rho + b.m_mat0[m];
    for (int t = tid; t < NP * NP; t += NT) {
        const int nu = t / NP, mu = t % NP;
        const float x = (nu < N && mu < N) ? (float)rg[mu * N + nu] : 0.f;
        const float h = umma::tf32_hi(x);
        const int o = umma::sw128(nu, mu, NSR);
        rho_h[o] = h;
        rho_l[o] = x - h;
    }
    for (int t = tid; t < NG * L::GF; t += NT) fs[L::grp(0) + t] = 0.f;
    float *shf = (float *)(shd + 3 * nsh);   // [nsh][10]: exps, cs, cp, (ao << 1 | kind) bits
    for (int sh = tid; sh < nsh; sh += NT) {
        const int gsh = s0 + sh;
        double *r = shd + 3 * sh;
        float *f = shf + 10 * sh;
        const double *A = b.a_xyz + 3 * b.s_atom[gsh];
        for (int d = 0; d < 3; ++d) {
            r[d] = A[d];
            f[d] = (float)b.s_exp[3 * gsh + d];
            f[3 + d] = (float)b.s_cs[3 * gsh + d];
            f[6 + d] = (float)b.s_cp[3 * gsh + d];
        }
        f[9] = __int_as_float((b.s_ao[gsh] << 1) | (b.s_kind[gsh] & 1));
    }
    if (warp == 0) umma::tmem_alloc(tbase, NG == 1 ? 256 : 512);
    if (tid == 0) {
        for (int k = 0; k < 2 * NG; ++k) umma::mbar_init(bars + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    // ---- this thread's group
    const int g = tid / XCG, tl = tid % XCG, wl = tl >> 5;
    const int gid = 1 + g, gfun = 1 + NG + g;                 // named barriers
    float *G = fs + L::grp(g);
    float *pha_h = G, *pha_l = G + L::PHA, *phv_l = G + 2 * L::PHA, *phv_h = phv_l + L::PHV;
    float *dphi = phv_h + L::PHV, *wv_h = dphi + 3 * L::PHV, *wv_l = wv_h + L::PHV;
    double *pt = (double *)(xsm + L::sc(g)), *dn = pt + 4 * BP, *fpt = dn + 4 * BP;
    float *part = (float *)fpt, *dw = (float *)(fpt + 10 * BP);
    uint64_t *bar_t = bars + 2 * g, *bar_v = bar_t + 1;
    // TMEM per group: three t accumulators (hi*lo, lo*hi, hi*hi: three independent MMA chains
    // instead of one dependent chain of 3 NP/8 MMAs), then V
    const uint32_t TT = *tbase + 256 * g, TV = TT + 3 * NP;
    const uint32_t sbr = NSR * 1024, sbp = NSP * 1024;
    const uint64_t dpha_h = umma::desc_sw128(umma::saddr(pha_h), sbr), dpha_l = umma::desc_sw128(umma::saddr(pha_l), sbr);
    const uint64_t drho_h = umma::desc_sw128(umma::saddr(rho_h), sbr), drho_l = umma::desc_sw128(umma::saddr(rho_l), sbr);
    const uint64_t dphv_h = umma::desc_sw128(umma::saddr(phv_h), sbp), dphv_l = umma::desc_sw128(umma::saddr(phv_l), sbp);
    const uint64_t dwv_h = umma::desc_sw128(umma::saddr(wv_h), sbp), dwv_l = umma::desc_sw128(umma::saddr(wv_l), sbp);
    constexpr uint32_t IT = umma::idesc_tf32(64, NP), IV = umma::idesc_tf32(MV, NP);
    double e_acc = 0.0;
    int bad = 0;
    const int64_t p0 = b.xc_p0[cta], p1 = b.xc_p1[cta];
    int s = 0;
#ifdef XC_PHASES
    long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tck = clock64();
#define XPH(k) do { const long long t_ = clock64(); ph[k] += t_ - tck; tck = t_; } while (0)
#else
#define XPH(k) do { } while (0)
#endif
    for (int64_t sb = p0 + (int64_t)g * BP; sb < p1; sb += (int64_t)NG * BP, ++s) {
        const int nb = (int)min((int64_t)BP, p1 - sb);
        if (s > 0 && wl == 0) umma::mbar_wait(bar_v, (uint32_t)((s - 1) & 1));   // V MMAs done with phi, wv
        if (tl < BP) {
            const int64_t gi = sb + min(tl, nb - 1);
            pt[4 * tl] = b.g_xyz[3 * gi];
            pt[4 * tl + 1] = b.g_xyz[3 * gi + 1];
            pt[4 * tl + 2] = b.g_xyz[3 * gi + 2];
            pt[4 * tl + 3] = tl < nb ? b.g_w[gi] : 0.0;
        }
        gbar(gid, XCG);
        XPH(0);
        // ---- AO values and gradients (f32) -> both phi layouts (hi / lo) + gradient planes
        for (int t = tl; t < BP * nsh; t += XCG) {
            const int p = t % BP, sh = t / BP;
            const double *r = shd + 3 * sh;
            const float *f = shf + 10 * sh;
            const int kao = __float_as_int(f[9]), kind = kao & 1, ao = kao >> 1;
            float v[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < 4; ++c) v[a][c] = 0.f;
            if (p < nb) {
                const double *q = pt + 4 * p;
                const float dx = (float)(q[0] - r[0]), dy = (float)(q[1] - r[1]), dz = (float)(q[2] - r[2]);
                const float r2 = dx * dx + dy * dy + dz * dz;
                float bs = 0, ds = 0, bp = 0, dp = 0;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const float a = f[k];
                    const float ar = a * r2;
                    const float e = ar < 88.f ? expf(-ar) : 0.f;
                    const float m2a = -2.f * a;
                    bs += f[3 + k] * e;
                    ds += f[3 + k] * m2a * e;
                    bp += f[6 + k] * e;
                    dp += f[6 + k] * m2a * e;
                }
                const float rel[3] = {dx, dy, dz};
                v[0][0] = bs;
#pragma unroll
                for (int d = 0; d < 3; ++d) v[d + 1][0] = rel[d] * ds;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    v[0][1 + c] = rel[c] * bp;
#pragma unroll
                    for (int d = 0; d < 3; ++d) v[d + 1][1 + c] = (c == d ? bp : 0.f) + rel[c] * rel[d] * dp;
                }
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (c > 0 && !kind) break;
                const float x = v[0][c], h = umma::tf32_hi(x);
                const int ov = umma::sw128(ao + c, p, NSP), oa = umma::sw128(p, ao + c, NSR);
                phv_h[ov] = h;
                phv_l[ov] = x - h;
                pha_h[oa] = h;
                pha_l[oa] = x - h;
#pragma unroll
                for (int d = 0; d < 3; ++d) dphi[d * L::PHV + ov] = v[d + 1][c];
            }
        }
        umma::fence_async_smem();
        umma::fence_before();
        gbar(gid, XCG);
        XPH(1);
        if (tl == 0) {   // ---- t = phi^T rho on the tensor cores
            umma::fence_after();
#pragma unroll
            for (int k = 0; k < NP / 8; ++k) {
                const uint64_t ah = umma::desc_step(dpha_h, k), al = umma::desc_step(dpha_l, k);
                const uint64_t bh = umma::desc_step(drho_h, k), bl = umma::desc_step(drho_l, k);
                umma::mma_tf32(TT, ah, bl, IT, k > 0);
                umma::mma_tf32(TT + NP, al, bh, IT, k > 0);
                umma::mma_tf32(TT + 2 * NP, ah, bh, IT, k > 0);
            }
            umma::commit(bar_t);
        }
        if (wl == 0) umma::mbar_wait(bar_t, (uint32_t)(s & 1));
        gbar(gid, XCG);
        umma::fence_after();
        XPH(2);
        {   // ---- n, grad n partials: warp -> lane quarter q (points 16q..16q+15), column half c
            const int q = warp & 3, c = wl >> 2;
            if (q < L::EQ) {
                float tv[NCS];
#pragma unroll
                for (int j = 0; j < NCS / 16; ++j) {
                    float a16[16], b16[16], c16[16];
                    const uint32_t ta = TT + ((uint32_t)(32 * q) << 16) + (uint32_t)(c * NCS + 16 * j);
                    umma::tld16(ta, a16);
                    umma::tld16(ta + NP, b16);
                    umma::tld16(ta + 2 * NP, c16);
                    umma::tld_wait();
#pragma unroll
                    for (int i = 0; i < 16; ++i) tv[16 * j + i] = (a16[i] + b16[i]) + c16[i];
                }
                const int p = 16 * q + lane;
                if (lane < 16) {
                    float n = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;
#pragma unroll
                    for (int i = 0; i < NCS; ++i) {
                        const int o = umma::sw128(c * NCS + i, p, NSP);
                        const float f = phv_h[o] + phv_l[o];
                        n += tv[i] * f;
                        gx += tv[i] * dphi[o];
                        gy += tv[i] * dphi[L::PHV + o];
                        gz += tv[i] * dphi[2 * L::PHV + o];
                    }
                    float *pp = part + 4 * (c * BP + p);
                    pp[0] = n; pp[1] = gx; pp[2] = gy; pp[3] = gz;
                }
            }
        }
        umma::fence_before();
        gbar(gid, XCG);
        if (tl < BP) {   // fixed-order combine of the two column halves
            const float *pa = part + 4 * tl, *pb = part + 4 * (BP + tl);
            double *d = dn + 4 * tl;
            d[0] = (double)(pa[0] + pb[0]);
            d[1] = (double)(2.f * (pa[1] + pb[1]));
            d[2] = (double)(2.f * (pa[2] + pb[2]));
            d[3] = (double)(2.f * (pa[3] + pb[3]));
        }
        gbar(gid, XCG);
        XPH(3);
        if (tl < 3 * BP) {   // ---- functional (f64): three parts on three thread groups
            const int pt_i = tl % BP, prt = tl / BP;
            const double *dq = dn + 4 * pt_i;
            double n = dq[0], sig = 0.0;
            {
                const float gx = (float)dq[1], gy = (float)dq[2], gz = (float)dq[3];
                sig = (double)(gx * gx + gy * gy + gz * gz);
            }
            const bool ok = pt_i < nb && b3lyp_clamp(n, sig);
            if (prt == 1) {
                const VPart v = ok ? b3lyp_vwn(n) : VPart{0.0, 0.0};
                fpt[5 * BP + pt_i] = v.f2;
                fpt[6 * BP + pt_i] = v.v2;
            } else if (prt == 2) {
                const LPart l = ok ? b3lyp_lyp(n, sig) : LPart{0.0, 0.0, 0.0};
                fpt[7 * BP + pt_i] = l.f3;
                fpt[8 * BP + pt_i] = l.v3;
                fpt[9 * BP + pt_i] = l.w3;
            }
            XPart x{0.0, 0.0, 0.0, 0.0, 0.0};
            if (prt == 0 && ok) x = b3lyp_x(n, sig);
            gbar(gfun, 3 * BP);
            if (prt == 0) {
                if (ok) {
                    const double gx = dq[1], gy = dq[2], gz = dq[3];
                    const XCOut o = xc_combine(n, x, VPart{fpt[5 * BP + pt_i], fpt[6 * BP + pt_i]},
                                               LPart{fpt[7 * BP + pt_i], fpt[8 * BP + pt_i], fpt[9 * BP + pt_i]});
                    if (!(isfinite(o.exc) && isfinite(o.vrho) && isfinite(o.vsigma))) bad = 1;
                    const double w = pt[4 * pt_i + 3];
                    e_acc += w * n * (double)(float)o.exc;
                    const double ww = (double)(float)w;
                    const double a = (double)(float)(0.5 * ww * (double)(float)o.vrho);
                    const double bb = (double)(float)(2.0 * ww * (double)(float)o.vsigma);
                    dw[pt_i] = (float)a;
                    dw[BP + pt_i] = (float)(bb * gx);
                    dw[2 * BP + pt_i] = (float)(bb * gy);
                    dw[3 * BP + pt_i] = (float)(bb * gz);
                } else {
                    dw[pt_i] = dw[BP + pt_i] = dw[2 * BP + pt_i] = dw[3 * BP + pt_i] = 0.f;
                }
            }
        }
        gbar(gid, XCG);
        XPH(4);
        {   // ---- wv = a phi + b . grad phi (split); this thread's point is fixed
            const int p = tl % BP;
            const float d0 = dw[p], d1 = dw[BP + p], d2 = dw[2 * BP + p], d3 = dw[3 * BP + p];
            for (int nu = tl / BP; nu < NP; nu += XCG / BP) {
                const int o = umma::sw128(nu, p, NSP);
                const float w = d0 * (phv_h[o] + phv_l[o]) + d1 * dphi[o] + d2 * dphi[L::PHV + o] +
                                d3 * dphi[2 * L::PHV + o];
                const float h = umma::tf32_hi(w);
                wv_h[o] = h;
                wv_l[o] = w - h;
            }
        }
        umma::fence_async_smem();
        umma::fence_before();
        gbar(gid, XCG);
        if (tl == 0) {   // ---- V += phi wv^T on the tensor cores (accumulated in TMEM)
            umma::fence_after();
#pragma unroll
            for (int k = 0; k < BP / 8; ++k) {
                const uint64_t ah = umma::desc_step(dphv_h, k), al = umma::desc_step(dphv_l, k);
                const uint64_t bh = umma::desc_step(dwv_h, k), bl = umma::desc_step(dwv_l, k);
                umma::mma_tf32(TV, ah, bl, IV, (s > 0 || k > 0) ? 1u : 0u);
                umma::mma_tf32(TV, al, bh, IV, 1);
                umma::mma_tf32(TV, ah, bh, IV, 1);
            }
            umma::commit(bar_v);
        }
        XPH(5);
    }
#ifdef XC_PHASES
    if (blockIdx.x < 2 && tl == 0)
        printf("xc cta %d group %d subblocks %d: pts+wait %lld  phi %lld  tmma %lld  epi %lld  func %lld  wv+vmma %lld\n",
               blockIdx.x, g, s, ph[0], ph[1], ph[2], ph[3], ph[4], ph[5]);
#endif
    if (s > 0 && wl == 0) umma::mbar_wait(bar_v, (uint32_t)((s - 1) & 1));
    __syncthreads();
    umma::fence_after();
    // ---- V partial = sum of the groups' accumulators (fixed order) -> f64 global
    const int nsb = (int)((p1 - p0 + BP - 1) / BP);        // sub-blocks of the CTA; group k ran ceil((nsb - k) / NG)
    const int local = cta - b.m_xccta0[m];
    double *Vp = b.Vpart + b.m_V0[m] + (int64_t)local * N * N;
    {
        constexpr int NW = NT / 32, NSPL = NW / 4, CPW = NP / NSPL;   // column split over the warps
        const int q = warp & 3, c = warp >> 2;
        float acc[CPW];
#pragma unroll
        for (int i = 0; i < CPW; ++i) acc[i] = 0.f;
        for (int k = 0; k < NG; ++k) {
            if (k >= nsb) break;
            const uint32_t base = *tbase + 256 * k + 3 * NP + ((uint32_t)(32 * q) << 16) + (uint32_t)(c * CPW);
#pragma unroll
            for (int j = 0; j < CPW / 16; ++j) {
                float t16[16];
                umma::tld16(base + 16 * j, t16);
                umma::tld_wait();
#pragma unroll
                for (int i = 0; i < 16; ++i) acc[16 * j + i] += t16[i];
            }
            if constexpr (CPW % 16) {
                float t4[4];
                umma::tld4(base + (CPW / 16) * 16, t4);
                umma::tld_wait();
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[(CPW / 16) * 16 + i] += t4[i];
            }
        }
        const int mu = MV == 64 ? (lane < 16 ? 16 * q + lane : NP) : 32 * q + lane;
        if (mu < N)
#pragma unroll
            for (int i = 0; i < CPW; ++i) {
                const int nu = c * CPW + i;
                if (nu < N) Vp[mu * N + nu] = (double)acc[i];
            }
    }
    umma::fence_before();
    const double e = block_sum(e_acc, red);
    if (tid == 0) b.Epart[cta] = e;
    if (bad) atomicOr(b.status + m, DFTB_ST_XC_NONFINITE);
    if (warp == 0) {
        umma::fence_after();
        umma::tmem_free(*tbase, NG == 1 ? 256 : 512);
    }
}

template <int NQ, int BP, int NG>
static void launch_bucket_mma(const DevBatch &b, const int *ctas, int n, int nsh_max, cudaStream_t s) {
    const size_t sm = XCM<NQ, BP, NG>::bytes(nsh_max);
    smem_optin((const void *)k_xc_mma<NQ, BP, NG>);
    k_xc_mma<NQ, BP, NG><<<n, NG * XCG, sm, s>>>(b, ctas);
}

template <typename W, int NQ, int BP>
static void launch_bucket(const DevBatch &b, const int *ctas, int n, int nsh_max, cudaStream_t s) {
    const size_t sm = XCL<W, NQ, BP>::bytes(nsh_max);
    smem_optin((const void *)k_xc<W, NQ, BP>);
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
#if XC_MMA
    if constexpr (sizeof(W) == 4) {
        if (bucket_n[3]) launch_bucket_mma<16, 32, 2>(b, c, bucket_n[3], nsh_max, s);
        c += bucket_n[3];
        if (bucket_n[4]) launch_bucket<W, 20, BPL>(b, c, bucket_n[4], nsh_max, s);
    } else
#endif
    {
        if (bucket_n[3]) launch_bucket<W, 16, BP>(b, c, bucket_n[3], nsh_max, s);
        c += bucket_n[3];
        if (bucket_n[4]) launch_bucket<W, 20, BPL>(b, c, bucket_n[4], nsh_max, s);
    }
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
