// J/K digestion over the ket-tiled ERI store — deterministic, no atomics.
//
// Reference: deskdft.integrals.build_jk (integrals.py:199-218) -> _jk_kernel
// (_kernels.py:650-693), which scatters each canonical entry to its <= 8 images.
//
// B200 formulation.  The store row P = (i, j) is the lower half of the symmetric ket
// matrix T_P (k, l <= i) in 4x4 tiles (common.cuh, "ket-tiled rows").  For a stored
// element the 8 images contribute J_P += v rho~_Q, J_Q += v rho~_P and — recording each
// K contribution at (a,d) or its transpose — only rows i and j of an intermediate G
// (K = -(G + G^T)/4 in the post kernel):
//     G_i += 2 T_P rho_j - c,   G_j = 2 T_P rho_i - c'   (c, c' = the (ij|ij) element's
//                                                      second image, subtracted once)
// A CTA owns a contiguous range of whole slabs i (all rows (i, .)), streamed in chunks of
// CR (= 4) consecutive rows by cp.async.bulk (TMA bulk copy, mbarrier completion) into a
// double-buffered shared-memory stage while the previous chunk is digested.  One warp
// digests one row.  With A = i/4 + 1 the 4-row blocks of the result vectors are paired
// (a1 = p, a2 = A-1-p); a pair is owned by S lanes, and for each of its two blocks they
// read the tiles of the block row (row part, T[a][b] rho[b]) and the block column (column
// part, T[a'][a]^T rho[a']).  Every pair then visits exactly A + 1 tiles in each of the two
// loops (no divergence between lanes); the S lanes split the tiles and are combined by a
// shuffle tree.  Diagonal tiles are used with their diagonal halved (in registers), which
// makes row part + column part the full symmetric product and gives the J_P dot product a
// uniform weight of 2.  G_i accumulates in registers over the slab's rows; the scattered
// J_Q contributions are a second sweep over the staged chunk with thread-owned 16-byte
// units, so they accumulate in registers across the CTA's whole slab range.  All products
// are formed in f64; every output is written once and summed in a fixed order by the
// post kernel.
//
// Algorithmic traffic: the store is read exactly once from HBM per SCF iteration.  Work per
// stored element: 4 DFMA for K (two visits x (rho_i, rho_j)), 1 for J_P, 1 for J_Q.
#include "common.cuh"

namespace dftb {


#ifndef JK_NBUF_MAX
#define JK_NBUF_MAX 2                          // staging buffers per CTA
#endif
// warps per CTA (one store row per warp): 4 for the buckets up to 64 AOs (3 CTAs per SM),
// 8 for the larger ones (measured on B200: NB = 80 f32 331 -> 221 us per launch, NB = 64
// 1.55 -> 1.59 ms)
template <int NB> constexpr int jk_warps() { return NB > 64 ? 8 : 4; }

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_copy(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// L2 prefetch of a byte range (no shared memory, no completion): the chunk after the one
// being copied is pulled into L2 while the current one is digested, so the next bulk copy,
// issued only when a stage buffer frees up, reads L2 instead of HBM
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
#ifndef JK_PREFETCH
#define JK_PREFETCH 1      // chunks of look-ahead prefetched into L2 (0: off; 1: 1.284 -> 1.232 ms, 2: 1.238, 4: 1.254)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

template <typename ST>
__device__ __forceinline__ void tile_ld(const ST *p, double (&t)[16]) {
    if constexpr (sizeof(ST) == 4) {
        const float4 *q = reinterpret_cast<const float4 *>(p);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const float4 v = q[r];
            t[4 * r] = v.x; t[4 * r + 1] = v.y; t[4 * r + 2] = v.z; t[4 * r + 3] = v.w;
        }
    } else {
        const double2 *q = reinterpret_cast<const double2 *>(p);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const double2 v = q[r];
            t[2 * r] = v.x; t[2 * r + 1] = v.y;
        }
    }
}

__device__ __forceinline__ void ld4(const double *p, double (&v)[4]) {
    const double2 a = *reinterpret_cast<const double2 *>(p);
    const double2 c = *reinterpret_cast<const double2 *>(p + 2);
    v[0] = a.x; v[1] = a.y; v[2] = c.x; v[3] = c.y;
}

__device__ __forceinline__ double shfl_x(double v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }

// Shared-memory plan of one bucket: NBUF staging buffers of CR rows, padded rho, G_i
// reduction scratch.  Double buffering (then rows per chunk) is reduced for the largest
// buckets to fit 227 KB.
template <typename ST, int NB, int JK_WARPS = jk_warps<NB>()>
struct JKPlan {
    static constexpr int JK_THREADS = 32 * JK_WARPS;
    static constexpr int AMAX = NB / 4;
    static constexpr int LMAX = 8 * AMAX * (AMAX + 1);
    static constexpr size_t row_bytes = (size_t)LMAX * sizeof(ST);
    static constexpr size_t fixed = 128 + sizeof(double) * ((size_t)NB * NB + 4 * JK_THREADS);
    static constexpr size_t cap = 227 * 1024;
    // resident CTAs per SM by shared memory (1 KB per-CTA reservation)
    static constexpr int ctas(size_t bytes) { return (int)((228 * 1024) / (bytes + 1024)); }
    // double-buffer unless a single stage buffer raises the CTAs per SM (measured on B200:
    // NB = 64 f32 2 -> 3 CTAs, J/K 1.66 -> 1.56 ms; NB = 80 f32 1 -> 2 CTAs)
    static constexpr int NBUF =
        JK_NBUF_MAX > 1 && fixed + 2 * JK_WARPS * row_bytes <= cap &&
                !(ctas(fixed + JK_WARPS * row_bytes) > ctas(fixed + 2 * JK_WARPS * row_bytes))
            ? 2 : 1;
    static constexpr int CR = fixed + NBUF * JK_WARPS * row_bytes <= cap       ? JK_WARPS
                              : fixed + NBUF * (JK_WARPS / 2) * row_bytes <= cap ? JK_WARPS / 2
                                                                                 : JK_WARPS / 4;
    static constexpr size_t bytes = fixed + NBUF * CR * row_bytes;
    static_assert(bytes <= 227 * 1024, "J/K bucket does not fit in shared memory");
};

// rho in shared memory: row-major with stride NP, 16-byte chunks XOR-swizzled by the row's
// 4-block so that the lanes of a warp (different blocks a, same column block) hit
// different banks.
template <int NP>
__device__ __forceinline__ int rsw(int r, int c) {
    static_assert(NP % 16 == 0, "chunk swizzle needs NP / 2 to be a multiple of 8");
    return r * NP + (((c >> 1) ^ ((r >> 2) & 7)) << 1) + (c & 1);
}

// 4 consecutive rho values of a swizzled row starting at column 2*c2 (c2 = 16-byte chunk
// index, even); key = that row's swizzle key ((r >> 2) & 7)
__device__ __forceinline__ void ld4k(const double *rowp, int c2, int key, double (&v)[4]) {
    const int k0 = c2 ^ key;
    const double2 a = *reinterpret_cast<const double2 *>(rowp + 2 * k0);
    const double2 c = *reinterpret_cast<const double2 *>(rowp + 2 * (k0 ^ 1));
    v[0] = a.x; v[1] = a.y; v[2] = c.x; v[3] = c.y;
}
__device__ __forceinline__ int tri32(int a) { return (a * (a + 1)) >> 1; }

// NB: AO-count bound of the bucket (multiple of 16) — fixes the padded rho stride, the
// staging size and the number of J_Q units each thread owns.
template <typename ST, int NB>
__global__ void __launch_bounds__(32 * jk_warps<NB>(), NB > 64 ? 2 : NB > 32 ? 3 : 4) k_jk(DevBatch b, const int *ctas) {
    using PL = JKPlan<ST, NB>;
    constexpr int JK_THREADS = PL::JK_THREADS;
    constexpr int VW = 16 / (int)sizeof(ST);                   // elements per 16-byte unit
    constexpr int LMAX = PL::LMAX, NBUF = PL::NBUF, CR = PL::CR;
    constexpr int KU = (LMAX / VW + JK_THREADS - 1) / JK_THREADS;
    constexpr int NP = NB;                                      // padded rho stride
    extern __shared__ __align__(128) unsigned char jsm[];
    uint64_t *bar = (uint64_t *)jsm;
    double *rho = (double *)(jsm + 128);                        // [NP][NP] swizzled, zero padded
    double *gred = rho + NP * NP;                               // [JK_THREADS][4]
    ST *stage = (ST *)(gred + 4 * JK_THREADS);                  // [NBUF][CR * LMAX]
    const int cta = ctas[blockIdx.x];
    const int m = b.jk_mol[cta];
    if (b.done[m]) return;
    const int N = b.m_nao[m];
    const int64_t npp = tri(N);
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    const ST *eri = (const ST *)b.eri + b.m_eri0[m];
    const int i0 = b.jk_i0[cta], i1 = b.jk_i1[cta];
    // chunk producer (thread 0): chunks = CR consecutive rows of one slab, slabs walked
    // from i1-1 down to i0
    int pi = i1 - 1, pj = 0;
    auto issue = [&](int slot) {
        const int nr = min(CR, pi + 1 - pj);
        const int64_t L = eri_rowlen(pi);
        bulk_copy(stage + (size_t)slot * CR * LMAX, eri + eri_row(pi, pj),
                  (uint32_t)(nr * L * sizeof(ST)), bar + slot);
        pj += CR;
        if (pj > pi) { --pi; pj = 0; }
    };
    if (tid == 0) {
        for (int k = 0; k < NBUF; ++k) mbar_init(bar + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int k = 0; k < NBUF && pi >= i0; ++k) issue(k);
    }
    const double *rg = b.rho + b.m_mat0[m];
    for (int t = tid; t < NP * NP; t += JK_THREADS) {
        const int r = t / NP, c = t % NP;
        rho[rsw<NP>(r, c)] = (r < N && c < N) ? rg[r * N + c] : 0.0;
    }
    // this CTA's exchange partial Kc (N x N, CTA-private): the rows G_j of its slabs are
    // accumulated here instead of being stored one slab row at a time, so the post kernel
    // reads ncta N^2 instead of tri(N) N.  The adds are fire-and-forget reductions (RED, no
    // latency on the row's critical path); an element gets at most one add per chunk and the
    // chunks are separated by CTA barriers, so the order of the adds - and the result - is
    // fixed (deterministic, batch invariant).
    double *Gp = b.Gpart + b.m_G0[m] + (int64_t)(cta - b.m_jkcta0[m]) * N * N;
    for (int t = tid; t < N * N; t += JK_THREADS) Gp[t] = 0.0;
    __syncthreads();
    double acc[KU][VW];
#pragma unroll
    for (int k = 0; k < KU; ++k)
#pragma unroll
        for (int v = 0; v < VW; ++v) acc[k][v] = 0.0;
    double *Jp = b.Jpart + b.m_Jp0[m];
    int chunk = 0;
    for (int i = i1 - 1; i >= i0; --i) {
        const int A = (i >> 2) + 1;
        // lanes: S per 4-block a of the result vectors, block a = lane / S
        const int S = A <= 1 ? 32 : A <= 2 ? 16 : A <= 4 ? 8 : A <= 8 ? 4 : A <= 16 ? 2 : 1;
        const int a = lane / S, s = lane % S;
        const bool lane_ok = a < A;
        const int key_a = a & 7, key_i = (i >> 2) & 7;
        const double *rhoA = rho + 4 * a * NP, *rhoI = rho + i * NP;
        const int64_t L = eri_rowlen(i);
        const int units = (int)(L / VW);
        double gi[4] = {0, 0, 0, 0};
        for (int j0 = 0; j0 <= i; j0 += CR, ++chunk) {
            const int slot = chunk % NBUF;
            const ST *cbuf = stage + (size_t)slot * CR * LMAX;
            mbar_wait(bar + slot, (uint32_t)((chunk / NBUF) & 1));
            const int j = j0 + w;
            if (w < CR && j <= i) {                    // warp-uniform
                const ST *row = cbuf + (int64_t)w * L;
                const double *rhoJ = rho + j * NP;
                const int key_j = (j >> 2) & 7;
                double oI[4] = {0, 0, 0, 0}, oJ[4] = {0, 0, 0, 0}, jp = 0.0;
                if (lane_ok) {
                    // block a: row part tiles (a, q), q = 0..a, then column part tiles
                    // (q-1, a), q = a+1..A (transposed); A + 1 tiles for every block
                    for (int q = s; q <= A; q += S) {
                        const bool rp = q <= a;
                        const int ta = rp ? a : q - 1, tb = rp ? q : a;   // tile (ta, tb)
                        const int beta = rp ? q : q - 1;                  // rho block of the product
                        const bool dg = ta == tb;
                        float tf[16];
                        {
                            const float4 *qp = reinterpret_cast<const float4 *>(row + 16 * (tri32(ta) + tb));
                            if constexpr (sizeof(ST) == 4) {
#pragma unroll
                                for (int r = 0; r < 4; ++r) {
                                    const float4 v = qp[r];
                                    tf[4 * r] = v.x; tf[4 * r + 1] = v.y; tf[4 * r + 2] = v.z; tf[4 * r + 3] = v.w;
                                }
                                if (dg) { tf[0] *= 0.5f; tf[5] *= 0.5f; tf[10] *= 0.5f; tf[15] *= 0.5f; }
                            }
                        }
                        double t[16];
                        if constexpr (sizeof(ST) == 4) {
#pragma unroll
                            for (int r = 0; r < 4; ++r)
#pragma unroll
                                for (int c = 0; c < 4; ++c)
                                    t[4 * r + c] = (double)(rp ? tf[4 * r + c] : tf[4 * c + r]);
                        } else {
                            double td[16];
                            const double2 *qp = reinterpret_cast<const double2 *>(row + 16 * (tri32(ta) + tb));
#pragma unroll
                            for (int r = 0; r < 8; ++r) {
                                const double2 v = qp[r];
                                td[2 * r] = v.x; td[2 * r + 1] = v.y;
                            }
#pragma unroll
                            for (int r = 0; r < 4; ++r)
#pragma unroll
                                for (int c = 0; c < 4; ++c) t[4 * r + c] = rp ? td[4 * r + c] : td[4 * c + r];
                            if (dg) { t[0] *= 0.5; t[5] *= 0.5; t[10] *= 0.5; t[15] *= 0.5; }
                        }
                        double jv[4], iv[4];
                        ld4k(rhoJ, 2 * beta, key_j, jv);
                        ld4k(rhoI, 2 * beta, key_i, iv);
                        const double jw = rp ? 1.0 : 0.0;      // J_P: row-part tiles only
#pragma unroll
                        for (int rr = 0; rr < 4; ++rr) {
                            double x[4];
                            ld4k(rhoA + rr * NP, 2 * beta, key_a, x);
                            double d = 0.0;
#pragma unroll
                            for (int cc = 0; cc < 4; ++cc) {
                                oJ[rr] = fma(t[4 * rr + cc], jv[cc], oJ[rr]);
                                oI[rr] = fma(t[4 * rr + cc], iv[cc], oI[rr]);
                                d = fma(t[4 * rr + cc], x[cc], d);
                            }
                            jp = fma(jw, d, jp);
                        }
                    }
                }
                // ---- G_i partials stay per lane (reduced at slab end); G_j and J_P reduced now
#pragma unroll
                for (int u = 0; u < 4; ++u) gi[u] = fma(2.0, oJ[u], gi[u]);
                for (int o = 1; o < S; o <<= 1)
#pragma unroll
                    for (int u = 0; u < 4; ++u) oI[u] += shfl_x(oI[u], o);
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) jp += shfl_x(jp, o);
                const double vp = (double)row[eri_ket(i, j)];
                const double rjI = rho[rsw<NP>(j, i)], rjJ = rho[rsw<NP>(j, j)];
                const double riI = rho[rsw<NP>(i, i)], riJ = rho[rsw<NP>(i, j)];
                if (lane_ok && s == 0) {
                    double *Gj = Gp + (int64_t)j * N;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int t = 4 * a + u;
                        double gJ = 2.0 * oI[u];
                        if (t == j) { gi[u] -= vp * rjI; gJ -= vp * riI; }
                        else if (t == i) { gi[u] -= vp * rjJ; gJ -= vp * riJ; }
                        if (j < i && t <= i) atomicAdd(Gj + t, gJ);   // RED, see Kc above
                    }
                }
                if (lane == 0) Jp[tri(i) + j] = 2.0 * jp - vp * riJ * (i != j ? 2.0 : 1.0);
            }
            // ---- J_Q += v_PQ rho~_P over the chunk's rows, thread-owned 16-byte units
            const int nr = min(CR, i + 1 - j0);
            for (int rr = 0; rr < nr; ++rr) {
                const int jj = j0 + rr;
                const double wgt = rho[rsw<NP>(i, jj)] * (i != jj ? 2.0 : 1.0);
                const ST *rowp = cbuf + (int64_t)rr * L;
#pragma unroll
                for (int k = 0; k < KU; ++k) {
                    const int u = tid + k * JK_THREADS;
                    const double wk = u < units ? wgt : 0.0;
                    const int uc = min(u, units - 1);
                    if constexpr (VW == 4) {
                        const float4 v = reinterpret_cast<const float4 *>(rowp)[uc];
                        acc[k][0] = fma((double)v.x, wk, acc[k][0]);
                        acc[k][1] = fma((double)v.y, wk, acc[k][1]);
                        acc[k][2] = fma((double)v.z, wk, acc[k][2]);
                        acc[k][3] = fma((double)v.w, wk, acc[k][3]);
                    } else {
                        const double2 v = reinterpret_cast<const double2 *>(rowp)[uc];
                        acc[k][0] = fma(v.x, wk, acc[k][0]);
                        acc[k][1] = fma(v.y, wk, acc[k][1]);
                    }
                }
            }
            __syncthreads();                           // chunk consumed
            if (tid == 0 && pi >= i0) issue(slot);
        }
        // ---- slab end: G_i = fixed-order sum over stride lanes, then over warps
        for (int o = 1; o < S; o <<= 1)
#pragma unroll
            for (int u = 0; u < 4; ++u) gi[u] += shfl_x(gi[u], o);
#pragma unroll
        for (int u = 0; u < 4; ++u) gred[tid * 4 + u] = gi[u];
        __syncthreads();
        if (tid < A) {                                 // thread tid handles block tid
            double *Gi = Gp + (int64_t)i * N;
            for (int u = 0; u < 4; ++u) {
                const int t = 4 * tid + u;
                if (t > i) break;
                double v = 0.0;
                for (int ww = 0; ww < CR; ++ww) v += gred[(ww * 32 + tid * S) * 4 + u];
                atomicAdd(Gi + t, v);
            }
        }
        __syncthreads();
    }
    // ---- this CTA's J_Q partial, every Q of the molecule written once
    const int local = cta - b.m_jkcta0[m];
    double *Js = Jp + (int64_t)(1 + local) * npp;
    const int64_t Lm = eri_rowlen(N - 1);
#pragma unroll
    for (int k = 0; k < KU; ++k)
#pragma unroll
        for (int v = 0; v < VW; ++v) {
            const int e = (tid + k * JK_THREADS) * VW + v;
            if (e >= Lm) continue;
            const int tau = e >> 4;
            int a = (int)((sqrt(8.0 * (double)tau + 1.0) - 1.0) * 0.5);
            while (tri(a + 1) <= tau) ++a;
            while (tri(a) > tau) --a;
            const int bb = tau - (int)tri(a);
            const int kk = 4 * a + ((e >> 2) & 3), ll = 4 * bb + (e & 3);
            if (kk < N && ll <= kk) Js[tri(kk) + ll] = acc[k][v];
        }
}

// ---------------------------------------------------------------------------- f32 build
// The f32 build stores the ERI values and the density in f32 (the reference's f32 working
// dtype, integrals.py:171, scf.py:169-174), so every product v * rho of the digestion is a
// product of two f32 numbers.  k_jk32 forms those products on the packed FP32 pipe (FFMA2,
// two lanes per instruction) in short f32 partial sums - four products per tile row / column
// for K and J_P, one slab of rows for J_Q - and accumulates the partials in f64.  Relative to
// the reference's exact f64 products that adds a rounding of ~2^-24 per partial, the size of
// the f32 rounding already in every stored value.  Removes the per-element f32 -> f64
// conversions (XU pipe) and DFMA of the f64 formulation; the digestion plan is the same as
// k_jk's (one warp per row, lane group per 4-block a, A + 1 tile visits per block).
template <int NB, int WARPS>
struct JKPlan32 {
    static constexpr int THREADS = 32 * WARPS;
    static constexpr int AMAX = NB / 4;
    static constexpr int LMAX = 8 * AMAX * (AMAX + 1);          // f32 elements of the longest row
    static constexpr size_t row_bytes = (size_t)LMAX * 4;
    // rho f32 [NB][NB] + J_Q accumulators f64 [LMAX] + G_i reduction [THREADS][4] f64
    static constexpr size_t fixed = 128 + 4 * (size_t)NB * NB + 8 * (size_t)LMAX + 32 * (size_t)THREADS;
    static constexpr size_t cap = 227 * 1024;
    static constexpr int ctas(size_t bytes) { return (int)((228 * 1024) / (bytes + 1024)); }
    static constexpr int NBUF =
        fixed + 2 * WARPS * row_bytes <= cap && !(ctas(fixed + WARPS * row_bytes) > ctas(fixed + 2 * WARPS * row_bytes))
            ? 2 : 1;
    static constexpr int CR = fixed + NBUF * WARPS * row_bytes <= cap ? WARPS : WARPS / 2;
    static constexpr size_t bytes = fixed + NBUF * CR * row_bytes;
    static_assert(bytes <= cap, "J/K bucket does not fit in shared memory");
};
#ifndef JK32
#define JK32 1   // 0: the f32 build digests through k_jk<float> (f64 products) - A/B only
#endif
#ifndef JK_QUNR
#define JK_QUNR 1      // unroll of the f32 kernel's tile-visit loop
#endif
constexpr int kJkQUnr = JK_QUNR;
template <int NB> constexpr int jk32_warps() { return NB > 64 ? 8 : 4; }

// rho f32 row-major, stride NB, 16-byte chunks XOR-swizzled by the row's 4-block (the
// lanes of a warp read the same column block of rows in different 4-blocks)
// (XOR over the low 3 chunk-index bits when a row holds a multiple of 8 chunks, else 2, so
// the permutation stays inside the row)
template <int NB>
__device__ __forceinline__ int sw32key(int r) { return (r >> 2) & ((NB / 4) % 8 == 0 ? 7 : 3); }
template <int NB>
__device__ __forceinline__ int rsw32(int r, int c) {
    return r * NB + (((c >> 2) ^ sw32key<NB>(r)) << 2) + (c & 3);
}
__device__ __forceinline__ float4 lds4(const float *p) { return *reinterpret_cast<const float4 *>(p); }

template <int NB>
__global__ void __launch_bounds__(32 * jk32_warps<NB>(), NB > 64 ? 1 : 3) k_jk32(DevBatch b, const int *ctas) {
    constexpr int WARPS = jk32_warps<NB>();
    using PL = JKPlan32<NB, WARPS>;
    constexpr int THREADS = PL::THREADS, LMAX = PL::LMAX, NBUF = PL::NBUF, CR = PL::CR;
    constexpr int KU = (LMAX / 4 + THREADS - 1) / THREADS;      // 16-byte units per thread
    extern __shared__ __align__(128) unsigned char jsm[];
    uint64_t *bar = (uint64_t *)jsm;
    float *rho = (float *)(jsm + 128);                          // [NB][NB] swizzled, zero padded
    double *jq = (double *)(rho + NB * NB);                     // [LMAX] J_Q by ket position
    double *gred = jq + LMAX;                                   // [THREADS][4]
    float *stage = (float *)(gred + 4 * THREADS);               // [NBUF][CR * LMAX]
    const int cta = ctas[blockIdx.x];
    const int m = b.jk_mol[cta];
    if (b.done[m]) return;
    const int N = b.m_nao[m];
    const int64_t npp = tri(N);
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    const float *eri = (const float *)b.eri + b.m_eri0[m];
    const int i0 = b.jk_i0[cta], i1 = b.jk_i1[cta];
    int pi = i1 - 1, pj = 0;
    auto issue = [&](int slot) {
        const int nr = min(CR, pi + 1 - pj);
        const int64_t L = eri_rowlen(pi);
        bulk_copy(stage + (size_t)slot * CR * LMAX, eri + eri_row(pi, pj), (uint32_t)(nr * L * 4), bar + slot);
        pj += CR;
        if (pj > pi) { --pi; pj = 0; }
        if (JK_PREFETCH > 0) {        // the chunk JK_PREFETCH ahead of the next one, into L2
            int qi = pi, qj = pj;
            for (int k = 0; k < JK_PREFETCH && qi >= i0; ++k) {
                qj += CR;
                if (qj > qi) { --qi; qj = 0; }
            }
            if (qi >= i0) {
                const int qr = min(CR, qi + 1 - qj);
                bulk_prefetch_l2(eri + eri_row(qi, qj), (uint32_t)(qr * eri_rowlen(qi) * 4));
            }
        }
    };
    if (tid == 0) {
        for (int k = 0; k < NBUF; ++k) mbar_init(bar + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int k = 0; k < NBUF && pi >= i0; ++k) issue(k);
    }
    const double *rg = b.rho + b.m_mat0[m];
    for (int t = tid; t < NB * NB; t += THREADS) {
        const int r = t / NB, c = t % NB;
        rho[rsw32<NB>(r, c)] = (r < N && c < N) ? (float)rg[r * N + c] : 0.f;   // f32-exact in this build
    }
    for (int t = tid; t < LMAX; t += THREADS) jq[t] = 0.0;
    // per-CTA exchange partial (see k_jk)
    double *Gp = b.Gpart + b.m_G0[m] + (int64_t)(cta - b.m_jkcta0[m]) * N * N;
    for (int t = tid; t < N * N; t += THREADS) Gp[t] = 0.0;
    __syncthreads();
    double *Jp = b.Jpart + b.m_Jp0[m];
    int chunk = 0;
    for (int i = i1 - 1; i >= i0; --i) {
        const int A = (i >> 2) + 1;
        const int S = A <= 1 ? 32 : A <= 2 ? 16 : A <= 4 ? 8 : A <= 8 ? 4 : A <= 16 ? 2 : 1;
        const int a = lane / S, s = lane % S;
        const bool lane_ok = a < A;
        const float *rhoA = rho + 4 * a * NB, *rhoI = rho + i * NB;
        const int64_t L = eri_rowlen(i);
        const int units = (int)(L / 4);
        double gi[4] = {0, 0, 0, 0};
        float2 jacc[KU][2];                                     // J_Q partials of this slab (f32)
#pragma unroll
        for (int k = 0; k < KU; ++k) jacc[k][0] = jacc[k][1] = make_float2(0.f, 0.f);
        for (int j0 = 0; j0 <= i; j0 += CR, ++chunk) {
            const int slot = chunk % NBUF;
            const float *cbuf = stage + (size_t)slot * CR * LMAX;
            mbar_wait(bar + slot, (uint32_t)((chunk / NBUF) & 1));
            const int j = j0 + w;
            if (w < CR && j <= i) {                             // warp-uniform
                const float *row = cbuf + (int64_t)w * L;
                const float *rhoJ = rho + j * NB;
                double oJ[4] = {0, 0, 0, 0}, oI[4] = {0, 0, 0, 0}, jp = 0.0;
                if (lane_ok) {
#pragma unroll kJkQUnr
                    for (int q = s; q <= A; q += S) {
                        const bool rp = q <= a;
                        const int ta = rp ? a : q - 1, tb = rp ? q : a;   // tile (ta, tb)
                        const int beta = rp ? q : q - 1;                  // rho block of the product
                        const float *tp = row + 16 * (tri32(ta) + tb);
                        float tf[16];
                        {
                            const float4 r0 = lds4(tp), r1 = lds4(tp + 4), r2 = lds4(tp + 8), r3 = lds4(tp + 12);
                            tf[0] = r0.x; tf[1] = r0.y; tf[2] = r0.z; tf[3] = r0.w;
                            tf[4] = r1.x; tf[5] = r1.y; tf[6] = r1.z; tf[7] = r1.w;
                            tf[8] = r2.x; tf[9] = r2.y; tf[10] = r2.z; tf[11] = r2.w;
                            tf[12] = r3.x; tf[13] = r3.y; tf[14] = r3.z; tf[15] = r3.w;
                        }
                        if (ta == tb) { tf[0] *= 0.5f; tf[5] *= 0.5f; tf[10] *= 0.5f; tf[15] *= 0.5f; }
                        float t[16];
#pragma unroll
                        for (int r = 0; r < 4; ++r)
#pragma unroll
                            for (int c = 0; c < 4; ++c) t[4 * r + c] = rp ? tf[4 * r + c] : tf[4 * c + r];
                        const float4 vj = lds4(rhoJ + ((beta ^ sw32key<NB>(j)) << 2));
                        const float4 vi = lds4(rhoI + ((beta ^ sw32key<NB>(i)) << 2));
                        const float2 u[4] = {make_float2(vj.x, vi.x), make_float2(vj.y, vi.y),
                                             make_float2(vj.z, vi.z), make_float2(vj.w, vi.w)};
                        // (T rho_j, T rho_i) per result row: one FFMA2 per product pair
                        float2 o2[4];
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                acc = __ffma2_rn(make_float2(t[4 * r + c], t[4 * r + c]), u[c], acc);
                            o2[r] = acc;
                        }
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            oJ[r] += (double)o2[r].x;
                            oI[r] += (double)o2[r].y;
                        }
                        if (rp) {                               // J_P: row-part tiles only
                            const int key = sw32key<NB>(4 * a);
                            float2 d2 = make_float2(0.f, 0.f);
#pragma unroll
                            for (int r = 0; r < 4; ++r) {
                                const float4 x = lds4(rhoA + r * NB + ((beta ^ key) << 2));
                                d2 = __ffma2_rn(make_float2(t[4 * r], t[4 * r + 1]), make_float2(x.x, x.y), d2);
                                d2 = __ffma2_rn(make_float2(t[4 * r + 2], t[4 * r + 3]), make_float2(x.z, x.w), d2);
                            }
                            jp += (double)d2.x + (double)d2.y;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) gi[u] = fma(2.0, oJ[u], gi[u]);
                for (int o = 1; o < S; o <<= 1)
#pragma unroll
                    for (int u = 0; u < 4; ++u) oI[u] += shfl_x(oI[u], o);
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) jp += shfl_x(jp, o);
                const double vp = (double)row[eri_ket(i, j)];
                const double rjI = rho[rsw32<NB>(j, i)], rjJ = rho[rsw32<NB>(j, j)];
                const double riI = rho[rsw32<NB>(i, i)], riJ = rho[rsw32<NB>(i, j)];
                if (lane_ok && s == 0) {
                    double *Gj = Gp + (int64_t)j * N;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int t = 4 * a + u;
                        double gJ = 2.0 * oI[u];
                        if (t == j) { gi[u] -= vp * rjI; gJ -= vp * riI; }
                        else if (t == i) { gi[u] -= vp * rjJ; gJ -= vp * riJ; }
                        if (j < i && t <= i) atomicAdd(Gj + t, gJ);   // RED, order fixed by the chunk barriers
                    }
                }
                if (lane == 0) Jp[tri(i) + j] = 2.0 * jp - vp * riJ * (i != j ? 2.0 : 1.0);
            }
            // ---- J_Q += v_PQ rho~_P over the chunk's rows (thread-owned 16-byte units, f32)
            const int nr = min(CR, i + 1 - j0);
            for (int rr = 0; rr < nr; ++rr) {
                const int jj = j0 + rr;
                const float wgt = rho[rsw32<NB>(i, jj)] * (i != jj ? 2.f : 1.f);   // exact
                const float2 w2 = make_float2(wgt, wgt);
                const float *rowp = cbuf + (int64_t)rr * L;
#pragma unroll
                for (int k = 0; k < KU; ++k) {
                    const int u = tid + k * THREADS;
                    if (u < units) {
                        const float4 v = lds4(rowp + 4 * u);
                        jacc[k][0] = __ffma2_rn(make_float2(v.x, v.y), w2, jacc[k][0]);
                        jacc[k][1] = __ffma2_rn(make_float2(v.z, v.w), w2, jacc[k][1]);
                    }
                }
            }
            __syncthreads();                           // chunk consumed
            if (tid == 0 && pi >= i0) issue(slot);
        }
        // ---- slab end: J_Q partials into the f64 accumulators; G_i fixed-order sums
#pragma unroll
        for (int k = 0; k < KU; ++k) {
            const int u = tid + k * THREADS;
            if (u < units) {
                double2 *q2 = reinterpret_cast<double2 *>(jq + 4 * u);
                double2 x = q2[0], y = q2[1];
                x.x += (double)jacc[k][0].x; x.y += (double)jacc[k][0].y;
                y.x += (double)jacc[k][1].x; y.y += (double)jacc[k][1].y;
                q2[0] = x;
                q2[1] = y;
            }
        }
        for (int o = 1; o < S; o <<= 1)
#pragma unroll
            for (int u = 0; u < 4; ++u) gi[u] += shfl_x(gi[u], o);
#pragma unroll
        for (int u = 0; u < 4; ++u) gred[tid * 4 + u] = gi[u];
        __syncthreads();
        if (tid < A) {                                 // thread tid handles block tid
            double *Gi = Gp + (int64_t)i * N;
            for (int u = 0; u < 4; ++u) {
                const int t = 4 * tid + u;
                if (t > i) break;
                double v = 0.0;
                for (int ww = 0; ww < CR; ++ww) v += gred[(ww * 32 + tid * S) * 4 + u];
                atomicAdd(Gi + t, v);
            }
        }
        __syncthreads();
    }
    // ---- this CTA's J_Q partial, every Q of the molecule written once
    const int local = cta - b.m_jkcta0[m];
    double *Js = Jp + (int64_t)(1 + local) * npp;
    const int64_t Lm = eri_rowlen(N - 1);
    for (int e = tid; e < Lm; e += THREADS) {
        const int tau = e >> 4;
        int a = (int)((sqrt(8.0 * (double)tau + 1.0) - 1.0) * 0.5);
        while (tri(a + 1) <= tau) ++a;
        while (tri(a) > tau) --a;
        const int bb = tau - (int)tri(a);
        const int kk = 4 * a + ((e >> 2) & 3), ll = 4 * bb + (e & 3);
        if (kk < N && ll <= kk) Js[tri(kk) + ll] = jq[e];
    }
}

template <int NB>
static void launch_bucket32(const DevBatch &b, const int *ctas, int n, cudaStream_t s) {
    using PL = JKPlan32<NB, jk32_warps<NB>()>;
    smem_optin((const void *)k_jk32<NB>);
    k_jk32<NB><<<n, PL::THREADS, PL::bytes, s>>>(b, ctas);
}

template <typename ST, int NB>
static void launch_bucket(const DevBatch &b, const int *ctas, int n, cudaStream_t s) {
    const size_t sm = JKPlan<ST, NB>::bytes;
    smem_optin((const void *)k_jk<ST, NB>);
    k_jk<ST, NB><<<n, JKPlan<ST, NB>::JK_THREADS, sm, s>>>(b, ctas);
}

template <typename ST>
static void launch_jk_t(const DevBatch &b, const int *bucket_ctas, const int *bucket_n, cudaStream_t s) {
    const int *c = bucket_ctas;
    if (bucket_n[0]) launch_bucket<ST, 16>(b, c, bucket_n[0], s);
    c += bucket_n[0];
    if (bucket_n[1]) launch_bucket<ST, 32>(b, c, bucket_n[1], s);
    c += bucket_n[1];
    if (bucket_n[2]) launch_bucket<ST, 48>(b, c, bucket_n[2], s);
    c += bucket_n[2];
    if (bucket_n[3]) launch_bucket<ST, 64>(b, c, bucket_n[3], s);
    c += bucket_n[3];
    if (bucket_n[4]) launch_bucket<ST, 80>(b, c, bucket_n[4], s);
    c += bucket_n[4];
    if (bucket_n[5]) launch_bucket<ST, 96>(b, c, bucket_n[5], s);
}

// bucket_ctas: device array of CTA indices grouped by AO-count bucket; bucket_n: host counts [6]
int launch_jk(const DevBatch &b, const int *bucket_ctas, const int *bucket_n, cudaStream_t s) {
    if (b.n_jk_cta == 0) return 0;
    if (b.eri64 || !JK32) {
        if (b.eri64) launch_jk_t<double>(b, bucket_ctas, bucket_n, s);
        else launch_jk_t<float>(b, bucket_ctas, bucket_n, s);
    } else {
        const int *c = bucket_ctas;
        if (bucket_n[0]) launch_bucket32<16>(b, c, bucket_n[0], s);
        c += bucket_n[0];
        if (bucket_n[1]) launch_bucket32<32>(b, c, bucket_n[1], s);
        c += bucket_n[1];
        if (bucket_n[2]) launch_bucket32<48>(b, c, bucket_n[2], s);
        c += bucket_n[2];
        if (bucket_n[3]) launch_bucket32<64>(b, c, bucket_n[3], s);
        c += bucket_n[3];
        if (bucket_n[4]) launch_bucket32<80>(b, c, bucket_n[4], s);
        c += bucket_n[4];
        if (bucket_n[5]) launch_bucket32<96>(b, c, bucket_n[5], s);
    }
    int k = 0;
    for (int i = 0; i < 6; ++i) k += bucket_n[i] > 0;
    return k;
}

}  // namespace dftb
