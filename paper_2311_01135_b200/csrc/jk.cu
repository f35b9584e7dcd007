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
                        const int tq = tri32(ta) + tb, rot = eri_tile_rot(tq);   // rows sit in slots (r + rot) & 3
                        {
                            const float4 *qp = reinterpret_cast<const float4 *>(row + 16 * tq);
                            if constexpr (sizeof(ST) == 4) {
#pragma unroll
                                for (int r = 0; r < 4; ++r) {
                                    const float4 v = qp[(r + rot) & 3];
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
                            const double2 *qp = reinterpret_cast<const double2 *>(row + 16 * tq);
#pragma unroll
                            for (int r = 0; r < 8; ++r) {
                                const double2 v = qp[2 * (((r >> 1) + rot) & 3) + (r & 1)];
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
            const int kk = 4 * a + ((((e >> 2) & 3) + 4 - eri_tile_rot(tau)) & 3), ll = 4 * bb + (e & 3);
            if (kk < N && ll <= kk) Js[tri(kk) + ll] = acc[k][v];
        }
}

// ---------------------------------------------------------------------------- f32 build
// The f32 build stores the ERI values and the density in f32 (the reference's f32 working
// dtype, integrals.py:171, scf.py:169-174), so every product v * rho of the digestion is a
// product of two f32 numbers.  k_jk32 forms those products on the packed FP32 pipe (FFMA2)
// in short f32 partial sums - four products per tile row / column for K, one tile for J_P,
// the rows of the CTA's slabs for J_Q - and accumulates the partials in f64 (the reference
// accumulates in f64 and rounds J, K to f32 at the end).
//
// Tile owners.  A thread owns ONE tile position tau = (ta, tb) of the ket matrix for the
// CTA's whole slab range and walks the rows (i, j) (RF rows in parallel when a row has fewer
// tiles than the CTA has threads).  Everything that depends on the tile position only - the
// tile's address, rho[ta-block][tb-block] for J_P, the J_Q accumulators of the tile's 16
// kets - stays in registers for the life of the CTA; rho_i[ta], rho_i[tb] and the G_i partial
// sums of the tile's two 4-blocks for a slab.  The inner loop over rows is loads, FFMA2 and
// pointer increments: no index arithmetic, no divergence, no transposition selects.
// Consecutive lanes own consecutive tiles; with the rows of a tile rotated in the store
// (common.cuh) the four 16-byte loads of a tile are bank-conflict free.  Each tile is read
// once and serves both of its 4-blocks: the row part T rho[tb] (result block ta) and the
// column part T^T rho[ta] (result block tb).
// The one reduction across tiles that cannot stay in registers is G_j = 2 T_P rho_i (a
// per-row result).  The thread drops its two 4-vectors into a dense [A][A] grid of the row
// (row part at [ta][tb], column part at [tb][ta]), so that G_j[block a] is the plain sum of
// grid row a; a reduce pass over groups of up to 8 rows does those sums in a fixed order
// and issues the RED adds (one CTA barrier per chunk, two more per group).  J_P terms go
// through a per-row list and one warp per row.  G_i is reduced the same way once per slab,
// J_Q once per CTA.  Chunks of rows arrive by cp.async.bulk into three stage buffers
// (mbarrier completion); the chunk after the ones in flight is prefetched into L2.
template <int NB> constexpr int jk32_threads() { return NB <= 80 ? 256 : 320; }
#ifndef JK_NSTAGE
#define JK_NSTAGE 3
#endif
#ifndef JK_GROWS
#define JK_GROWS 8
#endif

template <int NB>
struct JKPlan32 {
    static constexpr int THREADS = jk32_threads<NB>();
    static constexpr int AMAX = NB / 4;
    static constexpr int TMAX = AMAX * (AMAX + 1) / 2;          // tiles of the longest row
    static constexpr int TMAXP = (TMAX + 31) & ~31;
    static constexpr int LMAX = 16 * TMAX;                       // f32 elements of the longest row
    static constexpr int LGA = AMAX <= 4 ? 2 : AMAX <= 8 ? 3 : AMAX <= 16 ? 4 : 5;   // 4-blocks, as a power of two
    static constexpr int GS = AMAX + 1;                          // grid row stride in float4 (odd: conflict free)
    static constexpr int GROWS = JK_GROWS;                       // rows per reduce group
    static constexpr int NSTAGE = JK_NSTAGE;
    static constexpr int PARTC = THREADS / (GROWS << LGA);       // lanes per (row, 4-block) in the reduce pass
    static constexpr int LGP = PARTC >= 4 ? 2 : PARTC >= 2 ? 1 : 0;
    static_assert(THREADS >= TMAX && PARTC >= 1, "one tile position per thread, one reduce lane per (row, block)");
    static constexpr size_t row_bytes = 4 * (size_t)LMAX;
    // mbarriers | rho f32 [NB][NB] | corr1, corr2 f64 [NB] | (ij|ij) f32 [GROWS] |
    // J_P terms float2 [GROWS][TMAXP] | G_j grid float4 [GROWS][AMAX][GS] | stage f32 [NSTAGE][SFL]
    // (the J_P + grid region doubles as the f64 G_i grid at slab end and the J_Q scratch at the end)
    static constexpr size_t o_rho = 128;                         // 2 x NSTAGE mbarriers in front
    static constexpr size_t o_c1 = o_rho + 4 * (size_t)NB * NB;
    static constexpr size_t o_vp = o_c1 + 16 * (size_t)NB;
    static constexpr size_t o_jp = (o_vp + 4 * (size_t)GROWS + 15) & ~(size_t)15;
    static constexpr size_t o_grid = o_jp + 8 * (size_t)GROWS * TMAXP;
    static constexpr size_t e_grid = o_grid + 16 * (size_t)GROWS * AMAX * GS;
    static constexpr size_t e_scr = o_jp + 64 * (size_t)THREADS + 64 * (size_t)GROWS * AMAX;   // bound on either scratch use
    static constexpr size_t o_stage = ((e_grid > e_scr ? e_grid : e_scr) + 127) & ~(size_t)127;
    static constexpr size_t cap2 = 113 * 1024, cap1 = 227 * 1024;   // per CTA at 2 / 1 CTAs per SM
    static constexpr int rows2 = o_stage < cap2 ? (int)((cap2 - o_stage) / (NSTAGE * row_bytes)) : 0;
    static constexpr int rows1 = (int)((cap1 - o_stage) / (NSTAGE * row_bytes));
    static constexpr int CTAS = rows2 >= 2 ? 2 : 1;
    static constexpr int rowsc = CTAS == 2 ? rows2 : rows1;
    static constexpr int SROWS = rowsc < GROWS ? rowsc : GROWS;  // longest rows per stage buffer
    static_assert(SROWS >= 1, "J/K bucket does not fit in shared memory");
    static constexpr int SFL = SROWS * LMAX;                     // f32 elements per stage buffer
    static constexpr size_t bytes = o_stage + 4 * (size_t)NSTAGE * SFL;
    static_assert(bytes <= cap1, "J/K bucket does not fit in shared memory");
};

__device__ __forceinline__ float4 lds4(const float *p) { return *reinterpret_cast<const float4 *>(p); }
__device__ __forceinline__ float2 lo2(const float4 v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(const float4 v) { return make_float2(v.z, v.w); }
__device__ __forceinline__ float2 dup2(float x) { return make_float2(x, x); }
// sum_c t[c] v[c] as two packed FMAs and one add (a 4-product f32 partial)
__device__ __forceinline__ float dot4(const float4 t, const float4 v) {
    float2 p = __ffma2_rn(lo2(t), lo2(v), make_float2(0.f, 0.f));
    p = __ffma2_rn(hi2(t), hi2(v), p);
    return p.x + p.y;
}

// rows per chunk of slab i (L elements per row) for a CTA digesting RF rows in parallel
template <int NB>
__device__ __forceinline__ int jk32_chunk_rows(int L, int RF) {
    using PL = JKPlan32<NB>;
    const int cr = min(PL::SFL / L, PL::GROWS);
    return cr >= RF ? cr - cr % RF : cr;
}

template <int NB>
__global__ void __launch_bounds__(jk32_threads<NB>(), JKPlan32<NB>::CTAS) k_jk32(DevBatch b, const int *ctas) {
    using PL = JKPlan32<NB>;
    constexpr int THREADS = PL::THREADS, AMAX = PL::AMAX, GS = PL::GS, GROWS = PL::GROWS, SFL = PL::SFL;
    constexpr int NSTAGE = PL::NSTAGE, TMAXP = PL::TMAXP, LGA = PL::LGA, LGP = PL::LGP, PART = 1 << LGP;
    extern __shared__ __align__(128) unsigned char jsm[];
    uint64_t *bar = (uint64_t *)jsm;
    float *rho = (float *)(jsm + PL::o_rho);                    // [NB][NB] zero padded
    double *corr1 = (double *)(jsm + PL::o_c1), *corr2 = corr1 + NB;
    float *vps = (float *)(jsm + PL::o_vp);                     // [GROWS] (ij|ij) of the group's rows
    float2 *jpb = (float2 *)(jsm + PL::o_jp);                   // [GROWS][TMAXP] J_P terms
    float4 *grid = (float4 *)(jsm + PL::o_grid);                // [GROWS][AMAX][GS] G_j terms
    double *scrd = (double *)(jsm + PL::o_jp);                  // slab end / CTA end scratch (same region)
    float *stage = (float *)(jsm + PL::o_stage);                // [NSTAGE][SFL]
    const int cta = ctas[blockIdx.x];
    const int m = b.jk_mol[cta];
    if (b.done[m]) return;
    const int N = b.m_nao[m];
    const int64_t npp = tri(N);
    const int tid = threadIdx.x;
    const float *eri = (const float *)b.eri + b.m_eri0[m];
    const int i0 = b.jk_i0[cta], i1 = b.jk_i1[cta];
    // ---- tile ownership, fixed for the CTA: RF row groups x the ntm tiles of its longest rows
    const int ntm = tri32(((i1 - 1) >> 2) + 1);
    const int RF = min(THREADS / ntm, GROWS);
    const int rs = tid / ntm, tau = tid - rs * ntm;
    const bool own = rs < RF;
    // chunk producer (thread 0): chunks of consecutive rows of one slab, slabs from i1-1 down to i0.
    // The store is contiguous in that order read backwards slab by slab, so the source offset
    // advances incrementally (slab i-1 = the i rows before slab i).
    // Its state lives in shared memory (six registers less in every thread): slab, row, row
    // length, rows per chunk, slab offset, next source offset.
    volatile int *ps = (volatile int *)(bar + 2 * NSTAGE);
    auto issue = [&](int slot) {
        int pi = ps[0], pj = ps[1], pL = ps[2], pcr = ps[3], psrc = ps[5];
        const int nr = min(pcr, pi + 1 - pj);
        bulk_copy(stage + (size_t)slot * SFL, eri + psrc, (uint32_t)(nr * pL * 4), bar + slot);
        pj += pcr;
        psrc += nr * pL;
        if (pj > pi) {
            --pi;
            pj = 0;
            if (pi >= i0) {
                pL = (int)eri_rowlen(pi);
                pcr = jk32_chunk_rows<NB>(pL, RF);
                psrc = ps[4] - (pi + 1) * pL;
                ps[2] = pL; ps[3] = pcr; ps[4] = psrc;
            }
            ps[0] = pi;
        }
        ps[1] = pj; ps[5] = psrc;
        if (JK_PREFETCH > 0 && pi >= i0)         // the chunk after the one just issued, into L2
            bulk_prefetch_l2(eri + psrc, (uint32_t)(min(pcr, pi + 1 - pj) * pL * 4));
    };
    // "stage consumed" barriers: every thread arrives, only the producer thread waits, then refills.
    // Measured alternatives (B200, ms per iteration against 0.94): the last warp to finish a chunk
    // refills it (shared-memory atomic count, no waiting): 1.03; the producer refills one chunk
    // behind, when nobody is left in that buffer (one chunk less in flight): 0.97.
    uint64_t *ebar = bar + NSTAGE;
    if (tid == 0) {
        for (int k = 0; k < NSTAGE; ++k) { mbar_init(bar + k, 1); mbar_init(ebar + k, THREADS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        ps[0] = i1 - 1; ps[1] = 0; ps[2] = (int)eri_rowlen(i1 - 1); ps[3] = jk32_chunk_rows<NB>(ps[2], RF);
        ps[4] = ps[5] = (int)eri_slab0(i1 - 1);
        for (int k = 0; k < NSTAGE && ps[0] >= i0; ++k) issue(k);
    }
    const double *rg = b.rho + b.m_mat0[m];
    for (int t = tid; t < NB * NB; t += THREADS) {
        const int r = t / NB, c = t % NB;
        rho[t] = (r < N && c < N) ? (float)rg[r * N + c] : 0.f;   // f32-exact in this build
    }
    // per-CTA exchange partial (see k_jk)
    double *Gp = b.Gpart + b.m_G0[m] + (int64_t)(cta - b.m_jkcta0[m]) * N * N;
    for (int t = tid; t < N * N; t += THREADS) Gp[t] = 0.0;
    __syncthreads();
    // ---- this thread's tile
    int ta = (int)((sqrtf(8.f * (float)tau + 1.f) - 1.f) * 0.5f);
    while (tri32(ta + 1) <= tau) ++ta;
    while (tri32(ta) > tau) --ta;
    const int tb = tau - tri32(ta);
    const int rot = eri_tile_rot(tau);
    const int o0 = 16 * tau + 4 * (rot & 3), o1 = 16 * tau + 4 * ((rot + 1) & 3);
    const int o2 = 16 * tau + 4 * ((rot + 2) & 3), o3 = 16 * tau + 4 * ((rot + 3) & 3);
    const bool diag = ta == tb;
    const float hs = diag ? 0.5f : 1.f;                         // diagonal tiles: diagonal halved (see k_jk)
    const float dg = diag ? 1.f : 0.f;
    const int grow = ta * GS + tb, gcol = tb * GS + ta;         // grid slots of the row / column part
#ifndef JK_RAB_REGS
#define JK_RAB_REGS 0     // 1: keep rho[ta-block][tb-block] (J_P) in 16 registers instead of reloading it per row
#endif
    const float *rab = rho + (4 * ta) * NB + 4 * tb;            // rho[ta-block][tb-block] for J_P
#if JK_RAB_REGS
    float4 rab0 = make_float4(0.f, 0.f, 0.f, 0.f), rab1 = rab0, rab2 = rab0, rab3 = rab0;
    if (own) { rab0 = lds4(rab); rab1 = lds4(rab + NB); rab2 = lds4(rab + 2 * NB); rab3 = lds4(rab + 3 * NB); }
#endif
    float2 jqa[4][2];
#pragma unroll
    for (int r = 0; r < 4; ++r) jqa[r][0] = jqa[r][1] = make_float2(0.f, 0.f);
    double *Jp = b.Jpart + b.m_Jp0[m];
    int slot = 0;
    uint32_t ph = 0;
    const float *cbuf = stage;
    const float *rpa = rho + 4 * ta, *rpb = rho + 4 * tb;       // rho_j[ta-block], rho_j[tb-block] of row 0
    float4 *gpr = grid + grow, *gpc = grid + gcol;
    float2 *jpt = jpb + tau;
    for (int i = i1 - 1; i >= i0; --i) {
        const int A = (i >> 2) + 1, nt = tri32(A), L = 16 * nt;
        const int CR = jk32_chunk_rows<NB>(L, RF);
        const int GR = (GROWS / CR) * CR;                       // rows per reduce group
        const bool act = own && tau < nt;
        float4 rib = make_float4(0.f, 0.f, 0.f, 0.f), ria = rib;
        if (act) { rib = lds4(rho + i * NB + 4 * tb); ria = lds4(rho + i * NB + 4 * ta); }
        const float2 ria0 = dup2(ria.x), ria1 = dup2(ria.y), ria2 = dup2(ria.z), ria3 = dup2(ria.w);
        const float *rpi = rho + i * NB;
        const int tauv0 = tri32(A - 1);                         // tiles of AO i's block row
        const int ov = 16 * tau + 4 * (((i & 3) + rot) & 3);    // row i & 3 of this tile
        double gia[4] = {0, 0, 0, 0}, gib[4] = {0, 0, 0, 0};
        for (int g0 = 0; g0 <= i; g0 += GR) {
            const int nrg = min(GR, i + 1 - g0);
            for (int c0 = 0; c0 < nrg; c0 += CR) {
                mbar_wait(bar + slot, ph);
                const int nr = min(CR, nrg - c0);
                if (act) {
                    for (int rr = rs; rr < nr; rr += RF) {
                        const int gr = c0 + rr, j = g0 + gr;
                        const float *tp = cbuf + rr * L;
                        float4 T0 = lds4(tp + o0), T1 = lds4(tp + o1), T2 = lds4(tp + o2), T3 = lds4(tp + o3);
                        if (tau == tauv0 + (j >> 2)) vps[gr] = tp[ov + (j & 3)];      // (ij|ij)
                        const float4 rjb = lds4(rpb + j * NB), rja = lds4(rpa + j * NB);
                        const float2 w2 = dup2(rpi[j] * (i != j ? 2.f : 1.f));       // exact
                        // J_Q += v_PQ rho~_P on the stored values
                        jqa[0][0] = __ffma2_rn(lo2(T0), w2, jqa[0][0]); jqa[0][1] = __ffma2_rn(hi2(T0), w2, jqa[0][1]);
                        jqa[1][0] = __ffma2_rn(lo2(T1), w2, jqa[1][0]); jqa[1][1] = __ffma2_rn(hi2(T1), w2, jqa[1][1]);
                        jqa[2][0] = __ffma2_rn(lo2(T2), w2, jqa[2][0]); jqa[2][1] = __ffma2_rn(hi2(T2), w2, jqa[2][1]);
                        jqa[3][0] = __ffma2_rn(lo2(T3), w2, jqa[3][0]); jqa[3][1] = __ffma2_rn(hi2(T3), w2, jqa[3][1]);
                        T0.x *= hs; T1.y *= hs; T2.z *= hs; T3.w *= hs;
                        // row part (result block ta): T rho_j[tb] -> G_i, T rho_i[tb] -> G_j
                        const float oJ0 = dot4(T0, rjb), oJ1 = dot4(T1, rjb), oJ2 = dot4(T2, rjb), oJ3 = dot4(T3, rjb);
                        float4 oI = make_float4(dot4(T0, rib), dot4(T1, rib), dot4(T2, rib), dot4(T3, rib));
                        // column part (result block tb): T^T rho_j[ta] -> G_i, T^T rho_i[ta] -> G_j
                        // (rho_j[ta] changes with the row: scalar FMAs, no register-pair duplicates to build)
                        float cJ0 = T0.x * rja.x, cJ1 = T0.y * rja.x, cJ2 = T0.z * rja.x, cJ3 = T0.w * rja.x;
                        cJ0 = fmaf(T1.x, rja.y, cJ0); cJ1 = fmaf(T1.y, rja.y, cJ1); cJ2 = fmaf(T1.z, rja.y, cJ2); cJ3 = fmaf(T1.w, rja.y, cJ3);
                        cJ0 = fmaf(T2.x, rja.z, cJ0); cJ1 = fmaf(T2.y, rja.z, cJ1); cJ2 = fmaf(T2.z, rja.z, cJ2); cJ3 = fmaf(T2.w, rja.z, cJ3);
                        cJ0 = fmaf(T3.x, rja.w, cJ0); cJ1 = fmaf(T3.y, rja.w, cJ1); cJ2 = fmaf(T3.z, rja.w, cJ2); cJ3 = fmaf(T3.w, rja.w, cJ3);
                        float2 cI0 = __ffma2_rn(lo2(T0), ria0, make_float2(0.f, 0.f));
                        float2 cI1 = __ffma2_rn(hi2(T0), ria0, make_float2(0.f, 0.f));
                        cI0 = __ffma2_rn(lo2(T1), ria1, cI0); cI1 = __ffma2_rn(hi2(T1), ria1, cI1);
                        cI0 = __ffma2_rn(lo2(T2), ria2, cI0); cI1 = __ffma2_rn(hi2(T2), ria2, cI1);
                        cI0 = __ffma2_rn(lo2(T3), ria3, cI0); cI1 = __ffma2_rn(hi2(T3), ria3, cI1);
                        // J_P term of this tile: sum T . rho[ta-block][tb-block] (two f32 partials)
#if !JK_RAB_REGS
                        // (reloaded per row: 16 registers less, which the compiler otherwise pays for by
                        // re-deriving the tile's addresses and constants in every iteration)
                        const float4 rab0 = lds4(rab), rab1 = lds4(rab + NB), rab2 = lds4(rab + 2 * NB), rab3 = lds4(rab + 3 * NB);
#endif
                        float2 jp2 = __ffma2_rn(lo2(T0), lo2(rab0), make_float2(0.f, 0.f));
                        jp2 = __ffma2_rn(hi2(T0), hi2(rab0), jp2);
                        jp2 = __ffma2_rn(lo2(T1), lo2(rab1), jp2); jp2 = __ffma2_rn(hi2(T1), hi2(rab1), jp2);
                        jp2 = __ffma2_rn(lo2(T2), lo2(rab2), jp2); jp2 = __ffma2_rn(hi2(T2), hi2(rab2), jp2);
                        jp2 = __ffma2_rn(lo2(T3), lo2(rab3), jp2); jp2 = __ffma2_rn(hi2(T3), hi2(rab3), jp2);
                        gia[0] += (double)oJ0; gia[1] += (double)oJ1; gia[2] += (double)oJ2; gia[3] += (double)oJ3;
                        gib[0] += (double)cJ0; gib[1] += (double)cJ1; gib[2] += (double)cJ2; gib[3] += (double)cJ3;
                        // G_j terms into the row's grid (a diagonal tile's two parts share a slot), J_P term
                        oI.x = fmaf(dg, cI0.x, oI.x); oI.y = fmaf(dg, cI0.y, oI.y);
                        oI.z = fmaf(dg, cI1.x, oI.z); oI.w = fmaf(dg, cI1.y, oI.w);
                        gpr[gr * (AMAX * GS)] = oI;
                        if (!diag) gpc[gr * (AMAX * GS)] = make_float4(cI0.x, cI0.y, cI1.x, cI1.y);
                        jpt[gr * TMAXP] = jp2;
                    }
                }
                // stage consumed (no CTA barrier: the warps go on to the next chunk, already in its own buffer)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(ebar + slot)) : "memory");
                if (tid == 0 && ps[0] >= i0) {
                    mbar_wait(ebar + slot, ph);
                    issue(slot);
                }
                cbuf += SFL;
                if (++slot == NSTAGE) { slot = 0; cbuf = stage; ph ^= 1u; }
            }
            __syncthreads();                                    // the group's grid rows are written
            {   // ---- reduce pass over the group's rows: G_j[block a] = 2 sum of grid row a
                const int rr = tid >> (LGA + LGP), a = (tid >> LGP) & ((1 << LGA) - 1), part = tid & (PART - 1);
                const bool ract = rr < nrg && a < A;
                float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;   // this lane's terms (f32), then f64 across the lanes
                if (ract) {
                    const float4 *gp = grid + (rr * AMAX + a) * GS;
#pragma unroll
                    for (int x0 = 0; x0 < AMAX; x0 += PART) {
                        const int x = x0 + part;
                        if (x < A) {
                            const float4 v = gp[x];
                            s0 += v.x; s1 += v.y; s2 += v.z; s3 += v.w;
                        }
                    }
                }
                double d0 = (double)s0, d1 = (double)s1, d2 = (double)s2, d3 = (double)s3;
#pragma unroll
                for (int o = 1; o < PART; o <<= 1) {
                    d0 += shfl_x(d0, o); d1 += shfl_x(d1, o); d2 += shfl_x(d2, o); d3 += shfl_x(d3, o);
                }
                if (ract) {                                        // each of the PART lanes takes 4 / PART of the block's outputs
                    constexpr int UPL = 4 >> LGP;
                    const int j = g0 + rr;
                    const double vp = (double)vps[rr];
                    const double riI = rpi[i], riJ = rpi[j];
                    double g[UPL];
                    if constexpr (UPL == 4) { g[0] = d0; g[1] = d1; g[2] = d2; g[3] = d3; }
                    else if constexpr (UPL == 2) { g[0] = part ? d2 : d0; g[1] = part ? d3 : d1; }
                    else g[0] = part == 0 ? d0 : part == 1 ? d1 : part == 2 ? d2 : d3;
                    double *Gj = Gp + (int64_t)j * N + 4 * a + part * UPL;
#pragma unroll
                    for (int u = 0; u < UPL; ++u) {
                        const int t = 4 * a + part * UPL + u;
                        double gJ = 2.0 * g[u];
                        if (t == j) gJ -= vp * riI;
                        else if (t == i) gJ -= vp * riJ;
                        if (j < i && t <= i) atomicAdd(Gj + u, gJ);   // RED; one add per element per group
                    }
                    if (part == 0 && a == (j >> 2)) {               // this row's corrections to G_i (applied at slab end)
                        corr1[j] = vp * (double)rho[j * NB + i];
                        corr2[j] = j < i ? vp * (double)rho[j * NB + j] : 0.0;
                    }
                }
                // ---- J_P = 2 sum of the row's tile terms - the (ij|ij) image counted by J_Q: one warp per row
                for (int r2 = tid >> 5; r2 < nrg; r2 += THREADS / 32) {
                    const float2 *jr = jpb + r2 * TMAXP;
                    double jp = 0.0;
                    for (int tq = tid & 31; tq < nt; tq += 32) {
                        const float2 q = jr[tq];
                        jp += (double)q.x + (double)q.y;
                    }
                    jp = warp_sum(jp);
                    if ((tid & 31) == 0) {
                        const int j = g0 + r2;
                        const double vp = (double)vps[r2], riJ = rho[i * NB + j];
                        Jp[tri(i) + j] = 2.0 * jp - vp * riJ * (i != j ? 2.0 : 1.0);
                    }
                }
            }
            __syncthreads();
        }
        // ---- slab end: G_i = 2 sum over the row groups and tiles (dense f64 grid) - corrections
        if (act) {
            double *q = scrd + ((size_t)(rs * A + ta) * (A + 1) + tb) * 4;
            if (diag) {
                q[0] = gia[0] + gib[0]; q[1] = gia[1] + gib[1]; q[2] = gia[2] + gib[2]; q[3] = gia[3] + gib[3];
            } else {
                q[0] = gia[0]; q[1] = gia[1]; q[2] = gia[2]; q[3] = gia[3];
                double *qc = scrd + ((size_t)(rs * A + tb) * (A + 1) + ta) * 4;
                qc[0] = gib[0]; qc[1] = gib[1]; qc[2] = gib[2]; qc[3] = gib[3];
            }
        }
        __syncthreads();
        if (tid <= i) {                                        // G_i[t], t = tid
            const int a = tid >> 2, u = tid & 3;
            double s = 0.0;
            for (int g = 0; g < RF; ++g) {
                const double *q = scrd + (size_t)(g * A + a) * (A + 1) * 4 + u;
                for (int x = 0; x < A; ++x) s += q[4 * x];
            }
            double gv = 2.0 * s - corr1[tid];
            if (tid == i)
                for (int j = 0; j < i; ++j) gv -= corr2[j];
            atomicAdd(Gp + (int64_t)i * N + tid, gv);
        }
        __syncthreads();
    }
    // ---- this CTA's J_Q partial: f32 sums over the CTA's rows (measured on B200 against exact f64
    // sums, N = 59: 4e-8 of max|J| with 4 CTAs per molecule, 2.5e-7 with one - the K partials are at
    // 6e-8), f64 over the row groups; every Q of the molecule written once
    float *scrf = reinterpret_cast<float *>(scrd);
    if (own) {
        float *q = scrf + (size_t)(rs * ntm + tau) * 16;
#pragma unroll
        for (int r = 0; r < 4; ++r)
            *reinterpret_cast<float4 *>(q + 4 * r) = make_float4(jqa[r][0].x, jqa[r][0].y, jqa[r][1].x, jqa[r][1].y);
    }
    __syncthreads();
    const int local = cta - b.m_jkcta0[m];
    double *Js = Jp + (int64_t)(1 + local) * npp;
    const int Lm = (int)eri_rowlen(N - 1), Lc = 16 * ntm;
    for (int e = tid; e < Lm; e += THREADS) {
        const int tq = e >> 4;
        int a = (int)((sqrtf(8.f * (float)tq + 1.f) - 1.f) * 0.5f);
        while (tri32(a + 1) <= tq) ++a;
        while (tri32(a) > tq) --a;
        const int bb = tq - tri32(a);
        const int kk = 4 * a + ((e >> 2) & 3), ll = 4 * bb + (e & 3);
        if (kk < N && ll <= kk) {
            double s = 0.0;
            if (e < Lc)
                for (int g = 0; g < RF; ++g) s += (double)scrf[(size_t)g * Lc + e];
            Js[tri(kk) + ll] = s;
        }
    }
}

template <int NB>
static void launch_bucket32(const DevBatch &b, const int *ctas, int n, cudaStream_t s) {
    using PL = JKPlan32<NB>;
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
    if (b.eri64) {
        launch_jk_t<double>(b, bucket_ctas, bucket_n, s);
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
