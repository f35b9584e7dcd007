// J/K digestion over the dense 8-fold ERI store — deterministic, no atomics.
//
// Reference: deskdft.integrals.build_jk (integrals.py:199-218) -> _jk_kernel
// (_kernels.py:650-693), which scatters each canonical entry to its <= 8 images.
//
// B200 formulation ("row owner"): a CTA owns the store rows P = (i, j), j <= i,
// for one or two values of i.  Row P holds (ij|kl) for all Q = (k, l) <= P.  For a
// stored element the 8 images contribute J_P += v rho~_Q, J_Q += v rho~_P and —
// recording each K contribution at (a,d) or its transpose — only G[i][.] and G[j][.]
// updates (K = -(G + G^T)/4 at the end).  Per row the CTA computes two GEMVs with
// the row's symmetric ket matrix T (T rho_j, T rho_i), read straight from the
// staged packed row, and one dot product.  G_i accumulates in registers across the
// CTA's rows, the J_Q scatter accumulates in registers (thread t owns Q = t mod
// 256), G_j rows and J partials are written once and summed in a fixed order by the
// SCF post kernel.  One CTA barrier per row.
//
// Data movement: rows are 16-byte padded in HBM and prefetched whole with
// cp.async.bulk (TMA bulk copy, mbarrier completion) into a double-buffered
// staging area while the previous row is being digested; the store is streamed
// exactly once per SCF iteration.  In the f32 build rho is kept in f32 shared
// memory (it is f32-valued there); products are always formed in f64.
#include "common.cuh"

namespace dftb {

constexpr int JK_THREADS = 256;
constexpr int JK_NREG = (NMAX * (NMAX + 1) / 2 + JK_THREADS - 1) / JK_THREADS;  // owned J_Q slots

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_row(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

struct JKLayout {
    size_t stage, rho, lut, wpart, total;
};

constexpr int JK_MAXROWS = NMAX + 1;   // rows per CTA: (i0 + 1) + (i1 + 1) = N + 1

template <typename ST, typename RT_unused>
HD JKLayout jk_layout(int N, int nbuf) {
    using RT = double;
    const int g = 16 / (int)sizeof(ST);
    const size_t npp = (size_t)N * (N + 1) / 2;
    JKLayout L;
    size_t o = 64;                                    // mbarriers
    L.stage = o; o += (size_t)nbuf * rowpad((int64_t)npp, g) * sizeof(ST);
    o = (o + 15) & ~(size_t)15;
    L.rho = o; o += (size_t)N * N * sizeof(RT);
    o = (o + 15) & ~(size_t)15;
    L.lut = o; o += npp * sizeof(uint16_t);
    o = (o + 15) & ~(size_t)15;
    L.wpart = o; o += (size_t)JK_MAXROWS * (JK_THREADS / 32) * sizeof(double);
    L.total = o;
    return L;
}

// Row P = (i, j) of the packed store, staged in shared memory, is digested without
// expanding it: element (k, l) of the row sits at tri(k) + l, so the column t of the
// symmetric ket matrix T is {row[tri(n) + t] : n >= t} U {row[tri(t) + n] : n < t}.
// Across a warp, tri(t) + n hits 32 distinct banks (triangular numbers are a
// permutation mod 32), so both walks are conflict-free.
template <typename ST, typename RT>
__global__ void __launch_bounds__(JK_THREADS) k_jk(DevBatch b, int nbuf) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int cta = blockIdx.x;
    const int m = b.jk_mol[cta];
    if (b.done[m]) return;
    const int N = b.m_nao[m];
    const int g = 16 / (int)sizeof(ST);
    const int64_t npp = tri(N);
    const JKLayout L = jk_layout<ST, RT>(N, nbuf);
    uint64_t *bar = (uint64_t *)sm;
    ST *stage = (ST *)(sm + L.stage);
    const int64_t stride = rowpad(npp, g);
    double *rho = (double *)(sm + L.rho);
    uint16_t *lut = (uint16_t *)(sm + L.lut);
    double *wpart = (double *)(sm + L.wpart);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const ST *eri = (const ST *)b.eri + b.m_eri0[m];
    const int i0 = b.jk_i0[cta], i1 = b.jk_i1[cta];
    const int nrow0 = i0 + 1, nrows = nrow0 + (i1 >= 0 ? i1 + 1 : 0);
    auto row_ij = [&](int r, int &i, int &j) {
        if (r < nrow0) { i = i0; j = r; } else { i = i1; j = r - nrow0; }
    };
    auto issue = [&](int r) {
        int i, j;
        row_ij(r, i, j);
        const int64_t P = tri(i) + j;
        bulk_row(stage + (r % nbuf) * stride, eri + rowbase(P, g), (uint32_t)(rowpad(P + 1, g) * sizeof(ST)),
                 bar + (r % nbuf));
    };
    if (tid == 0) {
        for (int k = 0; k < nbuf; ++k) mbar_init(bar + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int r = 0; r < nbuf && r < nrows; ++r) issue(r);
    const double *rg = b.rho + b.m_mat0[m];
    for (int t = tid; t < N * N; t += JK_THREADS) rho[t] = rg[t];
    for (int k = tid; k < N; k += JK_THREADS)
        for (int l = 0; l <= k; ++l) lut[tri(k) + l] = (uint16_t)((k << 8) | l);
    __syncthreads();
    double jsc[JK_NREG];
#pragma unroll
    for (int q = 0; q < JK_NREG; ++q) jsc[q] = 0.0;
    double *Gp = b.Gpart + b.m_G0[m];
    double *Jp = b.Jpart + b.m_Jp0[m];
    double gi = 0.0;
    for (int r = 0; r < nrows; ++r) {
        int i, j;
        row_ij(r, i, j);
        const int64_t P = tri(i) + j;
        const ST *row = stage + (r % nbuf) * stride;
        mbar_wait(bar + (r % nbuf), (uint32_t)((r / nbuf) & 1));
        // ---- J: own dot product and the scattered J_Q (thread owns Q = tid mod 256)
        const double rt = rho[i * N + j] * (i != j ? 2.0 : 1.0);
        double jown = 0.0;
#pragma unroll
        for (int q = 0; q < JK_NREG; ++q) {
            const int64_t e = tid + (int64_t)q * JK_THREADS;
            if (e <= P) {
                const double v = (double)row[e];
                const int kl = lut[e], k = kl >> 8, l = kl & 255;
                jown += v * rho[k * N + l] * (k != l ? 2.0 : 1.0);
                if (e < P) jsc[q] += v * rt;
            }
        }
        // ---- K: G_i[t] += (T rho_j)[t] and G_j[t] = (T rho_i)[t], T read from the packed row.
        // One thread forms both dot products for output t over n = sl, sl+S, ... (S lanes per
        // output, combined by a shuffle tree).  T[n][t] = 2 v(e) except the row's own
        // element e = P (weight 1), corrected once; no per-element bounds checks.
        {
            const int ni = i + 1;
            const int S = ni * 8 <= JK_THREADS ? 8 : ni * 4 <= JK_THREADS ? 4 : ni * 2 <= JK_THREADS ? 2 : 1;
            const int t = tid / S, sl = tid % S;
            double ai = 0.0, aj = 0.0;
            if (t < ni) {
                const double *rj = rho + j * N, *ri = rho + i * N;
                const int tt = (int)tri(t);
                // walk 1: (t, n), n < n1 ; valid while tt + n <= P
                const int n1 = t < i ? t : min(t, j + 1);
                for (int n = sl; n < n1; n += S) {
                    const double v = (double)row[tt + n];
                    ai += v * rj[n];
                    aj += v * ri[n];
                }
                // walk 2: (n, t), t <= n <= n2 ; row index tri(n) + t
                const int n2 = t <= j ? i : i - 1;
                int n = t + sl;
                int e = (int)tri(n) + t;
                for (; n <= n2; n += S) {
                    const double v = (double)row[e];
                    ai += v * rj[n];
                    aj += v * ri[n];
                    // tri(n + S) - tri(n) = S n + S (S + 1) / 2
                    e += S * n + (S * (S + 1) >> 1);
                }
                ai *= 2.0;
                aj *= 2.0;
                if (sl == 0) {
                    const double vp = (double)row[P];
                    if (t == j) { ai -= vp * rj[i]; aj -= vp * ri[i]; }
                    else if (t == i) { ai -= vp * rj[j]; aj -= vp * ri[j]; }
                }
            }
            for (int o = S >> 1; o > 0; o >>= 1) {
                ai += __shfl_xor_sync(0xffffffffu, ai, o);
                aj += __shfl_xor_sync(0xffffffffu, aj, o);
            }
            if (sl == 0 && t < ni) {
                gi += ai;
                if (j < i) Gp[P * N + t] = aj;
                if (j == i) {
                    Gp[(tri(i) + i) * N + t] = gi;
                    gi = 0.0;
                }
            }
        }
        jown = warp_sum(jown);
        if (lane == 0) wpart[r * (JK_THREADS / 32) + warp] = jown;
        __syncthreads();                              // row r fully consumed: refill its buffer
        if (tid == 0 && r + nbuf < nrows) issue(r + nbuf);
    }
    for (int r = tid; r < nrows; r += JK_THREADS) {
        int i, j;
        row_ij(r, i, j);
        double s = 0.0;
        for (int w = 0; w < JK_THREADS / 32; ++w) s += wpart[r * (JK_THREADS / 32) + w];
        Jp[tri(i) + j] = s;
    }
    const int local = cta - b.m_jkcta0[m];
    double *Js = Jp + (int64_t)(1 + local) * npp;
#pragma unroll
    for (int q = 0; q < JK_NREG; ++q) {
        const int64_t e = tid + (int64_t)q * JK_THREADS;
        if (e < npp) Js[e] = jsc[q];
    }
}

template <typename ST, typename RT>
static void launch_jk_t(const DevBatch &b, int nmax, cudaStream_t s) {
    int nbuf = 2;
    size_t sm = jk_layout<ST, RT>(nmax, 2).total;
    if (sm > 227 * 1024) {
        nbuf = 1;
        sm = jk_layout<ST, RT>(nmax, 1).total;
    }
    cudaFuncSetAttribute(k_jk<ST, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_jk<ST, RT><<<b.n_jk_cta, JK_THREADS, sm, s>>>(b, nbuf);
}

void launch_jk(const DevBatch &b, int nmax, cudaStream_t s) {
    if (b.prec == 0) launch_jk_t<double, double>(b, nmax, s);
    else launch_jk_t<float, float>(b, nmax, s);
}

}  // namespace dftb
