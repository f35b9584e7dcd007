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

constexpr int JK_R = 4;                  // rows per chunk (one TMA bulk copy)
constexpr int JK_G = JK_THREADS / JK_R;  // threads per row (64)

struct JKLayout {
    size_t stage, rho, lut, gpart, total;
    int64_t chunk;                        // elements per staging buffer
};

template <typename ST>
HD JKLayout jk_layout(int N, int nbuf) {
    const int g = 16 / (int)sizeof(ST);
    const int64_t npp = (int64_t)N * (N + 1) / 2;
    JKLayout L;
    L.chunk = (int64_t)JK_R * rowpad(npp, g);
    size_t o = 64;                                    // mbarriers
    L.stage = o; o += (size_t)nbuf * L.chunk * sizeof(ST);
    o = (o + 15) & ~(size_t)15;
    L.rho = o; o += (size_t)N * N * sizeof(double);
    L.lut = o; o += (size_t)npp * sizeof(uint16_t);
    o = (o + 15) & ~(size_t)15;
    L.gpart = o; o += (size_t)JK_R * 2 * JK_G * sizeof(double);
    L.total = o;
    return L;
}

// A CTA digests the rows P = (i, j) of one or two i-slabs in chunks of JK_R consecutive
// rows (contiguous in HBM -> one cp.async.bulk per chunk, double buffered).  Within a
// chunk, 64 threads per row form the J_P dot product and the two K GEMVs with the
// row's symmetric ket matrix T, read straight from the staged packed row:
//   element (k, l) sits at tri(k) + l, so column t of T is row[tri(t) + n] (n < t) and
//   row[tri(n) + t] (n >= t); a single merged walk over n keeps every lane busy.
// The scattered J_Q contributions are done column-wise per chunk by the thread that owns
// Q (Q = tid mod 256), so they accumulate in registers across the CTA's rows.
template <typename ST>
__global__ void __launch_bounds__(JK_THREADS) k_jk(DevBatch b, int nbuf) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int cta = blockIdx.x;
    const int m = b.jk_mol[cta];
    if (b.done[m]) return;
    const int N = b.m_nao[m];
    const int g = 16 / (int)sizeof(ST);
    const int64_t npp = tri(N);
    const JKLayout L = jk_layout<ST>(N, nbuf);
    uint64_t *bar = (uint64_t *)sm;
    ST *stage = (ST *)(sm + L.stage);
    double *rho = (double *)(sm + L.rho);
    uint16_t *lut = (uint16_t *)(sm + L.lut);
    double *gpart = (double *)(sm + L.gpart);
    const int tid = threadIdx.x;
    const int grp = tid / JK_G, gt = tid % JK_G;      // row slot in the chunk, thread in the row
    const ST *eri = (const ST *)b.eri + b.m_eri0[m];
    const int iv[2] = {b.jk_i0[cta], b.jk_i1[cta]};
    // chunk list: (slab s, first j); nch0 chunks for the first slab
    const int nch0 = (iv[0] + JK_R) / JK_R;
    const int nch = nch0 + (iv[1] >= 0 ? (iv[1] + JK_R) / JK_R : 0);
    auto chunk_of = [&](int c, int &i, int &j0, int &nr) {
        const int s = c < nch0 ? 0 : 1, cc = c < nch0 ? c : c - nch0;
        i = iv[s];
        j0 = cc * JK_R;
        nr = min(JK_R, i + 1 - j0);
    };
    auto issue = [&](int c) {
        int i, j0, nr;
        chunk_of(c, i, j0, nr);
        const int64_t P0 = tri(i) + j0;
        const int64_t e0 = rowbase(P0, g), e1 = rowbase(P0 + nr, g);
        bulk_row(stage + (c % nbuf) * L.chunk, eri + e0, (uint32_t)((e1 - e0) * sizeof(ST)), bar + (c % nbuf));
    };
    if (tid == 0) {
        for (int k = 0; k < nbuf; ++k) mbar_init(bar + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int c = 0; c < nbuf && c < nch; ++c) issue(c);
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
    double gi0 = 0.0, gi1 = 0.0;                      // G_i[t] partials, t = gt and gt + 64
    for (int c = 0; c < nch; ++c) {
        int i, j0, nr;
        chunk_of(c, i, j0, nr);
        const int64_t P0 = tri(i) + j0;
        const ST *cbuf = stage + (c % nbuf) * L.chunk;
        mbar_wait(bar + (c % nbuf), (uint32_t)((c / nbuf) & 1));
        const int64_t rb0 = rowbase(P0, g);
        if (grp < nr) {
            const int j = j0 + grp;
            const int P = (int)(P0 + grp);
            const ST *row = cbuf + (rowbase(P, g) - rb0);
            // ---- J_P = sum_Q v_PQ rho~_Q  (64 threads, fixed shuffle tree + smem pair sum)
            double jown = 0.0;
            for (int e = gt; e <= P; e += JK_G) {
                const int kl = lut[e], k = kl >> 8, l = kl & 255;
                jown += (double)row[e] * rho[k * N + l] * (k != l ? 2.0 : 1.0);
            }
            jown = warp_sum(jown);
            // ---- K: G_i[t] += (T rho_j)[t], G_j[t] = (T rho_i)[t]
            const double *rj = rho + j * N, *ri = rho + i * N;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int t = gt + h * JK_G;
                if (t > i) break;
                const int tt = (int)tri(t);
                double ai = 0.0, aj = 0.0;
                int trin = 0;                         // tri(n)
                for (int n = 0; n <= i; ++n) {
                    const int e = n < t ? tt + n : trin + t;
                    trin += n + 1;
                    if (e <= P) {
                        const double v = (double)row[e];
                        ai += v * rj[n];
                        aj += v * ri[n];
                    }
                }
                // T = 2 v except the row's own element (weight 1): corrected once
                ai *= 2.0;
                aj *= 2.0;
                const double vp = (double)row[P];
                if (t == j) { ai -= vp * rj[i]; aj -= vp * ri[i]; }
                else if (t == i) { ai -= vp * rj[j]; aj -= vp * ri[j]; }
                if (h == 0) gi0 += ai; else gi1 += ai;
                if (j < i) Gp[(int64_t)P * N + t] = aj;
            }
            if ((tid & 31) == 0) gpart[2 * JK_G * JK_R - 1 - (tid >> 5)] = jown;   // 2 warps per row
        }
        // ---- scattered J_Q += v_PQ rho~_P for Q < P, thread-owned Q across the CTA's rows
        {
            int off[JK_R];
            double rt[JK_R];
#pragma unroll
            for (int r = 0; r < JK_R; ++r) {
                const int j = min(j0 + r, i);
                off[r] = (int)(rowbase(P0 + r, g) - rb0);
                rt[r] = r < nr ? rho[i * N + j] * (i != j ? 2.0 : 1.0) : 0.0;
            }
            const int Pend = (int)(P0 + nr - 1);      // Q < P for some row of the chunk
            const int Pfirst = (int)P0;
#pragma unroll
            for (int q = 0; q < JK_NREG; ++q) {
                const int Q = tid + q * JK_THREADS;
                if (Q >= Pend) break;
                double acc = 0.0;
                if (Q < Pfirst) {                     // below every row of the chunk
#pragma unroll
                    for (int r = 0; r < JK_R; ++r)
                        if (r < nr) acc += (double)cbuf[off[r] + Q] * rt[r];
                } else {
#pragma unroll
                    for (int r = 0; r < JK_R; ++r)
                        if (r < nr && Q < Pfirst + r) acc += (double)cbuf[off[r] + Q] * rt[r];
                }
                jsc[q] += acc;
            }
        }
        __syncthreads();                              // chunk consumed; J_P partials visible
        if (tid < nr) {
            const int w0 = 2 * JK_G * JK_R - 1 - 2 * tid;
            Jp[P0 + tid] = gpart[w0] + gpart[w0 - 1];
        }
        if (tid == 0 && c + nbuf < nch) issue(c + nbuf);
        if (j0 + nr == i + 1) {                       // slab complete: reduce G_i over the row groups
            __syncthreads();
            gpart[grp * 2 * JK_G + gt] = gi0;
            gpart[grp * 2 * JK_G + JK_G + gt] = gi1;
            __syncthreads();
            if (tid <= i) {
                double s = 0.0;
                for (int r = 0; r < JK_R; ++r) s += gpart[r * 2 * JK_G + tid];
                Gp[(tri(i) + i) * N + tid] = s;
            }
            gi0 = gi1 = 0.0;
            __syncthreads();
        }
    }
    const int local = cta - b.m_jkcta0[m];
    double *Js = Jp + (int64_t)(1 + local) * npp;
#pragma unroll
    for (int q = 0; q < JK_NREG; ++q) {
        const int64_t e = tid + (int64_t)q * JK_THREADS;
        if (e < npp) Js[e] = jsc[q];
    }
}

template <typename ST>
static void launch_jk_t(const DevBatch &b, int nmax, cudaStream_t s) {
    int nbuf = 2;
    size_t sm = jk_layout<ST>(nmax, 2).total;
    if (sm > 227 * 1024) {
        nbuf = 1;
        sm = jk_layout<ST>(nmax, 1).total;
    }
    cudaFuncSetAttribute(k_jk<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_jk<ST><<<b.n_jk_cta, JK_THREADS, sm, s>>>(b, nbuf);
}

void launch_jk(const DevBatch &b, int nmax, cudaStream_t s) {
    if (b.prec == 0) launch_jk_t<double>(b, nmax, s);
    else launch_jk_t<float>(b, nmax, s);
}

}  // namespace dftb
