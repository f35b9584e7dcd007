// Shell-pair tables, Schwarz bounds and the class-specialised ERI kernels.
//
// Reference path: deskdft.integrals.eri_packed (integrals.py:135-196) ->
// _schwarz_kernel / _fill_kernel / _quartet_block (_kernels.py:350-619).
//
// Layout decisions (B200-first):
//  * fused S / L(sp) shells; quartets grouped in 6 classes so every warp runs one
//    fully-unrolled code path (template on shell kinds and on the ket component
//    slice, which is warp-uniform because it is blockIdx.y);
//  * primitive-pair records are SoA with the pair index fastest, so the 32 lanes of
//    a warp (consecutive ket pairs) read one coalesced 256-byte line per field;
//  * results go to the dense per-molecule store in the "ket-tiled rows" layout
//    (common.cuh): one row per canonical bra pair P = (i, j), its kets as 4x4 tiles of
//    the symmetric ket matrix, so the J/K kernel streams whole rows with bulk copies and
//    16-byte tile loads; every canonical element has exactly one writer, and the stores
//    are streaming (evict-first: the store is next read by J/K, after the whole stage);
//  * the two ket-split classes (LL|LL, LL|LS) take two ket components per slice and
//    every class except SS|SS keeps its ket pair's nine primitive records in shared
//    memory (they are re-read once per bra primitive).
#include "common.cuh"
#include "md.cuh"

namespace dftb {

// --------------------------------------------------------------------------- pair records
__global__ void k_pairs(DevBatch b) {
    const int64_t pr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pr >= b.n_pair) return;
    const int sa = b.p_sa[pr], sb = b.p_sb[pr];
    const double *A = b.a_xyz + 3 * b.s_atom[sa];
    const double *B = b.a_xyz + 3 * b.s_atom[sb];
    double rab2 = 0.0;
    for (int d = 0; d < 3; ++d) {
        b.p_geo[(int64_t)d * b.n_pair + pr] = A[d];
        b.p_geo[(int64_t)(3 + d) * b.n_pair + pr] = B[d];
        rab2 += (A[d] - B[d]) * (A[d] - B[d]);
    }
    const int64_t np = b.n_pair;
    for (int i = 0; i < 3; ++i) {
        const double a = b.s_exp[3 * sa + i], csa = b.s_cs[3 * sa + i], cpa = b.s_cp[3 * sa + i];
        for (int j = 0; j < 3; ++j) {
            const double e = b.s_exp[3 * sb + j], csb = b.s_cs[3 * sb + j], cpb = b.s_cp[3 * sb + j];
            const double p = a + e;
            const double K = exp(-(a * e / p) * rab2);
            const int k = 3 * i + j;
            auto put = [&](int f, double v) { b.pp[((int64_t)f * 9 + k) * np + pr] = v; };
            put(PF_P, p);
            put(PF_X, (a * A[0] + e * B[0]) / p);
            put(PF_Y, (a * A[1] + e * B[1]) / p);
            put(PF_Z, (a * A[2] + e * B[2]) / p);
            put(PF_H, 0.5 / p);
            put(PF_CSS, csa * csb * K);
            put(PF_CSP, csa * cpb * K);
            put(PF_CPS, cpa * csb * K);
            put(PF_CPP, cpa * cpb * K);
            put(PF_BOUND, fmax(fabs(csa), fabs(cpa)) * fmax(fabs(csb), fabs(cpb)) * K);
        }
    }
}

// --------------------------------------------------------------------------- class geometry
// Pair lists per molecule: [LL | LS | SS] starting at m_pair0[m].
// class -> (bra list, ket list):  0 LL|LL  1 LL|LS  2 LL|SS  3 LS|LS  4 LS|SS  5 SS|SS
__device__ __forceinline__ void class_lists(const DevBatch &b, int m, int cls, int &b0, int &nb,
                                            int &k0, int &nk) {
    const int p0 = b.m_pair0[m];
    const int nll = b.m_npl[3 * m], nls = b.m_npl[3 * m + 1], nss = b.m_npl[3 * m + 2];
    const int s[3] = {p0, p0 + nll, p0 + nll + nls};
    const int n[3] = {nll, nls, nss};
    const int bl[NCLS] = {0, 0, 0, 1, 1, 2}, kl[NCLS] = {0, 1, 2, 1, 2, 2};
    b0 = s[bl[cls]]; nb = n[bl[cls]];
    k0 = s[kl[cls]]; nk = n[kl[cls]];
}

// ERI_TRANSPOSE bit c: class c enumerates its quartets transposed, so that consecutive lanes
// share the inner-loop (ket) pair - its records are then read by broadcast - and differ in
// the outer-loop (bra) pair; for the triangle classes the quartet (c | r), c <= r, is the
// same integral set as (r | c) (the store canonicalises every index quadruple).
#ifndef ERI_TRANSPOSE
#define ERI_TRANSPOSE 63   // all six classes (ERI stage 36.8 -> 34.0 ms)
#endif
__device__ __forceinline__ void decode_quartet_t(int cls, int64_t q, int nb, int nk, int &P, int &Q) {
    if (cls == 0 || cls == 3 || cls == 5) {            // triangle: ket r (uniform), bra c <= r
        int64_t r = (int64_t)((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
        while (tri(r + 1) <= q) ++r;
        while (tri(r) > q) --r;
        Q = (int)r;
        P = (int)(q - tri(r));
    } else {
        P = (int)(q % nb);
        Q = (int)(q / nb);
    }
}
__device__ __forceinline__ void decode_quartet(int cls, int64_t q, int nk, int &P, int &Q) {
    if (cls == 0 || cls == 3 || cls == 5) {  // triangle P >= Q
        int64_t r = (int64_t)((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
        while (tri(r + 1) <= q) ++r;
        while (tri(r) > q) --r;
        P = (int)r;
        Q = (int)(q - tri(r));
    } else {
        P = (int)(q / nk);
        Q = (int)(q % nk);
    }
}

template <int N, typename F>
__device__ __forceinline__ void static_switch(int c, F &&f) {
    // dispatch a runtime value in [0, N) to f(integral_constant) — c is warp-uniform here
    if constexpr (N >= 1) { if (c == 0) { f(std::integral_constant<int, 0>{}); return; } }
    if constexpr (N >= 2) { if (c == 1) { f(std::integral_constant<int, 1>{}); return; } }
    if constexpr (N >= 3) { if (c == 2) { f(std::integral_constant<int, 2>{}); return; } }
    if constexpr (N >= 4) { if (c == 3) { f(std::integral_constant<int, 3>{}); return; } }
    if constexpr (N >= 5) { if (c == 4) { f(std::integral_constant<int, 4>{}); return; } }
    if constexpr (N >= 6) { if (c == 5) { f(std::integral_constant<int, 5>{}); return; } }
    if constexpr (N >= 7) { if (c == 6) { f(std::integral_constant<int, 6>{}); return; } }
    if constexpr (N >= 8) { if (c == 7) { f(std::integral_constant<int, 7>{}); return; } }
    if constexpr (N >= 9) { if (c == 8) { f(std::integral_constant<int, 8>{}); return; } }
    if constexpr (N >= 10) { if (c == 9) { f(std::integral_constant<int, 9>{}); return; } }
    if constexpr (N >= 11) { if (c == 10) { f(std::integral_constant<int, 10>{}); return; } }
    if constexpr (N >= 12) { if (c == 11) { f(std::integral_constant<int, 11>{}); return; } }
    if constexpr (N >= 13) { if (c == 12) { f(std::integral_constant<int, 12>{}); return; } }
    if constexpr (N >= 14) { if (c == 13) { f(std::integral_constant<int, 13>{}); return; } }
    if constexpr (N >= 15) { if (c == 14) { f(std::integral_constant<int, 14>{}); return; } }
    if constexpr (N >= 16) { if (c == 15) { f(std::integral_constant<int, 15>{}); return; } }
}

__device__ __forceinline__ void load_geo(const DevBatch &b, int64_t pr, double *A, double *B) {
    for (int d = 0; d < 3; ++d) {
        A[d] = b.p_geo[(int64_t)d * b.n_pair + pr];
        B[d] = b.p_geo[(int64_t)(3 + d) * b.n_pair + pr];
    }
}

template <typename ST>
__device__ __forceinline__ void store_eri(ST *eri, int64_t base, int i, int j, int k, int l, double v) {
    // written once, read by the next stage: streaming (evict-first) store, so the output
    // does not push the primitive-pair tables out of L2
    __stcs(eri + base + eri_pos(i, j, k, l), (ST)v);
}

// --------------------------------------------------------------------------- ERI kernels
// Per-thread shared-memory copy of the ket pair's nine primitive records: the primitive
// loop reads each ket record once per bra primitive (81 times per quartet), so keeping them
// next to the SM removes ~8/9 of the kernel's load traffic.  Slots [slot][prim][thread];
// S-only kets need 7 fields (the screening bound goes to slot 6).
constexpr int ERI_T = 128;
// Only the latency-critical fields are cached (p, P, 1/2p, bound, and c_ss for L kets);
// the coefficient products read from global memory are consumed after the Boys / R_tuv
// chain, which hides their latency, and leaving them out keeps the cache small enough for
// 3 (L kets, 64.5 KB) or 4 (S kets, 55 KB) CTAs per SM.
template <bool LKET, int NS = (LKET ? 7 : 6)>
struct KetSmem {
    // 7 slots: p, P, 1/2p, c_ss, bound; 6 slots: p, P, 1/2p, bound (55 KB per CTA: 4 CTAs
    // per SM), c_ss from global as well
    static constexpr int NSLOT = NS;
    const double *s;
    int lane;
    PPView g;
    __device__ __forceinline__ static int slot(int f) { return f == PF_BOUND ? NSLOT - 1 : f; }
    __device__ __forceinline__ static int field(int sl) { return sl == NSLOT - 1 ? (int)PF_BOUND : sl; }
    __device__ __forceinline__ double get(int f, int k, int64_t pair) const {
        if (f == PF_CSP || f == PF_CPS || f == PF_CPP || (NS == 6 && f == PF_CSS)) return g.get(f, k, pair);
        return s[(slot(f) * 9 + k) * ERI_T + lane];
    }
};

// Per-warp copy of the inner (ket) pair's nine primitive records (all 10 fields) when every
// active lane of the warp has the same ket pair - the usual case with the transposed quartet
// enumeration - else the records come from global memory.  Reads are shared-memory broadcasts
// at constant offsets (no 64-bit address arithmetic per field).
struct WarpKet {
    const double *s;     // [10 fields][9 prims] of this warp, or null
    PPView g;
    __device__ __forceinline__ double get(int f, int k, int64_t pair) const {
        return s ? s[f * 9 + k] : g.get(f, k, pair);
    }
};
#ifndef ERI_WKC
#define ERI_WKC 2        // per-warp ket records: 1 every class, 2 the classes without the per-thread cache
#endif
#ifndef ERI_WKC_PAD
#define ERI_WKC_PAD 0    // A/B: extra shared memory for the classes that had the per-thread cache
#endif

// One thread = one screened shell quartet x one component slice (blockIdx.y).
// KPS: inner-pair components per slice (0 = all): a slice recomputes the Boys function and
// R_tuv of all 81 primitive quartets, so fewer slices trade registers for less recomputation.
// SW (swapped roles): lanes of a warp hold consecutive quartets of one bra pair P and
// consecutive ket pairs Q, so P's primitive records are warp-uniform and Q's per-lane.  The
// McMurchie-Davidson loop reads its inner pair's records 81 times per quartet and its outer
// pair's 9 times; with SW the per-lane ket pair is the outer one and the warp-uniform bra pair
// the inner one (broadcast loads from L1), i.e. (ab|cd) is evaluated as (cd|ab) and the
// slices run over bra components.  Without SW the ket records are re-read per bra primitive
// and KSM keeps them in shared memory.
template <int KA, int KB, int KC, int KD, int KPS, typename ST, bool KSM = true, int MINB = 1,
          int NS = ((KC || KD) ? 7 : 6), bool SW = false>
__global__ void __launch_bounds__(ERI_T, MINB) k_eri(DevBatch b, int cls, double eps, double prim_cut, ST *eri) {
    constexpr int NA = KA ? 4 : 1, NB = KB ? 4 : 1, NC = KC ? 4 : 1, ND = KD ? 4 : 1;
    constexpr int NOUT = SW ? NC * ND : NA * NB;              // outer-pair components
    constexpr int NIN = SW ? NA * NB : NC * ND;               // inner-pair components (sliced)
    constexpr int NKS = KPS ? KPS : NIN, NSL = NIN / NKS;
    static_assert(NIN % NKS == 0, "slice size must divide the inner component count");
    static_assert(!(SW && KSM), "the swapped form reads its inner (bra) records by broadcast");
    const int64_t *pre = b.cls0 + (int64_t)cls * (b.n_mol + 1);
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= pre[b.n_mol]) return;
    const int m = find_mol(pre, b.n_mol, g);
    int b0, nb, k0, nk;
    class_lists(b, m, cls, b0, nb, k0, nk);
    int P, Q;
    if ((ERI_TRANSPOSE >> cls) & 1) decode_quartet_t(cls, g - pre[m], nb, nk, P, Q);
    else decode_quartet(cls, g - pre[m], nk, P, Q);
    const int64_t Pp = b0 + P, Qp = k0 + Q;
    if (b.p_q[Pp] * b.p_q[Qp] < eps) return;
    double A[3], B[3], C[3], D[3];
    load_geo(b, Pp, A, B);
    load_geo(b, Qp, C, D);
    const PPView V{b.pp, b.n_pair};
    extern __shared__ double eri_ksm[];
    using KS = KetSmem<(KC || KD), NS>;
    const double *wk = nullptr;
    constexpr bool WK = ERI_WKC == 1 ? !SW : ERI_WKC == 2 ? (!SW && !KSM) : false;
    if constexpr (WK) {
        const unsigned mask = __activemask();
        const int lane = threadIdx.x & 31, lead = __ffs(mask) - 1;
        const int64_t q0 = __shfl_sync(mask, Qp, lead);
        if (__all_sync(mask, Qp == q0)) {
            double *ws = eri_ksm + (threadIdx.x >> 5) * 90;
            const int nact = __popc(mask), rk = __popc(mask & ((1u << lane) - 1));
            for (int e = rk; e < 90; e += nact) ws[e] = V.get(e / 9, e % 9, Qp);
            __syncwarp(mask);
            wk = ws;
        }
    }
    if constexpr (KSM && !WK) {
#pragma unroll
        for (int f = 0; f < KS::NSLOT; ++f) {
            const int field = KS::field(f);
#pragma unroll
            for (int k = 0; k < 9; ++k) eri_ksm[(f * 9 + k) * ERI_T + threadIdx.x] = V.get(field, k, Qp);
        }
    }
    const int ia = b.s_ao[b.p_sa[Pp]], ib = b.s_ao[b.p_sb[Pp]];
    const int ic = b.s_ao[b.p_sa[Qp]], id = b.s_ao[b.p_sb[Qp]];
    const int64_t base = b.m_eri0[m];
    static_switch<NSL>(blockIdx.y, [&](auto slc) {
        constexpr int KC0 = decltype(slc)::value * NKS;
        double out[NOUT][NKS];
#pragma unroll
        for (int x = 0; x < NOUT; ++x)
#pragma unroll
            for (int y = 0; y < NKS; ++y) out[x][y] = 0.0;
        if constexpr (SW) {
            eri_quartet_kv<KC, KD, KA, KB, KC0, NKS>(V, V, Qp, Pp, C, D, A, B, b.boys, prim_cut, out);
        } else if constexpr (WK) {
            const WarpKet VK{wk, V};
            eri_quartet_kv<KA, KB, KC, KD, KC0, NKS>(V, VK, Pp, Qp, A, B, C, D, b.boys, prim_cut, out);
        } else if constexpr (KSM) {
            const KS VK{eri_ksm, (int)threadIdx.x, V};
            eri_quartet_kv<KA, KB, KC, KD, KC0, NKS>(V, VK, Pp, Qp, A, B, C, D, b.boys, prim_cut, out);
        } else {
            eri_quartet_kv<KA, KB, KC, KD, KC0, NKS>(V, V, Pp, Qp, A, B, C, D, b.boys, prim_cut, out);
        }
        // single writer per canonical element: for a diagonal shell pair only the
        // (i >= j) component writes, for a diagonal quartet only the (ij >= kl) image
        const bool dab = b.p_sa[Pp] == b.p_sb[Pp], dcd = b.p_sa[Qp] == b.p_sb[Qp], dpq = Pp == Qp;
#pragma unroll
        for (int x = 0; x < NOUT; ++x)
#pragma unroll
            for (int y = 0; y < NKS; ++y) {
                const int xi = SW ? KC0 + y : x;          // bra component index (a, b)
                const int yk = SW ? x : KC0 + y;          // ket component index (c, d)
                const int i = ia + xi / NB, j = ib + xi % NB, k = ic + yk / ND, l = id + yk % ND;
                if (dab && i < j) continue;
                if (dcd && k < l) continue;
                if (dpq && pidx(i, j) < pidx(k, l)) continue;
                store_eri(eri, base, i, j, k, l, b.prec ? (double)(float)out[x][y] : out[x][y]);
            }
    });
}

// --------------------------------------------------------------------------- Schwarz
// q_ao[ij] = sqrt(max(0,(ij|ij))) for every AO pair of the pair; p_q = max over the pair.
// cls: 0 = LL pairs (16 slices, one diagonal component each), 1 = LS, 2 = SS.
template <int KA, int KB, int SPLIT>
__global__ void __launch_bounds__(128) k_schwarz(DevBatch b, int which) {
    constexpr int NA = KA ? 4 : 1, NB = KB ? 4 : 1, NKET = NA * NB;
    constexpr int NKS = SPLIT ? 1 : NKET, NSL = NKET / NKS;
    const int64_t *pre = b.cls0 + (int64_t)(NCLS) * (b.n_mol + 1) + (int64_t)which * (b.n_mol + 1);
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= pre[b.n_mol]) return;
    const int m = find_mol(pre, b.n_mol, g);
    const int p0 = b.m_pair0[m] + (which >= 1 ? b.m_npl[3 * m] : 0) + (which >= 2 ? b.m_npl[3 * m + 1] : 0);
    const int64_t Pp = p0 + (g - pre[m]);
    double A[3], B[3];
    load_geo(b, Pp, A, B);
    const PPView V{b.pp, b.n_pair};
    const int ia = b.s_ao[b.p_sa[Pp]], ib = b.s_ao[b.p_sb[Pp]];
    double *qao = b.qao + b.m_npp0[m];
    static_switch<NSL>(blockIdx.y, [&](auto slc) {
        constexpr int KC0 = decltype(slc)::value * NKS;
        double out[NKET][NKS];
#pragma unroll
        for (int x = 0; x < NKET; ++x)
#pragma unroll
            for (int y = 0; y < NKS; ++y) out[x][y] = 0.0;
        eri_quartet<KA, KB, KA, KB, KC0, NKS>(V, Pp, Pp, A, B, A, B, b.boys, 0.0, out);
        const bool dab = b.p_sa[Pp] == b.p_sb[Pp];
#pragma unroll
        for (int y = 0; y < NKS; ++y) {
            const int c = KC0 + y;
            const double v = out[c][y];
            if (dab && c / NB < c % NB) continue;   // single writer for symmetric components
            qao[pidx(ia + c / NB, ib + c % NB)] = sqrt(fmax(v, 0.0));
        }
    });
}

__global__ void k_pair_q(DevBatch b) {
    const int64_t pr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pr >= b.n_pair) return;
    // molecule of this pair: pairs are contiguous per molecule (m_pair0 prefix, int)
    int lo = 0, hi = b.n_mol;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (b.m_pair0[mid] <= pr) lo = mid; else hi = mid;
    }
    const int sa = b.p_sa[pr], sb = b.p_sb[pr];
    const int na = b.s_kind[sa] ? 4 : 1, nb = b.s_kind[sb] ? 4 : 1;
    const int ia = b.s_ao[sa], ib = b.s_ao[sb];
    const double *qao = b.qao + b.m_npp0[lo];
    double q = 0.0;
    for (int x = 0; x < na; ++x)
        for (int y = 0; y < nb; ++y) q = fmax(q, qao[pidx(ia + x, ib + y)]);
    b.p_q[pr] = q;
}

// --------------------------------------------------------------------------- launchers
static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

void launch_pairs(const DevBatch &b, cudaStream_t s) {
    if (b.n_pair) k_pairs<<<nblk(b.n_pair, 128), 128, 0, s>>>(b);
}

void launch_schwarz(const DevBatch &b, const int64_t *host_totals, cudaStream_t s) {
    // host_totals[3]: number of LL, LS, SS pairs in the batch
    if (host_totals[0]) k_schwarz<1, 1, 1><<<dim3(nblk(host_totals[0], 128), 16), 128, 0, s>>>(b, 0);
    if (host_totals[1]) k_schwarz<1, 0, 0><<<dim3(nblk(host_totals[1], 128), 1), 128, 0, s>>>(b, 1);
    if (host_totals[2]) k_schwarz<0, 0, 0><<<dim3(nblk(host_totals[2], 128), 1), 128, 0, s>>>(b, 2);
    if (b.n_pair) k_pair_q<<<nblk(b.n_pair, 128), 128, 0, s>>>(b);
}

template <int KA, int KB, int KC, int KD, int KPS, bool KSM = true, int MINB = 1, int NS = ((KC || KD) ? 7 : 6),
          bool SW = false, typename ST>
static void launch_cls(const DevBatch &b, int cls, int64_t n, double eps, double prim_cut, ST *eri,
                       cudaStream_t s, int *nlaunch) {
    if (!n) return;
    constexpr int NIN = SW ? (KA ? 4 : 1) * (KB ? 4 : 1) : (KC ? 4 : 1) * (KD ? 4 : 1);
    constexpr int NSL = NIN / (KPS ? KPS : NIN);
    constexpr bool WK = ERI_WKC == 1 ? !SW : ERI_WKC == 2 ? (!SW && !KSM) : false;
    const size_t sm = WK ? sizeof(double) * 90 * (ERI_T / 32) + ERI_WKC_PAD * KSM
                      : KSM ? sizeof(double) * KetSmem<(KC || KD), NS>::NSLOT * 9 * ERI_T : 0;
    auto kern = k_eri<KA, KB, KC, KD, KPS, ST, KSM, MINB, NS, SW>;
    smem_optin((const void *)kern);
    kern<<<dim3(nblk(n, ERI_T), NSL), ERI_T, sm, s>>>(b, cls, eps, prim_cut, eri);
    ++*nlaunch;
}

#ifndef ERI_S_MINB
#define ERI_S_MINB 4       // LL|SS, LS|SS: 4 CTAs per SM (55 KB ket cache, <= 128 registers)
#endif
#ifndef ERI_LSLS_MINB
#define ERI_LSLS_MINB 4    // LS|LS: 4 CTAs per SM (<= 128 registers, 6-slot ket cache)
#endif
#ifndef ERI_LSLS_NS
#define ERI_LSLS_NS 6
#endif
// Registers vs resident warps per class (B200, 256 x 9-heavy batch): the kernels are
// latency-bound, so more CTAs per SM pays even with some spills.  LL|LL at 3 CTAs (168
// registers): 5.65 -> 5.29 ms; LL|LS at 4 CTAs (128 registers, 6-slot ket cache): 10.97 ->
// 9.51 ms.
#ifndef ERI_LLLL_MINB
#define ERI_LLLL_MINB 3
#endif
#ifndef ERI_LLLL_NS
#define ERI_LLLL_NS 7
#endif
#ifndef ERI_LLLS_MINB
#define ERI_LLLS_MINB 4
#endif
#ifndef ERI_LLLS_NS
#define ERI_LLLS_NS 6
#endif
#ifndef ERI_LLLL_KSM
#define ERI_LLLL_KSM true
#endif
#ifndef ERI_LLLS_KSM
#define ERI_LLLS_KSM true
#endif
#ifndef ERI_LLSS_KSM
#define ERI_LLSS_KSM true
#endif
#ifndef ERI_LLSS_MINB
#define ERI_LLSS_MINB ERI_S_MINB
#endif
#ifndef ERI_LSLS_KSM
#define ERI_LSLS_KSM true
#endif
#ifndef ERI_LSSS_KSM
#define ERI_LSSS_KSM false     // LS|SS: no ket cache, 8 CTAs/SM (64 registers): 13.0 -> 12.2 ms
#endif
#ifndef ERI_LSSS_MINB
#define ERI_LSSS_MINB 8
#endif
#ifndef ERI_SSSS_MINB
#define ERI_SSSS_MINB 12      // SS|SS: 12 CTAs/SM by registers (40): 5.61 -> 5.10 ms
#endif
#ifndef ERI_KPS_LL
#define ERI_KPS_LL 2       // LL|LL: 8 slices of 2 ket components
#endif
#ifndef ERI_KPS_LS
#define ERI_KPS_LS 2       // LL|LS: 2 slices of 2
#endif

// Swapped roles (SW, see k_eri) per class, measured per class on B200 (ncu, kernels alone,
// 256 x 9-heavy batch, ms): LS|LS 7.33 -> 7.14, LS|SS 12.13 -> 11.61 (6 CTAs/SM), SS|SS 5.01 ->
// 4.56; LL|LL 5.28 -> 5.44, LL|SS 4.09 -> 4.88, LL|LS 9.60 -> 16.4 (the bra-component slices
// recompute R_tuv).  In the pipelined stage (one-electron / grid kernels on the aux stream, three
// batches in flight) the swapped S classes made the stage slower, 47.7 -> 49.5 ms, and the
// bench 2127 -> 2088 mol/s (same-box A/B), so every class runs unswapped by default.
#ifndef ERI_SW_LSLS
#define ERI_SW_LSLS 0
#endif
#ifndef ERI_SW_LSSS
#define ERI_SW_LSSS 0
#endif
#ifndef ERI_SW_SSSS
#define ERI_SW_SSSS 0
#endif

template <typename ST>
static void launch_eri_t(const DevBatch &b, const int64_t *tot, double eps, double prim_cut,
                         ST *eri, cudaStream_t s, int *nlaunch) {
    launch_cls<1, 1, 1, 1, ERI_KPS_LL, ERI_LLLL_KSM, ERI_LLLL_MINB, ERI_LLLL_NS>(b, 0, tot[0], eps, prim_cut, eri, s, nlaunch);
    launch_cls<1, 1, 1, 0, ERI_KPS_LS, ERI_LLLS_KSM, ERI_LLLS_MINB, ERI_LLLS_NS>(b, 1, tot[1], eps, prim_cut, eri, s, nlaunch);
    launch_cls<1, 1, 0, 0, 0, ERI_LLSS_KSM, ERI_LLSS_MINB>(b, 2, tot[2], eps, prim_cut, eri, s, nlaunch);
    if (ERI_SW_LSLS) launch_cls<1, 0, 1, 0, 0, false, ERI_LSLS_MINB, 7, true>(b, 3, tot[3], eps, prim_cut, eri, s, nlaunch);
    else launch_cls<1, 0, 1, 0, 0, ERI_LSLS_KSM, ERI_LSLS_MINB, ERI_LSLS_NS>(b, 3, tot[3], eps, prim_cut, eri, s, nlaunch);
    if (ERI_SW_LSSS) launch_cls<1, 0, 0, 0, 0, false, ERI_LSSS_MINB, 6, true>(b, 4, tot[4], eps, prim_cut, eri, s, nlaunch);
    else launch_cls<1, 0, 0, 0, 0, ERI_LSSS_KSM, ERI_LSSS_MINB>(b, 4, tot[4], eps, prim_cut, eri, s, nlaunch);
    if (ERI_SW_SSSS) launch_cls<0, 0, 0, 0, 0, false, ERI_SSSS_MINB, 6, true>(b, 5, tot[5], eps, prim_cut, eri, s, nlaunch);
    else launch_cls<0, 0, 0, 0, 0, false, ERI_SSSS_MINB>(b, 5, tot[5], eps, prim_cut, eri, s, nlaunch);
}

void launch_eri(const DevBatch &b, const int64_t *tot, double eps, double prim_cut, cudaStream_t s,
                int *nlaunch) {
    if (b.eri64) launch_eri_t<double>(b, tot, eps, prim_cut, (double *)b.eri, s, nlaunch);
    else launch_eri_t<float>(b, tot, eps, prim_cut, (float *)b.eri, s, nlaunch);
}

}  // namespace dftb
