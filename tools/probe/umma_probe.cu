// Standalone probe of the tcgen05 (UMMA) TF32 path used by the XC contractions:
// SWIZZLE_128B K-major / MN-major shared-memory descriptors, M=64 and M=128 TMEM
// accumulator layouts, 3xTF32 split products.  Build + run on a B200:
//   nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a tools/probe/umma_probe.cu -o /tmp/umma_probe && /tmp/umma_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#ifndef IL
#define IL 0
#endif
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// element (row, col) of a SW128 atom-tiled buffer with nseg 32-column segments per 8-row group
__device__ __forceinline__ int sw_idx(int row, int col, int nseg) {
    const int atom = (row >> 3) * nseg + (col >> 5);
    const int r = row & 7, ch = ((col & 31) >> 2) ^ r;
    return atom * 256 + r * 32 + ch * 4 + (col & 3);
}

// element (row, col) of an INTERLEAVE (no swizzle) buffer: 128-byte core blocks [8 rows][4 cols]
__device__ __forceinline__ int il_idx(int row, int col, int ncols) {
    return (((row >> 3) * (ncols >> 2) + (col >> 2)) << 5) + ((row & 7) << 2) + (col & 3);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t lt = 2) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;            // version (sm100)
    d |= (uint64_t)lt << 61;           // 2 = SWIZZLE_128B, 1 = SWIZZLE_128B_BASE32B
    return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int amaj, int bmaj) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(su32(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ float rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ float lo_part(float x) { return x - __int_as_float(__float_as_int(x) & 0xffffe000); }

template <int NC>
__device__ __forceinline__ void tld(uint32_t addr, float (&v)[NC]);
template <>
__device__ __forceinline__ void tld<16>(uint32_t addr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// phi: [64 mu][64 p], rho: [NP mu][NP nu] (general), wv: [NP nu][64 p]; NP = 64 or 80
// out_t[p][nu] = sum_mu phi[mu][p] rho[mu][nu]        (M = 64 points, MN-major A, K-major B)
// out_v[mu][nu] = sum_p phi[mu][p] wv[nu][p]          (M = 64 or 128 AOs, K-major A and B)
template <int NP, int MV>
__global__ void k_probe(const float *phi, const float *rho, const float *wv, float *out_t, float *out_v, int split,
                        int var) {
    constexpr int BP = 64, NSEG_P = 2, NSEG_R = (NP + 31) / 32;
    constexpr int PLANE = (NP / 8) * NSEG_P * 256;           // floats per phi/wv buffer
    constexpr int RHO = (NP / 8) * NSEG_R * 256;
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    float *sm = (float *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    float *s_phil = sm;                    // phi lo
    float *s_phi = s_phil + PLANE;         // phi (hi by truncation)
    float *s_pad = s_phi + PLANE;          // zero pad: M=128 reads past the AO rows
    float *s_wv = s_pad + 2 * PLANE;
    float *s_wvl = s_wv + PLANE;
    float *s_rho = s_wvl + PLANE;          // K-major B of the t phase: rows nu, cols mu
    float *s_rhol = s_rho + RHO;
    float *s_phiT = s_rhol + RHO;          // var 4: phi^T K-major, rows p, cols mu (SW128)
    float *s_phiTl = s_phiT + PLANE;
    float *s_p32 = s_phiTl + PLANE;        // var 5: phi MN-major SWIZZLE_128B_BASE32B (rows mu, 32 p per 128 B)
    float *s_p32l = s_p32 + PLANE;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    auto IX = [&](int r, int c, int nseg) { return IL ? il_idx(r, c, nseg * 32) : sw_idx(r, c, nseg); };
    for (int i = tid; i < NP * BP; i += blockDim.x) {
        const int mu = i / BP, p = i % BP;
        const float x = phi[i], w = wv[i];
        s_phi[IX(mu, p, NSEG_P)] = x;
        if (split == 2) {   // round-to-nearest hi, exact lo
            const float h = rna(x);
            s_phi[IX(mu, p, NSEG_P)] = h;
            s_phil[IX(mu, p, NSEG_P)] = x - h;
        } else {
            s_phil[IX(mu, p, NSEG_P)] = split ? lo_part(x) : 0.f;
        }
        s_wv[IX(mu, p, NSEG_P)] = w;
        if (split == 2) {
            const float h = rna(w);
            s_wv[IX(mu, p, NSEG_P)] = h;
            s_wvl[IX(mu, p, NSEG_P)] = w - h;
        } else {
            s_wvl[IX(mu, p, NSEG_P)] = split ? lo_part(w) : 0.f;
        }
    }
    for (int i = tid; i < 2 * PLANE; i += blockDim.x) s_pad[i] = 0.f;
    for (int i = tid; i < NP * BP; i += blockDim.x) {
        const int mu = i / BP, p = i % BP;
        const float x = phi[i], h = rna(x);
        s_phiT[sw_idx(p, mu, (NP + 31) / 32)] = h;
        s_phiTl[sw_idx(p, mu, (NP + 31) / 32)] = x - h;
        // BASE32B: 512-byte atoms of 4 rows (mu) x 128 B (32 p); 32-byte granule g ^ (row & 3)
        const int atom = (mu >> 2) * NSEG_P + (p >> 5), r = mu & 3, g = ((p & 31) >> 3) ^ r;
        const int o = atom * 128 + r * 32 + g * 8 + (p & 7);
        s_p32[o] = h;
        s_p32l[o] = x - h;
    }
    for (int i = tid; i < NP * NP; i += blockDim.x) {
        const int mu = i / NP, nu = i % NP;
        const float x = rho[i];
        s_rho[IX(nu, mu, NSEG_R)] = x;
        if (split == 2) {
            const float h = rna(x);
            s_rho[IX(nu, mu, NSEG_R)] = h;
            s_rhol[IX(nu, mu, NSEG_R)] = x - h;
        } else {
            s_rhol[IX(nu, mu, NSEG_R)] = split ? lo_part(x) : 0.f;
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t T = tbase, V = tbase + 128;
    if (tid == 0) {
        // t phase: A = phi MN-major (MN = p: LBO = segment stride 1 KB; K = mu: SBO = 8-row group stride)
        const uint32_t it = idesc_tf32(64, NP, 1, 0);
        for (int kk = 0; kk < NP / 8; ++kk) {
            uint32_t ao = kk * NSEG_P * 1024;                       // mu group kk
            uint32_t bo = (kk >> 2) * 1024 + (kk & 3) * 32;         // K = mu inside rho rows
            uint32_t L = (var & 1) ? NSEG_P * 1024 : 1024, S = (var & 1) ? 1024 : NSEG_P * 1024;
            uint32_t lt = (var & 2) ? 1 : 2;
            uint32_t bL = 16, bS = NSEG_R * 1024;
            if (IL) {   // A: core blocks (mu/8, p/4): MN = p chunks at 128 B (SBO), K groups at BP/4*128 (LBO)
                ao = kk * (BP / 4) * 128; bo = kk * 256;
                L = (var & 1) ? 128 : (BP / 4) * 128; S = (var & 1) ? (BP / 4) * 128 : 128; lt = 0;
                bL = 128; bS = NSEG_R * 1024;
            }
            const uint64_t a_hi = sdesc(su32(s_phi) + ao, L, S, lt);
            const uint64_t a_lo = sdesc(su32(s_phil) + ao, L, S, lt);
            const uint64_t b_hi = sdesc(su32(s_rho) + bo, bL, bS, IL ? 0 : 2);
            const uint64_t b_lo = sdesc(su32(s_rhol) + bo, bL, bS, IL ? 0 : 2);
            if (var == 4) {   // K-major A = phi^T rows p
                const uint32_t o = (kk >> 2) * 1024 + (kk & 3) * 32;
                const uint32_t NS = (NP + 31) / 32;
                const uint32_t it4 = idesc_tf32(64, NP, 0, 0);
                const uint64_t h = sdesc(su32(s_phiT) + o, 16, NS * 1024), l = sdesc(su32(s_phiTl) + o, 16, NS * 1024);
                const uint64_t bh = sdesc(su32(s_rho) + bo, bL, bS, IL ? 0 : 2), bl = sdesc(su32(s_rhol) + bo, bL, bS, IL ? 0 : 2);
                mma_tf32(T, h, bl, it4, kk > 0); mma_tf32(T, l, bh, it4, 1); mma_tf32(T, h, bh, it4, 1);
                continue;
            }
            if (var >= 5) {   // MN-major BASE32B: LBO = 32-point segment stride, SBO = 4-row group stride
                const uint32_t o = kk * 2 * NSEG_P * 512;
                const uint32_t LL = var == 5 ? 512 : NSEG_P * 512, SS = var == 5 ? NSEG_P * 512 : 512;
                const uint64_t h = sdesc(su32(s_p32) + o, LL, SS, 1), l = sdesc(su32(s_p32l) + o, LL, SS, 1);
                const uint64_t bh = sdesc(su32(s_rho) + bo, bL, bS, IL ? 0 : 2), bl = sdesc(su32(s_rhol) + bo, bL, bS, IL ? 0 : 2);
                mma_tf32(T, h, bl, it, kk > 0); mma_tf32(T, l, bh, it, 1); mma_tf32(T, h, bh, it, 1);
                continue;
            }
            mma_tf32(T, a_hi, b_lo, it, kk > 0);
            mma_tf32(T, a_lo, b_hi, it, 1);
            mma_tf32(T, a_hi, b_hi, it, 1);
        }
        // V phase: A = phi K-major (MN = mu rows, SBO = 8-row group stride), B = wv K-major
        const uint32_t iv = idesc_tf32(MV, NP, 0, 0);
        for (int kk = 0; kk < BP / 8; ++kk) {
            const uint32_t ko = IL ? kk * 256 : (kk >> 2) * 1024 + (kk & 3) * 32;
            const uint32_t L = IL ? 128 : 16, S = IL ? (BP / 4) * 128 : NSEG_P * 1024, lt = IL ? 0 : 2;
            const uint64_t a_hi = sdesc(su32(s_phi) + ko, L, S, lt);
            const uint64_t a_lo = sdesc(su32(s_phil) + ko, L, S, lt);
            const uint64_t b_hi = sdesc(su32(s_wv) + ko, L, S, lt);
            const uint64_t b_lo = sdesc(su32(s_wvl) + ko, L, S, lt);
            mma_tf32(V, a_hi, b_lo, iv, kk > 0);
            mma_tf32(V, a_lo, b_hi, iv, 1);
            mma_tf32(V, a_hi, b_hi, iv, 1);
        }
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // read back: warps 0-3 (one per lane quarter)
    if (warp < 4) {
        for (int c0 = 0; c0 < NP; c0 += 16) {
            float v[16];
            tld<16>(T + ((uint32_t)(warp * 32) << 16) + c0, v);
            if (lane < 16) {
                const int p = 16 * warp + lane;                   // M = 64 layout
                for (int i = 0; i < 16; ++i) out_t[p * NP + c0 + i] = v[i];
            }
            tld<16>(V + ((uint32_t)(warp * 32) << 16) + c0, v);
            if (MV == 128) {
                const int mu = 32 * warp + lane;
                if (mu < NP) for (int i = 0; i < 16; ++i) out_v[mu * NP + c0 + i] = v[i];
            } else if (lane < 16) {
                const int mu = 16 * warp + lane;
                for (int i = 0; i < 16; ++i) out_v[mu * NP + c0 + i] = v[i];
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(256));
}

template <int NP, int MV>
static void run(int split, int var = 0) {
    const int BP = 64;
    std::vector<float> phi(NP * BP), rho(NP * NP), wv(NP * BP), ot(BP * NP), ov(NP * NP);
    srand(7);
    auto rnd = [] { return (float)((rand() / (double)RAND_MAX) * 2.0 - 1.0) * 0.73f; };
    for (auto &x : phi) x = rnd();
    for (auto &x : rho) x = rnd();
    for (auto &x : wv) x = rnd();
    float *dphi, *drho, *dwv, *dt, *dv;
    CK(cudaMalloc(&dphi, phi.size() * 4)); CK(cudaMalloc(&drho, rho.size() * 4)); CK(cudaMalloc(&dwv, wv.size() * 4));
    CK(cudaMalloc(&dt, ot.size() * 4)); CK(cudaMalloc(&dv, ov.size() * 4));
    CK(cudaMemcpy(dphi, phi.data(), phi.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(drho, rho.data(), rho.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dwv, wv.data(), wv.size() * 4, cudaMemcpyHostToDevice));
    const int PLANE = (NP / 8) * 2 * 256, RHO = (NP / 8) * ((NP + 31) / 32) * 256;
    const size_t smem = (size_t)(10 * PLANE + 2 * RHO) * 4 + 1024;
    CK(cudaFuncSetAttribute(k_probe<NP, MV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_probe<NP, MV><<<1, 256, smem>>>(dphi, drho, dwv, dt, dv, split, var);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(ot.data(), dt, ot.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ov.data(), dv, ov.size() * 4, cudaMemcpyDeviceToHost));
    double et = 0, ev = 0, st = 0, sv = 0;
    for (int p = 0; p < BP; ++p)
        for (int nu = 0; nu < NP; ++nu) {
            double r = 0;
            for (int mu = 0; mu < NP; ++mu) r += (double)phi[mu * BP + p] * rho[mu * NP + nu];
            et = fmax(et, fabs(r - ot[p * NP + nu])); st = fmax(st, fabs(r));
        }
    for (int mu = 0; mu < NP; ++mu)
        for (int nu = 0; nu < NP; ++nu) {
            double r = 0;
            for (int p = 0; p < BP; ++p) r += (double)phi[mu * BP + p] * wv[nu * BP + p];
            ev = fmax(ev, fabs(r - ov[mu * NP + nu])); sv = fmax(sv, fabs(r));
        }
    printf("IL=%d var=%d NP=%d MV=%d split=%d: t max|err| %.3e (rel %.3e)   V max|err| %.3e (rel %.3e)\n", IL, var, NP, MV, split, et,
           et / st, ev, ev / sv);
    (void)var;
    cudaFree(dphi); cudaFree(drho); cudaFree(dwv); cudaFree(dt); cudaFree(dv);
}

int main() {
    for (int v = 4; v < 7; ++v) run<64, 64>(2, v);
    run<80, 128>(2, 4); run<80, 128>(2, 5); run<80, 128>(2, 6);
    run<64, 64>(0);
    run<64, 64>(2);
    run<64, 128>(1);
    run<80, 128>(1);
    return 0;
}
