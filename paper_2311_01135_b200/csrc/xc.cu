// Fused AO-on-grid + density + B3LYP + V_xc kernel.
//
// Reference: deskdft.xc.eval_ao (xc.py:165-194), density_on_grid (:309-317),
// b3lyp (:277-306) and xc_matrix (:320-350).  The reference stores phi and
// grad phi for the whole grid and runs two BLAS GEMMs per 8192-point batch.
//
// B200 formulation: one CTA owns a contiguous range of one molecule's grid
// points.  AO values and gradients are recomputed per 32-point sub-block into
// shared memory (never written to HBM), so each SCF iteration reads only the
// density matrix and writes one N x N partial per CTA:
//   pass A: phi -> t = phi rho (smem GEMM) -> n, grad n per point,
//   pass B: B3LYP per point (one thread per point, f64),
//   pass C: phi again -> wv = a phi + b . grad phi -> V += phi^T wv (register tiles).
// W is the arithmetic type of the contractions (double for the f64 build, float for
// the f32 build, as in the reference's f32 BLAS path); the functional is always f64.
#include "common.cuh"
#include "b3lyp.cuh"

namespace dftb {

constexpr int XC_THREADS = 256;
constexpr int XC_SB = 256;       // points per super-block (one per thread in pass B)
constexpr int XC_SHD = 13;       // doubles per shell record in smem

template <typename W>
struct XCSmem {
    W *rho, *phi, *tw;
    double *pt, *dn, *shd, *red;
};

template <typename W>
__device__ __forceinline__ void xc_eval_phi(const XCSmem<W> &s, int nsh, int NP, int BP, int sub, int nb) {
    const int plane = BP * NP;
    for (int t = threadIdx.x; t < BP * nsh; t += XC_THREADS) {
        const int p = t % BP, sh = t / BP;
        const double *r = s.shd + XC_SHD * sh;
        const int kind = (int)r[12] & 1, ao = (int)r[12] >> 1;
        W *o0 = s.phi + p * NP + ao;
        if (p >= nb) {
            const int nc = kind ? 4 : 1;
            for (int c = 0; c < nc; ++c) o0[c] = o0[plane + c] = o0[2 * plane + c] = o0[3 * plane + c] = (W)0;
            continue;
        }
        const double *q = s.pt + 4 * (sub + p);
        const double dx = q[0] - r[0], dy = q[1] - r[1], dz = q[2] - r[2];
        const double r2 = dx * dx + dy * dy + dz * dz;
        double bs = 0.0, ds = 0.0, bp = 0.0, dp = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double ar = r[3 + k] * r2;
            const double e = ar < 745.0 ? exp(-ar) : 0.0;
            const double m2a = -2.0 * r[3 + k];
            bs += r[6 + k] * e;
            ds += r[6 + k] * m2a * e;
            bp += r[9 + k] * e;
            dp += r[9 + k] * m2a * e;
        }
        o0[0] = (W)bs;
        o0[plane] = (W)(dx * ds);
        o0[2 * plane] = (W)(dy * ds);
        o0[3 * plane] = (W)(dz * ds);
        if (kind) {
            const double rel[3] = {dx, dy, dz};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                o0[1 + c] = (W)(rel[c] * bp);
#pragma unroll
                for (int d = 0; d < 3; ++d)
                    o0[(d + 1) * plane + 1 + c] = (W)((c == d ? bp : 0.0) + rel[c] * rel[d] * dp);
            }
        }
    }
}

template <typename W, int BP>
__global__ void __launch_bounds__(XC_THREADS) k_xc(DevBatch b) {
    extern __shared__ __align__(16) unsigned char xsm[];
    constexpr int G = XC_THREADS / BP;           // threads per point in the per-point phases
    const int cta = blockIdx.x;
    const int m = b.xc_mol[cta];
    if (b.done[m]) return;
    const int N = b.m_nao[m];
    const int NP = (N + 15) & ~15;
    const int nsh = b.m_nshell[m], s0 = b.m_shell0[m];
    XCSmem<W> s;
    s.rho = (W *)xsm;
    s.phi = s.rho + NP * NP;
    s.tw = s.phi + 4 * BP * NP;
    s.pt = (double *)(s.tw + BP * NP + ((BP * NP) & 1));
    s.pt = (double *)(((uintptr_t)s.pt + 15) & ~(uintptr_t)15);
    s.dn = s.pt + 4 * XC_SB;
    s.shd = s.dn + 4 * XC_SB;
    s.red = s.shd + XC_SHD * nsh;
    const int tid = threadIdx.x;
    const double *rg = b.rho + b.m_mat0[m];
    for (int t = tid; t < NP * NP; t += XC_THREADS) {
        const int r = t / NP, c = t % NP;
        s.rho[t] = (r < N && c < N) ? (W)rg[r * N + c] : (W)0;
    }
    for (int t = tid; t < 4 * BP * NP; t += XC_THREADS) s.phi[t] = (W)0;
    for (int t = tid; t < BP * NP; t += XC_THREADS) s.tw[t] = (W)0;
    for (int sh = tid; sh < nsh; sh += XC_THREADS) {
        const int g = s0 + sh;
        double *r = s.shd + XC_SHD * sh;
        const double *A = b.a_xyz + 3 * b.s_atom[g];
        for (int d = 0; d < 3; ++d) {
            r[d] = A[d];
            r[3 + d] = b.s_exp[3 * g + d];
            r[6 + d] = b.s_cs[3 * g + d];
            r[9 + d] = b.s_cp[3 * g + d];
        }
        r[12] = (double)((b.s_ao[g] << 1) | (b.s_kind[g] & 1));
    }
    // V accumulator tile: rows ty + 16 a, cols tx + 16 c
    const int ty = tid >> 4, tx = tid & 15;
    W acc[6][6];
#pragma unroll
    for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int c = 0; c < 6; ++c) acc[a][c] = (W)0;
    const int nblk16 = NP >> 4;
    double e_acc = 0.0;
    int bad = 0;
    const int64_t p0 = b.xc_p0[cta], p1 = b.xc_p1[cta];
    const int plane = BP * NP;
    const int gp = tid / G, gl = tid % G;         // point-group mapping
    for (int64_t sb0 = p0; sb0 < p1; sb0 += XC_SB) {
        const int nsb = (int)min((int64_t)XC_SB, p1 - sb0);
        __syncthreads();
        if (tid < nsb) {
            const int64_t gi = sb0 + tid;
            s.pt[4 * tid] = b.g_xyz[3 * gi];
            s.pt[4 * tid + 1] = b.g_xyz[3 * gi + 1];
            s.pt[4 * tid + 2] = b.g_xyz[3 * gi + 2];
            s.pt[4 * tid + 3] = b.g_w[gi];
        }
        __syncthreads();
        // ---- pass A: density and gradient
        for (int sub = 0; sub < nsb; sub += BP) {
            const int nb = min(BP, nsb - sub);
            xc_eval_phi(s, nsh, NP, BP, sub, nb);
            __syncthreads();
            {   // t = phi rho : point gp, columns gl + G r
                W t[96 / G];
#pragma unroll
                for (int r = 0; r < 96 / G; ++r) t[r] = (W)0;
                const W *ph = s.phi + gp * NP;
                for (int k = 0; k < N; ++k) {
                    const W a = ph[k];
                    const W *rr = s.rho + k * NP + gl;
#pragma unroll
                    for (int r = 0; r < 96 / G; ++r)
                        if (r * G < NP) t[r] += a * rr[r * G];
                }
#pragma unroll
                for (int r = 0; r < 96 / G; ++r)
                    if (r * G < NP) s.tw[gp * NP + gl + r * G] = t[r];
            }
            __syncthreads();
            {   // n = t . phi, grad n = 2 t . grad phi  (G lanes per point, shuffle tree)
                W n = 0, gx = 0, gy = 0, gz = 0;
                for (int mu = gl; mu < N; mu += G) {
                    const W tv = s.tw[gp * NP + mu];
                    n += tv * s.phi[gp * NP + mu];
                    gx += tv * s.phi[plane + gp * NP + mu];
                    gy += tv * s.phi[2 * plane + gp * NP + mu];
                    gz += tv * s.phi[3 * plane + gp * NP + mu];
                }
#pragma unroll
                for (int o = 1; o < G; o <<= 1) {
                    n += __shfl_xor_sync(0xffffffffu, n, o);
                    gx += __shfl_xor_sync(0xffffffffu, gx, o);
                    gy += __shfl_xor_sync(0xffffffffu, gy, o);
                    gz += __shfl_xor_sync(0xffffffffu, gz, o);
                }
                if (gl == 0 && gp < nb) {
                    double *d = s.dn + 4 * (sub + gp);
                    d[0] = (double)n;
                    d[1] = (double)(W)(2 * gx);
                    d[2] = (double)(W)(2 * gy);
                    d[3] = (double)(W)(2 * gz);
                }
            }
            __syncthreads();
        }
        // ---- pass B: functional, one thread per point
        if (tid < nsb) {
            double *d = s.dn + 4 * tid;
            const double n = d[0], gx = d[1], gy = d[2], gz = d[3];
            const double sig = (double)(W)((W)gx * (W)gx + (W)gy * (W)gy + (W)gz * (W)gz);
            const XCOut o = b3lyp_point(n, sig);
            if (!(isfinite(o.exc) && isfinite(o.vrho) && isfinite(o.vsigma))) bad = 1;
            const double w = s.pt[4 * tid + 3];
            e_acc += w * n * (double)(W)o.exc;
            const double ww = (double)(W)w;
            const double a = (double)(W)(0.5 * ww * (double)(W)o.vrho);
            const double bb = (double)(W)(2.0 * ww * (double)(W)o.vsigma);
            d[0] = a;
            d[1] = bb * gx;
            d[2] = bb * gy;
            d[3] = bb * gz;
        }
        __syncthreads();
        // ---- pass C: V += phi^T (a phi + b . grad phi)
        for (int sub = 0; sub < nsb; sub += BP) {
            const int nb = min(BP, nsb - sub);
            xc_eval_phi(s, nsh, NP, BP, sub, nb);
            __syncthreads();
            for (int t = tid; t < BP * NP; t += XC_THREADS) {
                const int p = t / NP;
                const double *d = s.dn + 4 * (sub + p);
                W v = (W)0;
                if (p < nb)
                    v = (W)d[0] * s.phi[t] + (W)d[1] * s.phi[plane + t] + (W)d[2] * s.phi[2 * plane + t] +
                        (W)d[3] * s.phi[3 * plane + t];
                s.tw[t] = v;
            }
            __syncthreads();
            for (int p = 0; p < nb; ++p) {
                const W *ph = s.phi + p * NP + ty;
                const W *wv = s.tw + p * NP + tx;
                W fa[6], fb[6];
#pragma unroll
                for (int a = 0; a < 6; ++a) {
                    fa[a] = a < nblk16 ? ph[16 * a] : (W)0;
                    fb[a] = a < nblk16 ? wv[16 * a] : (W)0;
                }
#pragma unroll
                for (int a = 0; a < 6; ++a)
#pragma unroll
                    for (int c = 0; c < 6; ++c) acc[a][c] += fa[a] * fb[c];
            }
            __syncthreads();
        }
    }
    double *Vp = b.Vpart + b.m_V0[m] + (int64_t)(cta - b.m_xccta0[m]) * N * N;
#pragma unroll
    for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            const int mu = ty + 16 * a, nu = tx + 16 * c;
            if (mu < N && nu < N) Vp[mu * N + nu] = (double)acc[a][c];
        }
    const double e = block_sum(e_acc, s.red);
    if (tid == 0) b.Epart[cta] = e;
    if (bad) atomicOr(b.status + m, DFTB_ST_XC_NONFINITE);
}

template <typename W>
static size_t xc_smem(int NP, int BP, int nsh_max) {
    size_t w = (size_t)NP * NP + 5 * (size_t)BP * NP + 2;
    return sizeof(W) * w + 16 + sizeof(double) * (8 * XC_SB + XC_SHD * (size_t)nsh_max + 32);
}

template <typename W>
static void launch_xc_t(const DevBatch &b, int nmax, int nsh_max, cudaStream_t s) {
    const int NP = (nmax + 15) & ~15;
    size_t sm = xc_smem<W>(NP, 32, nsh_max);
    if (sm <= 227 * 1024) {
        cudaFuncSetAttribute(k_xc<W, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_xc<W, 32><<<b.n_xc_cta, XC_THREADS, sm, s>>>(b);
    } else {
        sm = xc_smem<W>(NP, 16, nsh_max);
        cudaFuncSetAttribute(k_xc<W, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_xc<W, 16><<<b.n_xc_cta, XC_THREADS, sm, s>>>(b);
    }
}

void launch_xc(const DevBatch &b, int nmax, int nsh_max, cudaStream_t s) {
    if (b.n_xc_cta == 0) return;
    if (b.prec == 0) launch_xc_t<double>(b, nmax, nsh_max, s);
    else launch_xc_t<float>(b, nmax, nsh_max, s);
}

}  // namespace dftb
