// J/K digestion over the dense 8-fold ERI store — deterministic, no atomics.
//
// Reference: deskdft.integrals.build_jk (integrals.py:199-218) -> _jk_kernel
// (_kernels.py:650-693), which scatters each canonical entry to its <= 8 images.
//
// B200 formulation ("row owner"): a CTA owns the store rows P = (i, j), j <= i,
// for one or two values of i.  Row P holds (ij|kl) for all Q = (k, l) <= P.  For a
// stored element, the 8 images contribute J_P += v rho~_Q, J_Q += v rho~_P and,
// recording each K contribution at (a,d) or its transpose, G[i][.] and G[j][.]
// updates only (K = -(G + G^T)/4 at the end).  So per row the CTA expands the row
// into a symmetric N x N smem tile T and computes two GEMVs (T rho_j, T rho_i) plus
// one dot product; G rows for the owned i accumulate in registers, the j rows
// and the scattered J entries are written as partials and summed in a fixed order
// by the SCF post kernel.  The store is streamed exactly once per iteration.
#include "common.cuh"

namespace dftb {

template <typename ST>
__global__ void __launch_bounds__(128) k_jk(DevBatch b) {
    extern __shared__ double sm[];
    const int cta = blockIdx.x;
    const int m = b.jk_mol[cta];
    if (b.done[m]) return;
    const int N = b.m_nao[m];
    const int64_t npp = tri(N);
    double *rho = sm;                 // N*N
    double *Tm = rho + N * N;         // N*N
    double *Jsc = Tm + N * N;         // npp
    double *red = Jsc + npp;          // 32
    int *lut = (int *)(red + 32);     // npp  (k << 8 | l)
    const int tid = threadIdx.x, nt = blockDim.x;
    const double *rg = b.rho + b.m_mat0[m];
    for (int t = tid; t < N * N; t += nt) rho[t] = rg[t];
    for (int t = tid; t < npp; t += nt) Jsc[t] = 0.0;
    for (int k = tid; k < N; k += nt)
        for (int l = 0; l <= k; ++l) lut[tri(k) + l] = (k << 8) | l;
    __syncthreads();
    const ST *eri = (const ST *)b.eri + b.m_eri0[m];
    double *Gp = b.Gpart + b.m_G0[m];
    double *Jp = b.Jpart + b.m_Jp0[m];
    const int local = cta - b.m_jkcta0[m];
    const int iv[2] = {b.jk_i0[cta], b.jk_i1[cta]};
    for (int s = 0; s < 2; ++s) {
        const int i = iv[s];
        if (i < 0) continue;
        double gi = 0.0;
        for (int j = 0; j <= i; ++j) {
            const int64_t P = tri(i) + j;
            const ST *row = eri + tri(P);
            const double rt = rho[i * N + j] * (i != j ? 2.0 : 1.0);
            double jown = 0.0;
            for (int64_t e = tid; e <= P; e += nt) {
                const double v = (double)row[e];
                const int kl = lut[e], k = kl >> 8, l = kl & 255;
                const double c = e == P ? v : 2.0 * v;
                Tm[k * N + l] = c;
                Tm[l * N + k] = c;
                jown += v * rho[k * N + l] * (k != l ? 2.0 : 1.0);
                if (e < P) Jsc[e] += v * rt;
            }
            for (int l = j + 1 + tid; l <= i; l += nt) {
                Tm[i * N + l] = 0.0;
                Tm[l * N + i] = 0.0;
            }
            jown = block_sum(jown, red);  // also orders the Tm writes before the reads below
            if (tid == 0) Jp[P] = jown;
            if (tid <= i) {
                double a = 0.0, c2 = 0.0;
                const double *rj = rho + j * N, *ri = rho + i * N;
                for (int n = 0; n <= i; ++n) {
                    const double tv = Tm[n * N + tid];
                    a += tv * rj[n];
                    c2 += tv * ri[n];
                }
                gi += a;
                if (j < i) Gp[P * N + tid] = c2;
            }
            __syncthreads();
        }
        if (tid <= i) Gp[(tri(i) + i) * N + tid] = gi;
    }
    double *Js = Jp + (int64_t)(1 + local) * npp;
    for (int64_t t = tid; t < npp; t += nt) Js[t] = Jsc[t];
}

size_t jk_smem_bytes(int nmax) {
    const size_t npp = (size_t)nmax * (nmax + 1) / 2;
    return sizeof(double) * (2 * (size_t)nmax * nmax + npp + 32) + sizeof(int) * npp;
}

void launch_jk(const DevBatch &b, int nmax, cudaStream_t s) {
    const size_t sm = jk_smem_bytes(nmax);
    if (b.prec == 0) {
        cudaFuncSetAttribute(k_jk<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_jk<double><<<b.n_jk_cta, 128, sm, s>>>(b);
    } else {
        cudaFuncSetAttribute(k_jk<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_jk<float><<<b.n_jk_cta, 128, sm, s>>>(b);
    }
}

}  // namespace dftb
