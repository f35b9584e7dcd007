// Small operator-level kernels behind the C ABI: AO values on the grid
// (xc.eval_ao, xc.py:165-194), pointwise B3LYP (xc.b3lyp, xc.py:277-306), the
// reference-semantics compaction of the dense ERI store into eri_packed's
// canonical list (integrals.py:147-191), and an FMA-throughput probe used to
// state the FP64/FP32 roofline denominators.
#include "common.cuh"
#include "b3lyp.cuh"

namespace dftb {

__global__ void k_eval_ao(DevBatch b, int mol, double *out) {
    const int64_t g0 = b.m_grid0[mol], npts = b.m_grid0[mol + 1] - g0;
    const int N = b.m_nao[mol], nsh = b.m_nshell[mol], s0 = b.m_shell0[mol];
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= npts * nsh) return;
    const int64_t p = t % npts;
    const int sh = s0 + (int)(t / npts);
    const double *A = b.a_xyz + 3 * b.s_atom[sh];
    const double *q = b.g_xyz + 3 * (g0 + p);
    const double rel[3] = {q[0] - A[0], q[1] - A[1], q[2] - A[2]};
    const double r2 = rel[0] * rel[0] + rel[1] * rel[1] + rel[2] * rel[2];
    double bs = 0, ds = 0, bp = 0, dp = 0;
    for (int k = 0; k < 3; ++k) {
        const double a = b.s_exp[3 * sh + k], e = exp(-a * r2);
        bs += b.s_cs[3 * sh + k] * e;
        ds += b.s_cs[3 * sh + k] * (-2.0 * a) * e;
        bp += b.s_cp[3 * sh + k] * e;
        dp += b.s_cp[3 * sh + k] * (-2.0 * a) * e;
    }
    const int ao = b.s_ao[sh];
    const int64_t plane = npts * N;
    double *o = out + p * N + ao;
    o[0] = bs;
    for (int d = 0; d < 3; ++d) o[(d + 1) * plane] = rel[d] * ds;
    if (b.s_kind[sh]) {
        for (int c = 0; c < 3; ++c) {
            o[1 + c] = rel[c] * bp;
            for (int d = 0; d < 3; ++d) o[(d + 1) * plane + 1 + c] = (c == d ? bp : 0.0) + rel[c] * rel[d] * dp;
        }
    }
}

void launch_eval_ao(const DevBatch &b, int mol, double *out, cudaStream_t s) {
    int64_t npts = 0;
    int nsh = 0;
    cudaMemcpy(&npts, b.m_grid0 + mol + 1, sizeof(int64_t), cudaMemcpyDeviceToHost);
    int64_t g0 = 0;
    cudaMemcpy(&g0, b.m_grid0 + mol, sizeof(int64_t), cudaMemcpyDeviceToHost);
    cudaMemcpy(&nsh, b.m_nshell + mol, sizeof(int), cudaMemcpyDeviceToHost);
    npts -= g0;
    const int64_t n = npts * nsh;
    if (n > 0) k_eval_ao<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(b, mol, out);
}

__global__ void k_b3lyp(const double *n, const double *sg, int64_t np, double *e, double *vr, double *vs) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    const XCOut o = b3lyp_point(n[i], sg[i]);
    e[i] = o.exc;
    vr[i] = o.vrho;
    vs[i] = o.vsigma;
}

void launch_b3lyp(const double *n, const double *sg, int64_t np, double *e, double *vr, double *vs, cudaStream_t s) {
    k_b3lyp<<<(unsigned)((np + 255) / 256), 256, 0, s>>>(n, sg, np, e, vr, vs);
}

// ---------------------------------------------------------------- eri_packed compaction
__device__ __forceinline__ bool keep_entry(double v, int64_t P, int64_t Q, double eps, const double *qsp,
                                           const double *qao) {
    if (eps <= 0.0) return true;
    if (qsp[P] * qsp[Q] < eps) return false;      // shell-quartet screen (split-shell pairs)
    if (qao[P] * qao[Q] < eps) return false;      // AO-level screen
    return fabs(v) >= eps;                        // value screen
}

template <typename ST>
__global__ void k_compact(DevBatch b, int mol, double eps, const double *qsp, int64_t *rowcnt,
                          const int64_t *rowoff, uint16_t *oi, uint16_t *oj, uint16_t *ok, uint16_t *ol,
                          double *ov) {
    __shared__ int64_t scan[128];
    const int64_t P = blockIdx.x;
    int i = (int)((sqrt(8.0 * (double)P + 1.0) - 1.0) * 0.5);
    while (tri(i + 1) <= P) ++i;
    while (tri(i) > P) --i;
    const int j = (int)(P - tri(i));
    const ST *row = (const ST *)b.eri + b.m_eri0[mol] + eri_row(i, j);
    const double *qao = b.qao + b.m_npp0[mol];
    const int64_t len = P + 1, per = (len + 127) / 128;
    const int64_t lo = threadIdx.x * per, hi = min(len, lo + per);
    auto ket = [&](int64_t q, int &k) {
        k = (int)((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
        while (tri(k + 1) <= q) ++k;
        while (tri(k) > q) --k;
        return (double)row[eri_ket(k, (int)(q - tri(k)))];
    };
    int64_t c = 0;
    for (int64_t q = lo; q < hi; ++q) {
        int k;
        c += keep_entry(ket(q, k), P, q, eps, qsp, qao);
    }
    scan[threadIdx.x] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t s = 0;
        for (int k = 0; k < 128; ++k) { const int64_t t = scan[k]; scan[k] = s; s += t; }
        if (rowcnt) rowcnt[P] = s;
    }
    __syncthreads();
    if (!rowoff) return;
    int64_t pos = rowoff[P] + scan[threadIdx.x];
    for (int64_t q = lo; q < hi; ++q) {
        int k;
        const double v = ket(q, k);
        if (!keep_entry(v, P, q, eps, qsp, qao)) continue;
        oi[pos] = (uint16_t)i; oj[pos] = (uint16_t)j;
        ok[pos] = (uint16_t)k; ol[pos] = (uint16_t)(q - tri(k));
        ov[pos] = v;
        ++pos;
    }
}

static int mol_npp(const DevBatch &b, int mol) {
    int N = 0;
    cudaMemcpy(&N, b.m_nao + mol, sizeof(int), cudaMemcpyDeviceToHost);
    return N * (N + 1) / 2;
}

void launch_compact_count(const DevBatch &b, int mol, double eps, const double *qsp, int64_t *rowcnt, cudaStream_t s) {
    const int npp = mol_npp(b, mol);
    if (b.eri64) k_compact<double><<<npp, 128, 0, s>>>(b, mol, eps, qsp, rowcnt, nullptr, 0, 0, 0, 0, 0);
    else k_compact<float><<<npp, 128, 0, s>>>(b, mol, eps, qsp, rowcnt, nullptr, 0, 0, 0, 0, 0);
}

void launch_compact_write(const DevBatch &b, int mol, double eps, const double *qsp, const int64_t *rowoff,
                          uint16_t *oi, uint16_t *oj, uint16_t *ok, uint16_t *ol, double *ov, cudaStream_t s) {
    const int npp = mol_npp(b, mol);
    if (b.eri64) k_compact<double><<<npp, 128, 0, s>>>(b, mol, eps, qsp, nullptr, rowoff, oi, oj, ok, ol, ov);
    else k_compact<float><<<npp, 128, 0, s>>>(b, mol, eps, qsp, nullptr, rowoff, oi, oj, ok, ol, ov);
}

// ---------------------------------------------------------------- FMA throughput probe
template <typename T>
__global__ void __launch_bounds__(256) k_fma(T *out, int iters, T seed) {
    T a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed + (T)(threadIdx.x + k);
    const T m = (T)0.999999, c = (T)1e-7;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
    T s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == (T)-1) out[0] = s;  // never true; keeps the chains live
}

double fma_peak(int fp64, cudaStream_t st) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    void *out = nullptr;
    cudaMalloc(&out, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0, st);
        if (fp64) k_fma<double><<<blocks, threads, 0, st>>>((double *)out, iters, 1.0);
        else k_fma<float><<<blocks, threads, 0, st>>>((float *)out, iters, 1.0f);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
        if (rep > 0) best = fmax(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return best;
}

}  // namespace dftb
