// DMMA (mma.sync m8n8k4 f64) throughput / latency probe on sm_100a vs DFMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/dmma_probe tools/probe/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_dmma(double *out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double d[CH][2];
#pragma unroll
    for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void k_dfma(double *out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double d[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) d[c] = fma(a, b, d[c]);
    double s = 0;
    for (int c = 0; c < 8; ++c) s += d[c];
    if (s == 12345.0) out[0] = s;
}

int main() {
    double *o;
    cudaMalloc(&o, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    float ms;
    // throughput: many warps, 4 independent chains
    for (int w : {1, 2, 4, 8, 16}) {
        k_dmma<4><<<148, 32 * w>>>(o, 100);
        cudaEventRecord(e0);
        k_dmma<4><<<148, 32 * w>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 256 * 4 * (double)iters * 148 * 32 * w / 32;   // per warp: 4 MMAs of 8x8x4
        printf("DMMA  warps/SM %2d  4 chains: %.2f TFLOP/s\n", w, flops / ms / 1e9);
    }
    // latency: one warp, one chain
    k_dmma<1><<<1, 32>>>(o, 100);
    cudaEventRecord(e0);
    k_dmma<1><<<1, 32>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DMMA dependent-chain latency: %.1f ns per MMA\n", ms * 1e6 / iters);
    for (int w : {4, 8, 16}) {
        k_dfma<<<148, 32 * w>>>(o, 100);
        cudaEventRecord(e0);
        k_dfma<<<148, 32 * w>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 8 * (double)iters * 148 * 32 * w;
        printf("DFMA  warps/SM %2d  8 chains: %.2f TFLOP/s\n", w, flops / ms / 1e9);
    }
    return 0;
}
