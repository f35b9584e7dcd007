// Throughput probe: legacy mma.sync TF32 m16n8k8 vs FFMA on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_mma(float *out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
    float c[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma(float *out, int iters) {
    float c[16]; for (int j = 0; j < 16; ++j) c[j] = threadIdx.x + j;
    float a = 1.0001f, b = 0.9999f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) c[j] = fmaf(c[j], a, b);
    }
    float s = 0; for (int j = 0; j < 16; ++j) s += c[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float *o; cudaMalloc(&o, 148 * 8 * 256 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int blocks = 148 * 4, thr = 256, it = 4096; float ms;
    k_mma<<<blocks, thr>>>(o, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_mma<<<blocks, thr>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 8 * 8.0 * it * blocks * thr / 32;
    printf("mma.sync tf32 m16n8k8: %.1f TFLOP/s\n", fl / ms / 1e9);
    k_ffma<<<blocks, thr>>>(o, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_ffma<<<blocks, thr>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * it * (double)blocks * thr;
    printf("ffma: %.1f TFLOP/s\n", fl / ms / 1e9);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
