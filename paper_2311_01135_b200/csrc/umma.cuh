// tcgen05 (UMMA) helpers for the TF32 tensor-core contractions (sm_100a).
//
// Operands live in shared memory in the K-major SWIZZLE_128B canonical layout: a matrix
// with `rows` (the M or N index) and K columns is tiled into 1024-byte atoms of 8 rows x
// 128 bytes (32 f32); atom (row / 8, col / 32) sits at ((row / 8) * nseg + col / 32) KB,
// nseg = ceil(K / 32), and inside an atom the 16-byte chunk of a row is XOR-swizzled by
// (row % 8).  The descriptor's stride byte offset is the 8-row-group stride (nseg KB); one
// MMA consumes K = 8 (32 bytes) and the k-th step starts (k / 4) KB + (k % 4) * 32 bytes
// into the row.  (Measured on B200 with tools/probe/umma_probe.cu: TF32 operands that are
// MN-major need the SWIZZLE_128B_BASE32B layout instead, so every operand here is K-major.)
//
// Accumulators are f32 in tensor memory.  M = 64: row m is TMEM lane (m % 16) + 32 (m / 16);
// M = 128: row m is lane m.  Column n of the tile is TMEM column base + n.
#pragma once
#include <stdint.h>

namespace dftb {
namespace umma {

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// element offset (in 4-byte words) of (row, col) in a K-major SWIZZLE_128B buffer
__device__ __forceinline__ int sw128(int row, int col, int nseg) {
    return (((row >> 3) * nseg + (col >> 5)) << 8) + ((row & 7) << 5) + ((((col & 31) >> 2) ^ (row & 7)) << 2) +
           (col & 3);
}

__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// k-th K step (8 tf32) of a K-major SW128 operand starting at `base`
__device__ __forceinline__ uint64_t desc_k(uint32_t base, int k, uint32_t sbo) {
    return desc_sw128(base + (uint32_t)((k >> 2) << 10) + (uint32_t)((k & 3) << 5), sbo);
}

// descriptor of the k-th K step given the step-0 descriptor (start address field += offset / 16)
__device__ __forceinline__ uint64_t desc_step(uint64_t d0, int k) {
    return d0 + (uint64_t)(((k >> 2) << 6) | ((k & 3) << 1));
}

// instruction descriptor: kind::tf32, f32 accumulate, both operands K-major
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// arrive on `bar` once every previously issued tcgen05.mma of this thread has completed
__device__ __forceinline__ void commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nUW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra UW_%=;\n}" ::"r"(
            saddr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// warp-collective TMEM allocation of `ncols` (power of two >= 32) columns; address -> *dst
__device__ __forceinline__ void tmem_alloc(uint32_t *dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(dst)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free(uint32_t addr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(addr), "r"(ncols) : "memory");
}

// 32 lanes x 16 / 4 consecutive 32-bit columns (warp-collective; lane i <- TMEM lane quarter + i)
__device__ __forceinline__ void tld16(uint32_t addr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tld4(uint32_t addr, float (&v)[4]) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 3xTF32 split: x = hi + lo with hi exactly representable in TF32 (round to nearest)
__device__ __forceinline__ float tf32_hi(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

}  // namespace umma
}  // namespace dftb
