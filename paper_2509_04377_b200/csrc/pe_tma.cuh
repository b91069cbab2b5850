// Tensor-memory-accelerator staging helpers shared by the TMA kernels (K2, K3):
// mbarrier setup / wait and the 2-D tensor-map page load over the engine's
// pool tensor map (pages as [capacity * 2B rows][d] bf16, boxes of 64 columns
// x 32 rows, SWIZZLE_128B: 16-byte chunk c of box row r lives at c ^ (r & 7)).
#pragma once

#include <cuda.h>
#include <cstdint>

namespace pe {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Address of 16-byte chunk `chunk` (0..7) of row r in a 128-byte-wide
// SWIZZLE_128B box starting at half_base (1024-byte aligned).
__device__ __forceinline__ uint32_t sw128(uint32_t half_base, int r, int chunk) {
    return half_base + r * 128 + ((chunk ^ (r & 7)) << 4);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// One lane: order this thread's earlier generic-proxy reads of the stage
// before the async-proxy writes, arm the barrier for `bytes`, and load the
// `halves` 64-column boxes of box row `y` (page id * 32), starting at column
// `x0` (a PER_LAYER head's slice), into dst.
__device__ __forceinline__ void tma_load_page(uint32_t dst, uint64_t* bar, const CUtensorMap* tmap, int y, int x0,
                                              int halves, uint32_t bytes) {
    const uint32_t b = smem_u32(bar);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    for (int hf = 0; hf < halves; ++hf)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                dst + hf * 4096),
            "l"(tmap), "r"(x0 + hf * 64), "r"(y), "r"(b)
            : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t b = smem_u32(bar);
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
            : "=r"(done)
            : "r"(b), "r"(parity)
            : "memory");
}

// Rounds the dynamic shared memory base up to 1024 bytes (SWIZZLE_128B
// destinations); launches add 1 KB of slack.
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

}  // namespace pe
