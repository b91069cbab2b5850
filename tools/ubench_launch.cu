// Micro-benchmark (tools only): per-launch time of back-to-back dependent
// launches of a 256-CTA x 128-thread kernel whose threads do D dependent
// global loads (a pointer chase through DRAM-resident data), with and
// without programmatic dependent launch (every kernel waits at its top) —
// the floor for a latency-bound kernel like K0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_launch tools/ubench_launch.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void chase(const uint32_t* __restrict__ next, uint32_t* out, int depth, uint32_t seed) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    uint32_t i = (seed + blockIdx.x * 131u + threadIdx.x * 7919u) & ((1u << 26) - 1);
    for (int d = 0; d < depth; ++d) i = __ldcg(next + i);
    if (i == 0xFFFFFFFFu) out[0] = i;
}

int main() {
    const size_t n = 1u << 26;  // 256 MB of indices (> L2)
    uint32_t *next, *out;
    cudaMalloc(&next, n * 4);
    cudaMalloc(&out, 4);
    uint32_t* h = new uint32_t[n];
    uint64_t x = 88172645463325252ull;
    for (size_t k = 0; k < n; ++k) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        h[k] = (uint32_t)(x & (n - 1));
    }
    cudaMemcpy(next, h, n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int pdl = 0; pdl < 2; ++pdl) {
        for (int depth : {0, 1, 3, 5, 8}) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(256);
            cfg.blockDim = dim3(128);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = pdl;
            for (int w = 0; w < 32; ++w) cudaLaunchKernelEx(&cfg, chase, (const uint32_t*)next, out, depth, (uint32_t)w);
            cudaEventRecord(a);
            const int reps = 64;
            for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, chase, (const uint32_t*)next, out, depth, (uint32_t)r * 977u);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("pdl %d depth %d: %.2f us per launch\n", pdl, depth, ms * 1000 / reps);
        }
    }
    return 0;
}
