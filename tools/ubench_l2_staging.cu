// Micro-benchmark (tools only): does a freshly written staging buffer stay
// in L2 while a large stream of reads passes through it, depending on the
// cache-eviction hint of the streaming loads?  Sequence per trial:
//   write_kernel   writes the staging buffer S (stg_mb MB)
//   stream_kernel  reads stream_mb MB of X with hint h
//   read_kernel    reads S back
// Run under ncu (--cache-control none) and compare dram__bytes_read.sum of
// read_kernel across hints: ~0 means S survived in L2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_l2 tools/ubench_l2_staging.cu
//   ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
//       ./ubench_l2 64 134
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void write_kernel(uint4* s, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        s[i] = make_uint4(seed ^ (uint32_t)i, (uint32_t)i, seed, 1u);
}

// 256-bit loads (the .L2::evict_first qualifier requires .v8.b32)
struct u8x32 {
    uint32_t w[8];
};
template <int H>
__device__ __forceinline__ uint32_t ld_hint(const uint4* p) {
    u8x32 r;
    if constexpr (H == 0) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
                       "=r"(r.w[6]), "=r"(r.w[7]) : "l"(p));
    } else if constexpr (H == 1) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
                       "=r"(r.w[6]), "=r"(r.w[7]) : "l"(p));
    } else {
        asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.L2::256B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
                       "=r"(r.w[6]), "=r"(r.w[7]) : "l"(p));
    }
    uint32_t a = 0;
    for (int k = 0; k < 8; ++k) a ^= r.w[k];
    return a;
}

template <int H>
__global__ void stream_kernel(const uint4* x, size_t n, unsigned long long* sink) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; 2 * i < n; i += (size_t)gridDim.x * blockDim.x)
        acc ^= ld_hint<H>(x + 2 * i);
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void read_kernel(const uint4* s, size_t n, unsigned long long* sink) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const uint4 v = s[i];
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main(int argc, char** argv) {
    const size_t stg_mb = argc > 1 ? atoi(argv[1]) : 64;
    const size_t stream_mb = argc > 2 ? atoi(argv[2]) : 134;
    const size_t ns = stg_mb << 16, nx = (size_t)2048 << 16;  // uint4 elements; X = 2 GB
    uint4 *s, *x;
    unsigned long long* sink;
    cudaMalloc(&s, ns * 16);
    cudaMalloc(&x, nx * 16);
    cudaMalloc(&sink, 8);
    cudaMemset(x, 1, nx * 16);
    const size_t nstream = stream_mb << 16;
    size_t off = 0;
    for (int h = 0; h < 3; ++h) {
        for (int rep = 0; rep < 2; ++rep) {
            write_kernel<<<148 * 8, 256>>>(s, ns, 7u * h + rep);
            const uint4* xs = x + off;
            off = (off + nstream) % (nx - nstream);
            if (h == 0) stream_kernel<0><<<148 * 8, 256>>>(xs, nstream, sink);
            else if (h == 1) stream_kernel<1><<<148 * 8, 256>>>(xs, nstream, sink);
            else stream_kernel<2><<<148 * 8, 256>>>(xs, nstream, sink);
            read_kernel<<<148 * 8, 256>>>(s, ns, sink);
        }
    }
    cudaDeviceSynchronize();
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
