// Table-granular kernels behind the per-object reference API (pe_table_*,
// pe_pool_*; used by the C++ façade include/pe/pagedevict.hpp). These are
// the reference's single-table operations that have no batched hot-path
// counterpart; appends and PagedEviction decisions of the façade run through
// the hot kernels K0/K2 with an explicit table list (pe_decode.cu).
//
//   pool_allocate_kernel   PagePool::allocate        page_pool.cpp:24-33
//   pool_release_kernel    PagePool::release         page_pool.cpp:35-38
//   table_free_page_kernel BlockTable::free_page     block_table.cpp:21-31
//   table_clear_kernel     BlockTable::clear         block_table.cpp:72-78
//   table_attend_kernel    attend / attend_detailed  attention.cpp:15-99
#include "pe_kernels.cuh"

namespace pe {

__global__ void pool_allocate_kernel(DevState s, int32_t* out) {
    const int top = *s.top;
    if (top <= 0) {
        set_status(s.status, PE_POOL_EXHAUSTED);
        *out = -1;
        return;
    }
    const int id = s.stack[top - 1];
    *s.top = top - 1;
    *out = id;
}

__global__ void pool_release_kernel(DevState s, int32_t id) {
    const int top = *s.top;
    if (top >= s.capacity) {  // more releases than pages: the reference would grow its list
        set_status(s.status, PE_INVALID_STATE);
        return;
    }
    s.stack[top] = id;
    *s.top = top + 1;
}

// One warp. Every non-newest page is full (the engine never leaves holes),
// so the freed page holds B tokens unless it is the newest one.
__global__ void table_free_page_kernel(DevState s, int32_t t, int32_t idx) {
    const int lane = threadIdx.x & 31;
    const int N = s.num_pages[t];
    if (idx < 0 || idx >= N) {
        if (lane == 0) set_status(s.status, PE_INDEX_OUT_OF_RANGE);
        return;
    }
    int32_t* row = s.block_table + (int64_t)t * s.max_pages;
    const int page = row[idx];
    const int fill = (idx == N - 1) ? s.newest_fill[t] : s.B;
    for (int base = idx; base < N - 1; base += 32) {
        const int v = (base + lane + 1 < N) ? row[base + lane + 1] : 0;
        __syncwarp();
        if (base + lane < N - 1) row[base + lane] = v;
        __syncwarp();
    }
    if (lane == 0) {
        row[N - 1] = -1;
        s.num_pages[t] = N - 1;
        s.retained[t] -= fill;
        if (idx == N - 1) s.newest_fill[t] = (N - 1 > 0) ? s.B : 0;
        const int top = *s.top;
        s.stack[top] = page;
        *s.top = top + 1;
    }
}

// Releases every mapped page in logical order (the last one ends on top).
__global__ void table_clear_kernel(DevState s, int32_t t) {
    const int N = s.num_pages[t];
    int32_t* row = s.block_table + (int64_t)t * s.max_pages;
    const int top = *s.top;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        s.stack[top + j] = row[j];
        row[j] = -1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *s.top = top + N;
        s.num_pages[t] = 0;
        s.newest_fill[t] = 0;
        s.retained[t] = 0;
    }
}

__device__ __forceinline__ double row_elem(const uint8_t* row, int i, int dtype) {
    if (dtype == PE_DTYPE_BF16) {
        const uint16_t b = reinterpret_cast<const uint16_t*>(row)[i];
        return static_cast<double>(__uint_as_float(static_cast<uint32_t>(b) << 16));
    }
    return static_cast<double>(reinterpret_cast<const float*>(row)[i]);
}

// attend_impl (attention.cpp:15-99), one CTA per head, bit-for-bit the
// reference's arithmetic: logits are double dots in index order (float x
// float products are exact in double, so fma == mul+add), the softmax sum
// and the value accumulation run over tokens in logical order with separate
// IEEE multiply and add (no contraction: w is a full double). Only exp may
// differ from the host libm in the last ulp. `logits` is scratch [H][R].
__global__ void table_attend_kernel(DevState s, int32_t t, const float* __restrict__ q, int32_t head_dim,
                                    double* logits, float* out, double* weight_sums) {
    const int h = blockIdx.x;
    const int N = s.num_pages[t];
    const int R = s.retained[t];
    const int32_t* row = s.block_table + (int64_t)t * s.max_pages;
    const int64_t page_bytes = (int64_t)2 * s.B * s.pitch;
    const int64_t elt = s.dtype == PE_DTYPE_BF16 ? 2 : 4;
    const float* qh = q + (int64_t)h * head_dim;
    double* lg = logits + (int64_t)h * R;
    const double scale = 1.0 / sqrt(static_cast<double>(head_dim));
    (void)N;
    __shared__ double red[32];
    __shared__ double sh_max, sh_sum;
    // pass 1: logits
    double mx = -INFINITY;
    for (int i = threadIdx.x; i < R; i += blockDim.x) {
        const uint8_t* krow = s.pages + (int64_t)row[i / s.B] * page_bytes + (int64_t)(i % s.B) * s.pitch +
                              (int64_t)h * head_dim * elt;
        double dot = 0.0;
        for (int j = 0; j < head_dim; ++j) dot = fma(static_cast<double>(qh[j]), row_elem(krow, j, s.dtype), dot);
        const double l = __dmul_rn(dot, scale);
        lg[i] = l;
        mx = fmax(mx, l);
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = red[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
        sh_max = m;
    }
    __syncthreads();
    const double m = sh_max;
    for (int i = threadIdx.x; i < R; i += blockDim.x) lg[i] = exp(lg[i] - m);
    __syncthreads();
    if (threadIdx.x == 0) {  // sequential in logical order, as the reference
        double sum = 0.0;
        for (int i = 0; i < R; ++i) sum = __dadd_rn(sum, lg[i]);
        sh_sum = sum;
    }
    __syncthreads();
    const double ws = sh_sum;
    // pass 2: one accumulator per output element, tokens in logical order
    for (int j = threadIdx.x; j < head_dim; j += blockDim.x) {
        double acc = 0.0;
        for (int i = 0; i < R; ++i) {
            const uint8_t* vrow = s.pages + (int64_t)row[i / s.B] * page_bytes +
                                  (int64_t)(s.B + i % s.B) * s.pitch + (int64_t)h * head_dim * elt;
            const double w = __ddiv_rn(lg[i], ws);
            acc = __dadd_rn(acc, __dmul_rn(w, row_elem(vrow, j, s.dtype)));
        }
        out[(int64_t)h * head_dim + j] = static_cast<float>(acc);
    }
    if (weight_sums != nullptr && threadIdx.x == 0) {
        double tot = 0.0;
        for (int i = 0; i < R; ++i) tot = __dadd_rn(tot, __ddiv_rn(lg[i], ws));
        weight_sums[h] = tot;
    }
}

}  // namespace pe
