// Internal device-side definitions of the B200 PagedEviction engine.
//
// HBM layout:
//   pages        [capacity][2 (K,V)][B][row_pitch]   row_pitch = round_up(w*elt, 16)
//   positions    [capacity][B] int32
//   token_scores [capacity][B] double   (cached S of every written slot)
//   page_scores  [capacity] double      (mean S of a full page, set when it fills)
//   block_table  [n_tables][max_pages] int32, num_pages/newest_fill/retained [n_tables]
//   stack        [capacity] int32 + top   (LIFO free list, page_pool.cpp:18-38)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pe.h"

namespace pe {

constexpr int kWarp = 32;
constexpr double kNormEps = 1e-12;               // kNormEpsilon, importance.hpp:17

struct DevState {
    uint8_t* pages;
    int32_t* positions;
    double* token_scores;
    double* page_scores;
    int32_t* block_table;
    int32_t* num_pages;
    int32_t* newest_fill;
    int32_t* retained;
    int32_t* stack;
    int32_t* top;
    int32_t* status;
    unsigned long long* evict_count;
    unsigned long long* grid_ctr;   // monotonically increasing CTA completion tickets
    // Unstructured (per-token) eviction, table API only: bit s of holes[p]
    // marks an evicted slot of page p (Page::evict, page.hpp:47-56); cleared
    // when the page is released. holes_on = 0 until the first hole is made,
    // so the PagedEviction kernels never read the array before that.
    unsigned long long* holes;      // [capacity]
    int32_t holes_on;
    int32_t capacity, B, C, w, pitch, row_bytes, max_pages, n_tables;
    int32_t n_seqs, n_layers, tab_heads, dtype, policy;
};

// Occupied-slot count of a page whose first `cursor` slots were written.
__device__ __forceinline__ int page_fill(const DevState& s, int page, int cursor) {
    if (!s.holes_on) return cursor;
    const unsigned long long m = cursor >= 64 ? ~0ull : ((1ull << cursor) - 1ull);
    return cursor - __popcll(s.holes[page] & m);
}
__device__ __forceinline__ bool slot_hole(const DevState& s, int page, int slot) {
    return s.holes_on && slot < 64 && ((s.holes[page] >> slot) & 1ull);
}

// Per-launch control block written by the plan kernels.
struct LaunchCtl {
    int32_t abort;      // 1: the launch is a no-op (status set)
    int32_t pop_base;   // stack top before this launch's pops
    int32_t push_base;  // stack top before this launch's pushes
    int32_t count;      // number of flagged tables (evict work items)
    int32_t ready;      // unused (kept for layout)
    int32_t pad_;
    unsigned long long top_word;  // append look-back: epoch << 32 | stack top before the launch's pops
    // pop_flag[E & 1] = E: some table pops (or may pop) at append launch E.
    // Written by launch E-1 into the slot launch E reads and never into the
    // slot it reads itself (epochs alternate parity: period 0x3FFFFFFE), so a
    // CTA that starts after another CTA of its own launch has finished still
    // sees the previous launch's verdict.
    unsigned int pop_flag[2];
};

// Launch table set: decode launches cover every sequence for layers
// [layer_begin, layer_begin+n_layers); index i enumerates (seq, layer, head)
// seq-major, which is ascending table id. The table-granular API (pe_table_*,
// one reference BlockTable per call entry) instead passes an explicit
// ascending id list `ids` (device) whose entry i reads input row i.
struct TableSet {
    int32_t layer_begin, n_layers;
    const int32_t* ids = nullptr;
    int32_t n_ids = 0;
    __host__ __device__ int32_t size(const DevState& s) const {
        return ids ? n_ids : s.n_seqs * n_layers * s.tab_heads;
    }
    // index into the launch's positions array
    __host__ __device__ int64_t pos_index(const DevState& s, int32_t i) const {
        return ids ? i : input_row(s, i) / s.tab_heads % s.n_seqs;
    }
    __host__ __device__ int32_t table(const DevState& s, int32_t i) const {
        if (ids) return ids[i];
        const int32_t h = i % s.tab_heads;
        const int32_t rest = i / s.tab_heads;
        const int32_t li = rest % n_layers;
        const int32_t seq = rest / n_layers;
        return (seq * s.n_layers + layer_begin + li) * s.tab_heads + h;
    }
    // row index of launch table i in an input laid out [n_layers][n_seqs][tab_heads]
    __host__ __device__ int64_t input_row(const DevState& s, int32_t i) const {
        if (ids) return i;
        const int32_t h = i % s.tab_heads;
        const int32_t rest = i / s.tab_heads;
        const int32_t li = rest % n_layers;
        const int32_t seq = rest / n_layers;
        return ((int64_t)li * s.n_seqs + seq) * s.tab_heads + h;
    }
};

__device__ __forceinline__ void set_status(int32_t* status, int32_t code) {
    atomicCAS(status, 0, code);
}

// ------------------------------------------------------------------ async copy
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ uint4 ld_shared_v4(const void* p) {
    uint4 r;
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(s));
    return r;
}

// 2^768 as a double (exponent field 1791): undoes the 2^-768 scaling of the
// certified bf16 sums of squares (pe_score.cuh).
__device__ __forceinline__ double two_pow_768() { return __hiloint2double(0x6FF00000, 0); }

// S = ||V|| / max(||K||, eps) from the two sums of squares (importance.cpp:11-13).
__device__ __forceinline__ double token_score_from_sumsq(double k2, double v2) {
    const double kn = sqrt(k2);
    const double vn = sqrt(v2);
    return vn / fmax(kn, kNormEps);
}

// The same score computed by a lane pair holding the same (k2, v2): lane q
// takes one square root (q = 0: K, q = 1: V) and the pair exchanges them, so
// each lane runs one IEEE double sqrt instead of two (bit-identical result).
// Every lane of the warp must call it.
__device__ __forceinline__ double pair_score_from_sumsq(double k2, double v2) {
    const int q = threadIdx.x & 1;
    const double r = sqrt(q ? v2 : k2);
    const double o = __shfl_xor_sync(0xFFFFFFFFu, r, 1);
    return (q ? r : o) / fmax(q ? o : r, kNormEps);
}

// ------------------------------------------------------------------ warp/cta scans
__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Block-wide exclusive scan of one int per thread. `sm` needs 33 ints.
// Returns the exclusive prefix; *total receives the block total.
__device__ __forceinline__ int block_excl_scan(int v, int* sm, int* total) {
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    const int incl = warp_incl_scan(v);
    if (lane == 31) sm[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int x = lane < nw ? sm[lane] : 0;
        const int xi = warp_incl_scan(x);
        if (lane < nw) sm[lane] = xi - x;
        if (lane == 31) sm[32] = xi;
    }
    __syncthreads();
    const int r = sm[wid] + incl - v;
    *total = sm[32];
    __syncthreads();
    return r;
}

// Launch-level completion: every TABLE of the launch takes one ticket when it
// is settled (a non-triggered table at once, a triggered one after its
// finalize); whoever takes the launch's last ticket pushes the launch's
// released pages on the free stack in ascending table id (release,
// page_pool.cpp:35-38; canonical order DESIGN.md §1.6). `settled` is
// block-uniform.
// by_table (K2 recompute): vpage is indexed by table id, launch table i's
// entry is vpage[by_table->table(s, i)].
__device__ __forceinline__ void push_victims_if_last(const DevState& s, int n, int32_t* vpage,
                                                     unsigned long long grid_last, int settled,
                                                     const TableSet* by_table = nullptr) {
    __shared__ int is_last;
    __shared__ int scan_sm[33];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = settled > 0 && (atomicAdd(s.grid_ctr, (unsigned long long)settled) + settled - 1 >= grid_last);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    // tiles of 16 consecutive entries per thread: independent loads, one
    // block scan per tile (ascending table id = canonical push order)
    const int top = *s.top;
    int base = 0;
    for (int t0 = 0; t0 < n; t0 += blockDim.x * 16) {
        const int i0 = t0 + threadIdx.x * 16;
        int v[16];
        int cnt = 0;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            v[u] = (i0 + u < n) ? __ldcg(vpage + (by_table ? by_table->table(s, i0 + u) : i0 + u)) : -1;
            cnt += v[u] >= 0;
        }
        int total;
        int k = base + block_excl_scan(cnt, scan_sm, &total);
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (v[u] >= 0) s.stack[top + k++] = v[u];
        base += total;
    }
    __syncthreads();
    if (threadIdx.x == 0) *s.top = top + base;
}

// Programmatic dependent launch (PDL). A kernel launched with programmatic
// stream serialization may become resident while the previous kernel of the
// stream still runs; griddepcontrol.wait blocks until that kernel has
// completed and its memory is visible (a no-op for a normal launch), and
// griddepcontrol.launch_dependents lets the next PDL launch become resident.
// Kernels that start with pdl_top() behave exactly like normally ordered
// launches; PDL only hides the launch gap between them.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_top() {
    pdl_wait();
    pdl_launch_dependents();
}

}  // namespace pe
