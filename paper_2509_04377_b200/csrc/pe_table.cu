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
#include "pe_score.cuh"

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
    s.holes[id] = 0ull;  // Page::reset (page_pool.cpp:31)
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
    s.holes[id] = 0ull;
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
    const int fill = page_fill(s, page, (idx == N - 1) ? s.newest_fill[t] : s.B);
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
        s.holes[page] = 0ull;
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
        s.holes[row[j]] = 0ull;
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
    const int nf = s.newest_fill[t];
    const int X = N * s.B;  // slot index x = logical page * B + slot; holes and unwritten slots skipped
    const int32_t* row = s.block_table + (int64_t)t * s.max_pages;
    const int64_t page_bytes = (int64_t)2 * s.B * s.pitch;
    const int64_t elt = s.dtype == PE_DTYPE_BF16 ? 2 : 4;
    const float* qh = q + (int64_t)h * head_dim;
    double* lg = logits + (int64_t)h * X;
    const double scale = 1.0 / sqrt(static_cast<double>(head_dim));
    auto valid = [&](int x) {
        const int j = x / s.B, sl = x % s.B;
        return sl < (j == N - 1 ? nf : s.B) && !slot_hole(s, row[j], sl);
    };
    __shared__ double red[32];
    __shared__ double sh_max, sh_sum;
    // pass 1: logits
    double mx = -INFINITY;
    for (int x = threadIdx.x; x < X; x += blockDim.x) {
        if (!valid(x)) continue;
        const uint8_t* krow = s.pages + (int64_t)row[x / s.B] * page_bytes + (int64_t)(x % s.B) * s.pitch +
                              (int64_t)h * head_dim * elt;
        double dot = 0.0;
        for (int j = 0; j < head_dim; ++j) dot = fma(static_cast<double>(qh[j]), row_elem(krow, j, s.dtype), dot);
        const double l = __dmul_rn(dot, scale);
        lg[x] = l;
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
    for (int x = threadIdx.x; x < X; x += blockDim.x)
        if (valid(x)) lg[x] = exp(lg[x] - m);
    __syncthreads();
    if (threadIdx.x == 0) {  // sequential in logical order, as the reference
        double sum = 0.0;
        for (int x = 0; x < X; ++x)
            if (valid(x)) sum = __dadd_rn(sum, lg[x]);
        sh_sum = sum;
    }
    __syncthreads();
    const double ws = sh_sum;
    // pass 2: one accumulator per output element, tokens in logical order
    for (int j = threadIdx.x; j < head_dim; j += blockDim.x) {
        double acc = 0.0;
        for (int x = 0; x < X; ++x) {
            if (!valid(x)) continue;
            const uint8_t* vrow = s.pages + (int64_t)row[x / s.B] * page_bytes +
                                  (int64_t)(s.B + x % s.B) * s.pitch + (int64_t)h * head_dim * elt;
            const double w = __ddiv_rn(lg[x], ws);
            acc = __dadd_rn(acc, __dmul_rn(w, row_elem(vrow, j, s.dtype)));
        }
        out[(int64_t)h * head_dim + j] = static_cast<float>(acc);
    }
    if (weight_sums != nullptr && threadIdx.x == 0) {
        double tot = 0.0;
        for (int x = 0; x < X; ++x)
            if (valid(x)) tot = __dadd_rn(tot, __ddiv_rn(lg[x], ws));
        weight_sums[h] = tot;
    }
}

// ---------------------------------------------------------------------------
// Unstructured (per-token) eviction of one table (one CTA): picks a victim
// by `rule` among the retained tokens in logical order, then clears its slot
// (Page::evict, page.hpp:47-56) and auto-frees the page once it drains
// (BlockTable::evict_slot, block_table.cpp:33-46).
//   PE_TOKEN_AT_POSITION   the token at position `arg`          (evict_slot)
//   PE_TOKEN_STREAMING     oldest token with position >= arg    (StreamingLlmPolicy::evict, policy.cpp:184-206)
//   PE_TOKEN_MAX_KEY_NORM  largest ||K||, first on ties         (InvKeyL2Policy::evict, policy.cpp:219-237)
//   PE_TOKEN_KEY_DIFF      largest cos(K, mean K), first on ties (KeyDiffPolicy::evict, policy.cpp:263-283)
// The policies skip the step's own token (`newest`) and fire only when
// retained > C (C < 0: unconditional). *out = victim position or -1.
__device__ __forceinline__ double row_sumsq_f(const uint8_t* row, int w, int dtype) {
    double acc = 0.0;
    for (int i = 0; i < w; ++i) {
        const double x = row_elem(row, i, dtype);
        acc = fma(x, x, acc);
    }
    return acc;
}

// One table, executed by a whole CTA (<= 256 threads; `mean` holds w floats
// of shared or global scratch). Returns, on thread 0, the page released when
// the victim's page drained (the caller pushes it on the free stack) or -1;
// *out (thread 0) = victim position or -1.
__device__ int token_evict_table(const DevState& s, int t, int rule, long long arg, int C, long long newest,
                                 float* mean, long long* out) {
    __shared__ double sh_val[256];
    __shared__ int sh_x[256];
    __shared__ double sh_mnorm;
    const int N = s.num_pages[t];
    const int nf = s.newest_fill[t];
    const int X = N * s.B;
    int32_t* row = s.block_table + (int64_t)t * s.max_pages;
    const int64_t page_bytes = (int64_t)2 * s.B * s.pitch;
    if (C >= 0 && s.retained[t] <= C) {
        if (threadIdx.x == 0) *out = -1;
        return -1;
    }
    auto valid = [&](int x) {
        const int j = x / s.B, sl = x % s.B;
        return sl < (j == N - 1 ? nf : s.B) && !slot_hole(s, row[j], sl);
    };
    auto krow = [&](int x) { return s.pages + (int64_t)row[x / s.B] * page_bytes + (int64_t)(x % s.B) * s.pitch; };
    auto pos_of = [&](int x) { return (long long)s.positions[(int64_t)row[x / s.B] * s.B + x % s.B]; };
    if (rule == PE_TOKEN_KEY_DIFF) {
        // mean_key (policy.cpp:117-134): double sums in logical order, cast to float
        for (int i = threadIdx.x; i < s.w; i += blockDim.x) {
            double acc = 0.0;
            int cnt = 0;
            for (int x = 0; x < X; ++x) {
                if (!valid(x)) continue;
                acc = __dadd_rn(acc, row_elem(krow(x), i, s.dtype));
                ++cnt;
            }
            mean[i] = static_cast<float>(acc / static_cast<double>(cnt));
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double acc = 0.0;
            for (int i = 0; i < s.w; ++i) acc = fma(static_cast<double>(mean[i]), static_cast<double>(mean[i]), acc);
            sh_mnorm = sqrt(acc);
        }
        __syncthreads();
    }
    const double mnorm = sh_mnorm;
    double bv = -INFINITY;
    int bx = 0x7FFFFFFF;
    for (int x = threadIdx.x; x < X; x += blockDim.x) {
        if (!valid(x)) continue;
        const long long p = pos_of(x);
        double v;
        if (rule == PE_TOKEN_AT_POSITION) {
            if (p != arg) continue;
            v = 0.0;
        } else if (rule == PE_TOKEN_STREAMING) {
            if (p < arg) continue;
            v = 0.0;
        } else {
            if (p == newest) continue;
            const uint8_t* kr = krow(x);
            const double kn = sqrt(row_sumsq_f(kr, s.w, s.dtype));
            if (rule == PE_TOKEN_MAX_KEY_NORM) {
                v = kn;
            } else {  // cosine_similarity (policy.cpp:103-115)
                if (kn < kNormEps || mnorm < kNormEps) {
                    v = -1.0;
                } else {
                    double dot = 0.0;
                    for (int i = 0; i < s.w; ++i) dot = fma(row_elem(kr, i, s.dtype), static_cast<double>(mean[i]), dot);
                    v = __ddiv_rn(dot, __dmul_rn(kn, mnorm));
                }
            }
        }
        if (v > bv) {  // x ascending per thread: ties keep the first
            bv = v;
            bx = x;
        }
    }
    sh_val[threadIdx.x] = bv;
    sh_x[threadIdx.x] = bx;
    __syncthreads();
    if (threadIdx.x != 0) return -1;
    for (int i = 1; i < (int)blockDim.x; ++i) {
        if (sh_x[i] == 0x7FFFFFFF) continue;
        if (bx == 0x7FFFFFFF || sh_val[i] > bv || (sh_val[i] == bv && sh_x[i] < bx)) {
            bv = sh_val[i];
            bx = sh_x[i];
        }
    }
    if (bx == 0x7FFFFFFF) {
        if (rule == PE_TOKEN_AT_POSITION) set_status(s.status, PE_UNKNOWN_POSITION);
        *out = -1;
        return -1;
    }
    const int j = bx / s.B, sl = bx % s.B;
    const int page = row[j];
    *out = pos_of(bx);
    s.holes[page] |= 1ull << sl;
    s.retained[t] -= 1;
    const int cursor = (j == N - 1) ? nf : s.B;
    const int fill = page_fill(s, page, cursor);
    if (fill == 0) {  // drained: release whole (the caller pushes it) and close ranks
        s.holes[page] = 0ull;
        for (int k = j; k < N - 1; ++k) row[k] = row[k + 1];
        row[N - 1] = -1;
        s.num_pages[t] = N - 1;
        if (j == N - 1) s.newest_fill[t] = (N - 1 > 0) ? s.B : 0;
        return page;
    }
    if (cursor == s.B) {  // keep the cached page mean of a full page current
        double sum = 0.0;
        for (int k = 0; k < s.B; ++k)
            if (!slot_hole(s, page, k)) sum += s.token_scores[(int64_t)page * s.B + k];
        s.page_scores[page] = sum / static_cast<double>(fill);
    }
    return -1;
}

__global__ void token_evict_kernel(DevState s, int32_t t, int32_t rule, long long arg, int32_t C, long long newest,
                                   float* mean, long long* out) {
    const int released = token_evict_table(s, t, rule, arg, C, newest, mean, out);
    if (threadIdx.x == 0 && released >= 0) {  // release, page_pool.cpp:35-38
        const int top = *s.top;
        s.stack[top] = released;
        *s.top = top + 1;
    }
}

// Batched token eviction (the StreamingLLM / InvKeyL2 / KeyDiff decode step
// over every table of a layer range, after the step's append launch): one
// CTA per launch table, the table's mean key (KeyDiff) in shared memory;
// newest_pos[seq] is the step's appended position. Pages that drain are
// parked in vpage[y] and pushed by the grid's last CTA in ascending table
// id (canonical order: the append launch's pops, then these pushes).
__global__ void __launch_bounds__(256) token_evict_batch_kernel(DevState s, TableSet ts, int32_t rule, long long arg,
                                                                int32_t C, const int64_t* newest_pos,
                                                                int64_t* victims, int32_t* vpage,
                                                                unsigned long long grid_last) {
    extern __shared__ float mean_sm[];
    __shared__ long long vpos;
    const int y = blockIdx.x;
    const int t = ts.table(s, y);
    const int released = token_evict_table(s, t, rule, arg, C, newest_pos[ts.pos_index(s, y)], mean_sm, &vpos);
    if (threadIdx.x == 0) {
        vpage[y] = released;
        if (victims) victims[y] = vpos;
    }
    push_victims_if_last(s, ts.size(s), vpage, grid_last, 1);
}

// ---------------------------------------------------------------------------
// Prefill scoring + selection for the InvKeyL2 / KeyDiff baselines
// (compress_by_score, policy.cpp:90-101, with the scores of policy.cpp:212-216
// and :244-260): one thread per token scores it, a bitonic sort orders
// (score, position) ascending (rank_tokens, importance.cpp:41-60) and the
// first k are flagged.
__global__ void prompt_mean_key_kernel(const float* k, int n, int w, float* mean, double* mnorm) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < w; i += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int x = 0; x < n; ++x) acc = __dadd_rn(acc, static_cast<double>(k[(int64_t)x * w + i]));
        mean[i] = static_cast<float>(acc / static_cast<double>(n));
    }
    __threadfence();
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0 && gridDim.x == 1) {
        double acc = 0.0;
        for (int i = 0; i < w; ++i) acc = fma(static_cast<double>(mean[i]), static_cast<double>(mean[i]), acc);
        *mnorm = sqrt(acc);
    }
}

__global__ void prompt_score_kernel(const float* k, int n, int w, int rule, const float* mean, const double* mnorm,
                                    const long long* pos, int n_pad, double* score, long long* spos, int* sidx) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= n_pad) return;
    if (x >= n) {
        score[x] = INFINITY;
        spos[x] = 0x7FFFFFFFFFFFFFFFll;
        sidx[x] = x;
        return;
    }
    const float* kr = k + (int64_t)x * w;
    double acc = 0.0;
    for (int i = 0; i < w; ++i) acc = fma(static_cast<double>(kr[i]), static_cast<double>(kr[i]), acc);
    const double kn = sqrt(acc);
    double v;
    if (rule == PE_TOKEN_MAX_KEY_NORM) {
        v = 1.0 / fmax(kn, kNormEps);
    } else {
        const double mn = *mnorm;
        double c;
        if (kn < kNormEps || mn < kNormEps) {
            c = -1.0;
        } else {
            double dot = 0.0;
            for (int i = 0; i < w; ++i) dot = fma(static_cast<double>(kr[i]), static_cast<double>(mean[i]), dot);
            c = __ddiv_rn(dot, __dmul_rn(kn, mn));
        }
        v = -c;
    }
    score[x] = v;
    spos[x] = pos[x];
    sidx[x] = x;
}

__global__ void bitonic_step_kernel(double* score, long long* spos, int* sidx, int n_pad, int j, int k) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_pad) return;
    const int o = i ^ j;
    if (o <= i) return;
    const bool less_io = score[o] < score[i] || (score[o] == score[i] && spos[o] < spos[i]);
    const bool up = (i & k) == 0;
    if (less_io == up) {  // out of order for this direction: swap
        const double a = score[i];
        score[i] = score[o];
        score[o] = a;
        const long long b = spos[i];
        spos[i] = spos[o];
        spos[o] = b;
        const int c = sidx[i];
        sidx[i] = sidx[o];
        sidx[o] = c;
    }
}

__global__ void flag_first_kernel(const int* sidx, int k, uint8_t* flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k) flags[sidx[i]] = 1;
}


// ---------------------------------------------------------------------------
// Invariant checker (pe_check_invariants): one warp per table, then the free
// stack, then a per-page reference count pass. counters: [0] pages mapped,
// [1] page not full, [2] retained mismatch, [3] budget, [4] position order,
// [5] refcount.
__global__ void invariants_tables_kernel(DevState s, int32_t* refs, unsigned long long* counters) {
    const int lane = threadIdx.x & 31;
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (t >= s.n_tables) return;
    const int N = s.num_pages[t];
    const int nf = s.newest_fill[t];
    const int32_t* row = s.block_table + (int64_t)t * s.max_pages;
    int occupied = 0, not_full = 0, order = 0;
    long long prev_last = -1;  // last retained position of the previous chunk of pages
    for (int base = 0; base < N; base += 32) {
        const int j = base + lane;
        long long first = -1, last = -1;
        int cnt = 0;
        bool bad_order = false;
        if (j < N) {
            const int page = row[j];
            atomicAdd(refs + page, 1);
            const int cursor = j == N - 1 ? nf : s.B;
            long long pv = -1;
            for (int sl = 0; sl < cursor; ++sl) {
                if (slot_hole(s, page, sl)) continue;
                const long long p = s.positions[(int64_t)page * s.B + sl];
                if (pv >= 0 && p <= pv) bad_order = true;
                if (first < 0) first = p;
                pv = p;
                ++cnt;
            }
            last = pv;
            // page-aligned eviction: every non-newest page is full; with holes
            // (unstructured eviction) a mapped page holds >= 1 token (a page
            // that drains is released, block_table.cpp:33-46)
            if (!s.holes_on ? (j < N - 1 && cnt != s.B) : cnt == 0) ++not_full;
        }
        occupied += cnt;
        order += bad_order;
        // ordering across consecutive pages: page j's first > page j-1's last
        const long long left_last = __shfl_up_sync(0xFFFFFFFFu, last, 1);
        const long long chain = lane == 0 ? prev_last : left_last;
        if (j < N && first >= 0 && chain >= 0 && first <= chain) ++order;
        // carry the last non-empty page's last position into the next chunk
        long long carry = last;
        for (int o = 1; o < 32; o <<= 1) {  // inclusive "last valid" scan
            const long long v = __shfl_up_sync(0xFFFFFFFFu, carry, o);
            if (lane >= o && carry < 0) carry = v;
        }
        const long long chunk_last = __shfl_sync(0xFFFFFFFFu, carry, 31);
        if (chunk_last >= 0) prev_last = chunk_last;
    }
    for (int o = 16; o > 0; o >>= 1) {
        occupied += __shfl_xor_sync(0xFFFFFFFFu, occupied, o);
        not_full += __shfl_xor_sync(0xFFFFFFFFu, not_full, o);
        order += __shfl_xor_sync(0xFFFFFFFFu, order, o);
    }
    if (lane == 0) {
        atomicAdd(counters + 0, (unsigned long long)N);
        if (not_full) atomicAdd(counters + 1, (unsigned long long)not_full);
        if (occupied != s.retained[t]) atomicAdd(counters + 2, 1ull);
        if (s.policy == PE_POLICY_PAGED_EVICTION && s.retained[t] > s.C + s.B) atomicAdd(counters + 3, 1ull);
        if (order) atomicAdd(counters + 4, (unsigned long long)order);
    }
}

__global__ void invariants_free_kernel(DevState s, int32_t* refs) {
    const int top = *s.top;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < top; i += gridDim.x * blockDim.x) {
        const int page = s.stack[i];
        if (page >= 0 && page < s.capacity) atomicAdd(refs + page, 1);
    }
}

__global__ void invariants_refs_kernel(DevState s, const int32_t* refs, unsigned long long* counters) {
    unsigned long long bad = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s.capacity; i += gridDim.x * blockDim.x)
        bad += refs[i] != 1;
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xFFFFFFFFu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(counters + 5, bad);
}


// ---------------------------------------------------------------------------
// HBM probe (pe_probe_hbm): streaming read (256-bit loads, reduced so the
// loads are live) and copy over a buffer larger than L2, for the roofline
// denominators of read-dominated kernels (K2 reads 34.5 GB and writes 43 MB).
__global__ void probe_read_kernel(const uint4* __restrict__ src, size_t n16, unsigned long long* sink) {
    unsigned long long acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16 / 2; i += stride) {
        u32x8 v;
        asm("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]), "=r"(v.w[6]),
              "=r"(v.w[7])
            : "l"(src + 2 * i));
        acc += v.w[0] ^ v.w[3] ^ v.w[5] ^ v.w[7];
    }
    if (acc == 0x1234567890ull) atomicAdd(sink, acc);  // never true for the probe data; keeps the loads
}

__global__ void probe_copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) dst[i] = __ldcs(src + i);
}

// ---------------------------------------------------------------------------
// step_log_kernel: the engine-owned StepRecord fields of one decode step
// (metrics.hpp:18-28) per launch table: retained_len, page_count, the newest
// page's occupied slots (Page::fill, holes excluded) and the decision
// (victims[i], the evicted logical page or -1), for the host-side emitters.
__global__ void step_log_kernel(DevState s, TableSet ts, const int32_t* victims, pe_step_entry* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ts.size(s)) return;
    const int t = ts.table(s, i);
    const int np = s.num_pages[t];
    int fill = 0;
    if (np > 0) fill = page_fill(s, s.block_table[(int64_t)t * s.max_pages + np - 1], s.newest_fill[t]);
    pe_step_entry e;
    e.retained_len = s.retained[t];
    e.page_count = np;
    e.newest_fill = fill;
    e.victim = victims[i];
    out[i] = e;
}

}  // namespace pe
