// Decode-time kernels of the B200 PagedEviction engine:
//   plan_kernel          canonical-order free-list planning for one launch
//   append_kernel        K0: BlockTable::append_token for every table of the launch
//   evict_score_kernel   K2: recompute page scores from resident K/V bytes, last CTA per
//                        table takes the argmin and evicts (PagedEvictionPolicy::evict)
//   evict_cached_kernel  K2c: the same decision from page means cached at fill time
#include "pe_kernels.cuh"

namespace pe {

// ---------------------------------------------------------------------------
// plan_kernel: one CTA. Flags every table of the launch, ranks the flags in
// ascending table id (exclusive scan) and reserves the free-stack range.
//   APPEND: flag = the append opens a page (no page, or newest write-full:
//           block_table.cpp:12) -> pops, LIFO from the top (page_pool.cpp:29-31)
//   EVICT:  flag = PagedEviction trigger (newest write-full && retained > C:
//           policy.cpp:147-150) -> pushes (page_pool.cpp:37)
// Pops of one launch precede its pushes.
__global__ void __launch_bounds__(1024) plan_kernel(DevState s, TableSet ts, int mode,
                                                     int32_t* rank, int32_t* work,
                                                     int32_t* victims, LaunchCtl* ctl) {
    __shared__ int sm[33];
    __shared__ int bad;
    const int n = ts.size(s);
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int lo = min(n, (int)threadIdx.x * per);
    const int hi = min(n, lo + per);
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    int cnt = 0;
    for (int i = lo; i < hi; ++i) {
        const int t = ts.table(s, i);
        const int np = s.num_pages[t];
        int f;
        if (mode == kPlanAppend) {
            f = (np == 0 || s.newest_fill[t] == s.B) ? 1 : 0;
            if (f && np >= s.max_pages) atomicOr(&bad, 1);
        } else {
            f = (s.policy == PE_POLICY_PAGED_EVICTION && np > 0 && s.newest_fill[t] == s.B &&
                 s.retained[t] > s.C) ? 1 : 0;
        }
        cnt += f;
    }
    int total;
    int base = block_excl_scan(cnt, sm, &total);
    for (int i = lo; i < hi; ++i) {
        const int t = ts.table(s, i);
        const int np = s.num_pages[t];
        int f;
        if (mode == kPlanAppend) {
            f = (np == 0 || s.newest_fill[t] == s.B) ? 1 : 0;
        } else {
            f = (s.policy == PE_POLICY_PAGED_EVICTION && np > 0 && s.newest_fill[t] == s.B &&
                 s.retained[t] > s.C) ? 1 : 0;
            if (victims) victims[i] = -1;
        }
        rank[i] = f ? base : -1;
        if (f && work) work[base] = i;
        base += f;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int top = *s.top;
        if (mode == kPlanAppend) {
            if (bad) {
                set_status(s.status, PE_INVALID_STATE);
                ctl->abort = 1;
            } else if (total > top) {
                set_status(s.status, PE_POOL_EXHAUSTED);  // PoolExhausted, page_pool.cpp:26-28
                ctl->abort = 1;
            } else {
                ctl->abort = 0;
                ctl->pop_base = top;
                *s.top = top - total;
            }
        } else {
            ctl->abort = 0;
            ctl->push_base = top;
            ctl->count = total;
            *s.top = top + total;
        }
    }
}

// ---------------------------------------------------------------------------
// append_kernel (K0): one warp per 16 launch tables. Lanes 0-15 stream the K
// rows and lanes 16-31 the V rows of those tables (exact fp64 norms ->
// cached token score, kv_vector.hpp:42-43), the warp copies both rows into
// the newest page's write cursor (Page::write, page.hpp:39-44), opening a
// page popped in canonical order when needed (block_table.cpp:12-15).
// When the write fills the page its mean score is cached (importance.cpp:19-30).
__global__ void __launch_bounds__(kAppendThreads) append_kernel(DevState s, TableSet ts,
                                                                 const uint8_t* __restrict__ k_rows,
                                                                 const uint8_t* __restrict__ v_rows,
                                                                 const int64_t* __restrict__ positions,
                                                                 const int32_t* __restrict__ rank,
                                                                 const LaunchCtl* __restrict__ ctl) {
    extern __shared__ __align__(16) uint8_t smem[];
    if (ctl->abort) return;
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int n = ts.size(s);
    const int i0 = (blockIdx.x * (kAppendThreads / 32) + wid) * 16;
    if (i0 >= n) return;
    uint8_t* stage = smem + wid * (2 * kStageBytes);
    const int my_i = i0 + (lane & 15);
    const bool has = my_i < n;

    // Resolve (page, slot) for the lane's table (lanes l and l+16 agree).
    int t = 0, page = -1, slot = 0;
    if (has) {
        t = ts.table(s, my_i);
        const int np = s.num_pages[t];
        if (rank[my_i] >= 0) {
            page = s.stack[ctl->pop_base - 1 - rank[my_i]];
            slot = 0;
            if (lane < 16) {
                s.block_table[(int64_t)t * s.max_pages + np] = page;
                s.num_pages[t] = np + 1;
            }
        } else {
            page = s.block_table[(int64_t)t * s.max_pages + np - 1];
            slot = s.newest_fill[t];
        }
    }
    const int64_t in_row = has ? ts.input_row(s, my_i) : 0;
    const uint8_t* src = (lane < 16 ? k_rows : v_rows) + in_row * s.row_bytes;

    // copy: each half-warp lane copies its row (row_bytes multiple of 16)
    if (has) {
        uint8_t* dst = s.pages + (((int64_t)page * 2 + (lane >> 4)) * s.B + slot) * s.pitch;
        for (int off = 0; off < s.row_bytes; off += 16) {
            *reinterpret_cast<uint4*>(dst + off) = __ldg(reinterpret_cast<const uint4*>(src + off));
        }
    }
    // exact norms via the warp streamer (one set of 32 rows)
    double sq = 0.0;
    warp_stream_sumsq<2>(1, s.row_bytes, s.w, s.dtype, stage,
                         [&](int, int row) -> const uint8_t* {
                             const int ii = i0 + (row & 15);
                             if (ii >= n) return nullptr;
                             return (row < 16 ? k_rows : v_rows) + ts.input_row(s, ii) * s.row_bytes;
                         },
                         [&](int, double r, bool) { sq = r; });
    const double v2 = __shfl_down_sync(0xFFFFFFFFu, sq, 16);
    if (has && lane < 16) {
        const double S = token_score_from_sumsq(sq, v2);
        const int64_t ps = (int64_t)page * s.B + slot;
        s.positions[ps] = static_cast<int32_t>(positions[ts.input_row(s, my_i) / s.tab_heads % s.n_seqs]);
        s.token_scores[ps] = S;
        s.newest_fill[t] = slot + 1;
        s.retained[t] += 1;
        if (slot + 1 == s.B) {
            // page_score, importance.cpp:19-30: mean over the B slots in slot order
            double sum = 0.0;
            for (int j = 0; j < s.B - 1; ++j) sum += s.token_scores[(int64_t)page * s.B + j];
            sum += S;
            s.page_scores[page] = sum / static_cast<double>(s.B);
        }
    }
}

// ---------------------------------------------------------------------------
// Finalisation of one evicting table (shared by K2 and K2c), executed by one
// warp: rank_pages argmin (strict <, ties -> smaller index, importance.cpp:62-75),
// free_page (retained -= fill; erase -> entries shift left, block_table.cpp:21-31),
// release = push on the free stack at the canonical rank (page_pool.cpp:35-38).
__device__ __forceinline__ void finalize_evict(const DevState& s, int t, int i, int N,
                                               const double* scores, const int32_t* rank,
                                               const LaunchCtl* ctl, int32_t* victims,
                                               int32_t* /*unused*/) {
    const int lane = threadIdx.x & 31;
    double best = 0.0;
    int bj = 0x7FFFFFFF;
    for (int j = lane; j < N; j += 32) {
        const double v = __ldcg(scores + j);
        if (bj == 0x7FFFFFFF || v < best) {
            best = v;
            bj = j;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xFFFFFFFFu, best, o);
        const int oj = __shfl_xor_sync(0xFFFFFFFFu, bj, o);
        if (oj != 0x7FFFFFFF && (bj == 0x7FFFFFFF || ob < best || (ob == best && oj < bj))) {
            best = ob;
            bj = oj;
        }
    }
    const int victim = bj;
    int32_t* row = s.block_table + (int64_t)t * s.max_pages;
    const int victim_page = row[victim];
    // shift left in 32-entry chunks: every read of a chunk precedes its writes
    for (int base = victim; base < N - 1; base += 32) {
        const int v = (base + lane + 1 < N) ? row[base + lane + 1] : 0;
        __syncwarp();
        if (base + lane < N - 1) row[base + lane] = v;
        __syncwarp();
    }
    if (lane == 0) {
        row[N - 1] = -1;
        s.num_pages[t] = N - 1;
        s.retained[t] -= s.B;  // every page is full when the trigger fires
        s.newest_fill[t] = (N - 1 > 0) ? s.B : 0;
        s.stack[ctl->push_base + rank[i]] = victim_page;
        if (victims) victims[i] = victim;
        atomicAdd(s.evict_count, 1ull);
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// evict_score_kernel (K2, recompute): grid (work items, chunks). CTA (y, c)
// scores pages [c*P, c*P+P) of evicting table work[y]: warps stream whole
// pages (2B contiguous rows: K slots then V slots) through the exact fp64
// row streamer, S per slot = ||V||/max(||K||,eps), page mean = slot-order sum
// / fill (score_pages -> page_score, importance.cpp:19-39). The last CTA of
// the table (atomic ticket) takes the argmin and evicts.
__global__ void __launch_bounds__(kEvictThreads) evict_score_kernel(
    DevState s, TableSet ts, int pages_per_cta, const int32_t* __restrict__ work,
    const int32_t* __restrict__ rank, const LaunchCtl* __restrict__ ctl, double* scratch,
    int32_t* tickets, int32_t* victims) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ double page_mean[kMaxPagesPerCta];
    __shared__ int last;
    const int y = blockIdx.x;
    if (y >= ctl->count) return;
    const int i = work[y];
    const int t = ts.table(s, i);
    const int N = s.num_pages[t];
    const int n_cta = (N + pages_per_cta - 1) / pages_per_cta;
    const int c = blockIdx.y;
    if (c >= n_cta) return;
    const int p0 = c * pages_per_cta;
    const int np = min(pages_per_cta, N - p0);
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    const int32_t* row = s.block_table + (int64_t)t * s.max_pages;
    const int sets_per_page = (s.B + 15) / 16;
    uint8_t* stage = smem + wid * (kEvictStages * kStageBytes);

    // this warp's pages: p0 + wid, p0 + wid + nw, ...
    const int my_pages = np > wid ? (np - wid + nw - 1) / nw : 0;
    double sum = 0.0;  // running slot-order sum of the current page (lane 0)
    warp_stream_sumsq<kEvictStages>(
        my_pages * sets_per_page, s.row_bytes, s.w, s.dtype, stage,
        [&](int set, int r) -> const uint8_t* {
            const int pg = p0 + wid + (set / sets_per_page) * nw;
            const int q = set % sets_per_page;
            const int slot = q * 16 + (r & 15);
            if (slot >= s.B) return nullptr;
            const int id = row[pg];
            return s.pages + (((int64_t)id * 2 + (r >> 4)) * s.B + slot) * s.pitch;
        },
        [&](int set, double sq, bool present) {
            const double v2 = __shfl_down_sync(0xFFFFFFFFu, sq, 16);
            double S = 0.0;
            if (lane < 16 && present) S = token_score_from_sumsq(sq, v2);
            const int q = set % sets_per_page;
            const int nslots = min(16, s.B - q * 16);
            for (int j = 0; j < nslots; ++j) sum += __shfl_sync(0xFFFFFFFFu, S, j);
            if (q == sets_per_page - 1) {
                if (lane == 0) page_mean[(set / sets_per_page) * nw + wid] = sum / (double)s.B;
                sum = 0.0;
            }
        });
    __syncthreads();
    for (int j = threadIdx.x; j < np; j += blockDim.x) {
        scratch[(int64_t)y * s.max_pages + p0 + j] = page_mean[j];
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int tk = atomicAdd(&tickets[y], 1);
        last = (tk == n_cta - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (wid == 0) {
        const double* sc = scratch + (int64_t)y * s.max_pages;
        // volatile-free: other CTAs' writes are ordered by their fence + our ticket
        finalize_evict(s, t, i, N, sc, rank, ctl, victims, nullptr);
        if (lane == 0) tickets[y] = 0;
    }
}

// ---------------------------------------------------------------------------
// evict_cached_kernel (K2c): one warp per work item; page means were cached
// when each page filled, so the decision reads N doubles (gathered through
// the block table) instead of N pages. Bit-identical to K2.
__global__ void __launch_bounds__(256) evict_cached_kernel(DevState s, TableSet ts,
                                                           const int32_t* __restrict__ work,
                                                           const int32_t* __restrict__ rank,
                                                           const LaunchCtl* __restrict__ ctl,
                                                           double* scratch, int32_t* victims) {
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int y = blockIdx.x * 8 + wid;
    if (y >= ctl->count) return;
    const int i = work[y];
    const int t = ts.table(s, i);
    const int N = s.num_pages[t];
    const int32_t* row = s.block_table + (int64_t)t * s.max_pages;
    double* sc = scratch + (int64_t)y * s.max_pages;
    for (int j = lane; j < N; j += 32) sc[j] = s.page_scores[row[j]];
    __syncwarp();
    finalize_evict(s, t, i, N, sc, rank, ctl, victims, nullptr);
}

}  // namespace pe
