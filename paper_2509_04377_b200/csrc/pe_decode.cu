// Decode-time kernels of the B200 PagedEviction engine:
//   plan_kernel          canonical-order free-list planning for one launch
//   append_kernel        K0: BlockTable::append_token for every table of the launch
//   evict_score_kernel   K2: recompute page scores from resident K/V bytes, last CTA per
//                        table takes the argmin and evicts (PagedEvictionPolicy::evict)
//   evict_cached_kernel  K2c: the same decision from page means cached at fill time
#include "pe_kernels.cuh"
#include "pe_score.cuh"

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
// append_kernel (K0): one warp per 16 launch tables; lane pair r owns table
// i0 + r. The pair reads the new token's K and V rows once into registers,
// copies them into the newest page's write cursor (Page::write,
// page.hpp:39-44) and computes the token's exact score from the same
// registers (cached norms, kv_vector.hpp:42-43). A page is opened (popped in
// canonical order) when needed (block_table.cpp:12-15); when the write fills
// the page its mean score is cached (importance.cpp:19-30).
template <int SV>
__global__ void __launch_bounds__(kAppendThreads) append_kernel(DevState s, TableSet ts,
                                                                 const uint8_t* __restrict__ k_rows,
                                                                 const uint8_t* __restrict__ v_rows,
                                                                 const int64_t* __restrict__ positions,
                                                                 const int32_t* __restrict__ rank,
                                                                 const LaunchCtl* __restrict__ ctl) {
    if (ctl->abort) return;
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int n = ts.size(s);
    const int i0 = (blockIdx.x * (kAppendThreads / 32) + wid) * 16;
    if (i0 >= n) return;
    const int my_i = i0 + (lane >> 1);
    const bool has = my_i < n;
    const int q = lane & 1;

    int t = 0, page = 0, slot = 0, np = 0, rk = -1;
    if (has) {
        t = ts.table(s, my_i);
        np = s.num_pages[t];
        rk = rank[my_i];
        if (rk >= 0) {
            page = s.stack[ctl->pop_base - 1 - rk];
            slot = 0;
        } else {
            page = s.block_table[(int64_t)t * s.max_pages + np - 1];
            slot = s.newest_fill[t];
        }
    }
    __syncwarp();  // both lanes of a pair read the table state before lane 0 updates it
    if (has && q == 0 && rk >= 0) {
        s.block_table[(int64_t)t * s.max_pages + np] = page;
        s.num_pages[t] = np + 1;
    }
    const int64_t in_row = has ? ts.input_row(s, my_i) : 0;
    const uint8_t* krow = k_rows + in_row * s.row_bytes;
    const uint8_t* vrow = v_rows + in_row * s.row_bytes;
    uint8_t* kdst = s.pages + (((int64_t)page * 2 + 0) * s.B + slot) * s.pitch;
    uint8_t* vdst = s.pages + (((int64_t)page * 2 + 1) * s.B + slot) * s.pitch;
    const double S = pair_token_score<SV>(krow, vrow, has, s.w, s.dtype, has ? kdst : nullptr,
                                          has ? vdst : nullptr);
    if (has && q == 0) {
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
// scores pages [c*P, c*P+P) of evicting table work[y]; each warp takes whole
// pages: lane pair r scores slot r (K row r, V row r of the page, both
// 256-byte rows read straight into registers), the page mean is the
// slot-order sum / fill (score_pages -> page_score, importance.cpp:19-39).
// The last CTA of the table (atomic ticket) takes the argmin and evicts.
template <int SV>
__global__ void __launch_bounds__(kEvictThreads, 4) evict_score_kernel(
    DevState s, TableSet ts, int pages_per_cta, const int32_t* __restrict__ work,
    const int32_t* __restrict__ rank, const LaunchCtl* __restrict__ ctl, double* scratch,
    int32_t* tickets, int32_t* victims) {
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
    const int64_t page_bytes = (int64_t)2 * s.B * s.pitch;

    if (s.B == 16) {
        // one 16-slot group per page, read straight into registers (no
        // prefetch buffer: occupancy, i.e. warps in flight, hides HBM latency)
        const int slot = lane >> 1;
        const int64_t ko = (int64_t)slot * s.pitch, vo = (int64_t)(16 + slot) * s.pitch;
        for (int lp = wid; lp < np; lp += nw) {
            const uint8_t* base = s.pages + (int64_t)__ldg(row + p0 + lp) * page_bytes;
            const double S = pair_token_score<SV>(base + ko, base + vo, true, s.w, s.dtype);
            double sum = 0.0;
#pragma unroll
            for (int j = 0; j < 16; ++j) sum += __shfl_sync(0xFFFFFFFFu, S, 2 * j);
            if (lane == 0) page_mean[lp] = sum / 16.0;
        }
    } else {
        for (int lp = wid; lp < np; lp += nw) {
            const int id = __ldg(row + p0 + lp);
            const uint8_t* base = s.pages + (int64_t)id * page_bytes;
            double sum = 0.0;
            for (int s0 = 0; s0 < s.B; s0 += 16) {
                const int slot = s0 + (lane >> 1);
                const bool valid = slot < s.B;
                const double S = pair_token_score<SV>(base + (int64_t)slot * s.pitch,
                                                      base + (int64_t)(s.B + slot) * s.pitch, valid, s.w, s.dtype);
                const int ns = min(16, s.B - s0);
                for (int j = 0; j < ns; ++j) sum += __shfl_sync(0xFFFFFFFFu, S, 2 * j);
            }
            if (lane == 0) page_mean[lp] = sum / static_cast<double>(s.B);
        }
    }
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
        finalize_evict(s, t, i, N, scratch + (int64_t)y * s.max_pages, rank, ctl, victims, nullptr);
        if (lane == 0) tickets[y] = 0;
    }
}

template <int SV>
void launch_evict_score(dim3 grid, int threads, cudaStream_t st, const DevState& s, const TableSet& ts, int ppc,
                        const int32_t* work, const int32_t* rank, const LaunchCtl* ctl, double* scratch,
                        int32_t* tickets, int32_t* victims) {
    evict_score_kernel<SV><<<grid, threads, 0, st>>>(s, ts, ppc, work, rank, ctl, scratch, tickets, victims);
}

template <int SV>
void launch_append(int blocks, cudaStream_t st, const DevState& s, const TableSet& ts, const uint8_t* k,
                   const uint8_t* v, const int64_t* pos, const int32_t* rank, const LaunchCtl* ctl) {
    append_kernel<SV><<<blocks, kAppendThreads, 0, st>>>(s, ts, k, v, pos, rank, ctl);
}

void launch_evict_score_any(int variant, dim3 grid, int threads, cudaStream_t st, const DevState& s,
                            const TableSet& ts, int ppc, const int32_t* work, const int32_t* rank,
                            const LaunchCtl* ctl, double* scratch, int32_t* tickets, int32_t* victims) {
    PE_SCORE_DISPATCH(variant, (launch_evict_score<SV>(grid, threads, st, s, ts, ppc, work, rank, ctl, scratch,
                                                        tickets, victims)));
}

void launch_append_any(int variant, int blocks, cudaStream_t st, const DevState& s, const TableSet& ts,
                       const uint8_t* k, const uint8_t* v, const int64_t* pos, const int32_t* rank,
                       const LaunchCtl* ctl) {
    PE_SCORE_DISPATCH(variant, (launch_append<SV>(blocks, st, s, ts, k, v, pos, rank, ctl)));
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
