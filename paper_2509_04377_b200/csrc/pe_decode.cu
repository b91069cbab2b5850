// Decode-time kernels of the B200 PagedEviction engine:
//   append_kernel        K0: BlockTable::append_token for every table of the launch
//   evict_score_kernel   K2: recompute page scores from resident K/V bytes, last CTA per
//                        table takes the argmin and evicts (PagedEvictionPolicy::evict)
//   evict_cached_kernel  K2c: the same decision from page means cached at fill time
#include "pe_kernels.cuh"
#include "pe_score.cuh"

#ifdef PE_K0_TRACE
// Tooling build only (PE_NVCC_EXTRA=-DPE_K0_TRACE, tools/k0_trace.py):
// %globaltimer stamps of thread 0 of the first kTraceCtas CTAs of the last
// 64 append launches, read back with pe_debug_k0_trace.
namespace pe {
constexpr int kTraceCtas = 256, kTraceStamps = 10;
__device__ unsigned long long g_k0_trace[64 * kTraceCtas * kTraceStamps];
}  // namespace pe
extern "C" int pe_debug_k0_trace(void* out, size_t bytes) {
    return cudaMemcpyFromSymbol(out, pe::g_k0_trace, bytes < sizeof(pe::g_k0_trace) ? bytes : sizeof(pe::g_k0_trace)) ==
                   cudaSuccess
               ? 0
               : -1;
}
#endif

namespace pe {

// ---------------------------------------------------------------------------
// Single-pass canonical pop ranks for an append launch (decoupled look-back):
// CTAs take logical ids from a ticket counter (so a CTA only ever waits on
// CTAs that already started); logical CTA 0 publishes the stack top, every
// CTA publishes its pop count and looks back over its predecessors for its
// exclusive prefix, and the last CTA moves the stack top. Status words:
// epoch << 32 | flag << 30 | value.
//
// Pool exhaustion follows the reference's serial semantics: appends run in
// ascending table id; the first table whose pop finds the stack empty fails
// (PoolExhausted, page_pool.cpp:26-28) and no later table of the launch is
// appended (the exception would have stopped the loop).
constexpr unsigned long long kLbAgg = 1ull << 30;

// Every look-back word is self-contained (epoch, flag and value in one 64-bit
// word, nothing else published through it), so relaxed gpu-scope accesses
// suffice: no release fences (MEMBAR.GPU) on the critical path.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
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
                                                                 unsigned long long* lb_status,
                                                                 unsigned long long* lb_group, LaunchCtl* ctl,
                                                                 unsigned long long ticket_base, int epoch,
                                                                 int fast_ok) {
    __shared__ int sh_lid, sh_warp_cnt[kAppendThreads / 32], sh_prefix, sh_pop_base, sh_fast;
#ifdef PE_K0_TRACE
    unsigned long long tr[kTraceStamps] = {};
#define PE_TR(i) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr[i]))
#else
#define PE_TR(i)
#endif
    PE_TR(0);   // resident
    pdl_top();  // launched with PDL: the launch gap behind the previous kernel is hidden
    PE_TR(8);   // previous kernel complete
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nw = kAppendThreads / 32;
    const int n = ts.size(s);
    const int n_ctas = (n + 16 * nw - 1) / (16 * nw);
    if (threadIdx.x == 0) {
        sh_lid = static_cast<int>(atomicAdd(s.grid_ctr, 1ull) - ticket_base);
        // no-pop fast path: the previous append over the same tables (and no
        // other table operation since, fast_ok) flagged no table as popping
        // on this launch, so every pop rank is 0 and the look-back is skipped
        sh_fast = fast_ok &&
                  *reinterpret_cast<volatile unsigned int*>(&ctl->pop_flag[epoch & 1]) != static_cast<unsigned>(epoch);
    }
    __syncthreads();
    PE_TR(1);
    const int lid = sh_lid;
    const int i0 = (lid * nw + wid) * 16;
    const int my_i = i0 + (lane >> 1);
    const bool has = my_i < n;
    const int q = lane & 1;

    int t = 0, np = 0, slot = 0;
    bool pop = false;
    bool live = has;
    if (has) {
        t = ts.table(s, my_i);
        np = s.num_pages[t];
        slot = s.newest_fill[t];
        pop = (np == 0 || slot == s.B);
        if (pop && np >= s.max_pages) {  // table full (max_pages_per_table): skipped
            if (q == 0) set_status(s.status, PE_INVALID_STATE);
            pop = false;
            live = false;
        }
    }
    const unsigned pop_mask = __ballot_sync(0xFFFFFFFFu, pop && q == 0);
    if (lane == 0) sh_warp_cnt[wid] = __popc(pop_mask);
    __syncthreads();
    PE_TR(2);
    const bool fast = sh_fast;
    if (fast) {
        if (threadIdx.x == 0) {
            int local = 0;
            for (int w = 0; w < nw; ++w) local += sh_warp_cnt[w];
            if (local != 0) set_status(s.status, PE_INVALID_STATE);  // a mispredicted pop: never served below
            sh_prefix = 0;
            sh_pop_base = 0x7FFFFFFF;
        }
    } else if (wid == 0) {
        int local = 0;
        for (int w = 0; w < nw; ++w) local += sh_warp_cnt[w];
        const unsigned long long ep = static_cast<unsigned long long>(static_cast<unsigned>(epoch)) << 32;
        // Two-level look-back: CTA lid = 32g + r publishes its pop count; it
        // sums the counts of CTAs 32g .. lid-1 (lane l reads CTA 32g + l) and
        // the aggregates of groups 0 .. g-1, which the last CTA of each group
        // publishes after its own in-group sum. Every word waited on belongs
        // to a lower lid (deadlock-free in arrival order) and a CTA issues at
        // most 31 + ceil(g/32)*32 loads: all-pairs windows (O(n^2) loads on a
        // few status lines) congested their L2 slices for ~10 us.
        const int g = lid >> 5, r = lid & 31;
        if (lane == 0) {
            st_relaxed_u64(lb_status + lid, ep | kLbAgg | static_cast<unsigned long long>(local));
            if (lid == 0) {
                const int top0 = *s.top;
                st_relaxed_u64(&ctl->top_word, ep | static_cast<unsigned>(top0));
                sh_pop_base = top0;
            }
        }
        // the stack top CTA 0 publishes: first read issued now, re-polled below
        unsigned long long tw = (lane == 0 && lid != 0) ? ld_relaxed_u64(&ctl->top_word) : 0ull;
        unsigned long long w = 0;
        if (lane < r) {
            w = ld_relaxed_u64(lb_status + 32 * g + lane);
            while ((w >> 32) != static_cast<unsigned>(epoch)) {  // not yet published
                __nanosleep(64);
                w = ld_relaxed_u64(lb_status + 32 * g + lane);
            }
        }
        int in_grp = lane < r ? static_cast<int>(w & ((1ull << 30) - 1)) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) in_grp += __shfl_xor_sync(0xFFFFFFFFu, in_grp, o);
        if (lane == 0 && (r == 31 || lid == n_ctas - 1))
            st_relaxed_u64(lb_group + g, ep | static_cast<unsigned long long>(in_grp + local));
        int prefix = in_grp;
        for (int g0 = 0; g0 < g; g0 += 32) {
            unsigned long long gw = 0;
            if (g0 + lane < g) {
                gw = ld_relaxed_u64(lb_group + g0 + lane);
                while ((gw >> 32) != static_cast<unsigned>(epoch)) {
                    __nanosleep(64);
                    gw = ld_relaxed_u64(lb_group + g0 + lane);
                }
            }
            int v = g0 + lane < g ? static_cast<int>(gw & ((1ull << 30) - 1)) : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
            prefix += v;
        }
        PE_TR(6);
        if (lane == 0 && lid != 0) {
            while ((tw >> 32) != static_cast<unsigned>(epoch)) {
                __nanosleep(64);
                tw = ld_relaxed_u64(&ctl->top_word);
            }
            sh_pop_base = static_cast<int>(tw & 0xFFFFFFFFull);
            PE_TR(7);
        }
        if (lane == 0) {
            if (lid == n_ctas - 1) {
                const int total = prefix + local;
                *s.top = sh_pop_base - min(total, sh_pop_base);
            }
            sh_prefix = prefix;
        }
    }
    __syncthreads();
    PE_TR(3);

    // rank of this table's pop among the launch's pops (ascending table id);
    // for a non-popping table: the number of pops before it
    int rank = sh_prefix;
    for (int w = 0; w < wid; ++w) rank += sh_warp_cnt[w];
    rank += __popc(pop_mask & ((1u << (lane & ~1)) - 1u));
    const int top = sh_pop_base;
    if (!fast && pop && rank == top && q == 0) set_status(s.status, PE_POOL_EXHAUSTED);  // first failing pop
    const bool served = live && (pop ? !fast && rank < top : rank <= top);

    int page = 0;
    if (served) {
        if (pop) {
            page = s.stack[top - 1 - rank];
            slot = 0;
        } else {
            page = s.block_table[(int64_t)t * s.max_pages + np - 1];
        }
    }
    __syncwarp();
    if (served && q == 0 && pop) {
        s.block_table[(int64_t)t * s.max_pages + np] = page;
        s.num_pages[t] = np + 1;
    }
    uint8_t* kdst = s.pages + (((int64_t)page * 2 + 0) * s.B + slot) * s.pitch;
    uint8_t* vdst = s.pages + (((int64_t)page * 2 + 1) * s.B + slot) * s.pitch;
    PE_TR(4);
    const int64_t in_row = served ? ts.input_row(s, my_i) : 0;
    const double S = pair_token_score<SV>(k_rows + in_row * s.row_bytes, v_rows + in_row * s.row_bytes, served, s.w,
                                          s.dtype, served ? kdst : nullptr, served ? vdst : nullptr);
    PE_TR(5);
    if (served && q == 0) {
        const int64_t ps = (int64_t)page * s.B + slot;
        s.positions[ps] = static_cast<int32_t>(positions[ts.pos_index(s, my_i)]);
        s.token_scores[ps] = S;
        s.newest_fill[t] = slot + 1;
        s.retained[t] += 1;
        if (slot + 1 == s.B) {
            // page_score, importance.cpp:19-30: mean over the occupied slots in slot order
            double sum = 0.0;
            int cnt = 1;
            const double* ts_page = s.token_scores + (int64_t)page * s.B;
            if (s.B == 16 && !s.holes_on) {  // independent loads, then the slot-order sum
                double x[15];
#pragma unroll
                for (int j = 0; j < 15; ++j) x[j] = ts_page[j];
#pragma unroll
                for (int j = 0; j < 15; ++j) sum += x[j];
                cnt = 16;
            } else {
                for (int j = 0; j < s.B - 1; ++j) {
                    if (slot_hole(s, page, j)) continue;
                    sum += ts_page[j];
                    ++cnt;
                }
            }
            sum += S;
            s.page_scores[page] = sum / static_cast<double>(cnt);
        }
    }
    // will this table pop on the next append? (its newest page is now full;
    // an unserved table is flagged conservatively)
    const bool next_pop = has && q == 0 && (served ? slot + 1 == s.B : true);
    if (__syncthreads_or(next_pop) && threadIdx.x == 0) {
        const int next = epoch % kAppendEpochPeriod + 1;  // the next launch's epoch (opposite parity)
        *reinterpret_cast<volatile unsigned int*>(&ctl->pop_flag[next & 1]) = static_cast<unsigned>(next);
    }
#ifdef PE_K0_TRACE
    PE_TR(9);
    if (threadIdx.x == 0 && blockIdx.x < kTraceCtas) {
        unsigned long long* o = g_k0_trace + ((int64_t)(epoch % 64) * kTraceCtas + blockIdx.x) * kTraceStamps;
        for (int k = 0; k < kTraceStamps; ++k) o[k] = tr[k];
    }
#endif
    (void)nw;
}

// ---------------------------------------------------------------------------
// Finalisation of one evicting table (shared by K2 and K2c), executed by one
// warp: rank_pages argmin (strict <, ties -> smaller index, importance.cpp:62-75),
// free_page (retained -= fill; erase -> entries shift left, block_table.cpp:21-31).
// The released page id is parked in vpage[i]; the grid's last CTA pushes all
// of them on the free stack in ascending table id (push_victims below).
// The released page id goes to *vslot (the launch's vpage entry of the
// table), the logical victim to victims[i] (launch table i).
__device__ __forceinline__ void finalize_evict(const DevState& s, int t, int i, int N, const double* scores,
                                               int32_t* vslot, int32_t* victims) {
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
    // shift left: up to 8 x 32 entries per round are loaded (independent
    // loads, one round trip) before any of them is overwritten
    for (int base = victim; base < N - 1; base += 8 * 32) {
        int v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = base + u * 32 + lane + 1;
            v[u] = j < N ? __ldcg(row + j) : 0;
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = base + u * 32 + lane;
            if (j < N - 1) row[j] = v[u];
        }
        __syncwarp();
    }
    if (lane == 0) {
        row[N - 1] = -1;
        s.num_pages[t] = N - 1;
        // every page is write-full when the trigger fires; holes only come
        // from the table API's unstructured eviction
        s.retained[t] -= page_fill(s, victim_page, s.B);
        if (s.holes_on) s.holes[victim_page] = 0ull;
        s.newest_fill[t] = (N - 1 > 0) ? s.B : 0;
        *vslot = victim_page;
        if (victims) victims[i] = victim;
        atomicAdd(s.evict_count, 1ull);
    }
    __syncwarp();
}

// PagedEviction trigger, policy.cpp:147-150: newest page write-full and
// retained > C (num_pages > 0 implied).
__device__ __forceinline__ bool evict_triggered(const DevState& s, int t) {
    return s.policy == PE_POLICY_PAGED_EVICTION && s.num_pages[t] > 0 && s.newest_fill[t] == s.B &&
           s.retained[t] > s.C;
}


// Page mean of a 16-slot page from the lane-pair scores S (pair r = slot r),
// in slot order (score_pages -> page_score, importance.cpp:19-30); with holes,
// the mean over the occupied slots. Valid on every lane.
template <bool HOLES>
__device__ __forceinline__ double page_mean_b16(const DevState& s, int id, double S) {
    double sum = 0.0;
    if constexpr (!HOLES) {
#pragma unroll
        for (int j = 0; j < 16; ++j) sum += __shfl_sync(0xFFFFFFFFu, S, 2 * j);
        return sum / 16.0;
    } else {
        const unsigned long long hm = s.holes[id];
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const double x = __shfl_sync(0xFFFFFFFFu, S, 2 * j);
            const bool occ = !((hm >> j) & 1ull);
            sum += occ ? x : 0.0;  // S >= +0: adding +0 leaves the sum unchanged
            cnt += occ;
        }
        return sum / static_cast<double>(cnt);
    }
}

// End of a K2 chunk: publish this CTA's page means, take the table's ticket;
// the table's last CTA takes the argmin and evicts. Returns the tables settled.
// scratch rows, tickets and vpage are indexed by TABLE id t (launch-
// independent), so a programmatically overlapped next launch over other
// tables never touches this launch's entries.
__device__ __forceinline__ int publish_chunk(const DevState& s, int t, int y, int N, int p0, int np, int n_cta,
                                             const double* page_mean, double* scratch, int32_t* tickets,
                                             int32_t* vpage, int32_t* victims) {
    __shared__ int last;
    __syncthreads();
    for (int j = threadIdx.x; j < np; j += blockDim.x) scratch[(int64_t)t * s.max_pages + p0 + j] = page_mean[j];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(&tickets[t], 1) == n_cta - 1);
    __syncthreads();
    if (!last) return 0;
    __threadfence();
    if ((threadIdx.x >> 5) == 0) {
        finalize_evict(s, t, y, N, scratch + (int64_t)t * s.max_pages, vpage + t, victims);
        if ((threadIdx.x & 31) == 0) tickets[t] = 0;
    }
    return 1;
}


// ---------------------------------------------------------------------------
// evict_score_kernel (K2, recompute): grid (launch tables, chunks). CTA (y, c)
// scores pages [c*P, c*P+P) of table y if it triggers; each warp takes whole
// pages: lane pair r scores slot r (K row r, V row r of the page, both
// 256-byte rows read straight into registers), the page mean is the
// slot-order sum / fill (score_pages -> page_score, importance.cpp:19-39).
// The last CTA of the table (atomic ticket) takes the argmin and evicts; the
// last CTA of the grid pushes the released pages.
//
// early (PDL, per-layer launches back to back): the engine's previous launch
// on this stream was a K2 launch over OTHER tables, so everything up to the
// table's eviction touches state that launch never writes (this launch's
// tables, their pages, their table-indexed scratch / ticket / vpage
// entries); only the launch-level settle ticket and the free-stack push wait
// for it. The next launch may start as soon as every CTA of this one has.
template <int SV, bool HOLES>
__global__ void __launch_bounds__(kEvictThreads, 5) evict_score_kernel(
    DevState s, TableSet ts, int pages_per_cta, double* scratch, int32_t* tickets, int32_t* vpage,
    int32_t* victims, unsigned long long grid_last, int early) {
    __shared__ double page_mean[kMaxPagesPerCta];
    // not early: wait for the previous kernel BEFORE letting the next one
    // start, so an early launch always starts after the last non-K2 kernel
    // before the chain has completed
    if (!early) pdl_wait();
    pdl_launch_dependents();
    const int y = blockIdx.x;
    const int c = blockIdx.y;
    const int t = ts.table(s, y);
    const bool trig = evict_triggered(s, t);
    const int N = s.num_pages[t];
    const int n_cta = (N + pages_per_cta - 1) / pages_per_cta;
    int settled = 0;  // tables this CTA settles (block-uniform)
    if (!trig) {
        if (c == 0) {
            settled = 1;
            if (threadIdx.x == 0) {
                vpage[t] = -1;
                if (victims) victims[y] = -1;
            }
        }
    } else if (c < n_cta) {
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
                const int id = __ldg(row + p0 + lp);
                const uint8_t* base = s.pages + (int64_t)id * page_bytes;
                const double S = pair_token_score<SV>(base + ko, base + vo, true, s.w, s.dtype);
                const double mean = page_mean_b16<HOLES>(s, id, S);
                if (lane == 0) page_mean[lp] = mean;
            }
        } else {
            for (int lp = wid; lp < np; lp += nw) {
                const int id = __ldg(row + p0 + lp);
                const uint8_t* base = s.pages + (int64_t)id * page_bytes;
                double sum = 0.0;
                int cnt = 0;
                for (int s0 = 0; s0 < s.B; s0 += 16) {
                    const int slot = s0 + (lane >> 1);
                    const bool valid = slot < s.B;
                    const double S = pair_token_score<SV>(base + (int64_t)slot * s.pitch,
                                                          base + (int64_t)(s.B + slot) * s.pitch, valid, s.w,
                                                          s.dtype);
                    const int ns = min(16, s.B - s0);
                    for (int j = 0; j < ns; ++j) {
                        const double x = __shfl_sync(0xFFFFFFFFu, S, 2 * j);
                        if (!(HOLES && slot_hole(s, id, s0 + j))) {
                            sum += x;
                            ++cnt;
                        }
                    }
                }
                if (lane == 0) page_mean[lp] = sum / static_cast<double>(cnt);
            }
        }
        settled = publish_chunk(s, t, y, N, p0, np, n_cta, page_mean, scratch, tickets, vpage, victims);
    }
    if (early) pdl_wait();  // the previous launch's settle tickets and pushes come first
    push_victims_if_last(s, ts.size(s), vpage, grid_last, settled, &ts);
}

template <int SV, bool HOLES>
void launch_evict_score_t(dim3 grid, int threads, cudaStream_t st, const DevState& s, const TableSet& ts, int ppc,
                          double* scratch, int32_t* tickets, int32_t* vpage, int32_t* victims,
                          unsigned long long grid_last, bool early) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (early || pdl_enabled()) ? 1 : 0;  // a non-early launch waits at its top
    cudaLaunchKernelEx(&cfg, evict_score_kernel<SV, HOLES>, s, ts, ppc, scratch, tickets, vpage, victims, grid_last,
                       early ? 1 : 0);
}

template <int SV>
void launch_evict_score(dim3 grid, int threads, cudaStream_t st, const DevState& s, const TableSet& ts, int ppc,
                        double* scratch, int32_t* tickets, int32_t* vpage, int32_t* victims,
                        unsigned long long grid_last, bool early) {
    // hole-aware variant only after the table API made holes (no runtime check in the hot loop)
    if (s.holes_on)
        launch_evict_score_t<SV, true>(grid, threads, st, s, ts, ppc, scratch, tickets, vpage, victims, grid_last,
                                       early);
    else
        launch_evict_score_t<SV, false>(grid, threads, st, s, ts, ppc, scratch, tickets, vpage, victims, grid_last,
                                        early);
}

template <int SV>
void launch_append(int blocks, cudaStream_t st, const DevState& s, const TableSet& ts, const uint8_t* k,
                   const uint8_t* v, const int64_t* pos, unsigned long long* lb, unsigned long long* lbg,
                   LaunchCtl* ctl, int fast_ok,
                   unsigned long long ticket_base, int epoch) {
    launch_pdl(append_kernel<SV>, dim3(blocks), dim3(kAppendThreads), 0, st, s, ts, k, v, pos, lb, lbg, ctl,
               ticket_base, epoch, fast_ok);
}

void launch_evict_score_any(int variant, dim3 grid, int threads, cudaStream_t st, const DevState& s,
                            const TableSet& ts, int ppc, double* scratch, int32_t* tickets, int32_t* vpage,
                            int32_t* victims, unsigned long long grid_last, bool early) {
    PE_SCORE_DISPATCH(variant, (launch_evict_score<SV>(grid, threads, st, s, ts, ppc, scratch, tickets, vpage,
                                                        victims, grid_last, early)));
}

void launch_append_any(int variant, int blocks, cudaStream_t st, const DevState& s, const TableSet& ts,
                       const uint8_t* k, const uint8_t* v, const int64_t* pos, unsigned long long* lb,
                       unsigned long long* lbg,
                       LaunchCtl* ctl, unsigned long long ticket_base, int epoch, bool fast_ok) {
    PE_SCORE_DISPATCH(variant, (launch_append<SV>(blocks, st, s, ts, k, v, pos, lb, lbg, ctl, fast_ok ? 1 : 0,
                                                  ticket_base, epoch)));
}

// ---------------------------------------------------------------------------
// evict_cached_kernel (K2c): one warp per launch table; page means were
// cached when each page filled, so the decision reads N doubles (gathered
// through the block table) instead of N pages. Bit-identical to K2.
// Tables of up to 32*KR pages are handled in registers: the block-table row
// and the page means are loaded with two independent load levels, the argmin
// is a shuffle reduction, and free_page's left shift of the row is done with
// shuffles of the row held in registers (no dependent load chains).
template <int KR>
__device__ __forceinline__ void cached_evict_regs(const DevState& s, int t, int y, int32_t* vpage, int32_t* victims) {
    const int lane = threadIdx.x & 31;
    const int N = s.num_pages[t];
    int32_t* row = s.block_table + (int64_t)t * s.max_pages;
    int ids[KR];
    double sc[KR];
#pragma unroll
    for (int k = 0; k < KR; ++k) ids[k] = (lane + 32 * k < N) ? row[lane + 32 * k] : -1;
#pragma unroll
    for (int k = 0; k < KR; ++k) sc[k] = ids[k] >= 0 ? __ldcg(s.page_scores + ids[k]) : 0.0;
    // rank_pages (importance.cpp:62-75): strict <, ties -> smaller logical index
    double best = 0.0;
    int bj = 0x7FFFFFFF;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
        if (ids[k] >= 0 && (bj == 0x7FFFFFFF || sc[k] < best)) {
            best = sc[k];
            bj = lane + 32 * k;
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
    int victim_page = 0;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
        const int v = __shfl_sync(0xFFFFFFFFu, ids[k], victim & 31);
        if (k == (victim >> 5)) victim_page = v;
    }
    // free_page (block_table.cpp:21-31): entries after the victim move one left
#pragma unroll
    for (int k = 0; k < KR; ++k) {
        const int nxt_same = __shfl_down_sync(0xFFFFFFFFu, ids[k], 1);
        const int nxt_wrap = k + 1 < KR ? __shfl_sync(0xFFFFFFFFu, ids[k + 1 < KR ? k + 1 : k], 0) : -1;
        const int nxt = lane < 31 ? nxt_same : nxt_wrap;
        const int j = lane + 32 * k;
        if (j >= victim && j < N - 1) row[j] = nxt;
    }
    if (lane == 0) {
        row[N - 1] = -1;
        s.num_pages[t] = N - 1;
        s.retained[t] -= page_fill(s, victim_page, s.B);
        if (s.holes_on) s.holes[victim_page] = 0ull;
        s.newest_fill[t] = (N - 1 > 0) ? s.B : 0;
        vpage[t] = victim_page;
        if (victims) victims[y] = victim;
        atomicAdd(s.evict_count, 1ull);
    }
    __syncwarp();
}

// early (PDL, per-layer launches back to back, as K2's): everything up to the
// table's eviction touches only this launch's tables (vpage and scratch are
// indexed by table id); the settle ticket and the push wait for the
// previous launch.
__global__ void __launch_bounds__(256) evict_cached_kernel(DevState s, TableSet ts, double* scratch,
                                                           int32_t* vpage, int32_t* victims,
                                                           unsigned long long grid_last, int early) {
    if (!early) pdl_wait();
    pdl_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int y = blockIdx.x * 8 + wid;
    const int n = ts.size(s);
    if (y < n) {
        const int t = ts.table(s, y);
        if (!evict_triggered(s, t)) {
            if (lane == 0) {
                vpage[t] = -1;
                if (victims) victims[y] = -1;
            }
        } else if (s.max_pages <= 32 * 9) {
            cached_evict_regs<9>(s, t, y, vpage, victims);
        } else if (s.max_pages <= 32 * 16) {
            cached_evict_regs<16>(s, t, y, vpage, victims);
        } else {
            const int N = s.num_pages[t];
            const int32_t* row = s.block_table + (int64_t)t * s.max_pages;
            double* sc = scratch + (int64_t)t * s.max_pages;
            for (int j = lane; j < N; j += 32) sc[j] = s.page_scores[row[j]];
            __syncwarp();
            finalize_evict(s, t, y, N, sc, vpage + t, victims);
        }
    }
    if (early) pdl_wait();  // the previous launch's settle tickets and pushes come first
    push_victims_if_last(s, n, vpage, grid_last, min(8, n - static_cast<int>(blockIdx.x) * 8), &ts);
}

}  // namespace pe
