// K1: prefill prune+pack — scoring kernel + one thread-block cluster (8 CTAs) per table.
//
// Reference path (proj/core/): make_kv norms (kv_vector.hpp:36-48) ->
// EvictionPolicy::prefill_compress (policy.cpp:54-63) -> compress_by_score
// (policy.cpp:90-101): token_importance (importance.cpp:11-13) for every
// token, rank_tokens(k = L - C) (importance.cpp:41-60: k lowest by
// (score asc, position asc)), drop_positions (policy.cpp:75-86: survivors
// keep position order) -> append_token of every survivor
// (block_table.cpp:10-19, LIFO allocate page_pool.cpp:24-33).
//
// Device formulation (two kernels):
//  1. score   — prefill_score_kernel streams every token of every table of the
//               launch (lane pair per token, exact fp64 certificate scoring,
//               pe_score.cuh); key = IEEE bits of S (S >= +0 so the u64 order
//               is the double order), 8 B per token to a key buffer.
//  select/compact run in prefill_select_kernel, one cluster of 8 CTAs per
//  table, CTA r owning tokens [L*r/8, L*(r+1)/8) whose keys it loads to smem:
//  2. select  — cluster-wide MSB radix select (8-bit digits, histograms merged
//               through DSMEM) of the E-th smallest key: every key with a
//               smaller prefix is evicted; among keys equal to the final
//               prefix, the first k_rem in position order (the reference's
//               position tie rule).
//  3. compact — block scans + a DSMEM exchange of per-CTA counts give each
//               survivor its global rank q (position order) -> survivor list.
//  4. pack    — prefill_copy_kernel (warp per destination page): survivor q
//               goes to slot q%B of the table's (q/B)-th page; the
//               pages are the free-stack entries reserved in canonical order
//               by plan_prefill_kernel. Token scores and positions are stored
//               beside the page; full pages get their mean score cached.
#include <cooperative_groups.h>

#include "pe_kernels.cuh"
#include "pe_score.cuh"

namespace cg = cooperative_groups;

namespace pe {

__global__ void __launch_bounds__(1024) plan_prefill_kernel(DevState s, PrefillArgs a,
                                                             int32_t total_pages, LaunchCtl* ctl) {
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < a.n_tab; i += blockDim.x) {
        const int h = i % s.tab_heads;
        const int seq = a.seq_begin + i / s.tab_heads;
        const int t = (seq * s.n_layers + a.layer) * s.tab_heads + h;
        if (s.num_pages[t] != 0) atomicOr(&bad, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int top = *s.top;
        if (bad) {
            set_status(s.status, PE_INVALID_STATE);
            ctl->abort = 1;
        } else if (total_pages > top) {
            set_status(s.status, PE_POOL_EXHAUSTED);
            ctl->abort = 1;
        } else {
            ctl->abort = 0;
            ctl->pop_base = top;
            *s.top = top - total_pages;
        }
    }
}

// ---------------------------------------------------------------------------
// prefill_score_kernel: grid (ceil(maxL / 256), n_seqs of the launch), 4
// warps. The CTA scores tokens [256*bx, 256*bx+256) of one sequence for ALL
// its tables (heads): the input is token-major [tokens][heads][w], so the
// (token, head) rows of a token block are one contiguous span and every
// warp step (16 lane pairs = 16 consecutive (token, head) rows of K and of
// V) reads 4 KB of contiguous HBM.
template <int SV>
__global__ void __launch_bounds__(kPrefillThreads) prefill_score_kernel(DevState s, PrefillArgs a,
                                                                         const LaunchCtl* ctl) {
    if (ctl->abort) return;
    const int sq = blockIdx.y;  // sequence within the launch
    const int H = s.tab_heads;
    const int L = a.tab_len[sq * H];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    const int tok_lo = blockIdx.x * kScoreTokensPerCta;
    if (tok_lo >= L) return;
    const int tok_hi = min(L, tok_lo + kScoreTokensPerCta);
    const int64_t f_lo = (int64_t)tok_lo * H;
    const int64_t f_hi = (int64_t)tok_hi * H;
    const int64_t row0 = a.tab_tok0[sq * H] * H;  // first (token, head) row of the sequence
    const int64_t n_units = (f_hi - f_lo + 15) / 16;
    for (int64_t u = wid; u < n_units; u += nw) {
        const int64_t f = f_lo + u * 16 + (lane >> 1);
        const bool valid = f < f_hi;
        const int64_t off = (row0 + f) * s.row_bytes;
        const double S = pair_token_score<SV>(a.k + off, a.v + off, valid, s.w, s.dtype);
        if (valid && (lane & 1) == 0) {
            const int tok = static_cast<int>(f / H);
            const int h = static_cast<int>(f - (int64_t)tok * H);
            a.keys[a.tab_keybase[sq * H + h] + tok] = static_cast<unsigned long long>(__double_as_longlong(S));
        }
    }
}

template <int SV>
static void launch_score(dim3 grid, cudaStream_t st, const DevState& s, const PrefillArgs& a, const LaunchCtl* ctl) {
    prefill_score_kernel<SV><<<grid, kPrefillThreads, 0, st>>>(s, a, ctl);
}

void launch_prefill_score_any(int variant, dim3 grid, cudaStream_t st, const DevState& s, const PrefillArgs& a,
                              const LaunchCtl* ctl) {
    PE_SCORE_DISPATCH(variant, (launch_score<SV>(grid, st, s, a, ctl)));
}

// Warp-aggregated shared-memory histogram increment (many keys share a
// digit: S values of one table are concentrated).
__device__ __forceinline__ void hist_add(uint32_t* hb, uint32_t bin, bool active) {
    const uint32_t am = __ballot_sync(0xFFFFFFFFu, active);
    if (!active) return;
    const uint32_t peers = __match_any_sync(am, bin);
    if ((threadIdx.x & 31) == (__ffs(peers) - 1)) atomicAdd(&hb[bin], __popc(peers));
}

__global__ void __cluster_dims__(kPrefillCluster, 1, 1) __launch_bounds__(kPackThreads)
    prefill_select_kernel(DevState s, PrefillArgs a, const LaunchCtl* ctl) {
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint32_t hist[2][256];
    __shared__ uint32_t tot[256];
    __shared__ int scan_sm[33];
    __shared__ int xchg[2];
    __shared__ int bc[8];

    if (ctl->abort) return;  // uniform for the whole grid
    const int CL = kPrefillCluster;
    const int r = static_cast<int>(cluster.block_rank());
    const int i = blockIdx.y;
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const int lane = tid & 31;
    const int wid = tid >> 5;
    const int nw = nthr >> 5;

    const int L = a.tab_len[i];
    const int keep = (s.policy == PE_POLICY_PAGED_EVICTION && L > s.C) ? s.C : L;
    const int E = L - keep;
    const int lo = static_cast<int>((int64_t)L * r / CL);
    const int hi = static_cast<int>((int64_t)L * (r + 1) / CL);
    const int n = hi - lo;
    const int h = i % s.tab_heads;
    const int seq = a.seq_begin + i / s.tab_heads;
    const int t = (seq * s.n_layers + a.layer) * s.tab_heads + h;

    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);
    // survivor q of table i (position order) -> its token index
    int32_t* surv = a.surv + (int64_t)a.tab_pagebase[i] * s.B;

    // ---------------------------------------------------------------- 1. keys -> smem
    {
        const unsigned long long* g = a.keys + a.tab_keybase[i] + lo;
        for (int j = tid; j < n; j += nthr) keys[j] = __ldcs(g + j);
    }
    __syncthreads();

    // ---------------------------------------------------------------- 2. select
    int k_rem = 0;
    int final_shift = 64;
    unsigned long long prefix = 0;
    if (E > 0) {
        k_rem = E;
        int shift = 64;
        for (int pass = 0; pass < 8; ++pass) {
            shift -= 8;
            uint32_t* hb = hist[pass & 1];
            for (int b = tid; b < 256; b += nthr) hb[b] = 0;
            __syncthreads();
            const int n_round = (n + nthr - 1) / nthr * nthr;
            for (int j = tid; j < n_round; j += nthr) {
                const unsigned long long key = j < n ? keys[j] : 0ull;
                const bool match = j < n && ((pass == 0) || ((key >> (shift + 8)) == prefix));
                hist_add(hb, static_cast<uint32_t>((key >> shift) & 255u), match);
            }
            cluster.sync();
            for (int b = tid; b < 256; b += nthr) {
                uint32_t acc = 0;
                for (int rr = 0; rr < CL; ++rr) acc += cluster.map_shared_rank(hb, rr)[b];
                tot[b] = acc;
            }
            __syncthreads();
            if (wid == 0) {
                uint32_t part[8];
                uint32_t lsum = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    part[q] = tot[lane * 8 + q];
                    lsum += part[q];
                }
                const int incl = warp_incl_scan(static_cast<int>(lsum));
                int cum = incl - static_cast<int>(lsum);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (cum < k_rem && k_rem <= cum + static_cast<int>(part[q])) {
                        bc[0] = lane * 8 + q;
                        bc[1] = cum;
                    }
                    cum += static_cast<int>(part[q]);
                }
            }
            __syncthreads();
            const int d = bc[0];
            k_rem -= bc[1];
            prefix = (prefix << 8) | static_cast<unsigned long long>(d);
            final_shift = shift;
            const bool done = static_cast<int>(tot[d]) == k_rem;
            __syncthreads();
            if (done) break;
        }
    }

    // ---------------------------------------------------------------- 3. compact
    auto classify = [&](unsigned long long key, bool& less, bool& tie) {
        if (E == 0) {
            less = false;
            tie = false;
            return;
        }
        const unsigned long long top = key >> final_shift;
        less = top < prefix;
        tie = top == prefix;
    };
    const int seg = (n + nthr - 1) / nthr;
    const int a0 = min(n, tid * seg);
    const int a1 = min(n, a0 + seg);
    int less_t = 0, tie_t = 0;
    for (int j = a0; j < a1; ++j) {
        bool l, tt;
        classify(keys[j], l, tt);
        less_t += l;
        tie_t += tt;
    }
    int less_cta, tie_cta;
    block_excl_scan(less_t, scan_sm, &less_cta);
    const int tie_before = block_excl_scan(tie_t, scan_sm, &tie_cta);
    if (tid == 0) {
        xchg[0] = less_cta;
        xchg[1] = tie_cta;
    }
    cluster.sync();
    if (tid == 0) {
        int tie_base = 0, surv_base = 0, kept_me = 0, tb = 0;
        for (int rr = 0; rr < CL; ++rr) {
            const int* rx = cluster.map_shared_rank(xchg, rr);
            const int l_rr = rx[0];
            const int t_rr = rx[1];
            const int n_rr = static_cast<int>((int64_t)L * (rr + 1) / CL - (int64_t)L * rr / CL);
            const int ev_ties = max(0, min(k_rem - tb, t_rr));
            const int kept = n_rr - l_rr - ev_ties;
            if (rr < r) {
                tie_base += t_rr;
                surv_base += kept;
            }
            if (rr == r) kept_me = kept;
            tb += t_rr;
        }
        bc[2] = tie_base;
        bc[3] = surv_base;
        bc[4] = kept_me;
    }
    __syncthreads();
    const int tie_base = bc[2];
    const int surv_base = bc[3];
    const int kept_me = bc[4];
    const int my_tie0 = tie_base + tie_before;
    const int ev_ties_t = max(0, min(k_rem - my_tie0, tie_t));
    const int keep_t = (a1 - a0) - less_t - ev_ties_t;
    int keep_cta;
    int q_local = block_excl_scan(keep_t, scan_sm, &keep_cta);
    {
        int tr = my_tie0;
        for (int j = a0; j < a1; ++j) {
            bool l, tt;
            classify(keys[j], l, tt);
            const bool evict = l || (tt && tr < k_rem);
            tr += tt;
            if (!evict) surv[surv_base + q_local++] = lo + j;
        }
    }
    __syncthreads();

    // ---------------------------------------------------------------- table metadata
    const int B = s.B;
    const int n_pages = (keep + B - 1) / B;
    if (r == 0) {
        const int pop_base = ctl->pop_base;
        const int pagebase = a.tab_pagebase[i];
        for (int p = tid; p < n_pages; p += nthr) {
            s.block_table[(int64_t)t * s.max_pages + p] = s.stack[pop_base - 1 - (pagebase + p)];
        }
        if (tid == 0) {
            s.num_pages[t] = n_pages;
            s.newest_fill[t] = keep - (n_pages - 1) * B;
            s.retained[t] = keep;
            if (a.evicted_counts) a.evicted_counts[i] = E;
        }
    }
    // no CTA may leave while cluster peers can still read its shared memory
    cluster.sync();
    (void)kept_me;
    (void)lane;
    (void)wid;
    (void)nw;
}

// ---------------------------------------------------------------------------
// prefill_copy_kernel: one warp per destination page. Lane pair r moves the
// page's slot r: survivor q = page*B + r (position order) -> K and V rows
// with 256-bit loads/stores, position and cached score beside the page; the
// warp then sums the B scores in slot order (page_score, importance.cpp:19-30)
// for a full page. Grid (ceil(max pages / 4), n_tab).
__global__ void __launch_bounds__(128) prefill_copy_kernel(DevState s, PrefillArgs a, const LaunchCtl* ctl) {
    if (ctl->abort) return;
    const int i = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int j = blockIdx.x * (blockDim.x >> 5) + wid;
    const int L = a.tab_len[i];
    const int keep = (s.policy == PE_POLICY_PAGED_EVICTION && L > s.C) ? s.C : L;
    const int B = s.B;
    const int n_pages = (keep + B - 1) / B;
    if (j >= n_pages) return;
    const int h = i % s.tab_heads;
    const int64_t row0 = (a.tab_tok0[i] * s.tab_heads + h) * (int64_t)s.row_bytes;
    const uint8_t* kbase = a.k + row0;
    const uint8_t* vbase = a.v + row0;
    const int pagebase = a.tab_pagebase[i];
    const int page = s.stack[ctl->pop_base - 1 - (pagebase + j)];
    const int32_t* surv = a.surv + (int64_t)pagebase * B;
    const unsigned long long* keys = a.keys + a.tab_keybase[i];
    const int qq = lane & 1;
    double sum = 0.0;
    for (int s0 = 0; s0 < B; s0 += 16) {
        const int slot = s0 + (lane >> 1);
        const int q = j * B + slot;
        const bool valid = slot < B && q < keep;
        const int tok = valid ? __ldg(surv + q) : 0;
        double S = 0.0;
        if (valid) {
            const uint8_t* ks = kbase + (int64_t)tok * a.token_stride;
            const uint8_t* vs = vbase + (int64_t)tok * a.token_stride;
            uint8_t* kd = s.pages + (((int64_t)page * 2 + 0) * B + slot) * s.pitch;
            uint8_t* vd = s.pages + (((int64_t)page * 2 + 1) * B + slot) * s.pitch;
            if ((s.row_bytes & 63) == 0) {
                for (int off = qq * 32; off < s.row_bytes; off += 64) stg256(kd + off, ldg256(ks + off));
                for (int off = qq * 32; off < s.row_bytes; off += 64) stg256(vd + off, ldg256(vs + off));
            } else {
                for (int off = qq * 16; off < s.row_bytes; off += 32)
                    *reinterpret_cast<uint4*>(kd + off) = __ldcs(reinterpret_cast<const uint4*>(ks + off));
                for (int off = qq * 16; off < s.row_bytes; off += 32)
                    *reinterpret_cast<uint4*>(vd + off) = __ldcs(reinterpret_cast<const uint4*>(vs + off));
            }
            S = __longlong_as_double(static_cast<long long>(__ldg(keys + tok)));
            if (qq == 0) {
                s.positions[(int64_t)page * B + slot] = tok;
                s.token_scores[(int64_t)page * B + slot] = S;
            }
        }
        const int ns = min(16, B - s0);
        for (int u = 0; u < ns; ++u) sum += __shfl_sync(0xFFFFFFFFu, S, 2 * u);
    }
    if (lane == 0 && (j + 1) * B <= keep) s.page_scores[page] = sum / static_cast<double>(B);
}

}  // namespace pe
