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
//  2. select  — cluster-wide MSB radix select (8-bit digits after the common
//               prefix of the cluster min/max, candidate lists compacted each
//               pass, histograms merged through DSMEM) of the E-th smallest
//               key: every key with a
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
#include <cstdlib>
#include <cstring>

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
//
// SK (staged keys, a.score_tokens * heads <= kScoreKeysMax): the CTA's keys
// are gathered in shared memory and written per table as one contiguous run
// of score_tokens keys (full 32-byte sectors) instead of 2-key pieces from
// each warp step.
template <int SV, bool SK>
__global__ void __launch_bounds__(kPrefillThreads) prefill_score_kernel(DevState s, PrefillArgs a,
                                                                         const LaunchCtl* ctl) {
    __shared__ unsigned long long skeys[SK ? kScoreKeysMax : 1];
    if (ctl->abort) return;
    // 2-D grid (token block, sequence), or a compact 1-D grid over the
    // non-empty blocks of a call with mixed lengths (a.score_items)
    int sq = blockIdx.y, bx = blockIdx.x;  // sequence within the launch, token block
    if (a.score_items != nullptr) {
        const int d = __ldg(a.score_items + blockIdx.x);
        sq = (d >> 16) - a.item_seq0;
        bx = d & 0xFFFF;
    }
    const int H = s.tab_heads;
    const int L = a.tab_len[sq * H];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    const int tok_lo = bx * a.score_tokens;
    if (tok_lo >= L) return;
    const int tok_hi = min(L, tok_lo + a.score_tokens);
    const int64_t f_lo = (int64_t)tok_lo * H;
    const int64_t f_hi = (int64_t)tok_hi * H;
    const int64_t row0 = a.tab_tok0[sq * H] * H;  // first (token, head) row of the sequence
    const int64_t n_units = (f_hi - f_lo + 15) / 16;
    // a sequence whose tables keep every token (L <= C, or a non-evicting
    // policy) needs no select: its rows go straight into their pages here
    // (position p -> slot p % B of the table's (p / B)-th page), so they are
    // read once instead of twice; the copy kernel skips these tables
    const bool ident = SK && a.direct_identity &&
                       !(s.policy == PE_POLICY_PAGED_EVICTION && L > s.C);  // block-uniform
    const int B = s.B;
    for (int64_t u = wid; u < n_units; u += nw) {
        const int64_t f = f_lo + u * 16 + (lane >> 1);
        const bool valid = f < f_hi;
        const int64_t off = (row0 + f) * s.row_bytes;
        uint8_t* kd = nullptr;
        uint8_t* vd = nullptr;
        if (ident && valid) {
            const int tok = static_cast<int>(f / H);
            const int h = static_cast<int>(f - (int64_t)tok * H);
            const int page = s.stack[ctl->pop_base - 1 - (a.tab_pagebase[sq * H + h] + tok / B)];
            kd = s.pages + (((int64_t)page * 2 + 0) * B + tok % B) * s.pitch;
            vd = s.pages + (((int64_t)page * 2 + 1) * B + tok % B) * s.pitch;
        }
        const double S = pair_token_score<SV>(a.k + off, a.v + off, valid, s.w, s.dtype, kd, vd);
        if (valid && (lane & 1) == 0) {
            const unsigned long long key = static_cast<unsigned long long>(__double_as_longlong(S));
            if constexpr (SK) {
                skeys[f - f_lo] = key;  // (token, head) order
            } else {
                const int tok = static_cast<int>(f / H);
                const int h = static_cast<int>(f - (int64_t)tok * H);
                a.keys[a.tab_keybase[sq * H + h] + tok] = key;
            }
        }
    }
    if constexpr (SK) {
        __syncthreads();
        const int nt = tok_hi - tok_lo;
        for (int x = threadIdx.x; x < nt * H; x += blockDim.x) {  // head-major: one run per table
            const int h = x / nt, j = x - h * nt;
            a.keys[a.tab_keybase[sq * H + h] + tok_lo + j] = skeys[j * H + h];
        }
        if (ident) {
            // positions and cached token scores of the packed slots, and the
            // mean of every full page (slot-order sum / B, importance.cpp:19-30;
            // the block starts on a page boundary: score_tokens % B == 0)
            const int32_t* stk = s.stack + ctl->pop_base - 1;
            for (int x = threadIdx.x; x < nt * H; x += blockDim.x) {
                const int h = x / nt, j = x - h * nt;
                const int tok = tok_lo + j;
                const int page = stk[-(a.tab_pagebase[sq * H + h] + tok / B)];
                s.positions[(int64_t)page * B + tok % B] = tok;
                s.token_scores[(int64_t)page * B + tok % B] = __longlong_as_double(static_cast<long long>(skeys[j * H + h]));
            }
            const int pages_here = (nt + B - 1) / B;
            for (int x = threadIdx.x; x < pages_here * H; x += blockDim.x) {
                const int h = x / pages_here, pj = x - h * pages_here;
                if (tok_lo + (pj + 1) * B > L) continue;  // the newest, partial page has no cached mean
                double sum = 0.0;
                for (int sl = 0; sl < B; ++sl)
                    sum += __longlong_as_double(static_cast<long long>(skeys[(pj * B + sl) * H + h]));
                const int page = stk[-(a.tab_pagebase[sq * H + h] + tok_lo / B + pj)];
                s.page_scores[page] = sum / static_cast<double>(B);
            }
        }
    }
}

template <int SV>
static void launch_score(dim3 grid, cudaStream_t st, const DevState& s, const PrefillArgs& a, const LaunchCtl* ctl) {
    const char* sk = std::getenv("PE_SCORE_STAGED_KEYS");
    if ((int64_t)a.score_tokens * s.tab_heads <= kScoreKeysMax && !(sk != nullptr && std::strcmp(sk, "0") == 0))
        prefill_score_kernel<SV, true><<<grid, kPrefillThreads, 0, st>>>(s, a, ctl);
    else
        prefill_score_kernel<SV, false><<<grid, kPrefillThreads, 0, st>>>(s, a, ctl);
}

void launch_prefill_score_any(int variant, dim3 grid, cudaStream_t st, const DevState& s, const PrefillArgs& a,
                              const LaunchCtl* ctl) {
    PE_SCORE_DISPATCH(variant, (launch_score<SV>(grid, st, s, a, ctl)));
}

// Warp-interleaved position-order sweeps over n positions (conflict-free
// shared-memory access): warp w owns positions [w*span, (w+1)*span), visited
// in rounds of 32 consecutive positions (lane = position % 32); ranks come
// from ballots, so the order is exactly ascending position.
__device__ __forceinline__ int sweep_span(int n) {
    const int nw = blockDim.x >> 5;
    return ((n + nw * 32 - 1) / (nw * 32)) * 32;
}

template <typename F>
__device__ __forceinline__ void sweep_count(int n, F classify, int* warp_less, int* warp_tie) {
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int span = sweep_span(n);
    const int end = min(n, (wid + 1) * span);
    int lc = 0, tc = 0;
    for (int base = wid * span; base < end; base += 32) {
        const int p = base + lane;
        bool l = false, t = false;
        if (p < end) classify(p, l, t);
        lc += __popc(__ballot_sync(0xFFFFFFFFu, l));
        tc += __popc(__ballot_sync(0xFFFFFFFFu, t));
    }
    if (lane == 0) {
        warp_less[wid] = lc;
        warp_tie[wid] = tc;
    }
}

// Turns per-warp (less, tie) counts into per-warp tie / survivor bases (one
// thread), given the CTA's first tie rank and first survivor index.
__device__ __forceinline__ void sweep_bases(int n, int k_rem, int tie0, int surv0, const int* warp_less,
                                            const int* warp_tie, int* tie_base, int* keep_base) {
    const int nw = blockDim.x >> 5;
    const int span = sweep_span(n);
    int tb = tie0, kb = surv0;
    for (int w = 0; w < nw; ++w) {
        const int nwn = max(0, min(n, (w + 1) * span) - w * span);
        tie_base[w] = tb;
        keep_base[w] = kb;
        const int ev = max(0, min(k_rem - tb, warp_tie[w]));
        kb += nwn - warp_less[w] - ev;
        tb += warp_tie[w];
    }
}

template <typename F, typename EMIT>
__device__ __forceinline__ void sweep_emit(int n, F classify, int k_rem, const int* tie_base, const int* keep_base,
                                           EMIT emit) {
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int span = sweep_span(n);
    const int end = min(n, (wid + 1) * span);
    const unsigned lt = (1u << lane) - 1u;
    int tie_run = tie_base[wid];
    int keep_run = keep_base[wid];
    for (int base = wid * span; base < end; base += 32) {
        const int p = base + lane;
        bool l = false, t = false;
        if (p < end) classify(p, l, t);
        const unsigned tb = __ballot_sync(0xFFFFFFFFu, t);
        const bool evict = l || (t && tie_run + __popc(tb & lt) < k_rem);
        tie_run += __popc(tb);
        const bool keep = p < end && !evict;
        const unsigned kb = __ballot_sync(0xFFFFFFFFu, keep);
        if (keep) emit(keep_run + __popc(kb & lt), p);
        keep_run += __popc(kb);
    }
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
    __shared__ int xchg[2];
    __shared__ int bc[8];

    if (ctl->abort) return;  // uniform for the whole grid
    if (a.tab_len[blockIdx.y] <= a.cluster_len_min) return;  // mixed lengths: the CTA select's table (whole cluster)
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
    // candidate index lists (double-buffered) for the radix passes
    uint16_t* cand[2] = {reinterpret_cast<uint16_t*>(smem + (size_t)a.chunk_cap * 8),
                         reinterpret_cast<uint16_t*>(smem + (size_t)a.chunk_cap * 10)};
    __shared__ unsigned long long mm[2];
    __shared__ int cand_n[2];
    __shared__ uint32_t wh[8 * 256];  // per-warp histogram copies (reduced into hb)
    // survivor q of table i (position order) -> its token index
    int32_t* surv = a.surv + (int64_t)a.tab_pagebase[i] * s.B;

    // ---------------------------------------------------------------- 1. keys -> smem (+ min/max)
    unsigned long long kmin = ~0ull, kmax = 0ull;
    {
        const unsigned long long* g = a.keys + a.tab_keybase[i] + lo;
        for (int j0 = tid; j0 < n; j0 += 8 * nthr) {  // 8 independent loads in flight per thread
            unsigned long long kv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) kv[u] = (j0 + u * nthr < n) ? __ldcs(g + j0 + u * nthr) : 0ull;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (j0 + u * nthr < n) {
                    keys[j0 + u * nthr] = kv[u];
                    kmin = min(kmin, kv[u]);
                    kmax = max(kmax, kv[u]);
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xFFFFFFFFu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xFFFFFFFFu, kmax, o));
    }
    if (tid == 0) {
        mm[0] = ~0ull;
        mm[1] = 0ull;
    }
    __syncthreads();
    if (lane == 0) {
        atomicMin(&mm[0], kmin);
        atomicMax(&mm[1], kmax);
    }
    __syncthreads();

    // ---------------------------------------------------------------- 2. select
    // MSB radix select of the E-th smallest key. All keys share the common
    // prefix of the cluster-wide (min, max), so the passes start right after
    // it; each pass histograms only the candidates still matching the prefix
    // (compacted index lists), merged across the cluster through DSMEM.
    int k_rem = 0;
    int final_shift = 64;
    unsigned long long prefix = 0;
    if (E > 0) {
        k_rem = E;
        cluster.sync();
        unsigned long long gmin = ~0ull, gmax = 0ull;
        for (int rr = 0; rr < CL; ++rr) {
            const unsigned long long* rm = cluster.map_shared_rank(mm, rr);
            gmin = min(gmin, rm[0]);
            gmax = max(gmax, rm[1]);
        }
        const int cpl = (gmin == gmax) ? 64 : __clzll(gmin ^ gmax);
        int bitpos = 64 - cpl;  // unresolved low bits
        prefix = cpl == 0 ? 0ull : (cpl == 64 ? gmin : (gmin >> bitpos));
        final_shift = bitpos;
        int pass = 0;
        while (bitpos > 0) {
            const int bits = min(8, bitpos);
            const int shift = bitpos - bits;
            const unsigned long long dmask = (1ull << bits) - 1ull;
            uint32_t* hb = hist[pass & 1];
            uint16_t* out = cand[pass & 1];
            const uint16_t* in = cand[(pass & 1) ^ 1];
            const int n_in = pass == 0 ? n : cand_n[(pass & 1) ^ 1];
            for (int b = tid; b < 8 * 256; b += nthr) wh[b] = 0;
            __syncthreads();
            const int n_round = (n_in + nthr - 1) / nthr * nthr;
            for (int x = tid; x < n_round; x += nthr) {
                const bool act = x < n_in;
                const int j = act ? (pass == 0 ? x : in[x]) : 0;
                const unsigned long long key = act ? keys[j] : 0ull;
                hist_add(wh + (wid & 7) * 256, static_cast<uint32_t>((key >> shift) & dmask), act);
            }
            __syncthreads();
            for (int b = tid; b < 256; b += nthr) {
                uint32_t acc = 0;
#pragma unroll
                for (int c = 0; c < 8; ++c) acc += wh[c * 256 + b];
                hb[b] = acc;
            }
            cluster.sync();
            for (int b = tid; b < 256; b += nthr) {
                uint32_t acc = 0;
#pragma unroll
                for (int rr = 0; rr < kPrefillCluster; ++rr) acc += cluster.map_shared_rank(hb, rr)[b];
                tot[b] = acc;
            }
            if (tid == 0) cand_n[pass & 1] = 0;
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
            prefix = (prefix << bits) | static_cast<unsigned long long>(d);
            final_shift = shift;
            bitpos = shift;
            if (static_cast<int>(tot[d]) == k_rem || bitpos == 0) break;
            // compact the candidates that carry the chosen digit
            for (int x = tid; x < n_round; x += nthr) {
                const bool act = x < n_in;
                const int j = act ? (pass == 0 ? x : in[x]) : 0;
                const bool keep_c = act && static_cast<int>((keys[j] >> shift) & dmask) == d;
                const unsigned bal = __ballot_sync(0xFFFFFFFFu, keep_c);
                int base = 0;
                if (lane == 0 && bal) base = atomicAdd(&cand_n[pass & 1], __popc(bal));
                base = __shfl_sync(0xFFFFFFFFu, base, 0);
                if (keep_c) out[base + __popc(bal & ((1u << lane) - 1u))] = static_cast<uint16_t>(j);
            }
            __syncthreads();
            ++pass;
        }
    }

    // ---------------------------------------------------------------- 3. compact
    __shared__ int w_less[32], w_tie[32], w_tieb[32], w_keepb[32];
    auto classify = [&](int j, bool& less, bool& tie) {
        if (E == 0) {
            less = false;
            tie = false;
            return;
        }
        const unsigned long long top = keys[j] >> final_shift;
        less = top < prefix;
        tie = top == prefix;
    };
    sweep_count(n, classify, w_less, w_tie);
    __syncthreads();
    if (tid == 0) {
        int lc = 0, tc = 0;
        for (int w = 0; w < nw; ++w) {
            lc += w_less[w];
            tc += w_tie[w];
        }
        xchg[0] = lc;
        xchg[1] = tc;
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
        bc[4] = kept_me;
        sweep_bases(n, k_rem, tie_base, surv_base, w_less, w_tie, w_tieb, w_keepb);
    }
    __syncthreads();
    const int kept_me = bc[4];
    sweep_emit(n, classify, k_rem, w_tieb, w_keepb, [&](int q, int j) { surv[q] = lo + j; });
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
// prefill_select_cta_kernel: the select/compact step for tables of up to
// kSelectCtaMaxLen tokens with ONE CTA (1024 threads) per table and no
// cluster barriers. The high 32 bits of every key live in shared memory
// (the order of the high words is the order of the keys' high halves);
// radix passes of 11-bit digits after the common prefix of (min, max) run
// on them with block barriers only. If the boundary high word is shared by
// several keys, their low words (read from global memory, only for those
// keys) are resolved with further passes. Then one position-order sweep
// (block scans) emits the survivors. Same decisions as the cluster kernel.
__device__ __forceinline__ void reduce_hist_copies(const uint32_t* copies, uint32_t* out, int nbins, int ncopies) {
    for (int b = threadIdx.x; b < 2048; b += blockDim.x) {
        uint32_t acc = 0;
        if (b < nbins)
            for (int c = 0; c < ncopies; ++c) acc += copies[c * 2048 + b];
        out[b] = acc;
    }
    __syncthreads();
}

__device__ __forceinline__ int block_find_digit(const uint32_t* hist, int nbins, int k_rem, int* bc, int* scan_sm) {
    // exclusive scan over bins (2 per thread for 2048 bins / 1024 threads)
    const int per = (nbins + blockDim.x - 1) / blockDim.x;
    const int b0 = min(nbins, (int)threadIdx.x * per);
    const int b1 = min(nbins, b0 + per);
    int local = 0;
    for (int b = b0; b < b1; ++b) local += static_cast<int>(hist[b]);
    int total;
    int cum = block_excl_scan(local, scan_sm, &total);
    for (int b = b0; b < b1; ++b) {
        const int c = static_cast<int>(hist[b]);
        if (cum < k_rem && k_rem <= cum + c) {
            bc[0] = b;
            bc[1] = cum;
            bc[2] = c;
        }
        cum += c;
    }
    __syncthreads();
    return bc[0];
}

// Select of launch table i by the whole CTA (1024 threads); `smem` is the
// dynamic shared memory (hi words, histogram copies, candidates).
// SMEM_HI: the table's high key words are held in shared memory (tables up to
// kSelectCtaMaxLen tokens); otherwise every pass reads them from the keys in
// global memory (tables of any length, e.g. cfg5's 128K-token tables), with a
// larger candidate list in the shared memory the hi words would have used.
template <bool SMEM_HI>
__device__ __noinline__ void select_table_cta(const DevState& s, const PrefillArgs& a, int i, uint8_t* smem,
                                              const LaunchCtl* ctl) {
    __shared__ uint32_t hist[2048];  // reduced histogram
    __shared__ int scan_sm[33];
    __shared__ int bc[4];
    __shared__ unsigned int mm[2];
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const int L = a.tab_len[i];
    const int keep = (s.policy == PE_POLICY_PAGED_EVICTION && L > s.C) ? s.C : L;
    const int E = L - keep;
    const int h = i % s.tab_heads;
    const int seq = a.seq_begin + i / s.tab_heads;
    const int t = (seq * s.n_layers + a.layer) * s.tab_heads + h;
    const int B = s.B;
    uint32_t* hi = reinterpret_cast<uint32_t*>(smem);  // SMEM_HI only
    const int cand_cap = SMEM_HI ? kSelCandCap : a.cand_cap;
    // kSelHistCopies private histograms (warp w -> copy w % kSelHistCopies):
    // the early digits of a table's keys are concentrated in a few bins, so a
    // single histogram would serialise every warp's atomics on them
    uint32_t* hcopy =
        reinterpret_cast<uint32_t*>(SMEM_HI ? smem + (((size_t)a.chunk_cap * 4 + 15) & ~size_t(15)) : smem);
    uint32_t* my_hist = hcopy + ((threadIdx.x >> 5) % kSelHistCopies) * 2048;
    int32_t* cand = reinterpret_cast<int32_t*>(hcopy + kSelHistCopies * 2048);  // [cand_cap]
    // streamed select: one eviction bit per position (after the candidates)
    // when the table fits a.bits_cap — the windowed path then classifies and
    // emits from shared memory instead of re-reading every key
    uint32_t* evbits = reinterpret_cast<uint32_t*>(cand + cand_cap);
    const unsigned long long* gk = a.keys + a.tab_keybase[i];
    auto HI = [&](int j) -> uint32_t {
        if constexpr (SMEM_HI) return hi[j];
        else return static_cast<uint32_t>(__ldcg(gk + j) >> 32);
    };
    int32_t* surv = a.surv + (int64_t)a.tab_pagebase[i] * B;

    // ---- 0. pivot window from a sorted sample of 1024 high words: every key
    // whose high word lies in [p_lo, p_hi] is a candidate for the boundary,
    // the rest are counted as below / above during the load. When the E-th
    // key falls inside the window (the common case), the radix passes visit
    // only the candidates; otherwise the plain full-table passes run.
    const bool sampled = E > 0 && L >= 8192;
    const bool bits = !SMEM_HI && sampled && L <= a.bits_cap;
    unsigned int p_lo = 0u, p_hi = 0xFFFFFFFFu;
    uint32_t* seg = hcopy;  // per-warp candidate segments during the load
    constexpr int kSegCap = kSelHistCopies * 2048 / 32;
    if (sampled) {
        uint32_t* samp = hist;
        // bitonic sort of one sample per thread: partner distances >= 32 go
        // through shared memory (15 barrier stages for 1024), shorter ones are
        // warp shuffles on the value held in a register
        uint32_t x = static_cast<uint32_t>(__ldcg(gk + (int)(((int64_t)tid * L) / nthr)) >> 32);
        for (int k = 2; k <= nthr; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                const bool up = (tid & k) == 0;
                if (j >= 32) {
                    samp[tid] = x;
                    __syncthreads();
                    const uint32_t y = samp[tid ^ j];
                    __syncthreads();
                    const bool lower = (tid & j) == 0;
                    x = (lower == up) ? min(x, y) : max(x, y);
                } else {
                    const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, j);
                    const bool lower = (tid & j) == 0;
                    x = (lower == up) ? min(x, y) : max(x, y);
                }
            }
        }
        samp[tid] = x;
        __syncthreads();
        const int r = (int)(((int64_t)E * nthr) / L);
        const int win = nthr / 32 + 8;  // ~3.5 sigma of the sample quantile
        const int lo_i = r - win, hi_i = r + win;
        p_lo = lo_i <= 0 ? 0u : samp[lo_i];
        p_hi = hi_i >= nthr - 1 ? 0xFFFFFFFFu : samp[hi_i];
        __syncthreads();
    }

    // ---- 1. high words -> smem, min/max (+ window counts and candidates)
    unsigned int hmin = 0xFFFFFFFFu, hmax = 0u;
    int n_below = 0, seg_n = 0;
    const int lane_id = tid & 31, warp_id = tid >> 5;
    // warp w loads the position span the sweeps give it ([w*span, (w+1)*span)),
    // so its below-window count is already the sweep's per-warp "less" count
    const int wspan = sweep_span(L);
    const int w_beg = min(L, warp_id * wspan), w_end = min(L, w_beg + wspan);
    for (int j0 = w_beg; j0 < w_end; j0 += 8 * 32) {  // 8 independent loads in flight per thread
        unsigned long long kv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = j0 + u * 32 + lane_id;
            kv[u] = j < w_end ? __ldcs(gk + j) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = j0 + u * 32 + lane_id;
            const bool in = j < w_end;
            const uint32_t w = static_cast<uint32_t>(kv[u] >> 32);
            if (in) {
                if constexpr (SMEM_HI) hi[j] = w;
                hmin = min(hmin, w);
                hmax = max(hmax, w);
            }
            if (sampled) {
                if (bits) {
                    // below-window keys are evicted: one bitmap word per 32
                    // positions (spans are 32-aligned, lane = position % 32)
                    const unsigned bm = __ballot_sync(0xFFFFFFFFu, in && w < p_lo);
                    if (lane_id == 0 && j0 + u * 32 < w_end) evbits[(j0 + u * 32) >> 5] = bm;
                }
                n_below += in && w < p_lo;
                const bool c = in && w >= p_lo && w <= p_hi;
                const unsigned m = __ballot_sync(0xFFFFFFFFu, c);
                const int at = seg_n + __popc(m & ((1u << lane_id) - 1u));
                if (c && at < kSegCap) seg[warp_id * kSegCap + at] = j;
                seg_n += __popc(m);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        hmin = min(hmin, __shfl_xor_sync(0xFFFFFFFFu, hmin, o));
        hmax = max(hmax, __shfl_xor_sync(0xFFFFFFFFu, hmax, o));
        n_below += __shfl_xor_sync(0xFFFFFFFFu, n_below, o);
    }
    __shared__ int w_below[32], w_seg[32], win_ok, n_cand, below_sum;
    if (tid == 0) {
        mm[0] = 0xFFFFFFFFu;
        mm[1] = 0u;
    }
    __syncthreads();
    if ((tid & 31) == 0) {
        atomicMin(&mm[0], hmin);
        atomicMax(&mm[1], hmax);
        w_below[warp_id] = n_below;
        w_seg[warp_id] = seg_n;
    }
    __syncthreads();
    int below_total = 0;
    if (sampled) {
        if (tid == 0) {
            int b = 0, c = 0, over = 0;
            for (int w = 0; w < (nthr >> 5); ++w) {
                b += w_below[w];
                over |= w_seg[w] > kSegCap;
                c += w_seg[w];
            }
            win_ok = !over && c <= cand_cap && b < E && E <= b + c;
            below_sum = b;
            n_cand = c;
        }
        __syncthreads();
        below_total = below_sum;
        if (win_ok) {
            // contiguous candidate list (warp segments in warp order)
            int off = 0;
            for (int w = 0; w < warp_id; ++w) off += w_seg[w];
            for (int x = lane_id; x < w_seg[warp_id]; x += 32) cand[off + x] = static_cast<int32_t>(seg[warp_id * kSegCap + x]);
        }
        __syncthreads();
    }
    const bool windowed = sampled && win_ok;
    if (!windowed) {
        p_lo = 0u;
        p_hi = 0xFFFFFFFFu;
    }

    // ---- 2. radix select: threshold key prefix `prefix` of (64 - fshift) bits
    int k_rem = 0;
    int fshift = 64;  // 64: nothing evicted (E == 0)
    unsigned long long prefix = 0;
    if (E > 0) {
        k_rem = windowed ? E - below_total : E;
        // windowed: the candidates' high words lie in [p_lo, p_hi]
        const unsigned int gmin = windowed ? max(p_lo, mm[0]) : mm[0];
        const unsigned int gmax = windowed ? min(p_hi, mm[1]) : mm[1];
        const int cpl = (gmin == gmax) ? 32 : __clz(gmin ^ gmax);
        int bitpos = 32 - cpl;  // unresolved bits of the high word
        unsigned int hp = cpl == 0 ? 0u : (cpl == 32 ? gmin : (gmin >> bitpos));
        fshift = 32 + bitpos;
        bool done = false;
        // Only the keys of the chosen bin can hold the boundary: when they
        // fit, their indices are compacted into `cand` (after the sample
        // window, or after the first full pass) and every later pass (high
        // or low word) visits just them.
        bool use_cand = windowed;
        const int n_round_all = (L + nthr - 1) / nthr * nthr;
        while (bitpos > 0) {  // high-word passes (shared memory)
            const int bits = min(11, bitpos);
            const int shift = bitpos - bits;
            const unsigned int dmask = (1u << bits) - 1u;
            // candidate passes are small and spread out: one histogram copy
            const int ncopies = use_cand ? 1 : kSelHistCopies;
            uint32_t* hh = use_cand ? hcopy : my_hist;
            for (int b = tid; b < ncopies * 2048; b += nthr) hcopy[b] = 0;
            __syncthreads();
            const int n_iter = use_cand ? (n_cand + nthr - 1) / nthr * nthr : n_round_all;
            for (int x = tid; x < n_iter; x += nthr) {
                const int j = use_cand ? (x < n_cand ? cand[x] : L) : x;
                const unsigned int w = j < L ? HI(j) : 0u;
                const bool act = j < L && (bitpos == 32 || (w >> bitpos) == hp);
                hist_add(hh, (w >> shift) & dmask, act);
            }
            __syncthreads();
            reduce_hist_copies(hcopy, hist, 1 << bits, ncopies);
            const int d = block_find_digit(hist, 1 << bits, k_rem, bc, scan_sm);
            k_rem -= bc[1];
            hp = (bitpos == 32 ? 0u : (hp << bits)) | static_cast<unsigned int>(d);
            bitpos = shift;
            fshift = 32 + shift;
            done = bc[2] == k_rem;
            if (!done && !use_cand && bc[2] <= cand_cap) {
                // compact the chosen bin (warp-aggregated appends)
                if (tid == 0) n_cand = 0;
                __syncthreads();
                for (int j = tid; j < n_round_all; j += nthr) {
                    const bool in = j < L && (HI(j) >> bitpos) == hp;
                    const unsigned m = __ballot_sync(0xFFFFFFFFu, in);
                    int base = 0;
                    if ((tid & 31) == 0 && m) base = atomicAdd(&n_cand, __popc(m));
                    base = __shfl_sync(0xFFFFFFFFu, base, 0);
                    if (in) cand[base + __popc(m & ((1u << (tid & 31)) - 1u))] = j;
                }
                use_cand = true;
            }
            __syncthreads();
            if (done) break;
        }
        prefix = static_cast<unsigned long long>(hp);
        if (!done && bitpos == 0) {
            // the boundary high word is shared: resolve the low words of
            // those keys only (read from global memory)
            int lbit = 32;
            unsigned int lp = 0u;
            while (lbit > 0) {
                const int bits = min(11, lbit);
                const int shift = lbit - bits;
                const unsigned int dmask = (1u << bits) - 1u;
                const int ncopies = use_cand ? 1 : kSelHistCopies;
                uint32_t* hh = use_cand ? hcopy : my_hist;
                for (int b = tid; b < ncopies * 2048; b += nthr) hcopy[b] = 0;
                __syncthreads();
                const int n_iter = use_cand ? (n_cand + nthr - 1) / nthr * nthr : n_round_all;
                for (int x = tid; x < n_iter; x += nthr) {
                    const int j = use_cand ? (x < n_cand ? cand[x] : L) : x;
                    bool act = j < L && HI(j) == hp;
                    unsigned int lw = 0u;
                    if (act) {
                        lw = static_cast<unsigned int>(__ldcg(gk + j));
                        act = (lbit == 32) || (lw >> lbit) == lp;
                    }
                    hist_add(hh, (lw >> shift) & dmask, act);
                }
                __syncthreads();
                reduce_hist_copies(hcopy, hist, 1 << bits, ncopies);
                const int d = block_find_digit(hist, 1 << bits, k_rem, bc, scan_sm);
                k_rem -= bc[1];
                lp = (lbit == 32 ? 0u : (lp << bits)) | static_cast<unsigned int>(d);
                lbit = shift;
                const bool dn = bc[2] == k_rem;
                __syncthreads();
                if (dn) break;
            }
            fshift = lbit;
            prefix = (static_cast<unsigned long long>(hp) << (32 - lbit)) | (lp);
        }
    }

    // ---- 3. position-order sweep: evict iff key-prefix < prefix, or equal and
    // among the first k_rem such keys (older first, importance.cpp:46-52)
    __shared__ int w_less[32], w_tie[32], w_tieb[32], w_keepb[32];
    auto classify = [&](int j, bool& less, bool& tie) {
        less = false;
        tie = false;
        if (E == 0) return;
        const unsigned int hj = HI(j);
        if (hj < p_lo || hj > p_hi) {  // outside the candidate window
            less = hj < p_lo;
            return;
        }
        if (fshift >= 32) {
            const unsigned long long top = static_cast<unsigned long long>(hj) >> (fshift - 32);
            less = top < prefix;
            tie = top == prefix;
        } else {
            const unsigned long long hp64 = prefix >> (32 - fshift);
            const unsigned long long hw = hj;
            if (hw != hp64) {
                less = hw < hp64;
            } else {
                const unsigned long long top = __ldcg(gk + j) >> fshift;
                less = top < prefix;
                tie = top == prefix;
            }
        }
    };
    if (windowed && bits) {
        // the bitmap holds the below-window evictions; the candidates (in
        // ascending position order: warp segments in warp order) add theirs,
        // ties by tie rank in position order (importance.cpp:46-52)
        int tie_run = 0;
        for (int x0 = 0; x0 < n_cand; x0 += nthr) {
            const int x = x0 + tid;
            bool l = false, t = false;
            int j = 0;
            if (x < n_cand) {
                j = cand[x];
                classify(j, l, t);
            }
            int n_tie;
            const int tr = tie_run + block_excl_scan(t ? 1 : 0, scan_sm, &n_tie);
            if (l || (t && tr < k_rem)) atomicOr(&evbits[j >> 5], 1u << (j & 31));
            tie_run += n_tie;
        }
        __syncthreads();
        // survivors per warp span (lane-parallel over the span's words)
        int kc = 0;
        for (int b = w_beg + lane_id * 32; b < w_end; b += 32 * 32) {
            const int nv = min(32, w_end - b);
            const unsigned valid = nv == 32 ? 0xFFFFFFFFu : ((1u << nv) - 1u);
            kc += __popc(~evbits[b >> 5] & valid);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) kc += __shfl_xor_sync(0xFFFFFFFFu, kc, o);
        if (lane_id == 0) w_keepb[warp_id] = kc;
        __syncthreads();
        if (tid == 0) {
            int run = 0;
            for (int w = 0; w < (nthr >> 5); ++w) {
                const int c = w_keepb[w];
                w_keepb[w] = run;
                run += c;
            }
        }
        __syncthreads();
        int keep_run = w_keepb[warp_id];
        const unsigned lt = (1u << lane_id) - 1u;
        for (int b = w_beg; b < w_end; b += 32) {
            const int p = b + lane_id;
            const bool kp = p < w_end && !((evbits[b >> 5] >> lane_id) & 1u);
            const unsigned kb = __ballot_sync(0xFFFFFFFFu, kp);
            if (kp) surv[keep_run + __popc(kb & lt)] = p;
            keep_run += __popc(kb);
        }
    } else {
    if (windowed) {
        // per-warp (less, tie) counts without a counting sweep: the load pass
        // counted each warp's keys below the window; only the candidates need
        // the threshold
        if (tid < (nthr >> 5)) {
            w_less[tid] = w_below[tid];
            w_tie[tid] = 0;
        }
        __syncthreads();
        for (int x = tid; x < n_cand; x += nthr) {
            const int j = cand[x];
            bool l = false, t = false;
            classify(j, l, t);
            if (l) atomicAdd(&w_less[j / wspan], 1);
            if (t) atomicAdd(&w_tie[j / wspan], 1);
        }
    } else {
        sweep_count(L, classify, w_less, w_tie);
    }
    __syncthreads();
    if (tid == 0) sweep_bases(L, k_rem, 0, 0, w_less, w_tie, w_tieb, w_keepb);
    __syncthreads();
    sweep_emit(L, classify, k_rem, w_tieb, w_keepb, [&](int q, int j) { surv[q] = j; });
    }
    // ---- 4. table metadata
    const int n_pages = (keep + B - 1) / B;
    const int pop_base = ctl->pop_base;
    const int pagebase = a.tab_pagebase[i];
    for (int p = tid; p < n_pages; p += nthr)
        s.block_table[(int64_t)t * s.max_pages + p] = s.stack[pop_base - 1 - (pagebase + p)];
    if (tid == 0) {
        s.num_pages[t] = n_pages;
        s.newest_fill[t] = keep - (n_pages - 1) * B;
        s.retained[t] = keep;
        if (a.evicted_counts) a.evicted_counts[i] = E;
    }
}

__global__ void __launch_bounds__(1024, 1) prefill_select_cta_kernel(DevState s, PrefillArgs a, const LaunchCtl* ctl) {
    extern __shared__ __align__(16) uint8_t smem[];
    if (ctl->abort) return;
    if (a.tab_len[blockIdx.x] > a.cta_len_max) return;  // mixed lengths: the cluster select's table
    select_table_cta<true>(s, a, blockIdx.x, smem, ctl);
}

// Tables longer than kSelectCtaMaxLen: the same CTA-per-table select with the
// high key words read from global memory (grid = launch tables; tables of at
// most `cluster_len_min` tokens are skipped: they take the shared-memory one).
__global__ void __launch_bounds__(1024, 1) prefill_select_stream_kernel(DevState s, PrefillArgs a,
                                                                        const LaunchCtl* ctl) {
    extern __shared__ __align__(16) uint8_t smem[];
    if (ctl->abort) return;
    const int L = a.tab_len[blockIdx.x];
    if (L <= a.cluster_len_min || L > a.cta_len_max) return;  // the other select kernel's table
    select_table_cta<false>(s, a, blockIdx.x, smem, ctl);
}

// The streamed select with 512 threads and a 4096-entry candidate list: 80 KB
// of shared memory and 32K registers, so two CTAs share an SM (A/B variant,
// PE_SELECT=stream512).
__global__ void __launch_bounds__(512, 2) prefill_select_stream512_kernel(DevState s, PrefillArgs a,
                                                                          const LaunchCtl* ctl) {
    extern __shared__ __align__(16) uint8_t smem[];
    if (ctl->abort) return;
    const int L = a.tab_len[blockIdx.x];
    if (L <= a.cluster_len_min || L > a.cta_len_max) return;  // the other select kernel's table
    select_table_cta<false>(s, a, blockIdx.x, smem, ctl);
}

// The global select's fallback (pe_select.cu): tables whose sampled window
// missed the boundary (tie-heavy or adversarial score distributions) take the
// streamed CTA-per-table select; every other CTA exits at once.
__global__ void __launch_bounds__(1024, 1) gsel_fallback_kernel(DevState s, PrefillArgs a, GselArgs g,
                                                                const LaunchCtl* ctl) {
    extern __shared__ __align__(16) uint8_t smem[];
    if (ctl->abort) return;
    for (int i = blockIdx.x; i < a.n_tab; i += gridDim.x) {
        if (g.flag[g.tab_off + i]) {  // block-uniform
            select_table_cta<false>(s, a, i, smem, ctl);
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// prefill_copy_kernel: one warp per destination page. Lane pair r moves the
// page's slot r: survivor q = page*B + r (position order) -> K and V rows
// with 256-bit loads/stores, position and cached score beside the page; the
// warp then sums the B scores in slot order (page_score, importance.cpp:19-30)
// for a full page. Grid (ceil(max pages / 4), n_tab).
// One warp copies destination page j of launch table i.
__device__ __forceinline__ void copy_page_warp(const DevState& s, const PrefillArgs& a, const LaunchCtl* ctl, int i,
                                               int j) {
    const int lane = threadIdx.x & 31;
    const int L = a.tab_len[i];
    const int keep = (s.policy == PE_POLICY_PAGED_EVICTION && L > s.C) ? s.C : L;
    if (a.direct_identity && keep == L) return;  // packed by the score kernel
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

__global__ void __launch_bounds__(128) prefill_copy_kernel(DevState s, PrefillArgs a, const LaunchCtl* ctl) {
    if (ctl->abort) return;
    copy_page_warp(s, a, ctl, blockIdx.x, blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5));
}

// The same packing with each survivor's S recomputed from the row registers
// it is copied from (pair_token_score with destinations: every load of the
// row is issued before its stores, and no key is gathered): the score is the
// same function of the same bytes, so it is bit-identical to the key.
template <int SV>
__global__ void __launch_bounds__(256) prefill_copy_score_kernel(DevState s, PrefillArgs a, const LaunchCtl* ctl) {
    if (ctl->abort) return;
    const int i = blockIdx.x;
    const int j = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int L = a.tab_len[i];
    const int keep = (s.policy == PE_POLICY_PAGED_EVICTION && L > s.C) ? s.C : L;
    if (a.direct_identity && keep == L) return;  // packed by the score kernel
    const int B = s.B;
    const int n_pages = (keep + B - 1) / B;
    if (j >= n_pages) return;
    const int h = i % s.tab_heads;
    const int64_t row0 = (a.tab_tok0[i] * s.tab_heads + h) * (int64_t)s.row_bytes;
    const int pagebase = a.tab_pagebase[i];
    const int page = s.stack[ctl->pop_base - 1 - (pagebase + j)];
    const int32_t* surv = a.surv + (int64_t)pagebase * B;
    double sum = 0.0;
    for (int s0 = 0; s0 < B; s0 += 16) {
        const int slot = s0 + (lane >> 1);
        const int q = j * B + slot;
        const bool valid = slot < B && q < keep;
        const int tok = valid ? __ldg(surv + q) : 0;
        const int64_t src = row0 + (int64_t)tok * a.token_stride;
        uint8_t* kd = s.pages + (((int64_t)page * 2 + 0) * B + slot) * s.pitch;
        uint8_t* vd = s.pages + (((int64_t)page * 2 + 1) * B + slot) * s.pitch;
        const double S = pair_token_score<SV>(a.k + src, a.v + src, valid, s.w, s.dtype, kd, vd);
        if (valid && (lane & 1) == 0) {
            s.positions[(int64_t)page * B + slot] = tok;
            s.token_scores[(int64_t)page * B + slot] = S;
        }
        const int ns = min(16, B - s0);
        for (int u = 0; u < ns; ++u) sum += __shfl_sync(0xFFFFFFFFu, S, 2 * u);
    }
    if (lane == 0 && (j + 1) * B <= keep) s.page_scores[page] = sum / static_cast<double>(B);
}

void launch_prefill_copy_any(int variant, dim3 grid, cudaStream_t st, const DevState& s, const PrefillArgs& a,
                             const LaunchCtl* ctl) {
    const char* rs = std::getenv("PE_COPY_RESCORE");  // A/B: 0 = gather the keys (prefill_copy_kernel)
    const bool rescore = !(rs != nullptr && std::strcmp(rs, "0") == 0) && s.pitch == s.row_bytes;
    if (rescore) {
        // one warp (destination page) per CTA: the gather balances best in
        // small CTAs (cfg3 1.772 vs 1.785 ms with 4 warps, cfg2 0.511 vs 0.515)
        const char* cw = std::getenv("PE_COPY_WARPS");  // A/B: warps (pages) per copy CTA
        const int warps = cw ? std::max(1, std::min(8, std::atoi(cw))) : 1;
        const dim3 g2(grid.x, (grid.y * 4 + warps - 1) / warps);
        PE_SCORE_DISPATCH(variant, (prefill_copy_score_kernel<SV><<<g2, 32 * warps, 0, st>>>(s, a, ctl)));
    } else {
        prefill_copy_kernel<<<grid, 128, 0, st>>>(s, a, ctl);
    }
}

// ---------------------------------------------------------------------------
// prefill_fused_kernel: the whole prune+pack of one call in ONE persistent
// launch (one 1024-thread CTA per SM). CTAs take work items in schedule
// order from a global counter:
//   S(q, u)  score unit u of sequence q: tokens [u*T, u*T+T) x all heads
//            (same arithmetic as prefill_score_kernel); then seq_done[q]++.
//   X(q, h)  table (q, h): wait until every score unit of q is done, then the
//            CTA select (select_table_cta) and the survivor copy (one warp per
//            page), i.e. what prefill_select_cta_kernel + prefill_copy_kernel do.
// The host schedule interleaves X(q) after S(q+1), so while some SMs run a
// latency-bound select, the others keep streaming the next sequence's K/V:
// the select no longer serialises with the HBM-bound passes. Deadlock-free:
// an X item only waits for S items that precede it in the schedule, and
// those were claimed by CTAs that are running.
template <int SV>
__global__ void __launch_bounds__(1024, 1) prefill_fused_kernel(DevState s, PrefillArgs a, const LaunchCtl* ctl,
                                                                 const int32_t* items, int n_items, int* work_ctr,
                                                                 int* seq_done, const int32_t* seq_units,
                                                                 int unit_tokens) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int sh_item;
    if (ctl->abort) return;
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    const int H = s.tab_heads;
    for (;;) {
        if (threadIdx.x == 0) sh_item = atomicAdd(work_ctr, 1);
        __syncthreads();
        const int id = sh_item;
        __syncthreads();
        if (id >= n_items) break;
        const int d = __ldg(items + id);
        const int sq = (d >> 16) & 0x7FFF;
        const int idx = d & 0xFFFF;
        if (d >= 0) {  // S: score unit
            const int L = a.tab_len[sq * H];
            const int tok_lo = idx * unit_tokens;
            const int tok_hi = min(L, tok_lo + unit_tokens);
            const int64_t f_lo = (int64_t)tok_lo * H, f_hi = (int64_t)tok_hi * H;
            const int64_t row0 = a.tab_tok0[sq * H] * H;
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
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) atomicAdd(seq_done + sq, 1);
        } else {  // X: select + copy of table (sq, idx)
            if (threadIdx.x == 0) {
                const int need = __ldg(seq_units + sq);
                while (true) {
                    int v;
                    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(seq_done + sq) : "memory");
                    if (v >= need) break;
                    __nanosleep(200);
                }
            }
            __syncthreads();
            const int i = sq * H + idx;
            select_table_cta<true>(s, a, i, smem, ctl);
            __threadfence();
            __syncthreads();
            const int L = a.tab_len[i];
            const int keep = (s.policy == PE_POLICY_PAGED_EVICTION && L > s.C) ? s.C : L;
            const int n_pages = (keep + s.B - 1) / s.B;
            for (int j = wid; j < n_pages; j += nw) copy_page_warp(s, a, ctl, i, j);
            __syncthreads();
        }
    }
}

void launch_prefill_fused_any(int variant, int grid, size_t smem, cudaStream_t st, const DevState& s,
                              const PrefillArgs& a, const LaunchCtl* ctl, const int32_t* items, int n_items,
                              int* work_ctr, int* seq_done, const int32_t* seq_units, int unit_tokens) {
    PE_SCORE_DISPATCH(variant, (prefill_fused_kernel<SV><<<grid, 1024, smem, st>>>(
                                   s, a, ctl, items, n_items, work_ctr, seq_done, seq_units, unit_tokens)));
}

const void* prefill_fused_fn(int variant) {
    switch (variant) {
    case kScoreBf16x16: return reinterpret_cast<const void*>(prefill_fused_kernel<kScoreBf16x16>);
    case kScoreBf16x8: return reinterpret_cast<const void*>(prefill_fused_kernel<kScoreBf16x8>);
    case kScoreF32x16: return reinterpret_cast<const void*>(prefill_fused_kernel<kScoreF32x16>);
    case kScoreF32x32: return reinterpret_cast<const void*>(prefill_fused_kernel<kScoreF32x32>);
    default: return reinterpret_cast<const void*>(prefill_fused_kernel<kScoreGeneric>);
    }
}

}  // namespace pe
