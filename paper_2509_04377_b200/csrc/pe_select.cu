// K1 select, GPU-wide ("global select"): the E = L - C evicted tokens of
// every table of a prefill wave (rank_tokens, importance.cpp:41-60: the E
// smallest by (score asc, position asc); drop_positions, policy.cpp:75-86:
// survivors keep position order) as four short, fully parallel kernels
// instead of one long latency chain per table:
//
//   gsel_window_kernel   CTA per table: a strided sample of 1024 high key
//                        words, sorted; the window [p_lo, p_hi] of high
//                        words around the sample's boundary rank (+-3.5
//                        binomial sigma) holds the E-th key with
//                        overwhelming probability (checked exactly below)
//   gsel_count_kernel    CTA per (table, 2048-position chunk): classifies
//                        every key below / inside / above the window; below
//                        -> eviction bit (one ballot word per 32 positions),
//                        inside -> (key, position) appended to the table's
//                        candidate list; per-chunk below counts
//   gsel_resolve_kernel  CTA per table: k_rem = E - (keys below the window)
//                        must lie in [0, #candidates] (else the table is
//                        flagged for the CTA-per-table select,
//                        gsel_fallback_kernel); an MSB radix select over the
//                        candidates in shared memory finds the k_rem-th
//                        smallest key T: keys < T and the oldest of the keys
//                        equal to T get their eviction bit; per-chunk
//                        survivor bases (exclusive scan); table metadata
//   gsel_emit_kernel     CTA per (table, chunk): survivor ranks from the
//                        eviction bits (ballots) -> survivor list
//
// Keys are the IEEE bits of S >= +0 (u64 order = double order), so the
// decisions are exactly the reference's, ties included: keys equal to the
// threshold are evicted oldest first. The survivor list feeds
// prefill_copy_kernel unchanged.
#include "pe_kernels.cuh"

namespace pe {

__device__ __forceinline__ int table_keep(const DevState& s, int L) {
    return (s.policy == PE_POLICY_PAGED_EVICTION && L > s.C) ? s.C : L;
}

__global__ void __launch_bounds__(kGselSample) gsel_window_kernel(DevState s, PrefillArgs a, GselArgs g,
                                                                  const LaunchCtl* ctl) {
    __shared__ uint32_t samp[kGselSample];
    if (ctl->abort) return;
    const int i = blockIdx.x;
    const int gi = g.tab_off + i;
    const int tid = threadIdx.x;
    const int L = a.tab_len[i];
    const int E = L - table_keep(s, L);
    uint2 w = make_uint2(0u, 0xFFFFFFFFu);  // short tables: every key is a candidate
    if (E > 0 && L > kGselAll) {
        const unsigned long long* gk = a.keys + a.tab_keybase[i];
        const uint32_t x = static_cast<uint32_t>(__ldcg(gk + (int)(((int64_t)tid * L) / kGselSample)) >> 32);
        w = gsel_window_of_sample(x, samp, E, L);
    }
    if (tid == 0) {
        g.win[gi] = w;
        g.cand_n[gi] = 0;
        g.flag[gi] = g.force_fallback;  // test knob: every table through the fallback select
    }
}

__global__ void __launch_bounds__(256) gsel_count_kernel(DevState s, PrefillArgs a, GselArgs g,
                                                         const LaunchCtl* ctl) {
    __shared__ int red[8];
    __shared__ int n_loc, gbase;
    __shared__ unsigned long long lkey[kGselChunk];
    __shared__ int32_t lpos[kGselChunk];
    if (ctl->abort) return;
    const int i = blockIdx.x;
    const int c = blockIdx.y;
    const int gi = g.tab_off + i;
    const int L = a.tab_len[i];
    const int p0 = c * kGselChunk;
    if (p0 >= L || L - table_keep(s, L) == 0 || g.flag[gi]) return;
    if (threadIdx.x == 0) n_loc = 0;
    const uint2 w = g.win[gi];
    const unsigned long long* gk = a.keys + a.tab_keybase[i];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* eb = g.evbits + ((int64_t)gi * g.chunk_stride + c) * kGselWords;
    unsigned long long kv[kGselChunk / 256];
#pragma unroll
    for (int u = 0; u < kGselChunk / 256; ++u) {
        const int p = p0 + u * 256 + threadIdx.x;
        kv[u] = p < L ? __ldcg(gk + p) : 0ull;
    }
    __syncthreads();
    int below = 0;
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int u = 0; u < kGselChunk / 256; ++u) {
        const int p = p0 + u * 256 + threadIdx.x;
        const bool in = p < L;
        const uint32_t hw = static_cast<uint32_t>(kv[u] >> 32);
        const bool bl = in && hw < w.x;
        const bool cd = in && hw >= w.x && hw <= w.y;
        const unsigned bm = __ballot_sync(0xFFFFFFFFu, bl);
        if (lane == 0) eb[u * 8 + wid] = bm;  // positions p0 + u*256 + wid*32 + [0, 32)
        below += bl;
        const unsigned cm = __ballot_sync(0xFFFFFFFFu, cd);
        if (cm) {  // warp-aggregated append to the CTA's shared list
            const int leader = __ffs(cm) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(&n_loc, __popc(cm));
            base = __shfl_sync(0xFFFFFFFFu, base, leader);
            if (cd) {
                const int idx = base + __popc(cm & lt);
                lkey[idx] = kv[u];
                lpos[idx] = p;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) below += __shfl_xor_sync(0xFFFFFFFFu, below, o);
    if (lane == 0) red[wid] = below;
    __syncthreads();
    if (threadIdx.x == 0) {
        int b = 0;
        for (int x = 0; x < (int)(blockDim.x >> 5); ++x) b += red[x];
        g.chunk_cnt[(int64_t)gi * g.chunk_stride + c] = b;
        gbase = n_loc > 0 ? atomicAdd(&g.cand_n[gi], n_loc) : 0;  // one reservation per CTA
    }
    __syncthreads();
    unsigned long long* ck = g.cand_key + (int64_t)gi * g.cand_stride;
    int32_t* cp = g.cand_pos + (int64_t)gi * g.cand_stride;
    const int nl = n_loc, gb = gbase;
    for (int x = threadIdx.x; x < nl; x += blockDim.x) {
        if (gb + x < g.cand_stride) {
            ck[gb + x] = lkey[x];
            cp[gb + x] = lpos[x];
        }
    }
}

// Block-wide min / max of a u64 (every thread passes its value; result on all).
__device__ __forceinline__ void block_minmax_u64(unsigned long long lo, unsigned long long hi,
                                                 unsigned long long* sm, unsigned long long* out) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
    }
    const int nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        sm[threadIdx.x >> 5] = lo;
        sm[32 + (threadIdx.x >> 5)] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a = ~0ull, b = 0ull;
        for (int w = 0; w < nw; ++w) {
            a = min(a, sm[w]);
            b = max(b, sm[32 + w]);
        }
        out[0] = a;
        out[1] = b;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(512) gsel_resolve_kernel(DevState s, PrefillArgs a, GselArgs g,
                                                           const LaunchCtl* ctl) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int ev_chunk[kGselMaxChunks];
    __shared__ int red[16];
    __shared__ int sh[4];  // bad flag, n, k_rem, n_eq
    __shared__ unsigned long long mm_sm[64], mm[2];
    __shared__ uint32_t hist[256];
    __shared__ int dig[3];
    __shared__ int32_t eq[kGselMaxTies];  // indices of the candidates equal to the threshold
    if (ctl->abort) return;
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const int lane = tid & 31;
    const int i = blockIdx.x;
    const int gi = g.tab_off + i;
    const int L = a.tab_len[i];
    const int keep = table_keep(s, L);
    const int E = L - keep;
    const int nch = (L + kGselChunk - 1) / kGselChunk;
    int32_t* cc = g.chunk_cnt + (int64_t)gi * g.chunk_stride;
    if (g.flag[gi]) return;  // forced fallback (test knob)
    if (E > 0) {
        int b = 0;
        for (int c = tid; c < nch; c += nthr) b += cc[c];
        for (int c = tid; c < nch; c += nthr) ev_chunk[c] = 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xFFFFFFFFu, b, o);
        if (lane == 0) red[tid >> 5] = b;
        __syncthreads();
        if (tid == 0) {
            int below = 0;
            for (int x = 0; x < (nthr >> 5); ++x) below += red[x];
            const int n = g.cand_n[gi];
            const int k_rem = E - below;
            sh[0] = (n > g.cand_stride || k_rem < 0 || k_rem > n) ? 1 : 0;
            sh[1] = n;
            sh[2] = k_rem;
            sh[3] = 0;
            if (sh[0]) g.flag[gi] = 1;  // the CTA-per-table select takes this table
        }
        __syncthreads();
        if (sh[0]) return;
        const int n = sh[1];
        int k = sh[2];  // candidates to evict (the k smallest by (key, position))
        unsigned long long* sk = reinterpret_cast<unsigned long long*>(smem);
        int32_t* sp = reinterpret_cast<int32_t*>(sk + kGselCandCap);
        const unsigned long long* ck = g.cand_key + (int64_t)gi * g.cand_stride;
        const int32_t* cp = g.cand_pos + (int64_t)gi * g.cand_stride;
        unsigned long long lo = ~0ull, hi = 0ull;
        for (int j = tid; j < n; j += nthr) {
            const unsigned long long x = __ldcg(ck + j);
            sk[j] = x;
            sp[j] = __ldcg(cp + j);
            lo = min(lo, x);
            hi = max(hi, x);
        }
        uint32_t* eb = g.evbits + (int64_t)gi * g.chunk_stride * kGselWords;
        if (k > 0) {
            block_minmax_u64(lo, hi, mm_sm, mm);
            // MSB radix select of the k-th smallest key over the bits below
            // the candidates' common prefix (8-bit digits, shared histogram)
            const int cpl = mm[0] == mm[1] ? 64 : __clzll(mm[0] ^ mm[1]);
            int bitpos = 64 - cpl;  // unresolved low bits
            unsigned long long prefix = cpl == 64 ? mm[0] : (cpl == 0 ? 0ull : (mm[0] >> bitpos));
            while (bitpos > 0) {
                const int bits = min(8, bitpos);
                const int shift = bitpos - bits;
                for (int x = tid; x < 256; x += nthr) hist[x] = 0;
                __syncthreads();
                for (int j = tid; j < n; j += nthr) {
                    const unsigned long long x = sk[j];
                    if (bitpos == 64 || (x >> bitpos) == prefix)
                        atomicAdd(&hist[(x >> shift) & ((1u << bits) - 1u)], 1u);
                }
                __syncthreads();
                if (tid < 32) {  // warp scan over the 256 bins (8 per lane)
                    uint32_t c[8], sum = 0;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        c[u] = hist[lane * 8 + u];
                        sum += c[u];
                    }
                    uint32_t incl = sum;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    uint32_t cum = incl - sum;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        if (cum < (uint32_t)k && (uint32_t)k <= cum + c[u]) {
                            dig[0] = lane * 8 + u;
                            dig[1] = (int)cum;
                        }
                        cum += c[u];
                    }
                }
                __syncthreads();
                k -= dig[1];
                prefix = (bitpos == 64 ? 0ull : (prefix << bits)) | static_cast<unsigned long long>(dig[0]);
                bitpos = shift;
                __syncthreads();
            }
            // prefix = the threshold key T; k = how many keys equal to T are
            // evicted (the oldest, importance.cpp:46-52)
            const unsigned long long T = prefix;
            for (int j = tid; j < n; j += nthr) {
                const unsigned long long x = sk[j];
                if (x < T) {
                    const int p = sp[j];
                    atomicOr(&eb[p >> 5], 1u << (p & 31));
                    atomicAdd(&ev_chunk[p / kGselChunk], 1);
                } else if (x == T) {
                    const int e = atomicAdd(&sh[3], 1);
                    if (e < kGselMaxTies) eq[e] = j;
                }
            }
            __syncthreads();
            const int n_eq = sh[3];
            if (n_eq > kGselMaxTies) {  // massive ties: the CTA-per-table select (its position sweeps)
                if (tid == 0) g.flag[gi] = 1;
                return;
            }
            for (int e = tid; e < n_eq; e += nthr) {  // tie rank by position
                const int pe_ = sp[eq[e]];
                int r = 0;
                for (int f = 0; f < n_eq; ++f) r += sp[eq[f]] < pe_;
                if (r < k) {
                    atomicOr(&eb[pe_ >> 5], 1u << (pe_ & 31));
                    atomicAdd(&ev_chunk[pe_ / kGselChunk], 1);
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
            int run = 0;
            for (int c = 0; c < nch; ++c) {
                const int len = min(kGselChunk, L - c * kGselChunk);
                const int kc = len - cc[c] - ev_chunk[c];
                cc[c] = run;
                run += kc;
            }
        }
    } else {
        for (int c = tid; c < nch; c += nthr) cc[c] = c * kGselChunk;  // identity: every token survives
    }
    // table metadata (the survivors are packed by prefill_copy_kernel)
    const int h = i % s.tab_heads;
    const int seq = a.seq_begin + i / s.tab_heads;
    const int t = (seq * s.n_layers + a.layer) * s.tab_heads + h;
    const int n_pages = (keep + s.B - 1) / s.B;
    const int pop_base = ctl->pop_base;
    const int pagebase = a.tab_pagebase[i];
    for (int p = tid; p < n_pages; p += nthr)
        s.block_table[(int64_t)t * s.max_pages + p] = s.stack[pop_base - 1 - (pagebase + p)];
    if (tid == 0) {
        s.num_pages[t] = n_pages;
        s.newest_fill[t] = keep - (n_pages - 1) * s.B;
        s.retained[t] = keep;
        if (a.evicted_counts) a.evicted_counts[i] = E;
    }
}

__global__ void __launch_bounds__(64) gsel_emit_kernel(DevState s, PrefillArgs a, GselArgs g, const LaunchCtl* ctl) {
    __shared__ int warp0_keep;
    if (ctl->abort) return;
    const int i = blockIdx.x;
    const int c = blockIdx.y;
    const int gi = g.tab_off + i;
    const int L = a.tab_len[i];
    const int p0 = c * kGselChunk;
    if (p0 >= L || g.flag[gi]) return;  // flagged: gsel_fallback_kernel emits the table
    int32_t* surv = a.surv + (int64_t)a.tab_pagebase[i] * s.B;
    int base = g.chunk_cnt[(int64_t)gi * g.chunk_stride + c];
    const int len = min(kGselChunk, L - p0);
    if (L - table_keep(s, L) == 0) {
        for (int j = threadIdx.x; j < len; j += blockDim.x) surv[base + j] = p0 + j;
        return;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t* eb = g.evbits + ((int64_t)gi * g.chunk_stride + c) * kGselWords;
    // warp w: words [32w, 32w + 32) of the chunk; lane l holds word 32w + l
    const int wd = wid * 32 + lane;
    const int nv = min(32, max(0, len - wd * 32));
    const unsigned valid = nv >= 32 ? 0xFFFFFFFFu : ((1u << nv) - 1u);
    const unsigned km = nv > 0 ? (~__ldcg(eb + wd) & valid) : 0u;
    int cnt = __popc(km);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
    if (threadIdx.x == 0) warp0_keep = cnt;
    __syncthreads();
    if (wid == 1) base += warp0_keep;
    const unsigned lt = (1u << lane) - 1u;
    for (int q = 0; q < 32; ++q) {
        const unsigned wq = __shfl_sync(0xFFFFFFFFu, km, q);
        if ((wq >> lane) & 1u) surv[base + __popc(wq & lt)] = p0 + (wid * 32 + q) * 32 + lane;
        base += __popc(wq);
    }
}

}  // namespace pe
