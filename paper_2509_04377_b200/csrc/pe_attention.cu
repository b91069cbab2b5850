// K3: GQA paged decode attention over the pruned block tables.
//
// Reference: attend (attention.cpp:15-99) — per query head, logits
// q.k/sqrt(d) over the retained tokens in logical order (for_each_retained,
// block_table.hpp:81-91), max-subtracted softmax, weighted sum of values.
// The reference is MHA in double; GQA is the reference's attend called once
// per query head (head_count = 1) on its KV head's table (D3).
// Tolerance: relative L2 (output_deviation, attention.cpp:105-118) 1e-5 for
// fp32 caches, 1e-3 for bf16.
//
// Split-K: CTA (split, table) owns a contiguous range of the table's pages;
// each warp streams whole pages (K slots then V slots, 2B contiguous rows)
// into padded shared memory with cp.async, computes the G heads' logits with
// one lane per (token, head-pair), runs an online softmax in fp32 (exp2 with
// log2e folded into the scale) and accumulates P.V with one lane per
// d/32-dimension slice. Warp and split partials are merged with the usual
// (max, sum) log-sum-exp rescaling.
#include <cuda.h>
#include <cuda_bf16.h>

#include "pe_kernels.cuh"
#include "pe_tma.cuh"

namespace pe {

constexpr int kAttnThreads = 128;
constexpr int kAttnMaxG = 8;
constexpr int kAttnMaxDpl = 8;  // d <= 256
constexpr int kAttnStages = 2;

__device__ __forceinline__ float elem_f32(const uint8_t* row, int idx, int dtype) {
    if (dtype == PE_DTYPE_BF16) {
        return __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(row)[idx]) << 16);
    }
    return reinterpret_cast<const float*>(row)[idx];
}

// o / l, or 0 with PE_EMPTY_CACHE for a table without retained tokens (the
// reference's attend throws EmptyCache, attention.cpp:24-25).
__device__ __forceinline__ float empty_guard(const DevState& s, float o, float l) {
    if (l > 0.f) return o / l;
    set_status(s.status, PE_EMPTY_CACHE);
    return 0.f;
}

// Split-K completion: every split CTA of table i writes its partial, then
// takes a ticket; the CTA holding the last ticket merges all splits
// (out = sum_s o_s 2^(m_s - M) / sum_s l_s 2^(m_s - M)) and rearms the
// ticket. Replaces a separate merge launch.
__device__ __forceinline__ void merge_if_last(const DevState& s, const AttnArgs& a, int i, int d) {
    __shared__ int is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = atomicAdd(a.tickets + i, 1) == a.splits - 1;
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    const int H = a.kv_heads;
    const int h = i % H;
    const int seq = i / H;
    const int G = a.G;
    for (int x = threadIdx.x; x < G * d; x += blockDim.x) {
        const int g = x / d;
        float mm = -INFINITY;
        for (int sp = 0; sp < a.splits; ++sp) mm = fmaxf(mm, __ldcg(a.part_ml + (((int64_t)i * a.splits + sp) * G + g) * 2));
        float ll = 0.f, oo = 0.f;
        for (int sp = 0; sp < a.splits; ++sp) {
            const int64_t pidx = ((int64_t)i * a.splits + sp) * G + g;
            const float ms = __ldcg(a.part_ml + pidx * 2);
            const float c = (ms == -INFINITY) ? 0.f : exp2f(ms - mm);
            ll += __ldcg(a.part_ml + pidx * 2 + 1) * c;
            oo += __ldcg(a.part_o + pidx * d + (x % d)) * c;
        }
        a.out[((int64_t)seq * a.n_q_heads + h * G + g) * d + (x % d)] = empty_guard(s, oo, ll);
    }
    if (threadIdx.x == 0) a.tickets[i] = 0;
}

__global__ void __launch_bounds__(kAttnThreads) attention_split_kernel(DevState s, AttnArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    const int i = blockIdx.x;            // launch item: seq * kv_heads + h
    const int sp = blockIdx.y;           // split
    const int H = a.kv_heads;
    const int h = i % H;
    const int seq = i / H;
    const int t = a.table(s, i);
    const int G = a.G;
    const int d = a.d;
    const int B = s.B;
    const int N = s.num_pages[t];
    const int p_begin = sp * a.pages_per_split;
    const int p_end = min(N, p_begin + a.pages_per_split);
    const int elt = s.dtype == PE_DTYPE_BF16 ? 2 : 4;
    const int head_bytes = d * elt;       // this head's slice of each row
    const int col = a.col_elems(i) * elt;
    const int row_pitch = head_bytes + 16;
    const int stage_bytes = 2 * B * row_pitch;

    // shared layout: q [G][d] float | p [nw][G][16] float | warp partials | stages
    float* q_sm = reinterpret_cast<float*>(smem);
    float* p_sm = q_sm + G * d;
    float* wpart_o = p_sm + nw * G * 16;          // [nw][G][d]
    float* wpart_ml = wpart_o + nw * G * d;       // [nw][G][2]
    uint8_t* stages = reinterpret_cast<uint8_t*>(wpart_ml + nw * G * 2);
    stages = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(stages) + 15) & ~uintptr_t(15));
    uint8_t* my_stage = stages + wid * kAttnStages * stage_bytes;

    // load the G query heads of this table (as float, pre-scaled by log2e/sqrt(d))
    for (int x = threadIdx.x; x < G * d; x += blockDim.x) {
        const int g = x / d;
        const int dd = x % d;
        const uint8_t* qrow = a.q + ((int64_t)seq * a.n_q_heads + h * G + g) * head_bytes;
        q_sm[x] = elem_f32(qrow, dd, s.dtype) * a.scale_log2;
    }
    __syncthreads();

    const int dpl = (d + 31) / 32;  // dims per lane in P.V
    float o[kAttnMaxG][kAttnMaxDpl];
    float m[kAttnMaxG], l[kAttnMaxG];
#pragma unroll
    for (int g = 0; g < kAttnMaxG; ++g) {
        m[g] = -INFINITY;
        l[g] = 0.f;
#pragma unroll
        for (int k = 0; k < kAttnMaxDpl; ++k) o[g][k] = 0.f;
    }

    const int32_t* row = s.block_table + (int64_t)t * s.max_pages;
    const int my_n = (p_end - p_begin) > wid ? ((p_end - p_begin) - wid + nw - 1) / nw : 0;
    const int pieces = head_bytes / 16;
    auto issue = [&](int k) {
        if (k < my_n) {
            const int pg = p_begin + wid + k * nw;
            const uint8_t* base = s.pages + (int64_t)row[pg] * 2 * B * s.pitch + col;
            const int fill = (pg == N - 1) ? s.newest_fill[t] : B;
            uint8_t* st = my_stage + (k % kAttnStages) * stage_bytes;
            const int total = 2 * B * pieces;
            for (int x = lane; x < total; x += 32) {
                const int r = x / pieces;
                const int pc = x - r * pieces;
                const int slot = r % B;
                if (slot < fill) cp_async16(st + r * row_pitch + pc * 16, base + (int64_t)r * s.pitch + pc * 16);
            }
        }
        cp_async_commit();
    };
#pragma unroll
    for (int k = 0; k < kAttnStages - 1; ++k) issue(k);

    float* my_p = p_sm + wid * G * 16;
    for (int k = 0; k < my_n; ++k) {
        issue(k + kAttnStages - 1);
        cp_async_wait<kAttnStages - 1>();
        __syncwarp();
        const int pg = p_begin + wid + k * nw;
        const int fill = (pg == N - 1) ? s.newest_fill[t] : B;
        const uint8_t* st = my_stage + (k % kAttnStages) * stage_bytes;
        // process the page in groups of 16 slots
        for (int s0 = 0; s0 < fill; s0 += 16) {
            const int ns = min(16, fill - s0);
            // logits: lane -> slot s0 + (lane & 15), heads g = (lane>>4), +2, ...
            const int slot = s0 + (lane & 15);
            float sc[kAttnMaxG / 2];
#pragma unroll
            for (int gg = 0; gg < kAttnMaxG / 2; ++gg) sc[gg] = -INFINITY;
            if ((lane & 15) < ns) {
                const uint8_t* krow = st + slot * row_pitch;
                float acc[kAttnMaxG / 2];
#pragma unroll
                for (int gg = 0; gg < kAttnMaxG / 2; ++gg) acc[gg] = 0.f;
                for (int dd = 0; dd < d; dd += 4) {
                    float kv[4];
                    if (s.dtype == PE_DTYPE_BF16) {
                        const uint2 u = *reinterpret_cast<const uint2*>(krow + dd * 2);
                        kv[0] = __uint_as_float(u.x << 16);
                        kv[1] = __uint_as_float(u.x & 0xFFFF0000u);
                        kv[2] = __uint_as_float(u.y << 16);
                        kv[3] = __uint_as_float(u.y & 0xFFFF0000u);
                    } else {
                        const float4 f = *reinterpret_cast<const float4*>(krow + dd * 4);
                        kv[0] = f.x; kv[1] = f.y; kv[2] = f.z; kv[3] = f.w;
                    }
#pragma unroll
                    for (int gg = 0; gg < kAttnMaxG / 2; ++gg) {
                        const int g = (lane >> 4) + 2 * gg;
                        if (g < G) {
                            const float4 qv = *reinterpret_cast<const float4*>(q_sm + g * d + dd);
                            acc[gg] = fmaf(qv.x, kv[0], acc[gg]);
                            acc[gg] = fmaf(qv.y, kv[1], acc[gg]);
                            acc[gg] = fmaf(qv.z, kv[2], acc[gg]);
                            acc[gg] = fmaf(qv.w, kv[3], acc[gg]);
                        }
                    }
                }
#pragma unroll
                for (int gg = 0; gg < kAttnMaxG / 2; ++gg) sc[gg] = acc[gg];
            }
            // online softmax per head over the 16 slots (lanes of the same half)
#pragma unroll
            for (int gg = 0; gg < kAttnMaxG / 2; ++gg) {
                float mx = sc[gg];
#pragma unroll
                for (int off = 8; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, off));
                const int g = (lane >> 4) + 2 * gg;
                // both halves hold different heads; broadcast via smem
                const float mg_old = (g < G) ? m[g] : -INFINITY;
                const float mnew = fmaxf(mg_old, mx);
                const float pexp = (g < G && (lane & 15) < ns) ? exp2f(sc[gg] - mnew) : 0.f;
                float ps = pexp;
#pragma unroll
                for (int off = 8; off > 0; off >>= 1) ps += __shfl_xor_sync(0xFFFFFFFFu, ps, off);
                if (g < G) my_p[g * 16 + (lane & 15)] = pexp;
                const float mnew_b = mnew;
                const float ps_b = ps;
                // lanes 0 and 16 hold heads 2gg and 2gg+1: broadcast to every lane
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const int gh = half + 2 * gg;
                    const float mn = __shfl_sync(0xFFFFFFFFu, mnew_b, half * 16);
                    const float pss = __shfl_sync(0xFFFFFFFFu, ps_b, half * 16);
                    if (gh < G) {
                        const float corr = exp2f(m[gh] - mn);
                        l[gh] = l[gh] * corr + pss;
#pragma unroll
                        for (int kk = 0; kk < kAttnMaxDpl; ++kk) o[gh][kk] *= corr;
                        m[gh] = mn;
                    }
                }
            }
            __syncwarp();
            // P.V: lane owns dims lane + 32*k
            for (int j = 0; j < ns; ++j) {
                const uint8_t* vrow = st + (B + s0 + j) * row_pitch;
                float vv[kAttnMaxDpl];
#pragma unroll
                for (int kk = 0; kk < kAttnMaxDpl; ++kk) {
                    const int dd = lane + 32 * kk;
                    vv[kk] = (kk < dpl && dd < d) ? elem_f32(vrow, dd, s.dtype) : 0.f;
                }
#pragma unroll
                for (int g = 0; g < kAttnMaxG; ++g) {
                    if (g < G) {
                        const float p = my_p[g * 16 + j];
#pragma unroll
                        for (int kk = 0; kk < kAttnMaxDpl; ++kk) o[g][kk] = fmaf(p, vv[kk], o[g][kk]);
                    }
                }
            }
            __syncwarp();
        }
        __syncwarp();
    }
    cp_async_wait<0>();

    // warp partials -> smem
    float* wo = wpart_o + wid * G * d;
    float* wml = wpart_ml + wid * G * 2;
    for (int g = 0; g < G; ++g) {
#pragma unroll
        for (int kk = 0; kk < kAttnMaxDpl; ++kk) {
            const int dd = lane + 32 * kk;
            if (kk < dpl && dd < d) wo[g * d + dd] = o[g][kk];
        }
        if (lane == 0) {
            wml[g * 2] = m[g];
            wml[g * 2 + 1] = l[g];
        }
    }
    __syncthreads();
    // merge the warps and write the split partial
    const int n_splits = a.splits;
    for (int x = threadIdx.x; x < G * d; x += blockDim.x) {
        const int g = x / d;
        float mm = -INFINITY;
        for (int w2 = 0; w2 < nw; ++w2) mm = fmaxf(mm, wpart_ml[w2 * G * 2 + g * 2]);
        float ll = 0.f, oo = 0.f;
        for (int w2 = 0; w2 < nw; ++w2) {
            const float mw = wpart_ml[w2 * G * 2 + g * 2];
            const float c = (mw == -INFINITY) ? 0.f : exp2f(mw - mm);
            ll += wpart_ml[w2 * G * 2 + g * 2 + 1] * c;
            oo += wpart_o[w2 * G * d + x] * c;
        }
        const int64_t pidx = ((int64_t)i * n_splits + sp) * G + g;
        a.part_o[pidx * d + (x % d)] = oo;
        if (x % d == 0) {
            a.part_ml[pidx * 2] = mm;
            a.part_ml[pidx * 2 + 1] = ll;
        }
    }
    merge_if_last(s, a, i, d);
}

// ---------------------------------------------------------------------------
// Tensor-core variant for bf16 caches with B = 16 (one MMA k-step per page).
// Per warp and page: the page (16 K rows + 16 V rows) is staged into padded
// shared memory with cp.async (3-stage ring), then
//   S = Q K^T   mma.sync m16n8k16: M = query heads of the KV head (G <= 8,
//               zero-padded to 16), N = 8 tokens, K = 16 dims (ldmatrix);
//   online softmax on the S fragments in fp32 (exp2, log2e folded into the
//               scale; slots past the newest page's fill masked to -inf);
//   O += P V    M = heads, N = 8 dims, K = 16 tokens (ldmatrix.trans), with
//               P split into bf16 hi + lo halves (two MMAs) so the bf16
//               rounding of the weights stays ~2^-17 relative.
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void split_bf16x2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
    hi = pack_bf16x2(x0, x1);
    const float h0 = __uint_as_float(hi << 16);
    const float h1 = __uint_as_float(hi & 0xFFFF0000u);
    lo = pack_bf16x2(x0 - h0, x1 - h1);
}

constexpr int kAttnMaxSplitPages = 512;

template <int D>
__global__ void __launch_bounds__(kAttnThreads, 2) attention_mma_kernel(DevState s, AttnArgs a) {
    constexpr int RB = D * 2;          // bf16 row bytes
    constexpr int RP = RB + 16;        // padded smem row pitch (conflict-free ldmatrix)
    constexpr int PAGE_SM = 32 * RP;   // 16 K rows + 16 V rows
    constexpr int NST = 3;             // cp.async stages per warp
    constexpr int KS = D / 16;         // QK k-steps
    constexpr int NT = D / 8;          // PV n-tiles
    constexpr int PIECES = RB / 16;
    extern __shared__ __align__(16) uint8_t smem[];
    pdl_top();  // see attention_tma_kernel
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    const int i = blockIdx.x;
    const int sp = blockIdx.y;
    const int H = a.kv_heads;
    const int h = i % H;
    const int seq = i / H;
    const int t = a.table(s, i);
    const int col = a.col_elems(i) * 2;
    const int G = a.G;
    const int N = s.num_pages[t];
    const int p_begin = sp * a.pages_per_split;
    const int p_end = min(N, p_begin + a.pages_per_split);
    const int g = lane >> 2;
    const int tq = lane & 3;

    uint8_t* stage = smem + wid * NST * PAGE_SM;
    float* wpart_o = reinterpret_cast<float*>(smem + nw * NST * PAGE_SM);  // [nw][G][D]
    float* wpart_ml = wpart_o + nw * G * D;                                 // [nw][G][2]

    // Q fragments (A operand, rows g < G real)
    uint32_t qa[KS][2];
    {
        const uint8_t* qrow = a.q + ((int64_t)seq * a.n_q_heads + h * G + min(g, G - 1)) * RB;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            qa[ks][0] = g < G ? *reinterpret_cast<const uint32_t*>(qrow + (16 * ks + 2 * tq) * 2) : 0u;
            qa[ks][1] = g < G ? *reinterpret_cast<const uint32_t*>(qrow + (16 * ks + 2 * tq + 8) * 2) : 0u;
        }
    }
    float o[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    float m = -INFINITY, l = 0.f;

    const int32_t* row = s.block_table + (int64_t)t * s.max_pages;
    const int my_n = (p_end - p_begin) > wid ? ((p_end - p_begin) - wid + nw - 1) / nw : 0;
    // this split's page ids, read once up front: the cp.async of page k must
    // not wait for a dependent block-table load
    __shared__ int32_t ids[kAttnMaxSplitPages];
    const bool ids_sm = p_end - p_begin <= kAttnMaxSplitPages;
    if (ids_sm)
        for (int j = threadIdx.x; j < p_end - p_begin; j += blockDim.x) ids[j] = __ldg(row + p_begin + j);
    __syncthreads();
    auto issue = [&](int k) {
        if (k < my_n) {
            const int pg = p_begin + wid + k * nw;
            const int32_t id = ids_sm ? ids[pg - p_begin] : __ldg(row + pg);
            const uint8_t* base = s.pages + (int64_t)id * 32 * s.pitch + col;
            uint8_t* st = stage + (k % NST) * PAGE_SM;
#pragma unroll
            for (int x = lane; x < 32 * PIECES; x += 32) {
                const int r = x / PIECES;
                const int pc = x - r * PIECES;
                cp_async16(st + r * RP + pc * 16, base + (int64_t)r * s.pitch + pc * 16);
            }
        }
        cp_async_commit();
    };
#pragma unroll
    for (int k = 0; k < NST - 1; ++k) issue(k);

    const uint32_t stage_s = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
    const int lm_j = lane >> 3, lm_r = lane & 7;
    for (int k = 0; k < my_n; ++k) {
        issue(k + NST - 1);
        cp_async_wait<NST - 1>();
        __syncwarp();
        const int pg = p_begin + wid + k * nw;
        const int fill = (pg == N - 1) ? s.newest_fill[t] : 16;
        const uint32_t st = stage_s + (k % NST) * PAGE_SM;
        // ---- S = Q K^T (two n-tiles of 8 tokens)
        float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            uint32_t b0, b1, b2, b3;
            const int tok = (lm_j >> 1) * 8 + lm_r;
            const int dcol = 16 * ks + (lm_j & 1) * 8;
            ldsm_x4(st + tok * RP + dcol * 2, b0, b1, b2, b3);
            mma_bf16_16816(sc[0], qa[ks][0], qa[ks][1], b0, b1);
            mma_bf16_16816(sc[1], qa[ks][0], qa[ks][1], b2, b3);
        }
        // ---- online softmax on row g (columns: tokens 8nt + 2tq, +1)
        float x[2][2];
        float rmax = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int tok = 8 * nt + 2 * tq + j;
                x[nt][j] = tok < fill ? sc[nt][j] * a.scale_log2 : -INFINITY;
                rmax = fmaxf(rmax, x[nt][j]);
            }
        }
        rmax = fmaxf(rmax, __shfl_xor_sync(0xFFFFFFFFu, rmax, 1));
        rmax = fmaxf(rmax, __shfl_xor_sync(0xFFFFFFFFu, rmax, 2));
        const float m_new = fmaxf(m, rmax);
        const float corr = exp2f(m - m_new);
        float rsum = 0.f;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                x[nt][j] = exp2f(x[nt][j] - m_new);
                rsum += x[nt][j];
            }
        }
        rsum += __shfl_xor_sync(0xFFFFFFFFu, rsum, 1);
        rsum += __shfl_xor_sync(0xFFFFFFFFu, rsum, 2);
        l = l * corr + rsum;
        m = m_new;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            o[nt][0] *= corr;
            o[nt][1] *= corr;
        }
        // ---- O += P V (P = hi + lo bf16 halves)
        uint32_t ph0, pl0, ph1, pl1;
        split_bf16x2(x[0][0], x[0][1], ph0, pl0);
        split_bf16x2(x[1][0], x[1][1], ph1, pl1);
#pragma unroll
        for (int ntp = 0; ntp < NT / 2; ++ntp) {
            uint32_t b0, b1, b2, b3;
            const int tok = (lm_j & 1) * 8 + lm_r;
            const int dd = 16 * ntp + (lm_j >> 1) * 8;
            ldsm_x4_t(st + (16 + tok) * RP + dd * 2, b0, b1, b2, b3);
            mma_bf16_16816(o[2 * ntp], ph0, ph1, b0, b1);
            mma_bf16_16816(o[2 * ntp], pl0, pl1, b0, b1);
            mma_bf16_16816(o[2 * ntp + 1], ph0, ph1, b2, b3);
            mma_bf16_16816(o[2 * ntp + 1], pl0, pl1, b2, b3);
        }
        __syncwarp();
    }
    cp_async_wait<0>();
    __syncthreads();  // stage memory is reused for the partials below? (separate region) keep warps aligned

    // ---- warp partials -> smem (row g < G: dims 8nt + 2tq, +1)
    if (g < G) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            wpart_o[(wid * G + g) * D + 8 * nt + 2 * tq] = o[nt][0];
            wpart_o[(wid * G + g) * D + 8 * nt + 2 * tq + 1] = o[nt][1];
        }
        if (tq == 0) {
            wpart_ml[(wid * G + g) * 2] = m;
            wpart_ml[(wid * G + g) * 2 + 1] = l;
        }
    }
    __syncthreads();
    const int n_splits = a.splits;
    for (int xi = threadIdx.x; xi < G * D; xi += blockDim.x) {
        const int gg = xi / D;
        float mm = -INFINITY;
        for (int w2 = 0; w2 < nw; ++w2) mm = fmaxf(mm, wpart_ml[(w2 * G + gg) * 2]);
        float ll = 0.f, oo = 0.f;
        for (int w2 = 0; w2 < nw; ++w2) {
            const float mw = wpart_ml[(w2 * G + gg) * 2];
            const float c = (mw == -INFINITY) ? 0.f : exp2f(mw - mm);
            ll += wpart_ml[(w2 * G + gg) * 2 + 1] * c;
            oo += wpart_o[(w2 * G + gg) * D + (xi % D)] * c;
        }
        if (n_splits == 1) {  // the whole table: write the output directly
            a.out[((int64_t)seq * a.n_q_heads + h * G + gg) * D + (xi % D)] = empty_guard(s, oo, ll);
            continue;
        }
        const int64_t pidx = ((int64_t)i * n_splits + sp) * G + gg;
        a.part_o[pidx * D + (xi % D)] = oo;
        if (xi % D == 0) {
            a.part_ml[pidx * 2] = mm;
            a.part_ml[pidx * 2 + 1] = ll;
        }
    }
    if (n_splits > 1) merge_if_last(s, a, i, D);
}

size_t attention_mma_smem(int d, int G) {
    const int nw = kAttnThreads / 32;
    return (size_t)nw * 3 * 32 * (2 * d + 16) + (size_t)nw * G * d * 4 + (size_t)nw * G * 2 * 4;
}

void launch_attention_mma(int d, dim3 grid, size_t smem, cudaStream_t st, const DevState& s, const AttnArgs& a) {
    if (d == 128) launch_pdl(attention_mma_kernel<128>, grid, dim3(kAttnThreads), smem, st, s, a);
    else launch_pdl(attention_mma_kernel<64>, grid, dim3(kAttnThreads), smem, st, s, a);
}

const void* attention_mma_fn(int d) {
    return d == 128 ? reinterpret_cast<const void*>(attention_mma_kernel<128>)
                    : reinterpret_cast<const void*>(attention_mma_kernel<64>);
}


// ---------------------------------------------------------------------------
// TMA variant (bf16, d in {64, 128}, B = 16; the default): the same per-warp pipeline and math as
// attention_mma_kernel, but each page is staged by two 2-D tensor-map loads
// (cp.async.bulk.tensor, 64 columns x 32 rows each, SWIZZLE_128B) issued by
// one lane and completing on the stage's mbarrier, instead of 512 16-byte
// cp.async per page; ldmatrix addresses apply the 128-byte swizzle
// (16-byte chunk c of row r lives at chunk c ^ (r & 7)), so the unpadded
// 8 KB stage is bank-conflict free.
template <int D>
__global__ void __launch_bounds__(kAttnThreads, 2) attention_tma_kernel(DevState s, AttnArgs a,
                                                                         const __grid_constant__ CUtensorMap tmap) {
    constexpr int HALVES = D / 64;       // 64-column boxes per page row
    constexpr int PAGE_SM = 32 * 2 * D;  // HALVES x 4 KB (32 rows x 128 B each)
    constexpr int NST = 3;
    constexpr int KS = D / 16;
    constexpr int NT = D / 8;
    extern __shared__ __align__(16) uint8_t smem[];  // aligned to 1024 B by hand (align1024)
    __shared__ __align__(8) uint64_t bars[kAttnThreads / 32][NST];
    __shared__ int32_t ids[kAttnMaxSplitPages];
    // PDL: wait for the previous kernel (its block-table writes), then let
    // the next launch (a K2 over another layer may start early) become resident
    pdl_top();
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    const int i = blockIdx.x;
    const int sp = blockIdx.y;
    const int H = a.kv_heads;
    const int h = i % H;
    const int seq = i / H;
    const int t = a.table(s, i);
    const int col = a.col_elems(i);  // tensor-map column of this head's slice
    const int G = a.G;
    const int N = s.num_pages[t];
    const int p_begin = sp * a.pages_per_split;
    const int p_end = min(N, p_begin + a.pages_per_split);
    const int g = lane >> 2;
    const int tq = lane & 3;
    // SWIZZLE_128B destinations must be 1024-byte aligned: align the dynamic
    // shared memory base by hand (the launch adds 1 KB of slack)
    uint8_t* sbase = align1024(smem);
    uint8_t* stage = sbase + wid * NST * PAGE_SM;
    float* wpart_o = reinterpret_cast<float*>(sbase + nw * NST * PAGE_SM);
    float* wpart_ml = wpart_o + nw * G * D;
    uint32_t qa[KS][2];
    {
        const uint8_t* qrow = a.q + ((int64_t)seq * a.n_q_heads + h * G + min(g, G - 1)) * (D * 2);
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            qa[ks][0] = g < G ? *reinterpret_cast<const uint32_t*>(qrow + (16 * ks + 2 * tq) * 2) : 0u;
            qa[ks][1] = g < G ? *reinterpret_cast<const uint32_t*>(qrow + (16 * ks + 2 * tq + 8) * 2) : 0u;
        }
    }
    float o[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    float m = -INFINITY, l = 0.f;
    const int32_t* row = s.block_table + (int64_t)t * s.max_pages;
    const int my_n = (p_end - p_begin) > wid ? ((p_end - p_begin) - wid + nw - 1) / nw : 0;
    const bool ids_sm = p_end - p_begin <= kAttnMaxSplitPages;
    if (ids_sm)
        for (int j = threadIdx.x; j < p_end - p_begin; j += blockDim.x) ids[j] = __ldg(row + p_begin + j);
    if (lane < NST) mbar_init(&bars[wid][lane], 1);
    mbar_init_fence();
    __syncthreads();
    auto issue = [&](int k) {
        if (k < my_n && lane == 0) {
            const int pg = p_begin + wid + k * nw;
            const int32_t id = ids_sm ? ids[pg - p_begin] : __ldg(row + pg);
            tma_load_page(smem_u32(stage + (k % NST) * PAGE_SM), &bars[wid][k % NST], &tmap, id * 32, col, HALVES,
                          PAGE_SM);
        }
    };
    auto wait_stage = [&](int k) { mbar_wait(&bars[wid][k % NST], (k / NST) & 1); };
#pragma unroll
    for (int k = 0; k < NST - 1; ++k) issue(k);
    const uint32_t stage_s = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
    const int lm_j = lane >> 3, lm_r = lane & 7;
    for (int k = 0; k < my_n; ++k) {
        issue(k + NST - 1);
        wait_stage(k);
        const int pg = p_begin + wid + k * nw;
        const int fill = (pg == N - 1) ? s.newest_fill[t] : 16;
        const uint32_t st = stage_s + (k % NST) * PAGE_SM;
        float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            uint32_t b0, b1, b2, b3;
            const int tok = (lm_j >> 1) * 8 + lm_r;
            const int c = 2 * ks + (lm_j & 1);  // 16-byte chunk of d (8 elements)
            ldsm_x4(sw128(st + (c >> 3) * 4096, tok, c & 7), b0, b1, b2, b3);
            mma_bf16_16816(sc[0], qa[ks][0], qa[ks][1], b0, b1);
            mma_bf16_16816(sc[1], qa[ks][0], qa[ks][1], b2, b3);
        }
        float x[2][2];
        float rmax = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int tok = 8 * nt + 2 * tq + j;
                x[nt][j] = tok < fill ? sc[nt][j] * a.scale_log2 : -INFINITY;
                rmax = fmaxf(rmax, x[nt][j]);
            }
        }
        rmax = fmaxf(rmax, __shfl_xor_sync(0xFFFFFFFFu, rmax, 1));
        rmax = fmaxf(rmax, __shfl_xor_sync(0xFFFFFFFFu, rmax, 2));
        const float m_new = fmaxf(m, rmax);
        const float corr = exp2f(m - m_new);
        float rsum = 0.f;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                x[nt][j] = exp2f(x[nt][j] - m_new);
                rsum += x[nt][j];
            }
        }
        rsum += __shfl_xor_sync(0xFFFFFFFFu, rsum, 1);
        rsum += __shfl_xor_sync(0xFFFFFFFFu, rsum, 2);
        l = l * corr + rsum;
        m = m_new;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            o[nt][0] *= corr;
            o[nt][1] *= corr;
        }
        uint32_t ph0, pl0, ph1, pl1;
        split_bf16x2(x[0][0], x[0][1], ph0, pl0);
        split_bf16x2(x[1][0], x[1][1], ph1, pl1);
#pragma unroll
        for (int ntp = 0; ntp < NT / 2; ++ntp) {
            uint32_t b0, b1, b2, b3;
            const int tok = (lm_j & 1) * 8 + lm_r;
            const int c = 2 * ntp + (lm_j >> 1);
            ldsm_x4_t(sw128(st + (c >> 3) * 4096, 16 + tok, c & 7), b0, b1, b2, b3);
            mma_bf16_16816(o[2 * ntp], ph0, ph1, b0, b1);
            mma_bf16_16816(o[2 * ntp], pl0, pl1, b0, b1);
            mma_bf16_16816(o[2 * ntp + 1], ph0, ph1, b2, b3);
            mma_bf16_16816(o[2 * ntp + 1], pl0, pl1, b2, b3);
        }
        __syncwarp();
    }
    __syncthreads();
    if (g < G) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            wpart_o[(wid * G + g) * D + 8 * nt + 2 * tq] = o[nt][0];
            wpart_o[(wid * G + g) * D + 8 * nt + 2 * tq + 1] = o[nt][1];
        }
        if (tq == 0) {
            wpart_ml[(wid * G + g) * 2] = m;
            wpart_ml[(wid * G + g) * 2 + 1] = l;
        }
    }
    __syncthreads();
    const int n_splits = a.splits;
    for (int xi = threadIdx.x; xi < G * D; xi += blockDim.x) {
        const int gg = xi / D;
        float mm = -INFINITY;
        for (int w2 = 0; w2 < nw; ++w2) mm = fmaxf(mm, wpart_ml[(w2 * G + gg) * 2]);
        float ll = 0.f, oo = 0.f;
        for (int w2 = 0; w2 < nw; ++w2) {
            const float mw = wpart_ml[(w2 * G + gg) * 2];
            const float c = (mw == -INFINITY) ? 0.f : exp2f(mw - mm);
            ll += wpart_ml[(w2 * G + gg) * 2 + 1] * c;
            oo += wpart_o[(w2 * G + gg) * D + (xi % D)] * c;
        }
        if (n_splits == 1) {
            a.out[((int64_t)seq * a.n_q_heads + h * G + gg) * D + (xi % D)] = empty_guard(s, oo, ll);
            continue;
        }
        const int64_t pidx = ((int64_t)i * n_splits + sp) * G + gg;
        a.part_o[pidx * D + (xi % D)] = oo;
        if (xi % D == 0) {
            a.part_ml[pidx * 2] = mm;
            a.part_ml[pidx * 2 + 1] = ll;
        }
    }
    if (n_splits > 1) merge_if_last(s, a, i, D);
}

size_t attention_tma_smem(int d, int G) {
    const int nw = kAttnThreads / 32;
    return 1024 + (size_t)nw * 3 * 32 * 2 * d + (size_t)nw * G * d * 4 + (size_t)nw * G * 2 * 4;
}

void launch_attention_tma(int d, dim3 grid, size_t smem, cudaStream_t st, const DevState& s, const AttnArgs& a,
                          const void* tmap) {
    const CUtensorMap& tm = *reinterpret_cast<const CUtensorMap*>(tmap);
    if (d == 128) launch_pdl(attention_tma_kernel<128>, grid, dim3(kAttnThreads), smem, st, s, a, tm);
    else launch_pdl(attention_tma_kernel<64>, grid, dim3(kAttnThreads), smem, st, s, a, tm);
}

const void* attention_tma_fn(int d) {
    return d == 128 ? reinterpret_cast<const void*>(attention_tma_kernel<128>)
                    : reinterpret_cast<const void*>(attention_tma_kernel<64>);
}

}  // namespace pe
