// Kernel declarations and launch constants shared by the kernels and the
// host side of the engine.
#pragma once

#include <cstdlib>
#include <cstring>
#include <utility>

#include "pe_internal.cuh"

namespace pe {

constexpr int kAppendThreads = 128;      // 4 warps x 16 tables
constexpr int kAppendEpochPeriod = 0x3FFFFFFE;  // K0 epochs 1..period: even, so consecutive epochs alternate parity
constexpr int kEvictThreads = 128;       // 4 warps per CTA
constexpr int kMaxPagesPerCta = 288;
constexpr int kPrefillThreads = 128;     // score kernel: 4 warps per CTA
constexpr int kScoreTokensPerCta = 128;  // tokens (x all heads) per score CTA (64 when the keys would not fit)
constexpr int kScoreKeysMax = 1024;      // score CTA: keys staged in shared memory (8 KB)
constexpr int kPackThreads = 256;        // select kernel: 8 warps per CTA
constexpr int kPrefillCluster = 8;       // CTAs per table (portable cluster size)

struct PrefillArgs {
    const uint8_t* k;
    const uint8_t* v;
    int64_t token_stride;                // bytes between consecutive tokens of one table
    const int32_t* tab_len;              // [n_tab] L per launch table
    const int64_t* tab_tok0;             // [n_tab] first token index (cu_seqlens[s])
    const int32_t* tab_pagebase;         // [n_tab] exclusive prefix of pages popped
    int32_t* evicted_counts;             // [n_tab] or nullptr
    unsigned long long* keys;            // score keys, table i at tab_keybase[i]
    const int64_t* tab_keybase;          // [n_tab] exclusive prefix of L
    int32_t* surv;                       // survivor token indices, table i at tab_pagebase[i]*B
    int32_t n_tab;
    int32_t seq_begin, layer;
    int32_t chunk_cap;                   // max tokens per CTA (keys smem capacity)
    int32_t score_tokens;                // tokens (x all heads) per score CTA
    int32_t cta_len_max;                 // CTA select: tables longer than this are skipped
    int32_t cluster_len_min;             // cluster select: tables this short or shorter are skipped
    int32_t cand_cap;                    // streamed select: candidate list capacity (shared memory)
    int32_t bits_cap;                    // streamed select: eviction bitmap capacity in positions (0 = none)
    int32_t direct_identity;             // score kernel packs tables that keep every token (L <= C); copy skips them
    const int32_t* score_items;          // compact score grid: (sequence << 16 | token block) per CTA, or nullptr
    int32_t item_seq0;                   // sequence index (in the call) of the launch's first sequence
};

__global__ void evict_cached_kernel(DevState s, TableSet ts, double* scratch, int32_t* vpage, int32_t* victims,
                                    unsigned long long grid_last, int early);
__global__ void plan_prefill_kernel(DevState s, PrefillArgs a, int32_t total_pages, LaunchCtl* ctl);
__global__ void prefill_select_kernel(DevState s, PrefillArgs a, const LaunchCtl* ctl);
__global__ void prefill_select_cta_kernel(DevState s, PrefillArgs a, const LaunchCtl* ctl);
constexpr int kSelHistCopies = 8;        // private histogram copies in the CTA select kernel
constexpr int kSelCandCap = 4096;        // boundary-bin candidates compacted after the first radix pass
constexpr int kSelectCtaMaxLen = 34816;  // CTA-per-table select: 4 B of smem per token + 64 KB histograms + 16 KB candidates
constexpr int kSelCandCapStream = 16384;  // candidates of the streamed CTA select (no hi words in smem)
constexpr int kSelBitsMaxLen = 262144;    // streamed select: eviction bitmap (32 KB) for tables up to this length
__global__ void prefill_select_stream_kernel(DevState s, PrefillArgs a, const LaunchCtl* ctl);

// GPU-wide select (pe_select.cu): window / count / resolve / emit kernels
constexpr int kGselChunk = 2048;                    // positions per count / emit CTA
constexpr int kGselWords = kGselChunk / 32;         // eviction-bit words per chunk
constexpr int kGselSample = 1024;                   // sampled high words per table (window)
constexpr int kGselAll = 4096;                      // tables this short: every key is a candidate
constexpr int kGselCandCap = 8192;                  // candidates sorted in shared memory (96 KB)
constexpr int kGselMaxChunks = 128;                 // tables up to 128 chunks (262144 tokens)
constexpr int kGselMaxLen = kGselChunk * kGselMaxChunks;
constexpr int kGselMaxTies = 1024;                  // keys equal to the threshold resolved in the resolve kernel
constexpr int kGselMinLen = 16384;                  // calls with shorter tables only: the streamed CTA select
struct GselArgs {
    uint2* win;                          // [tables] high-word window (inclusive)
    int32_t* cand_n;                     // [tables] candidates appended
    unsigned long long* cand_key;        // [tables][cand_stride]
    int32_t* cand_pos;                   // [tables][cand_stride]
    int32_t* chunk_cnt;                  // [tables][chunk_stride] below counts, then survivor bases
    uint32_t* evbits;                    // [tables][chunk_stride][kGselWords] eviction bits
    int32_t* flag;                       // [tables] 1: the window missed, CTA-per-table select
    int32_t tab_off;                     // call-level index of the wave's first table
    int32_t cand_stride, chunk_stride;
    int32_t force_fallback;              // test knob (PE_SELECT=global_fallback)
};
__global__ void gsel_window_kernel(DevState s, PrefillArgs a, GselArgs g, const LaunchCtl* ctl);
__global__ void gsel_count_kernel(DevState s, PrefillArgs a, GselArgs g, const LaunchCtl* ctl);
__global__ void gsel_resolve_kernel(DevState s, PrefillArgs a, GselArgs g, const LaunchCtl* ctl);
__global__ void gsel_emit_kernel(DevState s, PrefillArgs a, GselArgs g, const LaunchCtl* ctl);
__global__ void gsel_fallback_kernel(DevState s, PrefillArgs a, GselArgs g, const LaunchCtl* ctl);
// The window from a strided sample of high words, one per thread of a
// kGselSample-thread CTA (both window kernels): bitonic sort (partner
// distances >= 32 through shared memory, shorter ones as warp shuffles),
// then the sample's boundary rank E*kGselSample/L +- 3.5 binomial sigma.
// The window holds the E-th key with overwhelming probability; the resolve
// kernel checks it exactly.
__device__ __forceinline__ uint2 gsel_window_of_sample(uint32_t x, uint32_t* samp, int E, int L) {
    const int tid = threadIdx.x;
    for (int k = 2; k <= kGselSample; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            const bool up = (tid & k) == 0;
            const bool lower = (tid & j) == 0;
            uint32_t y;
            if (j >= 32) {
                samp[tid] = x;
                __syncthreads();
                y = samp[tid ^ j];
                __syncthreads();
            } else {
                y = __shfl_xor_sync(0xFFFFFFFFu, x, j);
            }
            x = (lower == up) ? min(x, y) : max(x, y);
        }
    }
    samp[tid] = x;
    __syncthreads();
    const double p = static_cast<double>(E) / L;
    const int win = static_cast<int>(ceil(3.5 * sqrt(kGselSample * p * (1.0 - p)))) + 4;
    const int r = static_cast<int>(((int64_t)E * kGselSample) / L);
    const int lo = r - win, hi = r + win;
    return make_uint2(lo <= 0 ? 0u : samp[lo], hi >= kGselSample - 1 ? 0xFFFFFFFFu : samp[hi]);
}
__global__ void prefill_select_stream512_kernel(DevState s, PrefillArgs a, const LaunchCtl* ctl);
__global__ void prefill_copy_kernel(DevState s, PrefillArgs a, const LaunchCtl* ctl);
// the copy (PE_COPY_RESCORE=1: survivors rescored from the copied registers)
void launch_prefill_copy_any(int variant, dim3 grid, cudaStream_t st, const DevState& s, const PrefillArgs& a,
                             const LaunchCtl* ctl);
// persistent fused prefill (score units + per-table select/copy), pe_prefill.cu
void launch_prefill_fused_any(int variant, int grid, size_t smem, cudaStream_t st, const DevState& s,
                              const PrefillArgs& a, const LaunchCtl* ctl, const int32_t* items, int n_items,
                              int* work_ctr, int* seq_done, const int32_t* seq_units, int unit_tokens);
const void* prefill_fused_fn(int variant);

// host-side launchers of the row-geometry-specialised kernels (pe_score.cuh variants)
void launch_append_any(int variant, int blocks, cudaStream_t st, const DevState& s, const TableSet& ts,
                       const uint8_t* k, const uint8_t* v, const int64_t* pos, unsigned long long* lb,
                       unsigned long long* lbg,
                       LaunchCtl* ctl, unsigned long long ticket_base, int epoch, bool fast_ok);
void launch_evict_score_any(int variant, dim3 grid, int threads, cudaStream_t st, const DevState& s,
                            const TableSet& ts, int ppc, double* scratch, int32_t* tickets, int32_t* vpage,
                            int32_t* victims, unsigned long long grid_last, bool early);
void launch_prefill_score_any(int variant, dim3 grid, cudaStream_t st, const DevState& s, const PrefillArgs& a,
                              const LaunchCtl* ctl);

struct AttnArgs {
    const uint8_t* q;        // [n_seqs][n_q_heads][d]
    float* out;              // [n_seqs][n_q_heads][d]
    float* part_o;           // [n_tab][splits][G][d] split partial outputs
    float* part_ml;          // [n_tab][splits][G][2]  (max, sum)
    int32_t* tickets;        // [n_tab] split completion tickets (zero between launches)
    int32_t layer, G, n_q_heads, splits, pages_per_split;
    float scale_log2;        // log2(e)/sqrt(d)
    // Attention heads vs tables: launch item i = seq * kv_heads + h. A
    // PER_KV_HEAD table holds one KV head (heads_per_table = 1); a PER_LAYER
    // table holds every KV head of the layer, head h in columns
    // [h*d, (h+1)*d) of each row (kv_vector.hpp:23-27; attention.cpp:23-35
    // slices the concatenated row the same way).
    int32_t kv_heads, heads_per_table, d;
    __device__ __forceinline__ int table(const DevState& s, int i) const {
        const int seq = i / kv_heads, h = i - seq * kv_heads;
        return (seq * s.n_layers + layer) * s.tab_heads + h / heads_per_table;
    }
    __device__ __forceinline__ int col_elems(int i) const { return (i % kv_heads) % heads_per_table * d; }
};
__global__ void attention_split_kernel(DevState s, AttnArgs a);
// tensor-core variant (bf16, B = 16, d in {64, 128}, G <= 8)
size_t attention_mma_smem(int d, int G);
void launch_attention_mma(int d, dim3 grid, size_t smem, cudaStream_t st, const DevState& s, const AttnArgs& a);
const void* attention_mma_fn(int d);
// TMA (tensor map, SWIZZLE_128B) staging variant for d in {64, 128} (pe_attention.cu)
size_t attention_tma_smem(int d, int G);
void launch_attention_tma(int d, dim3 grid, size_t smem, cudaStream_t st, const DevState& s, const AttnArgs& a,
                          const void* tmap);
const void* attention_tma_fn(int d);

// table-granular kernels (pe_table.cu)
__global__ void pool_allocate_kernel(DevState s, int32_t* out);
__global__ void pool_release_kernel(DevState s, int32_t id);
__global__ void table_free_page_kernel(DevState s, int32_t t, int32_t idx);
__global__ void table_clear_kernel(DevState s, int32_t t);
__global__ void table_attend_kernel(DevState s, int32_t t, const float* q, int32_t head_dim, double* logits,
                                    float* out, double* weight_sums);
__global__ void token_evict_kernel(DevState s, int32_t t, int32_t rule, long long arg, int32_t C, long long newest,
                                   float* mean, long long* out);
__global__ void token_evict_batch_kernel(DevState s, TableSet ts, int32_t rule, long long arg, int32_t C,
                                         const int64_t* newest_pos, int64_t* victims, int32_t* vpage,
                                         unsigned long long grid_last);
__global__ void prompt_mean_key_kernel(const float* k, int n, int w, float* mean, double* mnorm);
__global__ void prompt_score_kernel(const float* k, int n, int w, int rule, const float* mean, const double* mnorm,
                                    const long long* pos, int n_pad, double* score, long long* spos, int* sidx);
__global__ void bitonic_step_kernel(double* score, long long* spos, int* sidx, int n_pad, int j, int k);
__global__ void flag_first_kernel(const int* sidx, int k, uint8_t* flags);
__global__ void invariants_tables_kernel(DevState s, int32_t* refs, unsigned long long* counters);
// step-log capture (pe_step_log_capture): one entry per launch table
__global__ void step_log_kernel(DevState s, TableSet ts, const int32_t* victims, pe_step_entry* out);
__global__ void invariants_free_kernel(DevState s, int32_t* refs);
__global__ void invariants_refs_kernel(DevState s, const int32_t* refs, unsigned long long* counters);
__global__ void probe_read_kernel(const uint4* src, size_t n16, unsigned long long* sink);
__global__ void probe_copy_kernel(const uint4* src, uint4* dst, size_t n16);

// Launch with programmatic stream serialization (kernels that start with
// pdl_top(), or K2's early path) unless PE_PDL=0.
inline bool pdl_enabled() {
    const char* v = std::getenv("PE_PDL");
    return !(v != nullptr && std::strcmp(v, "0") == 0);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace pe
