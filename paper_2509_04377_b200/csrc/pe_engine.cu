// Host side of the C-ABI (include/pe.h): engine lifecycle, argument
// validation (mirroring the reference's exceptions as pe_status codes),
// host-buffer staging, and the launch sequences of K0/K1/K2/K3.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "pe_kernels.cuh"
#include "pe_score.cuh"

using namespace pe;

namespace {

// append look-back words: one per K0 CTA (64 tables each), then one per
// group of 32 CTAs
size_t lb_cta_words(int64_t n_tables) { return (size_t)n_tables / 64 + 2; }
size_t lb_words(int64_t n_tables) { return lb_cta_words(n_tables) + lb_cta_words(n_tables) / 32 + 2; }

thread_local std::string g_err;

pe_status fail(pe_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

#define PE_CUDA(call)                                                                  \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess) {                                                       \
            return fail(PE_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_)); \
        }                                                                              \
    } while (0)

template <typename T>
cudaError_t dalloc(T** p, size_t n) {
    return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T));
}

bool is_device_ptr(const void* p) {
    if (p == nullptr) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

struct pe_engine {
    pe_config cfg{};
    DevState s{};
    int device = 0;
    int sm_count = 0;
    int32_t tab_heads = 0;
    // scratch
    LaunchCtl* ctl = nullptr;
    int32_t* rank = nullptr;
    int32_t* work = nullptr;
    int32_t* victims = nullptr;
    pe_step_entry* step_stage = nullptr;  // [n_tables] step-log staging for host destinations (lazy)
    int32_t* tickets = nullptr;
    int32_t* vpage = nullptr;           // per launch table released page id (or -1)
    unsigned long long* lb_status = nullptr;  // append look-back status words (one per CTA)
    int append_epoch = 0;
    // K0 no-pop fast path: the previous engine operation was an all-table
    // append over the same layer range (the device flag written by that
    // launch then says whether any table will pop on this one)
    bool append_chain = false;
    int32_t chain_layer0 = -1, chain_layers = 0;
    unsigned long long grid_tickets = 0;  // host mirror of DevState::grid_ctr
    // K2 PDL chain: the engine's last launch was a recompute K2 (or a
    // tensor-core attention) over the contiguous layer range
    // [k2_layer0, k2_layer0 + k2_layers) on k2_stream
    bool k2_chain = false;
    int32_t k2_layer0 = 0, k2_layers = 0;
    cudaStream_t k2_stream = nullptr;
    double* evict_scratch = nullptr;
    int32_t* tab_len = nullptr;
    int64_t* tab_tok0 = nullptr;
    int32_t* tab_pagebase = nullptr;
    int32_t* evicted_dev = nullptr;
    int64_t* tab_keybase = nullptr;
    int64_t* h_tab_keybase = nullptr;   // pinned
    unsigned long long* keys = nullptr;
    size_t keys_elems = 0;
    int32_t* surv = nullptr;
    size_t surv_elems = 0;
    // GPU-wide select scratch (pe_select.cu), sized per prefill call
    uint2* gs_win = nullptr;
    size_t gs_win_elems = 0;
    int32_t* gs_tab = nullptr;  // cand_n and flag, [2][tables]
    size_t gs_tab_elems = 0;
    unsigned long long* gs_ckey = nullptr;
    size_t gs_ckey_elems = 0;
    int32_t* gs_cpos = nullptr;
    size_t gs_cpos_elems = 0;
    int32_t* gs_chunk = nullptr;
    size_t gs_chunk_elems = 0;
    uint32_t* gs_bits = nullptr;
    size_t gs_bits_elems = 0;
    int variant = 0;
    int32_t* h_tab_len = nullptr;       // pinned
    int64_t* h_tab_tok0 = nullptr;      // pinned
    int32_t* h_tab_pagebase = nullptr;  // pinned
    // staging ring for host buffers: H2D copies run on copy_stream, overlapping
    // the engine's kernels; slot reuse is guarded by "consumed" events
    static constexpr int kRing = 64;  // a whole decode cycle of host inputs can be staged ahead
    static constexpr size_t kRingSlotCap = size_t(64) << 20;  // larger inputs get private buffers
    struct Slot {
        uint8_t* big = nullptr;          // private buffer for inputs > kRingSlotCap
        size_t big_bytes = 0;
        cudaEvent_t ready = nullptr;     // copy done (copy_stream)
        cudaEvent_t consumed = nullptr;  // last reader done (compute stream)
    } ring[kRing];
    int ring_next = 0;
    uint8_t* ring_arena = nullptr;       // kRing slots of ring_slot_bytes each
    size_t ring_slot_bytes = 0;
    int pending[4];                      // slots staged by the current call
    int n_pending = 0;
    cudaStream_t copy_stream = nullptr;
    cudaStream_t aux_stream = nullptr;   // second prefill wave stream
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_score = nullptr;      // prefill: the previous wave's score kernel is done (chained waves)
    cudaEvent_t ev_meta = nullptr;       // prefill metadata H2D copies done
    float* part_o = nullptr;
    size_t part_o_elems = 0;
    float* part_ml = nullptr;
    size_t part_ml_elems = 0;
    float* out_stage = nullptr;
    size_t out_stage_elems = 0;
    pe_stats stats{};
    int max_dyn_prefill = 0, max_dyn_attn = 0;
    // table-granular API (pe_table_*, pe_pool_*)
    int32_t* alloc_out = nullptr;
    int64_t* tok_out = nullptr;
    int64_t* tok_newest = nullptr;   // [n_seqs] staged newest positions (batched token eviction, lazy)
    size_t tok_newest_elems = 0;
    int64_t* tok_victims = nullptr;  // [n_tables] victim positions for host destinations (lazy)
    size_t tok_victims_elems = 0;
    int32_t* attn_tickets = nullptr;  // [n_tables] split-K completion tickets
    alignas(64) CUtensorMap pool_tmap;  // pages as [capacity*2*B rows][d] bf16, SWIZZLE_128B boxes of 32x64
    bool has_tmap = false;
    // fused prefill schedule (prefill_fused_kernel)
    int32_t* h_items = nullptr;          // pinned
    size_t h_items_elems = 0;
    int32_t* items = nullptr;
    size_t items_elems = 0;
    int32_t* h_seq_units = nullptr;      // pinned [n_seqs]
    int32_t* seq_units = nullptr;        // [n_seqs]
    int32_t* seq_done = nullptr;         // [n_seqs]
    int32_t* work_ctr = nullptr;
    double* attend_logits = nullptr;
    size_t attend_logits_elems = 0;
    float* attend_out = nullptr;
    size_t attend_out_elems = 0;
    double* attend_ws = nullptr;
    size_t attend_ws_elems = 0;
};

namespace {

template <typename T>
pe_status ensure_t(T** buf, size_t* have, size_t need) {
    if (*have >= need) return PE_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *have = 0;
    PE_CUDA(dalloc(buf, need));
    *have = need;
    return PE_OK;
}

// Device view of an input buffer: device pointers pass through; host
// buffers are copied into the next staging-ring slot on the engine's copy
// stream (so the H2D transfer overlaps kernels already queued on `st`), and
// `st` waits for that copy. mark_consumed() after the call's launches
// releases the slots.
pe_status as_device(pe_engine* e, const void* p, size_t bytes, cudaStream_t st, const uint8_t** out) {
    if (p == nullptr) return fail(PE_INVALID_ARG, "null buffer");
    if (is_device_ptr(p)) {
        *out = static_cast<const uint8_t*>(p);
        return PE_OK;
    }
    const int k = e->ring_next;
    e->ring_next = (e->ring_next + 1) % pe_engine::kRing;
    pe_engine::Slot& sl = e->ring[k];
    if (bytes > pe_engine::kRingSlotCap) {
        // large inputs (a prefill layer from host memory): a private buffer per slot
        if (sl.big_bytes < bytes) {
            PE_CUDA(cudaEventSynchronize(sl.consumed));
            if (sl.big) PE_CUDA(cudaFree(sl.big));
            sl.big = nullptr;
            sl.big_bytes = 0;
            PE_CUDA(cudaMalloc(&sl.big, bytes));
            sl.big_bytes = bytes;
        }
    } else if (e->ring_slot_bytes < bytes) {
        // grow the whole ring at once (one arena, every slot the same size)
        // so no slot has to grow later in the middle of a pipelined cycle
        for (auto& other : e->ring) PE_CUDA(cudaEventSynchronize(other.consumed));
        PE_CUDA(cudaStreamSynchronize(e->copy_stream));
        const size_t slot = (bytes + 255) & ~size_t(255);
        if (e->ring_arena) PE_CUDA(cudaFree(e->ring_arena));
        e->ring_arena = nullptr;
        e->ring_slot_bytes = 0;
        PE_CUDA(cudaMalloc(&e->ring_arena, slot * pe_engine::kRing));
        e->ring_slot_bytes = slot;
    }
    uint8_t* dst = bytes > pe_engine::kRingSlotCap ? sl.big : e->ring_arena + (size_t)k * e->ring_slot_bytes;
    PE_CUDA(cudaStreamWaitEvent(e->copy_stream, sl.consumed, 0));
    PE_CUDA(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, e->copy_stream));
    PE_CUDA(cudaEventRecord(sl.ready, e->copy_stream));
    PE_CUDA(cudaStreamWaitEvent(st, sl.ready, 0));
    if (e->n_pending < 4) e->pending[e->n_pending++] = k;
    *out = dst;
    return PE_OK;
}

void mark_consumed(pe_engine* e, cudaStream_t st) {
    for (int i = 0; i < e->n_pending; ++i) cudaEventRecord(e->ring[e->pending[i]].consumed, st);
    e->n_pending = 0;
}

int32_t elt_size(int32_t dtype) { return dtype == PE_DTYPE_BF16 ? 2 : 4; }

pe_status check_launch(pe_engine* e, const char* what) {
    if (e != nullptr) e->k2_chain = false;  // any other launch breaks the K2 PDL chain
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return fail(PE_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(err));
    return PE_OK;
}


}  // namespace

extern "C" {

int32_t pe_abi_version(void) { return PE_ABI_VERSION; }

const char* pe_last_error(void) { return g_err.c_str(); }

const char* pe_status_string(pe_status s) {
    switch (s) {
    case PE_OK: return "ok";
    case PE_ERROR: return "error";
    case PE_POOL_EXHAUSTED: return "page pool exhausted";
    case PE_INDEX_OUT_OF_RANGE: return "index out of range";
    case PE_UNKNOWN_POSITION: return "unknown position";
    case PE_OVERFLOW: return "overflow";
    case PE_EMPTY_PAGE: return "page has no occupied slots";
    case PE_K_TOO_LARGE: return "k too large";
    case PE_NO_ELIGIBLE_PAGE: return "no eligible page to rank";
    case PE_BUDGET_INVALID: return "budget invalid";
    case PE_EMPTY_CACHE: return "attention requires at least one retained token";
    case PE_LENGTH_MISMATCH: return "length mismatch";
    case PE_EMPTY_INPUT: return "empty input";
    case PE_IO_ERROR: return "io error";
    case PE_INVALID_ARG: return "invalid argument";
    case PE_INVALID_STATE: return "invalid state";
    case PE_CUDA_ERROR: return "cuda error";
    case PE_NO_DEVICE: return "no usable sm_100 device";
    }
    return "unknown status";
}

pe_status pe_engine_create(const pe_config* cfg_in, pe_engine** out) {
    if (cfg_in == nullptr || out == nullptr) return fail(PE_INVALID_ARG, "null argument");
    *out = nullptr;
    pe_config c = *cfg_in;
    // PolicyConfig::validate (policy.cpp:38-52)
    if (c.page_size <= 0) return fail(PE_BUDGET_INVALID, "page size must be positive");
    if (c.cache_budget < c.page_size)
        return fail(PE_BUDGET_INVALID, "budget must be at least one page (" + std::to_string(c.page_size) + " tokens)");
    if (c.cache_budget % c.page_size != 0) return fail(PE_BUDGET_INVALID, "budget must be a multiple of page size");
    if (c.policy != PE_POLICY_PAGED_EVICTION && c.policy != PE_POLICY_FULL_CACHE)
        return fail(PE_INVALID_ARG, "policy must be PagedEviction or FullCache");
    if (c.dtype != PE_DTYPE_F32 && c.dtype != PE_DTYPE_BF16) return fail(PE_INVALID_ARG, "dtype");
    if (c.granularity != PE_GRANULARITY_PER_KV_HEAD && c.granularity != PE_GRANULARITY_PER_LAYER)
        return fail(PE_INVALID_ARG, "granularity");
    if (c.n_seqs <= 0 || c.n_layers <= 0 || c.n_kv_heads <= 0 || c.head_dim <= 0)
        return fail(PE_INVALID_ARG, "geometry must be positive");
    const int32_t tab_heads = c.granularity == PE_GRANULARITY_PER_KV_HEAD ? c.n_kv_heads : 1;
    const int32_t w = c.granularity == PE_GRANULARITY_PER_KV_HEAD ? c.head_dim : c.n_kv_heads * c.head_dim;
    const int32_t row_bytes = w * elt_size(c.dtype);
    if (row_bytes % 16 != 0)
        return fail(PE_INVALID_ARG, "row width * element size must be a multiple of 16 bytes");
    const int64_t n_tables64 = (int64_t)c.n_seqs * c.n_layers * tab_heads;
    if (n_tables64 > (1 << 30)) return fail(PE_OVERFLOW, "too many tables");
    const int32_t n_tables = static_cast<int32_t>(n_tables64);
    int32_t max_pages = c.max_pages_per_table;
    if (max_pages <= 0) {
        if (c.policy == PE_POLICY_FULL_CACHE)
            return fail(PE_INVALID_ARG, "FullCache needs max_pages_per_table");
        max_pages = c.cache_budget / c.page_size + 1;
    }
    int64_t cap = c.capacity > 0 ? c.capacity : (int64_t)n_tables * max_pages;
    if (cap >= (int64_t)1 << 31) return fail(PE_OVERFLOW, "pool capacity exceeds int32 page ids");

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(PE_NO_DEVICE, "no CUDA device");
    }
    if (c.device < 0 || c.device >= ndev) return fail(PE_NO_DEVICE, "device ordinal out of range");
    cudaDeviceProp prop{};
    PE_CUDA(cudaGetDeviceProperties(&prop, c.device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(PE_NO_DEVICE, "engine is built for sm_100a (B200); device is sm_" +
                                      std::to_string(prop.major) + std::to_string(prop.minor));
    PE_CUDA(cudaSetDevice(c.device));

    auto* e = new pe_engine();
    e->cfg = c;
    e->device = c.device;
    e->sm_count = prop.multiProcessorCount;
    e->tab_heads = tab_heads;
    e->variant = score_variant(c.dtype, row_bytes);
    DevState& s = e->s;
    s.capacity = static_cast<int32_t>(cap);
    s.B = c.page_size;
    s.C = c.cache_budget;
    s.w = w;
    s.row_bytes = row_bytes;
    s.pitch = row_bytes;
    s.max_pages = max_pages;
    s.n_tables = n_tables;
    s.n_seqs = c.n_seqs;
    s.n_layers = c.n_layers;
    s.tab_heads = tab_heads;
    s.dtype = c.dtype;
    s.policy = c.policy;

    auto cleanup_fail = [&](pe_status st) {
        pe_engine_destroy(e);
        return st;
    };
    const size_t page_bytes = (size_t)2 * s.B * s.pitch;
    const size_t attn_items = std::max<size_t>((size_t)n_tables, (size_t)c.n_seqs * c.n_kv_heads);
    if (cudaMalloc(&s.pages, (size_t)cap * page_bytes) != cudaSuccess ||
        dalloc(&s.positions, (size_t)cap * s.B) != cudaSuccess ||
        dalloc(&s.token_scores, (size_t)cap * s.B) != cudaSuccess ||
        dalloc(&s.page_scores, (size_t)cap) != cudaSuccess ||
        dalloc(&s.block_table, (size_t)n_tables * max_pages) != cudaSuccess ||
        dalloc(&s.num_pages, n_tables) != cudaSuccess || dalloc(&s.newest_fill, n_tables) != cudaSuccess ||
        dalloc(&s.retained, n_tables) != cudaSuccess || dalloc(&s.stack, (size_t)cap) != cudaSuccess ||
        dalloc(&s.top, 1) != cudaSuccess || dalloc(&s.status, 1) != cudaSuccess ||
        dalloc(&s.evict_count, 1) != cudaSuccess || dalloc(&s.grid_ctr, 1) != cudaSuccess ||
        dalloc(&s.holes, (size_t)cap) != cudaSuccess ||
        dalloc(&e->vpage, n_tables) != cudaSuccess || dalloc(&e->ctl, 1) != cudaSuccess ||
        dalloc(&e->alloc_out, 1) != cudaSuccess || dalloc(&e->tok_out, 1) != cudaSuccess ||
        dalloc(&e->attn_tickets, attn_items) != cudaSuccess ||
        dalloc(&e->seq_units, c.n_seqs) != cudaSuccess || dalloc(&e->seq_done, c.n_seqs) != cudaSuccess ||
        dalloc(&e->work_ctr, 1) != cudaSuccess ||
        dalloc(&e->lb_status, lb_words(n_tables)) != cudaSuccess ||
        dalloc(&e->rank, n_tables) != cudaSuccess || dalloc(&e->work, n_tables) != cudaSuccess ||
        dalloc(&e->victims, n_tables) != cudaSuccess || dalloc(&e->tickets, n_tables) != cudaSuccess ||
        dalloc(&e->evict_scratch, (size_t)n_tables * max_pages) != cudaSuccess ||
        dalloc(&e->tab_len, (size_t)c.n_seqs * tab_heads) != cudaSuccess ||
        dalloc(&e->tab_tok0, (size_t)c.n_seqs * tab_heads) != cudaSuccess ||
        dalloc(&e->tab_pagebase, (size_t)c.n_seqs * tab_heads) != cudaSuccess ||
        dalloc(&e->evicted_dev, (size_t)c.n_seqs * tab_heads) != cudaSuccess ||
        dalloc(&e->tab_keybase, (size_t)c.n_seqs * tab_heads) != cudaSuccess) {
        cudaGetLastError();
        return cleanup_fail(fail(PE_CUDA_ERROR, "device allocation failed (pool of " +
                                                    std::to_string(cap) + " pages)"));
    }
    if (cudaMallocHost(&e->h_tab_len, sizeof(int32_t) * c.n_seqs * tab_heads) != cudaSuccess ||
        cudaMallocHost(&e->h_tab_tok0, sizeof(int64_t) * c.n_seqs * tab_heads) != cudaSuccess ||
        cudaMallocHost(&e->h_tab_pagebase, sizeof(int32_t) * c.n_seqs * tab_heads) != cudaSuccess ||
        cudaMallocHost(&e->h_tab_keybase, sizeof(int64_t) * c.n_seqs * tab_heads) != cudaSuccess ||
        cudaMallocHost(&e->h_seq_units, sizeof(int32_t) * c.n_seqs) != cudaSuccess) {
        cudaGetLastError();
        return cleanup_fail(fail(PE_CUDA_ERROR, "pinned allocation failed"));
    }
    // LIFO free list initialised [cap-1, ..., 0] (page_pool.cpp:18-21)
    {
        std::vector<int32_t> stack(cap);
        for (int64_t i = 0; i < cap; ++i) stack[i] = static_cast<int32_t>(cap - 1 - i);
        const int32_t top = static_cast<int32_t>(cap);
        if (cudaMemcpy(s.stack, stack.data(), sizeof(int32_t) * cap, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(s.top, &top, sizeof(int32_t), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemset(s.block_table, 0xFF, sizeof(int32_t) * (size_t)n_tables * max_pages) != cudaSuccess ||
            cudaMemset(s.num_pages, 0, sizeof(int32_t) * n_tables) != cudaSuccess ||
            cudaMemset(s.newest_fill, 0, sizeof(int32_t) * n_tables) != cudaSuccess ||
            cudaMemset(s.retained, 0, sizeof(int32_t) * n_tables) != cudaSuccess ||
            cudaMemset(s.status, 0, sizeof(int32_t)) != cudaSuccess ||
            cudaMemset(s.evict_count, 0, sizeof(unsigned long long)) != cudaSuccess ||
            cudaMemset(s.grid_ctr, 0, sizeof(unsigned long long)) != cudaSuccess ||
            cudaMemset(e->tickets, 0, sizeof(int32_t) * n_tables) != cudaSuccess ||
            cudaMemset(e->attn_tickets, 0, sizeof(int32_t) * attn_items) != cudaSuccess ||
            cudaMemset(e->lb_status, 0, sizeof(unsigned long long) * lb_words(n_tables)) != cudaSuccess ||
            cudaMemset(e->ctl, 0, sizeof(LaunchCtl)) != cudaSuccess ||
            cudaMemset(e->victims, 0xFF, sizeof(int32_t) * n_tables) != cudaSuccess ||
            cudaMemset(s.positions, 0xFF, sizeof(int32_t) * (size_t)cap * s.B) != cudaSuccess ||
            cudaMemset(s.holes, 0, sizeof(unsigned long long) * (size_t)cap) != cudaSuccess ||
            cudaMemset(s.pages, 0, (size_t)cap * page_bytes) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess) {
            cudaGetLastError();
            return cleanup_fail(fail(PE_CUDA_ERROR, "state initialisation failed"));
        }
    }
    if (cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&e->aux_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_score, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_meta, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return cleanup_fail(fail(PE_CUDA_ERROR, "copy stream creation failed"));
    }
    for (auto& sl : e->ring) {
        if (cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&sl.consumed, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            return cleanup_fail(fail(PE_CUDA_ERROR, "event creation failed"));
        }
    }
    // kernel attributes: allow dynamic smem up to the opt-in limit minus the static part
    {
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device);
        auto allow = [&](const void* fn, int* out) -> bool {
            cudaFuncAttributes fa{};
            if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess) return false;
            *out = optin - static_cast<int>(fa.sharedSizeBytes);
            return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, *out) == cudaSuccess;
        };
        int mma64 = 0, mma128 = 0, sel_cta = 0;
        if (!allow(reinterpret_cast<const void*>(prefill_select_kernel), &e->max_dyn_prefill) ||
            !allow(reinterpret_cast<const void*>(attention_split_kernel), &e->max_dyn_attn) ||
            !allow(attention_mma_fn(64), &mma64) || !allow(attention_mma_fn(128), &mma128) ||
            !allow(reinterpret_cast<const void*>(prefill_select_cta_kernel), &sel_cta) ||
            !allow(reinterpret_cast<const void*>(prefill_select_stream_kernel), &sel_cta) ||
            !allow(reinterpret_cast<const void*>(prefill_select_stream512_kernel), &sel_cta) ||
            !allow(reinterpret_cast<const void*>(gsel_resolve_kernel), &sel_cta) ||
            !allow(reinterpret_cast<const void*>(gsel_fallback_kernel), &sel_cta) ||
            !allow(prefill_fused_fn(e->variant), &sel_cta)) {
            cudaGetLastError();
            return cleanup_fail(fail(PE_CUDA_ERROR, "cudaFuncSetAttribute(max dynamic smem) failed"));
        }
    }
    // tensor map over the pool for the TMA attention variant (bf16, d = 128, B = 16)
    if (c.dtype == PE_DTYPE_BF16 && (c.head_dim == 128 || c.head_dim == 64) && s.B == 16) {
        using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                         const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                         CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                         CUtensorMapFloatOOBfill);
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) == cudaSuccess && fn) {
            const cuuint64_t dims[2] = {(cuuint64_t)s.w, (cuuint64_t)cap * 2 * s.B};
            const cuuint64_t strides[1] = {(cuuint64_t)s.pitch};
            const cuuint32_t box[2] = {64, 32};
            const cuuint32_t estr[2] = {1, 1};
            e->has_tmap = reinterpret_cast<EncodeTiled>(fn)(
                              &e->pool_tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, s.pages, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
        cudaGetLastError();
        int tma_smem = 0;
        cudaFuncAttributes fa{};
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device);
        if (cudaFuncGetAttributes(&fa, attention_tma_fn(c.head_dim)) == cudaSuccess) {
            tma_smem = optin - static_cast<int>(fa.sharedSizeBytes);
            cudaFuncSetAttribute(attention_tma_fn(c.head_dim), cudaFuncAttributeMaxDynamicSharedMemorySize, tma_smem);
        }
        cudaGetLastError();
    }
    *out = e;
    return PE_OK;
}

pe_status pe_engine_destroy(pe_engine* e) {
    if (e == nullptr) return PE_OK;
    cudaSetDevice(e->device);
    cudaDeviceSynchronize();
    DevState& s = e->s;
    void* dev[] = {s.holes, s.pages, s.positions, s.token_scores, s.page_scores, s.block_table, s.num_pages,
                   s.newest_fill, s.retained, s.stack, s.top, s.status, s.evict_count, s.grid_ctr, e->vpage,
                   e->ctl, e->rank,
                   e->work, e->victims, e->tickets, e->evict_scratch, e->tab_len, e->tab_tok0,
                   e->tab_pagebase, e->evicted_dev, e->part_o,
                   e->part_ml, e->out_stage, e->tab_keybase, e->keys, e->surv, e->gs_win, e->gs_tab, e->gs_ckey, e->gs_cpos,
                   e->gs_chunk, e->gs_bits, e->lb_status,
                   e->alloc_out, e->tok_out, e->attn_tickets, e->items, e->seq_units, e->seq_done, e->work_ctr, e->attend_logits, e->attend_out, e->attend_ws, e->step_stage, e->tok_newest, e->tok_victims};
    for (void* p : dev) {
        if (p) cudaFree(p);
    }
    if (e->ring_arena) cudaFree(e->ring_arena);
    for (auto& sl : e->ring) {
        if (sl.big) cudaFree(sl.big);
        if (sl.ready) cudaEventDestroy(sl.ready);
        if (sl.consumed) cudaEventDestroy(sl.consumed);
    }
    if (e->copy_stream) cudaStreamDestroy(e->copy_stream);
    if (e->aux_stream) cudaStreamDestroy(e->aux_stream);
    if (e->ev_fork) cudaEventDestroy(e->ev_fork);
    if (e->ev_join) cudaEventDestroy(e->ev_join);
    if (e->ev_score) cudaEventDestroy(e->ev_score);
    if (e->ev_meta) cudaEventDestroy(e->ev_meta);
    if (e->h_tab_len) cudaFreeHost(e->h_tab_len);
    if (e->h_tab_tok0) cudaFreeHost(e->h_tab_tok0);
    if (e->h_tab_pagebase) cudaFreeHost(e->h_tab_pagebase);
    if (e->h_tab_keybase) cudaFreeHost(e->h_tab_keybase);
    if (e->h_items) cudaFreeHost(e->h_items);
    if (e->h_seq_units) cudaFreeHost(e->h_seq_units);
    cudaGetLastError();
    delete e;
    return PE_OK;
}

// ------------------------------------------------------------------ K1
pe_status pe_prefill_prune_pack(pe_engine* e, int32_t layer, const void* k, const void* v,
                                const int32_t* cu_seqlens, int32_t seq_begin, int32_t n_seqs,
                                int32_t* evicted_counts, void* stream) {
    if (e != nullptr) e->append_chain = false;  // tables change outside the append chain
    if (e == nullptr) return fail(PE_INVALID_ARG, "null engine");
    const DevState& s = e->s;
    if (layer < 0 || layer >= s.n_layers) return fail(PE_INVALID_ARG, "layer out of range");
    if (seq_begin < 0 || n_seqs <= 0 || seq_begin + n_seqs > s.n_seqs)
        return fail(PE_INVALID_ARG, "sequence range out of range");
    if (cu_seqlens == nullptr) return fail(PE_INVALID_ARG, "cu_seqlens");
    if (cu_seqlens[0] != 0) return fail(PE_INVALID_ARG, "cu_seqlens[0] must be 0");
    cudaSetDevice(e->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int H = s.tab_heads;
    const int n_tab = n_seqs * H;
    int64_t total_pages = 0;
    int64_t total_keys = 0;
    int max_len = 0;
    int max_short = 0;  // longest table the CTA-per-table select can hold
    // the pinned per-table arrays are still being copied by the previous call
    // until its metadata event fires
    PE_CUDA(cudaEventSynchronize(e->ev_meta));
    for (int q = 0; q < n_seqs; ++q) {
        const int L = cu_seqlens[q + 1] - cu_seqlens[q];
        if (L <= 0) return fail(PE_ERROR, "prefill requires at least one token");  // policy.cpp:57-58
        const int keep = (s.policy == PE_POLICY_PAGED_EVICTION && L > s.C) ? s.C : L;
        const int np = (keep + s.B - 1) / s.B;
        if (np > s.max_pages)
            return fail(PE_INVALID_ARG, "prefill of " + std::to_string(L) + " tokens exceeds max_pages_per_table");
        max_len = std::max(max_len, L);
        if (L <= kSelectCtaMaxLen) max_short = std::max(max_short, L);
        for (int h = 0; h < H; ++h) {
            const int i = q * H + h;
            e->h_tab_len[i] = L;
            e->h_tab_tok0[i] = cu_seqlens[q];
            e->h_tab_pagebase[i] = static_cast<int32_t>(total_pages);
            e->h_tab_keybase[i] = total_keys;
            total_pages += np;
            total_keys += L;
        }
    }
    const int chunk_cap = (max_len + kPrefillCluster - 1) / kPrefillCluster;
    const size_t pack_smem = (size_t)chunk_cap * 12 + 16;  // keys + two u16 candidate lists
    const size_t tokens = cu_seqlens[n_seqs];
    const size_t in_bytes = tokens * (size_t)H * s.row_bytes;
    const uint8_t *dk = nullptr, *dv = nullptr;
    e->n_pending = 0;
    pe_status r = as_device(e, k, in_bytes, st, &dk);
    if (r != PE_OK) return r;
    r = as_device(e, v, in_bytes, st, &dv);
    if (r != PE_OK) return r;
    r = ensure_t(&e->keys, &e->keys_elems, (size_t)total_keys);
    if (r != PE_OK) return r;
    r = ensure_t(&e->surv, &e->surv_elems, (size_t)total_pages * s.B);
    if (r != PE_OK) return r;
    PE_CUDA(cudaMemcpyAsync(e->tab_len, e->h_tab_len, sizeof(int32_t) * n_tab, cudaMemcpyHostToDevice, st));
    PE_CUDA(cudaMemcpyAsync(e->tab_tok0, e->h_tab_tok0, sizeof(int64_t) * n_tab, cudaMemcpyHostToDevice, st));
    PE_CUDA(cudaMemcpyAsync(e->tab_pagebase, e->h_tab_pagebase, sizeof(int32_t) * n_tab, cudaMemcpyHostToDevice, st));
    PE_CUDA(cudaMemcpyAsync(e->tab_keybase, e->h_tab_keybase, sizeof(int64_t) * n_tab, cudaMemcpyHostToDevice, st));
    PE_CUDA(cudaEventRecord(e->ev_meta, st));
    const bool ev_dev = evicted_counts && is_device_ptr(evicted_counts);
    PrefillArgs a{};
    a.k = dk;
    a.v = dv;
    a.token_stride = (int64_t)H * s.row_bytes;
    a.tab_len = e->tab_len;
    a.tab_tok0 = e->tab_tok0;
    a.tab_pagebase = e->tab_pagebase;
    a.evicted_counts = evicted_counts ? (ev_dev ? evicted_counts : e->evicted_dev) : nullptr;
    a.keys = e->keys;
    a.tab_keybase = e->tab_keybase;
    a.surv = e->surv;
    a.n_tab = n_tab;
    a.seq_begin = seq_begin;
    a.layer = layer;
    // tokens (x all heads) per score CTA: 128 while the CTA's keys fit the
    // staged-key buffer (cfg3 1.827 -> 1.792 ms, cfg2 0.524 -> 0.518 against
    // 64 tokens), else 64
    a.score_tokens = (int64_t)kScoreTokensPerCta * H <= kScoreKeysMax ? kScoreTokensPerCta : 64;
    if (const char* stk = std::getenv("PE_SCORE_TOKENS")) a.score_tokens = std::max(16, std::atoi(stk));  // tuning
    {
        // tables that keep every token are packed by the score kernel (its
        // staged-key path, blocks aligned to pages); PE_PREFILL_DIRECT=0: by the copy
        const char* sk = std::getenv("PE_SCORE_STAGED_KEYS");
        const char* dv = std::getenv("PE_PREFILL_DIRECT");
        a.direct_identity = a.score_tokens % s.B == 0 && (int64_t)a.score_tokens * H <= kScoreKeysMax &&
                            !(sk != nullptr && std::strcmp(sk, "0") == 0) &&
                            !(dv != nullptr && std::strcmp(dv, "0") == 0);
    }
    // PE_SELECT=cluster forces the cluster kernel (tests exercise both paths)
    // Select kernels. Default: tables of up to kSelectCtaMaxLen tokens take the
    // 512-thread streamed CTA select (two CTAs per SM), longer ones the
    // 1024-thread streamed select with a 16K candidate list. A/B options:
    // PE_SELECT=smem (short tables: high words in shared memory, the previous
    // default), PE_SELECT=stream (every table: the 1024-thread streamed
    // select), PE_SELECT=cluster (every table: the 8-CTA cluster select),
    // PE_SELECT_LONG=cluster (long tables: the cluster select),
    // PE_SELECT_MIXED=0 (a call with long tables sends every table to the
    // long-table kernel).
    const char* sel_env = std::getenv("PE_SELECT");
    auto env_is = [](const char* v, const char* x) { return v != nullptr && std::strcmp(v, x) == 0; };
    // Default: the GPU-wide select (window / count / resolve / emit kernels,
    // pe_select.cu) for tables of up to kGselMaxLen tokens. PE_SELECT=stream512
    // restores the CTA-per-table selects below (the previous default).
    // A call with few short tables (fewer than half the SMs, every table
    // within the shared-memory select's capacity) takes the one-kernel
    // shared-memory CTA select instead: the GPU-wide select's five launches
    // dominate there (cfg1, 8 tables of 4096 tokens: 0.077 vs 0.095 ms per
    // layer).
    const bool small_call = sel_env == nullptr && n_tab < e->sm_count / 2 && max_len <= kSelectCtaMaxLen;
    // Calls whose tables are all at most kGselMinLen tokens take the 512-thread
    // streamed CTA select: its per-table latency grows with the table length,
    // the GPU-wide select's chain does not (cfg2, 16384-token tables: 0.509 vs
    // 0.540 ms per layer; cfg3, 32768: 1.805 vs 1.772; cfg4's mixed lengths up
    // to 64K: 1.899 vs 1.868 for the first prompt wave)
    const bool short_call = sel_env == nullptr && max_len <= kGselMinLen;
    const bool gsel_fb = env_is(sel_env, "global_fallback");  // test knob: the fallback for every table
    const bool use_gsel = (sel_env == nullptr || env_is(sel_env, "global") || gsel_fb) && !small_call &&
                          !short_call && !env_is(std::getenv("PE_SELECT_LONG"), "cluster") && max_len <= kGselMaxLen;
    if (env_is(sel_env, "stream512")) sel_env = nullptr;
    const bool force_cluster = env_is(sel_env, "cluster");
    const bool force_stream = env_is(sel_env, "stream");
    const bool smem_short = env_is(sel_env, "smem") || small_call;
    const bool has_long = max_len > kSelectCtaMaxLen;
    if (force_stream || force_cluster || (has_long && env_is(std::getenv("PE_SELECT_MIXED"), "0"))) max_short = 0;
    const bool long_cluster = force_cluster || env_is(std::getenv("PE_SELECT_LONG"), "cluster");
    const bool any_long = max_short == 0 || has_long;  // some table goes to the long-table kernel
    if (any_long && long_cluster) {  // the cluster select holds a chunk of keys per CTA (u16 indices)
        if (chunk_cap > 65535)
            return fail(PE_INVALID_ARG, "prefill length exceeds the cluster select's index range");
        if (pack_smem > (size_t)e->max_dyn_prefill)
            return fail(PE_INVALID_ARG, "prefill length " + std::to_string(max_len) +
                                            " exceeds the per-cluster shared-memory capacity");
    }
    // the shared-memory select (and the fused variant built on it) holds a
    // whole table's high words per CTA; the cluster select a chunk per CTA
    const bool smem_capable = !has_long && !force_cluster && !force_stream;
    a.chunk_cap = smem_capable ? max_len : chunk_cap;
    a.cta_len_max = 0x7FFFFFFF;
    a.cluster_len_min = -1;
    a.cand_cap = kSelCandCapStream;
    if (total_pages > INT32_MAX) return fail(PE_POOL_EXHAUSTED, "page pool exhausted");
    plan_prefill_kernel<<<1, 1024, 0, st>>>(s, a, static_cast<int32_t>(total_pages), e->ctl);
    // Opt-in (PE_PREFILL_FUSED=1): the persistent single-launch variant. On
    // cfg3 it measures 2.23-2.40 ms/layer against 1.99-2.01 ms for the
    // multi-kernel wave pipeline below (its 1024-thread CTAs keep fewer
    // loads in flight while scoring), so the wave pipeline is the default.
    const char* fz = std::getenv("PE_PREFILL_FUSED");
    if (smem_capable && fz != nullptr && std::strcmp(fz, "1") == 0) {
        // one persistent launch: score units and per-table select+copy items,
        // X(q) scheduled after S(q+1) (prefill_fused_kernel); its copies pack
        // every table
        a.direct_identity = 0;
        int kUnitTokens = 1024;
        if (const char* ut = std::getenv("PE_UNIT_TOKENS")) kUnitTokens = std::max(16, std::atoi(ut));
        int64_t n_items = 0;
        for (int q = 0; q < n_seqs; ++q)
            n_items += (cu_seqlens[q + 1] - cu_seqlens[q] + kUnitTokens - 1) / kUnitTokens + H;
        if (n_items >= INT32_MAX || n_seqs > 32767) return fail(PE_INVALID_ARG, "prefill schedule too large");
        if ((size_t)n_items > e->h_items_elems) {
            if (e->h_items) PE_CUDA(cudaFreeHost(e->h_items));
            e->h_items = nullptr;
            e->h_items_elems = 0;
            PE_CUDA(cudaMallocHost(&e->h_items, sizeof(int32_t) * n_items));
            e->h_items_elems = (size_t)n_items;
        }
        if ((r = ensure_t(&e->items, &e->items_elems, (size_t)n_items)) != PE_OK) return r;
        // lag: X(q) follows S(q + lag), with enough score units in between
        // (~2 per CTA) that the sequence's scoring has finished when its
        // select items are claimed (no CTA spins while others still score it)
        const int64_t units_total = n_items - (int64_t)n_seqs * H;
        const int64_t per_seq = std::max<int64_t>(1, units_total / n_seqs);
        int lag = (int)std::min<int64_t>(n_seqs, (2 * e->sm_count + per_seq - 1) / per_seq);
        if (const char* lg = std::getenv("PE_FUSED_LAG")) lag = std::max(1, std::atoi(lg));
        int64_t k = 0;
        for (int q = 0; q < n_seqs + lag; ++q) {
            if (q < n_seqs) {
                const int u = (cu_seqlens[q + 1] - cu_seqlens[q] + kUnitTokens - 1) / kUnitTokens;
                e->h_seq_units[q] = u;
                if (u > 0xFFFF) return fail(PE_INVALID_ARG, "prefill length exceeds the schedule encoding");
                for (int j = 0; j < u; ++j) e->h_items[k++] = (q << 16) | j;
            }
            const int qx = q - lag;
            if (qx >= 0 && qx < n_seqs)
                for (int h = 0; h < H; ++h) e->h_items[k++] = static_cast<int32_t>(0x80000000u | (qx << 16) | h);
        }
        PE_CUDA(cudaMemcpyAsync(e->items, e->h_items, sizeof(int32_t) * n_items, cudaMemcpyHostToDevice, st));
        PE_CUDA(cudaMemcpyAsync(e->seq_units, e->h_seq_units, sizeof(int32_t) * n_seqs, cudaMemcpyHostToDevice, st));
        PE_CUDA(cudaEventRecord(e->ev_meta, st));
        PE_CUDA(cudaMemsetAsync(e->seq_done, 0, sizeof(int32_t) * n_seqs, st));
        PE_CUDA(cudaMemsetAsync(e->work_ctr, 0, sizeof(int32_t), st));
        const size_t sel_smem =
            (((size_t)max_len * 4 + 15) & ~size_t(15)) + kSelHistCopies * 2048 * 4 + kSelCandCap * 4;
        const int grid = (int)std::min<int64_t>(e->sm_count, n_items);
        launch_prefill_fused_any(e->variant, grid, sel_smem, st, s, a, e->ctl, e->items, (int)n_items, e->work_ctr,
                                 e->seq_done, e->seq_units, kUnitTokens);
        mark_consumed(e, st);
        r = check_launch(e, "prefill_fused_kernel");
        if (r != PE_OK) return r;
        e->stats.kernel_launches += 2;
        e->stats.prefill_calls += 1;
        e->stats.tokens_scored += (int64_t)tokens * H;
        if (evicted_counts && !ev_dev) {
            PE_CUDA(cudaMemcpyAsync(evicted_counts, e->evicted_dev, sizeof(int32_t) * n_tab, cudaMemcpyDeviceToHost, st));
        }
        return PE_OK;
    }
    // Two sequence waves ping-pong between the caller's stream and the engine's
    // aux stream: while one wave is in its latency-bound select, the other
    // stream's HBM-bound score / copy kernels keep the memory system busy.
    // The canonical page reservation (plan) is made once for the whole call.
    // (the cluster select of long tables is kept out of the wave overlap: its
    // 8-CTA clusters co-schedule badly next to another stream's kernels)
    int waves = (any_long && long_cluster) ? 1 : (n_seqs >= 2 ? 2 : 1);
    if (const char* wv = std::getenv("PE_PREFILL_WAVES")) waves = std::max(1, std::min(n_seqs, std::atoi(wv)));
    // grid limits: the score grid's y (sequences of a wave) and the cluster
    // select's y (tables of a wave) are at most 65535
    waves = std::max(waves, (n_seqs + 65534) / 65535);
    if (any_long && long_cluster) waves = std::max(waves, (n_tab + 65534) / 65535);
    const int max_keep_pages = (std::min(max_len, s.policy == PE_POLICY_PAGED_EVICTION ? s.C : max_len) + s.B - 1) / s.B;
    const bool chain = env_is(std::getenv("PE_PREFILL_CHAIN"), "1");
    // Mixed lengths: a compact score grid over the non-empty (sequence,
    // token block) pairs instead of max_len/T blocks for every sequence (cfg4:
    // most of the 2-D grid's CTAs would exit at once). Items are built on the
    // host in sequence order, so wave w's items are one contiguous range.
    const int max_blocks = (max_len + a.score_tokens - 1) / a.score_tokens;
    std::vector<int> item_start;
    {
        int64_t n_items = 0;
        for (int q = 0; q < n_seqs; ++q)
            n_items += (cu_seqlens[q + 1] - cu_seqlens[q] + a.score_tokens - 1) / a.score_tokens;
        const char* cg = std::getenv("PE_SCORE_COMPACT");  // A/B: 0 = always the 2-D grid
        const bool compact = !(cg != nullptr && std::strcmp(cg, "0") == 0) && n_seqs <= 32767 &&
                             max_blocks <= 0xFFFF && n_items < (int64_t)n_seqs * max_blocks * 4 / 5;
        if (compact) {
            if ((size_t)n_items > e->h_items_elems) {
                if (e->h_items) PE_CUDA(cudaFreeHost(e->h_items));
                e->h_items = nullptr;
                e->h_items_elems = 0;
                PE_CUDA(cudaMallocHost(&e->h_items, sizeof(int32_t) * n_items));
                e->h_items_elems = (size_t)n_items;
            }
            if ((r = ensure_t(&e->items, &e->items_elems, (size_t)n_items)) != PE_OK) return r;
            item_start.resize(n_seqs + 1);
            int64_t k = 0;
            for (int q = 0; q < n_seqs; ++q) {
                item_start[q] = (int)k;
                const int nb = (cu_seqlens[q + 1] - cu_seqlens[q] + a.score_tokens - 1) / a.score_tokens;
                for (int b = 0; b < nb; ++b) e->h_items[k++] = (q << 16) | b;
            }
            item_start[n_seqs] = (int)k;
            PE_CUDA(cudaMemcpyAsync(e->items, e->h_items, sizeof(int32_t) * n_items, cudaMemcpyHostToDevice, st));
            PE_CUDA(cudaEventRecord(e->ev_meta, st));  // the next call rewrites h_items after this copy
        }
    }
    // the aux stream's waves start after everything above on the caller's stream
    if (waves > 1) {
        PE_CUDA(cudaEventRecord(e->ev_fork, st));
        PE_CUDA(cudaStreamWaitEvent(e->aux_stream, e->ev_fork, 0));
    }
    GselArgs gs{};
    if (use_gsel) {
        gs.cand_stride = std::min(kGselCandCap, max_len);
        gs.chunk_stride = (max_len + kGselChunk - 1) / kGselChunk;
        if ((r = ensure_t(&e->gs_win, &e->gs_win_elems, (size_t)n_tab)) != PE_OK ||
            (r = ensure_t(&e->gs_tab, &e->gs_tab_elems, (size_t)2 * n_tab)) != PE_OK ||
            (r = ensure_t(&e->gs_ckey, &e->gs_ckey_elems, (size_t)n_tab * gs.cand_stride)) != PE_OK ||
            (r = ensure_t(&e->gs_cpos, &e->gs_cpos_elems, (size_t)n_tab * gs.cand_stride)) != PE_OK ||
            (r = ensure_t(&e->gs_chunk, &e->gs_chunk_elems, (size_t)n_tab * gs.chunk_stride)) != PE_OK ||
            (r = ensure_t(&e->gs_bits, &e->gs_bits_elems, (size_t)n_tab * gs.chunk_stride * kGselWords)) != PE_OK)
            return r;
        gs.win = e->gs_win;
        gs.cand_n = e->gs_tab;
        gs.flag = e->gs_tab + n_tab;
        gs.cand_key = e->gs_ckey;
        gs.cand_pos = e->gs_cpos;
        gs.chunk_cnt = e->gs_chunk;
        gs.evbits = e->gs_bits;
        gs.force_fallback = gsel_fb ? 1 : 0;
    }
    for (int w = 0; w < waves; ++w) {
        const int q0 = (int)((int64_t)n_seqs * w / waves);
        const int q1 = (int)((int64_t)n_seqs * (w + 1) / waves);
        if (q1 <= q0) continue;
        cudaStream_t sw = (w & 1) ? e->aux_stream : st;
        PrefillArgs aw = a;
        aw.tab_len += q0 * H;
        aw.tab_tok0 += q0 * H;
        aw.tab_pagebase += q0 * H;
        aw.tab_keybase += q0 * H;
        if (aw.evicted_counts) aw.evicted_counts += q0 * H;
        aw.seq_begin = seq_begin + q0;
        aw.n_tab = (q1 - q0) * H;
        // chained waves: this wave's score starts when the previous wave's
        // score is done, so that wave's select and copy run beside this score
        if (chain && w > 0) PE_CUDA(cudaStreamWaitEvent(sw, e->ev_score, 0));
        if (!item_start.empty()) {
            aw.score_items = e->items + item_start[q0];
            aw.item_seq0 = q0;
            launch_prefill_score_any(e->variant, dim3(item_start[q1] - item_start[q0]), sw, s, aw, e->ctl);
        } else {
            launch_prefill_score_any(e->variant, dim3(max_blocks, q1 - q0), sw, s, aw, e->ctl);
        }
        if (chain && w + 1 < waves) PE_CUDA(cudaEventRecord(e->ev_score, sw));
        if (use_gsel) {
            GselArgs gw = gs;
            gw.tab_off = q0 * H;
            const dim3 chunk_grid(aw.n_tab, gs.chunk_stride);
            gsel_window_kernel<<<aw.n_tab, kGselSample, 0, sw>>>(s, aw, gw, e->ctl);
            gsel_count_kernel<<<chunk_grid, 256, 0, sw>>>(s, aw, gw, e->ctl);
            gsel_resolve_kernel<<<aw.n_tab, 512, kGselCandCap * 12, sw>>>(s, aw, gw, e->ctl);
            // tables whose window missed: the streamed CTA-per-table select
            PrefillArgs af = aw;
            af.bits_cap = std::min((max_len + 31) / 32 * 32, kSelBitsMaxLen);
            const size_t fb_smem = (size_t)kSelHistCopies * 2048 * 4 + (size_t)kSelCandCapStream * 4 +
                                   (size_t)af.bits_cap / 8;
            // strided over the wave's tables (only flagged ones do work)
            int fb_grid = std::min(aw.n_tab, e->sm_count);
            if (const char* fg = std::getenv("PE_FB_GRID")) fb_grid = std::max(1, std::min(aw.n_tab, std::atoi(fg)));
            gsel_fallback_kernel<<<fb_grid, 1024, fb_smem, sw>>>(s, af, gw, e->ctl);
            gsel_emit_kernel<<<chunk_grid, 64, 0, sw>>>(s, aw, gw, e->ctl);
            e->stats.kernel_launches += 5;
        } else if (max_short > 0) {  // tables of at most kSelectCtaMaxLen tokens
            PrefillArgs ac = aw;
            ac.cta_len_max = kSelectCtaMaxLen;
            if (smem_short) {
                ac.chunk_cap = max_short;
                const size_t sel_smem =
                    (((size_t)max_short * 4 + 15) & ~size_t(15)) + kSelHistCopies * 2048 * 4 + kSelCandCap * 4;
                prefill_select_cta_kernel<<<aw.n_tab, 1024, sel_smem, sw>>>(s, ac, e->ctl);
            } else {
                ac.cand_cap = kSelCandCap;
                ac.bits_cap = (kSelectCtaMaxLen + 31) / 32 * 32;  // eviction bitmap: 4.3 KB
                const size_t smem5 =
                    (size_t)kSelHistCopies * 2048 * 4 + (size_t)kSelCandCap * 4 + (size_t)ac.bits_cap / 8;
                prefill_select_stream512_kernel<<<aw.n_tab, 512, smem5, sw>>>(s, ac, e->ctl);
            }
            e->stats.kernel_launches += 1;
        }
        if (any_long && !use_gsel) {  // the longer tables (every table when max_short == 0)
            PrefillArgs al = aw;
            al.cluster_len_min = max_short > 0 ? kSelectCtaMaxLen : -1;
            if (long_cluster) {
                prefill_select_kernel<<<dim3(kPrefillCluster, aw.n_tab), kPackThreads, pack_smem, sw>>>(s, al,
                                                                                                     e->ctl);
            } else {
                // eviction bitmap for tables up to kSelBitsMaxLen tokens (longer: the sweeps)
                al.bits_cap = std::min((max_len + 31) / 32 * 32, kSelBitsMaxLen);
                const size_t st_smem = (size_t)kSelHistCopies * 2048 * 4 + (size_t)kSelCandCapStream * 4 +
                                       (size_t)al.bits_cap / 8;
                prefill_select_stream_kernel<<<aw.n_tab, 1024, st_smem, sw>>>(s, al, e->ctl);
            }
            e->stats.kernel_launches += 1;
        }
        launch_prefill_copy_any(e->variant, dim3(aw.n_tab, (max_keep_pages + 3) / 4), sw, s, aw, e->ctl);
        e->stats.kernel_launches += 2;  // score + copy (the selects counted above)
    }
    if (waves > 1) {
        PE_CUDA(cudaEventRecord(e->ev_join, e->aux_stream));
        PE_CUDA(cudaStreamWaitEvent(st, e->ev_join, 0));
    }
    mark_consumed(e, st);
    r = check_launch(e, "prefill_kernel");
    if (r != PE_OK) return r;
    e->stats.kernel_launches += 1;
    e->stats.prefill_calls += 1;
    e->stats.tokens_scored += (int64_t)tokens * H;
    if (evicted_counts && !ev_dev) {
        PE_CUDA(cudaMemcpyAsync(evicted_counts, e->evicted_dev, sizeof(int32_t) * n_tab, cudaMemcpyDeviceToHost, st));
    }
    return PE_OK;
}

}  // extern "C"

namespace {

// One eviction launch over table set `ts` (state `sc`: the engine's, or a
// copy with the table API's per-call budget).
pe_status launch_evict(pe_engine* e, const DevState& sc, const TableSet& ts, int32_t mode, int32_t* victims,
                       cudaStream_t st) {
    if (e != nullptr) e->append_chain = false;  // tables change outside the append chain
    const int n = ts.size(sc);
    const bool vic_dev = victims && is_device_ptr(victims);
    int32_t* vdst = vic_dev ? victims : e->victims;
    // one launch: the grid's last CTA pushes the released pages in ascending
    // table id (no separate planner)
    // PDL (programmatic dependent launch): a recompute launch right after one
    // over a disjoint layer range of the same engine on the same stream
    // scores and evicts while that launch drains (evict_score_kernel `early`)
    const char* pdl_env = std::getenv("PE_K2_PDL");  // A/B: 0 = plain stream order
    const bool early = !(pdl_env != nullptr && std::strcmp(pdl_env, "0") == 0) &&
                       e->k2_chain && e->k2_stream == st && ts.ids == nullptr &&
                       (ts.layer_begin >= e->k2_layer0 + e->k2_layers ||
                        ts.layer_begin + ts.n_layers <= e->k2_layer0);
    if (mode == PE_SCORE_RECOMPUTE) {
        // Pages per CTA: as many as possible (a CTA's warps stream their pages
        // without draining; one CTA per table reaches 97 % of the HBM peak on
        // an all-layer launch), but at least ~3 CTAs per SM on small launches
        // (cfg2's per-layer launch of 256 tables: 2 chunks of 65 pages; cfg3's
        // 512 tables: one CTA per table). With per-layer launches chained by
        // PDL the next launch fills the SMs a launch's tail leaves idle, so
        // fewer, longer CTAs win: cfg3 per-layer 195 -> 171 us (28 -> 3 CTAs
        // per SM target), cfg2 65 -> 45 us (tools/k2_ab.py).
        const int min_chunks = (sc.max_pages + kMaxPagesPerCta - 1) / kMaxPagesPerCta;
        const char* cps_env = std::getenv("PE_K2_CTAS_PER_SM");  // tuning override (read per call: A/B)
        const int ctas_per_sm = cps_env ? std::max(1, std::atoi(cps_env)) : 3;
        const int target_ctas = ctas_per_sm * e->sm_count;
        int chunks = std::max(min_chunks, (target_ctas + n - 1) / n);
        chunks = std::max(min_chunks, std::min(chunks, (sc.max_pages + 7) / 8));
        const int ppc = (sc.max_pages + chunks - 1) / chunks;
        chunks = (sc.max_pages + ppc - 1) / ppc;
        e->grid_tickets += (unsigned long long)n;  // one completion ticket per table
        launch_evict_score_any(e->variant, dim3(n, chunks), kEvictThreads, st, sc, ts, ppc,
                               e->evict_scratch, e->tickets, e->vpage, vdst, e->grid_tickets - 1, early);
    } else {
        e->grid_tickets += (unsigned long long)n;
        // PDL always (a non-early launch waits at its top); early: see K2
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((n + 7) / 8);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = (early || pdl_enabled()) ? 1 : 0;
        cudaLaunchKernelEx(&cfg, evict_cached_kernel, sc, ts, e->evict_scratch, e->vpage, vdst, e->grid_tickets - 1,
                           early ? 1 : 0);
    }
    pe_status r = check_launch(e, "evict kernel");
    if (r != PE_OK) return r;
    if (ts.ids == nullptr) {  // either score mode: both touch only their own tables before the push
        e->k2_chain = true;
        e->k2_layer0 = ts.layer_begin;
        e->k2_layers = ts.n_layers;
        e->k2_stream = st;
    }
    e->stats.kernel_launches += 1;
    e->stats.evict_calls += 1;
    if (victims && !vic_dev) {
        PE_CUDA(cudaMemcpyAsync(victims, e->victims, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    }
    return PE_OK;
}

// One append launch (K0) over table set `ts`; k/v/positions already on the device.
pe_status launch_append(pe_engine* e, const TableSet& ts, const uint8_t* dk, const uint8_t* dv,
                        const int64_t* dp, cudaStream_t st) {
    const DevState& s = e->s;
    const int n = ts.size(s);
    // one launch: canonical pop ranks by a single-pass decoupled look-back
    const int warps = kAppendThreads / 32;
    const int blocks = (n + 16 * warps - 1) / (16 * warps);
    const unsigned long long ticket_base = e->grid_tickets;
    e->grid_tickets += blocks;
    e->append_epoch = (e->append_epoch % kAppendEpochPeriod) + 1;  // 1 .. period, parity alternates
    const bool contiguous = ts.ids == nullptr;
    const char* ff = std::getenv("PE_APPEND_FAST");
    const bool fast_ok = contiguous && e->append_chain && e->chain_layer0 == ts.layer_begin &&
                         e->chain_layers == ts.n_layers && !(ff != nullptr && std::strcmp(ff, "0") == 0);
    launch_append_any(e->variant, blocks, st, s, ts, dk, dv, dp, e->lb_status,
                      e->lb_status + lb_cta_words(s.n_tables), e->ctl, ticket_base, e->append_epoch, fast_ok);
    mark_consumed(e, st);
    e->append_chain = contiguous;
    e->chain_layer0 = ts.layer_begin;
    e->chain_layers = ts.n_layers;
    pe_status r = check_launch(e, "append_kernel");
    if (r != PE_OK) return r;
    e->stats.kernel_launches += 1;
    e->stats.append_calls += 1;
    return PE_OK;
}

}  // namespace

extern "C" {

// ------------------------------------------------------------------ K0
pe_status pe_decode_append(pe_engine* e, int32_t layer_begin, int32_t n_layers, const void* k_rows,
                           const void* v_rows, const int64_t* positions, void* stream) {
    if (e == nullptr) return fail(PE_INVALID_ARG, "null engine");
    const DevState& s = e->s;
    if (layer_begin < 0 || n_layers <= 0 || layer_begin + n_layers > s.n_layers)
        return fail(PE_INVALID_ARG, "layer range out of range");
    cudaSetDevice(e->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TableSet ts{layer_begin, n_layers};
    const int n = ts.size(s);
    const size_t bytes = (size_t)n * s.row_bytes;
    const uint8_t *dk = nullptr, *dv = nullptr, *dp = nullptr;
    e->n_pending = 0;
    pe_status r = as_device(e, k_rows, bytes, st, &dk);
    if (r != PE_OK) return r;
    r = as_device(e, v_rows, bytes, st, &dv);
    if (r != PE_OK) return r;
    r = as_device(e, positions, sizeof(int64_t) * s.n_seqs, st, &dp);
    if (r != PE_OK) return r;
    return launch_append(e, ts, dk, dv, reinterpret_cast<const int64_t*>(dp), st);
}

// ------------------------------------------------------------------ K2 / K2c
pe_status pe_decode_evict(pe_engine* e, int32_t layer_begin, int32_t n_layers, int64_t step,
                          int32_t mode, int32_t* victims, void* stream) {
    (void)step;
    if (e == nullptr) return fail(PE_INVALID_ARG, "null engine");
    const DevState& s = e->s;
    if (layer_begin < 0 || n_layers <= 0 || layer_begin + n_layers > s.n_layers)
        return fail(PE_INVALID_ARG, "layer range out of range");
    if (mode != PE_SCORE_RECOMPUTE && mode != PE_SCORE_CACHED) return fail(PE_INVALID_ARG, "score mode");
    cudaSetDevice(e->device);
    TableSet ts{layer_begin, n_layers};
    return launch_evict(e, s, ts, mode, victims, static_cast<cudaStream_t>(stream));
}

pe_status pe_decode_step(pe_engine* e, int32_t layer_begin, int32_t n_layers, const void* k_rows,
                         const void* v_rows, const int64_t* positions, int64_t step, int32_t mode,
                         int32_t* victims, void* stream) {
    pe_status r = pe_decode_append(e, layer_begin, n_layers, k_rows, v_rows, positions, stream);
    if (r != PE_OK) return r;
    return pe_decode_evict(e, layer_begin, n_layers, step, mode, victims, stream);
}

pe_status pe_step_log_capture(pe_engine* e, int32_t layer_begin, int32_t n_layers, const int32_t* victims,
                              pe_step_entry* out, void* stream) {
    if (e == nullptr || out == nullptr) return fail(PE_INVALID_ARG, "null argument");
    const DevState& s = e->s;
    if (layer_begin < 0 || n_layers <= 0 || layer_begin + n_layers > s.n_layers)
        return fail(PE_INVALID_ARG, "layer range out of range");
    if (victims != nullptr && !is_device_ptr(victims))
        return fail(PE_INVALID_ARG, "victims must be a device array (or NULL for the engine's copy)");
    cudaSetDevice(e->device);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    TableSet ts{layer_begin, n_layers};
    const int n = ts.size(s);
    const bool out_dev = is_device_ptr(out);
    if (!out_dev && e->step_stage == nullptr && dalloc(&e->step_stage, (size_t)s.n_tables) != cudaSuccess)
        return fail(PE_CUDA_ERROR, "step-log staging allocation failed");
    pe_step_entry* dst = out_dev ? out : e->step_stage;
    step_log_kernel<<<(n + 255) / 256, 256, 0, st>>>(s, ts, victims ? victims : e->victims, dst);
    pe_status r = check_launch(e, "step_log_kernel");
    if (r != PE_OK) return r;
    e->stats.kernel_launches += 1;
    if (!out_dev) PE_CUDA(cudaMemcpyAsync(out, dst, sizeof(pe_step_entry) * n, cudaMemcpyDeviceToHost, st));
    return PE_OK;
}

// ------------------------------------------------------------------ K3
pe_status pe_paged_decode_attention(pe_engine* e, int32_t layer, const void* q, float* out,
                                    int32_t n_q_heads, void* stream) {
    if (e == nullptr) return fail(PE_INVALID_ARG, "null engine");
    const DevState& s = e->s;
    if (s.holes_on)
        return fail(PE_INVALID_STATE, "tables with evicted slots (unstructured eviction): use pe_table_attend");
    if (layer < 0 || layer >= s.n_layers) return fail(PE_INVALID_ARG, "layer out of range");
    // attention heads: the model's KV heads (a PER_LAYER table holds all of a
    // layer's KV heads side by side in each row, kv_vector.hpp:23-27)
    const int Hk = e->cfg.n_kv_heads;
    const int hd = e->cfg.head_dim;
    if (n_q_heads <= 0 || n_q_heads % Hk != 0)
        return fail(PE_LENGTH_MISMATCH, "query heads must be a multiple of KV heads");
    const int G = n_q_heads / Hk;
    if (G > 8) return fail(PE_INVALID_ARG, "at most 8 query heads per KV head");
    if (hd > 256) return fail(PE_INVALID_ARG, "head_dim > 256 unsupported");
    if ((hd * (s.dtype == PE_DTYPE_BF16 ? 2 : 4)) % 16 != 0)
        return fail(PE_INVALID_ARG, "head_dim * element size must be a multiple of 16 bytes");
    cudaSetDevice(e->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int n_tab = s.n_seqs * Hk;  // launch items (sequence, KV head)
    const size_t head_bytes = (size_t)hd * (s.dtype == PE_DTYPE_BF16 ? 2 : 4);
    const uint8_t* dq = nullptr;
    e->n_pending = 0;
    pe_status r = as_device(e, q, (size_t)s.n_seqs * n_q_heads * head_bytes, st, &dq);
    if (r != PE_OK) return r;
    // as many splits as fit in one wave of CTAs (2 per SM), rounding down: a
    // CTA's warps stream their pages without draining, so long CTAs beat
    // extra waves (cfg3: one split per table 181 us vs three 191 us; cfg2's
    // 256 tables: one split 47 us vs two 53 us)
    int splits = std::max(1, (e->sm_count * 2) / n_tab);
    if (const char* sv = std::getenv("PE_ATTN_SPLITS")) splits = std::max(1, std::atoi(sv));
    splits = std::min(splits, std::max(1, (s.max_pages + 3) / 4));
    const int pps = (s.max_pages + splits - 1) / splits;
    splits = (s.max_pages + pps - 1) / pps;
    if (splits > 65535) return fail(PE_INVALID_ARG, "attention split count exceeds the grid limit");
    r = ensure_t(&e->part_o, &e->part_o_elems, (size_t)n_tab * splits * G * hd);
    if (r != PE_OK) return r;
    r = ensure_t(&e->part_ml, &e->part_ml_elems, (size_t)n_tab * splits * G * 2);
    if (r != PE_OK) return r;
    const bool out_dev = is_device_ptr(out);
    const size_t out_elems = (size_t)s.n_seqs * n_q_heads * hd;
    if (!out_dev) {
        r = ensure_t(&e->out_stage, &e->out_stage_elems, out_elems);
        if (r != PE_OK) return r;
    }
    AttnArgs a{};
    a.q = dq;
    a.out = out_dev ? out : e->out_stage;
    a.part_o = e->part_o;
    a.part_ml = e->part_ml;
    a.tickets = e->attn_tickets;
    a.layer = layer;
    a.G = G;
    a.n_q_heads = n_q_heads;
    a.splits = splits;
    a.pages_per_split = pps;
    a.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(hd)));
    a.kv_heads = Hk;
    a.heads_per_table = Hk / s.tab_heads;
    a.d = hd;
    const bool use_mma = s.dtype == PE_DTYPE_BF16 && s.B == 16 && (hd == 64 || hd == 128);
    // TMA staging (tensor map, 128-byte swizzle) unless PE_ATTN_TMA=0: 7 % faster
    // than the cp.async staging at cfg3 (160 vs 172 us), 11 % on the unpruned layer
    const char* tv = std::getenv("PE_ATTN_TMA");
    const bool use_tma = use_mma && e->has_tmap && !(tv != nullptr && std::strcmp(tv, "0") == 0);
    if (use_tma) {
        launch_attention_tma(hd, dim3(n_tab, splits), attention_tma_smem(hd, G), st, s, a, &e->pool_tmap);
    } else if (use_mma) {
        // tensor-core path (mma.sync bf16, P split hi/lo), pe_attention.cu
        const size_t smem = attention_mma_smem(hd, G);
        launch_attention_mma(hd, dim3(n_tab, splits), smem, st, s, a);
    } else {
        const int nw = 4;
        size_t smem = (size_t)G * hd * 4 + (size_t)nw * G * 16 * 4 + (size_t)nw * G * hd * 4 +
                      (size_t)nw * G * 2 * 4 + 16 + (size_t)nw * 2 * (2 * s.B * (head_bytes + 16));
        if (smem > (size_t)e->max_dyn_attn) return fail(PE_INVALID_ARG, "attention tile exceeds shared memory");
        attention_split_kernel<<<dim3(n_tab, splits), 128, smem, st>>>(s, a);
    }
    mark_consumed(e, st);
    r = check_launch(e, "attention");
    if (r != PE_OK) return r;
    if (use_mma) {
        // the tensor-core attention writes only its partials, tickets and
        // output: a recompute K2 over another layer may follow it through PDL
        // (decode order attend(l) -> evict(l + 1): the eviction streams its
        // pages while this launch drains)
        e->k2_chain = true;
        e->k2_layer0 = layer;
        e->k2_layers = 1;
        e->k2_stream = st;
    }
    e->stats.kernel_launches += 1;
    e->stats.attention_calls += 1;
    if (!out_dev) {
        PE_CUDA(cudaMemcpyAsync(out, e->out_stage, sizeof(float) * out_elems, cudaMemcpyDeviceToHost, st));
    }
    return PE_OK;
}

// ------------------------------------------------------------------ sync / readback
pe_status pe_sync(pe_engine* e) {
    if (e == nullptr) return fail(PE_INVALID_ARG, "null engine");
    cudaSetDevice(e->device);
    PE_CUDA(cudaDeviceSynchronize());
    int32_t st = 0;
    PE_CUDA(cudaMemcpy(&st, e->s.status, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (st != 0) {
        PE_CUDA(cudaMemset(e->s.status, 0, sizeof(int32_t)));
        return fail(static_cast<pe_status>(st), pe_status_string(static_cast<pe_status>(st)));
    }
    return PE_OK;
}

pe_status pe_get_info(pe_engine* e, pe_info* out) {
    if (e == nullptr || out == nullptr) return fail(PE_INVALID_ARG, "null argument");
    const DevState& s = e->s;
    cudaSetDevice(e->device);
    std::memset(out, 0, sizeof(*out));
    out->n_tables = s.n_tables;
    out->tab_heads = s.tab_heads;
    out->width = s.w;
    out->page_size = s.B;
    out->cache_budget = s.C;
    out->capacity = s.capacity;
    out->max_pages = s.max_pages;
    out->dtype = s.dtype;
    out->policy = s.policy;
    out->granularity = e->cfg.granularity;
    out->row_pitch_bytes = s.pitch;
    out->sm_count = e->sm_count;
    out->pool_bytes = (int64_t)s.capacity * 2 * s.B * s.pitch;
    out->state_bytes = (int64_t)s.capacity * s.B * 12 + (int64_t)s.capacity * 12 +
                       (int64_t)s.n_tables * (s.max_pages + 3) * 4;
    PE_CUDA(cudaDeviceSynchronize());
    PE_CUDA(cudaMemcpy(&out->free_pages, s.top, sizeof(int32_t), cudaMemcpyDeviceToHost));
    return PE_OK;
}

pe_status pe_get_stats(pe_engine* e, pe_stats* out) {
    if (e == nullptr || out == nullptr) return fail(PE_INVALID_ARG, "null argument");
    cudaSetDevice(e->device);
    *out = e->stats;
    unsigned long long ev = 0;
    PE_CUDA(cudaDeviceSynchronize());
    PE_CUDA(cudaMemcpy(&ev, e->s.evict_count, sizeof(ev), cudaMemcpyDeviceToHost));
    out->pages_evicted = static_cast<int64_t>(ev);
    return PE_OK;
}

pe_status pe_read_tables(pe_engine* e, int32_t* block_table, int32_t* num_pages, int32_t* newest_fill,
                         int32_t* retained) {
    if (e == nullptr) return fail(PE_INVALID_ARG, "null engine");
    const DevState& s = e->s;
    cudaSetDevice(e->device);
    PE_CUDA(cudaDeviceSynchronize());
    if (block_table)
        PE_CUDA(cudaMemcpy(block_table, s.block_table, sizeof(int32_t) * (size_t)s.n_tables * s.max_pages,
                           cudaMemcpyDeviceToHost));
    if (num_pages) PE_CUDA(cudaMemcpy(num_pages, s.num_pages, sizeof(int32_t) * s.n_tables, cudaMemcpyDeviceToHost));
    if (newest_fill)
        PE_CUDA(cudaMemcpy(newest_fill, s.newest_fill, sizeof(int32_t) * s.n_tables, cudaMemcpyDeviceToHost));
    if (retained) PE_CUDA(cudaMemcpy(retained, s.retained, sizeof(int32_t) * s.n_tables, cudaMemcpyDeviceToHost));
    return PE_OK;
}

pe_status pe_read_free_list(pe_engine* e, int32_t* stack_out, int32_t* n_free) {
    if (e == nullptr) return fail(PE_INVALID_ARG, "null engine");
    cudaSetDevice(e->device);
    PE_CUDA(cudaDeviceSynchronize());
    int32_t top = 0;
    PE_CUDA(cudaMemcpy(&top, e->s.top, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (n_free) *n_free = top;
    if (stack_out && top > 0)
        PE_CUDA(cudaMemcpy(stack_out, e->s.stack, sizeof(int32_t) * top, cudaMemcpyDeviceToHost));
    return PE_OK;
}

pe_status pe_read_positions(pe_engine* e, int32_t page_begin, int32_t n_pages, int32_t* positions,
                            double* token_scores, double* page_scores) {
    if (e == nullptr) return fail(PE_INVALID_ARG, "null engine");
    const DevState& s = e->s;
    if (page_begin < 0 || n_pages < 0 || page_begin + n_pages > s.capacity)
        return fail(PE_INDEX_OUT_OF_RANGE, "page range out of range");
    cudaSetDevice(e->device);
    PE_CUDA(cudaDeviceSynchronize());
    if (positions)
        PE_CUDA(cudaMemcpy(positions, s.positions + (size_t)page_begin * s.B, sizeof(int32_t) * (size_t)n_pages * s.B,
                           cudaMemcpyDeviceToHost));
    if (token_scores)
        PE_CUDA(cudaMemcpy(token_scores, s.token_scores + (size_t)page_begin * s.B,
                           sizeof(double) * (size_t)n_pages * s.B, cudaMemcpyDeviceToHost));
    if (page_scores)
        PE_CUDA(cudaMemcpy(page_scores, s.page_scores + page_begin, sizeof(double) * n_pages, cudaMemcpyDeviceToHost));
    return PE_OK;
}

pe_status pe_read_pages(pe_engine* e, int32_t page_begin, int32_t n_pages, void* out) {
    if (e == nullptr || out == nullptr) return fail(PE_INVALID_ARG, "null argument");
    const DevState& s = e->s;
    if (page_begin < 0 || n_pages < 0 || page_begin + n_pages > s.capacity)
        return fail(PE_INDEX_OUT_OF_RANGE, "page range out of range");
    cudaSetDevice(e->device);
    PE_CUDA(cudaDeviceSynchronize());
    const size_t pb = (size_t)2 * s.B * s.pitch;
    PE_CUDA(cudaMemcpy(out, s.pages + (size_t)page_begin * pb, pb * n_pages, cudaMemcpyDeviceToHost));
    return PE_OK;
}

pe_status pe_get_device_view(pe_engine* e, pe_device_view* out) {
    if (e == nullptr || out == nullptr) return fail(PE_INVALID_ARG, "null argument");
    out->pages = e->s.pages;
    out->block_table = e->s.block_table;
    out->num_pages = e->s.num_pages;
    out->newest_fill = e->s.newest_fill;
    out->retained = e->s.retained;
    out->positions = e->s.positions;
    return PE_OK;
}

// ------------------------------------------------------------------ table-granular API
}  // extern "C"

namespace {

pe_status check_table_list(pe_engine* e, int32_t n, const int32_t* ids) {
    if (e == nullptr) return fail(PE_INVALID_ARG, "null engine");
    if (n <= 0 || n > e->s.n_tables) return fail(PE_INVALID_ARG, "table count out of range");
    if (ids == nullptr) return fail(PE_INVALID_ARG, "null table list");
    if (is_device_ptr(ids)) return fail(PE_INVALID_ARG, "table list must be a host array");
    for (int32_t i = 0; i < n; ++i) {
        if (ids[i] < 0 || ids[i] >= e->s.n_tables) return fail(PE_INDEX_OUT_OF_RANGE, "table id out of range");
        if (i > 0 && ids[i] <= ids[i - 1]) return fail(PE_INVALID_ARG, "table ids must be strictly ascending");
    }
    return PE_OK;
}

pe_status check_table(pe_engine* e, int32_t t) {
    if (e == nullptr) return fail(PE_INVALID_ARG, "null engine");
    if (t < 0 || t >= e->s.n_tables) return fail(PE_INDEX_OUT_OF_RANGE, "table id out of range");
    return PE_OK;
}

}  // namespace

extern "C" {

pe_status pe_table_append(pe_engine* e, int32_t n, const int32_t* table_ids, const void* k_rows,
                          const void* v_rows, const int64_t* positions, void* stream) {
    pe_status r = check_table_list(e, n, table_ids);
    if (r != PE_OK) return r;
    const DevState& s = e->s;
    cudaSetDevice(e->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t bytes = (size_t)n * s.row_bytes;
    const uint8_t *dk = nullptr, *dv = nullptr, *dp = nullptr, *di = nullptr;
    e->n_pending = 0;
    if ((r = as_device(e, table_ids, sizeof(int32_t) * n, st, &di)) != PE_OK) return r;
    if ((r = as_device(e, k_rows, bytes, st, &dk)) != PE_OK) return r;
    if ((r = as_device(e, v_rows, bytes, st, &dv)) != PE_OK) return r;
    if ((r = as_device(e, positions, sizeof(int64_t) * n, st, &dp)) != PE_OK) return r;
    TableSet ts{0, 1, reinterpret_cast<const int32_t*>(di), n};
    return launch_append(e, ts, dk, dv, reinterpret_cast<const int64_t*>(dp), st);
}

pe_status pe_table_evict(pe_engine* e, int32_t n, const int32_t* table_ids, int32_t cache_budget, int32_t mode,
                         int32_t* victims, void* stream) {
    if (e != nullptr) e->append_chain = false;  // tables change outside the append chain
    pe_status r = check_table_list(e, n, table_ids);
    if (r != PE_OK) return r;
    if (cache_budget < 0) return fail(PE_BUDGET_INVALID, "negative budget");
    if (mode != PE_SCORE_RECOMPUTE && mode != PE_SCORE_CACHED) return fail(PE_INVALID_ARG, "score mode");
    cudaSetDevice(e->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint8_t* di = nullptr;
    e->n_pending = 0;
    if ((r = as_device(e, table_ids, sizeof(int32_t) * n, st, &di)) != PE_OK) return r;
    DevState sc = e->s;  // PagedEviction decision with this call's budget C
    sc.policy = PE_POLICY_PAGED_EVICTION;
    sc.C = cache_budget;
    TableSet ts{0, 1, reinterpret_cast<const int32_t*>(di), n};
    r = launch_evict(e, sc, ts, mode, victims, st);
    mark_consumed(e, st);
    return r;
}

pe_status pe_table_free_page(pe_engine* e, int32_t table, int32_t logical_index, void* stream) {
    if (e != nullptr) e->append_chain = false;  // tables change outside the append chain
    pe_status r = check_table(e, table);
    if (r != PE_OK) return r;
    cudaSetDevice(e->device);
    table_free_page_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(e->s, table, logical_index);
    e->stats.kernel_launches += 1;
    return check_launch(e, "table_free_page_kernel");
}

pe_status pe_table_clear(pe_engine* e, int32_t table, void* stream) {
    if (e != nullptr) e->append_chain = false;  // tables change outside the append chain
    pe_status r = check_table(e, table);
    if (r != PE_OK) return r;
    cudaSetDevice(e->device);
    table_clear_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(e->s, table);
    e->stats.kernel_launches += 1;
    return check_launch(e, "table_clear_kernel");
}

pe_status pe_table_attend(pe_engine* e, int32_t table, const float* query, int32_t head_count, int32_t head_dim,
                          float* out, double* weight_sums, void* stream) {
    pe_status r = check_table(e, table);
    if (r != PE_OK) return r;
    const DevState& s = e->s;
    if (query == nullptr || out == nullptr) return fail(PE_INVALID_ARG, "null buffer");
    if (head_count <= 0 || head_dim <= 0 || (int64_t)head_count * head_dim > s.w)
        return fail(PE_LENGTH_MISMATCH, "head_count * head_dim exceeds the pool row width");
    cudaSetDevice(e->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int32_t R = 0, NP = 0;
    PE_CUDA(cudaStreamSynchronize(st));
    PE_CUDA(cudaMemcpy(&R, s.retained + table, sizeof(int32_t), cudaMemcpyDeviceToHost));
    PE_CUDA(cudaMemcpy(&NP, s.num_pages + table, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (R <= 0) return fail(PE_EMPTY_CACHE, "attention requires at least one retained token");
    const size_t width = (size_t)head_count * head_dim;
    e->n_pending = 0;
    const uint8_t* dq = nullptr;
    if ((r = as_device(e, query, sizeof(float) * width, st, &dq)) != PE_OK) return r;
    if ((r = ensure_t(&e->attend_logits, &e->attend_logits_elems, (size_t)NP * s.B * head_count)) != PE_OK) return r;
    if ((r = ensure_t(&e->attend_out, &e->attend_out_elems, width)) != PE_OK) return r;
    if ((r = ensure_t(&e->attend_ws, &e->attend_ws_elems, (size_t)head_count)) != PE_OK) return r;
    const bool out_dev = is_device_ptr(out);
    const bool ws_dev = weight_sums && is_device_ptr(weight_sums);
    table_attend_kernel<<<head_count, 256, 0, st>>>(s, table, reinterpret_cast<const float*>(dq), head_dim,
                                                    e->attend_logits, out_dev ? out : e->attend_out,
                                                    weight_sums ? (ws_dev ? weight_sums : e->attend_ws) : nullptr);
    mark_consumed(e, st);
    if ((r = check_launch(e, "table_attend_kernel")) != PE_OK) return r;
    e->stats.kernel_launches += 1;
    e->stats.attention_calls += 1;
    if (!out_dev) PE_CUDA(cudaMemcpyAsync(out, e->attend_out, sizeof(float) * width, cudaMemcpyDeviceToHost, st));
    if (weight_sums && !ws_dev)
        PE_CUDA(cudaMemcpyAsync(weight_sums, e->attend_ws, sizeof(double) * head_count, cudaMemcpyDeviceToHost, st));
    return PE_OK;
}

pe_status pe_read_table(pe_engine* e, int32_t table, int32_t* page_ids, int32_t* num_pages, int32_t* newest_fill,
                        int32_t* retained) {
    pe_status r = check_table(e, table);
    if (r != PE_OK) return r;
    const DevState& s = e->s;
    cudaSetDevice(e->device);
    PE_CUDA(cudaDeviceSynchronize());
    int32_t np = 0;
    PE_CUDA(cudaMemcpy(&np, s.num_pages + table, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (num_pages) *num_pages = np;
    if (page_ids && np > 0)
        PE_CUDA(cudaMemcpy(page_ids, s.block_table + (size_t)table * s.max_pages, sizeof(int32_t) * np,
                           cudaMemcpyDeviceToHost));
    if (newest_fill) PE_CUDA(cudaMemcpy(newest_fill, s.newest_fill + table, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (retained) PE_CUDA(cudaMemcpy(retained, s.retained + table, sizeof(int32_t), cudaMemcpyDeviceToHost));
    return PE_OK;
}

pe_status pe_table_evict_token(pe_engine* e, int32_t table, int32_t rule, int64_t arg, int32_t cache_budget,
                               int64_t newest_position, int64_t* victim_position, void* stream) {
    if (e != nullptr) e->append_chain = false;  // tables change outside the append chain
    pe_status r = check_table(e, table);
    if (r != PE_OK) return r;
    if (rule < PE_TOKEN_AT_POSITION || rule > PE_TOKEN_KEY_DIFF) return fail(PE_INVALID_ARG, "token rule");
    if (e->s.B > 64) return fail(PE_INVALID_ARG, "unstructured eviction needs page_size <= 64");
    cudaSetDevice(e->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    e->s.holes_on = 1;  // from now on every kernel honours the hole masks
    if ((r = ensure_t(&e->attend_out, &e->attend_out_elems, (size_t)e->s.w)) != PE_OK) return r;
    token_evict_kernel<<<1, 256, 0, st>>>(e->s, table, rule, static_cast<long long>(arg), cache_budget,
                                          static_cast<long long>(newest_position), e->attend_out,
                                          reinterpret_cast<long long*>(e->tok_out));
    if ((r = check_launch(e, "token_evict_kernel")) != PE_OK) return r;
    e->stats.kernel_launches += 1;
    if (victim_position != nullptr)
        PE_CUDA(cudaMemcpyAsync(victim_position, e->tok_out, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    return PE_OK;
}

pe_status pe_decode_evict_tokens(pe_engine* e, int32_t layer_begin, int32_t n_layers, int32_t rule, int64_t arg,
                                 const int64_t* newest_positions, int64_t* victim_positions, void* stream) {
    if (e != nullptr) e->append_chain = false;  // tables change outside the append chain
    if (e == nullptr || newest_positions == nullptr) return fail(PE_INVALID_ARG, "null argument");
    DevState& s = e->s;
    if (layer_begin < 0 || n_layers <= 0 || layer_begin + n_layers > s.n_layers)
        return fail(PE_INVALID_ARG, "layer range out of range");
    if (rule != PE_TOKEN_STREAMING && rule != PE_TOKEN_MAX_KEY_NORM && rule != PE_TOKEN_KEY_DIFF)
        return fail(PE_INVALID_ARG, "token rule (STREAMING, MAX_KEY_NORM or KEY_DIFF)");
    if (s.B > 64) return fail(PE_INVALID_ARG, "unstructured eviction needs page_size <= 64");
    cudaSetDevice(e->device);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    TableSet ts{layer_begin, n_layers};
    const int n = ts.size(s);
    pe_status r;
    const int64_t* dnew = newest_positions;
    if (!is_device_ptr(newest_positions)) {
        if ((r = ensure_t(&e->tok_newest, &e->tok_newest_elems, (size_t)s.n_seqs)) != PE_OK) return r;
        PE_CUDA(cudaMemcpyAsync(e->tok_newest, newest_positions, sizeof(int64_t) * s.n_seqs, cudaMemcpyHostToDevice,
                                st));
        dnew = e->tok_newest;
    }
    const bool vic_dev = victim_positions != nullptr && is_device_ptr(victim_positions);
    int64_t* dvic = vic_dev ? victim_positions : nullptr;
    if (victim_positions != nullptr && !vic_dev) {
        if ((r = ensure_t(&e->tok_victims, &e->tok_victims_elems, (size_t)s.n_tables)) != PE_OK) return r;
        dvic = e->tok_victims;
    }
    s.holes_on = 1;  // from now on every kernel honours the hole masks
    e->grid_tickets += (unsigned long long)n;  // one completion ticket per table
    token_evict_batch_kernel<<<n, 256, sizeof(float) * s.w, st>>>(s, ts, rule, static_cast<long long>(arg), s.C,
                                                                   dnew, dvic, e->vpage, e->grid_tickets - 1);
    if ((r = check_launch(e, "token_evict_batch_kernel")) != PE_OK) return r;
    e->stats.kernel_launches += 1;
    e->stats.evict_calls += 1;
    if (victim_positions != nullptr && !vic_dev)
        PE_CUDA(cudaMemcpyAsync(victim_positions, dvic, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
    return PE_OK;
}

pe_status pe_read_page_holes(pe_engine* e, int32_t page_begin, int32_t n_pages, uint64_t* holes) {
    if (e == nullptr || holes == nullptr) return fail(PE_INVALID_ARG, "null argument");
    const DevState& s = e->s;
    if (page_begin < 0 || n_pages < 0 || page_begin + n_pages > s.capacity)
        return fail(PE_INDEX_OUT_OF_RANGE, "page range out of range");
    cudaSetDevice(e->device);
    PE_CUDA(cudaDeviceSynchronize());
    PE_CUDA(cudaMemcpy(holes, s.holes + page_begin, sizeof(uint64_t) * n_pages, cudaMemcpyDeviceToHost));
    return PE_OK;
}

pe_status pe_check_invariants(pe_engine* e, pe_invariants* out) {
    if (e == nullptr || out == nullptr) return fail(PE_INVALID_ARG, "null argument");
    const DevState& s = e->s;
    cudaSetDevice(e->device);
    int32_t* refs = nullptr;
    unsigned long long* ctr = nullptr;
    if (dalloc(&refs, (size_t)s.capacity) != cudaSuccess || dalloc(&ctr, 8) != cudaSuccess) {
        cudaGetLastError();
        if (refs) cudaFree(refs);
        return fail(PE_CUDA_ERROR, "invariant scratch allocation failed");
    }
    cudaError_t ce = cudaMemset(refs, 0, sizeof(int32_t) * (size_t)s.capacity);
    if (ce == cudaSuccess) ce = cudaMemset(ctr, 0, sizeof(unsigned long long) * 8);
    if (ce == cudaSuccess) {
        invariants_tables_kernel<<<(s.n_tables + 7) / 8, 256>>>(s, refs, ctr);
        invariants_free_kernel<<<e->sm_count * 4, 256>>>(s, refs);
        invariants_refs_kernel<<<e->sm_count * 4, 256>>>(s, refs, ctr);
        ce = cudaGetLastError();
    }
    unsigned long long h[8] = {};
    int32_t top = 0;
    if (ce == cudaSuccess) ce = cudaMemcpy(h, ctr, sizeof(h), cudaMemcpyDeviceToHost);
    if (ce == cudaSuccess) ce = cudaMemcpy(&top, s.top, sizeof(int32_t), cudaMemcpyDeviceToHost);
    cudaFree(refs);
    cudaFree(ctr);
    if (ce != cudaSuccess) return fail(PE_CUDA_ERROR, std::string("invariant check: ") + cudaGetErrorString(ce));
    e->stats.kernel_launches += 3;
    std::memset(out, 0, sizeof(*out));
    out->tables_checked = s.n_tables;
    out->pages_mapped = (int64_t)h[0];
    out->free_pages = top;
    out->page_not_full = (int64_t)h[1];
    out->retained_mismatch = (int64_t)h[2];
    out->budget_violations = (int64_t)h[3];
    out->position_order = (int64_t)h[4];
    out->page_refcount = (int64_t)h[5];
    out->violations = out->page_not_full + out->retained_mismatch + out->budget_violations + out->position_order +
                      out->page_refcount;
    return PE_OK;
}

pe_status pe_pool_allocate(pe_engine* e, int32_t* page_id) {
    if (e != nullptr) e->append_chain = false;  // tables change outside the append chain
    if (e == nullptr || page_id == nullptr) return fail(PE_INVALID_ARG, "null argument");
    cudaSetDevice(e->device);
    pool_allocate_kernel<<<1, 1>>>(e->s, e->alloc_out);
    pe_status r = check_launch(e, "pool_allocate_kernel");
    if (r != PE_OK) return r;
    e->stats.kernel_launches += 1;
    if ((r = pe_sync(e)) != PE_OK) return r;
    PE_CUDA(cudaMemcpy(page_id, e->alloc_out, sizeof(int32_t), cudaMemcpyDeviceToHost));
    return PE_OK;
}

pe_status pe_pool_release(pe_engine* e, int32_t page_id) {
    if (e != nullptr) e->append_chain = false;  // tables change outside the append chain
    if (e == nullptr) return fail(PE_INVALID_ARG, "null engine");
    if (page_id < 0 || page_id >= e->s.capacity) return fail(PE_INDEX_OUT_OF_RANGE, "page id out of range");
    cudaSetDevice(e->device);
    pool_release_kernel<<<1, 1>>>(e->s, page_id);
    pe_status r = check_launch(e, "pool_release_kernel");
    if (r != PE_OK) return r;
    e->stats.kernel_launches += 1;
    return pe_sync(e);
}

// ------------------------------------------------------------------ baseline prefill selection
pe_status pe_prompt_select(int32_t device, int32_t rule, const float* keys, int32_t n, int32_t w,
                           const int64_t* positions, int32_t k, uint8_t* evicted_flags) {
    if (rule != PE_TOKEN_MAX_KEY_NORM && rule != PE_TOKEN_KEY_DIFF) return fail(PE_INVALID_ARG, "prompt rule");
    if (keys == nullptr || positions == nullptr || evicted_flags == nullptr) return fail(PE_INVALID_ARG, "null buffer");
    if (n <= 0 || w <= 0) return fail(PE_EMPTY_INPUT, "empty prompt");
    if (k < 0 || k > n) return fail(PE_K_TOO_LARGE, "k exceeds the scored tokens");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(PE_NO_DEVICE, "no CUDA device");
    }
    if (device < 0 || device >= ndev) return fail(PE_NO_DEVICE, "device ordinal out of range");
    PE_CUDA(cudaSetDevice(device));
    int n_pad = 1;
    while (n_pad < n) n_pad <<= 1;
    float *dk = nullptr, *mean = nullptr;
    double *score = nullptr, *mnorm = nullptr;
    long long *pos = nullptr, *spos = nullptr;
    int* sidx = nullptr;
    uint8_t* flags = nullptr;
    auto release = [&]() {
        void* ps[] = {dk, mean, score, mnorm, pos, spos, sidx, flags};
        for (void* p : ps)
            if (p) cudaFree(p);
    };
    if (dalloc(&dk, (size_t)n * w) != cudaSuccess || dalloc(&mean, (size_t)w) != cudaSuccess ||
        dalloc(&score, (size_t)n_pad) != cudaSuccess || dalloc(&mnorm, 1) != cudaSuccess ||
        dalloc(&pos, (size_t)n) != cudaSuccess || dalloc(&spos, (size_t)n_pad) != cudaSuccess ||
        dalloc(&sidx, (size_t)n_pad) != cudaSuccess || dalloc(&flags, (size_t)n) != cudaSuccess) {
        cudaGetLastError();
        release();
        return fail(PE_CUDA_ERROR, "device allocation failed");
    }
    cudaError_t ce = cudaMemcpy(dk, keys, sizeof(float) * (size_t)n * w, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaMemcpy(pos, positions, sizeof(int64_t) * n, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaMemset(flags, 0, n);
    if (ce == cudaSuccess && rule == PE_TOKEN_KEY_DIFF) {
        prompt_mean_key_kernel<<<1, 256>>>(dk, n, w, mean, mnorm);
        ce = cudaGetLastError();
    }
    if (ce == cudaSuccess) {
        prompt_score_kernel<<<(n_pad + 255) / 256, 256>>>(dk, n, w, rule, mean, mnorm, pos, n_pad, score, spos, sidx);
        for (int kk = 2; kk <= n_pad; kk <<= 1)
            for (int j = kk >> 1; j > 0; j >>= 1)
                bitonic_step_kernel<<<(n_pad + 255) / 256, 256>>>(score, spos, sidx, n_pad, j, kk);
        if (k > 0) flag_first_kernel<<<(k + 255) / 256, 256>>>(sidx, k, flags);
        ce = cudaGetLastError();
    }
    if (ce == cudaSuccess) ce = cudaMemcpy(evicted_flags, flags, (size_t)n, cudaMemcpyDeviceToHost);
    release();
    if (ce != cudaSuccess) return fail(PE_CUDA_ERROR, std::string("prompt select: ") + cudaGetErrorString(ce));
    return PE_OK;
}

pe_status pe_current_device(int32_t* device) {
    if (device == nullptr) return fail(PE_INVALID_ARG, "null argument");
    int ndev = 0, d = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(PE_NO_DEVICE, "no CUDA device");
    }
    PE_CUDA(cudaGetDevice(&d));
    *device = d;
    return PE_OK;
}

// ------------------------------------------------------------------ HBM probe
pe_status pe_probe_hbm(int32_t device, int64_t bytes, int32_t iters, double* read_gbs, double* copy_gbs) {
    if (bytes < (int64_t)(64 << 20) || iters <= 0) return fail(PE_INVALID_ARG, "probe needs >= 64 MB and iters > 0");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(PE_NO_DEVICE, "no CUDA device");
    }
    PE_CUDA(cudaSetDevice(device));
    int sms = 0;
    PE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const size_t n16 = (size_t)bytes / 32 * 2;  // multiple of 32 bytes
    uint4 *a = nullptr, *b = nullptr;
    unsigned long long* sink = nullptr;
    if (cudaMalloc(&a, n16 * 16) != cudaSuccess || cudaMalloc(&b, n16 * 16) != cudaSuccess ||
        cudaMalloc(&sink, 8) != cudaSuccess) {
        cudaGetLastError();
        if (a) cudaFree(a);
        if (b) cudaFree(b);
        return fail(PE_CUDA_ERROR, "probe allocation failed");
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaMemset(a, 0x5A, n16 * 16);
    const int grid = sms * 16;
    float best_r = 1e30f, best_c = 1e30f;
    for (int it = 0; it < iters + 1; ++it) {  // first pass warms up
        float ms = 0.f;
        cudaEventRecord(e0);
        probe_read_kernel<<<grid, 256>>>(a, n16, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (it > 0) best_r = std::min(best_r, ms);
        cudaEventRecord(e0);
        probe_copy_kernel<<<grid, 256>>>(a, b, n16);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (it > 0) best_c = std::min(best_c, ms);
    }
    const cudaError_t ce = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(a);
    cudaFree(b);
    cudaFree(sink);
    if (ce != cudaSuccess) return fail(PE_CUDA_ERROR, std::string("probe: ") + cudaGetErrorString(ce));
    if (read_gbs) *read_gbs = (double)n16 * 16 / (best_r * 1e-3) / 1e9;
    if (copy_gbs) *copy_gbs = 2.0 * (double)n16 * 16 / (best_c * 1e-3) / 1e9;
    return PE_OK;
}

}  // extern "C"
