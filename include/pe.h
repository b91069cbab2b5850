/*
 * pe.h — C-ABI of the B200-native PagedEviction engine (libpe_b200.so).
 *
 * This is the drop-in boundary for the reference's C++ cache-manager API
 * (/root/reference/proj/core/include/pagedevict/<header>.hpp). One engine owns, in
 * HBM of one GPU: the paged KV pool (PagePool), every table's block table
 * (BlockTable), the LIFO free list, the eviction policy and its budget
 * config (PolicyConfig). All compute runs in hand-written sm_100a kernels;
 * there is no CPU fallback: without a usable device every call returns
 * PE_NO_DEVICE.
 *
 * Mapping to the reference (file:line under proj/core/):
 *   pe_engine_create        PagePool(capacity, page_size)      page_pool.hpp:19-24, page_pool.cpp:8-22
 *                           + one BlockTable per table          block_table.hpp:21-24
 *                           + make_policy(PolicyConfig)          policy.hpp:31-39,122, policy.cpp:38-52,308-322
 *   pe_prefill_prune_pack   EvictionPolicy::prefill_compress    policy.hpp:106, policy.cpp:54-63,90-101,139-141
 *                           + BlockTable::append_token loop      block_table.cpp:10-19 (simulator.cpp:181-186)
 *   pe_decode_append        BlockTable::append_token            block_table.cpp:10-19, page_pool.cpp:24-33
 *   pe_decode_evict         PagedEvictionPolicy::evict           policy.cpp:143-155 -> score_pages/rank_pages
 *                                                               (importance.cpp:19-39,62-75) -> free_page
 *                                                               (block_table.cpp:21-31) -> release (page_pool.cpp:35-38)
 *   pe_decode_step          EvictionPolicy::decode_step         policy.hpp:110, policy.cpp:65-70
 *   pe_paged_decode_attention attend (per query head)           attention.hpp:26, attention.cpp:15-99
 *   pe_read_*               BlockTable accessors / PagePool     block_table.hpp:61-91, page_pool.hpp:30-38
 *   pe_status               the 12 pagedevict::Error classes    errors.hpp:12-88
 *
 * Tables. A table is the reference's (sequence, layer) BlockTable. With
 * PE_GRANULARITY_PER_KV_HEAD (default) there is one table per (sequence,
 * layer, kv_head) with row width w = head_dim; with PE_GRANULARITY_PER_LAYER
 * one table per (sequence, layer) with w = n_kv_heads*head_dim (heads
 * concatenated, exactly the reference's KvVector, kv_vector.hpp:23-27).
 * Table id: t = (seq*n_layers + layer)*tab_heads + head.
 *
 * Canonical batched order (the reference is per-sequence serial,
 * simulator.cpp:288-317): calls execute in stream order; inside one call,
 * tables are processed in ascending table id, and all free-list pops of a
 * call precede all of its pushes.
 *
 * Memory: K/V/Q/out/positions/victims pointers may be device pointers or
 * host pointers (host buffers are staged through the engine with
 * cudaMemcpyAsync on `stream`). Calls are asynchronous and stream-ordered;
 * device-side failures (pool exhaustion, table overflow) set a device status
 * word and make the failing launch a no-op; pe_sync() returns it.
 * Calls on one engine must be serialised by the caller (the reference's
 * BlockTable/EvictionPolicy are single-threaded, block_table.hpp:17-20).
 * The decode-path kernels (append, evict, attention) are launched with
 * programmatic dependent launch: each becomes resident behind the previous
 * kernel of the stream and waits for it before it reads inputs or table
 * state (plain stream-order semantics, without the launch gap); a per-layer
 * evict that directly follows an evict or attention call over other layers
 * of the same engine starts scoring early. Environment PE_PDL=0 /
 * PE_K2_PDL=0 turn this off.
 */
#ifndef PE_PE_H
#define PE_PE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PE_ABI_VERSION 1

typedef enum pe_status {
    PE_OK = 0,
    PE_ERROR = 1,                /* pagedevict::Error            errors.hpp:12-15 */
    PE_POOL_EXHAUSTED = 2,       /* PoolExhausted                errors.hpp:18-22 */
    PE_INDEX_OUT_OF_RANGE = 3,   /* IndexOutOfRange              errors.hpp:25-28 */
    PE_UNKNOWN_POSITION = 4,     /* UnknownPosition              errors.hpp:31-34 */
    PE_OVERFLOW = 5,             /* Overflow                     errors.hpp:37-40 */
    PE_EMPTY_PAGE = 6,           /* EmptyPage                    errors.hpp:43-46 */
    PE_K_TOO_LARGE = 7,          /* KTooLarge                    errors.hpp:49-52 */
    PE_NO_ELIGIBLE_PAGE = 8,     /* NoEligiblePage               errors.hpp:55-58 */
    PE_BUDGET_INVALID = 9,       /* BudgetInvalid                errors.hpp:61-64 */
    PE_EMPTY_CACHE = 10,         /* EmptyCache                   errors.hpp:67-70 */
    PE_LENGTH_MISMATCH = 11,     /* LengthMismatch               errors.hpp:73-76 */
    PE_EMPTY_INPUT = 12,         /* EmptyInput                   errors.hpp:79-82 */
    PE_IO_ERROR = 13,            /* IoError                      errors.hpp:85-88 */
    PE_INVALID_ARG = 20,         /* bad argument (engine-level)                     */
    PE_INVALID_STATE = 21,       /* e.g. prefill into a non-empty table, table full */
    PE_CUDA_ERROR = 30,          /* a CUDA runtime call failed                     */
    PE_NO_DEVICE = 31            /* no usable sm_100 device                        */
} pe_status;

typedef enum pe_dtype { PE_DTYPE_F32 = 0, PE_DTYPE_BF16 = 1 } pe_dtype;

/* PolicyKind (policy.hpp:17-23); the engine implements PagedEviction and
 * FullCache (the unpruned comparison). */
typedef enum pe_policy_kind {
    PE_POLICY_PAGED_EVICTION = 0,
    PE_POLICY_FULL_CACHE = 4
} pe_policy_kind;

typedef enum pe_granularity {
    PE_GRANULARITY_PER_KV_HEAD = 0,
    PE_GRANULARITY_PER_LAYER = 1
} pe_granularity;

/* How pe_decode_evict obtains page scores. RECOMPUTE reads every resident
 * page's K/V bytes and recomputes the fp64 token scores (the headline
 * eviction kernel); CACHED takes the page means cached when each page
 * filled (the reference caches norms at make_kv time, kv_vector.hpp:42-43).
 * Both give bit-identical decisions. */
typedef enum pe_score_mode { PE_SCORE_RECOMPUTE = 0, PE_SCORE_CACHED = 1 } pe_score_mode;

typedef struct pe_config {
    int32_t n_seqs;              /* sequences held by this engine (rank shard)   */
    int32_t n_layers;
    int32_t n_kv_heads;          /* KV heads per token in the input layout       */
    int32_t head_dim;
    int32_t granularity;         /* pe_granularity                               */
    int32_t page_size;           /* B  (PolicyConfig::page_size, default 16)      */
    int32_t cache_budget;        /* C  (PolicyConfig::cache_budget, default 256)  */
    int32_t dtype;               /* pe_dtype of K/V/Q                             */
    int32_t policy;              /* pe_policy_kind                                */
    int32_t capacity;            /* pool pages; 0 = n_tables*(C/B+1)              */
    int32_t max_pages_per_table; /* 0 = C/B+1 (PagedEviction); FullCache needs it */
    int32_t device;              /* CUDA device ordinal                           */
} pe_config;

typedef struct pe_engine pe_engine;

typedef struct pe_info {
    int32_t n_tables, tab_heads, width, page_size, cache_budget, capacity, max_pages;
    int32_t dtype, policy, granularity, row_pitch_bytes, sm_count;
    int64_t pool_bytes, state_bytes;
    int32_t free_pages;          /* synchronous read of the device stack top      */
    int32_t pad_;
} pe_info;

typedef struct pe_stats {
    int64_t prefill_calls, append_calls, evict_calls, attention_calls;
    int64_t tokens_scored;       /* prefill tokens scored on device               */
    int64_t pages_evicted;       /* synchronous read of the device counter        */
    int64_t kernel_launches;     /* engine kernels launched so far                */
} pe_stats;

/* Lifecycle. Validates the config like PolicyConfig::validate
 * (policy.cpp:38-52 -> PE_BUDGET_INVALID). */
pe_status pe_engine_create(const pe_config* cfg, pe_engine** out);
pe_status pe_engine_destroy(pe_engine* eng);

/* Prefill prune+pack of one layer for sequences [seq_begin, seq_begin+n_seqs).
 * k, v: [cu_seqlens[n_seqs], n_kv_heads, head_dim] (token-major). cu_seqlens
 * is a HOST array of n_seqs+1 prefix offsets. Token positions are 0..L-1.
 * Per table: if L > C (PagedEviction) the E = L-C lowest (score, position)
 * tokens are evicted and the survivors are packed in position order into
 * ceil(C/B) fresh pages; otherwise all L are packed. Target tables must be
 * empty. evicted_counts (nullable, host or device, [n_seqs*tab_heads] int32)
 * receives E per table in launch order. */
pe_status pe_prefill_prune_pack(pe_engine* eng, int32_t layer, const void* k, const void* v,
                                const int32_t* cu_seqlens, int32_t seq_begin, int32_t n_seqs,
                                int32_t* evicted_counts, void* stream);

/* Decode append of one token to every table of layers
 * [layer_begin, layer_begin+n_layers): k_rows/v_rows
 * [n_layers][n_seqs][n_kv_heads][head_dim]; positions [n_seqs] int64. */
pe_status pe_decode_append(pe_engine* eng, int32_t layer_begin, int32_t n_layers,
                           const void* k_rows, const void* v_rows, const int64_t* positions,
                           void* stream);

/* Decode eviction over the same table set. victims (nullable, host or
 * device) [n_layers*n_seqs*tab_heads] int32 receives the evicted logical
 * page index per table in launch order, or -1. */
pe_status pe_decode_evict(pe_engine* eng, int32_t layer_begin, int32_t n_layers, int64_t step,
                          int32_t mode, int32_t* victims, void* stream);

/* append + evict (EvictionPolicy::decode_step). */
pe_status pe_decode_step(pe_engine* eng, int32_t layer_begin, int32_t n_layers,
                         const void* k_rows, const void* v_rows, const int64_t* positions,
                         int64_t step, int32_t mode, int32_t* victims, void* stream);

/* GQA paged decode attention for one layer over the (pruned) tables.
 * q: [n_seqs][n_q_heads][head_dim] (dtype of the engine); out: float32
 * [n_seqs][n_q_heads][head_dim]. n_q_heads must be a multiple of
 * n_kv_heads (PER_KV_HEAD only). softmax(q.k/sqrt(d)).V per query head. */
pe_status pe_paged_decode_attention(pe_engine* eng, int32_t layer, const void* q, float* out,
                                    int32_t n_q_heads, void* stream);

/* Step-log capture (StepRecord, metrics.hpp:18-28; schemas/steplog.jsonl.md):
 * the engine-owned fields of one decode step per table. retained_len and
 * page_count as BlockTable::retained_len / page_count, newest_fill = occupied
 * slots of the newest page (Page::fill), victim = the evicted logical page
 * or -1 (EvictionDecision::Page / None). fragmentation and
 * fragmentation_excl_newest follow from these exactly as in
 * block_table.cpp:48-63 (pagedevict::step_records in the C++ façade,
 * paper_2509_04377_b200.steplog in Python). */
typedef struct pe_step_entry {
    int32_t retained_len;
    int32_t page_count;
    int32_t newest_fill;
    int32_t victim;
} pe_step_entry;

/* Writes one pe_step_entry per table of layers [layer_begin,
 * layer_begin+n_layers) in launch order into out (host or device,
 * stream-ordered). victims: the array (device) given to the preceding
 * pe_decode_evict / pe_decode_step over the same tables, or NULL for that
 * call's engine-side copy (when it was given a host array or none). */
pe_status pe_step_log_capture(pe_engine* eng, int32_t layer_begin, int32_t n_layers, const int32_t* victims,
                              pe_step_entry* out, void* stream);

/* Synchronises the engine's device work and returns the device status word
 * (PE_OK or the first failure since the last pe_sync). */
pe_status pe_sync(pe_engine* eng);

/* Readback (synchronous, host buffers, for parity checks and the façade). */
pe_status pe_get_info(pe_engine* eng, pe_info* out);
pe_status pe_get_stats(pe_engine* eng, pe_stats* out);
/* block_table [n_tables*max_pages] (-1 past num_pages), num_pages,
 * newest_fill, retained [n_tables]; any pointer may be NULL. */
pe_status pe_read_tables(pe_engine* eng, int32_t* block_table, int32_t* num_pages,
                         int32_t* newest_fill, int32_t* retained);
/* free stack bottom..top (top = next page handed out); *n_free = top. */
pe_status pe_read_free_list(pe_engine* eng, int32_t* stack_out, int32_t* n_free);
/* positions [n_pages][B] int32 and, if non-NULL, cached token scores
 * [n_pages][B] and page scores [n_pages] (double) for pages
 * [page_begin, page_begin+n_pages). */
pe_status pe_read_positions(pe_engine* eng, int32_t page_begin, int32_t n_pages,
                            int32_t* positions, double* token_scores, double* page_scores);
/* page bytes [n_pages][2][B][w] (dense rows, dtype of the engine). */
pe_status pe_read_pages(pe_engine* eng, int32_t page_begin, int32_t n_pages, void* out);

/* Raw device pointers of the engine state (advanced integration, e.g. a
 * serving stack's own attention kernel reading the pruned tables). */
typedef struct pe_device_view {
    void* pages;                 /* [capacity][2][B][row_pitch_bytes]            */
    int32_t* block_table;        /* [n_tables][max_pages]                        */
    int32_t* num_pages;
    int32_t* newest_fill;
    int32_t* retained;
    int32_t* positions;          /* [capacity][B]                                */
} pe_device_view;
pe_status pe_get_device_view(pe_engine* eng, pe_device_view* out);

/* ------------------------------------------------------------------------
 * Table-granular API: the reference's per-object calls, one BlockTable per
 * table id. This is what the C++ façade (include/pe/pagedevict.hpp,
 * libpagedevict_b200.so) binds; appends and PagedEviction decisions go
 * through the same kernels as the batched calls (K0, K2/K2c) with an
 * explicit table list. Table lists are HOST arrays of strictly ascending ids
 * (the canonical order); row i of k_rows/v_rows/positions belongs to
 * table_ids[i]. Device-side failures set the status word read by pe_sync.
 * ---------------------------------------------------------------------- */

/* BlockTable::append_token for each listed table (block_table.cpp:10-19):
 * writes into the newest page's next slot, opening a page (PagePool::allocate,
 * page_pool.cpp:24-33) when the newest page is write-full or none exists.
 * Pool exhaustion -> PE_POOL_EXHAUSTED at pe_sync; tables before the failing
 * one (ascending id) are appended, later ones are not (reference loop order). */
pe_status pe_table_append(pe_engine* eng, int32_t n, const int32_t* table_ids, const void* k_rows,
                          const void* v_rows, const int64_t* positions, void* stream);

/* PagedEvictionPolicy::evict (policy.cpp:143-155) with C = cache_budget for
 * each listed table: trigger iff the newest page is write-full and
 * retained > C; then score_pages -> rank_pages -> free_page. victims
 * (nullable, host or device) [n] receives the evicted logical index or -1. */
pe_status pe_table_evict(pe_engine* eng, int32_t n, const int32_t* table_ids, int32_t cache_budget,
                         int32_t mode, int32_t* victims, void* stream);

/* BlockTable::free_page (block_table.cpp:21-31): releases the page at
 * logical_index whole, later entries close ranks. Out of range ->
 * PE_INDEX_OUT_OF_RANGE at pe_sync (no-op). */
pe_status pe_table_free_page(pe_engine* eng, int32_t table, int32_t logical_index, void* stream);

/* BlockTable::clear (block_table.cpp:72-78): releases every mapped page in
 * logical order. */
pe_status pe_table_clear(pe_engine* eng, int32_t table, void* stream);

/* attend_detailed (attention.cpp:15-99) over one table: per head h, softmax
 * of q_h.k_h/sqrt(head_dim) over the retained tokens in logical order,
 * heads concatenated in the row (head h = elements [h*head_dim, (h+1)*head_dim)).
 * Double-precision in the reference's order (bit-identical up to the last
 * ulp of exp). query float32 [head_count*head_dim]; out float32 (same
 * length); weight_sums (nullable) double [head_count]. No retained token ->
 * PE_EMPTY_CACHE; head_count*head_dim wider than the rows -> PE_LENGTH_MISMATCH. */
pe_status pe_table_attend(pe_engine* eng, int32_t table, const float* query, int32_t head_count,
                          int32_t head_dim, float* out, double* weight_sums, void* stream);

/* Unstructured (per-token) eviction of one table: picks a victim among the
 * retained tokens (logical order) by `rule`, clears its slot and releases
 * its page once drained (BlockTable::evict_slot, block_table.cpp:33-46).
 * Rules:
 *   PE_TOKEN_AT_POSITION   the token at position `arg`; none -> PE_UNKNOWN_POSITION
 *   PE_TOKEN_STREAMING     oldest token with position >= arg (sink count)  policy.cpp:184-206
 *   PE_TOKEN_MAX_KEY_NORM  largest ||K||, first on ties                    policy.cpp:219-237
 *   PE_TOKEN_KEY_DIFF      largest cos(K, mean retained K), first on ties  policy.cpp:263-283
 * The policy rules skip the token at newest_position and fire only when
 * retained > cache_budget (cache_budget < 0: unconditional).
 * *victim_position (nullable) <- evicted position or -1. Needs page_size <= 64;
 * afterwards pe_paged_decode_attention refuses the engine (holes). */
typedef enum pe_token_rule {
    PE_TOKEN_AT_POSITION = 0,
    PE_TOKEN_STREAMING = 1,
    PE_TOKEN_MAX_KEY_NORM = 2,
    PE_TOKEN_KEY_DIFF = 3
} pe_token_rule;
pe_status pe_table_evict_token(pe_engine* eng, int32_t table, int32_t rule, int64_t arg, int32_t cache_budget,
                               int64_t newest_position, int64_t* victim_position, void* stream);

/* Batched token eviction: the decode step of the StreamingLLM / InvKeyL2 /
 * KeyDiff baselines (StreamingLlmPolicy / InvKeyL2Policy / KeyDiffPolicy::
 * evict, policy.cpp:184-283) over every table of layers [layer_begin,
 * layer_begin+n_layers), after the step's pe_decode_append. Every table
 * holding more than the engine's budget C evicts one token by `rule`:
 * PE_TOKEN_STREAMING (arg = sink count), PE_TOKEN_MAX_KEY_NORM or
 * PE_TOKEN_KEY_DIFF; a page that drains is released (pushed in ascending
 * table id after the append launch's pops). newest_positions [n_seqs] int64
 * (host or device): the step's appended position, never a candidate.
 * victim_positions (nullable, host or device) [n_layers*n_seqs*tab_heads]
 * int64: the evicted position per table in launch order, or -1. */
pe_status pe_decode_evict_tokens(pe_engine* eng, int32_t layer_begin, int32_t n_layers, int32_t rule, int64_t arg,
                                 const int64_t* newest_positions, int64_t* victim_positions, void* stream);

/* Evicted-slot masks (bit s = slot s is a hole) of pages [page_begin, +n_pages). */
pe_status pe_read_page_holes(pe_engine* eng, int32_t page_begin, int32_t n_pages, uint64_t* holes);

/* Prefill selection of the score-based baselines (compress_by_score,
 * policy.cpp:90-101): scores every prompt token on `device` —
 * PE_TOKEN_MAX_KEY_NORM: 1 / max(||K||, 1e-12) (InvKeyL2, policy.cpp:212-216);
 * PE_TOKEN_KEY_DIFF: -cos(K, mean prompt K) (KeyDiff, policy.cpp:244-260) —
 * and flags the k lowest (score, position) tokens (rank_tokens,
 * importance.cpp:41-60). keys: HOST float32 [n][w]; positions: HOST [n];
 * evicted_flags: HOST [n]. Stateless (no engine). */
pe_status pe_prompt_select(int32_t device, int32_t rule, const float* keys, int32_t n, int32_t w,
                           const int64_t* positions, int32_t k, uint8_t* evicted_flags);

/* Structural invariants of the whole engine state, checked on the device
 * (selfcheck.cpp:19-75, test_policies.cpp:220-234,437-473):
 * every non-newest page full and hole-free, retained == the occupied slots,
 * PagedEviction retained <= C + B, positions strictly increasing in logical
 * order, every page id either mapped exactly once or free exactly once
 * (page conservation, allocated + free == capacity). Synchronous. */
typedef struct pe_invariants {
    int64_t tables_checked;
    int64_t pages_mapped;
    int64_t free_pages;
    int64_t violations;          /* sum of the counts below */
    int64_t page_not_full;       /* a non-newest page with holes                 */
    int64_t retained_mismatch;   /* retained != occupied slots of the table      */
    int64_t budget_violations;   /* PagedEviction engine: retained > C + B       */
    int64_t position_order;      /* positions not strictly increasing            */
    int64_t page_refcount;       /* page ids mapped/free != exactly once         */
} pe_invariants;
pe_status pe_check_invariants(pe_engine* eng, pe_invariants* out);

/* HBM roofline probe: best-of-iters streaming read and copy bandwidth (GB/s,
 * bytes counted once per direction) over a `bytes` buffer (>= 64 MB; use
 * more than L2) on `device`. Synchronous; allocates 2 x bytes. */
pe_status pe_probe_hbm(int32_t device, int64_t bytes, int32_t iters, double* read_gbs, double* copy_gbs);

/* One table's block-table row (page_ids [num_pages], nullable) and counters. */
pe_status pe_read_table(pe_engine* eng, int32_t table, int32_t* page_ids, int32_t* num_pages,
                        int32_t* newest_fill, int32_t* retained);

/* PagePool::allocate / release (page_pool.cpp:24-38) on the device free
 * list, synchronous. Empty list -> PE_POOL_EXHAUSTED. */
pe_status pe_pool_allocate(pe_engine* eng, int32_t* page_id);
pe_status pe_pool_release(pe_engine* eng, int32_t page_id);

/* The calling host thread's current CUDA device (cudaGetDevice): the device
 * stateless helpers such as the façade's prefill selection run on, so a
 * multi-GPU process (one host thread per GPU) never funnels
 * them onto device 0. PE_NO_DEVICE without a CUDA device. */
pe_status pe_current_device(int32_t* device);

/* Thread-local message for the last non-OK status returned on this thread. */
const char* pe_last_error(void);
const char* pe_status_string(pe_status s);
int32_t pe_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PE_PE_H */
