/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT PATH.
 *
 * pe_oracle: a plain-C restatement of the reference PagedEviction hot path
 * (arxiv 2509.04377 reference, /root/reference/proj/core), restated over the
 * SAME flat data layout the CUDA engine keeps in HBM so that every engine
 * array (pages, positions, block tables, free stack, decisions) can be
 * compared byte for byte. Each function cites the reference file:line it
 * follows. Parity of this restatement is pinned against the reference
 * library itself (oracle/_ref, built from the reference sources) in
 * tests/test_oracle_pinning.py and against the golden fixtures in
 * tests/golden/.
 *
 * Batched canonical order (the reference is per-sequence serial,
 * simulator.cpp:288-317): within one launch, tables are
 * visited in ascending table id; all free-list pops happen before all pushes.
 */
#ifndef PE_ORACLE_H
#define PE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { PEO_F32 = 0, PEO_BF16 = 1 };
enum { PEO_PAGED_EVICTION = 0, PEO_FULL_CACHE = 4 };

/* kNormEpsilon, importance.hpp:17 */
#define PEO_NORM_EPS 1e-12

/* l2_norm, kv_vector.hpp:15-21: double accumulation in index order. */
double peo_l2_norm(const void* x, size_t n, int dtype);
/* token_importance, importance.cpp:11-13 over make_kv's cached norms
 * (kv_vector.hpp:42-43). */
double peo_token_score(const void* k, const void* v, size_t w, int dtype);
/* rank_tokens, importance.cpp:41-60: the k lowest (score, position) keys,
 * output sorted by position. Returns 0, or 7 (KTooLarge) when k > n. */
int peo_rank_tokens(const int64_t* positions, const double* scores, size_t n, size_t k,
                    int64_t* out);
/* rank_pages, importance.cpp:62-75: argmin, strict <, ties -> smaller index.
 * Returns -1 on empty input (NoEligiblePage). */
int64_t peo_rank_pages(const double* scores, size_t n);
/* output_deviation, attention.cpp:105-118 */
double peo_output_deviation(const float* a, const float* b, size_t n);
/* attend (head_count = 1 over a contiguous token list), attention.cpp:15-93 */
void peo_attend_dense(const float* q, const float* keys, const float* values, size_t n,
                      size_t d, float* out);

typedef struct peo_engine {
    /* geometry */
    int32_t n_seqs, n_layers, n_tab_heads; /* tables per (seq, layer) */
    int32_t width;                         /* row width w (elements) */
    int32_t page_size;                     /* B */
    int32_t budget;                        /* C */
    int32_t dtype, policy;
    int32_t capacity, max_pages;
    int32_t n_tables;
    /* state (same layout as the device engine) */
    uint8_t* pages;          /* [cap][2][B][w] elements */
    int32_t* positions;      /* [cap][B] */
    double* token_scores;    /* [cap][B] */
    double* page_scores;     /* [cap] (valid for full pages) */
    int32_t* block_table;    /* [n_tables][max_pages] */
    int32_t* num_pages;      /* [n_tables] */
    int32_t* newest_fill;    /* [n_tables] */
    int32_t* retained;       /* [n_tables] */
    int32_t* stack;          /* [cap], stack[0..top) free, top-1 popped first */
    int32_t top;
    int32_t status;
} peo_engine;

int peo_engine_create(peo_engine** out, int32_t n_seqs, int32_t n_layers, int32_t n_tab_heads,
                      int32_t width, int32_t page_size, int32_t budget, int32_t dtype,
                      int32_t policy, int32_t capacity, int32_t max_pages);
void peo_engine_destroy(peo_engine* e);

/* Prefill prune+pack for one layer: K/V [tokens][n_tab_heads][w] with
 * sequence s of the launch spanning cu_seqlens[s]..cu_seqlens[s+1],
 * positions 0..L-1. Tables must be empty. Policy: prefill_compress
 * (policy.cpp:54-63) -> compress_by_score (policy.cpp:90-101) -> append
 * survivors (block_table.cpp:10-19). `evicted_count` [n_seqs*n_tab_heads]
 * receives E per table. */
int peo_prefill(peo_engine* e, int32_t layer, const void* k, const void* v,
                const int32_t* cu_seqlens, int32_t seq_begin, int32_t n_seqs,
                int32_t* evicted_count);

/* Decode append of one token per table for layers [layer_begin,
 * layer_begin+n_layers): rows [n_layers][n_seqs][n_tab_heads][w]; position
 * per sequence. BlockTable::append_token (block_table.cpp:10-19) with the
 * LIFO PagePool::allocate (page_pool.cpp:24-33), serially in ascending table
 * id: the first failing pop stops the launch (PoolExhausted). */
int peo_decode_append(peo_engine* e, int32_t layer_begin, int32_t n_layers, const void* k,
                      const void* v, const int64_t* positions);

/* Decode eviction over the same table set: PagedEvictionPolicy::evict
 * (policy.cpp:143-155) with scores recomputed from page bytes.
 * victims [n_layers*n_seqs*n_tab_heads] in launch-table order: logical index
 * or -1. */
int peo_decode_evict(peo_engine* e, int32_t layer_begin, int32_t n_layers, int32_t* victims);

/* GQA paged decode attention for one layer: q [n_seqs][n_tab_heads*G][d]
 * (PER_KV_HEAD, w == d); out float [n_seqs][n_tab_heads*G][d]. attend per
 * query head with head_count 1 (attention.cpp:15-93). */
int peo_attention(peo_engine* e, int32_t layer, const void* q, int32_t G, float* out);

int32_t peo_table_id(const peo_engine* e, int32_t seq, int32_t layer, int32_t head);

#ifdef __cplusplus
}
#endif
#endif
