/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT PATH.
 * Plain-C restatement of the reference PagedEviction hot path; see
 * pe_oracle.h for the contract and the parity pins. Compiled with
 * -ffp-contract=off so every double operation is the separately rounded IEEE
 * operation the reference performs. */
#include "pe_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* status numbering follows include/pe/pe.h */
enum {
    ST_OK = 0,
    ST_POOL_EXHAUSTED = 2,
    ST_INDEX_OUT_OF_RANGE = 3,
    ST_K_TOO_LARGE = 7,
    ST_BUDGET_INVALID = 9,
    ST_EMPTY_CACHE = 10,
    ST_INVALID_ARG = 20,
    ST_INVALID_STATE = 21,
};

static float bf16_to_f32(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

static float elem(const void* base, size_t i, int dtype) {
    if (dtype == PEO_BF16) return bf16_to_f32(((const uint16_t*)base)[i]);
    return ((const float*)base)[i];
}

static size_t esize(int dtype) { return dtype == PEO_BF16 ? 2 : 4; }

/* kv_vector.hpp:15-21 */
double peo_l2_norm(const void* x, size_t n, int dtype) {
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double xi = (double)elem(x, i, dtype);
        acc += xi * xi;
    }
    return sqrt(acc);
}

/* importance.cpp:11-13: value_norm / max(key_norm, kNormEpsilon) */
double peo_token_score(const void* k, const void* v, size_t w, int dtype) {
    const double kn = peo_l2_norm(k, w, dtype);
    const double vn = peo_l2_norm(v, w, dtype);
    return vn / (kn > PEO_NORM_EPS ? kn : PEO_NORM_EPS);
}

/* importance.cpp:19-30: mean over occupied slots, sum in slot order. */
static double page_mean(const double* slot_scores, int32_t fill) {
    double sum = 0.0;
    for (int32_t s = 0; s < fill; ++s) sum += slot_scores[s];
    return sum / (double)fill;
}

typedef struct {
    double score;
    int64_t pos;
} key_t_;

/* Comparator of importance.cpp:47-52: score asc, then position asc. */
static int key_cmp(const void* a, const void* b) {
    const key_t_* x = (const key_t_*)a;
    const key_t_* y = (const key_t_*)b;
    if (x->score != y->score) return x->score < y->score ? -1 : 1;
    return (x->pos > y->pos) - (x->pos < y->pos);
}

static int i64_cmp(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* importance.cpp:41-60 */
int peo_rank_tokens(const int64_t* positions, const double* scores, size_t n, size_t k,
                    int64_t* out) {
    if (k > n) return ST_K_TOO_LARGE;
    key_t_* order = (key_t_*)malloc((n ? n : 1) * sizeof(key_t_));
    for (size_t i = 0; i < n; ++i) {
        order[i].score = scores[i];
        order[i].pos = positions[i];
    }
    qsort(order, n, sizeof(key_t_), key_cmp);
    for (size_t i = 0; i < k; ++i) out[i] = order[i].pos;
    qsort(out, k, sizeof(int64_t), i64_cmp);
    free(order);
    return ST_OK;
}

/* importance.cpp:62-75 */
int64_t peo_rank_pages(const double* scores, size_t n) {
    if (n == 0) return -1;
    size_t best = 0;
    for (size_t i = 1; i < n; ++i) {
        if (scores[i] < scores[best]) best = i; /* equal scores keep the smaller index */
    }
    return (int64_t)best;
}

/* attention.cpp:105-118 */
double peo_output_deviation(const float* a, const float* b, size_t n) {
    double diff = 0.0, ref = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double d = (double)a[i] - (double)b[i];
        diff += d * d;
        ref += (double)b[i] * (double)b[i];
    }
    const double r = sqrt(ref);
    return sqrt(diff) / (r > 1e-12 ? r : 1e-12);
}

/* attention.cpp:15-93 with heads = 1 */
void peo_attend_dense(const float* q, const float* keys, const float* values, size_t n,
                      size_t d, float* out) {
    const double scale = 1.0 / sqrt((double)d);
    double* logits = (double*)malloc((n ? n : 1) * sizeof(double));
    double* acc = (double*)calloc(d, sizeof(double));
    for (size_t t = 0; t < n; ++t) {
        double dot = 0.0;
        for (size_t i = 0; i < d; ++i) dot += (double)q[i] * (double)keys[t * d + i];
        logits[t] = dot * scale;
    }
    double mx = -INFINITY;
    for (size_t t = 0; t < n; ++t) mx = logits[t] > mx ? logits[t] : mx;
    double wsum = 0.0;
    for (size_t t = 0; t < n; ++t) {
        logits[t] = exp(logits[t] - mx);
        wsum += logits[t];
    }
    for (size_t t = 0; t < n; ++t) {
        const double w = logits[t] / wsum;
        for (size_t i = 0; i < d; ++i) acc[i] += w * (double)values[t * d + i];
    }
    for (size_t i = 0; i < d; ++i) out[i] = (float)acc[i];
    free(logits);
    free(acc);
}

/* ------------------------------------------------------------------ engine */

int peo_engine_create(peo_engine** out, int32_t n_seqs, int32_t n_layers, int32_t n_tab_heads,
                      int32_t width, int32_t page_size, int32_t budget, int32_t dtype,
                      int32_t policy, int32_t capacity, int32_t max_pages) {
    /* PolicyConfig::validate, policy.cpp:38-52 */
    if (page_size <= 0 || budget < page_size || budget % page_size != 0) return ST_BUDGET_INVALID;
    if (n_seqs <= 0 || n_layers <= 0 || n_tab_heads <= 0 || width <= 0 || capacity < 0 ||
        max_pages <= 0)
        return ST_INVALID_ARG;
    if (dtype != PEO_F32 && dtype != PEO_BF16) return ST_INVALID_ARG;
    if (policy != PEO_PAGED_EVICTION && policy != PEO_FULL_CACHE) return ST_INVALID_ARG;
    peo_engine* e = (peo_engine*)calloc(1, sizeof(peo_engine));
    e->n_seqs = n_seqs;
    e->n_layers = n_layers;
    e->n_tab_heads = n_tab_heads;
    e->width = width;
    e->page_size = page_size;
    e->budget = budget;
    e->dtype = dtype;
    e->policy = policy;
    e->capacity = capacity;
    e->max_pages = max_pages;
    e->n_tables = n_seqs * n_layers * n_tab_heads;
    const size_t cap = (size_t)(capacity ? capacity : 1);
    e->pages = (uint8_t*)calloc(cap * 2 * page_size * (size_t)width, esize(dtype));
    e->positions = (int32_t*)calloc(cap * page_size, sizeof(int32_t));
    e->token_scores = (double*)calloc(cap * page_size, sizeof(double));
    e->page_scores = (double*)calloc(cap, sizeof(double));
    e->block_table = (int32_t*)malloc((size_t)e->n_tables * max_pages * sizeof(int32_t));
    for (size_t i = 0; i < (size_t)e->n_tables * max_pages; ++i) e->block_table[i] = -1;
    e->num_pages = (int32_t*)calloc(e->n_tables, sizeof(int32_t));
    e->newest_fill = (int32_t*)calloc(e->n_tables, sizeof(int32_t));
    e->retained = (int32_t*)calloc(e->n_tables, sizeof(int32_t));
    /* LIFO free list initialised [cap-1, ..., 0]; the back (top) is popped
     * first, so low ids are handed out first: page_pool.cpp:18-21 */
    e->stack = (int32_t*)malloc(cap * sizeof(int32_t));
    for (int32_t i = 0; i < capacity; ++i) e->stack[i] = capacity - 1 - i;
    e->top = capacity;
    *out = e;
    return ST_OK;
}

void peo_engine_destroy(peo_engine* e) {
    if (!e) return;
    free(e->pages);
    free(e->positions);
    free(e->token_scores);
    free(e->page_scores);
    free(e->block_table);
    free(e->num_pages);
    free(e->newest_fill);
    free(e->retained);
    free(e->stack);
    free(e);
}

int32_t peo_table_id(const peo_engine* e, int32_t seq, int32_t layer, int32_t head) {
    return (seq * e->n_layers + layer) * e->n_tab_heads + head;
}

static uint8_t* page_row(peo_engine* e, int32_t page, int kv, int32_t slot) {
    const size_t es = esize(e->dtype);
    return e->pages + (((size_t)page * 2 + kv) * e->page_size + slot) * e->width * es;
}

/* Page::write at the cursor (page.hpp:39-44) plus the cached score. */
static void write_slot(peo_engine* e, int32_t page, int32_t slot, const void* krow,
                       const void* vrow, int32_t pos, double score) {
    const size_t rb = (size_t)e->width * esize(e->dtype);
    memcpy(page_row(e, page, 0, slot), krow, rb);
    memcpy(page_row(e, page, 1, slot), vrow, rb);
    e->positions[(size_t)page * e->page_size + slot] = pos;
    e->token_scores[(size_t)page * e->page_size + slot] = score;
    if (slot == e->page_size - 1) {
        e->page_scores[page] =
            page_mean(e->token_scores + (size_t)page * e->page_size, e->page_size);
    }
}

static int32_t pages_for(int32_t n, int32_t b) { return (n + b - 1) / b; }

int peo_prefill(peo_engine* e, int32_t layer, const void* k, const void* v,
                const int32_t* cu_seqlens, int32_t seq_begin, int32_t n_seqs,
                int32_t* evicted_count) {
    const int32_t H = e->n_tab_heads, B = e->page_size, C = e->budget, w = e->width;
    const size_t es = esize(e->dtype);
    if (layer < 0 || layer >= e->n_layers || seq_begin < 0 || n_seqs < 0 ||
        seq_begin + n_seqs > e->n_seqs)
        return ST_INVALID_ARG;
    /* Whole-launch pre-checks (the device engine is all-or-nothing). */
    int64_t need = 0;
    for (int32_t s = 0; s < n_seqs; ++s) {
        const int32_t L = cu_seqlens[s + 1] - cu_seqlens[s];
        if (L <= 0) return ST_INVALID_ARG; /* policy.cpp:57-58: empty prefill */
        const int32_t keep = (e->policy == PEO_PAGED_EVICTION && L > C) ? C : L;
        if (pages_for(keep, B) > e->max_pages) return ST_INVALID_ARG;
        for (int32_t h = 0; h < H; ++h) {
            if (e->num_pages[peo_table_id(e, seq_begin + s, layer, h)] != 0)
                return ST_INVALID_STATE;
        }
        need += (int64_t)pages_for(keep, B) * H;
    }
    if (need > e->top) {
        e->status = ST_POOL_EXHAUSTED;
        return ST_POOL_EXHAUSTED;
    }
    for (int32_t s = 0; s < n_seqs; ++s) {
        const int32_t L = cu_seqlens[s + 1] - cu_seqlens[s];
        for (int32_t h = 0; h < H; ++h) {
            const int32_t t = peo_table_id(e, seq_begin + s, layer, h);
            const uint8_t* kb = (const uint8_t*)k;
            const uint8_t* vb = (const uint8_t*)v;
#define ROW(base, i) ((base) + (((size_t)(cu_seqlens[s] + (i)) * H + h) * w) * es)
            /* make_kv norms + token_importance for every token. */
            double* sc = (double*)malloc((size_t)L * sizeof(double));
            for (int32_t i = 0; i < L; ++i)
                sc[i] = peo_token_score(ROW(kb, i), ROW(vb, i), (size_t)w, e->dtype);
            uint8_t* evict = (uint8_t*)calloc((size_t)L, 1);
            int32_t E = 0;
            if (e->policy == PEO_PAGED_EVICTION && L > C) {
                /* compress_by_score, policy.cpp:90-101: rank_tokens(k = L - C)
                 * then drop_positions (policy.cpp:75-86) */
                E = L - C;
                int64_t* pos = (int64_t*)malloc((size_t)L * sizeof(int64_t));
                int64_t* out = (int64_t*)malloc((size_t)E * sizeof(int64_t));
                for (int32_t i = 0; i < L; ++i) pos[i] = i;
                peo_rank_tokens(pos, sc, (size_t)L, (size_t)E, out);
                for (int32_t i = 0; i < E; ++i) evict[out[i]] = 1;
                free(pos);
                free(out);
            }
            if (evicted_count) evicted_count[s * H + h] = E;
            /* append survivors in position order: block_table.cpp:10-19 */
            int32_t q = 0;
            for (int32_t i = 0; i < L; ++i) {
                if (evict[i]) continue;
                const int32_t slot = q % B;
                if (slot == 0) {
                    const int32_t page = e->stack[--e->top]; /* page_pool.cpp:29-31 */
                    e->block_table[(size_t)t * e->max_pages + e->num_pages[t]] = page;
                    e->num_pages[t] += 1;
                }
                const int32_t page = e->block_table[(size_t)t * e->max_pages + e->num_pages[t] - 1];
                write_slot(e, page, slot, ROW(kb, i), ROW(vb, i), i, sc[i]);
                ++q;
            }
#undef ROW
            e->retained[t] = q;
            e->newest_fill[t] = q - (e->num_pages[t] - 1) * B;
            free(sc);
            free(evict);
        }
    }
    return ST_OK;
}

/* Appends run serially in ascending table id, like the reference's loop of
 * append_token calls (block_table.cpp:10-19): the first pop that finds the
 * free list empty fails with PoolExhausted (page_pool.cpp:26-28) and stops
 * the launch (later tables are not appended). A popping table already at
 * max_pages is skipped with PE_INVALID_STATE. Errors are sticky in
 * e->status; the first one is returned. */
int peo_decode_append(peo_engine* e, int32_t layer_begin, int32_t n_layers, const void* k,
                      const void* v, const int64_t* positions) {
    const int32_t H = e->n_tab_heads, B = e->page_size, w = e->width, S = e->n_seqs;
    const size_t es = esize(e->dtype);
    if (layer_begin < 0 || n_layers <= 0 || layer_begin + n_layers > e->n_layers)
        return ST_INVALID_ARG;
    int rc = ST_OK;
    /* ascending table id == seq-major, then layer, then head */
    for (int32_t s = 0; s < S; ++s)
        for (int32_t l = layer_begin; l < layer_begin + n_layers; ++l)
            for (int32_t h = 0; h < H; ++h) {
                const int32_t t = peo_table_id(e, s, l, h);
                const size_t off = ((((size_t)(l - layer_begin) * S + s) * H + h) * w) * es;
                const uint8_t* kr = (const uint8_t*)k + off;
                const uint8_t* vr = (const uint8_t*)v + off;
                if (e->num_pages[t] == 0 || e->newest_fill[t] == B) {
                    if (e->num_pages[t] >= e->max_pages) {
                        if (!e->status) e->status = ST_INVALID_STATE;
                        if (!rc) rc = ST_INVALID_STATE;
                        continue;
                    }
                    if (e->top == 0) {
                        if (!e->status) e->status = ST_POOL_EXHAUSTED;
                        if (!rc) rc = ST_POOL_EXHAUSTED;
                        return rc;
                    }
                    const int32_t page = e->stack[--e->top];
                    e->block_table[(size_t)t * e->max_pages + e->num_pages[t]] = page;
                    e->num_pages[t] += 1;
                    e->newest_fill[t] = 0;
                }
                const int32_t page = e->block_table[(size_t)t * e->max_pages + e->num_pages[t] - 1];
                write_slot(e, page, e->newest_fill[t], kr, vr, (int32_t)positions[s],
                           peo_token_score(kr, vr, (size_t)w, e->dtype));
                e->newest_fill[t] += 1;
                e->retained[t] += 1;
            }
    return rc;
}

int peo_decode_evict(peo_engine* e, int32_t layer_begin, int32_t n_layers, int32_t* victims) {
    const int32_t H = e->n_tab_heads, B = e->page_size, C = e->budget, S = e->n_seqs;
    if (layer_begin < 0 || n_layers <= 0 || layer_begin + n_layers > e->n_layers)
        return ST_INVALID_ARG;
    double* ps = (double*)malloc((size_t)e->max_pages * sizeof(double));
    double* ts = (double*)malloc((size_t)B * sizeof(double));
    int32_t idx = 0;
    for (int32_t s = 0; s < S; ++s)
        for (int32_t l = layer_begin; l < layer_begin + n_layers; ++l)
            for (int32_t h = 0; h < H; ++h, ++idx) {
                const int32_t t = peo_table_id(e, s, l, h);
                victims[idx] = -1;
                /* trigger: newest page write-full and retained > C,
                 * policy.cpp:147-150 */
                if (e->policy != PEO_PAGED_EVICTION || e->num_pages[t] == 0 ||
                    e->newest_fill[t] != B || e->retained[t] <= C)
                    continue;
                const int32_t N = e->num_pages[t];
                int32_t* row = e->block_table + (size_t)t * e->max_pages;
                /* score_pages -> page_score, importance.cpp:19-39, with token
                 * scores recomputed from the resident K/V bytes */
                for (int32_t j = 0; j < N; ++j) {
                    const int32_t fill = (j == N - 1) ? e->newest_fill[t] : B;
                    for (int32_t sl = 0; sl < fill; ++sl)
                        ts[sl] = peo_token_score(page_row(e, row[j], 0, sl),
                                                 page_row(e, row[j], 1, sl), (size_t)e->width,
                                                 e->dtype);
                    ps[j] = page_mean(ts, fill);
                }
                const int64_t victim = peo_rank_pages(ps, (size_t)N); /* importance.cpp:62-75 */
                /* free_page: retained -= fill, release, erase (shift left),
                 * block_table.cpp:21-31 + page_pool.cpp:35-38 */
                const int32_t page = row[victim];
                e->retained[t] -= B; /* every page is full at a trigger */
                for (int32_t j = (int32_t)victim; j < N - 1; ++j) row[j] = row[j + 1];
                row[N - 1] = -1;
                e->num_pages[t] = N - 1;
                e->newest_fill[t] = N - 1 > 0 ? B : 0;
                e->stack[e->top++] = page;
                victims[idx] = (int32_t)victim;
            }
    free(ps);
    free(ts);
    return ST_OK;
}

int peo_attention(peo_engine* e, int32_t layer, const void* q, int32_t G, float* out) {
    const int32_t H = e->n_tab_heads, B = e->page_size, d = e->width, S = e->n_seqs;
    if (layer < 0 || layer >= e->n_layers || G <= 0) return ST_INVALID_ARG;
    int32_t maxr = 0;
    for (int32_t t = 0; t < e->n_tables; ++t) maxr = e->retained[t] > maxr ? e->retained[t] : maxr;
    float* kk = (float*)malloc((size_t)(maxr ? maxr : 1) * d * sizeof(float));
    float* vv = (float*)malloc((size_t)(maxr ? maxr : 1) * d * sizeof(float));
    float* qq = (float*)malloc((size_t)d * sizeof(float));
    for (int32_t s = 0; s < S; ++s)
        for (int32_t h = 0; h < H; ++h) {
            const int32_t t = peo_table_id(e, s, layer, h);
            const int32_t R = e->retained[t];
            if (R == 0) {
                free(kk);
                free(vv);
                free(qq);
                return ST_EMPTY_CACHE; /* attention.cpp:24-26 */
            }
            /* for_each_retained in logical order, block_table.hpp:81-91 */
            int32_t n = 0;
            for (int32_t j = 0; j < e->num_pages[t]; ++j) {
                const int32_t page = e->block_table[(size_t)t * e->max_pages + j];
                const int32_t fill = (j == e->num_pages[t] - 1) ? e->newest_fill[t] : B;
                for (int32_t sl = 0; sl < fill; ++sl, ++n)
                    for (int32_t i = 0; i < d; ++i) {
                        kk[(size_t)n * d + i] = elem(page_row(e, page, 0, sl), i, e->dtype);
                        vv[(size_t)n * d + i] = elem(page_row(e, page, 1, sl), i, e->dtype);
                    }
            }
            for (int32_t g = 0; g < G; ++g) {
                const size_t qo = ((size_t)s * H * G + (size_t)h * G + g) * d;
                for (int32_t i = 0; i < d; ++i) qq[i] = elem(q, qo + i, e->dtype);
                peo_attend_dense(qq, kk, vv, (size_t)n, (size_t)d, out + qo);
            }
        }
    free(kk);
    free(vv);
    free(qq);
    return ST_OK;
}
