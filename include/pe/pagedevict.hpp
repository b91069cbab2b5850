// pagedevict.hpp — C++ façade: the reference's `pagedevict::` cache-manager
// API (/root/reference/proj/core/include/pagedevict/*.hpp) served by the
// B200 engine through the C-ABI in pe.h. Reference code that includes
// "pagedevict/<header>.hpp" compiles unchanged against include/pagedevict/
// (one-line forwarding headers) and links libpagedevict_b200.so.
//
// Where the state lives. Everything a PagePool owns — page bytes, token
// positions, every BlockTable's page list and counters, the LIFO free list —
// lives in HBM inside one pe_engine; a BlockTable is one table slot of that
// engine. Every mutation (append_token, free_page, clear, allocate,
// release, EvictionPolicy::decode_step, prefill_compress's scoring and
// selection, attend) is a device kernel; the façade only moves the caller's
// host vectors in and the results out, synchronously, and rethrows device
// status codes as the reference exception types (errors.hpp:12-88).
//
// Page objects returned by PagePool::page / BlockTable::page_at are host
// snapshots of a device page, refreshed on each call; mutating a snapshot
// (Page::write / evict / reset) does not write back.
//
// Differences from the reference:
//  * a pool's row width is fixed by the first token appended (or
//    PoolOptions::row_width): narrower tokens are zero-padded (norms,
//    scores and dot products are unchanged), wider ones throw LengthMismatch;
//  * unstructured eviction (BlockTable::evict_slot, the StreamingLLM /
//    InvKeyL2 / KeyDiff baselines) marks holes on the device; afterwards
//    the pool's batched GQA attention (pe_paged_decode_attention) refuses
//    the engine, attend() here handles holes;
//  * token positions must be < 2^31 (the device stores int32, D10);
//  * scores are computed from the token's bytes, not from KvVector's cached
//    key_norm/value_norm fields (identical for vectors built by make_kv).
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "pe.h"

namespace pagedevict {

// ---------------------------------------------------------------- errors
// The reference's exception hierarchy (errors.hpp:12-88); pe_status codes
// map 1:1 onto these classes (pe.h).
class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

#define PAGEDEVICT_ERROR_CLASS(Name, default_message)                 \
    class Name : public Error {                                       \
    public:                                                           \
        Name() : Error(default_message) {}                            \
        explicit Name(const std::string& what) : Error(what) {}       \
    };
PAGEDEVICT_ERROR_CLASS(PoolExhausted, "page pool exhausted")
PAGEDEVICT_ERROR_CLASS(IndexOutOfRange, "index out of range")
PAGEDEVICT_ERROR_CLASS(UnknownPosition, "unknown position")
PAGEDEVICT_ERROR_CLASS(Overflow, "overflow")
PAGEDEVICT_ERROR_CLASS(EmptyPage, "page has no occupied slots")
PAGEDEVICT_ERROR_CLASS(KTooLarge, "k too large")
PAGEDEVICT_ERROR_CLASS(NoEligiblePage, "no eligible page to rank")
PAGEDEVICT_ERROR_CLASS(BudgetInvalid, "budget invalid")
PAGEDEVICT_ERROR_CLASS(EmptyCache, "attention requires at least one retained token")
PAGEDEVICT_ERROR_CLASS(LengthMismatch, "length mismatch")
PAGEDEVICT_ERROR_CLASS(EmptyInput, "empty input")
PAGEDEVICT_ERROR_CLASS(IoError, "io error")
#undef PAGEDEVICT_ERROR_CLASS

// Throws the reference exception matching a non-OK engine status.
[[noreturn]] void throw_status(pe_status status, const std::string& context);

// ---------------------------------------------------------------- tokens
// kv_vector.hpp:15-48. A token's K and V rows for one table plus its absolute
// position; key_norm/value_norm are the cached L2 norms (double sum of
// squares in index order).
inline double l2_norm(std::span<const float> v) {
    double sum_sq = 0.0;
    for (const float x : v) sum_sq += static_cast<double>(x) * static_cast<double>(x);
    return std::sqrt(sum_sq);
}

struct KvVector {
    std::vector<float> key;
    std::vector<float> value;
    std::uint64_t position = 0;
    double key_norm = 0.0;
    double value_norm = 0.0;
};

inline KvVector make_kv(std::vector<float> key, std::vector<float> value, std::uint64_t position) {
    if (key.empty() || key.size() != value.size())
        throw LengthMismatch("key and value must have identical nonzero length");
    KvVector kv;
    kv.position = position;
    kv.key_norm = l2_norm(key);
    kv.value_norm = l2_norm(value);
    kv.key = std::move(key);
    kv.value = std::move(value);
    return kv;
}

using PageId = std::uint32_t;

// ---------------------------------------------------------------- Page
// page.hpp:21-71 as a host snapshot of one device page.
class Page {
public:
    Page() = default;
    Page(std::uint32_t slot_count, PageId physical_id) : slots_(slot_count), id_(physical_id) {}

    std::uint32_t slot_count() const { return static_cast<std::uint32_t>(slots_.size()); }
    std::uint32_t fill() const { return fill_; }
    std::uint32_t write_cursor() const { return cursor_; }
    bool write_full() const { return cursor_ == slots_.size(); }
    PageId physical_id() const { return id_; }
    bool occupied(std::uint32_t slot) const { return slot < slots_.size() && slots_[slot].has_value(); }
    const KvVector& at(std::uint32_t slot) const;

    void write(KvVector kv);
    bool evict(std::uint64_t position);
    void reset();

private:
    friend class PagePool;
    std::vector<std::optional<KvVector>> slots_;
    std::uint32_t cursor_ = 0;
    std::uint32_t fill_ = 0;
    PageId id_ = 0;
};

// ---------------------------------------------------------------- PagePool
// Engine sizing beyond the reference's (capacity, page_size).
struct PoolOptions {
    std::uint32_t row_width = 0;            // floats per K/V row; 0 = the first appended token's width
    std::uint32_t max_tables = 256;         // BlockTables that may be alive at once on this pool
    std::uint32_t max_pages_per_table = 0;  // 0 = the whole pool (bounded by a 256 MB block-table budget)
    int device = 0;                          // CUDA ordinal
    pe_dtype dtype = PE_DTYPE_F32;          // storage type of the K/V rows (bf16: values are rounded)
};

// page_pool.hpp:19-42: fixed pool of pages with a LIFO free list, safe to
// share between threads (one mutex serialises the device calls).
class PagePool {
public:
    PagePool(std::size_t capacity, std::uint32_t page_size, PoolOptions options = {});
    ~PagePool();
    PagePool(const PagePool&) = delete;
    PagePool& operator=(const PagePool&) = delete;

    PageId allocate();
    void release(PageId id);

    Page& page(PageId id);
    const Page& page(PageId id) const;

    std::uint32_t page_size() const;
    std::size_t capacity() const;
    std::size_t free_count() const;
    std::size_t allocated() const;

    // --- extensions: the engine behind the pool (created on first use)
    pe_engine* engine() const;
    std::uint32_t row_width() const;  // 0 until fixed

    struct Impl;
    Impl& impl() const { return *impl_; }  // façade internals

private:
    std::unique_ptr<Impl> impl_;
};

std::uint64_t memory_bytes(std::uint64_t seq_len, std::uint64_t layer_count, std::uint64_t head_count,
                           std::uint64_t head_dim, std::uint64_t bytes_per_scalar);

// ---------------------------------------------------------------- BlockTable
struct AppendOutcome {
    bool page_opened = false;
};

// block_table.hpp:21-102: one table slot of the pool's engine.
class BlockTable {
public:
    explicit BlockTable(PagePool& pool);
    ~BlockTable();
    BlockTable(const BlockTable&) = delete;
    BlockTable& operator=(const BlockTable&) = delete;
    BlockTable(BlockTable&& other) noexcept;
    BlockTable& operator=(BlockTable&& other) noexcept;

    AppendOutcome append_token(KvVector kv);
    void free_page(std::size_t logical_index);
    void evict_slot(std::uint64_t position);

    std::size_t page_count() const;
    std::size_t retained_len() const;
    bool empty() const { return retained_len() == 0; }
    const Page& page_at(std::size_t logical_index) const;
    PageId physical_id_at(std::size_t logical_index) const;

    double fragmentation_ratio() const;
    double fragmentation_ratio_excluding_newest() const;
    std::vector<std::uint64_t> retained_positions() const;

    template <typename Fn>
    void for_each_retained(Fn&& fn) const {
        const std::size_t n = page_count();
        for (std::size_t j = 0; j < n; ++j) {
            const Page& pg = page_at(j);
            for (std::uint32_t s = 0; s < pg.write_cursor(); ++s)
                if (pg.occupied(s)) fn(pg.at(s));
        }
    }

    void clear();
    PagePool& pool() { return *pool_; }

    // --- extensions
    std::int32_t table_id() const { return slot_; }  // engine table slot (-1 when moved-from)

private:
    friend class PagePool;
    friend class EvictionPolicy;
    struct View {                 // last device readback
        bool valid = false;
        std::vector<std::int32_t> pages;
        std::int32_t newest_fill = 0;
        std::int32_t retained = 0;
    };
    const View& view() const;
    void invalidate() const { view_.valid = false; }
    void release_slot() noexcept;

    PagePool* pool_ = nullptr;
    std::int32_t slot_ = -1;
    mutable View view_;
};

// ---------------------------------------------------------------- importance
// importance.hpp:17-48. Pure functions over caller-held values.
inline constexpr double kNormEpsilon = 1e-12;

struct TokenScore {
    std::uint64_t position = 0;
    double score = 0.0;
};

struct PageScore {
    std::size_t logical_index = 0;
    double score = 0.0;
    std::uint32_t token_count = 0;
};

double token_importance(const KvVector& kv);
TokenScore token_score(const KvVector& kv);
PageScore page_score(const Page& page, std::size_t logical_index);
std::vector<PageScore> score_pages(const BlockTable& table);
std::vector<std::uint64_t> rank_tokens(std::span<const TokenScore> scores, std::size_t k);
std::size_t rank_pages(std::span<const PageScore> scores);

// ---------------------------------------------------------------- policy
// policy.hpp:17-122.
enum class PolicyKind { PagedEviction, StreamingLlm, InvKeyL2, KeyDiff, FullCache };

std::string_view to_string(PolicyKind kind);
std::optional<PolicyKind> parse_policy_kind(std::string_view name);

struct PolicyConfig {
    std::size_t cache_budget = 256;
    std::uint32_t page_size = 16;
    std::size_t sink_count = 4;
    PolicyKind kind = PolicyKind::PagedEviction;
    void validate() const;
};

struct EvictionDecision {
    enum class Kind { None, Tokens, Page };

    Kind kind = Kind::None;
    std::vector<std::uint64_t> positions;
    std::size_t logical_index = 0;
    std::int64_t trigger_step = 0;

    static EvictionDecision none(std::int64_t step) {
        EvictionDecision d;
        d.trigger_step = step;
        return d;
    }
    static EvictionDecision tokens(std::vector<std::uint64_t> evicted, std::int64_t step) {
        EvictionDecision d;
        d.kind = Kind::Tokens;
        d.positions = std::move(evicted);
        d.trigger_step = step;
        return d;
    }
    static EvictionDecision page(std::size_t index, std::int64_t step) {
        EvictionDecision d;
        d.kind = Kind::Page;
        d.logical_index = index;
        d.trigger_step = step;
        return d;
    }
    std::uint64_t tokens_removed(std::uint32_t page_size) const {
        if (kind == Kind::Tokens) return positions.size();
        if (kind == Kind::Page) return page_size;
        return 0;
    }
};

struct PrefillResult {
    std::vector<KvVector> retained;
    EvictionDecision decision;
};

// The plugin point (policy.hpp:95-120): prefill_compress validates and
// short-circuits, then calls compress(); decode_step appends the token and
// calls evict(). Subclasses may be written against the same protected hooks.
class EvictionPolicy {
public:
    explicit EvictionPolicy(PolicyConfig config) : config_(config) { config_.validate(); }
    virtual ~EvictionPolicy() = default;

    const PolicyConfig& config() const { return config_; }
    PolicyKind kind() const { return config_.kind; }

    PrefillResult prefill_compress(std::vector<KvVector> tokens) const;
    EvictionDecision decode_step(BlockTable& table, KvVector kv, std::int64_t step);

protected:
    virtual PrefillResult compress(std::vector<KvVector> tokens) const = 0;
    virtual EvictionDecision evict(BlockTable& table, std::uint64_t newest_position, std::int64_t step) = 0;

    // device helpers for subclasses
    static std::vector<std::size_t> device_select_survivors(const std::vector<KvVector>& tokens,
                                                            const PolicyConfig& config);
    static std::int64_t device_paged_evict(BlockTable& table, std::size_t cache_budget);
    // unstructured eviction of one token by a pe_token_rule; -1 = none
    static std::int64_t device_token_evict(BlockTable& table, pe_token_rule rule, std::int64_t arg,
                                           std::size_t cache_budget, std::uint64_t newest_position);
    // score-based baseline prefill: flags of the k lowest-scoring prompt tokens
    static std::vector<char> device_prompt_select(const std::vector<KvVector>& tokens, pe_token_rule rule,
                                                  std::size_t k);

    PolicyConfig config_;
};

std::unique_ptr<EvictionPolicy> make_policy(PolicyConfig config);

// ---------------------------------------------------------------- attention
// attention.hpp:14-38.
struct AttentionInputs {
    std::span<const float> query;
    const BlockTable* table = nullptr;
    std::uint32_t head_count = 0;
    std::uint32_t head_dim = 0;
};

struct AttentionDetail {
    std::vector<float> output;
    std::vector<double> weight_sums;
};

std::vector<float> attend(const AttentionInputs& inputs);
AttentionDetail attend_detailed(const AttentionInputs& inputs);
double output_deviation(std::span<const float> a, std::span<const float> b);

// ------------------------------------------------------------------ metrics
// metrics.hpp:16-80 and schemas/{steplog.jsonl,metrics.csv}.md: the per-step
// log record, the per-run CSV record, their emitters and the per-policy
// summary. Byte-identical output to the reference for the same records
// (tests/cpp/scenario_trace.cpp runs both builds). Device-side capture of
// the engine-owned StepRecord fields: pe_step_log_capture (pe.h) and
// step_records() below.
struct StepRecord {
    std::uint32_t run = 0;
    std::uint32_t sequence = 0;
    std::uint32_t layer = 0;
    std::int64_t step = 0;  // 1-based
    std::size_t retained_len = 0;
    EvictionDecision decision;
    double fragmentation = 0.0;
    double fragmentation_excl_newest = 0.0;
    double deviation = 0.0;  // NaN: no FullCache shadow
};

struct MetricsRecord {
    std::string policy;
    std::uint64_t cache_budget = 0;
    std::uint32_t page_size = 0;
    std::uint64_t prefill_len = 0;
    std::uint64_t decode_steps = 0;
    std::uint64_t batch = 0;
    std::uint64_t layer_count = 0;
    std::uint64_t seed = 0;
    std::uint64_t prefill_evicted = 0;
    std::uint64_t evictions_total = 0;
    std::uint64_t page_evictions = 0;
    std::uint64_t token_evictions = 0;
    std::uint64_t block_table_updates = 0;
    double mean_fragmentation = 0.0;
    double max_fragmentation = 0.0;
    double max_fragmentation_excl_newest = 0.0;
    double mean_deviation = 0.0;
    double p95_deviation = 0.0;
    std::uint64_t retained_bytes = 0;
    std::uint64_t prefill_wall_ns = 0;
    std::uint64_t decode_wall_ns = 0;
};

std::string emit_csv(std::span<const MetricsRecord> records);
std::string emit_jsonl(std::span<const StepRecord> steps);

struct SummaryRow {
    std::string policy;
    std::uint64_t runs = 0;
    std::uint64_t evictions_total = 0;
    std::uint64_t block_table_updates = 0;
    double cadence_ratio = 0.0;  // NaN without a PagedEviction record
    double max_fragmentation_excl_newest = 0.0;
    double mean_deviation = 0.0;
};

std::vector<SummaryRow> summarize(std::span<const MetricsRecord> records);
std::string format_summary(std::span<const SummaryRow> rows);

// StepRecords (decision, retained length, both fragmentation ratios) for the
// tables of one pe_step_log_capture, in the capture's table order; page
// decisions carry trigger_step = step. `page_size` is the engine's B.
std::vector<StepRecord> step_records(std::span<const pe_step_entry> entries, std::uint32_t page_size,
                                     std::int64_t step, std::uint32_t run = 0);

}  // namespace pagedevict

// Integration self-test (one PagedEviction table on the device, invariants
// checked); returns 0 and a summary in msg, or 1 and the error.
extern "C" int pagedevict_facade_selftest(char* msg, int cap);
