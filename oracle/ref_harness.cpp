// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT PATH.
//
// C-ABI harness over the UNMODIFIED reference library (pagedevict::core,
// compiled from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libpagedevict_ref.so). It drives the reference's own objects
// directly — PagePool, BlockTable, make_policy(PolicyConfig), attend — one
// BlockTable + EvictionPolicy per engine table, in the canonical batched
// order the device engine documents: the Python test driver
// issues the per-table calls in that order.
//
// Uses: (1) pin the C restatement in oracle/pe_oracle.c against the real
// reference; (2) parity checks of the CUDA engine; (3) the CPU baseline /
// `bench.py --impl reference` arm.  Only tests/, __graft_entry__.smoke() and
// bench.py's reference/cpu_baseline legs may load this library.
//
// Free-list observability: PagePool::free_list_ is private
// (proj/core/include/pagedevict/page_pool.hpp:40). The session keeps a mirror
// stack, initialised [cap-1..0] like page_pool.cpp:18-21, popped on every
// append that opened a page (checked against physical_id_at(last)) and pushed
// with the victim's physical id on every Page decision (captured before the
// step). `ref_drain_free_list` drains the real pool with allocate() and
// compares it against the mirror.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "pagedevict/attention.hpp"
#include "pagedevict/block_table.hpp"
#include "pagedevict/errors.hpp"
#include "pagedevict/importance.hpp"
#include "pagedevict/kv_vector.hpp"
#include "pagedevict/page_pool.hpp"
#include "pagedevict/policy.hpp"
#include "pagedevict/rng.hpp"

using namespace pagedevict;

namespace {

// Status codes: same numbering as include/pe.h (pe_status).
enum : int {
    RS_OK = 0,
    RS_ERROR = 1,
    RS_POOL_EXHAUSTED = 2,
    RS_INDEX_OUT_OF_RANGE = 3,
    RS_UNKNOWN_POSITION = 4,
    RS_OVERFLOW = 5,
    RS_EMPTY_PAGE = 6,
    RS_K_TOO_LARGE = 7,
    RS_NO_ELIGIBLE_PAGE = 8,
    RS_BUDGET_INVALID = 9,
    RS_EMPTY_CACHE = 10,
    RS_LENGTH_MISMATCH = 11,
    RS_EMPTY_INPUT = 12,
    RS_IO_ERROR = 13,
    RS_MIRROR_MISMATCH = 100,
};

thread_local std::string g_last_error;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return RS_OK;
    } catch (const PoolExhausted& e) {
        g_last_error = e.what();
        return RS_POOL_EXHAUSTED;
    } catch (const IndexOutOfRange& e) {
        g_last_error = e.what();
        return RS_INDEX_OUT_OF_RANGE;
    } catch (const UnknownPosition& e) {
        g_last_error = e.what();
        return RS_UNKNOWN_POSITION;
    } catch (const Overflow& e) {
        g_last_error = e.what();
        return RS_OVERFLOW;
    } catch (const EmptyPage& e) {
        g_last_error = e.what();
        return RS_EMPTY_PAGE;
    } catch (const KTooLarge& e) {
        g_last_error = e.what();
        return RS_K_TOO_LARGE;
    } catch (const NoEligiblePage& e) {
        g_last_error = e.what();
        return RS_NO_ELIGIBLE_PAGE;
    } catch (const BudgetInvalid& e) {
        g_last_error = e.what();
        return RS_BUDGET_INVALID;
    } catch (const EmptyCache& e) {
        g_last_error = e.what();
        return RS_EMPTY_CACHE;
    } catch (const LengthMismatch& e) {
        g_last_error = e.what();
        return RS_LENGTH_MISMATCH;
    } catch (const EmptyInput& e) {
        g_last_error = e.what();
        return RS_EMPTY_INPUT;
    } catch (const IoError& e) {
        g_last_error = e.what();
        return RS_IO_ERROR;
    } catch (const Error& e) {
        g_last_error = e.what();
        return RS_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return RS_ERROR;
    }
}

PolicyKind kind_from_int(int k) {
    switch (k) {
    case 0: return PolicyKind::PagedEviction;
    case 1: return PolicyKind::StreamingLlm;
    case 2: return PolicyKind::InvKeyL2;
    case 3: return PolicyKind::KeyDiff;
    case 4: return PolicyKind::FullCache;
    default: throw Error("unknown policy kind " + std::to_string(k));
    }
}

struct Session {
    PagePool pool;
    std::vector<BlockTable> tables;
    std::vector<std::unique_ptr<EvictionPolicy>> policies;
    std::vector<PageId> mirror;  // free-list mirror, back = top of stack
    std::uint32_t width = 0;

    Session(std::size_t cap, std::uint32_t page_size, const PolicyConfig& cfg, std::size_t n)
        : pool(cap, page_size) {
        tables.reserve(n);
        policies.reserve(n);
        for (std::size_t i = 0; i < n; ++i) {
            tables.emplace_back(pool);
            policies.push_back(make_policy(cfg));
        }
        for (std::size_t i = cap; i > 0; --i) {
            mirror.push_back(static_cast<PageId>(i - 1));
        }
    }

    // Records a pop on the mirror after an append that opened a page.
    void mirror_pop(const BlockTable& table) {
        if (mirror.empty()) {
            throw Error("free-list mirror underflow");
        }
        const PageId expect = mirror.back();
        mirror.pop_back();
        const PageId got = table.physical_id_at(table.page_count() - 1);
        if (got != expect) {
            throw Error("free-list mirror mismatch on pop: pool gave " + std::to_string(got) +
                        ", mirror expected " + std::to_string(expect));
        }
    }
};

KvVector kv_from(const float* k, const float* v, std::size_t w, std::uint64_t pos) {
    return make_kv(std::vector<float>(k, k + w), std::vector<float>(v, v + w), pos);
}

}  // namespace

// The policies' protected evict (policy.hpp:113-117), reached through a
// member pointer formed in a derived class: the two-phase decode of the
// engine's canonical batched order (all of a step's appends, then all
// evictions) drives append_token and evict separately.
struct EvictAccess : EvictionPolicy {
    using Fn = EvictionDecision (EvictionPolicy::*)(BlockTable&, std::uint64_t, std::int64_t);
    static Fn fn() { return &EvictAccess::evict; }
};

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

// ---------------------------------------------------------------- free functions
// l2_norm: proj/core/include/pagedevict/kv_vector.hpp:15-21
double ref_l2_norm(const float* x, std::size_t n) {
    return l2_norm(std::span<const float>(x, n));
}

// token_importance on a make_kv record: importance.cpp:11-13, kv_vector.hpp:36-48
int ref_token_importance(const float* k, const float* v, std::size_t w, double* out) {
    return guarded([&] { *out = token_importance(kv_from(k, v, w, 0)); });
}

// rank_tokens: importance.cpp:41-60
int ref_rank_tokens(const std::uint64_t* positions, const double* scores, std::size_t n,
                    std::size_t k, std::uint64_t* out) {
    return guarded([&] {
        std::vector<TokenScore> s(n);
        for (std::size_t i = 0; i < n; ++i) {
            s[i] = TokenScore{positions[i], scores[i]};
        }
        auto sel = rank_tokens(s, k);
        std::copy(sel.begin(), sel.end(), out);
    });
}

// rank_pages: importance.cpp:62-75 (logical index = array index)
int ref_rank_pages(const double* scores, std::size_t n, std::size_t* out) {
    return guarded([&] {
        std::vector<PageScore> s(n);
        for (std::size_t i = 0; i < n; ++i) {
            s[i] = PageScore{i, scores[i], 1};
        }
        *out = rank_pages(s);
    });
}

// PolicyConfig::validate: policy.cpp:38-52
int ref_validate_config(std::size_t budget, std::uint32_t page_size, std::size_t sinks, int kind) {
    return guarded([&] {
        PolicyConfig c;
        c.cache_budget = budget;
        c.page_size = page_size;
        c.sink_count = sinks;
        c.kind = kind_from_int(kind);
        c.validate();
    });
}

// memory_bytes: page_pool.cpp:50-61
int ref_memory_bytes(std::uint64_t seq_len, std::uint64_t layers, std::uint64_t heads,
                     std::uint64_t dim, std::uint64_t bytes, std::uint64_t* out) {
    return guarded([&] { *out = memory_bytes(seq_len, layers, heads, dim, bytes); });
}

// attend over a contiguous token list packed into a private pool (MHA with
// `heads` heads of `dim`): attention.cpp:15-99
int ref_attend_dense(const float* keys, const float* values, std::size_t n_tokens,
                     const float* query, std::uint32_t heads, std::uint32_t dim,
                     std::uint32_t page_size, float* out) {
    return guarded([&] {
        const std::size_t w = static_cast<std::size_t>(heads) * dim;
        PagePool pool(n_tokens / page_size + 2, page_size);
        BlockTable table(pool);
        for (std::size_t i = 0; i < n_tokens; ++i) {
            table.append_token(kv_from(keys + i * w, values + i * w, w, i));
        }
        auto o = attend({std::span<const float>(query, w), &table, heads, dim});
        std::copy(o.begin(), o.end(), out);
    });
}

int ref_output_deviation(const float* a, std::size_t na, const float* b, std::size_t nb,
                         double* out) {
    return guarded([&] {
        *out = output_deviation(std::span<const float>(a, na), std::span<const float>(b, nb));
    });
}

// ---------------------------------------------------------------- sessions
void* ref_session_create(std::size_t capacity, std::uint32_t page_size, std::size_t budget,
                         int kind, std::size_t n_tables, std::uint32_t width, int* status) {
    Session* s = nullptr;
    *status = guarded([&] {
        PolicyConfig c;
        c.cache_budget = budget;
        c.page_size = page_size;
        c.kind = kind_from_int(kind);
        c.validate();
        s = new Session(capacity, page_size, c, n_tables);
        s->width = width;
    });
    return s;
}

void ref_session_destroy(void* h) { delete static_cast<Session*>(h); }

// Prefill one table: EvictionPolicy::prefill_compress (policy.cpp:54-63) then
// append every survivor in order (simulator.cpp:181-186). `evicted` receives
// the Tokens decision's positions (sorted) — caller sizes it >= L.
int ref_prefill(void* h, std::size_t t, const float* k, const float* v, std::size_t L,
                const std::uint64_t* positions, std::uint64_t* evicted, std::size_t* n_evicted) {
    auto* s = static_cast<Session*>(h);
    return guarded([&] {
        const std::size_t w = s->width;
        std::vector<KvVector> tokens;
        tokens.reserve(L);
        for (std::size_t i = 0; i < L; ++i) {
            tokens.push_back(kv_from(k + i * w, v + i * w, w, positions[i]));
        }
        auto result = s->policies.at(t)->prefill_compress(std::move(tokens));
        *n_evicted = result.decision.positions.size();
        std::copy(result.decision.positions.begin(), result.decision.positions.end(), evicted);
        BlockTable& table = s->tables.at(t);
        for (auto& kv : result.retained) {
            if (table.append_token(std::move(kv)).page_opened) {
                s->mirror_pop(table);
            }
        }
    });
}

// One EvictionPolicy::decode_step (policy.cpp:65-70). Outputs the decision
// kind (0 None, 1 Tokens, 2 Page) and its logical index (Page).
int ref_decode_step(void* h, std::size_t t, const float* k, const float* v,
                    std::uint64_t position, std::int64_t step, int* kind,
                    std::int64_t* logical_index) {
    auto* s = static_cast<Session*>(h);
    return guarded([&] {
        BlockTable& table = s->tables.at(t);
        std::vector<PageId> before(table.page_count());
        for (std::size_t j = 0; j < before.size(); ++j) {
            before[j] = table.physical_id_at(j);
        }
        const bool will_open = table.page_count() == 0 ||
                               table.page_at(table.page_count() - 1).write_full();
        auto d = s->policies.at(t)->decode_step(table, kv_from(k, v, s->width, position), step);
        if (will_open) {
            // The append opened a page. If the same step then evicted, the new
            // page sits at the end of `before` + [new].
            PageId opened;
            if (d.kind == EvictionDecision::Kind::Page &&
                d.logical_index == before.size()) {
                opened = PageId(-1);  // evicted the page it just opened
            } else {
                opened = table.physical_id_at(table.page_count() - 1);
            }
            if (s->mirror.empty()) {
                throw Error("free-list mirror underflow");
            }
            const PageId expect = s->mirror.back();
            s->mirror.pop_back();
            if (opened != PageId(-1) && opened != expect) {
                throw Error("free-list mirror mismatch on decode pop");
            }
            before.push_back(expect);
        }
        *kind = static_cast<int>(d.kind);
        *logical_index = -1;
        if (d.kind == EvictionDecision::Kind::Page) {
            *logical_index = static_cast<std::int64_t>(d.logical_index);
            s->mirror.push_back(before.at(d.logical_index));
        }
    });
}

// BlockTable::append_token (block_table.cpp:10-19) alone: phase 1 of a
// two-phase decode step (no free-list mirror bookkeeping).
int ref_append_token(void* h, std::size_t t, const float* k, const float* v, std::uint64_t position) {
    auto* s = static_cast<Session*>(h);
    return guarded([&] { s->tables.at(t).append_token(kv_from(k, v, s->width, position)); });
}

// The policy's evict after the append (phase 2): kind 0 None, 1 Tokens, 2
// Page; *victim = the evicted position (Tokens, one per step for the
// baselines) or logical page (Page), else -1.
int ref_policy_evict(void* h, std::size_t t, std::uint64_t newest, std::int64_t step, int* kind,
                     std::int64_t* victim) {
    auto* s = static_cast<Session*>(h);
    return guarded([&] {
        EvictionPolicy& p = *s->policies.at(t);
        const EvictionDecision d = (p.*EvictAccess::fn())(s->tables.at(t), newest, step);
        *kind = static_cast<int>(d.kind);
        *victim = -1;
        if (d.kind == EvictionDecision::Kind::Tokens && !d.positions.empty())
            *victim = static_cast<std::int64_t>(d.positions.front());
        if (d.kind == EvictionDecision::Kind::Page) *victim = static_cast<std::int64_t>(d.logical_index);
    });
}

std::size_t ref_page_count(void* h, std::size_t t) {
    return static_cast<Session*>(h)->tables.at(t).page_count();
}
std::size_t ref_retained_len(void* h, std::size_t t) {
    return static_cast<Session*>(h)->tables.at(t).retained_len();
}
std::size_t ref_free_count(void* h) { return static_cast<Session*>(h)->pool.free_count(); }
// BlockTable::fragmentation_ratio / _excluding_newest (step-log fields)
void ref_fragmentation(void* h, std::size_t t, double* out2) {
    const auto& table = static_cast<Session*>(h)->tables.at(t);
    out2[0] = table.fragmentation_ratio();
    out2[1] = table.fragmentation_ratio_excluding_newest();
}

// Logical-order readback of one table: physical ids [page_count], per page
// fill [page_count], and per retained token (logical order, holes skipped)
// position, key and value (w floats each).
int ref_read_table(void* h, std::size_t t, std::uint32_t* phys, std::uint32_t* fills,
                   std::uint64_t* positions, float* keys, float* values) {
    auto* s = static_cast<Session*>(h);
    return guarded([&] {
        const BlockTable& table = s->tables.at(t);
        for (std::size_t j = 0; j < table.page_count(); ++j) {
            phys[j] = table.physical_id_at(j);
            fills[j] = table.page_at(j).fill();
        }
        std::size_t i = 0;
        const std::size_t w = s->width;
        table.for_each_retained([&](const KvVector& kv) {
            positions[i] = kv.position;
            if (keys) std::memcpy(keys + i * w, kv.key.data(), w * sizeof(float));
            if (values) std::memcpy(values + i * w, kv.value.data(), w * sizeof(float));
            ++i;
        });
    });
}

// Mirror of the free list, bottom..top (top = next id allocate() returns).
std::size_t ref_mirror_free_list(void* h, std::uint32_t* out) {
    auto* s = static_cast<Session*>(h);
    std::copy(s->mirror.begin(), s->mirror.end(), out);
    return s->mirror.size();
}

// Drains the real pool with allocate() (page_pool.cpp:24-33) and checks the
// order against the mirror (check_mirror). Destroys the session's usefulness
// afterwards.
int ref_drain_free_list(void* h, std::uint32_t* out, std::size_t* n, int check_mirror) {
    auto* s = static_cast<Session*>(h);
    int st = guarded([&] {
        std::size_t i = 0;
        while (s->pool.free_count() > 0) {
            out[i++] = s->pool.allocate();
        }
        *n = i;
    });
    if (st != RS_OK || !check_mirror) return st;  // (the two-phase calls keep no mirror)
    // allocate() pops from the back: out[i] must equal mirror[size-1-i].
    if (*n != s->mirror.size()) return RS_MIRROR_MISMATCH;
    for (std::size_t i = 0; i < *n; ++i) {
        if (out[i] != s->mirror[s->mirror.size() - 1 - i]) return RS_MIRROR_MISMATCH;
    }
    return RS_OK;
}

// attend() on one table with head_count = heads (GQA: caller passes one
// query head at a time with heads=1, dim=w). attention.cpp:97-99
int ref_attend_table(void* h, std::size_t t, const float* query, std::uint32_t heads,
                     std::uint32_t dim, float* out) {
    auto* s = static_cast<Session*>(h);
    return guarded([&] {
        const std::size_t w = static_cast<std::size_t>(heads) * dim;
        auto o = attend({std::span<const float>(query, w), &s->tables.at(t), heads, dim});
        std::copy(o.begin(), o.end(), out);
    });
}

// ---------------------------------------------------------------- CPU baseline timing
// Each worker thread owns a PagePool and a contiguous slice of tables
// (timing runs need no physical-id parity). Inputs are drawn with the
// reference's own GaussianStream (rng.hpp:24-46) before the clock starts.

}  // extern "C"

namespace {

struct Worker {
    std::unique_ptr<PagePool> pool;
    std::vector<BlockTable> tables;
    std::vector<std::unique_ptr<EvictionPolicy>> policies;
    std::vector<std::uint64_t> next_pos;
};

template <typename Fn>
double timed_parallel(std::size_t n_threads, Fn&& fn) {
    std::vector<std::thread> th;
    std::atomic<std::size_t> ready{0};
    std::atomic<bool> go{false};
    std::vector<double> secs(n_threads, 0.0);
    for (std::size_t i = 0; i < n_threads; ++i) {
        th.emplace_back([&, i] {
            ++ready;
            while (!go.load()) {
            }
            fn(i);
        });
    }
    while (ready.load() < n_threads) {
    }
    const auto t0 = std::chrono::steady_clock::now();
    go = true;
    for (auto& x : th) x.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

// Decode eviction cycles: `n_tables` tables of width w, each set up with an
// identity prefill of `budget` tokens (untimed), then timed: `cycles` × B
// decode steps per table (make_kv + EvictionPolicy::decode_step), so every
// table triggers exactly one PagedEviction page eviction per cycle
// (policy.cpp:143-155). Returns seconds; *evictions = Page decisions seen.
int ref_bench_decode_cycles(std::size_t n_tables, std::size_t budget, std::uint32_t page_size,
                            std::uint32_t w, std::size_t n_threads, std::size_t warmup_cycles,
                            std::size_t cycles, std::uint64_t seed, double* seconds,
                            std::uint64_t* evictions) {
    return guarded([&] {
        n_threads = std::max<std::size_t>(1, std::min(n_threads, n_tables));
        PolicyConfig cfg;
        cfg.cache_budget = budget;
        cfg.page_size = page_size;
        cfg.kind = PolicyKind::PagedEviction;
        std::vector<Worker> workers(n_threads);
        // Pre-drawn decode inputs: one stream of (warmup+timed)*B tokens per
        // thread, re-used across that thread's tables.
        const std::size_t warm_steps = warmup_cycles * page_size;
        const std::size_t steps = (warmup_cycles + cycles) * page_size;
        std::vector<std::vector<float>> dk(n_threads), dv(n_threads);
        std::vector<std::atomic<std::uint64_t>> ev(n_threads);
        std::vector<std::thread> setup;
        for (std::size_t ti = 0; ti < n_threads; ++ti) {
            setup.emplace_back([&, ti] {
                const std::size_t lo = n_tables * ti / n_threads;
                const std::size_t hi = n_tables * (ti + 1) / n_threads;
                Worker& wk = workers[ti];
                const std::size_t pages = (hi - lo) * (budget / page_size + 2);
                wk.pool = std::make_unique<PagePool>(pages, page_size);
                GaussianStream rng(derive_seed(seed, ti));
                for (std::size_t t = lo; t < hi; ++t) {
                    wk.tables.emplace_back(*wk.pool);
                    wk.policies.push_back(make_policy(cfg));
                    std::vector<KvVector> prompt;
                    prompt.reserve(budget);
                    for (std::size_t i = 0; i < budget; ++i) {
                        prompt.push_back(make_kv(rng.draw(w), rng.draw(w), i));
                    }
                    auto r = wk.policies.back()->prefill_compress(std::move(prompt));
                    for (auto& kv : r.retained) wk.tables.back().append_token(std::move(kv));
                    wk.next_pos.push_back(budget);
                }
                dk[ti] = rng.draw(steps * w);
                dv[ti] = rng.draw(steps * w);
                ev[ti] = 0;
            });
        }
        for (auto& x : setup) x.join();
        auto run_steps = [&](std::size_t ti, std::size_t s0, std::size_t s1) {
            Worker& wk = workers[ti];
            std::uint64_t e = 0;
            for (std::size_t st = s0; st < s1; ++st) {
                const float* kr = dk[ti].data() + st * w;
                const float* vr = dv[ti].data() + st * w;
                for (std::size_t j = 0; j < wk.tables.size(); ++j) {
                    auto kv = make_kv(std::vector<float>(kr, kr + w),
                                      std::vector<float>(vr, vr + w), wk.next_pos[j]++);
                    auto d = wk.policies[j]->decode_step(wk.tables[j], std::move(kv),
                                                         static_cast<std::int64_t>(st + 1));
                    e += d.kind == EvictionDecision::Kind::Page;
                }
            }
            return e;
        };
        if (warm_steps > 0) {  // untimed warm-up cycles
            std::vector<std::thread> warm;
            for (std::size_t ti = 0; ti < n_threads; ++ti)
                warm.emplace_back([&, ti] { run_steps(ti, 0, warm_steps); });
            for (auto& x : warm) x.join();
        }
        *seconds = timed_parallel(n_threads, [&](std::size_t ti) { ev[ti] = run_steps(ti, warm_steps, steps); });
        std::uint64_t tot = 0;
        for (auto& x : ev) tot += x.load();
        *evictions = tot;
    });
}

// Prefill prune+pack: `n_tables` tables of L tokens of width w each
// (inputs drawn untimed), timed: make_kv (norms) + prefill_compress +
// append of every survivor (simulator.cpp:170-187 minus the toy projection).
int ref_bench_prefill(std::size_t n_tables, std::size_t L, std::size_t budget,
                      std::uint32_t page_size, std::uint32_t w, std::size_t n_threads,
                      std::uint64_t seed, double* seconds) {
    return guarded([&] {
        n_threads = std::max<std::size_t>(1, std::min(n_threads, n_tables));
        PolicyConfig cfg;
        cfg.cache_budget = budget;
        cfg.page_size = page_size;
        cfg.kind = PolicyKind::PagedEviction;
        std::vector<std::vector<float>> raw_k(n_threads), raw_v(n_threads);
        std::vector<std::thread> setup;
        for (std::size_t ti = 0; ti < n_threads; ++ti) {
            setup.emplace_back([&, ti] {
                GaussianStream rng(derive_seed(seed, 1000 + ti));
                raw_k[ti] = rng.draw(L * w);
                raw_v[ti] = rng.draw(L * w);
            });
        }
        for (auto& x : setup) x.join();
        *seconds = timed_parallel(n_threads, [&](std::size_t ti) {
            const std::size_t lo = n_tables * ti / n_threads;
            const std::size_t hi = n_tables * (ti + 1) / n_threads;
            PagePool pool((hi - lo) * (std::min(L, budget) / page_size + 2), page_size);
            std::vector<BlockTable> tables;
            tables.reserve(hi - lo);
            auto policy = make_policy(cfg);
            for (std::size_t t = lo; t < hi; ++t) {
                std::vector<KvVector> tokens;
                tokens.reserve(L);
                for (std::size_t i = 0; i < L; ++i) {
                    const float* kr = raw_k[ti].data() + i * w;
                    const float* vr = raw_v[ti].data() + i * w;
                    tokens.push_back(make_kv(std::vector<float>(kr, kr + w),
                                             std::vector<float>(vr, vr + w), i));
                }
                auto r = policy->prefill_compress(std::move(tokens));
                tables.emplace_back(pool);
                for (auto& kv : r.retained) tables.back().append_token(std::move(kv));
            }
        });
    });
}

// Paged attention: n_tables tables of R tokens (width d), G query heads
// each, attend() per query head (head_count = 1). Timed: one attend per
// (table, q-head).
int ref_bench_attend(std::size_t n_tables, std::size_t R, std::uint32_t page_size,
                     std::uint32_t d, std::uint32_t G, std::size_t n_threads,
                     std::uint64_t seed, double* seconds) {
    return guarded([&] {
        n_threads = std::max<std::size_t>(1, std::min(n_threads, n_tables));
        std::vector<std::unique_ptr<PagePool>> pools(n_threads);
        std::vector<std::vector<BlockTable>> tabs(n_threads);
        std::vector<std::vector<float>> qs(n_threads);
        std::vector<std::thread> setup;
        for (std::size_t ti = 0; ti < n_threads; ++ti) {
            setup.emplace_back([&, ti] {
                const std::size_t lo = n_tables * ti / n_threads;
                const std::size_t hi = n_tables * (ti + 1) / n_threads;
                GaussianStream rng(derive_seed(seed, 2000 + ti));
                pools[ti] = std::make_unique<PagePool>((hi - lo) * (R / page_size + 2), page_size);
                tabs[ti].reserve(hi - lo);
                for (std::size_t t = lo; t < hi; ++t) {
                    tabs[ti].emplace_back(*pools[ti]);
                    for (std::size_t i = 0; i < R; ++i) {
                        tabs[ti].back().append_token(make_kv(rng.draw(d), rng.draw(d), i));
                    }
                }
                qs[ti] = rng.draw(static_cast<std::size_t>(G) * d);
            });
        }
        for (auto& x : setup) x.join();
        *seconds = timed_parallel(n_threads, [&](std::size_t ti) {
            volatile float sink = 0.0f;
            for (auto& table : tabs[ti]) {
                for (std::uint32_t g = 0; g < G; ++g) {
                    auto o = attend({std::span<const float>(qs[ti].data() + g * d, d), &table, 1, d});
                    sink = sink + o[0];
                }
            }
        });
    });
}

}  // extern "C"
