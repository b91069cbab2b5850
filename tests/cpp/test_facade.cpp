// Façade conformance tests (test infrastructure): the C++ pagedevict::
// API (include/pe/pagedevict.hpp) running on the B200 engine, checked
// against the plain-C oracle (oracle/pe_oracle.c — the checker only) on
// identical synthetic inputs: survivors, eviction victims, block tables,
// the free list and attention outputs.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

#include "doctest.h"
#include "pagedevict/attention.hpp"
#include "pagedevict/block_table.hpp"
#include "pagedevict/importance.hpp"
#include "pagedevict/policy.hpp"

extern "C" {
#include "../../oracle/pe_oracle.h"
}

using namespace pagedevict;

namespace {

struct Gen {
    std::mt19937_64 rng;
    explicit Gen(std::uint64_t seed) : rng(seed) {}
    std::vector<float> row(std::size_t w) {
        std::normal_distribution<float> nd(0.0f, 1.0f);
        std::vector<float> r(w);
        for (auto& x : r) x = nd(rng);
        return r;
    }
    KvVector token(std::size_t w, std::uint64_t pos) { return make_kv(row(w), row(w), pos); }
};

PolicyConfig paged(std::size_t C, std::uint32_t B) {
    PolicyConfig c;
    c.cache_budget = C;
    c.page_size = B;
    c.kind = PolicyKind::PagedEviction;
    return c;
}

// Single-table oracle engine with the same pool as the façade.
struct OracleTable {
    peo_engine* e = nullptr;
    std::int32_t w;
    OracleTable(std::int32_t width, std::int32_t B, std::int32_t C, std::int32_t cap) : w(width) {
        REQUIRE(peo_engine_create(&e, 1, 1, 1, width, B, C, PEO_F32, PEO_PAGED_EVICTION, cap, cap) == 0);
    }
    ~OracleTable() { peo_engine_destroy(e); }
    std::vector<std::int32_t> pages() const {
        return std::vector<std::int32_t>(e->block_table, e->block_table + e->num_pages[0]);
    }
};

std::vector<float> padded(const std::vector<float>& x, std::size_t w) {
    std::vector<float> r(w, 0.0f);
    std::copy(x.begin(), x.end(), r.begin());
    return r;
}

}  // namespace

TEST_CASE("facade prefill selection and decode evictions match the C oracle") {
    const std::uint32_t B = 16;
    for (const std::size_t w : {16u, 40u, 128u}) {
        for (const std::size_t C : {64u, 256u}) {
            const std::size_t L = 3 * C + 7;
            const std::int32_t cap = static_cast<std::int32_t>(C / B + 2);
            Gen g(1000 + w + C);
            std::vector<KvVector> prompt;
            for (std::uint64_t i = 0; i < L; ++i) prompt.push_back(g.token(w, i));
            // oracle prefill over the same bytes (rows padded to the pool width)
            const std::size_t W = (w + 3) / 4 * 4;
            OracleTable o(static_cast<std::int32_t>(W), B, static_cast<std::int32_t>(C), cap);
            std::vector<float> K, V;
            for (const auto& kv : prompt) {
                auto k = padded(kv.key, W), v = padded(kv.value, W);
                K.insert(K.end(), k.begin(), k.end());
                V.insert(V.end(), v.begin(), v.end());
            }
            const std::int32_t cu[2] = {0, static_cast<std::int32_t>(L)};
            std::int32_t evicted = 0;
            REQUIRE(peo_prefill(o.e, 0, K.data(), V.data(), cu, 0, 1, &evicted) == 0);

            PagePool pool(static_cast<std::size_t>(cap), B);
            BlockTable table(pool);
            auto policy = make_policy(paged(C, B));
            auto pre = policy->prefill_compress(prompt);
            CHECK(pre.retained.size() == C);
            CHECK(pre.decision.kind == EvictionDecision::Kind::Tokens);
            CHECK(pre.decision.positions.size() == L - C);
            CHECK(static_cast<std::size_t>(evicted) == L - C);
            for (auto& kv : pre.retained) table.append_token(std::move(kv));
            // survivors: identical positions and physical pages
            std::vector<std::uint64_t> opos;
            for (std::int32_t j = 0; j < o.e->num_pages[0]; ++j) {
                const std::int32_t id = o.e->block_table[j];
                const std::int32_t cur = j + 1 == o.e->num_pages[0] ? o.e->newest_fill[0] : static_cast<std::int32_t>(B);
                for (std::int32_t s = 0; s < cur; ++s) opos.push_back(static_cast<std::uint64_t>(o.e->positions[id * B + s]));
            }
            CHECK(table.retained_positions() == opos);
            REQUIRE(table.page_count() == o.pages().size());
            for (std::size_t j = 0; j < table.page_count(); ++j)
                CHECK(static_cast<std::int32_t>(table.physical_id_at(j)) == o.pages()[j]);
            // decode: 4 eviction cycles
            for (std::int64_t step = 1; step <= static_cast<std::int64_t>(4 * B); ++step) {
                const std::uint64_t pos = L + static_cast<std::uint64_t>(step) - 1;
                KvVector kv = g.token(w, pos);
                auto k = padded(kv.key, W), v = padded(kv.value, W);
                const std::int64_t p64 = static_cast<std::int64_t>(pos);
                REQUIRE(peo_decode_append(o.e, 0, 1, k.data(), v.data(), &p64) == 0);
                std::int32_t ovic = -1;
                REQUIRE(peo_decode_evict(o.e, 0, 1, &ovic) == 0);
                const auto d = policy->decode_step(table, std::move(kv), step);
                if (ovic < 0) {
                    CHECK(d.kind == EvictionDecision::Kind::None);
                } else {
                    CHECK(d.kind == EvictionDecision::Kind::Page);
                    CHECK(d.logical_index == static_cast<std::size_t>(ovic));
                }
                CHECK(d.trigger_step == step);
            }
            CHECK(table.retained_len() == static_cast<std::size_t>(o.e->retained[0]));
            std::vector<std::int32_t> ids;
            for (std::size_t j = 0; j < table.page_count(); ++j) ids.push_back(static_cast<std::int32_t>(table.physical_id_at(j)));
            CHECK(ids == o.pages());
            CHECK(pool.free_count() == static_cast<std::size_t>(o.e->top));
            // the free list drains in the oracle's LIFO order
            std::vector<std::int32_t> drained, expect;
            for (std::int32_t i = o.e->top - 1; i >= 0; --i) expect.push_back(o.e->stack[i]);
            while (pool.free_count() > 0) drained.push_back(static_cast<std::int32_t>(pool.allocate()));
            CHECK(drained == expect);
        }
    }
}

TEST_CASE("facade attend is the reference's double-precision attention") {
    const std::uint32_t B = 16, H = 4, D = 32;
    Gen g(77);
    PagePool pool(64, B);
    BlockTable table(pool);
    std::vector<KvVector> toks;
    for (std::uint64_t i = 0; i < 150; ++i) {
        toks.push_back(g.token(H * D, i));
        table.append_token(toks.back());
    }
    table.free_page(2);  // retained tokens: logical order without page 2
    std::vector<KvVector> kept;
    for (const auto& t : toks)
        if (t.position < 32 || t.position >= 48) kept.push_back(t);
    const std::vector<float> q = g.row(H * D);
    const auto det = attend_detailed(AttentionInputs{q, &table, H, D});
    for (std::uint32_t h = 0; h < H; ++h) {
        std::vector<float> kk, vv;
        for (const auto& t : kept) {
            kk.insert(kk.end(), t.key.begin() + h * D, t.key.begin() + (h + 1) * D);
            vv.insert(vv.end(), t.value.begin() + h * D, t.value.begin() + (h + 1) * D);
        }
        std::vector<float> ref(D);
        peo_attend_dense(q.data() + h * D, kk.data(), vv.data(), kept.size(), D, ref.data());
        const std::vector<float> got(det.output.begin() + h * D, det.output.begin() + (h + 1) * D);
        CHECK(output_deviation(got, ref) <= 1e-12);
        CHECK(det.weight_sums[h] == doctest::Approx(1.0).epsilon(1e-12));
    }
    CHECK_THROWS_AS(attend(AttentionInputs{std::vector<float>(3), &table, H, D}), LengthMismatch);
    BlockTable empty(pool);
    CHECK_THROWS_AS(attend(AttentionInputs{q, &empty, H, D}), EmptyCache);
}

TEST_CASE("many tables share one device pool in LIFO order") {
    const std::uint32_t B = 8;
    PagePool pool(40, B);
    std::vector<BlockTable> tables;
    for (int t = 0; t < 5; ++t) tables.emplace_back(pool);
    Gen g(5);
    for (std::uint64_t i = 0; i < 30; ++i)
        for (auto& t : tables) t.append_token(g.token(8, i));
    // pages were popped 0,1,2,... in append order: table t's page j is 5*j+t
    for (std::size_t t = 0; t < tables.size(); ++t)
        for (std::size_t j = 0; j < tables[t].page_count(); ++j)
            CHECK(tables[t].physical_id_at(j) == static_cast<PageId>(5 * j + t));
    CHECK(pool.free_count() == 40 - 20);
    tables[1].clear();
    CHECK(pool.free_count() == 40 - 16);
    // released in logical order: the table's last page is handed out first
    BlockTable fresh(pool);
    fresh.append_token(g.token(8, 0));
    CHECK(fresh.physical_id_at(0) == 16);
    CHECK(pool.allocated() + pool.free_count() == pool.capacity());
}

TEST_CASE("bf16 pools store rounded rows and keep decisions exact") {
    PoolOptions opt;
    opt.dtype = PE_DTYPE_BF16;
    PagePool pool(20, 16, opt);
    BlockTable table(pool);
    auto policy = make_policy(paged(64, 16));
    Gen g(9);
    std::int64_t pages = 0;
    for (std::int64_t step = 1; step <= 200; ++step) {
        const auto d = policy->decode_step(table, g.token(64, static_cast<std::uint64_t>(step - 1)), step);
        pages += d.kind == EvictionDecision::Kind::Page;
        REQUIRE(table.retained_len() <= 64 + 16);
    }
    CHECK(pages == (200 - 64) / 16);
    const Page& p = table.page_at(0);
    CHECK(p.write_full());
    CHECK(p.at(0).key.size() == 64);
}

TEST_CASE("facade error mapping") {
    CHECK_THROWS_AS(paged(8, 16).validate(), BudgetInvalid);
    CHECK_THROWS_AS(make_policy(paged(100, 16)), BudgetInvalid);
    PagePool pool(1, 4);
    BlockTable table(pool);
    Gen g(1);
    for (int i = 0; i < 4; ++i) table.append_token(g.token(4, static_cast<std::uint64_t>(i)));
    CHECK_THROWS_AS(table.append_token(g.token(4, 4)), PoolExhausted);
    CHECK(table.retained_len() == 4);
    CHECK_THROWS_AS(table.free_page(3), IndexOutOfRange);
    CHECK_THROWS_AS(table.append_token(g.token(64, 5)), LengthMismatch);
    CHECK_THROWS_AS(make_kv({1.0f}, {1.0f, 2.0f}, 0), LengthMismatch);
    CHECK_THROWS_AS(make_policy(paged(64, 16)).get()->prefill_compress({}), Error);
    PagePool none(0, 4);
    BlockTable t0(none);
    CHECK_THROWS_AS(t0.append_token(g.token(4, 0)), PoolExhausted);
    CHECK_THROWS_AS(none.allocate(), PoolExhausted);
}
