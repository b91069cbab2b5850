// One program, two backends (test infrastructure): randomized cache-manager
// traces written ONLY against the reference's public pagedevict:: API.
// tests/cpp/build_conformance.py compiles it twice — against the reference
// sources (oracle/_ref/scenario_ref, CPU) and against the B200 façade
// (tests/cpp/_build/scenario_b200) — and tests/test_facade_gpu.py requires
// the two decision / state logs to be identical (attention outputs within
// 1e-12 relative: exp may differ in the last ulp).
//
// Every policy (PagedEviction, StreamingLLM, InvKeyL2, KeyDiff, FullCache),
// several tables sharing one pool, prefill over and under budget, decode
// with evictions, free_page / evict_slot / clear, attention.
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "pagedevict/attention.hpp"
#include "pagedevict/block_table.hpp"
#include "pagedevict/importance.hpp"
#include "pagedevict/policy.hpp"

using namespace pagedevict;

namespace {

// Box-Muller over a 64-bit LCG: identical streams on both builds
struct Rng {
    std::uint64_t x;
    explicit Rng(std::uint64_t seed) : x(seed * 6364136223846793005ull + 1442695040888963407ull) {}
    double uni() {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        return (static_cast<double>(x >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    }
    float normal() {
        const double u = uni(), v = uni();
        return static_cast<float>(std::sqrt(-2.0 * std::log(u)) * std::cos(6.283185307179586 * v));
    }
    std::uint32_t below(std::uint32_t n) { return static_cast<std::uint32_t>(uni() * n); }
};

KvVector token(Rng& r, std::size_t w, std::uint64_t pos) {
    std::vector<float> k(w), v(w);
    for (auto& a : k) a = r.normal();
    for (auto& a : v) a = r.normal();
    return make_kv(std::move(k), std::move(v), pos);
}

std::uint64_t fnv(const std::vector<std::uint64_t>& xs) {
    std::uint64_t h = 1469598103934665603ull;
    for (const auto x : xs) h = (h ^ x) * 1099511628211ull;
    return h;
}

void state(const char* tag, const BlockTable& t, const PagePool& pool) {
    const auto pos = t.retained_positions();
    std::printf("S %s n=%zu ret=%zu free=%zu frag=%.17g fragx=%.17g pos=%016" PRIx64 " ids=", tag, t.page_count(),
                t.retained_len(), pool.free_count(), t.fragmentation_ratio(), t.fragmentation_ratio_excluding_newest(),
                fnv(pos));
    for (std::size_t j = 0; j < t.page_count(); ++j) std::printf("%u,", t.physical_id_at(j));
    std::printf("\n");
}

void decision(std::int64_t step, const EvictionDecision& d) {
    std::printf("D %" PRId64 " kind=%d", step, static_cast<int>(d.kind));
    if (d.kind == EvictionDecision::Kind::Page) std::printf(" page=%zu", d.logical_index);
    if (d.kind == EvictionDecision::Kind::Tokens) {
        std::printf(" n=%zu h=%016" PRIx64, d.positions.size(), fnv(d.positions));
        if (d.positions.size() == 1) std::printf(" p=%" PRIu64, d.positions[0]);
    }
    std::printf("\n");
}

}  // namespace

int main() {
    const PolicyKind kinds[] = {PolicyKind::PagedEviction, PolicyKind::StreamingLlm, PolicyKind::InvKeyL2,
                                PolicyKind::KeyDiff, PolicyKind::FullCache};
    Rng rng(20250904);
    int scenario = 0;
    for (const PolicyKind kind : kinds) {
        for (int round = 0; round < 6; ++round, ++scenario) {
            const std::uint32_t B = round % 2 ? 8 : 16;
            const std::size_t C = B * (2 + rng.below(5));
            const std::size_t w = std::vector<std::size_t>{4, 16, 40, 64}[rng.below(4)];
            const std::uint32_t heads = w % 8 == 0 ? 4 : 2;
            const int n_tables = 1 + static_cast<int>(rng.below(3));
            std::vector<std::size_t> L(n_tables);
            std::size_t need = 0;
            const std::size_t D = 2 * C + rng.below(static_cast<std::uint32_t>(C));
            for (auto& l : L) {
                l = 1 + rng.below(static_cast<std::uint32_t>(3 * C));
                need += (kind == PolicyKind::PagedEviction ? C + B : l + D) / B + 2;
            }
            std::printf("# scenario %d kind=%d B=%u C=%zu w=%zu tables=%d D=%zu\n", scenario, static_cast<int>(kind),
                        B, C, w, n_tables, D);
            PagePool pool(need, B);
            std::vector<BlockTable> tables;
            std::vector<std::unique_ptr<EvictionPolicy>> pols;
            PolicyConfig cfg;
            cfg.kind = kind;
            cfg.cache_budget = C;
            cfg.page_size = B;
            cfg.sink_count = round % 3;
            for (int t = 0; t < n_tables; ++t) {
                tables.emplace_back(pool);
                pols.push_back(make_policy(cfg));
                std::vector<KvVector> prompt;
                for (std::uint64_t i = 0; i < L[t]; ++i) prompt.push_back(token(rng, w, i));
                auto res = pols[t]->prefill_compress(std::move(prompt));
                decision(0, res.decision);
                for (auto& kv : res.retained) tables[t].append_token(std::move(kv));
                state("prefill", tables[t], pool);
            }
            for (std::size_t step = 1; step <= D; ++step) {
                for (int t = 0; t < n_tables; ++t) {
                    const auto d = pols[t]->decode_step(tables[t], token(rng, w, L[t] + step - 1),
                                                        static_cast<std::int64_t>(step));
                    decision(static_cast<std::int64_t>(step), d);
                    if (step % 5 == 0) state("decode", tables[t], pool);
                }
            }
            for (int t = 0; t < n_tables; ++t) {
                std::vector<float> q(heads * (w / heads));
                for (auto& a : q) a = rng.normal();
                const auto det = attend_detailed(AttentionInputs{q, &tables[t], heads, static_cast<std::uint32_t>(w / heads)});
                for (std::size_t i = 0; i < det.output.size(); ++i) std::printf("A %zu %.9e\n", i, det.output[i]);
                for (const double ws : det.weight_sums) std::printf("W %.15f\n", ws);
                const auto scores = score_pages(tables[t]);
                std::printf("R %zu\n", scores.empty() ? 0 : rank_pages(scores));
            }
            // structural ops on the first table, then release everything
            BlockTable& t0 = tables[0];
            if (t0.page_count() > 1) {
                t0.free_page(t0.page_count() / 2);
                state("free_page", t0, pool);
            }
            const auto pos = t0.retained_positions();
            if (!pos.empty()) {
                t0.evict_slot(pos[pos.size() / 3]);
                state("evict_slot", t0, pool);
            }
            try {
                t0.evict_slot(1u << 30);
            } catch (const UnknownPosition&) {
                std::printf("E unknown-position\n");
            }
            t0.clear();
            state("clear", t0, pool);
            std::printf("F %zu %zu\n", pool.free_count(), pool.allocated());
        }
    }
    return 0;
}
