// Metrics emitters on both builds (test infrastructure): a fixed set of
// StepRecords / MetricsRecords with awkward numbers (signed zero, integral
// doubles, the exponent thresholds, NaN, repeating fractions, quoting)
// printed through emit_jsonl, emit_csv and format_summary(summarize(...)).
// tests/cpp/build_conformance.py compiles it against the reference sources
// (metrics.cpp + its JSON library) and against the B200 façade;
// tests/test_steplog.py requires byte-identical output from both and from
// the Python mirror (paper_2509_04377_b200/steplog.py), which reads the same
// records from tests/golden/metrics_records.json.
#include <cmath>
#include <cstdio>
#include <limits>
#include <string>
#include <vector>

#include "pagedevict/metrics.hpp"

using namespace pagedevict;

int main() {
    const double nan = std::numeric_limits<double>::quiet_NaN();
    const double vals[] = {0.0,     -0.0,    1.0,     0.5,      0.1,       1.0 / 3.0, 2.0 / 3.0, 1e-4,
                           1e-5,    1.5e-5,  0.00031, 123.25,   1e15,      1e16,      1.5e20,    9.999e14,
                           12345678901234567890.0,  4.9e-324, 1.7976931348623157e308, 0.0039215686274509665,
                           0.015625, 0.99609375, 0.9375,  nan};
    std::vector<StepRecord> steps;
    std::uint32_t k = 0;
    for (const double v : vals) {
        StepRecord r;
        r.run = k % 3;
        r.sequence = k % 5;
        r.layer = k % 7;
        r.step = 1 + static_cast<std::int64_t>(k);
        r.retained_len = 4096 + k;
        if (k % 3 == 0) r.decision = EvictionDecision::page(k % 11, r.step);
        else if (k % 3 == 1) r.decision = EvictionDecision::tokens({k, 7ull * k, 1ull << 40}, r.step);
        else r.decision = EvictionDecision::none(r.step);
        r.fragmentation = v;
        r.deviation = vals[(k + 5) % (sizeof vals / sizeof vals[0])];
        steps.push_back(r);
        ++k;
    }
    StepRecord empty_tokens;
    empty_tokens.decision = EvictionDecision::tokens({}, 3);
    empty_tokens.deviation = nan;
    steps.push_back(empty_tokens);
    std::fputs(emit_jsonl(steps).c_str(), stdout);

    std::vector<MetricsRecord> recs;
    const char* policies[] = {"paged-eviction", "streaming-llm", "inv-key-l2", "key-diff", "full",
                              "paged-eviction", "odd,\"name\""};
    for (int i = 0; i < 7; ++i) {
        MetricsRecord m;
        m.policy = policies[i];
        m.cache_budget = 1024u << (i % 3);
        m.page_size = 16;
        m.prefill_len = 4096 + 13 * i;
        m.decode_steps = 256;
        m.batch = 1 + i;
        m.layer_count = 16;
        m.seed = 20250904 + i;
        m.prefill_evicted = 3072u * (i + 1);
        m.evictions_total = 17u * i;
        m.page_evictions = 16u * i;
        m.token_evictions = 5u * i;
        m.block_table_updates = 17u * i + (i == 1 ? 3 : 0);
        m.mean_fragmentation = vals[i];
        m.max_fragmentation = vals[i + 3];
        m.max_fragmentation_excl_newest = vals[i + 9];
        m.mean_deviation = vals[(i + 12) % 23];
        m.p95_deviation = 1.0 / (3.0 + i);
        m.retained_bytes = 1ull << (30 + i);
        recs.push_back(m);
    }
    std::fputs(emit_csv(recs).c_str(), stdout);
    const auto rows = summarize(recs);
    std::fputs(format_summary(rows).c_str(), stdout);
    // no PagedEviction record: cadence n/a
    std::vector<MetricsRecord> only_full(recs.begin() + 4, recs.begin() + 5);
    const auto rows2 = summarize(only_full);
    std::fputs(format_summary(rows2).c_str(), stdout);
    try {
        summarize(std::vector<MetricsRecord>{});
    } catch (const EmptyInput&) {
        std::puts("EmptyInput");
    }
    return 0;
}
