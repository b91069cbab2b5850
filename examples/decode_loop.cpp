// decode_loop — the reference simulator's prefill/decode loop
// (proj/core/src/simulator.cpp:158-251) written as C++ host code against the
// engine's C-ABI (include/pe.h) with device-resident buffers: one engine per
// GPU, one prefill_prune_pack call per layer for the whole batch, then
// eviction cycles of B decode appends (all layers per call) and one
// PagedEviction launch, plus the GQA decode attention of every layer. No
// Python anywhere on this path; the CUDA runtime is used only for buffers,
// streams and events. Prints one JSON line and exits non-zero if the device
// invariant checker finds a violation.
//
// usage: decode_loop [seqs layers kv_heads head_dim prompt budget cycles [score]]
//        (defaults: BASELINE config 3 — 64 32 8 128 32768 4096 4; score:
//        0 = PE_SCORE_RECOMPUTE (default), 1 = PE_SCORE_CACHED)
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "pe.h"

namespace {

void check(pe_status st, const char* what) {
    if (st != PE_OK) {
        std::fprintf(stderr, "%s: %s (%s)\n", what, pe_status_string(st), pe_last_error());
        std::exit(2);
    }
}

void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        std::fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
        std::exit(2);
    }
}

uint16_t bf16(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

// Fills `bytes` of device memory with N(0,1) bf16 values: a 64 MB random
// block from the host, tiled device to device (distinct per `salt`).
void fill_bf16(void* dst, size_t bytes, uint64_t salt) {
    const size_t block = std::min<size_t>(bytes, size_t(64) << 20) & ~size_t(1);
    std::vector<uint16_t> h(block / 2);
    std::mt19937_64 rng(20250904 + salt);
    std::normal_distribution<float> nd(0.f, 1.f);
    for (auto& x : h) x = bf16(nd(rng));
    cuda(cudaMemcpy(dst, h.data(), block, cudaMemcpyHostToDevice), "fill");
    for (size_t off = block; off < bytes; off += block)
        cuda(cudaMemcpy(static_cast<char*>(dst) + off, dst, std::min(block, bytes - off), cudaMemcpyDeviceToDevice),
             "tile");
}

}  // namespace

int main(int argc, char** argv) {
    int S = 64, NL = 32, H = 8, d = 128, L = 32768, C = 4096, cycles = 4, score = PE_SCORE_RECOMPUTE;
    const int B = 16, G = 4;
    if (argc >= 8) {
        S = std::atoi(argv[1]);
        NL = std::atoi(argv[2]);
        H = std::atoi(argv[3]);
        d = std::atoi(argv[4]);
        L = std::atoi(argv[5]);
        C = std::atoi(argv[6]);
        cycles = std::atoi(argv[7]);
    }
    if (argc >= 9 && std::atoi(argv[8]) == 1) score = PE_SCORE_CACHED;
    pe_config cfg{};
    cfg.n_seqs = S;
    cfg.n_layers = NL;
    cfg.n_kv_heads = H;
    cfg.head_dim = d;
    cfg.granularity = PE_GRANULARITY_PER_KV_HEAD;
    cfg.page_size = B;
    cfg.cache_budget = C;
    cfg.dtype = PE_DTYPE_BF16;
    cfg.policy = PE_POLICY_PAGED_EVICTION;
    pe_engine* eng = nullptr;
    check(pe_engine_create(&cfg, &eng), "pe_engine_create");
    cudaStream_t st;
    cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);

    // ---- prefill prune+pack of every layer (simulator.cpp:170-187)
    const size_t row = size_t(d) * 2;
    const size_t in_bytes = size_t(S) * L * H * row;
    void *k = nullptr, *v = nullptr;
    cuda(cudaMalloc(&k, in_bytes), "k");
    cuda(cudaMalloc(&v, in_bytes), "v");
    fill_bf16(k, in_bytes, 1);
    fill_bf16(v, in_bytes, 2);
    std::vector<int32_t> cu(S + 1);
    for (int q = 0; q <= S; ++q) cu[q] = q * L;
    std::vector<float> pre_ms;
    for (int layer = 0; layer < NL; ++layer) {
        cudaEventRecord(e0, st);
        check(pe_prefill_prune_pack(eng, layer, k, v, cu.data(), 0, S, nullptr, st), "prefill");
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        pre_ms.push_back(ms);
    }
    check(pe_sync(eng), "prefill status");
    cudaFree(k);
    cudaFree(v);

    // ---- decode: cycles of B appends (all layers per call) + one eviction launch
    const size_t step_rows = size_t(NL) * S * H;
    void *rk = nullptr, *rv = nullptr, *q = nullptr;
    float* out = nullptr;
    int64_t* pos = nullptr;
    cuda(cudaMalloc(&rk, B * step_rows * row), "rows k");
    cuda(cudaMalloc(&rv, B * step_rows * row), "rows v");
    cuda(cudaMalloc(&q, size_t(S) * H * G * row), "q");
    cuda(cudaMalloc(&out, size_t(S) * H * G * d * sizeof(float)), "out");
    const int total_steps = (cycles + 1) * B;
    cuda(cudaMalloc(&pos, size_t(total_steps) * S * sizeof(int64_t)), "positions");
    {
        std::vector<int64_t> hp(size_t(total_steps) * S);
        for (int j = 0; j < total_steps; ++j)
            for (int s = 0; s < S; ++s) hp[size_t(j) * S + s] = int64_t(L) + j;
        cuda(cudaMemcpy(pos, hp.data(), hp.size() * sizeof(int64_t), cudaMemcpyHostToDevice), "positions");
    }
    fill_bf16(rk, B * step_rows * row, 3);
    fill_bf16(rv, B * step_rows * row, 4);
    fill_bf16(q, size_t(S) * H * G * row, 5);
    int step = 0;
    auto cycle = [&]() {
        for (int j = 0; j < B; ++j, ++step)
            check(pe_decode_append(eng, 0, NL, static_cast<char*>(rk) + j * step_rows * row,
                                   static_cast<char*>(rv) + j * step_rows * row, pos + size_t(step) * S, st),
                  "append");
        check(pe_decode_evict(eng, 0, NL, step, static_cast<pe_score_mode>(score), nullptr, st), "evict");
    };
    cycle();  // warm-up
    cudaEventRecord(e0, st);
    for (int c = 0; c < cycles; ++c) cycle();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float cyc_ms = 0.f;
    cudaEventElapsedTime(&cyc_ms, e0, e1);
    cyc_ms /= cycles;
    check(pe_sync(eng), "decode status");

    // ---- attention of every layer over the pruned tables
    std::vector<float> att_ms;
    for (int layer = 0; layer < NL; ++layer) {
        cudaEventRecord(e0, st);
        check(pe_paged_decode_attention(eng, layer, q, out, H * G, st), "attention");
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        att_ms.push_back(ms);
    }
    std::vector<float> h_out(size_t(S) * H * G * d);
    cuda(cudaMemcpy(h_out.data(), out, h_out.size() * sizeof(float), cudaMemcpyDeviceToHost), "out");
    bool finite = true;
    for (float x : h_out) finite = finite && std::isfinite(x);

    pe_invariants inv{};
    check(pe_check_invariants(eng, &inv), "invariants");
    pe_stats stt{};
    check(pe_get_stats(eng, &stt), "stats");
    const int64_t tables = int64_t(S) * NL * H;
    // algorithmic bytes as in DESIGN.md §3 (rkv = one token's K + V row)
    const double rkv = 2.0 * row;
    const double k2_bytes = double(tables) * ((C + B) * rkv + 8.0 * (C / B + 1) + 4);
    const double k0_bytes = double(tables) * B * (2.0 * rkv + 4);
    std::sort(pre_ms.begin(), pre_ms.end());
    std::sort(att_ms.begin(), att_ms.end());
    const int keep = std::min(L, C);
    const double k1_bytes = double(S) * H * (double(L) * rkv + keep * rkv + 4.0 * keep + 4.0 * ((keep + B - 1) / B));
    std::printf(
        "{\"tool\": \"examples/decode_loop\", \"seqs\": %d, \"layers\": %d, \"tables\": %lld, \"prompt\": %d, "
        "\"budget\": %d, \"prefill_ms_per_layer_p50\": %.4f, \"prefill_gbs\": %.1f, \"eviction_cycle_ms\": %.4f, "
        "\"eviction_cycle_gbs\": %.1f, \"attention_us_per_layer_p50\": %.2f, \"pages_evicted\": %lld, "
        "\"invariant_violations\": %lld, \"outputs_finite\": %s}\n",
        S, NL, static_cast<long long>(tables), L, C, pre_ms[pre_ms.size() / 2],
        k1_bytes / (pre_ms[pre_ms.size() / 2] * 1e-3) / 1e9, cyc_ms, (k2_bytes + k0_bytes) / (cyc_ms * 1e-3) / 1e9,
        att_ms[att_ms.size() / 2] * 1e3, static_cast<long long>(stt.pages_evicted),
        static_cast<long long>(inv.violations), finite ? "true" : "false");
    pe_engine_destroy(eng);
    return inv.violations == 0 && finite && stt.pages_evicted == tables * (cycles + 1) ? 0 : 1;
}
