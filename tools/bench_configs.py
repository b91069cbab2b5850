#!/usr/bin/env python3
"""Measures the PagedEviction kernels on every BASELINE.json config (one
JSON line each). bench.py is the driver-facing headline (cfg3); this script
covers the rest:

  cfg1  Llama-3.2-1B KV geometry, 1 seq x 4K fp32 prefill, C=1024 (full)
  cfg2  Llama-3.2-3B geometry, batch 32 x 16K, C=2048, bf16 (full)
  cfg4  mixed-length serving trace: 256 sequences, lengths log-uniform in
        [1K, 64K] (seeded), 8B geometry, C=4096, shared pool; decode with
        continuous block eviction + paged attention every step
  cfg5  8B geometry, 128K context, one layer's tables of 1024 sequences
        (prefill streamed in sequence waves), eviction cycles

Per config: prefill GB/s (K1), eviction-step GB/s + p50 µs (K2), cached
eviction p50 (K2c), attention GB/s (K3), decode tokens/s. Algorithmic bytes
as in DESIGN.md §3. Synthetic N(0,1) data.
"""
import argparse
import json
import math
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2509_04377_b200 as pe  # noqa: E402

B = 16
PEAK = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else 6650.0


def ev():
    return torch.cuda.Event(enable_timing=True)


def timed(fn, stream):
    a, b = ev(), ev()
    a.record(stream)
    fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b)


def k1_bytes(lens, C, row):
    return sum(L * row + min(L, C) * row + 4 * min(L, C) + 4 * math.ceil(min(L, C) / B) for L in lens)


def run(name, layers, kvh, d, qh, lens, C, dtype, decode_steps, waves=1, pool_layers=None):
    torch.cuda.empty_cache()
    bf16 = dtype == "bf16"
    tdt = torch.bfloat16 if bf16 else torch.float32
    elt = 2 if bf16 else 4
    row = 2 * d * elt
    S = len(lens)
    G = qh // kvh
    eng = pe.PagedEvictionEngine(pe.EngineGeometry(n_seqs=S, n_layers=layers, n_kv_heads=kvh, head_dim=d,
                                                   dtype=pe.DTYPE_BF16 if bf16 else pe.DTYPE_F32),
                                 pe.PolicyConfig(cache_budget=C, page_size=B))
    st = torch.cuda.current_stream()
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1234)
    # ---- prefill (sequence waves when the raw prompt does not fit)
    per_wave = math.ceil(S / waves)
    pre_layer_ms = []
    max_tok = max(sum(lens[w0:w0 + per_wave]) for w0 in range(0, S, per_wave))
    k_in = torch.empty((max_tok, kvh, d), dtype=tdt, device="cuda")
    v_in = torch.empty_like(k_in)
    for layer in range(layers):
        ms = 0.0
        for w0 in range(0, S, per_wave):
            wl = lens[w0:w0 + per_wave]
            n = sum(wl)
            k_in[:n].normal_(generator=gen)
            v_in[:n].normal_(generator=gen)
            cu = np.concatenate([[0], np.cumsum(wl)]).astype(np.int32)
            ms += timed(lambda: eng.prefill_compress(layer, k_in[:n], v_in[:n], cu, seq_begin=w0), st)
        pre_layer_ms.append(ms)
    eng.sync()
    # per-layer p50 without the first layer (first calls load modules and
    # allocate the select's scratch); one layer only: that layer
    pre_p50 = statistics.median(pre_layer_ms[1:] or pre_layer_ms)
    del k_in, v_in
    torch.cuda.empty_cache()
    n_tab = S * layers * kvh
    pre_gbs = k1_bytes(lens, C, row) * kvh / (pre_p50 * 1e-3) / 1e9
    # ---- decode: K0 (all layers per token) + K2 at triggers + K3 per layer
    pos = torch.tensor(lens, dtype=torch.int64, device="cuda")
    rk = torch.randn((B, layers, S, kvh, d), generator=gen, device="cuda", dtype=torch.float32).to(tdt)
    rv = torch.randn((B, layers, S, kvh, d), generator=gen, device="cuda", dtype=torch.float32).to(tdt)
    q = torch.randn((S, qh, d), generator=gen, device="cuda", dtype=torch.float32).to(tdt)
    out = torch.empty((S, qh, d), dtype=torch.float32, device="cuda")
    evicted0 = eng.stats().pages_evicted
    # (1) serving loop, timed as a whole (no events between launches, so
    # consecutive launches overlap through PDL as in a real serving loop):
    # per decode token, K0 on every layer, then per layer evict(l) + attend(l)
    t0, t1 = ev(), ev()
    torch.cuda.synchronize()
    t0.record(st)
    for step in range(decode_steps):
        j = step % B
        eng.append_token(0, layers, rk[j], rv[j], pos)
        pos.add_(1)
        for layer in range(layers):
            eng.evict(layer, 1, step=step + 1)
            eng.attend(layer, q, out, qh)
    t1.record(st)
    t1.synchronize()
    dec_ms = t0.elapsed_time(t1)
    steps_run = decode_steps

    # (2) kernel timings over 2B more tokens: each token's per-layer evictions
    # back to back (one event pair around the layer loop; recompute scores in
    # the first B tokens, cached in the next B), then the per-layer attention
    # back to back
    k2_groups, k2c_groups, k2_other, k3_groups = [], [], [], []
    for step in range(2 * B):
        j = step % B
        eng.append_token(0, layers, rk[j], rv[j], pos)
        pos.add_(1)
        steps_run += 1
        cached = step >= B
        a, b = ev(), ev()
        a.record(st)
        for layer in range(layers):
            eng.evict(layer, 1, step=steps_run, mode=pe.ScoreMode.CACHED if cached else pe.ScoreMode.RECOMPUTE)
        b.record(st)
        if steps_run % B == 0:  # uniform prompts >= C: every table triggers at these steps
            (k2c_groups if cached else k2_groups).append((a, b))
        else:
            k2_other.append((a, b))
        a3, b3 = ev(), ev()
        a3.record(st)
        for layer in range(layers):
            eng.attend(layer, q, out, qh)
        b3.record(st)
        k3_groups.append((a3, b3))
    # all-layer eviction launches (one per decode step, as bench.py): B more steps
    all_ms = []
    for j in range(B):
        eng.append_token(0, layers, rk[j], rv[j], pos)
        pos.add_(1)
        steps_run += 1
        a, b = ev(), ev()
        a.record(st)
        eng.evict(0, layers, step=steps_run, mode=pe.ScoreMode.RECOMPUTE)
        b.record(st)
        all_ms.append((a, b))
    torch.cuda.synchronize()
    per_layer = lambda grp: [a.elapsed_time(b) / layers for a, b in grp]  # noqa: E731
    k2_ms, k2c_ms, k3_ms = per_layer(k2_groups), per_layer(k2c_groups), per_layer(k3_groups)
    all_ms = [a.elapsed_time(b) for a, b in all_ms]
    evicted = eng.stats().pages_evicted - evicted0
    # checks (untimed): the device invariant checker over the whole state and
    # the eviction cadence — a table that starts decode at R0 = min(L, C)
    # retained tokens has made max(0, floor((R0 + D) / B) - C / B) page
    # evictions after D decode tokens (policy.cpp:147-150; pages never have
    # holes, so the newest page is full exactly when retained % B == 0)
    D = steps_run
    expect = layers * kvh * sum(max(0, (min(L, C) + D) // B - C // B) for L in lens)
    inv = eng.check_invariants()
    # eviction launches at a trigger step (all tables of the layer triggered together in uniform configs)
    trig = k2_ms
    _, _, _, retained = eng.tables()
    mean_R = float(retained.mean())
    k3 = k3_ms
    k3_bytes = S * kvh * (mean_R * row + 4 * math.ceil(mean_R / B) + G * d * (elt + 4))
    line = {
        "config": name, "tables": n_tab, "dtype": dtype, "seqs": S, "C": C,
        "prompt_len": {"min": int(min(lens)), "max": int(max(lens)), "mean": float(np.mean(lens))},
        "prefill": {"ms_per_layer_p50": round(pre_p50, 4), "ms_first_layer": round(pre_layer_ms[0], 3),
                    "gbs": round(pre_gbs, 1), "frac": round(pre_gbs / PEAK, 4), "waves": waves},
        "evict_recompute_us": {"p50": round(statistics.median(trig) * 1e3, 2), "max": round(max(trig) * 1e3, 2),
                               "timing": "per-layer launches back to back, mean per launch, trigger steps"},
        "evict_nontrigger_step_us_p50": round(statistics.median(per_layer(k2_other)) * 1e3, 2),
        "evict_cached_us_p50": round(statistics.median(k2c_ms) * 1e3, 2),
        "pages_evicted": int(evicted),
        "checks": {"evictions_expected": int(expect), "evictions_observed": int(evicted),
                   "cadence_ok": int(expect) == int(evicted), "invariant_violations": int(inv["violations"]),
                   "tables_checked": n_tab},
        "attention": {"us_p50": round(statistics.median(k3) * 1e3, 2),
                      "gbs": round(k3_bytes / (statistics.median(k3) * 1e-3) / 1e9, 1),
                      "mean_retained": round(mean_R, 1)},
        "decode": {"steps": decode_steps, "tokens_per_s": round(S * decode_steps / (dec_ms * 1e-3), 1),
                   "ms_per_step_all_layers": round(dec_ms / decode_steps, 4),
                   "loop": "per token: K0 on all layers, then per layer K2 (recompute) + K3; timed as a whole"},
    }
    # eviction-step GB/s for a uniform config: all tables of a layer trigger at the same step
    if min(lens) == max(lens) and min(lens) >= C:
        k2_bytes = S * kvh * ((C + B) * row + 8 * (C // B + 1) + 4)
        p50 = statistics.median(trig)
        line["evict_step_gbs"] = round(k2_bytes / (p50 * 1e-3) / 1e9, 1)
        line["evict_step_frac"] = round(line["evict_step_gbs"] / PEAK, 4)
        # one launch for all layers at the trigger step (the last of the B steps)
        line["evict_all_layers_us"] = round(all_ms[-1] * 1e3, 2)
        line["evict_all_layers_gbs"] = round(layers * k2_bytes / (all_ms[-1] * 1e-3) / 1e9, 1)
        line["evict_all_layers_frac"] = round(line["evict_all_layers_gbs"] / PEAK, 4)
    else:
        line["evict_all_layers_us_mean"] = round(statistics.mean(all_ms) * 1e3, 2)
    print(json.dumps(line), flush=True)
    del eng
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg1,cfg2,cfg4,cfg5")
    ap.add_argument("--decode-steps", type=int, default=64)
    a = ap.parse_args()
    todo = a.configs.split(",")
    if "cfg1" in todo:
        run("cfg1", 16, 8, 64, 32, [4096], 1024, "f32", a.decode_steps)
    if "cfg2" in todo:
        run("cfg2", 28, 8, 128, 24, [16384] * 32, 2048, "bf16", a.decode_steps)
    if "cfg4" in todo:
        rng = np.random.default_rng(20250904 + 4)
        lens = np.exp(rng.uniform(np.log(1024), np.log(65536), 256)).astype(int).tolist()
        run("cfg4", 32, 8, 128, 32, lens, 4096, "bf16", a.decode_steps, waves=2)
    if "cfg5" in todo:
        run("cfg5(1 layer, 1 GPU)", 1, 8, 128, 32, [131072] * 1024, 4096, "bf16", a.decode_steps, waves=64)


if __name__ == "__main__":
    main()
