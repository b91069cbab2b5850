#!/usr/bin/env python3
"""K2 eviction A/B on one box at cfg3 shape (or cfg2): one engine prefilled
once, then eviction cycles (B appends on all layers + the eviction), each
cycle's eviction run under one variant (PE_* environment values, read by the
engine at launch time), variants interleaved cycle by cycle. Reports, per
variant, the per-launch time of per-layer launches issued back to back
(--launch layer) or of one all-layer launch (--launch step), and GB/s over
the K2 algorithmic bytes. Every variant runs the same decision semantics, so
the device invariant checker closes the run.

  python tools/k2_ab.py --launch layer --cycles 12 --variant base: --variant c14:PE_K2_CTAS_PER_SM=14
"""
import argparse
import re
import json
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2509_04377_b200 as pe  # noqa: E402

CONFIGS = {  # name: (seqs, layers, L, kv_heads, d, C)
    "cfg2": (32, 28, 16384, 8, 128, 2048),
    "cfg3": (64, 32, 32768, 8, 128, 4096),
}
B = 16


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--launch", default="layer", choices=["layer", "step", "serve"],
                    help="serve: per decode token, append on every layer, then per layer evict(l) + attend(l) "
                         "(GQA, 4 query heads per KV head); the time is per decode token")
    ap.add_argument("--cycles", type=int, default=12)
    ap.add_argument("--variant", action="append", required=True, help="name:VAR=val,VAR=val")
    args = ap.parse_args()
    S, NL, L, H, d, C = CONFIGS[args.config]
    variants = []
    for v in args.variant:
        name, _, envs = v.partition(":")
        variants.append((name, dict(kv.split("=", 1) for kv in re.split(r",(?=[A-Z_0-9]+=)", envs) if kv)))
    keys = sorted({k for _, e in variants for k in e})
    eng = pe.PagedEvictionEngine(
        pe.EngineGeometry(n_seqs=S, n_layers=NL, n_kv_heads=H, head_dim=d, dtype=pe.DTYPE_BF16),
        pe.PolicyConfig(cache_budget=C, page_size=B))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(2509)
    wave = 16
    k = torch.empty((wave * L, H, d), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    for layer in range(NL):
        for w0 in range(0, S, wave):
            k.normal_(generator=gen)
            v.normal_(generator=gen)
            eng.prefill_compress(layer, k, v, np.arange(wave + 1, dtype=np.int32) * L, seq_begin=w0)
    del k, v
    torch.cuda.empty_cache()
    rows_k = torch.randn((B, NL, S, H, d), generator=gen, device="cuda").to(torch.bfloat16)
    rows_v = torch.randn((B, NL, S, H, d), generator=gen, device="cuda").to(torch.bfloat16)
    stream = torch.cuda.current_stream()
    row = 2 * d * 2
    per_table = (C + B) * row + 8 * (C // B + 1) + 4
    n_tab = S * NL * H
    spans = [(0, NL)] if args.launch == "step" else [(ly, 1) for ly in range(NL)]
    G = 4
    q = torch.randn((S, H * G, d), generator=gen, device="cuda").to(torch.bfloat16)
    out = torch.empty((S, H * G, d), dtype=torch.float32, device="cuda")
    launch_bytes = per_table * (n_tab if args.launch == "step" else S * H)
    times = {n: [] for n, _ in variants}
    pos = L
    for c in range(args.cycles + 1):
        for name, env in variants:
            for kk in keys:
                os.environ.pop(kk, None)
            os.environ.update(env)
            if args.launch == "serve":
                ps = [torch.full((S,), pos + j, dtype=torch.int64, device="cuda") for j in range(B)]
                pos += B
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for j in range(B):
                    eng.append_token(0, NL, rows_k[j], rows_v[j], ps[j])
                    for ly in range(NL):
                        eng.evict(ly, 1, step=j + 1)
                        eng.attend(ly, q, out, H * G)
                b.record(stream)
                b.synchronize()
                if c > 0:
                    times[name].append(a.elapsed_time(b) / B)
                continue
            for j in range(B):
                p = torch.full((S,), pos, dtype=torch.int64, device="cuda")
                eng.append_token(0, NL, rows_k[j], rows_v[j], p)
                pos += 1
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for l0, nl in spans:
                eng.evict(l0, nl)
            b.record(stream)
            b.synchronize()
            if c > 0:  # cycle 0 warms every variant
                times[name].append(a.elapsed_time(b) / len(spans))
    for kk in keys:
        os.environ.pop(kk, None)
    eng.sync()
    inv = eng.check_invariants()
    res = {"config": args.config, "launch": args.launch, "bytes_per_launch": launch_bytes, "invariants": inv,
           "variants": {}}
    for name, env in variants:
        ms = statistics.median(times[name])
        res["variants"][name] = {"env": env, "us_per_launch_p50": round(ms * 1e3, 2),
                                 "us_all": [round(x * 1e3, 1) for x in times[name]],
                                 "gbs": round(launch_bytes / (ms * 1e-3) / 1e9, 1)}
        if args.launch == "serve":
            res["variants"][name]["tokens_per_s"] = round(S / (ms * 1e-3), 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
