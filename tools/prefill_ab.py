#!/usr/bin/env python3
"""K1 prefill A/B on one box: one engine, one synthetic cfg-shaped prompt
batch, every variant (a set of PE_* environment values, read by the engine at
call time) prefilling its own fresh layer, variants interleaved round by
round. Prints ms per layer (median) and GB/s against the BASELINE.md
algorithmic bytes, and checks that every variant's retained positions and
packed page bytes equal the first variant's on sampled tables.

  python tools/prefill_ab.py --config cfg3 --rounds 3 \
      --variant base: --variant l2:PE_PREFILL_L2=1,PE_WAVE_SEQS=2
"""
import argparse
import re
import json
import math
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2509_04377_b200 as pe  # noqa: E402

CONFIGS = {  # name: (seqs, L, kv_heads, d, C, dtype)
    "cfg1": (1, 4096, 8, 64, 1024, "f32"),
    "cfg2": (32, 16384, 8, 128, 2048, "bf16"),
    "cfg3": (64, 32768, 8, 128, 4096, "bf16"),
    "cfg5w": (16, 131072, 8, 128, 4096, "bf16"),  # one prompt wave of cfg5
    "cfg4h": (128, 0, 8, 128, 4096, "bf16"),  # the first prompt wave of cfg4 (lengths as bench_configs)
}


def cfg4_lengths():
    rng = np.random.default_rng(20250904 + 4)
    return np.exp(rng.uniform(np.log(1024), np.log(65536), 256)).astype(int)[:128]
B = 16


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--variant", action="append", required=True, help="name:VAR=val,VAR=val")
    args = ap.parse_args()
    S, L, H, d, C, dt = CONFIGS[args.config]
    tdt, pdt, elt = (torch.bfloat16, pe.DTYPE_BF16, 2) if dt == "bf16" else (torch.float32, pe.DTYPE_F32, 4)
    variants = []
    for v in args.variant:
        name, _, envs = v.partition(":")
        variants.append((name, dict(kv.split("=", 1) for kv in re.split(r",(?=[A-Z_0-9]+=)", envs) if kv)))
    keys = sorted({k for _, e in variants for k in e})
    n_layers = args.rounds * len(variants)
    eng = pe.PagedEvictionEngine(
        pe.EngineGeometry(n_seqs=S, n_layers=n_layers, n_kv_heads=H, head_dim=d, dtype=pdt),
        pe.PolicyConfig(cache_budget=C, page_size=B))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(2509)
    lens = cfg4_lengths() if args.config == "cfg4h" else np.full(S, L)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    k = torch.empty((int(cu[-1]), H, d), dtype=tdt, device="cuda").normal_(generator=gen)
    v = torch.empty_like(k).normal_(generator=gen)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    row = 2 * d * elt
    alg = H * sum(int(x) * row + min(int(x), C) * (row + 4) + 4 * math.ceil(min(int(x), C) / B) for x in lens)
    times = {n: [] for n, _ in variants}
    layer_of = {n: [] for n, _ in variants}
    stream = torch.cuda.current_stream()
    layer = 0
    for r in range(args.rounds):
        for name, env in variants:
            for kk in keys:
                os.environ.pop(kk, None)
            os.environ.update(env)
            flush.zero_()  # L2 holds nothing of the prompt
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            eng.prefill_compress(layer, k, v, cu)
            e1.record(stream)
            e1.synchronize()
            times[name].append(e0.elapsed_time(e1))
            layer_of[name].append(layer)
            layer += 1
    for kk in keys:
        os.environ.pop(kk, None)
    eng.sync()
    # parity across variants: sampled tables' positions and page bytes
    rng = np.random.default_rng(7)
    ref_layer = layer_of[variants[0][0]][0]
    mism = 0
    for s_ in rng.choice(S, size=min(S, 4), replace=False):
        for h in rng.choice(H, size=2, replace=False):
            t0 = eng.table_id(int(s_), ref_layer, int(h))
            p0 = eng.retained_positions(t0)
            pg0 = [eng.pages(eng.physical_id_at(t0, j), 1) for j in (0, eng.page_count(t0) - 1)]
            for name, _ in variants:
                for ly in layer_of[name]:
                    t = eng.table_id(int(s_), ly, int(h))
                    if not np.array_equal(eng.retained_positions(t), p0):
                        mism += 1
                        continue
                    pg = [eng.pages(eng.physical_id_at(t, j), 1) for j in (0, eng.page_count(t) - 1)]
                    mism += sum(not np.array_equal(a, b) for a, b in zip(pg, pg0))
    inv = eng.check_invariants()
    out = {"config": args.config, "algorithmic_bytes_per_layer": alg, "parity_mismatches": mism,
           "invariants": inv, "variants": {}}
    for name, env in variants:
        ms = statistics.median(times[name])
        out["variants"][name] = {"env": env, "ms_per_layer_p50": round(ms, 4),
                                 "ms_all": [round(x, 4) for x in times[name]],
                                 "gbs": round(alg / (ms * 1e-3) / 1e9, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
