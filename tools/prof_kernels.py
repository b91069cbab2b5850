"""Small driver for ncu captures: cfg3 geometry (64 seqs, 8 KV heads, d=128,
L=32768, C=4096, bf16) with a reduced layer count. Runs K1 prefill per
layer, two eviction cycles (K0 x16 + K2 per layer, recompute), one K2c
cycle and one attention call per layer."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2509_04377_b200 as pe

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--seqs", type=int, default=64)
ap.add_argument("--L", type=int, default=32768)
ap.add_argument("--C", type=int, default=4096)
ap.add_argument("--cycles", type=int, default=2)
a = ap.parse_args()
S, NL, H, d, B, QH = a.seqs, a.layers, 8, 128, 16, 32
eng = pe.PagedEvictionEngine(pe.EngineGeometry(n_seqs=S, n_layers=NL, n_kv_heads=H, head_dim=d,
                                               dtype=pe.DTYPE_BF16),
                             pe.PolicyConfig(cache_budget=a.C, page_size=B))
g = torch.Generator(device="cuda")
g.manual_seed(1)
cu = np.arange(S + 1, dtype=np.int32) * a.L
k = torch.empty((S * a.L, H, d), dtype=torch.bfloat16, device="cuda")
v = torch.empty_like(k)
for layer in range(NL):
    k.normal_(generator=g)
    v.normal_(generator=g)
    eng.prefill_compress(layer, k, v, cu)
eng.sync()
del k, v
rk = torch.randn((B, NL, S, H, d), device="cuda").bfloat16()
rv = torch.randn((B, NL, S, H, d), device="cuda").bfloat16()
pos = torch.full((S,), a.L, dtype=torch.int64, device="cuda")
for c in range(a.cycles + 1):
    for j in range(B):
        eng.append_token(0, NL, rk[j], rv[j], pos)
        pos.add_(1)
    for layer in range(NL):
        eng.evict(layer, 1, mode=pe.ScoreMode.CACHED if c == a.cycles else pe.ScoreMode.RECOMPUTE)
q = torch.randn((S, QH, d), device="cuda").bfloat16()
out = torch.empty((S, QH, d), dtype=torch.float32, device="cuda")
for layer in range(NL):
    eng.attend(layer, q, out, QH)
eng.sync()
print("done", eng.stats().pages_evicted)
