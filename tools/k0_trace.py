#!/usr/bin/env python3
"""K0 timeline from a tooling build (nvcc -DPE_K0_TRACE, loaded with PE_LIB):
%globaltimer stamps of the first 256 CTAs of each of the last append
launches, for one cfg3 eviction cycle (16 appends back to back, as bench.py
issues them). Per launch: when its CTAs became resident, when the previous
kernel had completed (griddepcontrol.wait returned), the phases, and the last
CTA's end; between launches: the gap from one launch's last CTA to the next
launch's release.

  PE_LIB=ab/libpe_b200_trace.so python tools/k0_trace.py
"""
import ctypes
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2509_04377_b200 as pe  # noqa: E402

S, NL, H, d, C, B, L = 64, 32, 8, 128, 4096, 16, 4096
eng = pe.PagedEvictionEngine(pe.EngineGeometry(n_seqs=S, n_layers=NL, n_kv_heads=H, head_dim=d, dtype=pe.DTYPE_BF16),
                             pe.PolicyConfig(cache_budget=C, page_size=B))
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
k = torch.empty((S * L, H, d), dtype=torch.bfloat16, device="cuda")
for layer in range(NL):
    k.normal_(generator=gen)
    eng.prefill_compress(layer, k, k, np.arange(S + 1, dtype=np.int32) * L)
del k
rows = torch.randn((B, NL, S, H, d), generator=gen, device="cuda").to(torch.bfloat16)
pos = torch.arange(100000, device="cuda", dtype=torch.int64).unsqueeze(1).expand(100000, S).contiguous() + L
t = 0
for cycle in range(4):
    for j in range(B):
        eng.append_token(0, NL, rows[j], rows[j], pos[t])
        t += 1
    eng.evict(0, NL)
eng.sync()
lib = ctypes.CDLL(os.environ["PE_LIB"])
buf = np.zeros(64 * 256 * 10, dtype=np.uint64)
assert lib.pe_debug_k0_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
tr = buf.reshape(64, 256, 10).astype(np.int64)
epochs = [e for e in range(64) if tr[e, 0, 0] > 0]
launches = sorted(epochs, key=lambda e: tr[e, :, 0].min())[-16:]  # the last cycle's appends
t0 = tr[launches[0], :, 0].min()
names = {0: "resident", 8: "waited", 1: "ticket", 2: "meta", 3: "lookback", 4: "pre-score", 5: "scored", 9: "end"}
prev_end = None
for e in launches:
    x = tr[e]
    row = {n: (int(np.median(x[:, i])) - t0) / 1000 for i, n in names.items()}
    first_res, last_end = (x[:, 0].min() - t0) / 1000, (x[:, 9].max() - t0) / 1000
    wait_min = (x[:, 8].min() - t0) / 1000
    gap = None if prev_end is None else wait_min - prev_end
    print(f"epoch {e:2d}: resident {first_res:8.2f}  released {wait_min:8.2f}  "
          + "  ".join(f"{n} {v:8.2f}" for n, v in row.items() if n not in ('resident',))
          + f"  last end {last_end:8.2f}  gap-after-prev-end {gap if gap is None else round(gap, 2)}")
    prev_end = last_end
spans = [(tr[e, :, 9].max() - tr[e, :, 8].min()) / 1000 for e in launches]
print("span (release -> last end) median us:", statistics.median(spans))

# phase durations across CTAs (last 15 launches), percentiles in us
ph = {"wait->ticket": (8, 1), "ticket->meta": (1, 2), "meta->lookback": (2, 3), "lookback->prescore": (3, 4),
      "prescore->scored": (4, 5), "scored->end": (5, 9), "release->end": (8, 9)}
for name, (a, b) in ph.items():
    v = np.concatenate([(tr[e, :, b] - tr[e, :, a]) / 1000 for e in launches[1:]])
    print(f"{name:20s} p10 {np.percentile(v, 10):6.2f} p50 {np.percentile(v, 50):6.2f} p90 {np.percentile(v, 90):6.2f} "
          f"p99 {np.percentile(v, 99):6.2f} max {v.max():6.2f}")
rel = np.concatenate([(tr[e, :, 8] - tr[e, :, 8].min()) / 1000 for e in launches[1:]])
print(f"release skew across CTAs: p50 {np.percentile(rel, 50):.2f} p99 {np.percentile(rel, 99):.2f} max {rel.max():.2f}")
