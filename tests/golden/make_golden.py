"""Generates the golden fixtures in this directory FROM THE REFERENCE ITSELF
(oracle/_ref/libpagedevict_ref.so, compiled from /root/reference/proj/core by
oracle/Makefile). Run in the dev container:

    python tests/golden/make_golden.py

Fixtures (small, committed):
  scores.npz  per-row K/V inputs (fp32 values, bf16-exact) and the
              reference's token_importance (kv_vector.hpp:36-48,
              importance.cpp:11-13) as uint64 bit patterns; includes zero rows
              and lattice rows (fallback path of the exact scorer).
  trace.npz   an engine-shaped trace (2 seqs x 2 layers x 2 KV heads, w=16,
              B=8, C=32, mixed prompt lengths incl. an identity prefill),
              driven through the reference's PagePool / BlockTable /
              make_policy(PagedEviction) in the canonical order: prefill
              evicted counts, per-step decode victims, final block tables
              (physical ids), retained positions, the free list (drained
              from the reference pool), and attend outputs for a GQA query.
All input values are bf16-representable, so the same fixture checks an
engine run in fp32 and in bf16.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from tests.harness import RefReplay  # noqa: E402

OUT = Path(__file__).resolve().parent


def bf16_exact(x):
    return oracle.bf16_bits_to_f32(oracle.f32_to_bf16_bits(x))


def make_scores(ref):
    rng = np.random.default_rng(20250904)
    rows = []
    for w in (8, 16, 64, 128):
        for _ in range(24):
            rows.append((w, bf16_exact(rng.standard_normal(w).astype(np.float32)),
                         bf16_exact(rng.standard_normal(w).astype(np.float32))))
        lat = (rng.integers(-3, 4, size=(4, w)) / 8.0).astype(np.float32)  # zeros + ties
        rows.append((w, lat[0], lat[1]))
        rows.append((w, np.zeros(w, np.float32), lat[2]))                 # zero key -> eps guard
        rows.append((w, lat[3], np.zeros(w, np.float32)))                 # zero value -> S = 0
        tiny = bf16_exact((rng.standard_normal(w) * 1e-30).astype(np.float32))
        rows.append((w, tiny, bf16_exact(rng.standard_normal(w).astype(np.float32))))
    out = {}
    for i, (w, k, v) in enumerate(rows):
        out[f"k{i}"] = k
        out[f"v{i}"] = v
        out[f"s{i}"] = np.array([ref.token_importance(k, v)], np.float64).view(np.uint64)
    out["n"] = np.array([len(rows)])
    np.savez_compressed(OUT / "scores.npz", **out)


def make_trace(ref):
    rng = np.random.default_rng(2509)
    S, NL, H, w, B, C, G = 2, 2, 2, 16, 8, 32, 2
    lens = np.array([70, 20])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    cap = S * NL * H * (C // B + 1) + 5
    rep = RefReplay(ref, n_seqs=S, n_layers=NL, n_tab_heads=H, width=w, page_size=B, budget=C,
                    capacity=cap)
    data = dict(S=S, NL=NL, H=H, w=w, B=B, C=C, G=G, cap=cap, cu=cu)
    for layer in range(NL):
        k = bf16_exact(rng.standard_normal((cu[-1], H, w)).astype(np.float32))
        v = bf16_exact(rng.standard_normal((cu[-1], H, w)).astype(np.float32))
        ev = rep.prefill(layer, k, v, cu)
        data[f"pk{layer}"], data[f"pv{layer}"] = k, v
        data[f"pev{layer}"] = np.array([len(e) for e in ev], np.int32)
    steps = 3 * B + 2
    pos = lens.astype(np.int64).copy()
    dk = bf16_exact(rng.standard_normal((steps, NL, S, H, w)).astype(np.float32))
    dv = bf16_exact(rng.standard_normal((steps, NL, S, H, w)).astype(np.float32))
    vic = np.zeros((steps, NL * S * H), np.int32)
    for st in range(steps):
        vic[st] = rep.decode(0, NL, dk[st], dv[st], pos, st + 1)
        pos += 1
    data.update(dk=dk, dv=dv, victims=vic)
    n = rep.n_tables
    phys = np.full((n, C // B + 1), -1, np.int32)
    npg = np.zeros(n, np.int32)
    retained = []
    for t in range(n):
        r = rep.sess.read_table(t, with_data=False)
        npg[t] = len(r["phys"])
        phys[t, : npg[t]] = r["phys"]
        retained.append(r["positions"])
    data.update(phys=phys, num_pages=npg,
                retained_len=np.array([len(r) for r in retained], np.int32),
                retained=np.concatenate(retained).astype(np.int64))
    q = bf16_exact(rng.standard_normal((S, H * G, w)).astype(np.float32))
    data["q"] = q
    data["attn"] = np.stack([rep.attend(layer, q, G) for layer in range(NL)])
    data["free_list"] = rep.sess.mirror_free_list()
    data["drain"] = rep.sess.drain_free_list()
    np.savez_compressed(OUT / "trace.npz", **data)


if __name__ == "__main__":
    r = oracle.Reference()
    make_scores(r)
    make_trace(r)
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))
