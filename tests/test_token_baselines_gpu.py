"""Batched unstructured baselines on the device: the
StreamingLLM / InvKeyL2 / KeyDiff decode step over every table of a layer
range in one launch (pe_decode_evict_tokens), against the reference's own
policy objects driven in the engine's canonical batched order — all of a
step's appends (ascending table id), then all evictions (ascending table id)
— through oracle/ref_harness.cpp's two-phase calls.

Bit-exact: the evicted position of every table at every step, page ids in
logical order, retained positions (holes skipped), retained lengths, and the
free list (drained at the end). The paper's cadence comparison
(acceptance_main.cpp:208-241): a token baseline updates the block table every
step once over budget, PagedEviction every B steps, ratio B.
"""
import numpy as np
import pytest

import oracle
from tests.harness import grid_kv, random_kv

torch = pytest.importorskip("torch")
pe = pytest.importorskip("paper_2509_04377_b200")

pytestmark = pytest.mark.gpu

KIND = {pe.TokenRule.STREAMING: 1, pe.TokenRule.MAX_KEY_NORM: 2, pe.TokenRule.KEY_DIFF: 3}
SINKS = 4  # PolicyConfig::sink_count default (policy.hpp:31-39), the harness sessions' value


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def engine_retained(eng, holes, t, bt, npg, nf, pos):
    out = []
    for j in range(int(npg[t])):
        pid = int(bt[t, j])
        cursor = eng.B if j < npg[t] - 1 else int(nf[t])
        for sl in range(cursor):
            if not (int(holes[pid]) >> sl) & 1:
                out.append(int(pos[pid, sl]))
    return out


@pytest.mark.parametrize("rule", [pe.TokenRule.STREAMING, pe.TokenRule.MAX_KEY_NORM, pe.TokenRule.KEY_DIFF])
@pytest.mark.parametrize("dtype,gran", [(oracle.F32, 0), (oracle.BF16, 0), (oracle.BF16, 1)])
def test_batched_token_eviction_matches_reference(reference, rule, dtype, gran):
    """gran 1: PER_LAYER tables (one table per (sequence, layer), rows of all
    KV heads, width H*d)."""
    rng = np.random.default_rng(100 + int(rule) * 7 + dtype + 31 * gran)
    B, C, d, Hkv, S, NL = 8, 32, 16, 2, 3, 2
    H, w = (1, Hkv * d) if gran else (Hkv, d)  # table heads, table row width
    lens = np.array([C, 5, C - 9])  # identity prefill (L <= C) for every policy
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    geo = pe.EngineGeometry(n_seqs=S, n_layers=NL, n_kv_heads=Hkv, head_dim=d, dtype=dtype,
                            granularity=pe.Granularity(gran), max_pages_per_table=C // B + 8)
    # the batched baselines run on a FullCache-kind engine (identity prefill,
    # no PagedEviction trigger); the budget C drives pe_decode_evict_tokens
    eng = pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=C, page_size=B,
                                                      kind=pe.PolicyKind.FullCache))
    sess = reference.session(eng.capacity, B, C, eng.n_tables, w, KIND[rule])
    tid = lambda s, l, h: (s * NL + l) * H + h  # noqa: E731
    for layer in range(NL):
        k, k32 = random_kv(rng, (cu[-1], H, w), dtype)
        v, v32 = random_kv(rng, (cu[-1], H, w), dtype)
        eng.prefill_compress(layer, dev(k), dev(v), cu)
        for s in range(S):
            for h in range(H):
                ev = sess.prefill(tid(s, layer, h), k32[cu[s]:cu[s + 1], h], v32[cu[s]:cu[s + 1], h])
                assert len(ev) == 0
    pos = lens.astype(np.int64).copy()
    updates = 0
    for step in range(1, 3 * B + 6):
        gen = grid_kv if step % 3 == 0 else random_kv  # ties in ||K|| and cosine
        k, k32 = gen(rng, (NL, S, H, w), dtype)
        v, v32 = random_kv(rng, (NL, S, H, w), dtype)
        eng.append_token(0, NL, dev(k), dev(v), dev(pos))
        vic = eng.evict_tokens(0, NL, rule, SINKS, dev(pos), victims=True)
        order = [(s, li, h) for s in range(S) for li in range(NL) for h in range(H)]
        for s, li, h in order:  # phase 1: appends, ascending table id
            sess.append_token(tid(s, li, h), k32[li, s, h], v32[li, s, h], pos[s])
        want = []
        for s, li, h in order:  # phase 2: evictions, ascending table id
            kind, victim = sess.policy_evict(tid(s, li, h), pos[s], step)
            want.append(victim if kind == 1 else -1)
        np.testing.assert_array_equal(vic, np.array(want, dtype=np.int64), err_msg=f"step {step}")
        updates += int((vic >= 0).sum())
        pos += 1
        eng.sync()
        bt, npg, nf, rt = eng.tables()
        holes = eng.page_holes()
        positions = eng.positions()
        for t in range(eng.n_tables):
            r = sess.read_table(t, with_data=False)
            np.testing.assert_array_equal(bt[t, :npg[t]], r["phys"], err_msg=f"step {step} table {t} pages")
            assert int(rt[t]) == len(r["positions"])
            assert engine_retained(eng, holes, t, bt, npg, nf, positions) == r["positions"].tolist(), \
                f"step {step} table {t}"
    assert updates > 0
    np.testing.assert_array_equal(sess.drain_free_list(check_mirror=False), eng.free_list()[::-1])
    assert eng.check_invariants()["page_refcount"] == 0


def test_cadence_ratio_is_page_size():
    """acceptance_main.cpp:208-241 at GPU scale: over the same decode run the
    StreamingLLM engine updates block tables B times as often as the
    PagedEviction engine (one update per step vs one per B steps, once over
    budget)."""
    rng = np.random.default_rng(3)
    B, C, d, H, S, NL = 16, 64, 32, 4, 8, 4
    L = C
    cu = np.arange(S + 1, dtype=np.int32) * L
    counts = {}
    for kind in (0, 1):
        geo = pe.EngineGeometry(n_seqs=S, n_layers=NL, n_kv_heads=H, head_dim=d, dtype=oracle.BF16,
                                max_pages_per_table=C // B + 8)
        eng = pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=C, page_size=B,
                                                          kind=pe.PolicyKind(0 if kind == 0 else 4)))
        r2 = np.random.default_rng(5)
        for layer in range(NL):
            k, _ = random_kv(r2, (cu[-1], H, d), oracle.BF16)
            v, _ = random_kv(r2, (cu[-1], H, d), oracle.BF16)
            eng.prefill_compress(layer, dev(k), dev(v), cu)
        pos = np.full(S, L, dtype=np.int64)
        n_upd = 0
        for step in range(1, 4 * B + 1):
            k, _ = random_kv(r2, (NL, S, H, d), oracle.BF16)
            v, _ = random_kv(r2, (NL, S, H, d), oracle.BF16)
            eng.append_token(0, NL, dev(k), dev(v), dev(pos))
            if kind == 0:
                vic = eng.evict(0, NL, step=step, victims=True)
            else:
                vic = eng.evict_tokens(0, NL, pe.TokenRule.STREAMING, SINKS, dev(pos), victims=True)
            n_upd += int((vic >= 0).sum())
            pos += 1
        counts[kind] = n_upd
        assert eng.check_invariants()["violations"] == 0
    assert counts[0] > 0 and counts[1] == B * counts[0], counts
