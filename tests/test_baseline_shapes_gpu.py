"""Parity at the BASELINE.json configurations' own shapes, and at the
reference's own table granularity (PER_LAYER).

Every check compares the CUDA engine (through the C-ABI) with the
UNMODIFIED reference (oracle/_ref: PagePool / BlockTable /
make_policy(PagedEviction) / attend) or with the pinned C restatement, on the
same bytes:

* PER_LAYER (kv_vector.hpp:23-27, simulator.cpp:105-108): one table per
  (sequence, layer), rows of all KV heads side by side (w = H*d = 1024 bf16,
  512 fp32); prefill (K1), decode append + block eviction (K0, K2, K2c) and
  the GQA attention (K3) slicing head h's columns.
* cfg2 (Llama-3.2-3B geometry, 32 x 16K, C=2048) at full size for one
  layer: G=3 attention (24 query heads over 8 KV heads).
* cfg5 (Llama-3.1-8B geometry at 128K context, C=4096): tables of 131 072
  tokens through the streamed long-table select, on Gaussian and on the
  tie-heavy lattice data, every table bit-exact against the oracle.
* cfg4 (mixed-length serving trace): 256 sequences of log-uniform lengths in
  [1K, 64K] in one shared pool, continuous eviction with K3 every step: the
  eviction cadence of every table against the trigger rule
  (policy.cpp:147-150), the device invariant checker, and sampled tables
  replayed through the reference (survivors, every victim, attention).
"""
import numpy as np
import pytest

import oracle
from tests.harness import RefReplay, compare_states_vectorized, compare_with_reference, grid_kv, oracle_state, \
    random_kv

torch = pytest.importorskip("torch")
pe = pytest.importorskip("paper_2509_04377_b200")

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def to_f32(a):
    """bf16 bits (uint16) or float32 numpy -> float32."""
    return oracle.bf16_bits_to_f32(a) if a.dtype == np.uint16 else a


def bf16_randn(shape, gen):
    return torch.randn(shape, generator=gen, device="cuda", dtype=torch.float32).to(torch.bfloat16)


def t_f32(x):
    return x.float().cpu().numpy()


def ref_gqa_attend(sess, t, q_heads, H, G, d):
    """The reference's attend over a PER_LAYER table for GQA: for each group
    member g one MHA call over the H heads of the concatenated row, the query
    row being q[h*G + g] for h = 0..H-1 (attention.cpp:23-35 slices head h's
    columns). Returns [H*G, d]."""
    out = np.zeros((H * G, d), np.float32)
    for g in range(G):
        qg = np.concatenate([q_heads[h * G + g] for h in range(H)])
        o = sess.attend(t, qg, H, d).reshape(H, d)
        for h in range(H):
            out[h * G + g] = o[h]
    return out


# ----------------------------------------------------------------- PER_LAYER
@pytest.mark.parametrize("dtype,d,tol", [(oracle.BF16, 128, 1e-3), (oracle.F32, 64, 1e-5)])
@pytest.mark.parametrize("mode", [0, 1])
def test_per_layer_batched_against_reference(reference, dtype, d, tol, mode):
    """Batched PagedEviction at the reference's PER_LAYER granularity, w = 8
    heads x d, through K1 / K0 / K2 (or K2c) / K3 against RefReplay (the
    reference objects driven in the engine's canonical order)."""
    rng = np.random.default_rng(1024 + dtype + 10 * mode)
    H, G, B, C, n_layers = 8, 4, 16, 128, 2
    lens = np.array([600, 90, 129, 1000])
    S = len(lens)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    geo = pe.EngineGeometry(n_seqs=S, n_layers=n_layers, n_kv_heads=H, head_dim=d, dtype=dtype,
                            granularity=pe.Granularity.PER_LAYER)
    eng = pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=C, page_size=B))
    assert eng.width == H * d and eng.n_tables == S * n_layers
    rep = RefReplay(reference, n_seqs=S, n_layers=n_layers, n_tab_heads=1, width=H * d, page_size=B,
                    budget=C, capacity=eng.capacity)
    for layer in range(n_layers):
        k, k32 = (random_kv if layer == 0 else grid_kv)(rng, (cu[-1], H, d), dtype)
        v, v32 = random_kv(rng, (cu[-1], H, d), dtype)
        ev = eng.prefill_compress(layer, dev(k), dev(v), cu, evicted_counts=True)
        out = rep.prefill(layer, k32.reshape(-1, 1, H * d), v32.reshape(-1, 1, H * d), cu)
        np.testing.assert_array_equal(ev, [len(x) for x in out])
    pos = lens.astype(np.int64).copy()
    for step in range(1, 2 * B + 5):
        k, k32 = random_kv(rng, (n_layers, S, H, d), dtype)
        v, v32 = random_kv(rng, (n_layers, S, H, d), dtype)
        vic = eng.decode_step(0, n_layers, dev(k), dev(v), dev(pos), step, mode=mode, victims=True)
        want = rep.decode(0, n_layers, k32.reshape(n_layers, S, 1, H * d), v32.reshape(n_layers, S, 1, H * d),
                          pos, step)
        np.testing.assert_array_equal(vic, want, err_msg=f"step {step}")
        pos += 1
        if step % B == 0 or step == 2 * B + 4:
            q, q32 = random_kv(rng, (S, H * G, d), dtype)
            for layer in range(n_layers):
                o = torch.empty((S, H * G, d), dtype=torch.float32, device="cuda")
                eng.attend(layer, dev(q), o, H * G)
                got = o.cpu().numpy()
                for sq in range(S):
                    ref = ref_gqa_attend(rep.sess, rep.tid(sq, layer, 0), q32[sq], H, G, d)
                    for hq in range(H * G):
                        dv = oracle.Oracle().output_deviation(got[sq, hq], ref[hq])
                        assert dv <= tol, (step, layer, sq, hq, dv)
    eng.sync()
    assert eng.stats().pages_evicted > 0
    compare_with_reference(rep, eng.state())
    assert eng.check_invariants()["violations"] == 0


# ----------------------------------------------------------------- cfg2 (G = 3)
@pytest.mark.slow
def test_cfg2_full_layer_g3_sampled_against_reference(reference):
    """BASELINE config 2 at full size for one layer — Llama-3.2-3B KV geometry
    (8 KV heads, d=128, 24 query heads: G=3), 32 sequences x 16 384 tokens,
    C=2048, B=16, bf16 — prefill, 16 decode tokens (one block eviction per
    table), GQA attention. Eight sampled tables are replayed through the
    reference on the same bytes (survivors, every decision, attention <=
    1e-3); every table's eviction and the device invariants are checked."""
    S, H, d, L, C, B, G = 32, 8, 128, 16384, 2048, 16, 3
    geo = pe.EngineGeometry(n_seqs=S, n_layers=1, n_kv_heads=H, head_dim=d, dtype=oracle.BF16)
    eng = pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=C, page_size=B))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(2)
    k_in, v_in = bf16_randn((S * L, H, d), gen), bf16_randn((S * L, H, d), gen)
    cu = np.arange(S + 1, dtype=np.int32) * L
    eng.prefill_compress(0, k_in, v_in, cu)
    eng.sync()
    samples = [(0, 0), (5, 3), (11, 7), (17, 1), (20, 4), (26, 6), (30, 2), (31, 5)]
    ref = {}
    for sq, h in samples:
        sess = oracle.RefSession(reference, capacity=C // B + 2, page_size=B, budget=C, n_tables=1, width=d,
                                 kind=0)
        sess.prefill(0, t_f32(k_in[sq * L:(sq + 1) * L, h]), t_f32(v_in[sq * L:(sq + 1) * L, h]))
        ref[(sq, h)] = sess
        np.testing.assert_array_equal(eng.retained_positions(sq * H + h), sess.read_table(0, False)["positions"])
    del k_in, v_in
    torch.cuda.empty_cache()
    pos = torch.full((S,), L, dtype=torch.int64, device="cuda")
    for step in range(1, B + 1):
        rk, rv = bf16_randn((1, S, H, d), gen), bf16_randn((1, S, H, d), gen)
        vic = eng.decode_step(0, 1, rk, rv, pos, step, victims=True)
        for (sq, h), sess in ref.items():
            kind, idx = sess.decode_step(0, t_f32(rk[0, sq, h]), t_f32(rv[0, sq, h]), L + step - 1, step)
            assert int(vic[sq * H + h]) == (idx if kind == 2 else -1), (step, sq, h)
        # the trigger fires exactly once per table, on the 16th token
        assert np.all(vic == -1) if step < B else np.all(vic >= 0)
        pos += 1
    eng.sync()
    assert eng.stats().pages_evicted == S * H
    assert eng.check_invariants()["violations"] == 0
    q = bf16_randn((S, H * G, d), gen)
    out = torch.empty((S, H * G, d), dtype=torch.float32, device="cuda")
    eng.attend(0, q, out, H * G)
    qf, of = t_f32(q), out.cpu().numpy()
    o = oracle.Oracle()
    for (sq, h), sess in ref.items():
        np.testing.assert_array_equal(eng.retained_positions(sq * H + h), sess.read_table(0, False)["positions"])
        for g in range(G):
            want = sess.attend(0, qf[sq, h * G + g], 1, d)
            assert o.output_deviation(of[sq, h * G + g], want) <= 1e-3, (sq, h, g)


# ----------------------------------------------------------------- cfg5 (128K)
@pytest.mark.slow
@pytest.mark.parametrize("gen", [random_kv, grid_kv])
def test_cfg5_128k_tables_against_oracle(gen):
    """BASELINE config 5's table length: 2 sequences x 8 KV heads at
    L = 131 072 tokens, C = 4096 (rank_tokens with k = 126 976,
    importance.cpp:41-60) through the streamed long-table select; Gaussian
    and tie-heavy lattice keys. Evicted counts, block tables, positions and
    page bytes bit-exact against the oracle, then one eviction cycle."""
    rng = np.random.default_rng(131072)
    S, H, d, L, C, B = 2, 8, 128, 131072, 4096, 16
    geo = pe.EngineGeometry(n_seqs=S, n_layers=1, n_kv_heads=H, head_dim=d, dtype=oracle.BF16)
    eng = pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=C, page_size=B))
    orc = oracle.OracleEngine(n_seqs=S, n_layers=1, n_tab_heads=H, width=d, page_size=B, budget=C,
                              dtype=oracle.BF16, capacity=eng.capacity, max_pages=eng.max_pages)
    cu = np.arange(S + 1, dtype=np.int32) * L
    k, _ = gen(rng, (S * L, H, d), oracle.BF16)
    v, _ = random_kv(rng, (S * L, H, d), oracle.BF16)
    ev = eng.prefill_compress(0, dev(k), dev(v), cu, evicted_counts=True)
    st, oev = orc.prefill(0, k, v, cu)
    assert st == 0
    np.testing.assert_array_equal(ev, oev)
    assert np.all(ev == L - C)
    eng.sync()
    compare_states_vectorized(eng.state(), oracle_state(orc), B, what="cfg5 prefill: ")
    pos = np.full(S, L, np.int64)
    for step in range(1, B + 1):
        kk, _ = random_kv(rng, (1, S, H, d), oracle.BF16)
        vv, _ = random_kv(rng, (1, S, H, d), oracle.BF16)
        vic = eng.decode_step(0, 1, dev(kk), dev(vv), dev(pos), step, victims=True)
        orc.decode_append(0, 1, kk, vv, pos)
        _, ovic = orc.decode_evict(0, 1)
        np.testing.assert_array_equal(vic, ovic)
        pos += 1
    eng.sync()
    compare_states_vectorized(eng.state(), oracle_state(orc), B, what="cfg5 decode: ")


# ----------------------------------------------------------------- cfg4 (mixed trace)
def trigger_sim(num_pages, fill, retained, B, C):
    """One decode step of every table on counts only: append_token
    (block_table.cpp:10-19) then the PagedEviction trigger
    (policy.cpp:147-150) and free_page's bookkeeping. Returns the trigger mask."""
    pop = (num_pages == 0) | (fill == B)
    num_pages += pop
    fill[:] = np.where(pop, 1, fill + 1)
    retained += 1
    trig = (fill == B) & (retained > C)
    num_pages -= trig
    retained -= B * trig
    fill[:] = np.where(trig, np.where(num_pages > 0, B, 0), fill)
    return trig


@pytest.mark.slow
def test_cfg4_mixed_trace_shared_pool(reference):
    """BASELINE config 4: 256 concurrent sequences, lengths log-uniform in
    [1024, 65536] (seeded), 8B geometry (8 KV heads, d=128, G=4), C=4096,
    one shared pool for all 2048 tables of the layer; 48 decode steps with
    continuous block eviction and the paged attention every step. Checks:
    every table's eviction cadence equals the trigger rule, the device
    invariants (pages mapped + free == capacity), and 8 sampled tables
    (short identity-prefill ones and long ones) replayed through the
    reference: survivors, every victim, attention <= 1e-3."""
    S, H, d, C, B, G, steps = 256, 8, 128, 4096, 16, 4, 48
    rng = np.random.default_rng(4)
    lens = np.exp(rng.uniform(np.log(1024), np.log(65536), size=S)).astype(np.int64)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    geo = pe.EngineGeometry(n_seqs=S, n_layers=1, n_kv_heads=H, head_dim=d, dtype=oracle.BF16)
    eng = pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=C, page_size=B))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(44)
    k_in, v_in = bf16_randn((int(cu[-1]), H, d), gen), bf16_randn((int(cu[-1]), H, d), gen)
    ev = eng.prefill_compress(0, k_in, v_in, cu, evicted_counts=True)
    np.testing.assert_array_equal(ev, np.repeat(np.maximum(lens - C, 0), H))
    order = np.argsort(lens)
    pick = [order[0], order[1], order[S // 4], order[S // 2], order[3 * S // 4], order[-2], order[-1],
            int(np.argmin(np.abs(lens - C)))]
    samples = [(int(sq), int(sq * 5 + 3) % H) for sq in pick]
    ref = {}
    for sq, h in samples:
        sess = oracle.RefSession(reference, capacity=C // B + 2, page_size=B, budget=C, n_tables=1, width=d,
                                 kind=0)
        a, b = int(cu[sq]), int(cu[sq + 1])
        sess.prefill(0, t_f32(k_in[a:b, h]), t_f32(v_in[a:b, h]))
        ref[(sq, h)] = sess
        np.testing.assert_array_equal(eng.retained_positions(sq * H + h), sess.read_table(0, False)["positions"])
    del k_in, v_in
    torch.cuda.empty_cache()
    _, npg, nf, rt = eng.tables()
    npg, nf, rt = npg.astype(np.int64), nf.astype(np.int64), rt.astype(np.int64)
    pos = torch.from_numpy(lens.copy()).cuda()
    o = oracle.Oracle()
    for step in range(1, steps + 1):
        rk, rv = bf16_randn((1, S, H, d), gen), bf16_randn((1, S, H, d), gen)
        vic = eng.decode_step(0, 1, rk, rv, pos, step, victims=True)
        want = trigger_sim(npg, nf, rt, B, C)
        np.testing.assert_array_equal(vic >= 0, want, err_msg=f"cadence, step {step}")
        for (sq, h), sess in ref.items():
            kind, idx = sess.decode_step(0, t_f32(rk[0, sq, h]), t_f32(rv[0, sq, h]), int(lens[sq]) + step - 1,
                                         step)
            assert int(vic[sq * H + h]) == (idx if kind == 2 else -1), (step, sq, h)
        q = bf16_randn((S, H * G, d), gen)
        out = torch.empty((S, H * G, d), dtype=torch.float32, device="cuda")
        eng.attend(0, q, out, H * G)
        if step % 8 == 0:
            qf, of = t_f32(q), out.cpu().numpy()
            for (sq, h), sess in ref.items():
                for g in range(G):
                    want_o = sess.attend(0, qf[sq, h * G + g], 1, d)
                    assert o.output_deviation(of[sq, h * G + g], want_o) <= 1e-3, (step, sq, h, g)
        pos += 1
    eng.sync()
    _, npg2, nf2, rt2 = eng.tables()
    np.testing.assert_array_equal(npg2, npg)
    np.testing.assert_array_equal(rt2, rt)
    inv = eng.check_invariants()
    assert inv["violations"] == 0, inv
    assert inv["pages_mapped"] + inv["free_pages"] == eng.capacity
    for (sq, h), sess in ref.items():
        np.testing.assert_array_equal(eng.retained_positions(sq * H + h), sess.read_table(0, False)["positions"])


def test_prefill_longer_than_the_cluster_shared_memory():
    """A 200 000-token prompt (beyond what the cluster select's shared memory
    holds) goes through the streamed select: accepted and bit-exact."""
    rng = np.random.default_rng(200000)
    L, C, B, d = 200000, 4096, 16, 128
    geo = pe.EngineGeometry(n_seqs=1, n_layers=1, n_kv_heads=1, head_dim=d, dtype=oracle.BF16)
    eng = pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=C, page_size=B))
    orc = oracle.OracleEngine(n_seqs=1, n_layers=1, n_tab_heads=1, width=d, page_size=B, budget=C,
                              dtype=oracle.BF16, capacity=eng.capacity, max_pages=eng.max_pages)
    k, _ = random_kv(rng, (L, 1, d), oracle.BF16)
    v, _ = random_kv(rng, (L, 1, d), oracle.BF16)
    cu = np.array([0, L], np.int32)
    ev = eng.prefill_compress(0, dev(k), dev(v), cu, evicted_counts=True)
    _, oev = orc.prefill(0, k, v, cu)
    np.testing.assert_array_equal(ev, oev)
    compare_states_vectorized(eng.state(), oracle_state(orc), B, what="200K prefill: ")
