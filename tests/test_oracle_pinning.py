"""Pins the C restatement (oracle/pe_oracle.c) to the REAL reference library
(oracle/_ref, compiled from /root/reference/proj/core) — CPU only.

Known answers are the reference's own unit-test pins
(proj/tests/test_importance.cpp, test_paged_store.cpp, test_policies.cpp,
test_attention.cpp); randomized cases compare the restatement and the
reference bit for bit.
"""
import numpy as np
import pytest

import oracle
from tests.harness import RefReplay, compare_with_reference, grid_kv, oracle_state, random_kv

# ----------------------------------------------------------------- known answers


def test_score_known_answers(oracle_lib, reference):
    # test_importance.cpp:13-22
    k = np.array([1, 0, 0], np.float32)
    v = np.array([0, 2, 0], np.float32)
    assert oracle_lib.token_score(k, v) == 2.0 == reference.token_importance(k, v)
    k = np.array([0.5, -1.5], np.float32)
    assert oracle_lib.token_score(k, k) == 1.0 == reference.token_importance(k, k)
    # zero key: eps-guarded, >= 1e11 (test_importance.cpp:24-29)
    z = np.zeros(2, np.float32)
    s = oracle_lib.token_score(z, np.array([1, 0], np.float32))
    assert np.isfinite(s) and s >= 1e11
    assert s == reference.token_importance(z, np.array([1, 0], np.float32))


def test_rank_tokens_known_answers(oracle_lib, reference):
    # test_importance.cpp:87-96
    pos = [0, 1, 2]
    assert list(oracle_lib.rank_tokens(pos, [3.0, 1.0, 2.0], 1)) == [1]
    assert list(oracle_lib.rank_tokens(pos, [1.0, 1.0, 1.0], 2)) == [0, 1]
    assert oracle_lib.rank_tokens(pos, [3.0, 1.0, 2.0], 0).size == 0
    with pytest.raises(oracle.KTooLarge):
        oracle_lib.rank_tokens(pos, [3.0, 1.0, 2.0], 4)
    with pytest.raises(oracle.RefError):
        reference.rank_tokens(pos, [3.0, 1.0, 2.0], 4)


def test_rank_pages_known_answers(oracle_lib, reference):
    # ties break toward the smaller logical index (importance.cpp:66-72)
    for sc in ([2.0, 1.0, 1.0, 3.0], [1.0, 1.0], [5.0], [0.5, 0.25, 0.25, 0.125, 0.125]):
        assert oracle_lib.rank_pages(sc) == reference.rank_pages(sc)
    assert oracle_lib.rank_pages([2.0, 1.0, 1.0, 3.0]) == 1
    with pytest.raises(oracle.NoEligiblePage):
        oracle_lib.rank_pages([])


# ----------------------------------------------------------------- randomized pins


@pytest.mark.parametrize("dtype", [oracle.F32, oracle.BF16])
@pytest.mark.parametrize("w", [1, 8, 40, 64, 128])
def test_token_scores_bit_exact(oracle_lib, reference, dtype, w):
    rng = np.random.default_rng(11 + w)
    for _ in range(50):
        k, k32 = random_kv(rng, (w,), dtype)
        v, v32 = random_kv(rng, (w,), dtype)
        a = oracle_lib.token_score(k, v)
        b = reference.token_importance(k32, v32)
        assert a == b  # bit-exact double
        assert oracle_lib.l2_norm(k) == reference.l2_norm(k32)


def test_rank_tokens_matches_reference_with_ties(oracle_lib, reference):
    rng = np.random.default_rng(21)
    for n in (1, 7, 64, 513):
        sc = np.round(rng.uniform(0, 2, n) * 8) / 8  # quantized: many ties
        pos = rng.permutation(n)
        for k in {0, 1, n // 3, n - 1, n}:
            np.testing.assert_array_equal(oracle_lib.rank_tokens(pos, sc, k),
                                          reference.rank_tokens(pos, sc, k))


def test_attend_matches_reference(oracle_lib, reference):
    rng = np.random.default_rng(31)
    for n in (1, 5, 48, 300):
        d = 16
        keys = rng.standard_normal((n, d), dtype=np.float32)
        vals = rng.standard_normal((n, d), dtype=np.float32)
        q = rng.standard_normal(d, dtype=np.float32)
        a = oracle_lib.attend_dense(q, keys, vals)
        b = reference.attend_dense(keys, vals, q, 1, d)
        np.testing.assert_array_equal(a, b)
    # single token returns its value exactly (test_attention.cpp:12-19)
    out = oracle_lib.attend_dense(np.ones(2, np.float32), np.array([[0.3, -0.7]], np.float32),
                                  np.array([[4.0, 3.0]], np.float32))
    np.testing.assert_array_equal(out, [4.0, 3.0])


def test_output_deviation(oracle_lib, reference):
    a = np.array([1, 2, -3], np.float32)
    assert oracle_lib.output_deviation(a, a) == 0.0
    assert oracle_lib.output_deviation(2 * a, a) == pytest.approx(1.0)
    assert oracle_lib.output_deviation(2 * a, a) == reference.output_deviation(2 * a, a)


def test_config_validation_matches_reference(reference):
    # policy.cpp:38-52 / test_policies.cpp:56-65
    assert reference.validate_config(1000, 16) == 9
    assert reference.validate_config(8, 16) == 9
    assert reference.validate_config(256, 16) == 0
    eng_args = dict(n_seqs=1, n_layers=1, n_tab_heads=1, width=4, dtype=oracle.F32,
                    capacity=4, max_pages=4)
    for C, B, ok in ((1000, 16, False), (8, 16, False), (256, 16, True), (16, 16, True)):
        if ok:
            oracle.OracleEngine(page_size=B, budget=C, **eng_args)
        else:
            with pytest.raises(oracle.OracleError):
                oracle.OracleEngine(page_size=B, budget=C, **eng_args)


# ----------------------------------------------------------------- engine replay


def _engine_pair(reference, *, n_seqs, n_layers, H, w, B, C, cap, max_pages, dtype,
                 kind=oracle.PAGED_EVICTION):
    eng = oracle.OracleEngine(n_seqs=n_seqs, n_layers=n_layers, n_tab_heads=H, width=w,
                              page_size=B, budget=C, dtype=dtype, capacity=cap,
                              max_pages=max_pages, policy=kind)
    rep = RefReplay(reference, n_seqs=n_seqs, n_layers=n_layers, n_tab_heads=H, width=w,
                    page_size=B, budget=C, capacity=cap, kind=kind)
    return eng, rep


@pytest.mark.parametrize("dtype", [oracle.F32, oracle.BF16])
@pytest.mark.parametrize("gen", [random_kv, grid_kv])
@pytest.mark.parametrize("B,C", [(16, 64), (4, 16), (8, 40)])
def test_engine_replay_matches_reference(reference, dtype, gen, B, C):
    """Mixed-length prefill (identity L<=C and pruned L>C), then decode steps
    with appends, page evictions and free-list reuse, all layers in one
    decode launch and also per-layer launches."""
    rng = np.random.default_rng(B * 1000 + C + dtype)
    n_seqs, n_layers, H, w = 3, 2, 2, 8
    lens = np.array([C + 3 * B + 5, max(1, C - 3), 2 * C + 1])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    max_pages = C // B + 1
    cap = n_seqs * n_layers * H * max_pages + 3
    eng, rep = _engine_pair(reference, n_seqs=n_seqs, n_layers=n_layers, H=H, w=w, B=B, C=C,
                            cap=cap, max_pages=max_pages, dtype=dtype)
    for layer in range(n_layers):
        k, k32 = gen(rng, (cu[-1], H, w), dtype)
        v, v32 = gen(rng, (cu[-1], H, w), dtype)
        st, ev = eng.prefill(layer, k, v, cu)
        assert st == 0
        ref_ev = rep.prefill(layer, k32, v32, cu)
        assert [len(x) for x in ref_ev] == list(ev)
    compare_with_reference(rep, oracle_state(eng))
    pos = lens.copy()
    for step in range(1, 3 * B + 3):
        per_layer = step % 2 == 0
        k, k32 = gen(rng, (n_layers, n_seqs, H, w), dtype)
        v, v32 = gen(rng, (n_layers, n_seqs, H, w), dtype)
        if per_layer:
            for layer in range(n_layers):
                assert eng.decode_append(layer, 1, k[layer:layer + 1], v[layer:layer + 1], pos) == 0
                st, vic = eng.decode_evict(layer, 1)
                ref_vic = rep.decode(layer, 1, k32[layer:layer + 1], v32[layer:layer + 1], pos,
                                     step)
                np.testing.assert_array_equal(vic, ref_vic)
        else:
            assert eng.decode_append(0, n_layers, k, v, pos) == 0
            st, vic = eng.decode_evict(0, n_layers)
            ref_vic = rep.decode(0, n_layers, k32, v32, pos, step)
            np.testing.assert_array_equal(vic, ref_vic)
        pos += 1
        compare_with_reference(rep, oracle_state(eng), check_pages=(step % 5 == 0))
    drained = rep.sess.drain_free_list()
    np.testing.assert_array_equal(drained, eng.free_stack()[::-1])


def test_engine_attention_matches_reference(reference):
    rng = np.random.default_rng(5)
    n_seqs, H, G, d, B, C = 2, 2, 3, 16, 8, 32
    lens = np.array([70, 20])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, rep = _engine_pair(reference, n_seqs=n_seqs, n_layers=1, H=H, w=d, B=B, C=C,
                            cap=64, max_pages=C // B + 1, dtype=oracle.F32)
    k, _ = random_kv(rng, (cu[-1], H, d), oracle.F32)
    v, _ = random_kv(rng, (cu[-1], H, d), oracle.F32)
    eng.prefill(0, k, v, cu)
    rep.prefill(0, k, v, cu)
    q = rng.standard_normal((n_seqs, H * G, d), dtype=np.float32)
    st, out = eng.attention(0, q, G)
    assert st == 0
    np.testing.assert_array_equal(out, rep.attend(0, q, G))


def test_full_cache_policy_never_evicts(reference):
    rng = np.random.default_rng(6)
    B, C = 4, 8
    eng, rep = _engine_pair(reference, n_seqs=1, n_layers=1, H=1, w=4, B=B, C=C, cap=40,
                            max_pages=30, dtype=oracle.F32, kind=oracle.FULL_CACHE)
    cu = np.array([0, 30], np.int32)
    k, _ = random_kv(rng, (30, 1, 4), oracle.F32)
    v, _ = random_kv(rng, (30, 1, 4), oracle.F32)
    st, ev = eng.prefill(0, k, v, cu)
    assert st == 0 and ev[0] == 0
    rep.prefill(0, k, v, cu)
    pos = np.array([30])
    for step in range(1, 20):
        kk, _ = random_kv(rng, (1, 1, 1, 4), oracle.F32)
        vv, _ = random_kv(rng, (1, 1, 1, 4), oracle.F32)
        eng.decode_append(0, 1, kk, vv, pos)
        st, vic = eng.decode_evict(0, 1)
        assert vic[0] == -1
        rep.decode(0, 1, kk, vv, pos, step)
        pos += 1
    compare_with_reference(rep, oracle_state(eng))


def test_pool_exhaustion_is_all_or_nothing():
    eng = oracle.OracleEngine(n_seqs=2, n_layers=1, n_tab_heads=1, width=4, page_size=4,
                              budget=8, dtype=oracle.F32, capacity=3, max_pages=3)
    k = np.ones((16, 1, 4), np.float32)
    cu = np.array([0, 8, 16], np.int32)  # needs 2 + 2 pages, pool has 3
    st, _ = eng.prefill(0, k, k, cu)
    assert st == 2  # PoolExhausted
    assert eng.top == 3 and eng.num_pages().sum() == 0
