"""GPU parity of the CUDA engine against the C oracle (and, for small cases,
the compiled reference itself), all through the C-ABI.

Bit-exact: block tables, num_pages/newest_fill/retained, the free list,
positions, page bytes, victims, evicted counts, token and page scores.
Attention: relative L2 (output_deviation) <= 1e-5 (fp32) / 1e-3 (bf16).
"""
import numpy as np
import pytest

import oracle
from tests.harness import (RefReplay, compare_states, compare_states_vectorized, compare_with_reference, grid_kv,
                           oracle_state, random_kv)

torch = pytest.importorskip("torch")
pe = pytest.importorskip("paper_2509_04377_b200")

pytestmark = pytest.mark.gpu


def make_pair(*, n_seqs, n_layers, H, d, B, C, dtype, cap=0, max_pages=0, kind=0):
    geo = pe.EngineGeometry(n_seqs=n_seqs, n_layers=n_layers, n_kv_heads=H, head_dim=d,
                            dtype=dtype, capacity=cap, max_pages_per_table=max_pages)
    eng = pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=C, page_size=B,
                                                      kind=pe.PolicyKind(kind)))
    orc = oracle.OracleEngine(n_seqs=n_seqs, n_layers=n_layers, n_tab_heads=H, width=d,
                              page_size=B, budget=C, dtype=dtype, capacity=eng.capacity,
                              max_pages=eng.max_pages, policy=kind)
    return eng, orc


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(eng, orc, what="", pages=True):
    st = eng.state(with_pages=pages)
    ost = oracle_state(orc)
    compare_states(st, ost, eng.n_tables, eng.B, check_pages=pages, what=what)
    # cached scores of every live slot / full page are the oracle's bit for bit
    for t in range(eng.n_tables):
        n = int(st["num_pages"][t])
        for j in range(n):
            pid = int(st["block_table"][t, j])
            fill = eng.B if j < n - 1 else int(st["newest_fill"][t])
            np.testing.assert_array_equal(st["token_scores"][pid, :fill],
                                          orc.token_scores()[pid, :fill], err_msg=f"{what}token scores")
            if fill == eng.B:
                assert st["page_scores"][pid] == ost["page_scores"][pid], f"{what}page score {pid}"


@pytest.fixture(params=["default", "global", "global_fallback", "stream512", "smem", "stream", "cluster"])
def select_path(request, monkeypatch):
    """Run prefill through every select kernel: the default (for these small
    calls, fewer tables than half the SMs: the shared-memory CTA select), the
    GPU-wide select (window / count / resolve / emit, pe_select.cu; the
    default for larger calls) forced with PE_SELECT=global, its fallback forced for
    every table (PE_SELECT=global_fallback), the 512-thread streamed
    CTA select, the shared-memory CTA select, the 1024-thread streamed
    select and the 8-CTA cluster select."""
    if request.param == "default":
        monkeypatch.delenv("PE_SELECT", raising=False)
    else:
        monkeypatch.setenv("PE_SELECT", request.param)
    return request.param


@pytest.mark.parametrize("dtype", [oracle.F32, oracle.BF16])
@pytest.mark.parametrize("gen", [random_kv, grid_kv])
def test_prefill_parity(dtype, gen, select_path):
    rng = np.random.default_rng(100 + dtype)
    B, C, d, H = 16, 64, 64 if dtype == oracle.F32 else 128, 2
    lens = np.array([C + 1, 3 * C + 7, C, 5, 1, 2 * C, 1000])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, orc = make_pair(n_seqs=len(lens), n_layers=2, H=H, d=d, B=B, C=C, dtype=dtype)
    for layer in range(2):
        k, _ = gen(rng, (cu[-1], H, d), dtype)
        v, _ = gen(rng, (cu[-1], H, d), dtype)
        ev = eng.prefill_compress(layer, dev(k), dev(v), cu, evicted_counts=True)
        st, oev = orc.prefill(layer, k, v, cu)
        assert st == 0
        np.testing.assert_array_equal(ev, oev)
    eng.sync()
    check(eng, orc, "prefill: ")


@pytest.mark.parametrize("variant", ["copy_gather", "unstaged_keys", "fallback_grid2", "identity_by_copy",
                                     "score_grid_2d"])
@pytest.mark.parametrize("dtype", [oracle.F32, oracle.BF16])
@pytest.mark.parametrize("gen", [random_kv, grid_kv])
def test_prefill_kernel_variants(variant, dtype, gen, monkeypatch):
    """The K1 A/B paths beside the defaults: the copy that gathers each
    survivor's key instead of rescoring its row (PE_COPY_RESCORE=0), per-warp
    key stores instead of the CTA-staged runs (PE_SCORE_STAGED_KEYS=0), and
    the global select's fallback looping over a wave's flagged tables with 2
    CTAs (PE_FB_GRID=2, every table flagged), and tables that keep every
    token (L <= C) packed by the copy kernel instead of by the score kernel
    (PE_PREFILL_DIRECT=0), and the score kernel on its full 2-D grid instead
    of the compact grid over non-empty blocks (PE_SCORE_COMPACT=0).
    Bit-exact against the oracle."""
    env = {"copy_gather": {"PE_COPY_RESCORE": "0"},
           "unstaged_keys": {"PE_SCORE_STAGED_KEYS": "0"},
           "fallback_grid2": {"PE_FB_GRID": "2", "PE_SELECT": "global_fallback"},
           "identity_by_copy": {"PE_PREFILL_DIRECT": "0"},
           "score_grid_2d": {"PE_SCORE_COMPACT": "0"}}[variant]
    monkeypatch.delenv("PE_SELECT", raising=False)
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    rng = np.random.default_rng(300 + dtype)
    B, C, d, H = 16, 512, 64 if dtype == oracle.F32 else 128, 2
    lens = np.array([C + 1, 9000, C, 5, 3 * C + 7, 4097])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, orc = make_pair(n_seqs=len(lens), n_layers=1, H=H, d=d, B=B, C=C, dtype=dtype)
    k, _ = gen(rng, (cu[-1], H, d), dtype)
    v, _ = gen(rng, (cu[-1], H, d), dtype)
    ev = eng.prefill_compress(0, dev(k), dev(v), cu, evicted_counts=True)
    st, oev = orc.prefill(0, k, v, cu)
    assert st == 0
    np.testing.assert_array_equal(ev, oev)
    eng.sync()
    check(eng, orc, f"{variant}: ")


def test_prefill_ties_across_cta_boundaries(select_path):
    """Every token of a table scores identically: the E evicted tokens must be
    exactly the oldest E (position tie rule, importance.cpp:46-52), even
    though the ties straddle the 8 CTAs of the cluster."""
    B, C, d, H = 16, 256, 128, 1
    L = 2000
    k = np.tile(oracle.f32_to_bf16_bits(np.full(d, 0.5, np.float32)), (L, H, 1))
    cu = np.array([0, L], np.int32)
    eng, orc = make_pair(n_seqs=1, n_layers=1, H=H, d=d, B=B, C=C, dtype=oracle.BF16)
    eng.prefill_compress(0, dev(k), dev(k), cu)
    orc.prefill(0, k, k, cu)
    eng.sync()
    check(eng, orc, "ties: ")
    np.testing.assert_array_equal(eng.retained_positions(0), np.arange(L - C, L))


@pytest.fixture(params=["waves", "fused"])
def prefill_variant(request, monkeypatch):
    """The default multi-kernel wave pipeline and the opt-in persistent kernel."""
    monkeypatch.setenv("PE_PREFILL_FUSED", "1" if request.param == "fused" else "0")
    return request.param


@pytest.mark.parametrize("sel", ["default", "global", "global_fallback", "stream512", "smem"])
@pytest.mark.parametrize("gen", [random_kv, grid_kv])
def test_prefill_long_tables_windowed_select(gen, prefill_variant, sel, monkeypatch):
    """Tables of >= 8192 tokens take the sampled pivot window (the GPU-wide
    select's window kernel, or the CTA selects'); tie-heavy grid data
    overflows the window and exercises the fallbacks (the CTA-per-table
    select behind the global select, the full passes inside the CTA
    selects). Bit-exact against the oracle."""
    if sel == "default":
        monkeypatch.delenv("PE_SELECT", raising=False)
    else:
        monkeypatch.setenv("PE_SELECT", sel)
    rng = np.random.default_rng(8192)
    B, C, d, H = 16, 2048, 128, 2
    lens = np.array([8192, 32768, 20001, 9000, 4096 + 1])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, orc = make_pair(n_seqs=len(lens), n_layers=1, H=H, d=d, B=B, C=C, dtype=oracle.BF16)
    k, _ = gen(rng, (cu[-1], H, d), oracle.BF16)
    v, _ = gen(rng, (cu[-1], H, d), oracle.BF16)
    ev = eng.prefill_compress(0, dev(k), dev(v), cu, evicted_counts=True)
    st, oev = orc.prefill(0, k, v, cu)
    assert st == 0
    np.testing.assert_array_equal(ev, oev)
    eng.sync()
    check(eng, orc, "windowed: ")


@pytest.mark.parametrize("dtype", [oracle.F32, oracle.BF16])
@pytest.mark.parametrize("mode,k2", [(0, "flat"), (0, "grid"), (1, "cached")])
def test_decode_parity(dtype, mode, k2, monkeypatch):
    """K0 + K2 (recompute: the flat persistent kernel of small launches, or
    the (table, chunk) grid with PE_K2_FLAT=0) or K2c, all-layer and
    per-layer launches, bit-exact against the oracle."""
    monkeypatch.setenv("PE_K2_FLAT", "0" if k2 == "grid" else "1")
    rng = np.random.default_rng(7 + 10 * dtype + mode)
    B, C, H, n_layers, S = 16, 64, 2, 3, 3
    d = 64 if dtype == oracle.F32 else 128
    lens = np.array([C + 20, C - 5, 200])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, orc = make_pair(n_seqs=S, n_layers=n_layers, H=H, d=d, B=B, C=C, dtype=dtype)
    for layer in range(n_layers):
        k, _ = random_kv(rng, (cu[-1], H, d), dtype)
        v, _ = random_kv(rng, (cu[-1], H, d), dtype)
        eng.prefill_compress(layer, dev(k), dev(v), cu)
        orc.prefill(layer, k, v, cu)
    pos = lens.astype(np.int64).copy()
    for step in range(1, 3 * B + 4):
        k, _ = random_kv(rng, (n_layers, S, H, d), dtype)
        v, _ = random_kv(rng, (n_layers, S, H, d), dtype)
        if step % 3 == 1 and mode == 0:
            # one append over all layers, then per-layer evictions back to
            # back with device-side victims (no host copy in between: the K2
            # launches chain through programmatic dependent launch)
            eng.append_token(0, n_layers, dev(k), dev(v), dev(pos))
            assert orc.decode_append(0, n_layers, k, v, pos) == 0
            vics = [torch.full((S * H,), -7, dtype=torch.int32, device="cuda") for _ in range(n_layers)]
            for layer in range(n_layers):
                eng.evict(layer, 1, step=step, mode=mode, victims=vics[layer])
            for layer in range(n_layers):
                _, ovic = orc.decode_evict(layer, 1)
                np.testing.assert_array_equal(vics[layer].cpu().numpy(), ovic, err_msg=f"step {step} layer {layer}")
        elif step % 3 == 0:  # per-layer launches
            for layer in range(n_layers):
                vic = eng.decode_step(layer, 1, dev(k[layer:layer + 1]), dev(v[layer:layer + 1]),
                                      dev(pos), step, mode=mode, victims=True)
                assert orc.decode_append(layer, 1, k[layer:layer + 1], v[layer:layer + 1], pos) == 0
                _, ovic = orc.decode_evict(layer, 1)
                np.testing.assert_array_equal(vic, ovic, err_msg=f"step {step} layer {layer}")
        else:
            vic = eng.decode_step(0, n_layers, dev(k), dev(v), dev(pos), step, mode=mode,
                                  victims=True)
            assert orc.decode_append(0, n_layers, k, v, pos) == 0
            _, ovic = orc.decode_evict(0, n_layers)
            np.testing.assert_array_equal(vic, ovic, err_msg=f"step {step}")
        pos += 1
        if step % 8 == 0:
            eng.sync()
            check(eng, orc, f"step {step}: ", pages=(step % 16 == 0))
    eng.sync()
    check(eng, orc, "final: ")
    assert eng.stats().pages_evicted > 0


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("pdl", ["1", "0"])
def test_per_layer_evictions_back_to_back(pdl, mode, monkeypatch):
    """Per-layer K2 launches issued back to back on one stream (a serving
    loop's eviction of every layer): with PE_K2_PDL=1 each launch after the
    first overlaps its predecessor (programmatic dependent launch: scoring
    and table eviction before griddepcontrol.wait, the free-stack push after).
    16 x 4 x 8 = 512 tables of C + B = 1040 tokens, 9 chunks per table;
    victims, block tables, positions, page bytes and the free list bit-exact
    against the oracle after every cycle, the pushes in launch order."""
    monkeypatch.setenv("PE_K2_PDL", pdl)
    rng = np.random.default_rng(4096)
    B, C, H, n_layers, S, d = 16, 1024, 8, 4, 16, 128
    lens = np.full(S, 2048)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, orc = make_pair(n_seqs=S, n_layers=n_layers, H=H, d=d, B=B, C=C, dtype=oracle.BF16)
    for layer in range(n_layers):
        k, _ = random_kv(rng, (cu[-1], H, d), oracle.BF16)
        v, _ = random_kv(rng, (cu[-1], H, d), oracle.BF16)
        eng.prefill_compress(layer, dev(k), dev(v), cu)
        orc.prefill(layer, k, v, cu)
    pos = lens.astype(np.int64).copy()
    for cycle in range(3):
        for j in range(B):
            k, _ = random_kv(rng, (n_layers, S, H, d), oracle.BF16)
            v, _ = random_kv(rng, (n_layers, S, H, d), oracle.BF16)
            eng.append_token(0, n_layers, dev(k), dev(v), dev(pos))
            assert orc.decode_append(0, n_layers, k, v, pos) == 0
            pos += 1
        vics = [torch.full((S * H,), -7, dtype=torch.int32, device="cuda") for _ in range(n_layers)]
        for layer in range(n_layers):
            # alternate the score modes across layers in mode 1 (K2c and K2
            # launches chained through PDL in both orders)
            m = pe.ScoreMode.CACHED if (mode == 1 and (layer + cycle) % 2 == 0) else pe.ScoreMode.RECOMPUTE
            eng.evict(layer, 1, step=(cycle + 1) * B, victims=vics[layer], mode=m)
        for layer in range(n_layers):
            _, ovic = orc.decode_evict(layer, 1)
            np.testing.assert_array_equal(vics[layer].cpu().numpy(), ovic, err_msg=f"cycle {cycle} layer {layer}")
        eng.sync()
        st = eng.state(with_pages=(cycle == 2))
        compare_states_vectorized(st, oracle_state(orc), B, check_pages=(cycle == 2), what=f"cycle {cycle}: ")
    assert eng.stats().pages_evicted == 3 * S * n_layers * H


@pytest.mark.parametrize("pdl", ["1", "0"])
def test_serving_order_evict_attend_interleaved(pdl, monkeypatch):
    """A serving loop's per-layer order: append on every layer, then per
    layer evict(l) -> attend(l). With PE_K2_PDL=1 each evict(l + 1) launches
    behind attend(l) through programmatic dependent launch (the attention
    writes only its own partials and output; the eviction of another layer's
    tables streams while it drains). Victims of every layer and the GQA
    outputs (bf16 tolerance 1e-3) against the oracle at every step; the whole
    state bit-exact at the end. PE_PDL=0 also turns off the PDL launches of
    K0, K2c and K3 (each waits at its top, so only the launch gap differs)."""
    monkeypatch.setenv("PE_K2_PDL", pdl)
    monkeypatch.setenv("PE_PDL", pdl)
    rng = np.random.default_rng(5150)
    B, C, H, G, n_layers, S, d = 16, 512, 4, 4, 3, 8, 128
    lens = np.full(S, 1200)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, orc = make_pair(n_seqs=S, n_layers=n_layers, H=H, d=d, B=B, C=C, dtype=oracle.BF16)
    for layer in range(n_layers):
        k, _ = random_kv(rng, (cu[-1], H, d), oracle.BF16)
        v, _ = random_kv(rng, (cu[-1], H, d), oracle.BF16)
        eng.prefill_compress(layer, dev(k), dev(v), cu)
        orc.prefill(layer, k, v, cu)
    pos = lens.astype(np.int64).copy()
    for step in range(1, 2 * B + 3):
        k, _ = random_kv(rng, (n_layers, S, H, d), oracle.BF16)
        v, _ = random_kv(rng, (n_layers, S, H, d), oracle.BF16)
        eng.append_token(0, n_layers, dev(k), dev(v), dev(pos))
        assert orc.decode_append(0, n_layers, k, v, pos) == 0
        pos += 1
        q, _ = random_kv(rng, (n_layers, S, H * G, d), oracle.BF16)
        outs, vics = [], []
        for layer in range(n_layers):
            vics.append(torch.full((S * H,), -7, dtype=torch.int32, device="cuda"))
            eng.evict(layer, 1, step=step, victims=vics[-1])
            outs.append(torch.empty((S, H * G, d), dtype=torch.float32, device="cuda"))
            eng.attend(layer, dev(np.ascontiguousarray(q[layer])), outs[-1], H * G)
        for layer in range(n_layers):
            _, ovic = orc.decode_evict(layer, 1)
            np.testing.assert_array_equal(vics[layer].cpu().numpy(), ovic, err_msg=f"step {step} layer {layer}")
            _, ref = orc.attention(layer, np.ascontiguousarray(q[layer]), G)
            got = outs[layer].cpu().numpy()
            for s_ in range(S):
                for hq in range(H * G):
                    dv = oracle.Oracle().output_deviation(got[s_, hq], ref[s_, hq])
                    assert dv <= 1e-3, f"step {step} layer {layer} seq {s_} head {hq}: deviation {dv}"
    eng.sync()
    check(eng, orc, "serving order: ")
    assert eng.stats().pages_evicted == 2 * S * n_layers * H


@pytest.mark.parametrize("fast", ["1", "0"])
def test_append_chain_parity(fast, monkeypatch):
    """Runs of consecutive appends (the K0 no-pop fast path: the previous
    append over the same layer range flagged no popping table), broken by
    evictions and per-layer appends (a range change); an initially empty
    layer and mixed lengths so pops happen at different steps
    in different tables. Bit-exact against the oracle after every launch;
    PE_APPEND_FAST=0 runs the same schedule through the look-back only."""
    monkeypatch.setenv("PE_APPEND_FAST", fast)
    rng = np.random.default_rng(77)
    B, C, H, n_layers, S, d = 8, 32, 2, 3, 4, 64
    lens = np.array([C + 3, 7, 2 * C, 1])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    # evictions every B steps only: tables may hold up to C + 2B tokens
    eng, orc = make_pair(n_seqs=S, n_layers=n_layers, H=H, d=d, B=B, C=C, dtype=oracle.F32,
                         max_pages=C // B + 4)
    for layer in range(n_layers - 1):  # the last layer starts empty (its first append pops)
        k, _ = random_kv(rng, (cu[-1], H, d), oracle.F32)
        v, _ = random_kv(rng, (cu[-1], H, d), oracle.F32)
        eng.prefill_compress(layer, dev(k), dev(v), cu)
        orc.prefill(layer, k, v, cu)
    pos = lens.astype(np.int64).copy()
    for step in range(1, 4 * B + 3):
        k, _ = random_kv(rng, (n_layers, S, H, d), oracle.F32)
        v, _ = random_kv(rng, (n_layers, S, H, d), oracle.F32)
        if step % 11 == 5:  # per-layer appends (range change breaks the chain)
            for layer in range(n_layers):
                eng.append_token(layer, 1, dev(k[layer:layer + 1]), dev(v[layer:layer + 1]), dev(pos))
                assert orc.decode_append(layer, 1, k[layer:layer + 1], v[layer:layer + 1], pos) == 0
        else:
            eng.append_token(0, n_layers, dev(k), dev(v), dev(pos))
            assert orc.decode_append(0, n_layers, k, v, pos) == 0
        if step % B == 0:
            vic = eng.evict(0, n_layers, step=step, victims=True)
            _, ovic = orc.decode_evict(0, n_layers)
            np.testing.assert_array_equal(vic, ovic, err_msg=f"step {step}")
        pos += 1
        eng.sync()
        check(eng, orc, f"step {step}: ", pages=(step % 8 == 0))


@pytest.mark.slow
@pytest.mark.parametrize("fast", ["1", "0"])
def test_append_chain_parity_grid_exceeds_residency(fast, monkeypatch):
    """The K0 fast-path verdict must be the same in every CTA of a launch
    even when the grid is larger than what the GPU holds at once (CTAs that
    start after others finished). 4096 seqs x 2 layers x 64 heads
    = 524 288 tables = 8192 append CTAs (> 148 SMs x 32 resident CTAs);
    mixed prompt lengths so some tables pop on every launch while others
    fill, and one layer starts empty. Bit-exact against the oracle."""
    monkeypatch.setenv("PE_APPEND_FAST", fast)
    rng = np.random.default_rng(8192)
    B, C, H, n_layers, S, d = 4, 8, 64, 2, 4096, 4
    lens = rng.integers(1, 3 * C, size=S)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, orc = make_pair(n_seqs=S, n_layers=n_layers, H=H, d=d, B=B, C=C, dtype=oracle.F32,
                         max_pages=C // B + 4)
    assert eng.n_tables == 524288
    k, _ = random_kv(rng, (cu[-1], H, d), oracle.F32)
    v, _ = random_kv(rng, (cu[-1], H, d), oracle.F32)
    eng.prefill_compress(0, dev(k), dev(v), cu)
    orc.prefill(0, k, v, cu)
    pos = lens.astype(np.int64).copy()
    for step in range(1, 2 * B + 3):
        k, _ = random_kv(rng, (n_layers, S, H, d), oracle.F32)
        v, _ = random_kv(rng, (n_layers, S, H, d), oracle.F32)
        eng.append_token(0, n_layers, dev(k), dev(v), dev(pos))
        assert orc.decode_append(0, n_layers, k, v, pos) == 0
        if step % B == 0:
            vic = eng.evict(0, n_layers, step=step, victims=True)
            _, ovic = orc.decode_evict(0, n_layers)
            np.testing.assert_array_equal(vic, ovic, err_msg=f"step {step}")
        pos += 1
        eng.sync()
        st = eng.state(with_pages=(step == 2 * B + 2))
        compare_states_vectorized(st, oracle_state(orc), B, check_pages=(step == 2 * B + 2),
                                  what=f"step {step}: ")
    inv = eng.check_invariants()
    # evictions only every B appends: tables may hold up to C + 2B tokens, so
    # the budget bound does not apply here; every structural invariant does
    assert inv["violations"] == inv["budget_violations"], inv
    assert inv["pages_mapped"] + inv["free_pages"] == eng.capacity and inv["page_refcount"] == 0, inv


def test_engine_matches_compiled_reference(reference):
    """Direct replay through the reference's own PagePool/BlockTable/policy."""
    rng = np.random.default_rng(42)
    B, C, d, H, S, n_layers = 8, 40, 16, 2, 3, 2
    lens = np.array([100, 17, 41])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, _ = make_pair(n_seqs=S, n_layers=n_layers, H=H, d=d, B=B, C=C, dtype=oracle.F32)
    rep = RefReplay(reference, n_seqs=S, n_layers=n_layers, n_tab_heads=H, width=d, page_size=B,
                    budget=C, capacity=eng.capacity)
    for layer in range(n_layers):
        k, _ = grid_kv(rng, (cu[-1], H, d), oracle.F32)
        v, _ = random_kv(rng, (cu[-1], H, d), oracle.F32)
        eng.prefill_compress(layer, dev(k), dev(v), cu)
        rep.prefill(layer, k, v, cu)
    pos = lens.astype(np.int64).copy()
    for step in range(1, 30):
        k, _ = random_kv(rng, (n_layers, S, H, d), oracle.F32)
        v, _ = grid_kv(rng, (n_layers, S, H, d), oracle.F32)
        vic = eng.decode_step(0, n_layers, dev(k), dev(v), dev(pos), step, victims=True)
        np.testing.assert_array_equal(vic, rep.decode(0, n_layers, k, v, pos, step))
        pos += 1
    eng.sync()
    st = eng.state()
    compare_with_reference(rep, st)
    np.testing.assert_array_equal(rep.sess.drain_free_list(), st["free_stack"][::-1])


@pytest.mark.parametrize("dtype,tol", [(oracle.F32, 1e-5), (oracle.BF16, 1e-3)])
def test_attention_parity(dtype, tol):
    rng = np.random.default_rng(9)
    B, C, H, G = 16, 128, 2, 4
    d = 64 if dtype == oracle.F32 else 128
    lens = np.array([300, 50, 128, 7])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, orc = make_pair(n_seqs=len(lens), n_layers=1, H=H, d=d, B=B, C=C, dtype=dtype)
    k, _ = random_kv(rng, (cu[-1], H, d), dtype)
    v, _ = random_kv(rng, (cu[-1], H, d), dtype)
    eng.prefill_compress(0, dev(k), dev(v), cu)
    orc.prefill(0, k, v, cu)
    pos = lens.astype(np.int64).copy()
    for step in range(1, 20):
        kk, _ = random_kv(rng, (1, len(lens), H, d), dtype)
        vv, _ = random_kv(rng, (1, len(lens), H, d), dtype)
        eng.decode_step(0, 1, dev(kk), dev(vv), dev(pos), step)
        orc.decode_append(0, 1, kk, vv, pos)
        orc.decode_evict(0, 1)
        pos += 1
        q, _ = random_kv(rng, (len(lens), H * G, d), dtype)
        out = torch.empty((len(lens), H * G, d), dtype=torch.float32, device="cuda")
        eng.attend(0, dev(q), out, H * G)
        _, ref = orc.attention(0, q, G)
        got = out.cpu().numpy()
        for s in range(len(lens)):
            for hq in range(H * G):
                dev_ = oracle.Oracle().output_deviation(got[s, hq], ref[s, hq])
                assert dev_ <= tol, f"step {step} seq {s} head {hq}: deviation {dev_}"


@pytest.mark.parametrize("B", [8, 32])
@pytest.mark.parametrize("dtype", [oracle.F32, oracle.BF16])
@pytest.mark.parametrize("mode", [0, 1])
def test_page_sizes_full_flow(B, dtype, mode):
    """Page sizes other than 16 through the whole path: prefill (every select
    path the call shape picks, tables below and above the budget, so the
    score kernel's direct packing and the copy both run), decode cycles with
    block evictions (recompute or cached scores) and attention (the CUDA-core
    kernel: the tensor-core ones take B = 16 only). State bit-exact and
    attention within tolerance against the oracle."""
    rng = np.random.default_rng(3200 + B + dtype + 10 * mode)
    C, H, G = 4 * B, 2, 2
    d = 64 if dtype == oracle.F32 else 128
    lens = np.array([C - 3, 7 * B + 5, C, 3 * C + 1, 2 * B])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, orc = make_pair(n_seqs=len(lens), n_layers=2, H=H, d=d, B=B, C=C, dtype=dtype)
    for layer in range(2):
        k, _ = random_kv(rng, (cu[-1], H, d), dtype)
        v, _ = random_kv(rng, (cu[-1], H, d), dtype)
        ev = eng.prefill_compress(layer, dev(k), dev(v), cu, evicted_counts=True)
        st, oev = orc.prefill(layer, k, v, cu)
        assert st == 0
        np.testing.assert_array_equal(ev, oev)
    pos = lens.astype(np.int64).copy()
    tol = 1e-5 if dtype == oracle.F32 else 1e-3
    for step in range(1, 2 * B + 3):
        kk, _ = random_kv(rng, (2, len(lens), H, d), dtype)
        vv, _ = random_kv(rng, (2, len(lens), H, d), dtype)
        vic = eng.decode_step(0, 2, dev(kk), dev(vv), dev(pos), step, mode=mode, victims=True)
        orc.decode_append(0, 2, kk, vv, pos)
        _, ovic = orc.decode_evict(0, 2)
        np.testing.assert_array_equal(vic, ovic, err_msg=f"step {step}")
        pos += 1
        if step % B == 0:
            q, _ = random_kv(rng, (len(lens), H * G, d), dtype)
            out = torch.empty((len(lens), H * G, d), dtype=torch.float32, device="cuda")
            eng.attend(1, dev(q), out, H * G)
            _, ref = orc.attention(1, q, G)
            got = out.cpu().numpy()
            for sq in range(len(lens)):
                for hq in range(H * G):
                    assert oracle.Oracle().output_deviation(got[sq, hq], ref[sq, hq]) <= tol
    eng.sync()
    check(eng, orc, f"B={B}: ")
    assert eng.stats().pages_evicted > 0


@pytest.mark.parametrize("H", [16, 32])
def test_prefill_many_kv_heads(H):
    """More KV heads per sequence than the defaults plan for: 16 heads (score
    CTAs of 64 tokens so the keys still fit the staging buffer) and 32 heads
    (per-warp key stores, no direct packing of tables that keep every
    token). Prefill and one eviction cycle bit-exact against the oracle."""
    rng = np.random.default_rng(1600 + H)
    B, C, d = 16, 64, 64
    lens = np.array([C + 17, 40, 5 * C + 3, C])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, orc = make_pair(n_seqs=len(lens), n_layers=1, H=H, d=d, B=B, C=C, dtype=oracle.BF16)
    k, _ = random_kv(rng, (cu[-1], H, d), oracle.BF16)
    v, _ = random_kv(rng, (cu[-1], H, d), oracle.BF16)
    ev = eng.prefill_compress(0, dev(k), dev(v), cu, evicted_counts=True)
    st, oev = orc.prefill(0, k, v, cu)
    assert st == 0
    np.testing.assert_array_equal(ev, oev)
    pos = lens.astype(np.int64).copy()
    for step in range(1, B + 1):
        kk, _ = random_kv(rng, (1, len(lens), H, d), oracle.BF16)
        vv, _ = random_kv(rng, (1, len(lens), H, d), oracle.BF16)
        vic = eng.decode_step(0, 1, dev(kk), dev(vv), dev(pos), step, victims=True)
        orc.decode_append(0, 1, kk, vv, pos)
        _, ovic = orc.decode_evict(0, 1)
        np.testing.assert_array_equal(vic, ovic, err_msg=f"step {step}")
        pos += 1
    eng.sync()
    check(eng, orc, f"H={H}: ")


def test_host_buffers_match_device_buffers():
    rng = np.random.default_rng(3)
    B, C, d, H = 16, 64, 128, 2
    lens = np.array([150, 90])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    a, _ = make_pair(n_seqs=2, n_layers=1, H=H, d=d, B=B, C=C, dtype=oracle.BF16)
    b, _ = make_pair(n_seqs=2, n_layers=1, H=H, d=d, B=B, C=C, dtype=oracle.BF16)
    k, _ = random_kv(rng, (cu[-1], H, d), oracle.BF16)
    v, _ = random_kv(rng, (cu[-1], H, d), oracle.BF16)
    a.prefill_compress(0, dev(k), dev(v), cu)
    b.prefill_compress(0, k, v, cu)  # numpy host buffers
    pos = lens.astype(np.int64)
    for step in range(1, 18):
        kk, _ = random_kv(rng, (1, 2, H, d), oracle.BF16)
        vv, _ = random_kv(rng, (1, 2, H, d), oracle.BF16)
        va = a.decode_step(0, 1, dev(kk), dev(vv), dev(pos), step, victims=True)
        vb = b.decode_step(0, 1, kk, vv, pos, step, victims=True)
        np.testing.assert_array_equal(va, vb)
        pos = pos + 1
    a.sync()
    b.sync()
    compare_states(a.state(), b.state(), a.n_tables, B)


def test_error_statuses():
    # PolicyConfig::validate -> BudgetInvalid (policy.cpp:38-52)
    geo = pe.EngineGeometry(n_seqs=1, n_layers=1, n_kv_heads=1, head_dim=8, dtype=oracle.F32)
    with pytest.raises(pe.BudgetInvalid):
        pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=1000, page_size=16))
    with pytest.raises(pe.BudgetInvalid):
        pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=8, page_size=16))
    # PoolExhausted (page_pool.cpp:26-28): all-or-nothing, status via sync()
    geo = pe.EngineGeometry(n_seqs=2, n_layers=1, n_kv_heads=1, head_dim=8, dtype=oracle.F32,
                            capacity=3)
    eng = pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=8, page_size=4))
    k = np.ones((16, 1, 8), np.float32)
    eng.prefill_compress(0, dev(k), dev(k), np.array([0, 8, 16], np.int32))
    with pytest.raises(pe.PoolExhausted):
        eng.sync()
    assert eng.free_count() == 3
    # prefill into a non-empty table -> InvalidState
    eng.prefill_compress(0, dev(k[:8]), dev(k[:8]), np.array([0, 8], np.int32))
    eng.sync()
    eng.prefill_compress(0, dev(k[:8]), dev(k[:8]), np.array([0, 8], np.int32))
    with pytest.raises(pe.InvalidState):
        eng.sync()
    # empty prefill -> Error (policy.cpp:57-58)
    with pytest.raises(pe.Error):
        eng.prefill_compress(0, dev(k), dev(k), np.array([0, 0], np.int32), seq_begin=1)
    # GQA shape mismatch -> LengthMismatch (3 query heads over 2 KV heads)
    geo = pe.EngineGeometry(n_seqs=1, n_layers=1, n_kv_heads=2, head_dim=8, dtype=oracle.F32)
    eng2 = pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=8, page_size=4))
    out = torch.empty((1, 3, 8), dtype=torch.float32, device="cuda")
    with pytest.raises(pe.LengthMismatch):
        eng2.attend(0, dev(np.ones((1, 3, 8), np.float32)), out, 3)
    # attention over a table with no retained token -> EmptyCache (attention.cpp:24-25),
    # output zeros instead of 0/0
    geo = pe.EngineGeometry(n_seqs=2, n_layers=1, n_kv_heads=1, head_dim=64, dtype=oracle.BF16)
    eng3 = pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=16, page_size=16))
    kb = np.tile(oracle.f32_to_bf16_bits(np.full(64, 0.25, np.float32)), (20, 1, 1))
    eng3.prefill_compress(0, dev(kb), dev(kb), np.array([0, 20], np.int32), seq_begin=0)  # seq 1 stays empty
    eng3.sync()
    out3 = torch.full((2, 4, 64), 7.0, dtype=torch.float32, device="cuda")
    eng3.attend(0, dev(np.zeros((2, 4, 64), np.uint16)), out3, 4)
    with pytest.raises(pe.EmptyCache):
        eng3.sync()
    assert torch.all(out3[1] == 0) and torch.isfinite(out3).all()


@pytest.mark.slow
def test_cfg1_full_parity():
    """BASELINE config 1 in full: Llama-3.2-1B KV geometry (16 layers, 8 KV
    heads, d=64), fp32, 1 sequence of 4096 tokens, C=1024, B=16: prefill all
    layers, then 64 decode steps (4 triggers per table), recompute eviction."""
    rng = np.random.default_rng(20250905)
    eng, orc = make_pair(n_seqs=1, n_layers=16, H=8, d=64, B=16, C=1024, dtype=oracle.F32)
    cu = np.array([0, 4096], np.int32)
    for layer in range(16):
        k, _ = random_kv(rng, (4096, 8, 64), oracle.F32)
        v, _ = random_kv(rng, (4096, 8, 64), oracle.F32)
        eng.prefill_compress(layer, dev(k), dev(v), cu)
        orc.prefill(layer, k, v, cu)
    eng.sync()
    check(eng, orc, "cfg1 prefill: ", pages=False)
    pos = np.array([4096], np.int64)
    for step in range(1, 65):
        k, _ = random_kv(rng, (16, 1, 8, 64), oracle.F32)
        v, _ = random_kv(rng, (16, 1, 8, 64), oracle.F32)
        vic = eng.decode_step(0, 16, dev(k), dev(v), dev(pos), step, victims=True)
        orc.decode_append(0, 16, k, v, pos)
        _, ovic = orc.decode_evict(0, 16)
        np.testing.assert_array_equal(vic, ovic)
        pos += 1
    eng.sync()
    check(eng, orc, "cfg1 decode: ")


def test_decode_pool_exhaustion_matches_serial_semantics():
    """A decode append that runs out of pages behaves like the reference's
    serial loop of append_token calls: tables before the first failing pop
    (ascending table id) are appended, the failing one and all later ones are
    not, and PoolExhausted is reported (page_pool.cpp:26-28)."""
    rng = np.random.default_rng(12)
    B, C, d, H, S = 4, 8, 8, 1, 6
    lens = np.array([8, 7, 8, 3, 8, 8])  # tables 0, 2, 4, 5 will need a page on the next append
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    need = int(sum((L + B - 1) // B for L in lens))
    eng, orc = make_pair(n_seqs=S, n_layers=1, H=H, d=d, B=B, C=C, dtype=oracle.F32, cap=need + 2)
    k, _ = random_kv(rng, (cu[-1], H, d), oracle.F32)
    v, _ = random_kv(rng, (cu[-1], H, d), oracle.F32)
    eng.prefill_compress(0, dev(k), dev(v), cu)
    orc.prefill(0, k, v, cu)
    eng.sync()
    kk, _ = random_kv(rng, (1, S, H, d), oracle.F32)
    vv, _ = random_kv(rng, (1, S, H, d), oracle.F32)
    pos = lens.astype(np.int64)
    eng.append_token(0, 1, dev(kk), dev(vv), dev(pos))
    with pytest.raises(pe.PoolExhausted):
        eng.sync()
    assert orc.decode_append(0, 1, kk, vv, pos) == 2
    check(eng, orc, "exhaustion: ")
    assert list(eng.tables()[3]) == [9, 8, 9, 4, 8, 8]  # tables 0..3 appended, 4 failed, 5 stopped


@pytest.mark.slow
@pytest.mark.parametrize("long_path", ["stream", "cluster"])
def test_prefill_long_context_cluster_select(long_path, monkeypatch):
    """Tables longer than the CTA select limit (34816 tokens): the streamed
    CTA select (default) or the cluster select (PE_SELECT_LONG=cluster),
    2 sequences x 2 KV heads at 60000 / 50001 tokens."""
    if long_path == "cluster":
        monkeypatch.setenv("PE_SELECT_LONG", "cluster")
    rng = np.random.default_rng(60000)
    B, C, d, H = 16, 4096, 128, 2
    lens = np.array([60000, 50001])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, orc = make_pair(n_seqs=2, n_layers=1, H=H, d=d, B=B, C=C, dtype=oracle.BF16)
    k, _ = random_kv(rng, (cu[-1], H, d), oracle.BF16)
    v, _ = random_kv(rng, (cu[-1], H, d), oracle.BF16)
    ev = eng.prefill_compress(0, dev(k), dev(v), cu, evicted_counts=True)
    _, oev = orc.prefill(0, k, v, cu)
    np.testing.assert_array_equal(ev, oev)
    check(eng, orc, "long: ")


@pytest.mark.parametrize("long_path,mixed", [("stream", "1"), ("cluster", "1"), ("cluster", "0")])
def test_prefill_mixed_lengths_split_select(long_path, mixed, monkeypatch):
    """One prefill call with tables on both sides of the CTA select's limit
    (34816 tokens): the short ones take the shared-memory CTA select, the long
    ones the streamed CTA select (default) or the cluster select
    (PE_SELECT_LONG=cluster; with PE_SELECT_MIXED=0 every table takes it).
    Tie-heavy keys on one sequence; identity tables (L <= C) included."""
    monkeypatch.setenv("PE_SELECT_MIXED", mixed)
    if long_path == "cluster":
        monkeypatch.setenv("PE_SELECT_LONG", "cluster")
    rng = np.random.default_rng(34816)
    B, C, d, H = 16, 2048, 128, 2
    lens = np.array([40000, 1500, 34816, 9000, 34817, 700])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, orc = make_pair(n_seqs=len(lens), n_layers=1, H=H, d=d, B=B, C=C, dtype=oracle.BF16)
    k, _ = random_kv(rng, (cu[-1], H, d), oracle.BF16)
    v, _ = random_kv(rng, (cu[-1], H, d), oracle.BF16)
    kg, _ = grid_kv(rng, (lens[3], H, d), oracle.BF16)
    k[cu[3]:cu[4]] = kg
    ev = eng.prefill_compress(0, dev(k), dev(v), cu, evicted_counts=True)
    _, oev = orc.prefill(0, k, v, cu)
    np.testing.assert_array_equal(ev, oev)
    check(eng, orc, "mixed: ")


@pytest.mark.parametrize("mode", [0, 1])
def test_invariants_hold_after_prefill_and_decode(mode):
    """pe_check_invariants on a decoded engine: no violation, pages mapped +
    free == capacity; then a corrupted block table is detected."""
    rng = np.random.default_rng(77)
    B, C, d, H = 16, 64, 128, 2
    lens = np.array([300, 64, 17, 150])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    eng, orc = make_pair(n_seqs=len(lens), n_layers=2, H=H, d=d, B=B, C=C, dtype=oracle.BF16)
    for layer in range(2):
        k, _ = random_kv(rng, (cu[-1], H, d), oracle.BF16)
        v, _ = random_kv(rng, (cu[-1], H, d), oracle.BF16)
        eng.prefill_compress(layer, dev(k), dev(v), cu)
    pos = lens.astype(np.int64).copy()
    for step in range(1, 3 * B + 1):
        kk, _ = random_kv(rng, (2, len(lens), H, d), oracle.BF16)
        vv, _ = random_kv(rng, (2, len(lens), H, d), oracle.BF16)
        eng.decode_step(0, 2, dev(kk), dev(vv), torch.from_numpy(pos).cuda(), step, mode=mode)
        pos += 1
    eng.sync()
    inv = eng.check_invariants()
    assert inv["violations"] == 0, inv
    assert inv["pages_mapped"] + inv["free_pages"] == eng.capacity
    assert inv["tables_checked"] == eng.n_tables
    # corrupt: release a page that table 0 still maps (a double owner)
    bt, npg, _, _ = eng.tables()
    pid = int(bt[0, 0])
    assert eng.lib.pe_pool_release(eng.h, pid) == 0
    bad = eng.check_invariants()
    assert bad["page_refcount"] > 0 and bad["violations"] > 0, bad


@pytest.mark.slow
def test_cfg3_full_layer_sampled_against_reference(reference):
    """BASELINE config 3 at full size for one layer — Llama-3.1-8B KV geometry,
    64 sequences x 32768 tokens x 8 KV heads, C=4096, B=16, bf16 — then 16
    decode tokens (one block eviction per table). Six sampled tables are
    replayed through the UNMODIFIED reference (oracle/_ref: PagePool /
    BlockTable / make_policy(PagedEviction) / attend) on the same bytes:
    retained positions after prefill and after decode, every eviction
    decision, and the GQA attention output (<= 1e-3, bf16) must agree."""
    import oracle

    S, H, d, L, C, B, G = 64, 8, 128, 32768, 4096, 16, 4
    eng, _ = None, None
    geo = pe.EngineGeometry(n_seqs=S, n_layers=1, n_kv_heads=H, head_dim=d, dtype=oracle.BF16)
    eng = pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=C, page_size=B))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    k_in = torch.randn((S * L, H, d), generator=gen, device="cuda", dtype=torch.float32).to(torch.bfloat16)
    v_in = torch.randn((S * L, H, d), generator=gen, device="cuda", dtype=torch.float32).to(torch.bfloat16)
    cu = np.arange(S + 1, dtype=np.int32) * L
    eng.prefill_compress(0, k_in, v_in, cu)
    eng.sync()
    samples = [(0, 0), (13, 5), (31, 7), (42, 2), (50, 6), (63, 3)]
    ref = {}
    for sq, h in samples:
        sess = oracle.RefSession(reference, capacity=C // B + 2, page_size=B, budget=C, n_tables=1,
                                 width=d, kind=0)
        kk = k_in[sq * L:(sq + 1) * L, h].float().cpu().numpy()
        vv = v_in[sq * L:(sq + 1) * L, h].float().cpu().numpy()
        sess.prefill(0, kk, vv)
        ref[(sq, h)] = sess
        np.testing.assert_array_equal(eng.retained_positions(sq * H + h), sess.read_table(0, False)["positions"],
                                      err_msg=f"prefill survivors of table {(sq, h)}")
    del k_in, v_in
    torch.cuda.empty_cache()
    pos = torch.full((S,), L, dtype=torch.int64, device="cuda")
    for step in range(1, B + 1):
        rk = torch.randn((1, S, H, d), generator=gen, device="cuda", dtype=torch.float32).to(torch.bfloat16)
        rv = torch.randn((1, S, H, d), generator=gen, device="cuda", dtype=torch.float32).to(torch.bfloat16)
        vic = eng.decode_step(0, 1, rk, rv, pos, step, victims=True)
        for (sq, h), sess in ref.items():
            kind, idx = sess.decode_step(0, rk[0, sq, h].float().cpu().numpy(), rv[0, sq, h].float().cpu().numpy(),
                                         L + step - 1, step)
            want = idx if kind == 2 else -1
            assert int(vic[sq * H + h]) == want, (step, sq, h, int(vic[sq * H + h]), kind, idx)
        pos += 1
    eng.sync()
    assert eng.stats().pages_evicted == S * H  # one block per table
    q = torch.randn((S, H * G, d), generator=gen, device="cuda", dtype=torch.float32).to(torch.bfloat16)
    out = torch.empty((S, H * G, d), dtype=torch.float32, device="cuda")
    eng.attend(0, q, out, H * G)
    qf, of = q.float().cpu().numpy(), out.cpu().numpy()
    o = oracle.Oracle()
    for (sq, h), sess in ref.items():
        np.testing.assert_array_equal(eng.retained_positions(sq * H + h), sess.read_table(0, False)["positions"])
        for g in range(G):
            want = sess.attend(0, qf[sq, h * G + g], 1, d)
            assert o.output_deviation(of[sq, h * G + g], want) <= 1e-3


def test_hbm_probe_is_plausible():
    """pe_probe_hbm: the streaming-read and copy bandwidths the bench reports
    beside the roofline are in the B200's physical range."""
    import ctypes

    from paper_2509_04377_b200 import _lib

    rd, cp = ctypes.c_double(), ctypes.c_double()
    assert _lib.load().pe_probe_hbm(0, 1 << 30, 3, ctypes.byref(rd), ctypes.byref(cp)) == 0
    assert 3000 < rd.value < 9000, rd.value
    assert 2000 < cp.value < 9000, cp.value
