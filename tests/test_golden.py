"""Golden fixtures produced by the compiled reference (tests/golden/
make_golden.py): the C oracle (CPU) and the CUDA engine (GPU) must
reproduce them bit for bit (attention within tolerance)."""
from pathlib import Path

import numpy as np
import pytest

import oracle

GOLD = Path(__file__).resolve().parent / "golden"


def load(name):
    return dict(np.load(GOLD / name))


def score_rows():
    d = load("scores.npz")
    for i in range(int(d["n"][0])):
        yield d[f"k{i}"], d[f"v{i}"], d[f"s{i}"].view(np.float64)[0]


@pytest.mark.parametrize("dtype", [oracle.F32, oracle.BF16])
def test_oracle_scores_match_golden(oracle_lib, dtype):
    for k, v, s in score_rows():
        if dtype == oracle.BF16:
            k, v = oracle.f32_to_bf16_bits(k), oracle.f32_to_bf16_bits(v)
        assert oracle_lib.token_score(k, v) == s


def _cast(x, dtype):
    return oracle.f32_to_bf16_bits(x) if dtype == oracle.BF16 else np.ascontiguousarray(x, np.float32)


def _check_trace_state(d, bt, npg, nf, retained_pos_fn, free_list):
    n = d["num_pages"].size
    np.testing.assert_array_equal(npg, d["num_pages"])
    off = 0
    for t in range(n):
        np.testing.assert_array_equal(bt[t, : npg[t]], d["phys"][t, : npg[t]])
        L = int(d["retained_len"][t])
        np.testing.assert_array_equal(retained_pos_fn(t), d["retained"][off: off + L])
        off += L
    np.testing.assert_array_equal(free_list, d["free_list"])
    np.testing.assert_array_equal(free_list[::-1], d["drain"])


@pytest.mark.parametrize("dtype", [oracle.F32, oracle.BF16])
def test_oracle_trace_matches_golden(dtype):
    d = load("trace.npz")
    S, NL, H, w, B, C = (int(d[x]) for x in ("S", "NL", "H", "w", "B", "C"))
    eng = oracle.OracleEngine(n_seqs=S, n_layers=NL, n_tab_heads=H, width=w, page_size=B,
                              budget=C, dtype=dtype, capacity=int(d["cap"]), max_pages=C // B + 1)
    for layer in range(NL):
        st, ev = eng.prefill(layer, _cast(d[f"pk{layer}"], dtype), _cast(d[f"pv{layer}"], dtype),
                             d["cu"])
        assert st == 0
        np.testing.assert_array_equal(ev, d[f"pev{layer}"])
    pos = np.diff(d["cu"]).astype(np.int64)
    for stp in range(d["dk"].shape[0]):
        assert eng.decode_append(0, NL, _cast(d["dk"][stp], dtype), _cast(d["dv"][stp], dtype), pos) == 0
        _, vic = eng.decode_evict(0, NL)
        np.testing.assert_array_equal(vic, d["victims"][stp])
        pos += 1
    bt, npg, nf = eng.block_table(), eng.num_pages(), eng.newest_fill()
    positions = eng.positions()

    def retained(t):
        out = []
        for j in range(npg[t]):
            fill = B if j < npg[t] - 1 else nf[t]
            out.append(positions[bt[t, j], :fill])
        return np.concatenate(out)

    _check_trace_state(d, bt, npg, nf, retained, eng.free_stack())
    for layer in range(NL):
        st, out = eng.attention(layer, _cast(d["q"], dtype), int(d["G"]))
        np.testing.assert_array_equal(out, d["attn"][layer])  # same double arithmetic


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [oracle.F32, oracle.BF16])
def test_engine_scores_match_golden(dtype):
    torch = pytest.importorskip("torch")
    import paper_2509_04377_b200 as pe

    by_w = {}
    for k, v, s in score_rows():
        by_w.setdefault(k.size, []).append((k, v, s))
    for w, rows in by_w.items():
        n = len(rows)
        C = ((n + 15) // 16) * 16
        eng = pe.PagedEvictionEngine(
            pe.EngineGeometry(n_seqs=1, n_layers=1, n_kv_heads=1, head_dim=w, dtype=dtype),
            pe.PolicyConfig(cache_budget=C, page_size=16))
        k = np.stack([_cast(r[0], dtype) for r in rows])[:, None, :]
        v = np.stack([_cast(r[1], dtype) for r in rows])[:, None, :]
        eng.prefill_compress(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(),
                             np.array([0, n], np.int32))
        eng.sync()
        bt, npg, nf, _ = eng.tables()
        _, ts, _ = eng.positions(scores=True)
        got = np.concatenate([ts[bt[0, j], :(16 if j < npg[0] - 1 else nf[0])] for j in range(npg[0])])
        want = np.array([r[2] for r in rows])
        np.testing.assert_array_equal(got.view(np.uint64), want.view(np.uint64), err_msg=f"w={w}")


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [oracle.F32, oracle.BF16])
def test_engine_trace_matches_golden(dtype):
    torch = pytest.importorskip("torch")
    import paper_2509_04377_b200 as pe

    d = load("trace.npz")
    S, NL, H, w, B, C, G = (int(d[x]) for x in ("S", "NL", "H", "w", "B", "C", "G"))
    eng = pe.PagedEvictionEngine(
        pe.EngineGeometry(n_seqs=S, n_layers=NL, n_kv_heads=H, head_dim=w, dtype=dtype,
                          capacity=int(d["cap"])),
        pe.PolicyConfig(cache_budget=C, page_size=B))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    for layer in range(NL):
        ev = eng.prefill_compress(layer, dev(_cast(d[f"pk{layer}"], dtype)),
                                  dev(_cast(d[f"pv{layer}"], dtype)), d["cu"], evicted_counts=True)
        np.testing.assert_array_equal(ev, d[f"pev{layer}"])
    pos = np.diff(d["cu"]).astype(np.int64)
    for stp in range(d["dk"].shape[0]):
        vic = eng.decode_step(0, NL, dev(_cast(d["dk"][stp], dtype)), dev(_cast(d["dv"][stp], dtype)),
                              dev(pos), stp + 1, victims=True)
        np.testing.assert_array_equal(vic, d["victims"][stp])
        pos += 1
    eng.sync()
    bt, npg, nf, _ = eng.tables()
    _check_trace_state(d, bt, npg, nf, eng.retained_positions, eng.free_list())
    tol = 1e-5 if dtype == oracle.F32 else 1e-3
    orc = oracle.Oracle()
    for layer in range(NL):
        out = torch.empty((S, H * G, w), dtype=torch.float32, device="cuda")
        eng.attend(layer, dev(_cast(d["q"], dtype)), out, H * G)
        got = out.cpu().numpy()
        for s in range(S):
            for hq in range(H * G):
                assert orc.output_deviation(got[s, hq], d["attn"][layer, s, hq]) <= tol
