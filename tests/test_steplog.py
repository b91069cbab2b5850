"""Step log and run metrics in the reference's formats.

CPU:
* tests/cpp/metrics_fmt.cpp prints a fixed set of StepRecords / MetricsRecords
  through emit_jsonl / emit_csv / format_summary. The reference build
  (oracle/_ref/metrics_fmt_ref: metrics.cpp + its JSON library), the B200
  façade build and the Python mirror (steplog.py) must agree byte for byte,
  and with the committed output tests/golden/metrics_fmt_ref.txt.
* step_records' fragmentation ratios are the reference BlockTable's, bit for
  bit, on states driven through the reference objects.
GPU:
* the engine's device capture (pe_step_log_capture) over a decode run gives
  the same step-log JSONL and metrics CSV as the reference objects driven
  through the same run.
"""
from __future__ import annotations

import math
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2509_04377_b200 import steplog as sl
from tests.harness import RefReplay, grid_kv, random_kv

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden" / "metrics_fmt_ref.txt"

VALS = [0.0, -0.0, 1.0, 0.5, 0.1, 1.0 / 3.0, 2.0 / 3.0, 1e-4, 1e-5, 1.5e-5, 0.00031, 123.25, 1e15, 1e16, 1.5e20,
        9.999e14, 12345678901234567890.0, 4.9e-324, 1.7976931348623157e308, 0.0039215686274509665, 0.015625,
        0.99609375, 0.9375, math.nan]


def python_metrics_fmt() -> str:
    """The records of tests/cpp/metrics_fmt.cpp, through steplog.py."""
    steps = []
    n = len(VALS)
    for k, v in enumerate(VALS):
        r = sl.StepRecord(run=k % 3, sequence=k % 5, layer=k % 7, step=1 + k, retained_len=4096 + k,
                          fragmentation=v, deviation=VALS[(k + 5) % n])
        if k % 3 == 0:
            r.kind, r.logical_index = "page", k % 11
        elif k % 3 == 1:
            r.kind, r.positions = "tokens", [k, 7 * k, 1 << 40]
        steps.append(r)
    steps.append(sl.StepRecord(kind="tokens", positions=[], deviation=math.nan))
    out = sl.emit_jsonl(steps)
    policies = ["paged-eviction", "streaming-llm", "inv-key-l2", "key-diff", "full", "paged-eviction",
                'odd,"name"']
    recs = []
    for i, p in enumerate(policies):
        recs.append(sl.MetricsRecord(
            policy=p, cache_budget=1024 << (i % 3), page_size=16, prefill_len=4096 + 13 * i, decode_steps=256,
            batch=1 + i, layer_count=16, seed=20250904 + i, prefill_evicted=3072 * (i + 1),
            evictions_total=17 * i, page_evictions=16 * i, token_evictions=5 * i,
            block_table_updates=17 * i + (3 if i == 1 else 0), mean_fragmentation=VALS[i],
            max_fragmentation=VALS[i + 3], max_fragmentation_excl_newest=VALS[i + 9],
            mean_deviation=VALS[(i + 12) % 23], p95_deviation=1.0 / (3.0 + i), retained_bytes=1 << (30 + i)))
    out += sl.emit_csv(recs)
    out += sl.format_summary(sl.summarize(recs))
    out += sl.format_summary(sl.summarize(recs[4:5]))
    try:
        sl.summarize([])
    except ValueError:
        out += "EmptyInput\n"
    return out


def _run(binary: Path) -> str:
    if not binary.exists():
        pytest.skip(f"{binary.name} not built (tests/cpp/build_conformance.py)")
    return subprocess.run([str(binary)], capture_output=True, text=True, check=True, timeout=120).stdout


def test_reference_build_matches_golden():
    assert _run(ROOT / "oracle" / "_ref" / "metrics_fmt_ref") == GOLDEN.read_text()


def test_facade_emitters_byte_identical_to_reference():
    assert _run(ROOT / "tests" / "cpp" / "_build" / "metrics_fmt_b200") == GOLDEN.read_text()


def test_python_emitters_byte_identical_to_reference():
    got, want = python_metrics_fmt(), GOLDEN.read_text()
    for i, (a, b) in enumerate(zip(got.splitlines(), want.splitlines())):
        assert a == b, f"line {i}: python {a!r} vs reference {b!r}"
    assert got == want


def _ref_step_records(rep: RefReplay, victims, step):
    out = []
    for i, t in enumerate(_launch_tables(rep)):
        frag, fragx = rep.sess.fragmentation(t)
        v = int(victims[i])
        out.append(sl.StepRecord(sequence=i, step=step, retained_len=rep.sess.retained_len(t),
                                 kind="page" if v >= 0 else None, logical_index=max(v, 0), fragmentation=frag,
                                 fragmentation_excl_newest=fragx))
    return out


def _launch_tables(rep: RefReplay):
    return [rep.tid(s, li, h) for s in range(rep.n_seqs) for li in range(rep.n_layers) for h in range(rep.H)]


def _entries_from_reference(rep: RefReplay, victims):
    e = []
    for i, t in enumerate(_launch_tables(rep)):
        n = rep.sess.page_count(t)
        e.append([rep.sess.retained_len(t), n, rep._newest_fill(t) if n else 0, int(victims[i])])
    return np.array(e, dtype=np.int32)


def test_step_record_fragmentation_is_the_reference_blocktable(reference):
    """step_records' ratios == BlockTable::fragmentation_ratio[_excluding_newest]
    bit for bit, over prefill (identity and pruned) and decode with evictions."""
    rng = np.random.default_rng(11)
    B, C, w, H, S, NL = 8, 40, 8, 2, 3, 2
    lens = np.array([100, 17, 41])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    rep = RefReplay(reference, n_seqs=S, n_layers=NL, n_tab_heads=H, width=w, page_size=B, budget=C,
                    capacity=S * NL * H * (C // B + 2) + 8)
    for layer in range(NL):
        _, k = random_kv(rng, (cu[-1], H, w), oracle.F32)
        _, v = random_kv(rng, (cu[-1], H, w), oracle.F32)
        rep.prefill(layer, k, v, cu)
    pos = lens.astype(np.int64).copy()
    evictions = 0
    for step in range(1, 3 * B + 2):
        _, k = grid_kv(rng, (NL, S, H, w), oracle.F32)
        _, v = random_kv(rng, (NL, S, H, w), oracle.F32)
        vic = rep.decode(0, NL, k, v, pos, step)
        pos += 1
        got = sl.step_records(_entries_from_reference(rep, vic), B, step)
        want = _ref_step_records(rep, vic, step)
        for a, b in zip(got, want):
            assert a.fragmentation.hex() == b.fragmentation.hex()
            assert a.fragmentation_excl_newest.hex() == b.fragmentation_excl_newest.hex()
        assert sl.emit_jsonl(got) == sl.emit_jsonl(want)
        evictions += int((vic >= 0).sum())
    assert evictions > 0


@pytest.mark.gpu
def test_engine_step_log_matches_reference(reference):
    """Device capture after every decode step of the CUDA engine == the
    reference objects' StepRecords (JSONL byte-identical), and the run's
    metrics CSV row is identical."""
    torch = pytest.importorskip("torch")
    import paper_2509_04377_b200 as pe

    rng = np.random.default_rng(7)
    B, C, d, H, S, NL = 8, 40, 16, 2, 3, 2
    lens = np.array([100, 17, 41])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    geo = pe.EngineGeometry(n_seqs=S, n_layers=NL, n_kv_heads=H, head_dim=d, dtype=oracle.F32)
    eng = pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=C, page_size=B))
    rep = RefReplay(reference, n_seqs=S, n_layers=NL, n_tab_heads=H, width=d, page_size=B, budget=C,
                    capacity=eng.capacity)

    def dev(a):
        return torch.from_numpy(np.ascontiguousarray(a)).cuda()

    prefill_evicted = 0
    for layer in range(NL):
        k, _ = grid_kv(rng, (cu[-1], H, d), oracle.F32)
        v, _ = random_kv(rng, (cu[-1], H, d), oracle.F32)
        eng.prefill_compress(layer, dev(k), dev(v), cu)
        prefill_evicted += sum(len(x) for x in rep.prefill(layer, k, v, cu))
    pos = lens.astype(np.int64).copy()
    got_steps = [[] for _ in range(S)]
    want_steps = [[] for _ in range(S)]
    D = 3 * B + 5
    for step in range(1, D + 1):
        k, _ = random_kv(rng, (NL, S, H, d), oracle.F32)
        v, _ = grid_kv(rng, (NL, S, H, d), oracle.F32)
        vic = eng.decode_step(0, NL, dev(k), dev(v), dev(pos), step, victims=True)
        ref_vic = rep.decode(0, NL, k, v, pos, step)
        np.testing.assert_array_equal(vic, ref_vic)
        pos += 1
        entries = eng.step_log(0, NL)
        np.testing.assert_array_equal(entries, _entries_from_reference(rep, ref_vic))
        got = sl.step_records(entries, B, step)
        want = _ref_step_records(rep, ref_vic, step)
        assert sl.emit_jsonl(got) == sl.emit_jsonl(want)
        # per sequence, layer-minor (simulator order); one record per table
        per_seq = NL * H
        for s in range(S):
            got_steps[s] += got[s * per_seq:(s + 1) * per_seq]
            want_steps[s] += want[s * per_seq:(s + 1) * per_seq]
    _, _, _, retained = eng.tables()
    final = [[int(retained[rep.tid(s, li, h)]) for li in range(NL) for h in range(H)] for s in range(S)]
    kw = dict(policy="paged-eviction", cache_budget=C, page_size=B, prefill_len=int(lens.max()), decode_steps=D,
              layer_count=NL, seed=7, prefill_evicted=prefill_evicted, final_retained=final, head_count=1,
              head_dim=d)
    got_rec = sl.build_record(got_steps, **kw)
    want_rec = sl.build_record(want_steps, **kw)
    assert sl.emit_csv([got_rec]) == sl.emit_csv([want_rec])
    assert got_rec.page_evictions > 0
    # schemas/metrics.csv.md invariant: page_evictions * B + token_evictions
    # = tokens removed during decode = appended - (final - after prefill)
    after_prefill = sum(min(int(L), C) for L in lens) * NL * H
    removed = S * NL * H * D - (int(np.asarray(final).sum()) - after_prefill)
    assert got_rec.page_evictions * B + got_rec.token_evictions == removed
