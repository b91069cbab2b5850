"""Step log and run metrics in the reference's formats.

The reference's simulator logs one StepRecord per decode step per
(sequence, layer) and aggregates a run into one MetricsRecord
(metrics.hpp:16-80, simulator.cpp:203-249 and 355-400). Its emitters write
schemas/steplog.jsonl.md and schemas/metrics.csv.md. This module is the
Python side of the same formats for the batched engine:

* `PagedEvictionEngine.step_log()` captures, on the device, the engine-owned
  fields of every table after a decode step (pe_step_log_capture): retained
  length, page count, occupied slots of the newest page, evicted page.
* `step_records()` turns one capture into StepRecords. Fragmentation follows
  block_table.cpp:48-63 exactly.
* `build_record()` aggregates StepRecords like simulator.cpp:355-400.
* `emit_jsonl()`, `emit_csv()`, `summarize()` and `format_summary()` produce
  text byte-identical to the reference's for the same records. This is pinned
  by tests/test_steplog.py against the reference build
  (oracle/_ref/metrics_fmt_ref) and tests/golden/metrics_fmt_ref.txt.

The C++ façade offers the same functions (pagedevict::emit_jsonl, ...).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from decimal import Decimal
from typing import Iterable, Sequence

import numpy as np

__all__ = ["StepRecord", "MetricsRecord", "SummaryRow", "step_records", "build_record", "emit_jsonl",
           "emit_csv", "summarize", "format_summary", "POLICY_ORDER"]

# PolicyKind order and spellings (policy.hpp:17-29, policy.cpp to_string)
POLICY_ORDER = ["paged-eviction", "streaming-llm", "inv-key-l2", "key-diff", "full"]


@dataclass
class StepRecord:
    run: int = 0
    sequence: int = 0
    layer: int = 0
    step: int = 0
    retained_len: int = 0
    kind: str | None = None          # None | "tokens" | "page"
    positions: list[int] = field(default_factory=list)
    logical_index: int = 0
    fragmentation: float = 0.0
    fragmentation_excl_newest: float = 0.0
    deviation: float = math.nan      # NaN: no FullCache shadow


@dataclass
class MetricsRecord:
    policy: str = ""
    cache_budget: int = 0
    page_size: int = 0
    prefill_len: int = 0
    decode_steps: int = 0
    batch: int = 0
    layer_count: int = 0
    seed: int = 0
    prefill_evicted: int = 0
    evictions_total: int = 0
    page_evictions: int = 0
    token_evictions: int = 0
    block_table_updates: int = 0
    mean_fragmentation: float = 0.0
    max_fragmentation: float = 0.0
    max_fragmentation_excl_newest: float = 0.0
    mean_deviation: float = 0.0
    p95_deviation: float = 0.0
    retained_bytes: int = 0
    prefill_wall_ns: int = 0
    decode_wall_ns: int = 0


@dataclass
class SummaryRow:
    policy: str
    runs: int = 0
    evictions_total: int = 0
    block_table_updates: int = 0
    cadence_ratio: float = 0.0
    max_fragmentation_excl_newest: float = 0.0
    mean_deviation: float = 0.0


# ---------------------------------------------------------------- numbers
def _shortest(v: float) -> tuple[str, int, str]:
    """(sign, shortest round-trip digits, n) with |v| = 0.digits * 10**n."""
    t = Decimal(repr(abs(v))).as_tuple()
    digits = "".join(map(str, t.digits)).rstrip("0") or "0"
    n = len(t.digits) + t.exponent
    return ("-" if math.copysign(1.0, v) < 0 else ""), digits, n


def _exp(e: int) -> str:
    return ("e-" if e < 0 else "e+") + f"{abs(e):02d}"


def json_double(v: float) -> str:
    """The reference JSON library's double layout: shortest digits, '.0' on
    integral values, exponent form outside 1e-5 <= |v| < 1e15, NaN/inf null."""
    if not math.isfinite(v):
        return "null"
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    sign, d, n = _shortest(v)
    k = len(d)
    if k <= n <= 15:
        return sign + d + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + d[:n] + "." + d[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + d
    return sign + d[0] + ("." + d[1:] if k > 1 else "") + _exp(n - 1)


def csv_double(v: float) -> str:
    """std::to_chars(double) shortest form: the shorter of fixed and
    scientific notation over the shortest round-trip digits (ties: fixed)."""
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    if v == 0.0:
        return "-0" if math.copysign(1.0, v) < 0 else "0"
    sign, d, n = _shortest(v)
    k = len(d)
    if n >= k:  # integral: std::to_chars prints the exact integer value, not padded digits
        fixed = str(int(abs(v)))
    elif n > 0:
        fixed = d[:n] + "." + d[n:]
    else:
        fixed = "0." + "0" * (-n) + d
    sci = d[0] + ("." + d[1:] if k > 1 else "") + _exp(n - 1)
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def _csv_field(s: str) -> str:
    if not any(c in s for c in ',"\n'):
        return s
    return '"' + s.replace('"', '""') + '"'


# ---------------------------------------------------------------- emitters
def emit_jsonl(steps: Iterable[StepRecord]) -> str:
    """schemas/steplog.jsonl.md (metrics.cpp emit_jsonl)."""
    out = []
    for s in steps:
        if s.kind is None:
            dec = '{"kind":null}'
        elif s.kind == "tokens":
            dec = '{"kind":"tokens","positions":[' + ",".join(str(int(p)) for p in s.positions) + "]}"
        else:
            dec = '{"kind":"page","logical_index":' + str(int(s.logical_index)) + "}"
        out.append(f'{{"run":{s.run},"seq":{s.sequence},"layer":{s.layer},"step":{s.step},'
                   f'"retained_len":{s.retained_len},"decision":{dec},'
                   f'"fragmentation":{json_double(s.fragmentation)},"deviation":{json_double(s.deviation)}}}\n')
    return "".join(out)


CSV_HEADER = ("policy,cache_budget,page_size,prefill_len,decode_steps,batch,layer_count,seed,"
              "prefill_evicted,evictions_total,page_evictions,token_evictions,"
              "block_table_updates,mean_fragmentation,max_fragmentation,"
              "max_fragmentation_excl_newest,mean_deviation,p95_deviation,retained_bytes,"
              "prefill_wall_ns,decode_wall_ns\n")


def emit_csv(records: Iterable[MetricsRecord]) -> str:
    """schemas/metrics.csv.md (metrics.cpp emit_csv)."""
    out = [CSV_HEADER]
    for r in records:
        ints = [r.cache_budget, r.page_size, r.prefill_len, r.decode_steps, r.batch, r.layer_count, r.seed,
                r.prefill_evicted, r.evictions_total, r.page_evictions, r.token_evictions, r.block_table_updates]
        dbl = [r.mean_fragmentation, r.max_fragmentation, r.max_fragmentation_excl_newest, r.mean_deviation,
               r.p95_deviation]
        out.append(",".join([_csv_field(r.policy), *map(str, ints), *map(csv_double, dbl),
                             str(r.retained_bytes), str(r.prefill_wall_ns), str(r.decode_wall_ns)]) + "\n")
    return "".join(out)


def summarize(records: Sequence[MetricsRecord]) -> list[SummaryRow]:
    """Per-policy rows in PolicyKind order (metrics.cpp summarize)."""
    if not records:
        raise ValueError("EmptyInput: summarize requires at least one record")
    rows: dict[str, SummaryRow] = {}
    for r in records:
        row = rows.setdefault(r.policy, SummaryRow(r.policy))
        row.runs += 1
        row.evictions_total += r.evictions_total
        row.block_table_updates += r.block_table_updates
        row.max_fragmentation_excl_newest = max(row.max_fragmentation_excl_newest, r.max_fragmentation_excl_newest)
        row.mean_deviation += r.mean_deviation
    paged = float(rows["paged-eviction"].block_table_updates) if "paged-eviction" in rows else 0.0
    out = []
    for name in POLICY_ORDER:
        if name not in rows:
            continue
        row = rows[name]
        row.mean_deviation /= row.runs
        row.cadence_ratio = row.block_table_updates / paged if paged > 0.0 else math.nan
        out.append(row)
    return out


def format_summary(rows: Iterable[SummaryRow]) -> str:
    out = [f"{'policy':<16}{'runs':>6}{'evictions':>11}{'table_updates':>15}{'cadence':>10}"
           f"{'max_frag_excl_newest':>22}{'mean_deviation':>16}\n"]
    for r in rows:
        cad = "n/a" if math.isnan(r.cadence_ratio) else f"{r.cadence_ratio:.4f}"
        out.append(f"{r.policy:<16}{r.runs:>6}{r.evictions_total:>11}{r.block_table_updates:>15}{cad:>10}"
                   f"{r.max_fragmentation_excl_newest:>22.4f}{r.mean_deviation:>16.4f}\n")
    return "".join(out)


# ---------------------------------------------------------------- engine side
def step_records(entries: np.ndarray, page_size: int, step: int, run: int = 0,
                 sequences: Sequence[int] | None = None, layers: Sequence[int] | None = None) -> list[StepRecord]:
    """StepRecords of one pe_step_log_capture (entries [n, 4] int32:
    retained_len, page_count, newest_fill, victim), in capture order;
    `sequences` / `layers` label each entry (default: its index / 0)."""
    e = np.asarray(entries, dtype=np.int64).reshape(-1, 4)
    out = []
    for i, (ret, npg, fill, vic) in enumerate(e.tolist()):
        frag = 1.0 - float(ret) / (float(npg) * page_size) if npg > 0 else 0.0
        fragx = 1.0 - float(ret - fill) / (float(npg - 1) * page_size) if npg > 1 else 0.0
        out.append(StepRecord(run=run, sequence=int(sequences[i]) if sequences is not None else i,
                              layer=int(layers[i]) if layers is not None else 0, step=step, retained_len=int(ret),
                              kind="page" if vic >= 0 else None, logical_index=max(int(vic), 0),
                              fragmentation=frag, fragmentation_excl_newest=fragx))
    return out


def memory_bytes(seq_len: int, layer_count: int, head_count: int, head_dim: int, bytes_per_elem: int) -> int:
    """page_pool.cpp memory_bytes: 2 (K and V) * S * L * H * d * bytes."""
    return 2 * seq_len * layer_count * head_count * head_dim * bytes_per_elem


def build_record(steps_by_sequence: Sequence[Sequence[StepRecord]], *, policy: str, cache_budget: int,
                 page_size: int, prefill_len: int, decode_steps: int, layer_count: int, seed: int,
                 prefill_evicted: int, final_retained: Sequence[Sequence[int]], head_count: int,
                 head_dim: int) -> MetricsRecord:
    """Aggregates a run like simulator.cpp:355-400: sums in sequence-major,
    step-major, layer-minor order (the order of `steps_by_sequence[s]`)."""
    rec = MetricsRecord(policy=policy, cache_budget=cache_budget, page_size=page_size, prefill_len=prefill_len,
                        decode_steps=decode_steps, batch=len(steps_by_sequence), layer_count=layer_count, seed=seed,
                        prefill_evicted=prefill_evicted)
    frag_sum, frag_n, devs = 0.0, 0, []
    for seq_steps, retained in zip(steps_by_sequence, final_retained):
        for s in seq_steps:
            if s.kind == "tokens":
                rec.evictions_total += 1
                rec.block_table_updates += 1
                rec.token_evictions += len(s.positions)
            elif s.kind == "page":
                rec.evictions_total += 1
                rec.block_table_updates += 1
                rec.page_evictions += 1
            frag_sum += s.fragmentation
            frag_n += 1
            rec.max_fragmentation = max(rec.max_fragmentation, s.fragmentation)
            rec.max_fragmentation_excl_newest = max(rec.max_fragmentation_excl_newest, s.fragmentation_excl_newest)
            if not math.isnan(s.deviation):
                devs.append(s.deviation)
        for r in retained:
            rec.retained_bytes += memory_bytes(int(r), 1, head_count, head_dim, 2)
    if frag_n:
        rec.mean_fragmentation = frag_sum / frag_n
    if devs:
        total = 0.0
        for d in devs:
            total += d
        rec.mean_deviation = total / len(devs)
        devs.sort()
        rec.p95_deviation = devs[min(math.ceil(0.95 * len(devs)) - 1, len(devs) - 1)]
    return rec
