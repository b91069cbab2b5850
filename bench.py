#!/usr/bin/env python3
"""PagedEviction hot-path benchmark (BASELINE.json metric):

    eviction step HBM GB/s (% of peak); p50 evict-step µs; pruned decode tokens/s

Workload (default, the N=1 line): BASELINE config 3 — Llama-3.1-8B KV
geometry (32 layers, 8 KV heads, head_dim 128, 32 query heads), batch 64,
32K-token prompts, budget C=4096, page size B=16, bf16, PER_KV_HEAD tables
(16384 per GPU). Weak scaling: every rank holds its own 64 sequences (own
pool, tables and free list; no data-path collective).

`--config cfg5`: BASELINE config 5 — 1024 sequences at 128K context, sharded
by sequence across the ranks (strong scaling: 1024/N sequences per rank, one
layer's 8192 tables in total); prefill streamed in sequence waves.

`--gpus N`: N ranks, one per GPU. Launched by the driver under torchrun
(WORLD_SIZE/RANK/LOCAL_RANK from the environment); run directly with N > 1
it re-executes itself under `torch.distributed.run`. N larger than the
visible GPUs is an error. NCCL carries only the barrier, the max-over-ranks
time and one small stats gather.

Setup (untimed, measured with CUDA events and reported under "prefill"): K1
prefill prune+pack of every layer from synthetic N(0,1) K/V.

One bench STEP = one eviction cycle of the whole batch: B=16 decode tokens
appended to every table (K0, one launch per token over all layers) followed
by the PagedEviction block eviction of every table (K2, pages rescored from
their resident K/V bytes; by default one launch per layer, issued back to
back as a serving loop does, consecutive launches overlapping through
programmatic dependent launch; `--evict-launch step` runs ONE launch
covering all layers — each table's decision depends only on that table; the
other granularity is reported too). `value` =
algorithmic bytes of the step, summed over ranks (K2: (C+B)*row + 8*(C/B+1)
+ 4 per table; K0: 2*row+4 per table per token) / the max over ranks of the
step's device time.

`e2e`: the same cycle through the C-ABI with HOST buffers: every token's K/V
rows are copied from pinned host memory inside the timed region and the
victims are read back to host after every eviction launch (recompute scores;
`e2e.cached` the same with the cached-score eviction K2c).

`decode`: pruned decode tokens/s (K0 + K2 or K2c at the trigger + K3 on every
layer) against FullCache (no eviction, the unpruned table growing from L:
K0 + K3, measured on one layer and multiplied by the layer count).

`--impl reference`: the reference's own CPU implementation (oracle/_ref,
compiled from the reference sources) on the same config, all host threads,
on a bounded sample of tables; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "eviction step HBM GB/s (% of peak); p50 evict-step µs; pruned decode tokens/s"

CONFIGS = {
    # seqs: per rank (weak scaling) or in total (strong scaling, sharded by sequence)
    "cfg1": dict(layers=16, kvh=8, d=64, qh=32, seqs=1, L=4096, C=1024, dtype="f32", scaling="weak",
                 desc="Llama-3.2-1B KV geometry, 1 seq, 4K fp32 prefill, C=1024"),
    "cfg2": dict(layers=28, kvh=8, d=128, qh=24, seqs=32, L=16384, C=2048, dtype="bf16", scaling="weak",
                 desc="Llama-3.2-3B KV geometry, batch 32, 16K context, C=2048, bf16"),
    "cfg3": dict(layers=32, kvh=8, d=128, qh=32, seqs=64, L=32768, C=4096, dtype="bf16", scaling="weak",
                 desc="Llama-3.1-8B KV geometry, batch 64, 32K context, C=4096, bf16"),
    "cfg5": dict(layers=1, kvh=8, d=128, qh=32, seqs=1024, L=131072, C=4096, dtype="bf16", scaling="strong",
                 wave_seqs=16,
                 desc="Llama-3.1-8B KV geometry, 1024 sequences x 128K context sharded by sequence across "
                      "the ranks, one layer (8192 tables in total), C=4096, bf16"),
    # a small configuration for the multi-rank plumbing tests
    "tiny": dict(layers=2, kvh=8, d=128, qh=32, seqs=4, L=8192, C=1024, dtype="bf16", scaling="weak",
                 desc="test configuration: 8B KV geometry, 2 layers, 4 x 8K, C=1024"),
}
B = 16


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def ncu_traffic(kernel_substr="evict_score_kernel", expect_bytes=None):
    """Mean DRAM bytes (read+write) per launch of `kernel_substr` from the
    committed ncu launch list of this command (profiles/*bench_launches*.csv,
    `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
    dram__bytes_write.sum ... python bench.py`), or None."""
    import csv
    import glob

    files = sorted(glob.glob(str(ROOT / "profiles" / "*bench_launches*.csv")))
    if not files:
        return None
    rows = list(csv.reader(open(files[-1])))
    try:
        h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    except IndexError:
        return None
    hdr = rows[h]
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = {}
    for r in rows[h + 1:]:
        if kernel_substr in r[ki] and r[mi].startswith("dram__bytes"):
            per[r[ii]] = per.get(r[ii], 0.0) + float(r[vi].replace(",", "")) * (
                1e9 if "Gbyte" in r[hdr.index("Metric Unit")] else 1e6 if "Mbyte" in r[hdr.index("Metric Unit")]
                else 1.0)
    vals = list(per.values())
    if expect_bytes:  # launches of the same size as the measured one (the list holds both granularities)
        vals = [v for v in vals if 0.5 * expect_bytes < v < 2.0 * expect_bytes]
    return round(sum(vals) / len(vals)) if vals else None


# --------------------------------------------------------------------------- helpers
def k2_bytes_per_table(C, row):
    return (C + B) * row + 8 * (C // B + 1) + 4


def k1_bytes_per_table(L, C, row):
    keep = min(L, C)
    return L * row + keep * row + 4 * keep + 4 * ((keep + B - 1) // B)


def k3_bytes_per_table(R, row, G, d, q_elt):
    return R * row + 4 * ((R + B - 1) // B) + G * d * (q_elt + 4)


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def rank_seqs(cfg, world, rank):
    """(first sequence, sequence count) of this rank: weak scaling gives every
    rank cfg['seqs'] sequences of its own; strong scaling shards cfg['seqs']."""
    if cfg["scaling"] == "strong":
        from paper_2509_04377_b200.dist import shard

        lo, hi = shard(cfg["seqs"], world, rank)
        return lo, hi - lo
    return rank * cfg["seqs"], cfg["seqs"]


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args) -> int:
    """`python bench.py --gpus N` (N > 1) outside torchrun: one rank per GPU
    under torch.distributed.run, rendezvous on 127.0.0.1."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(Path(__file__).resolve())]
    cmd += sys.argv[1:]
    return subprocess.call(cmd)


# --------------------------------------------------------------------------- CPU reference
def cpu_legs(cfg, threads, decode_tables, decode_cycles, single: bool):
    """The reference's own CPU implementation of the three kernels' work, on
    bounded samples, with `threads` host threads (and a single-thread run
    when `single`): decode eviction cycles (make_kv + decode_step x16, one
    PagedEviction trigger), prefill (make_kv + prefill_compress + append of
    the survivors, policy.cpp:54-63) and attention (attend per query head,
    attention.cpp:97-99). Rates are converted to "equivalent GB/s" over the
    same algorithmic bytes as the GPU kernels."""
    import oracle

    ref = oracle.Reference()
    C, d, L = cfg["C"], cfg["d"], cfg["L"]
    G = cfg["qh"] // cfg["kvh"]
    elt = 2 if cfg["dtype"] == "bf16" else 4
    row_alg = 2 * d * elt
    cycle_bytes = k2_bytes_per_table(C, row_alg) + B * (2 * row_alg + 4)
    out = {}

    def leg(name, fn, n_tables, unit_bytes, th, sample):
        secs = fn(n_tables, th)
        return {"tables_per_s": round(n_tables / secs, 2), "gbs": round(n_tables * unit_bytes / secs / 1e9, 3),
                "seconds": round(secs, 4), "threads": th, "sample": sample}

    def dec(n, th):
        secs, ev = ref.bench_decode_cycles(n, C, B, d, th, decode_cycles, seed=7, warmup_cycles=1)
        assert ev == n * decode_cycles, (ev, n)
        return secs / decode_cycles

    runs = [(threads, 1)] + ([(1, 16)] if single and threads > 1 else [])
    for th, div in runs:
        key = "all_cores" if th == threads else "single_thread"
        nt_dec = max(th, decode_tables // div)
        nt_pre = max(th, (4 * threads) // div)
        nt_att = max(th, (16 * threads) // div)
        out[key] = {
            "decode_cycle": leg("decode", dec, nt_dec, cycle_bytes, th,
                                f"{nt_dec} tables x {decode_cycles} cycles, identity-prefilled to C"),
            "prefill": leg("prefill", lambda n, t: ref.bench_prefill(n, L, C, B, d, t), nt_pre,
                           k1_bytes_per_table(L, C, row_alg), th, f"{nt_pre} tables of {L} tokens"),
            "attention": leg("attention", lambda n, t: ref.bench_attend(n, C + B // 2, B, d, G, t), nt_att,
                             k3_bytes_per_table(C + B // 2, row_alg, G, d, elt), th,
                             f"{nt_att} tables of {C + B // 2} tokens x {G} query heads"),
        }
    return out


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return
    import oracle

    ref = oracle.Reference()
    threads = os.cpu_count() or 1
    row_alg = 2 * cfg["d"] * (2 if cfg["dtype"] == "bf16" else 4)
    C = cfg["C"]
    # bounded sample: `tables` tables per step, `cps` eviction cycles each
    tables = args.ref_tables or 1024
    cps = 8
    secs, ev = ref.bench_decode_cycles(tables, C, B, cfg["d"], threads, args.steps * cps, seed=1,
                                       warmup_cycles=args.warmup)
    assert ev == tables * args.steps * cps, (ev, tables)
    per_step = secs / args.steps
    bytes_step = cps * tables * (k2_bytes_per_table(C, row_alg) + B * (2 * row_alg + 4))
    value = bytes_step / per_step / 1e9
    legs = cpu_legs(cfg, threads, 1024, 16, single=True)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(per_step * 1e3, 3), "higher_is_better": True, "scaling": cfg["scaling"],
        "vs_baseline": None, "dtype": "f64", "data": "synthetic N(0,1) (reference GaussianStream)",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "tables_sampled": tables,
                   "cycle": "B=16 decode_step calls per table incl. one PagedEviction trigger",
                   "cycles_per_step": cps},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"{tables} tables x {cps} eviction cycles per step "
                                   f"(make_kv + EvictionPolicy::decode_step x16), identity-prefilled to C",
                         "legs": legs},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "p50_evict_step_us_per_table": round(per_step / cps / tables * threads * 1e6, 3),
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, args):
    """Reference CPU path on the host cores, bounded sample (~10-30 s)."""
    try:
        import oracle

        ref = oracle.Reference()
    except Exception as exc:  # reference library not built
        return {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference",
                "sample": f"unavailable: {exc}"}
    threads = os.cpu_count() or 1
    tables = args.ref_tables or 1024
    cycles = 256
    row_alg = 2 * cfg["d"] * (2 if cfg["dtype"] == "bf16" else 4)
    secs, ev = ref.bench_decode_cycles(tables, cfg["C"], B, cfg["d"], threads, cycles, seed=7,
                                       warmup_cycles=1)
    bytes_step = cycles * tables * (k2_bytes_per_table(cfg["C"], row_alg) + B * (2 * row_alg + 4))
    return {"value": round(bytes_step / secs / 1e9, 3), "unit": "GB/s", "cores": threads,
            "kind": "reference", "cpu_model": cpu_model(),
            "sample": f"{tables} of the {args.config} tables x {cycles} eviction cycles (16 make_kv + "
                      f"EvictionPolicy::decode_step each, one PagedEviction trigger), {secs:.3f} s timed "
                      f"on {threads} threads; identity-prefilled to C (setup untimed)",
            "evictions": int(ev),
            "legs": cpu_legs(cfg, threads, 1024, 16, single=True)}


# --------------------------------------------------------------------------- B200 arm
def run_b200(args, cfg, world, rank, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2509_04377_b200 as pe
    from paper_2509_04377_b200.dist import RankStats, gather_stats, max_over_ranks as _mor, sum_over_ranks as _sor

    n_dev = torch.cuda.device_count()
    if args.share_device:  # test-only: every rank on device 0, gloo plumbing
        local_dev = 0
    else:
        if world > n_dev:
            raise SystemExit(f"bench.py: --gpus {world} needs {world} visible GPUs, found {n_dev}")
        local_dev = local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if args.share_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def max_over_ranks(x):
        return _mor(x, device=None if args.share_device else dev)

    def sum_over_ranks(x):
        return _sor(x, device=None if args.share_device else dev)

    peak, peak_kind = load_peaks()
    # live HBM probe (untimed): K2 is read-only traffic, so its roofline is
    # also reported against the streaming-read bandwidth of this GPU
    import ctypes as _C

    from paper_2509_04377_b200 import _lib as _pl

    _rd, _cp = _C.c_double(0.0), _C.c_double(0.0)
    probe_ok = _pl.load().pe_probe_hbm(local_dev, 8 << 30, 5, _C.byref(_rd), _C.byref(_cp)) == 0
    probe = {"read_gbs": round(_rd.value, 1), "kind": "256-bit streaming read of 8 GiB, best of 5 (pe_probe_hbm)"} \
        if probe_ok else None
    bf16 = cfg["dtype"] == "bf16"
    tdt = torch.bfloat16 if bf16 else torch.float32
    elt = 2 if bf16 else 4
    NL, H, d, L, C, QH = cfg["layers"], cfg["kvh"], cfg["d"], cfg["L"], cfg["C"], cfg["qh"]
    seq0, S = rank_seqs(cfg, world, rank)
    G = QH // H
    row = 2 * d * elt  # K+V
    geo = pe.EngineGeometry(n_seqs=S, n_layers=NL, n_kv_heads=H, head_dim=d,
                            dtype=pe.DTYPE_BF16 if bf16 else pe.DTYPE_F32, device=local_dev)
    eng = pe.PagedEvictionEngine(geo, pe.PolicyConfig(cache_budget=C, page_size=B))
    stream = torch.cuda.current_stream()
    gen = torch.Generator(device=dev)
    gen.manual_seed(20250904 + 3 + 1000 * rank)

    # ---------------- setup: K1 prefill prune+pack of every layer (event-timed),
    # in sequence waves when the raw prompts of the rank do not fit at once
    wave = min(S, cfg.get("wave_seqs", S))
    k_in = torch.empty((wave * L, H, d), dtype=tdt, device=dev)
    v_in = torch.empty_like(k_in)
    pre_ms = []
    for layer in range(NL):
        ms = 0.0
        for w0 in range(0, S, wave):
            nw = min(wave, S - w0)
            k_in[: nw * L].normal_(generator=gen)
            v_in[: nw * L].normal_(generator=gen)
            cu = np.arange(nw + 1, dtype=np.int32) * L
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            eng.prefill_compress(layer, k_in[: nw * L], v_in[: nw * L], cu, seq_begin=w0)
            e1.record(stream)
            e1.synchronize()
            ms += e0.elapsed_time(e1)
        pre_ms.append(ms)
    eng.sync()
    del k_in, v_in
    torch.cuda.empty_cache()
    n_tab_layer = S * H
    k1_bytes = n_tab_layer * k1_bytes_per_table(L, C, row)
    pre_p50 = statistics.median(pre_ms[1:] or pre_ms)
    prefill = {"kernel": "K1 prefill_prune_pack: score + GPU-wide select (window/count/resolve/emit) + rescoring copy, "
                         "2 sequence waves on 2 streams",
               "ms_per_layer_p50": round(pre_p50, 4),
               "gbs": round(k1_bytes / (pre_p50 * 1e-3) / 1e9, 1),
               "tables_per_layer": n_tab_layer, "prompt_waves": (S + wave - 1) // wave,
               "algorithmic_bytes_per_layer": k1_bytes}
    prefill["frac"] = round(prefill["gbs"] / peak, 4)

    # ---------------- decode inputs: B tokens of rows for every table (device + pinned host)
    # every decode token's positions, precomputed (no per-token increment kernel)
    # cycles that append: warm-up W + timed K + p50 extras max(0, 100 - K) + 4
    # cached + 2 other-granularity + 2 x (1 + K) e2e + 2 decode (+ margin)
    max_tokens = B * (args.warmup + 3 * max(1, args.steps) + max(0, 100 - args.steps) + 16)
    pos_all = (L + torch.arange(max_tokens, device=dev, dtype=torch.int64)).unsqueeze(1).expand(
        max_tokens, S).contiguous()
    tok = [0]

    def next_pos():
        p = pos_all[tok[0]]
        tok[0] += 1
        return p
    rows_k = torch.randn((B, NL, S, H, d), generator=gen, device=dev, dtype=torch.float32).to(tdt)
    rows_v = torch.randn((B, NL, S, H, d), generator=gen, device=dev, dtype=torch.float32).to(tdt)
    h_k = rows_k.cpu().pin_memory()
    h_v = rows_v.cpu().pin_memory()
    n_tab = S * NL * H
    k2_alg = n_tab * k2_bytes_per_table(C, row)          # per step (all layers)
    k0_alg = n_tab * B * (2 * row + 4)                   # read + write rows, positions
    step_bytes = k2_alg + k0_alg
    k2_per_launch = (n_tab if args.evict_launch == "step" else n_tab_layer) * k2_bytes_per_table(C, row)

    cycles = [0]  # eviction cycles run on every table (cadence check)
    k0_evs = []  # (start, end) around each cycle's B append launches (timed cycles only)

    def cycle(record=None, host=False, mode=pe.ScoreMode.RECOMPUTE, victims_host=None):
        cycles[0] += 1
        if record is not None and not host and mode == pe.ScoreMode.RECOMPUTE:
            k0_evs.append((torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)))
            k0_evs[-1][0].record(stream)
        for j in range(B):
            if host:
                eng.append_token(0, NL, h_k[j], h_v[j], next_pos())
            else:
                eng.append_token(0, NL, rows_k[j], rows_v[j], next_pos())
        if record is not None and not host and mode == pe.ScoreMode.RECOMPUTE:
            k0_evs[-1][1].record(stream)
        spans = [(0, NL)] if args.evict_launch == "step" else [(layer, 1) for layer in range(NL)]
        # one event pair around the cycle's eviction launches: per-layer
        # launches run back to back (consecutive K2 launches over disjoint
        # layers overlap through programmatic dependent launch); each recorded
        # entry is (start, end, launches) -> per-launch time = elapsed / launches
        if record is not None:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if mode == pe.ScoreMode.CACHED:
                # a ~50 us launch: keep the GPU busy so the event pair brackets
                # device time, not the host's launch latency
                torch.cuda._sleep(200_000)
            a.record(stream)
        for l0, nl in spans:
            # e2e: every launch writes its victims into the step's device
            # buffer, read back to host ONCE per step below (a serving loop
            # reads the step's decisions, not one small copy per layer)
            vd = vict_dev[l0 * n_tab_layer: (l0 + nl) * n_tab_layer] if victims_host is not None else None
            eng.evict(l0, nl, step=0, mode=mode, victims=vd)
        if victims_host is not None:
            victims_host.copy_(vict_dev, non_blocking=True)
        if record is not None:
            b.record(stream)
            record.append((a, b, len(spans)))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        cycle()
    eng.sync()

    launches0 = eng.stats().kernel_launches
    evs = []
    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_dev) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            cycle(record=evs)
        t1.record(stream)
        barrier()
    eng.sync()
    launches = eng.stats().kernel_launches - launches0
    ms_total = max_over_ranks(t0.elapsed_time(t1))
    ms_step = ms_total / args.steps
    total_step_bytes = sum_over_ranks(float(step_bytes))
    k2_ms = [a.elapsed_time(b) / n for a, b, n in evs]
    k2_mean = statistics.mean(k2_ms)
    value = total_step_bytes / (ms_step * 1e-3) / 1e9
    k2_gbs = k2_per_launch / (k2_mean * 1e-3) / 1e9
    # p50 evict-step µs over >= 100 trigger launches: extra
    # cycles after the timed region when --steps is smaller (not in `value`)
    evs_p50 = list(evs)
    while sum(n for _, _, n in evs_p50) < 100 * (1 if args.evict_launch == "step" else NL):
        cycle(record=evs_p50)
    eng.sync()
    k2_p50_ms = statistics.median(a.elapsed_time(b) / n for a, b, n in evs_p50)  # per launch
    # the whole eviction step of a cycle (every layer), whatever the launch granularity
    k2_step_p50_ms = statistics.median(a.elapsed_time(b) for a, b, _ in evs_p50)

    # ---------------- cached-score variant (K2c): p50 of the evict launch
    evc = []
    for _ in range(4):
        cycle(record=evc, mode=pe.ScoreMode.CACHED)
    eng.sync()
    k2c_us = statistics.median([a.elapsed_time(b) * 1e3 / n for a, b, n in evc])  # per launch
    k2c_step_us = statistics.median([a.elapsed_time(b) * 1e3 for a, b, _ in evc])

    # ---------------- the other launch granularity, for reference
    other = "layer" if args.evict_launch == "step" else "step"
    saved = args.evict_launch
    args.evict_launch = other
    evo = []
    for _ in range(2):
        cycle(record=evo)
    eng.sync()
    args.evict_launch = saved
    other_us = statistics.median([a.elapsed_time(b) * 1e3 / n for a, b, n in evo])
    other_bytes = (n_tab if other == "step" else n_tab_layer) * k2_bytes_per_table(C, row)

    # ---------------- e2e: host buffers through the C-ABI (recompute, then cached scores)
    vict_host = torch.zeros(n_tab, dtype=torch.int32).pin_memory()  # step result read back
    vict_dev = torch.zeros(n_tab, dtype=torch.int32, device=dev)

    def e2e_run(mode):
        cycle(host=True, victims_host=vict_host, mode=mode)  # warm the host-staging ring (untimed)
        eng.sync()
        barrier()
        w0 = time.perf_counter()
        for _ in range(max(1, args.steps)):
            cycle(host=True, victims_host=vict_host, mode=mode)
        eng.sync()
        barrier()
        return max_over_ranks((time.perf_counter() - w0) / max(1, args.steps))

    e2e_s = e2e_run(pe.ScoreMode.RECOMPUTE)
    e2e_c = e2e_run(pe.ScoreMode.CACHED)
    e2e = {"value": round(total_step_bytes / e2e_s / 1e9, 3), "unit": "GB/s",
           "h2d_bytes_per_step": int(B * 2 * NL * S * H * d * elt + B * S * 8),
           "d2h_bytes_per_step": int(n_tab * 4),
           "ms_per_step": round(e2e_s * 1e3, 3), "score_mode": "recompute (K2)",
           # the same cycle with the cached-score eviction (K2c reads 12 B per
           # page instead of the pages): its time, and the recompute step's
           # bytes over it as an "equivalent" rate (not an HBM rate)
           "cached": {"ms_per_step": round(e2e_c * 1e3, 3), "score_mode": "cached (K2c)",
                      "equivalent_gbs": round(total_step_bytes / e2e_c / 1e9, 3),
                      "hbm_bytes_per_step": int(sum_over_ranks(float(k0_alg + n_tab * 12 * (C // B + 1)))),
                      "hbm_gbs": round(sum_over_ranks(float(k0_alg + n_tab * 12 * (C // B + 1))) / e2e_c / 1e9,
                                       3)}}

    # ---------------- pruned decode tokens/s (K0 + K2/K2c + K3, all layers) vs FullCache
    decode = None
    total_seqs = int(round(sum_over_ranks(float(S))))
    if not args.no_decode:
        q = torch.randn((S, QH, d), generator=gen, device=dev, dtype=torch.float32).to(tdt)
        out = torch.empty((S, QH, d), dtype=torch.float32, device=dev)

        def decode_tokens(mode):
            """B decode tokens: per token K0 over all layers, then per layer the
            trigger's eviction (on the B-th token) and K3; no events between
            launches (consecutive launches overlap through PDL, as in serving)."""
            barrier()
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            d0.record(stream)
            for j in range(B):
                eng.append_token(0, NL, rows_k[j], rows_v[j], next_pos())
                for layer in range(NL):
                    if j == B - 1:
                        eng.evict(layer, 1, mode=mode)
                    eng.attend(layer, q, out, QH)
            d1.record(stream)
            d1.synchronize()
            cycles[0] += 1
            return max_over_ranks(d0.elapsed_time(d1))

        dec_ms = decode_tokens(pe.ScoreMode.RECOMPUTE)
        dec_ms_c = decode_tokens(pe.ScoreMode.CACHED)
        # K3 alone: every layer's attention back to back, one event pair per
        # pass over the layers (per-layer time = pass / NL), 8 passes
        attn_ms = []
        for _ in range(8):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for layer in range(NL):
                eng.attend(layer, q, out, QH)
            b.record(stream)
            attn_ms.append((a, b))
        torch.cuda.synchronize()
        at = [a.elapsed_time(b) / NL for a, b in attn_ms]
        k3_bytes = n_tab_layer * k3_bytes_per_table(C + B // 2, row, G, d, elt)
        decode = {"tokens_per_s": round(total_seqs * B / (dec_ms * 1e-3), 1),
                  "ms_per_token_all_layers": round(dec_ms / B, 4),
                  "score_mode": "recompute (K2 at the trigger)",
                  "tokens_per_s_cached": round(total_seqs * B / (dec_ms_c * 1e-3), 1),
                  "ms_per_token_all_layers_cached": round(dec_ms_c / B, 4),
                  "attention_us_per_layer_p50": round(statistics.median(at) * 1e3, 2),
                  "attention_gbs": round(k3_bytes / (statistics.median(at) * 1e-3) / 1e9, 1)}
        decode["full_cache"] = full_cache_decode(args, cfg, pe, torch, np, gen, dev, local_dev, stream, S, q, out,
                                                 statistics.median(at) * 1e3, max_over_ranks, total_seqs)

    st = eng.stats()
    # full-size parity by size-independent properties (untimed): every table
    # evicted exactly once per 16-token cycle (policy.cpp:147-150 cadence) and
    # the device invariant checker over all tables and the whole pool
    inv = eng.check_invariants()
    checks = {"evictions_expected": n_tab * cycles[0], "evictions_observed": int(st.pages_evicted),
              "cadence_ok": int(st.pages_evicted) == n_tab * cycles[0],
              "invariant_violations": inv["violations"], "tables_checked": inv["tables_checked"],
              "pages_mapped_plus_free": inv["pages_mapped"] + inv["free_pages"],
              "pool_capacity": int(eng.capacity)}
    ranks = gather_stats(RankStats(rank=rank, tables=n_tab, tokens_scored=int(st.tokens_scored),
                                   pages_evicted=int(st.pages_evicted),
                                   algorithmic_bytes=int(step_bytes * args.steps), kernel_ms=k2_ms))
    for r, c in zip(ranks, _gather_obj(world, {"seq_begin": seq0, "seqs": S, "device": local_dev,
                                               "ms_per_step": round(t0.elapsed_time(t1) / args.steps, 4),
                                               "checks_ok": checks["cadence_ok"]
                                               and checks["invariant_violations"] == 0})):
        r.update(c)
    cpu = cpu_baseline(cfg, args) if (rank == 0 and not args.no_cpu) else None
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None, "dtype": cfg["dtype"],
            "data": "synthetic N(0,1) K/V/Q (torch.randn); inputs resident in HBM",
            "config": {"workload": f"{args.config}: {cfg['desc']}", "tables_per_gpu": n_tab,
                       "tables_total": n_tab * world if cfg["scaling"] == "weak" else cfg["seqs"] * NL * H,
                       "page_size": B, "step": "one eviction cycle: 16 decode appends (K0, all layers per launch) "
                       "+ block eviction of every table (K2, " + ("one launch for all layers)" if args.evict_launch
                                                                  == "step" else "one launch per layer)"),
                       "l2": "inputs larger than L2 (pool %.1f GB per GPU)" % (eng.info().pool_bytes / 1e9),
                       "parallelism": f"sequence-sharded x{world}, no data-path collective"},
            "pct_of_peak": round(100 * value / world / peak, 2),
            # p50 of the eviction step (all tables of every layer, the per-layer
            # launches of a cycle together in layer mode) and of one launch
            "p50_evict_step_us": round(k2_step_p50_ms * 1e3, 2),
            "p50_evict_step_samples": len(evs_p50),
            "p50_evict_launch_us": round(k2_p50_ms * 1e3, 2),
            "p50_evict_launch_samples": sum(n for _, _, n in evs_p50),
            "p50_evict_step_us_cached": round(k2c_step_us, 2),
            "p50_evict_launch_us_cached": round(k2c_us, 2),
            "append_us_per_launch_p50": round(statistics.median(a.elapsed_time(b) for a, b in k0_evs) * 1e3 / B, 2),
            "evict_launch": args.evict_launch,
            f"p50_evict_{other}_launch_us": round(other_us, 2),
            f"evict_{other}_launch_gbs": round(other_bytes / (other_us * 1e-6) / 1e9, 1),
            f"evict_{other}_launch_frac": round(other_bytes / (other_us * 1e-6) / 1e9 / peak, 4),
            "roofline": {"bound": "hbm", "achieved": round(k2_gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(k2_gbs / peak, 4), "traffic": ncu_traffic(expect_bytes=k2_per_launch),
                         "traffic_source": "ncu dram__bytes_read+write per launch, profiles/*bench_launches*.csv",
                         "kernel": "K2 evict_score_kernel, " + (f"one launch per decode step (all {NL} layers)"
                                                                  if args.evict_launch == "step" else "per-layer launch"),
                         "algorithmic_bytes_per_launch": k2_per_launch, "peak_kind": peak_kind,
                         "probe": probe,
                         "frac_of_probe_read": round(k2_gbs / probe["read_gbs"], 4) if probe else None},
            "prefill": prefill,
            "decode": decode,
            "e2e": e2e,
            "checks": checks,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "ranks": ranks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _gather_obj(world, obj):
    import torch.distributed as dist

    if world == 1:
        return [obj]
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


def full_cache_decode(args, cfg, pe, torch, np, gen, dev, local_dev, stream, S, q, out, pruned_attn_us,
                      max_over_ranks, total_seqs):
    """FullCache decode (policy.cpp:292-304: no eviction, the table keeps
    every token and grows from L) on one layer — K0 + K3 per token — and the
    tokens/s of the whole model (× layers). When the unpruned layer of all S
    sequences does not fit beside the pruned pool, a stated subset of the
    sequences is measured (attention time is linear in the sequences)."""
    bf16 = cfg["dtype"] == "bf16"
    tdt = torch.bfloat16 if bf16 else torch.float32
    elt = 2 if bf16 else 4
    NL, H, d, L, QH = cfg["layers"], cfg["kvh"], cfg["d"], cfg["L"], cfg["qh"]
    G = QH // H
    row = 2 * d * elt
    free_b, _ = torch.cuda.mem_get_info(dev)
    per_seq = H * ((L + 2 * B) // B + 1) * 2 * B * row // 2 + L * H * row  # pool + prompt staging
    S_f = max(1, min(S, int(0.6 * free_b // per_seq)))
    try:
        fgeo = pe.EngineGeometry(n_seqs=S_f, n_layers=1, n_kv_heads=H, head_dim=d,
                                 dtype=pe.DTYPE_BF16 if bf16 else pe.DTYPE_F32, device=local_dev,
                                 max_pages_per_table=(L + 2 * B) // B + 1)
        feng = pe.PagedEvictionEngine(fgeo, pe.PolicyConfig(cache_budget=cfg["C"], page_size=B,
                                                            kind=pe.PolicyKind.FullCache))
        fk = torch.empty((S_f * L, H, d), dtype=tdt, device=dev).normal_(generator=gen)
        cu = np.arange(S_f + 1, dtype=np.int32) * L
        feng.prefill_compress(0, fk, torch.empty_like(fk).normal_(generator=gen), cu)
        del fk
        torch.cuda.empty_cache()
        fq, fo = q[:S_f].contiguous(), out[:S_f]
        rk = torch.randn((B, 1, S_f, H, d), generator=gen, device=dev, dtype=torch.float32).to(tdt)
        rv = torch.randn((B, 1, S_f, H, d), generator=gen, device=dev, dtype=torch.float32).to(tdt)
        pos = L + torch.arange(B, device=dev, dtype=torch.int64).unsqueeze(1).expand(B, S_f).contiguous()
        feng.attend(0, fq, fo, QH)  # warm
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        att = []
        a.record(stream)
        for j in range(B):
            feng.append_token(0, 1, rk[j], rv[j], pos[j])
            x, y = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            x.record(stream)
            feng.attend(0, fq, fo, QH)
            y.record(stream)
            att.append((x, y))
        b.record(stream)
        b.synchronize()
        layer_ms = max_over_ranks(a.elapsed_time(b) / B)  # one token on one layer
        f_us = statistics.median(x.elapsed_time(y) for x, y in att) * 1e3
        ok = feng.check_invariants()["violations"] == 0 and feng.stats().pages_evicted == 0
        feng.close()
        torch.cuda.empty_cache()
        f_bytes = S_f * H * k3_bytes_per_table(L + B // 2, row, G, d, elt)
        scale = S / S_f  # attention time is linear in the sequences
        return {"tokens_per_s": round(total_seqs / (NL * layer_ms * scale * 1e-3), 1),
                "ms_per_token_all_layers": round(NL * layer_ms * scale, 4),
                "measured": f"K0 + K3 on one layer of {S_f} of the rank's {S} sequences (unpruned, "
                            f"~{L + B // 2} tokens per table), x {NL} layers" + (
                                f", x {scale:.2f} for the other sequences" if S_f < S else ""),
                "attention_us_per_layer_p50": round(f_us, 2),
                "attention_gbs": round(f_bytes / (f_us * 1e-6) / 1e9, 1),
                "retained_tokens_per_table": L + B // 2,
                "attention_speedup_pruned": round(f_us * scale / pruned_attn_us, 2),
                "no_evictions_ok": bool(ok)}
    except Exception as exc:  # pool for the unpruned layer does not fit: report why
        torch.cuda.empty_cache()
        return {"unavailable": str(exc)[:200]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--ref-tables", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--evict-launch", default="layer", choices=["layer", "step"],
                    help="one K2 launch per layer (default: the serving granularity; consecutive launches "
                         "overlap through PDL), or one per decode step covering all layers")
    ap.add_argument("--share-device", action="store_true",
                    help="test only: every rank on device 0 with the gloo backend")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ:
        if args.gpus > 1 and args.impl == "b200":
            sys.exit(relaunch(args))
        world, rank, local = args.gpus if args.impl == "reference" else 1, 0, 0
    else:
        world, rank, local = dist_setup()
        if world != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
    else:
        run_b200(args, cfg, world, rank, local)


if __name__ == "__main__":
    main()
