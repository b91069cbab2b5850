"""Multi-rank host logic on CPU (gloo, world_size 2): sequences are sharded
across ranks, each rank runs its own engine (here the C oracle engine, the
CPU stand-in for the per-GPU CUDA engine) with its own pool and free list,
and only the timing max and a stats struct cross ranks. The union of the
ranks' decisions must equal a single-rank run over all sequences (tables
are independent; only physical page ids differ, since pools differ)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2509_04377_b200.dist import RankStats, gather_stats, max_over_ranks, shard
from tests.harness import random_kv

S, NL, H, W, B, C = 5, 2, 2, 16, 8, 32
LENS = np.array([70, 20, 33, 90, 41])
STEPS = 20


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def inputs():
    rng = np.random.default_rng(77)
    cu = np.concatenate([[0], np.cumsum(LENS)]).astype(np.int32)
    pk = [random_kv(rng, (cu[-1], H, W), oracle.F32)[0] for _ in range(NL)]
    pv = [random_kv(rng, (cu[-1], H, W), oracle.F32)[0] for _ in range(NL)]
    dk = random_kv(rng, (STEPS, NL, S, H, W), oracle.F32)[0]
    dv = random_kv(rng, (STEPS, NL, S, H, W), oracle.F32)[0]
    return cu, pk, pv, dk, dv


def run_shard(seq_lo, seq_hi):
    """Runs sequences [seq_lo, seq_hi) on a private engine; returns per
    (global seq, layer, head) victims per step and final retained positions."""
    cu, pk, pv, dk, dv = inputs()
    n = seq_hi - seq_lo
    eng = oracle.OracleEngine(n_seqs=n, n_layers=NL, n_tab_heads=H, width=W, page_size=B, budget=C,
                              dtype=oracle.F32, capacity=n * NL * H * (C // B + 1), max_pages=C // B + 1)
    lcu = (cu[seq_lo:seq_hi + 1] - cu[seq_lo]).astype(np.int32)
    for layer in range(NL):
        rows = slice(cu[seq_lo], cu[seq_hi])
        assert eng.prefill(layer, pk[layer][rows], pv[layer][rows], lcu)[0] == 0
    pos = LENS[seq_lo:seq_hi].astype(np.int64).copy()
    victims = {}
    evicted = 0
    for st in range(STEPS):
        assert eng.decode_append(0, NL, dk[st][:, seq_lo:seq_hi], dv[st][:, seq_lo:seq_hi], pos) == 0
        _, vic = eng.decode_evict(0, NL)
        i = 0
        for s in range(n):
            for layer in range(NL):
                for h in range(H):
                    victims[(seq_lo + s, layer, h, st)] = int(vic[i])
                    evicted += vic[i] >= 0
                    i += 1
        pos += 1
    bt, npg, nf, posn = eng.block_table(), eng.num_pages(), eng.newest_fill(), eng.positions()
    retained = {}
    for s in range(n):
        for layer in range(NL):
            for h in range(H):
                t = eng.table_id(s, layer, h)
                retained[(seq_lo + s, layer, h)] = np.concatenate(
                    [posn[bt[t, j], : (B if j < npg[t] - 1 else nf[t])] for j in range(npg[t])]).tolist()
    return victims, retained, int(evicted)


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard(S, world, rank)
    victims, retained, evicted = run_shard(lo, hi)
    t = max_over_ranks(float(rank + 1))
    stats = gather_stats(RankStats(rank=rank, tables=(hi - lo) * NL * H, pages_evicted=evicted,
                                   kernel_ms=[1.0 + rank]))
    gathered = [None] * world
    dist.all_gather_object(gathered, (victims, retained))
    if rank == 0:
        q.put((t, stats, gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_partition():
    for n in (1, 5, 64, 1024):
        for world in (1, 2, 3, 8):
            spans = [shard(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1


def test_two_rank_gloo_equals_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, stats, gathered = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 2.0  # max over ranks
    assert [s["rank"] for s in stats] == [0, 1]
    assert sum(s["tables"] for s in stats) == S * NL * H
    victims, retained, _ = run_shard(0, S)
    merged_v, merged_r = {}, {}
    for v, r in gathered:
        merged_v.update(v)
        merged_r.update(r)
    assert merged_v == victims
    assert merged_r == retained
    assert sum(s["pages_evicted"] for s in stats) == sum(1 for x in victims.values() if x >= 0)
