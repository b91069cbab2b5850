"""Multi-rank host logic (gloo, world_size 2): sequences are sharded across
ranks, each rank runs its own engine with its own pool and free list, and
only the timing max and a stats struct cross ranks. The union of the ranks'
decisions must equal a single-rank run over all sequences (tables are
independent; only physical page ids differ, since pools differ).

Backends: the C oracle engine (CPU, runs everywhere) and the CUDA engine
(`-m gpu`: two processes, each with its own engine on cuda:0, gloo between
them — the single-GPU stand-in for one engine per GPU). The bench's own
multi-rank path (`bench.py --gpus 2`, re-executed under torchrun) is run
the same way with --share-device."""
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


class _CudaShard:
    """The CUDA engine behind the oracle engine's calls (same state readback)."""

    def __init__(self, n):
        import torch

        import paper_2509_04377_b200 as pe

        self.torch = torch
        self.eng = pe.PagedEvictionEngine(
            pe.EngineGeometry(n_seqs=n, n_layers=NL, n_kv_heads=H, head_dim=W, dtype=pe.DTYPE_F32, device=0),
            pe.PolicyConfig(cache_budget=C, page_size=B))

    def _d(self, a):
        return self.torch.from_numpy(np.ascontiguousarray(a)).cuda(0)

    def prefill(self, layer, k, v, cu):
        self.eng.prefill_compress(layer, self._d(k), self._d(v), cu)
        return (0,)

    def decode(self, k, v, pos, step):
        return self.eng.decode_step(0, NL, self._d(k), self._d(v), self._d(pos), step, victims=True)

    def state(self):
        bt, npg, nf, _ = self.eng.tables()
        return bt, npg, nf, self.eng.positions()

    def table_id(self, s, layer, h):
        return self.eng.table_id(s, layer, h)


def run_shard(seq_lo, seq_hi, backend="oracle"):
    """Runs sequences [seq_lo, seq_hi) on a private engine; returns per
    (global seq, layer, head) victims per step and final retained positions."""
    cu, pk, pv, dk, dv = inputs()
    n = seq_hi - seq_lo
    if backend == "cuda":
        eng = _CudaShard(n)
    else:
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
        if backend == "cuda":
            vic = eng.decode(dk[st][:, seq_lo:seq_hi], dv[st][:, seq_lo:seq_hi], pos, st + 1)
        else:
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
    if backend == "cuda":
        bt, npg, nf, posn = eng.state()
    else:
        bt, npg, nf, posn = eng.block_table(), eng.num_pages(), eng.newest_fill(), eng.positions()
    retained = {}
    for s in range(n):
        for layer in range(NL):
            for h in range(H):
                t = eng.table_id(s, layer, h)
                retained[(seq_lo + s, layer, h)] = np.concatenate(
                    [posn[bt[t, j], : (B if j < npg[t] - 1 else nf[t])] for j in range(npg[t])]).tolist()
    return victims, retained, int(evicted)


def worker(rank, world, port, q, backend="oracle"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard(S, world, rank)
    victims, retained, evicted = run_shard(lo, hi, backend)
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


@pytest.mark.parametrize("backend", ["oracle", pytest.param("cuda", marks=pytest.mark.gpu)])
def test_two_rank_gloo_equals_single_rank(backend):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q, backend)) for r in range(2)]
    for p in procs:
        p.start()
    t, stats, gathered = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 2.0  # max over ranks
    assert [s["rank"] for s in stats] == [0, 1]
    assert sum(s["tables"] for s in stats) == S * NL * H
    victims, retained, _ = run_shard(0, S, backend)
    merged_v, merged_r = {}, {}
    for v, r in gathered:
        merged_v.update(v)
        merged_r.update(r)
    assert merged_v == victims
    assert merged_r == retained
    assert sum(s["pages_evicted"] for s in stats) == sum(1 for x in victims.values() if x >= 0)


def _bench_line(out: str) -> dict:
    import json

    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_two_ranks_share_device():
    """bench.py --gpus 2 re-executes itself under torch.distributed.run: two
    ranks, each with its own engine and sequence shard (here both on cuda:0
    with gloo, --share-device), one JSON line from rank 0 with n_gpus 2,
    both ranks' stats, clean checks, and the whole-job value."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--share-device", "--config",
                          "tiny", "--steps", "3", "--warmup", "3", "--no-cpu"], capture_output=True, text=True,
                         timeout=600, env=env, cwd=root)
    assert res.returncode == 0, res.stderr[-3000:]
    line = _bench_line(res.stdout)
    assert line["n_gpus"] == 2 and len(line["ranks"]) == 2
    assert [r["rank"] for r in line["ranks"]] == [0, 1]
    assert all(r["checks_ok"] for r in line["ranks"])
    assert line["checks"]["cadence_ok"] and line["checks"]["invariant_violations"] == 0
    assert line["config"]["tables_total"] == 2 * line["config"]["tables_per_gpu"]
    assert line["value"] > 0 and line["e2e"]["value"] > 0


def test_bench_rejects_inconsistent_world():
    """--gpus must match the launcher's WORLD_SIZE (no silent single rank)."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "4"], capture_output=True, text=True,
                         timeout=300, env=env, cwd=root)
    assert res.returncode != 0 and "WORLD_SIZE=1" in res.stderr


def test_bench_fails_loudly_without_enough_gpus():
    """`bench.py --gpus 2` with fewer visible GPUs: the torchrun re-exec
    starts two ranks and each refuses (no silent oversubscription)."""
    import subprocess
    import sys
    from pathlib import Path

    import torch

    if torch.cuda.device_count() >= 2:
        pytest.skip("two GPUs visible")
    root = Path(__file__).resolve().parent.parent
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--config", "tiny"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert res.returncode != 0
    assert "needs 2 visible GPUs" in res.stderr + res.stdout
