"""Multi-GPU plumbing for the PagedEviction engine.

Tables are independent (one reference BlockTable per sequence/layer/head), so
the path shards by sequence with no collective on the data path: every rank
owns its own engine (pool, block tables, free list) for a contiguous block of
sequences. torch.distributed (NCCL on GPUs, gloo on CPU) is used only to
agree on timing (max over ranks) and to gather a small per-rank stats
struct at the end of a run.
"""
from __future__ import annotations

import os
from dataclasses import asdict, dataclass, field


def shard(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [begin, end) of `n_items` owned by `rank`
    (the first n_items % world ranks get one extra)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def env_rank() -> tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


@dataclass
class RankStats:
    rank: int = 0
    tables: int = 0
    tokens_scored: int = 0
    pages_evicted: int = 0
    algorithmic_bytes: int = 0
    kernel_ms: list = field(default_factory=list)

    def summary(self) -> dict:
        d = asdict(self)
        ms = sorted(self.kernel_ms)
        d.pop("kernel_ms")
        d["kernel_ms_p50"] = ms[len(ms) // 2] if ms else None
        d["kernel_ms_p99"] = ms[min(len(ms) - 1, int(0.99 * len(ms)))] if ms else None
        return d


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (identity when not distributed)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    """Sum of a scalar over all ranks (identity when not distributed)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_stats(stats: RankStats) -> list[dict]:
    """All ranks' stats summaries (one small all_gather at the end of a run)."""
    import torch.distributed as dist

    s = stats.summary()
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [s]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, s)
    return out
