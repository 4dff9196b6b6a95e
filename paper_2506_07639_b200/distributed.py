"""Multi-GPU plumbing for batched rollouts (BASELINE config 4).

Episodes are independent (each `run_episode` owns its runner and cache,
reference `schedulers.py:818`), so the path shards with no data-path
collective: episode e runs on rank e mod world, every rank drives its shard
on its own engine (weights regenerated locally from the seed), and one
object gather at the end collects the per-episode results ("scaling":
"weak" per GPU for a fixed shard, or a fixed episode set split over ranks).

The same functions run under NCCL (bench.py, one process per GPU) and gloo
(the CPU tests), so the N > 1 host logic is exercised without GPUs.
"""

from __future__ import annotations

import os
from typing import Any, Sequence


def shard_episodes(episodes: Sequence[int], world: int, rank: int) -> list[int]:
    """Episode ids of `rank`: e for position i with i mod world == rank
    (round-robin keeps the shards within one episode of each other)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return [e for i, e in enumerate(episodes) if i % world == rank]


def init_from_env(backend: str) -> tuple[int, int, int]:
    """(rank, world, local_rank) from torchrun's environment; initialises the
    process group when world > 1 (rendezvous on 127.0.0.1)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if not dist.is_initialized():
            dist.init_process_group(backend=backend)
    return rank, world, local


def gather_to_all(obj: Any, world: int) -> list[Any]:
    """Every rank's `obj`, in rank order (all_gather_object; world 1: [obj])."""
    if world == 1:
        return [obj]
    import torch.distributed as dist
    out: list[Any] = [None] * world
    dist.all_gather_object(out, obj)
    return out


def merge_shards(per_rank: Sequence[dict], episodes: Sequence[int]) -> list[Any]:
    """Per-rank {episode id: result} dicts -> results in `episodes` order;
    raises if an episode is missing or produced twice."""
    merged: dict = {}
    for shard in per_rank:
        for e, res in shard.items():
            if e in merged:
                raise ValueError(f"episode {e} reported by two ranks")
            merged[e] = res
    missing = [e for e in episodes if e not in merged]
    if missing:
        raise ValueError(f"episodes {missing} missing from the gathered shards")
    return [merged[e] for e in episodes]


def episode_tokens(results) -> list:
    """One episode's per-timestep step contents as plain int tuples
    [(step name, tokens), ...] -- what ranks gather (the episode's results)."""
    return [tuple((name, tuple(int(t) for t in toks)) for name, toks in r.trace.steps) for r in results]
