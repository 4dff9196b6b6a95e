"""N > 1 host path on CPU (gloo, world size 2): episode sharding, each rank
driving its shard as one `BatchedEpisodes` batch on its own engine (a fake
device engine here), and the token gather -- the same functions bench.py
uses over NCCL.  The gathered traces must equal a single-process batch of
every episode (episodes are independent)."""

import os
import socket
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

from paper_2506_07639_b200 import distributed as D

EPISODES = [0, 1, 2, 3, 4]
T = 3


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_tokens(seeds) -> dict:
    """{episode: [per-timestep step token tuples]} from one batched engine."""
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import ecot_sched
    from fake_engine import fake_backend

    from paper_2506_07639_b200 import BatchedEpisodes
    schema = ecot_sched.trace.default_schema()
    be, _ = fake_backend()
    batch = BatchedEpisodes(ecot_sched.SchedulerConfig(mode="parallel_sync", slots=8), be, schema, seeds)
    steps = [batch.step(t) for t in range(T)]
    return {e: D.episode_tokens([steps[t][i] for t in range(T)]) for i, e in enumerate(seeds)}


def _worker(rank: int, world: int, port: int, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    r, w, _ = D.init_from_env("gloo")
    mine = D.shard_episodes(EPISODES, w, r)
    gathered = D.gather_to_all(_shard_tokens(mine), w)
    if r == 0:
        out.put(D.merge_shards(gathered, EPISODES))
    import torch.distributed as dist
    dist.barrier()
    dist.destroy_process_group()


def test_shard_episodes_round_robin():
    assert D.shard_episodes(list(range(7)), 3, 0) == [0, 3, 6]
    assert D.shard_episodes(list(range(7)), 3, 2) == [2, 5]
    shards = [D.shard_episodes(list(range(64)), 8, r) for r in range(8)]
    assert sorted(e for s in shards for e in s) == list(range(64))
    assert {len(s) for s in shards} == {8}
    with pytest.raises(ValueError):
        D.shard_episodes([1], 2, 2)


def test_merge_shards_detects_gaps_and_duplicates():
    assert D.merge_shards([{0: "a", 2: "c"}, {1: "b"}], [0, 1, 2]) == ["a", "b", "c"]
    with pytest.raises(ValueError):
        D.merge_shards([{0: "a"}, {0: "b"}], [0])
    with pytest.raises(ValueError):
        D.merge_shards([{0: "a"}], [0, 1])


def test_gloo_world2_sharded_episodes_equal_single_process():
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    got = out.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = _shard_tokens(EPISODES)
    assert got == [want[e] for e in EPISODES]
