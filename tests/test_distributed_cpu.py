"""N > 1 host path on CPU (gloo, world size 2): episode sharding, per-rank
episodes driven by the package runners, and the result gather -- the same
functions bench.py uses over NCCL.  The gathered traces must equal a
single-process run of every episode (episodes are independent)."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2506_07639_b200 import distributed as D

EPISODES = [0, 1, 2, 3, 4]
T = 3


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _episode_bytes(seed: int) -> list[bytes]:
    from paper_2506_07639_b200 import schedulers as S
    from paper_2506_07639_b200.backends import SyntheticBackend, default_profile
    from paper_2506_07639_b200.trace import default_schema, trace_content_bytes
    schema = default_schema()
    res, _ = S.run_episode(S.SchedulerConfig(mode="parallel_sync", slots=8), T,
                           SyntheticBackend(default_profile(0)), schema, seed=seed)
    return [trace_content_bytes(r.trace, schema) for r in res]


def _worker(rank: int, world: int, port: int, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    r, w, _ = D.init_from_env("gloo")
    mine = D.shard_episodes(EPISODES, w, r)
    local = {e: _episode_bytes(e) for e in mine}
    gathered = D.gather_to_all(local, w)
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
    want = [_episode_bytes(e) for e in EPISODES]
    assert got == want
