"""The reference's cross-mode scheduler laws
(`/root/reference/pkg/tests/test_schedulers.py`) with the device backend in
place of `SyntheticBackend`: the unmodified reference runners (`run_episode`,
`MODES`) drive `EngineBackend` (tiny, fp32), so the laws hold for the
engine's decoded content, not only for synthetic tokens.

Reference tests mirrored:
  test_all_modes_reduce_to_warmup_at_t1          test_schedulers.py:289
  test_action_available_in_every_mode            test_schedulers.py:301
  test_episode_determinism_byte_identical_logs   test_schedulers.py:321
  test_sync_warmup_equals_sequential             test_schedulers.py:102
"""

import math

import pytest

from ecot_sched.backends import default_profile
from ecot_sched.batching import LatencyModel
from ecot_sched.schedulers import MODES, SchedulerConfig, run_episode
from ecot_sched.trace import serialize_trace
from paper_2506_07639_b200.engine_backend import EngineBackend

pytestmark = pytest.mark.gpu


def episode(mode, profile_seed, schema, T, seed=0, k=5, slots=8):
    """One episode of the reference runner on a fresh device backend (its own
    engine: an async runner may leave reasoning requests in flight at the end
    of an episode, which belong to that backend)."""
    be = EngineBackend("tiny", dtype="f32", seed=0, kv_pages=1024, profile=default_profile(profile_seed))
    try:
        cfg = SchedulerConfig(mode=mode, k=k, slots=slots, latency=LatencyModel(), failure_policy="reuse_stale")
        return run_episode(cfg, T, be, schema, seed=seed)
    finally:
        be.close()


def test_all_modes_reduce_to_warmup_at_t1(schema):
    results = {}
    for mode in MODES:
        r, _ = episode(mode, 9, schema, 1, seed=9)
        results[mode] = r[0]
    ref = results["sequential"]
    for mode, r in results.items():
        assert r.trace == ref.trace, mode
        assert r.latency_ms == ref.latency_ms, mode


def test_action_available_in_every_mode(schema):
    for mode in MODES:
        results, _ = episode(mode, 1, schema, 5, seed=1)
        for r in results:
            assert r.action is not None
            assert len(r.action) == schema.action_dim
            assert all(math.isfinite(c) for c in r.action.components)


def test_episode_determinism_byte_identical_logs(schema):
    for mode in MODES:
        runs = []
        for _ in range(2):
            results, _ = episode(mode, 13, schema, 8, seed=13)
            runs.append(b"\n".join(serialize_trace(r.trace, schema, wall_ms=r.latency_ms) for r in results))
        assert runs[0] == runs[1], mode


def test_sync_warmup_equals_sequential(schema):
    seq, _ = episode("sequential", 3, schema, 1, seed=3)
    syn, _ = episode("parallel_sync", 3, schema, 1, seed=3)
    assert seq[0].trace == syn[0].trace
    assert seq[0].latency_ms == syn[0].latency_ms
