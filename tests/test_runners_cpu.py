"""Runner semantics of the mirror (CPU): the reference's own scheduler tests
that pin the hot-path modes (tests/test_schedulers.py of the reference),
re-run against this package's runners, plus golden-trace parity of the
runners over the CPU oracle."""

import math
import threading

import numpy as np
import pytest

from conftest import FailingBackend, FixedBackend
from paper_2506_07639_b200 import backends as B
from paper_2506_07639_b200 import schedulers as S
from paper_2506_07639_b200 import trace as T
from paper_2506_07639_b200.batching import LatencyModel

MODEL = LatencyModel(c_iter=10, c_slot=1, c_encode=20, c_decode=5)
HOT_MODES = ("sequential", "parallel_sync", "parallel_async")


def episode(mode, backend, schema, T_, seed=0, slots=8, model=None, policy="reuse_stale"):
    cfg = S.SchedulerConfig(mode=mode, slots=slots, latency=model or LatencyModel(), failure_policy=policy)
    return S.run_episode(cfg, T_, backend, schema, seed=seed)


def fixed_profile(schema, lengths, p=1.0, seed=0):
    return B.SyntheticProfile({s.name: B.StepProfile(lengths[s.name], 0, p) for s in schema.steps}, seed=seed)


def test_sequential_latency_closed_form():
    schema = T.StepSchema((T.StepSpec("think", "high", 32), T.StepSpec("action", "low", 16)))
    be = B.SyntheticBackend(fixed_profile(schema, {"think": 5, "action": 7}))
    r = S.SequentialRunner(be, schema, S.SchedulerConfig(latency=MODEL)).step(be.encode("i", b"o"), 0)
    assert r.latency_ms == 12 * 11 + 20 + 5


def test_sync_makespan_matches_fig5_lengths():
    schema = T.StepSchema((T.StepSpec("a", "high", 16), T.StepSpec("b", "high", 16),
                           T.StepSpec("c", "low", 16), T.StepSpec("action", "low", 16)))
    be = B.SyntheticBackend(fixed_profile(schema, {"a": 3, "b": 6, "c": 8, "action": 9}))
    res, _ = episode("parallel_sync", be, schema, 2, slots=4, model=MODEL)
    assert res[1].latency_ms == 9 * 10 + 26 * 1 + 20 + 5
    assert res[1].generated_tokens == 26


def test_async_action_latency_closed_form(schema):
    lengths = {"task": 50, "plan": 75, "subtask": 70, "move": 18, "gripper": 15,
               "visible_objects": 120, "action": 7}
    res, _ = episode("parallel_async", B.SyntheticBackend(fixed_profile(schema, lengths)), schema, 2,
                     model=MODEL)
    assert res[1].latency_ms == 7 * (10 + 7 * 1) + 20 + 5


def test_async_staleness_bound(schema):
    res, _ = episode("parallel_async", B.SyntheticBackend(B.default_profile(5)), schema, 60, seed=5)
    max_len = {s.name: 0 for s in schema.reasoning_steps}
    for r in res:
        for name, toks in r.trace.steps[:-1]:
            max_len[name] = max(max_len[name], len(toks))
    for name, L in max_len.items():
        assert all(r.staleness[name] <= math.ceil(L / 7) + 1 for r in res)


def test_dominance_per_timestep(schema):
    seq = episode("sequential", B.SyntheticBackend(B.default_profile(0)), schema, 12)[0]
    syn = episode("parallel_sync", B.SyntheticBackend(B.default_profile(0)), schema, 12)[0]
    asy = episode("parallel_async", B.SyntheticBackend(B.default_profile(0)), schema, 12)[0]
    for t in range(12):
        assert asy[t].latency_ms <= syn[t].latency_ms <= seq[t].latency_ms


def test_prefix_independent_backend_gives_identical_traces(schema):
    contents = {s.name: tuple(range(5 + i)) for i, s in enumerate(schema.steps)}
    logs = {m: b"\n".join(T.trace_content_bytes(r.trace, schema)
                          for r in episode(m, FixedBackend(contents), schema, 10)[0]) for m in HOT_MODES}
    assert len(set(logs.values())) == 1


def test_sync_reuse_stale_substitutes_previous_step(schema):
    be = FailingBackend(B.SyntheticBackend(B.default_profile(0)), fail_steps={"plan"}, fail_from_timestep=1)
    res, summary = episode("parallel_sync", be, schema, 4)
    for r in res[1:]:
        assert r.trace.tokens_of("plan") == res[0].trace.tokens_of("plan")
        assert "plan" in r.failures
    assert summary["failures"] == 3


def test_sync_abort_policy_stops_episode(schema):
    be = FailingBackend(B.SyntheticBackend(B.default_profile(0)), fail_steps={"plan"}, fail_from_timestep=2)
    with pytest.raises(S.EpisodeAborted) as exc:
        episode("parallel_sync", be, schema, 6, policy="abort_episode")
    assert len(exc.value.partial_results) == 2


def test_sequential_failure_aborts_with_partial_trace(schema):
    be = FailingBackend(B.SyntheticBackend(B.default_profile(0)), fail_steps={"subtask"})
    with pytest.raises(S.EpisodeAborted) as exc:
        episode("sequential", be, schema, 3)
    assert exc.value.partial_trace.names == ("task", "plan")


def test_async_background_failure_keeps_stale_value(schema):
    be = FailingBackend(B.SyntheticBackend(B.default_profile(0)), fail_steps={"visible_objects"},
                        fail_from_timestep=1)
    res, summary = episode("parallel_async", be, schema, 5)
    for r in res[1:]:
        assert r.trace.tokens_of("visible_objects") == res[0].trace.tokens_of("visible_objects")
    assert summary["failures"] >= 1


def test_cache_concurrent_stress_no_torn_snapshots(schema):
    registry = {}
    cache = S.CachedTrace(schema.names, recorder=lambda v, fp: registry.__setitem__(v, fp))
    names = list(schema.names)
    stop, torn = threading.Event(), []

    def writer(w):
        rng = np.random.default_rng(w)
        for _ in range(1000):
            cache.write(names[int(rng.integers(0, len(names)))],
                        tuple(int(x) for x in rng.integers(0, 100, 4)), 0)

    def reader():
        while not stop.is_set():
            snap = cache.snapshot()
            if snap.version and S.snapshot_fingerprint(snap.steps) != registry.get(snap.version):
                torn.append(snap.version)

    rs = [threading.Thread(target=reader) for _ in range(3)]
    ws = [threading.Thread(target=writer, args=(w,)) for w in range(3)]
    for th in rs + ws:
        th.start()
    for th in ws:
        th.join()
    stop.set()
    for th in rs:
        th.join()
    assert cache.snapshot().version == 3000 and torn == []


def test_summary_reports_percentiles(schema):
    _, summary = episode("parallel_sync", B.SyntheticBackend(B.default_profile(0)), schema, 8)
    assert summary["latency_p50_ms"] <= summary["latency_p99_ms"]


def test_mirror_runners_over_oracle_reproduce_reference_golden(schema, golden_traces):
    """The golden lines were produced by the REFERENCE runners over the CPU
    oracle; this package's runners over the same oracle must match byte for
    byte (and in simulated latency, staleness and token accounting)."""
    from oracle.backend import OracleBackend, OracleModel
    model = OracleModel("tiny", seed=0)
    for mode in HOT_MODES:
        g = golden_traces["modes"][mode]
        res, _ = episode(mode, OracleBackend("tiny", seed=0, model=model), schema, golden_traces["T"])
        assert [T.trace_content_bytes(r.trace, schema).decode() for r in res] == g["lines"], mode
        assert [r.latency_ms for r in res] == g["latency_ms"]
        assert [r.staleness for r in res] == g["staleness"]
        assert [r.generated_tokens for r in res] == g["generated_tokens"]
