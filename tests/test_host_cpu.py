"""Host logic of the engine (CPU, fake device engine): the REFERENCE runners
(`ecot_sched`, imported unmodified) drive `EngineBackend`; batching,
deferred generators, the device async engines, failure policies and cache
coherence are checked against the reference's own simulated path.

`HashBackend` computes, one request at a time, the tokens the fake engine
produces for the same framed request, so any difference between the two
runs is a host-logic difference (ordering, batching, landing)."""

import threading
import time

import numpy as np
import pytest
from fake_engine import FakeEngine, HashBackend, fake_backend

import ecot_sched
from ecot_sched import schedulers as RS
from ecot_sched.batching import LatencyModel
from ecot_sched.trace import StepSchema, StepSpec, default_schema, trace_content_bytes
from paper_2506_07639_b200 import BatchedEpisodes, EngineError, runners
from paper_2506_07639_b200.backends import BackendError, StepProfile, SyntheticProfile, default_profile
from paper_2506_07639_b200.engine_backend import DeviceTokens, EngineBackend

HOT_MODES = ("sequential", "parallel_sync", "parallel_async")
MODEL = LatencyModel(c_iter=10, c_slot=1, c_encode=20, c_decode=5)


def episode(mode, backend, schema, T, seed=0, policy="reuse_stale", slots=8):
    cfg = RS.SchedulerConfig(mode=mode, slots=slots, latency=MODEL, failure_policy=policy)
    return ecot_sched.run_episode(cfg, T, backend, schema, seed=seed)


def lines(results, schema):
    return [trace_content_bytes(r.trace, schema) for r in results]


def test_engine_error_is_a_reference_backend_error():
    assert issubclass(EngineError, ecot_sched.BackendError)
    assert BackendError is ecot_sched.BackendError


def test_registry_serves_parallel_async_through_the_engine_runner():
    assert RS._RUNNERS["parallel_async"] is runners.EngineParallelAsyncRunner
    assert issubclass(runners.EngineParallelAsyncRunner, RS.ParallelAsyncRunner)


@pytest.mark.parametrize("mode", HOT_MODES)
def test_reference_runners_over_engine_match_synchronous_backend(mode):
    """Byte-identical traces AND identical simulated latency, staleness and
    token accounting: the deferred/batched engine path is invisible to the
    reference runners (async: lockstep device engine == reference
    `_MicroEngine` landing order)."""
    schema = default_schema()
    be, eng = fake_backend()
    got, gs = episode(mode, be, schema, 12, seed=3)
    want, ws = episode(mode, HashBackend(), schema, 12, seed=3)
    assert lines(got, schema) == lines(want, schema)
    assert [r.latency_ms for r in got] == [r.latency_ms for r in want]
    assert [r.staleness for r in got] == [r.staleness for r in want]
    assert [r.generated_tokens for r in got] == [r.generated_tokens for r in want]
    assert gs == ws


def test_parallel_sync_branches_decode_as_one_batch():
    schema = default_schema()
    be, eng = fake_backend()
    episode("parallel_sync", be, schema, 3)
    occ = [o for lane, o in eng.occupancy_log]
    assert max(occ) == len(schema.steps)   # all N+1 branches in one batch


def test_sequential_decodes_one_request_at_a_time():
    schema = default_schema()
    be, eng = fake_backend()
    episode("sequential", be, schema, 2)
    assert {o for _, o in eng.occupancy_log} == {1}


def test_trunk_prefix_is_prefilled_once_per_timestep():
    """All branches of a parallel_sync timestep fork one trunk: the prefill
    covers the context + previous reasoning once (not once per branch)."""
    schema = default_schema()
    be, eng = fake_backend()
    res, _ = episode("parallel_sync", be, schema, 2)
    before, calls = eng.prefilled_tokens, eng.prefill_calls
    runner = RS.ParallelSyncRunner(be, schema, RS.SchedulerConfig(mode="parallel_sync"))
    runner._prev_trace = res[-1].trace
    runner.step(be.encode("pick up the object and place it on the target", b"obs-x"), 2)
    ctx_len = 1 + be.cfg.n_vision + 16
    assert eng.prefilled_tokens - before == ctx_len + sum(len(t) for _, t in res[-1].trace.steps[:-1])
    assert eng.prefill_calls - calls == 1   # longest branch first: one prefill, every other branch forks it


def test_generators_are_lazy_until_read():
    schema = default_schema()
    be, eng = fake_backend()
    ctx = be.encode("i", b"o")
    gens = [be.begin_step(ctx, (), s, ()) for s in schema.steps]
    assert eng.occupancy_log == []
    assert all(isinstance(g.drain(), DeviceTokens) for g in gens)
    assert [len(g.tokens) for g in gens] == [len(HashBackend().begin_step(ctx, (), s, ()).tokens)
                                             for s in schema.steps]
    first = tuple(gens[0].tokens)
    assert first == HashBackend().begin_step(ctx, (), schema.steps[0], ()).tokens
    assert max(o for _, o in eng.occupancy_log) == len(schema.steps)


def test_batched_episodes_equal_independent_episodes():
    schema = default_schema()
    be, eng = fake_backend()
    cfg = RS.SchedulerConfig(mode="parallel_sync", slots=8, latency=MODEL)
    batch = BatchedEpisodes(cfg, be, schema, seeds=[0, 1, 2, 3])
    got = [batch.step(t) for t in range(4)]
    for e, seed in enumerate([0, 1, 2, 3]):
        want, _ = ecot_sched.run_episode(cfg, 4, HashBackend(), schema, seed=seed)
        assert [trace_content_bytes(got[t][e].trace, schema) for t in range(4)] == lines(want, schema)
        assert [got[t][e].latency_ms for t in range(4)] == [r.latency_ms for r in want]
    assert max(o for _, o in eng.occupancy_log) == 4 * len(schema.steps)
    assert be._live == 0 and not be._owners and not be._pending


# --- failure policies of the REFERENCE runners over the engine ----------------

class FailingEngine:
    """Fault injection around EngineBackend (reference tests/conftest.py:34-53)."""

    deterministic = True
    supports_prefix_conditioning = True

    def __init__(self, inner, fail_steps=(), fail_from_timestep=0):
        self.inner, self.fail_steps, self.fail_from = inner, set(fail_steps), fail_from_timestep
        self._encodes = -1

    def encode(self, instruction, observation):
        self._encodes += 1
        return self.inner.encode(instruction, observation)

    def begin_step(self, context, prefix, step, prev_content):
        if step.name in self.fail_steps and self._encodes >= self.fail_from:
            raise EngineError(f"injected engine failure for {step.name}")
        return self.inner.begin_step(context, prefix, step, prev_content)


def test_sync_reuse_stale_on_engine_error():
    schema = default_schema()
    be, _ = fake_backend()
    res, summary = episode("parallel_sync", FailingEngine(be, {"plan"}, 1), schema, 4)
    for r in res[1:]:
        assert r.trace.tokens_of("plan") == res[0].trace.tokens_of("plan")
        assert "plan" in r.failures
    assert summary["failures"] == 3
    assert be._live == 0


def test_sync_abort_on_engine_error():
    schema = default_schema()
    be, _ = fake_backend()
    with pytest.raises(RS.EpisodeAborted) as exc:
        episode("parallel_sync", FailingEngine(be, {"plan"}, 2), schema, 6, policy="abort_episode")
    assert len(exc.value.partial_results) == 2


def test_async_reuse_stale_and_abort_on_engine_error():
    schema = default_schema()
    be, _ = fake_backend()
    res, summary = episode("parallel_async", FailingEngine(be, {"visible_objects"}, 1), schema, 5)
    for r in res[1:]:
        assert r.trace.tokens_of("visible_objects") == res[0].trace.tokens_of("visible_objects")
    assert summary["failures"] >= 1
    be2, _ = fake_backend()
    with pytest.raises(RS.EpisodeAborted):
        episode("parallel_async", FailingEngine(be2, {"action"}, 2), schema, 5, policy="abort_episode")


def test_device_limits_surface_as_policy_errors():
    """A request the device would reject (here: longer than the 1024-token
    request cap) fails in begin_step, before any fork, so the reference
    reuse_stale policy handles it and no KV is leaked."""
    schema = StepSchema((StepSpec("essay", "high", 4096), StepSpec("action", "low", 16)))
    prof = SyntheticProfile({"essay": StepProfile(50, 0, 1.0), "action": StepProfile(7, 0, 1.0)})
    be, _ = fake_backend(profile=prof)
    res, _ = episode("parallel_sync", be, schema, 2)
    be.profile = SyntheticProfile({"essay": StepProfile(2000, 0, 1.0), "action": StepProfile(7, 0, 1.0)})
    runner = RS.ParallelSyncRunner(be, schema, RS.SchedulerConfig(mode="parallel_sync"))
    runner._prev_trace = res[-1].trace
    r = runner.step(be.encode("i", b"x"), 2)
    assert r.failures == ("essay",) and r.trace.tokens_of("essay") == res[-1].trace.tokens_of("essay")
    assert be._live == 0


# --- background async ----------------------------------------------------------

def test_background_async_per_request_parity_and_coherence():
    """Background ticker under the reference async runner: every landed request equals
    the synchronous backend's answer for the same (context, prefix, step,
    prev_content), and every snapshot the runner took was an atomic cache
    state (recorder fingerprints, reference tests/test_schedulers.py:397-429)."""
    schema = default_schema()
    log: list = []
    be, eng = fake_backend(async_mode="background", request_log=log)
    eng.tick_delay = 2e-4
    registry, torn = {}, []
    cfg = RS.SchedulerConfig(mode="parallel_async", slots=8, latency=MODEL)
    runner = RS.make_runner(cfg, be, schema)
    runner.cache.recorder = lambda v, fp: registry.__setitem__(v, fp)
    orig_snapshot = runner.cache.snapshot

    def audited():
        snap = orig_snapshot()
        if snap.version and RS.snapshot_fingerprint(snap.steps) != registry.get(snap.version):
            torn.append(snap.version)
        return snap

    runner.cache.snapshot = audited
    between = []
    try:
        for t in range(20):
            runner.step(be.encode("pick up", RS.observation_for(0, t)), t)
            n0 = len(eng.occupancy_log)
            time.sleep(0.005)             # control loop idle: reasoning keeps decoding
            between.append(len(eng.occupancy_log) - n0)
        runner.engine.drain(timeout=30.0)
    finally:
        runner.close()
    assert torn == []
    assert sum(between) > 0
    ref = HashBackend()
    assert len(log) > 20
    by_name = {s.name: s for s in schema.steps}
    for ctx, prefix, name, prev, tokens in log:
        assert tokens == tuple(ref.begin_step(ctx, prefix, by_name[name], prev).tokens)
    assert be._live == 0


def test_background_in_flight_covers_the_landing_window():
    """A request whose tokens are landing (cache write pending) still counts
    as in flight, so the runner cannot re-issue the same step from a snapshot
    that lacks it (advisor finding, round 1)."""
    schema = default_schema()
    be, eng = fake_backend(async_mode="background")
    aeng = be.make_async_engine(8)
    seen = []
    gate = threading.Event()
    ctx = be.encode("i", b"o")
    spec = schema.steps[1]
    g = be.begin_step(ctx, (), spec, ())

    def land(req, t):
        seen.append(aeng.in_flight_names())
        gate.set()

    req = RS._EngineRequest(name=spec.name, tokens=g.drain(), remaining=len(g.tokens), issue_timestep=0,
                            priority="reasoning", seqno=0, on_complete=land)
    aeng.submit(req)
    assert gate.wait(10.0)
    aeng.drain(10.0)
    aeng.close()
    assert spec.name in seen[0]
    assert not aeng.in_flight_names()


def test_background_released_id_reused_while_landing():
    """The id of a request released by the background ticker can be reused by
    a submit made while the first is still landing."""
    schema = default_schema()
    be, eng = fake_backend(async_mode="background")
    aeng = be.make_async_engine(8)
    ctx = be.encode("i", b"o")
    landed = []
    specs = schema.steps[0], schema.steps[1]
    gens = [be.begin_step(ctx, (), s, ()) for s in specs]
    reqs = [RS._EngineRequest(name=s.name, tokens=g.drain(), remaining=len(g.tokens), issue_timestep=0,
                              priority="reasoning", seqno=0, on_complete=lambda r, t: landed.append(r.name))
            for s, g in zip(specs, gens)]
    eng.on_release = lambda: aeng.submit(reqs[1])
    aeng.submit(reqs[0])
    aeng.drain(10.0)
    aeng.close()
    assert sorted(landed) == sorted(s.name for s in specs)
    assert gens[0].handle.req == gens[1].handle.req
    assert reqs[1].tokens == HashBackend().begin_step(ctx, (), specs[1], ()).tokens


def test_summary_adds_percentiles():
    schema = default_schema()
    res, _ = episode("parallel_sync", HashBackend(), schema, 8)
    s = runners.summarize("parallel_sync", res, schema)
    assert s["latency_p50_ms"] <= s["latency_p99_ms"]
    assert s["latency_mean_ms"] == pytest.approx(float(np.mean([r.latency_ms for r in res])))


def test_kv_pool_exhaustion_is_a_policy_error():
    """Page reservations fail in begin_step (a BackendError) when the pool
    cannot hold the request, so the reference reuse_stale policy applies
    instead of a device allocation failing mid-tick."""
    schema = default_schema()
    be, eng = fake_backend(trunk_cache=1)
    runner = RS.make_runner(RS.SchedulerConfig(mode="parallel_sync", slots=8), be, schema)
    for t in range(2):
        runner.step(be.encode("i", RS.observation_for(0, t)), t)
    eng.pages_total = eng.stats()["pages_used"] + 16
    r = runner.step(be.encode("i", RS.observation_for(0, 2)), 2)
    assert r.failures                       # some branches could not reserve their pages
    assert len(r.failures) < len(schema.steps)
    assert be._live == 0 and be._reserved == 0


# ------------------------------------------------------- reuse-as-draft ----
def _fixed_obs_episode(mode, backend, schema, T, obs=b"same-frame"):
    """Episode whose observation never changes (repeated control steps on one
    frame): the reasoning a branch emits at t equals the content it was
    conditioned on at t - 1, so prev_content is a correct greedy draft."""
    runner = RS.make_runner(RS.SchedulerConfig(mode=mode, slots=8, latency=MODEL), backend, schema)
    ctx_instr = "pick up the object and place it on the target"
    return [runner.step(backend.encode(ctx_instr, obs), t) for t in range(T)]


@pytest.mark.parametrize("mode", ("sequential", "parallel_sync"))
@pytest.mark.parametrize("fixed", (True, False))
def test_draft_reuse_is_exactly_greedy(mode, fixed):
    """Reuse-as-draft changes how tokens are produced,
    not which: traces are byte-identical with and without it, over an
    autoregressive stand-in model.  On a fixed frame the drafts are accepted
    (decode iterations skipped); with a new frame every step they are not."""
    schema = default_schema()
    runs = {}
    for draft in (False, True):
        be, eng = fake_backend(autoregressive=True, draft_reuse=draft)
        if fixed:
            res = _fixed_obs_episode(mode, be, schema, 6)
        else:
            res, _ = episode(mode, be, schema, 6, seed=5)
        runs[draft] = (lines(res, schema), be.draft_stats, eng)
    assert runs[True][0] == runs[False][0]
    st = runs[True][1]
    assert st["drafted"] > 0 and runs[True][2].verify_calls > 0
    if fixed:
        assert st["accepted_tokens"] > 0.9 * st["draft_tokens"], st
        assert st["resolved_by_verify"] > 0, st
    else:
        assert st["accepted_tokens"] < 0.05 * st["draft_tokens"], st
    assert runs[False][1]["drafted"] == 0


def test_draft_reuse_skips_decode_ticks_on_a_fixed_frame():
    schema = default_schema()
    ticks = {}
    for draft in (False, True):
        be, eng = fake_backend(autoregressive=True, draft_reuse=draft)
        _fixed_obs_episode("parallel_sync", be, schema, 5)
        ticks[draft] = len(eng.occupancy_log)
    assert ticks[True] < 0.5 * ticks[False], ticks


# --------------------------------------------------- experiments harness ----
def test_reference_experiment_harness_runs_on_the_engine(tmp_path):
    """The unmodified reference `run_experiment` (every mode cell, traces.jsonl,
    comparison rows) with its backend factory served by EngineBackend
    (paper_2506_07639_b200.experiments): the cell traces equal the same
    harness over the synchronous HashBackend stand-in."""
    from ecot_sched.experiments import spec_from_dict
    from fake_engine import HashBackend

    from paper_2506_07639_b200.experiments import engine_backends, run_engine_experiment
    spec = spec_from_dict({"name": "eng", "modes": [{"mode": "sequential"}, {"mode": "parallel_sync"},
                                                    {"mode": "parallel_async"}],
                           "episode_len": 4, "repetitions": 2, "seed": 3, "slots": 8})
    be, _ = fake_backend(profile=spec.profile)
    out = run_engine_experiment(spec, tmp_path / "engine", backend=be)
    with engine_backends(lambda sp, rep: HashBackend(profile=sp.profile.with_seed(sp.profile.seed + rep))):
        ref = ecot_sched.experiments.run_experiment(spec, tmp_path / "hash")
    assert not out.aborted and len(out.cell_summaries) == len(spec.modes) * spec.repetitions
    for cell in sorted((tmp_path / "engine" / "eng").rglob("traces.jsonl")):
        other = tmp_path / "hash" / "eng" / cell.relative_to(tmp_path / "engine" / "eng")
        a = [line.split(b'"wall_ms"')[0] for line in cell.read_bytes().splitlines()]
        b = [line.split(b'"wall_ms"')[0] for line in other.read_bytes().splitlines()]
        assert a == b, cell
    assert ecot_sched.experiments._make_backend.__module__ == "ecot_sched.experiments"


@pytest.mark.parametrize("mode", ("sequential", "parallel_sync"))
def test_tag_in_prefill_is_exactly_greedy(mode):
    """The trunk owner's first token computed by the trunk prefill (its TAG row
    riding along) instead of a decode tick: identical traces, fewer ticks."""
    schema = default_schema()
    runs = {}
    for tag in (False, True):
        be, eng = fake_backend(autoregressive=True, tag_in_prefill=tag)
        res, _ = episode(mode, be, schema, 5, seed=2)
        runs[tag] = (lines(res, schema), len(eng.occupancy_log))
    assert runs[True][0] == runs[False][0]
    assert runs[True][1] < runs[False][1]


def test_close_leaves_a_shared_engine_open():
    """A backend built over a passed-in engine does not close it (another
    backend may share it); a backend that created its engine closes it."""
    class CountingEngine(FakeEngine):
        closed = 0

        def close(self):
            CountingEngine.closed += 1

    eng = CountingEngine()
    be = EngineBackend("tiny", engine=eng)
    be.close()
    assert CountingEngine.closed == 0
