"""`EngineBackend`: the reference `GenerationBackend` served by the B200 engine.

Drop-in for the protocol of `pkg/src/ecot_sched/backends.py:98-110`
(`encode`, `begin_step`, `deterministic`, `supports_prefix_conditioning`),
plus the two runner-level extensions the GPU-aware runners use
(schedulers.py in this package):

* `begin_steps(ctx, jobs)` -- the N+1 branch jobs of one Fast-ECoT timestep
  (reference `ParallelSyncRunner`, schedulers.py:399-420) decoded as one
  batch: the longest prefix is prefilled once as a *trunk*, every job forks
  the trunk's paged KV at its own prefix length (copy-on-write of the partial
  page only) and all branches decode together;
* `make_async_engine(slots)` -- the continuous batcher for Fast ECoT async
  (reference `_MicroEngine`, schedulers.py:244-299) whose ticks are real
  decode iterations.

Reuse across timesteps: trunks live in a content-addressed prefix cache keyed
by (vision seed, input ids); a request whose context and prefix extend a
cached trunk forks it at the longest common prefix and prefills only the
remainder (sequential ECoT extends the trunk step by step; repeated
contexts reuse whole trunks).

Errors from the engine surface as `BackendError` subclasses (`EngineError`)
so the runners' `reuse_stale` / `abort_episode` policies apply unchanged
(schedulers.py:422-434, :510-517).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from .backends import (BackendError, EngineError, StepGenerator, SyntheticProfile, default_profile,
                       encode_tokens, length_plan)
from .batching import ACTION
from .engine import Engine, PRIO_ACTION, PRIO_REASONING
from .model import VIS_ID, context_ids, get_config, step_tag, text_ids, vision_seed
from .trace import Context, StepSpec, TokenSeq


@dataclass
class _Trunk:
    vseed: int
    ids: np.ndarray
    seq: int
    stamp: int


@dataclass
class EngineRequest:
    """A prepared branch request (async engine handle)."""

    name: str
    step: StepSpec
    length: int
    truncated: bool
    tag: int
    branch: int
    priority: int
    issue_timestep: int = 0
    lane: int = 0
    req: int = -1
    tokens: TokenSeq = ()
    on_complete: Optional[Callable[["EngineRequest", int], None]] = None
    done: bool = False


class EngineBackend:
    deterministic = True
    supports_prefix_conditioning = True

    def __init__(self, config="tiny", dtype: str = "f32", seed: int = 0,
                 profile: SyntheticProfile | None = None, device: int = 0,
                 engine: Engine | None = None, trunk_cache: int = 64, async_streams: int = 1,
                 request_log: list | None = None, **engine_kw):
        """`async_streams=1`: lockstep async batcher (reference landing order,
        byte-comparable traces); `2`: two-stream async scheduler (action on the
        high-priority lane, reasoning refresh running on the low-priority lane in
        the background, across control steps).  `request_log`: if a list,
        every completed request appends (context, prefix, step name,
        prev_content, tokens) -- used by per-request parity checks."""
        self.cfg = get_config(config)
        self.async_streams = async_streams
        self.request_log = request_log
        self.engine = engine or Engine(self.cfg, dtype=dtype, device=device, seed=seed, **engine_kw)
        self.profile = profile or default_profile(seed)
        self._trunks: list[_Trunk] = []
        self._trunk_cap = trunk_cache
        self._clock = 0
        # request -> handle, shared by every backend driving this engine (a
        # request left in flight by one backend may complete in another's run)
        if not hasattr(self.engine, "owners"):
            self.engine.owners = {}
        self._owners: dict[int, EngineRequest] = self.engine.owners
        self._async_engines: list = []
        self._slots = 8
        self.requests = 0

    # -- protocol ------------------------------------------------------------
    def encode(self, instruction: str, observation: bytes) -> Context:
        return Context(instruction, observation, encode_tokens(instruction, observation))

    def begin_step(self, context: Context, prefix: TokenSeq, step: StepSpec,
                   prev_content: TokenSeq) -> StepGenerator:
        out = self.begin_steps(context, [(step, prefix, prev_content)], priorities=[PRIO_ACTION])[0]
        if isinstance(out, BackendError):
            raise out
        return out

    def begin_steps(self, context: Context, jobs: Sequence[tuple[StepSpec, TokenSeq, TokenSeq]],
                    priorities: Sequence[int] | None = None) -> list:
        """Decode several branch requests of one context as one batch.
        Returns a StepGenerator or a BackendError per job (job order)."""
        if priorities is None:  # reference fan-out order: the action step is last
            priorities = [PRIO_REASONING] * (len(jobs) - 1) + [PRIO_ACTION]
        outcomes: list = [None] * len(jobs)
        handles: dict[int, EngineRequest] = {}
        order = sorted(range(len(jobs)), key=lambda i: -len(jobs[i][1]))  # longest trunk first
        for i in order:
            spec, prefix, prev = jobs[i]
            try:
                handles[i] = self._prepare(context, prefix, spec, prev, priorities[i])
            except BackendError as exc:
                outcomes[i] = exc
        for i in sorted(handles):
            self._submit(handles[i], None)
        for i in sorted(handles):
            h = handles[i]
            if not h.done:
                self._run(h.req, 0)
            outcomes[i] = StepGenerator(h.tokens, truncated=h.truncated)
        return outcomes

    def begin_steps_multi(self, contexts: Sequence[Context], jobs_per_context: Sequence[Sequence],
                          priorities=None) -> list[list]:
        """Branch jobs of several independent contexts (episodes) decoded as one
        batch (BASELINE config 4).  Returns per context a list of
        StepGenerator / BackendError in job order."""
        outcomes: list[list] = [[None] * len(j) for j in jobs_per_context]
        handles: dict[tuple[int, int], EngineRequest] = {}
        self._ensure_slots(sum(len(j) for j in jobs_per_context))
        for e, (ctx, jobs) in enumerate(zip(contexts, jobs_per_context)):
            prios = priorities[e] if priorities else [PRIO_REASONING] * (len(jobs) - 1) + [PRIO_ACTION]
            for i in sorted(range(len(jobs)), key=lambda i: -len(jobs[i][1])):
                spec, prefix, prev = jobs[i]
                try:
                    handles[(e, i)] = self._prepare(ctx, prefix, spec, prev, prios[i])
                except BackendError as exc:
                    outcomes[e][i] = exc
        for key in sorted(handles):
            self._submit(handles[key], None)
        for key in sorted(handles):
            h = handles[key]
            if not h.done:
                self._run(h.req, 0)
            outcomes[key[0]][key[1]] = StepGenerator(h.tokens, truncated=h.truncated)
        return outcomes

    def make_async_engine(self, slots: int):
        if self.async_streams == 2:
            return TwoStreamAsyncEngine(self, slots)
        return AsyncEngine(self, slots)

    def _ensure_slots(self, n: int) -> None:
        """Grow the batcher so a multi-episode barrier fits in one batch."""
        if n > self._slots:
            self._slots = min(n, self.engine.max_slots)
            self.engine.set_slots(self._slots)

    # -- trunks & branches -----------------------------------------------------
    def _branch_point(self, vseed: int, ids: np.ndarray) -> tuple[int, bool]:
        """Sequence whose KV covers ids exactly up to len(ids) (possibly longer)."""
        n = ids.size
        best, best_lcp = None, 0
        for tr in self._trunks:
            if tr.vseed != vseed:
                continue
            m = min(n, tr.ids.size)
            neq = np.flatnonzero(tr.ids[:m] != ids[:m])
            lcp = int(neq[0]) if neq.size else m
            if lcp > best_lcp or (lcp == best_lcp and best is not None and tr.ids.size < best.ids.size):
                best, best_lcp = tr, lcp
        self._clock += 1
        if best is not None and best_lcp == n:
            best.stamp = self._clock
            return best.seq, False
        eng = self.engine
        seq = eng.seq_fork(best.seq, best_lcp) if best is not None and best_lcp > 0 else eng.seq_create()
        try:
            eng.prefill(seq, ids[best_lcp:], vseed, VIS_ID)
        except EngineError:
            eng.seq_free(seq)
            raise
        self._trunks.append(_Trunk(vseed, ids.copy(), seq, self._clock))
        if len(self._trunks) > self._trunk_cap:
            victim = min(self._trunks, key=lambda t: t.stamp)
            self._trunks.remove(victim)
            eng.seq_free(victim.seq)
        return seq, True

    def _prepare(self, ctx: Context, prefix: TokenSeq, spec: StepSpec, prev: TokenSeq,
                 priority: int, timestep: int = 0) -> EngineRequest:
        plan = length_plan(self.profile, ctx, spec, prev)  # BackendError on unknown step
        ids = np.asarray(context_ids(ctx, self.cfg) + text_ids(prefix), dtype=np.int32)
        vseed = vision_seed(ctx.observation)
        trunk, _ = self._branch_point(vseed, ids)
        branch = self.engine.seq_fork(trunk, ids.size)
        h = EngineRequest(spec.name, spec, plan.length, plan.truncated, step_tag(spec), branch,
                          priority, issue_timestep=timestep)
        if self.request_log is not None:
            h.log = (ctx, tuple(prefix), spec.name, tuple(prev))
        return h

    def _submit(self, h: EngineRequest, on_complete) -> None:
        h.on_complete = on_complete
        h.req = self.engine.submit(h.branch, h.tag, h.length, h.priority)
        self._owners[h.req] = h
        self.requests += 1

    def _run(self, stop_req: int, timestep: int) -> list[int]:
        occupancy, done = self.engine.run(stop_req)
        for req, _tick in done:
            h = self._owners.pop(req, None)
            if h is None:
                raise EngineError(f"request {req} completed without an owner")
            h.tokens = tuple(self.engine.request_tokens(req, h.length))
            h.done = True
            self._log(h)
            self.engine.request_release(req)
            self.engine.seq_free(h.branch)
            if h.on_complete is not None:
                h.on_complete(h, timestep)
        return occupancy

    def _log(self, h: EngineRequest) -> None:
        if self.request_log is not None and getattr(h, "log", None) is not None:
            self.request_log.append(h.log + (h.tokens,))

    def close(self) -> None:
        for eng in list(self._async_engines):
            eng.close()
        self.engine.close()


class AsyncEngine:
    """Continuous batcher facade used by `ParallelAsyncRunner`: same surface
    as the reference `_MicroEngine` (submit / in_flight_names), but each tick
    is one decode iteration of every admitted row on the GPU."""

    def __init__(self, backend: EngineBackend, slots: int):
        self.backend = backend
        backend.engine.set_slots(slots)
        backend._slots = slots
        self._inflight: dict[int, EngineRequest] = {}

    def prepare(self, ctx, prefix, spec, prev_content, priority: str, timestep: int) -> EngineRequest:
        prio = PRIO_ACTION if priority == ACTION else PRIO_REASONING
        return self.backend._prepare(ctx, prefix, spec, prev_content, prio, timestep)

    def submit(self, h: EngineRequest, on_complete) -> None:
        def landed(req: EngineRequest, t: int) -> None:
            self._inflight.pop(req.req, None)
            if on_complete is not None:
                on_complete(req, t)

        self.backend._submit(h, landed)
        self._inflight[h.req] = h

    def in_flight_names(self) -> set[str]:
        return {h.name for h in self._inflight.values()}

    def idle(self) -> bool:
        return not self._inflight

    def run_until_complete(self, h: EngineRequest, timestep: int) -> list[int]:
        self._now = timestep
        return self.backend._run(h.req, timestep)

    def drain(self) -> None:
        """Decode every request still in flight (they land at the last control
        timestep) so the engine is idle before it is handed to another runner."""
        if self._inflight:
            self.backend._run(-1, getattr(self, "_now", 0))

    def close(self) -> None:
        pass


class TwoStreamAsyncEngine:
    """Fast ECoT async as two CUDA streams (north_star item 4).

    The action request of each control step decodes on lane 0 (highest stream
    priority) against the last committed reasoning; reasoning-refresh requests
    decode on lane 1 (lowest priority), driven by a background host thread
    that keeps ticking across control steps.  A request's content is fixed at
    issue (the snapshot it was prepared against, as in the reference,
    `schedulers.py:471-492`); it lands into the cache at the control timestep
    current when it completes.  Landing order is real-time, so traces are
    checked per request (identical (context, prefix, step) -> identical tokens)
    rather than byte-for-byte against the simulated clock."""

    def __init__(self, backend: EngineBackend, slots: int):
        self.backend = backend
        eng = backend.engine
        eng.set_slots(slots)
        eng.set_slots_lane(1, slots)
        backend._slots = slots
        self._lock = threading.Lock()
        self._inflight: dict[int, EngineRequest] = {}
        self._landing = 0  # completed requests the background thread is still landing
        self._now = 0
        self._errors: list[BaseException] = []
        self._stop = threading.Event()
        self._work = threading.Event()
        self._thread = threading.Thread(target=self._loop, name="fastecot-reasoning-lane", daemon=True)
        self._thread.start()
        backend._async_engines.append(self)

    # -- runner surface (same as AsyncEngine / the reference _MicroEngine) ----
    def prepare(self, ctx, prefix, spec, prev_content, priority: str, timestep: int) -> EngineRequest:
        prio = PRIO_ACTION if priority == ACTION else PRIO_REASONING
        with self._lock:  # trunk cache / prefill / fork all happen on lane 0
            h = self.backend._prepare(ctx, prefix, spec, prev_content, prio, timestep)
        h.lane = 0 if prio == PRIO_ACTION else 1
        return h

    def submit(self, h: EngineRequest, on_complete) -> None:
        h.on_complete = on_complete
        if h.lane == 0:
            h.req = self.backend.engine.submit_lane(0, h.branch, h.tag, h.length, h.priority)
            return
        with self._lock:
            h.req = self.backend.engine.submit_lane(1, h.branch, h.tag, h.length, h.priority)
            self._inflight[h.req] = h
        self._work.set()

    def in_flight_names(self) -> set[str]:
        with self._lock:
            return {h.name for h in self._inflight.values()}

    def idle(self) -> bool:
        with self._lock:
            return not self._inflight and not self._landing

    def run_until_complete(self, h: EngineRequest, timestep: int) -> list[int]:
        self._raise_background_error()
        self._now = timestep
        eng = self.backend.engine
        occupancy, _ = eng.run(h.req, lane=0)
        h.tokens = tuple(eng.request_tokens(h.req, h.length))
        h.done = True
        eng.request_release(h.req)
        eng.seq_free(h.branch)
        self.backend._log(h)
        return occupancy

    def set_timestep(self, timestep: int) -> None:
        self._now = timestep

    # -- background lane ----------------------------------------------------
    def _loop(self) -> None:
        eng = self.backend.engine
        while not self._stop.is_set():
            with self._lock:
                busy = bool(self._inflight)
            if not busy:
                self._work.wait(0.05)
                self._work.clear()
                continue
            try:
                _, done = eng.run(-1, lane=1, max_ticks=4)
                for req, _tick in done:
                    # take the handle out before the id is released: a submit on
                    # the runner thread may reuse the id right after the release
                    with self._lock:
                        h = self._inflight.pop(req)
                        self._landing += 1
                    try:
                        h.tokens = tuple(eng.request_tokens(req, h.length))
                        h.done = True
                        eng.request_release(req)
                        eng.seq_free(h.branch)
                        self.backend._log(h)
                        if h.on_complete is not None:
                            h.on_complete(h, self._now)
                    finally:
                        with self._lock:
                            self._landing -= 1
            except BaseException as exc:  # surfaced on the runner thread
                self._errors.append(exc)
                self._stop.set()

    def _raise_background_error(self) -> None:
        if self._errors:
            raise EngineError(f"background reasoning lane failed: {self._errors[0]!r}")

    def drain(self, timeout: float = 60.0) -> None:
        """Wait until every background request has landed."""
        import time
        t0 = time.time()
        while not self.idle() and time.time() - t0 < timeout:
            self._raise_background_error()
            time.sleep(0.002)

    def close(self) -> None:
        self._stop.set()
        self._work.set()
        self._thread.join(timeout=10.0)
