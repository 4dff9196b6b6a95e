"""Engine-aware additions to the reference runners (`ecot_sched.schedulers`).

The reference runners are used as they are: `SequentialRunner` and
`ParallelSyncRunner` already batch on the GPU through `EngineBackend`'s
deferred generators (engine_backend.py).  This module adds only what the
reference cannot express:

* `EngineParallelAsyncRunner` -- the reference `ParallelAsyncRunner`
  (Alg. 1, `schedulers.py:459-552`) with its simulated `_MicroEngine`
  (`:244-299`) replaced by the backend's device engine when the backend has
  one (`make_async_engine`); with any other backend it *is* the reference
  runner.  `register()` installs it in the reference's runner table
  (`_RUNNERS`, `schedulers.py:719-730`), so `ecot_sched.run_episode` /
  `make_runner` pick it up;
* `BatchedEpisodes` -- BASELINE config 4: E independent episodes (each with
  its own reference runner and cache, as `run_episode` gives them,
  `schedulers.py:818`) stepped together so that every timestep's E x (N+1)
  branch requests decode as one batch;
* `summarize` -- the reference `summarize_results` (`schedulers.py:830-849`)
  plus p50/p99 latency.
"""

from __future__ import annotations

import dataclasses
import time
from typing import Sequence

import numpy as np

from .refapi import backends as _rb
from .refapi import schedulers as _rs
from .refapi import trace as _rt

DEFAULT_INSTRUCTION = "pick up the object and place it on the target"   # schedulers.py:813


class EngineParallelAsyncRunner(_rs.ParallelAsyncRunner):
    """Reference Fast-ECoT async runner over the device batcher (see module doc)."""

    def __init__(self, backend, schema, config):
        super().__init__(backend, schema, config)
        factory = getattr(backend, "make_async_engine", None)
        if factory is not None:
            self.engine = factory(config.slots)

    def step(self, ctx, timestep: int):
        hold = getattr(self.engine, "hold", None)
        if hold is None or not self._warm:
            return super().step(ctx, timestep)
        hold()               # the device engine pauses background ticks until the action is submitted
        try:
            return super().step(ctx, timestep)
        finally:
            self.engine.release()

    def close(self) -> None:
        close = getattr(self.engine, "close", None)
        if close is not None:
            close()


def register() -> None:
    """Install the engine-aware runner in the reference's runner table."""
    _rs._RUNNERS["parallel_async"] = EngineParallelAsyncRunner


class _Prefetched:
    """Backend proxy that serves requests issued ahead of a runner's step
    (keyed by (prefix, step name, prev_content)), so the reference runner
    consumes generators that were batched with other episodes' requests."""

    deterministic = True
    supports_prefix_conditioning = True

    def __init__(self, inner, table: dict):
        self.inner = inner
        self.table = table

    def encode(self, instruction: str, observation: bytes):
        return self.inner.encode(instruction, observation)

    def begin_step(self, context, prefix, step, prev_content):
        out = self.table.pop((tuple(prefix), step.name, tuple(prev_content)), None)
        if out is None:
            return self.inner.begin_step(context, prefix, step, prev_content)
        if isinstance(out, BaseException):
            raise out
        return out


class BatchedEpisodes:
    """BASELINE config 4: independent episodes stepped in lockstep.

    Each episode keeps its own reference `ParallelSyncRunner` (cache, previous
    trace, accounting).  Per timestep, the branch requests of every episode
    are issued first -- the reference job construction, `prefix_i =
    prev.steps[:i]`, `prev_content = prev.steps[i]` (`schedulers.py:399-404`)
    -- so they decode as one batch, then each runner's own `step` consumes
    its episode's generators.  Timestep 0 is the reference warm-up
    (sequential pass, `schedulers.py:329-351`), batched across episodes step
    by step."""

    def __init__(self, config, backend, schema, seeds: Sequence[int],
                 instruction: str = DEFAULT_INSTRUCTION):
        if config.mode != "parallel_sync":
            raise _rs.ConfigError("mode", "batched episodes drive the parallel_sync runner")
        self.backend, self.schema, self.config = backend, schema, config
        self.seeds = list(seeds)
        self.instruction = instruction
        self.runners = [_rs.make_runner(config, backend, schema) for _ in self.seeds]

    def _issue(self, table: dict, ctx, prefix: tuple, spec, prev: tuple):
        try:
            g = self.backend.begin_step(ctx, prefix, spec, prev)
        except _rb.BackendError as exc:
            table[(prefix, spec.name, prev)] = exc
            return None
        table[(prefix, spec.name, prev)] = g
        return g

    def step(self, timestep: int) -> list:
        t0 = time.perf_counter()
        ctxs = [self.backend.encode(self.instruction, _rs.observation_for(s, timestep)) for s in self.seeds]
        tables: list[dict] = [{} for _ in self.seeds]
        if self.runners[0]._prev_trace is None:
            prefixes: list[list[int]] = [[] for _ in self.seeds]
            alive = [True] * len(self.seeds)
            for spec in self.schema.steps:
                gens = [self._issue(tables[e], ctxs[e], tuple(prefixes[e]), spec, ()) if alive[e] else None
                        for e in range(len(self.seeds))]
                for e, g in enumerate(gens):
                    if g is None:
                        alive[e] = False
                    else:
                        prefixes[e].extend(g.tokens)   # the first read decodes the whole level
        else:
            for e, r in enumerate(self.runners):
                prefix: list[int] = []
                for i, spec in enumerate(self.schema.steps):
                    prev = tuple(r._prev_trace.steps[i][1])
                    self._issue(tables[e], ctxs[e], tuple(prefix), spec, prev)
                    prefix.extend(prev)
        results = []
        try:
            for e, r in enumerate(self.runners):
                r.backend = _Prefetched(self.backend, tables[e])
                try:
                    results.append(r.step(ctxs[e], timestep))
                finally:
                    r.backend = self.backend
        finally:
            discard = getattr(self.backend, "discard", None)
            for table in tables:   # requests no runner consumed (an aborted episode)
                for g in table.values():
                    if discard is not None and hasattr(g, "handle"):
                        discard(g.handle)
        if self.config.wall_clock:
            ms = (time.perf_counter() - t0) * 1000.0
            results = [dataclasses.replace(r, latency_ms=ms) for r in results]
        return results


def summarize(mode: str, results: Sequence, schema) -> dict:
    """Reference summary (`summarize_results`: mean / population std,
    staleness histogram) plus p50 / p99 latency."""
    out = _rs.summarize_results(mode, results, schema)
    lat = np.asarray([r.latency_ms for r in results], dtype=np.float64)
    out["latency_p50_ms"] = float(np.percentile(lat, 50))
    out["latency_p99_ms"] = float(np.percentile(lat, 99))
    return out


def plain_trace(trace: _rt.ReasoningTrace) -> _rt.ReasoningTrace:
    """The trace with every step's tokens as a plain tuple (device sequences
    resolved), e.g. before pickling or gathering across ranks."""
    return dataclasses.replace(trace, steps=tuple((n, tuple(int(t) for t in toks)) for n, toks in trace.steps))
