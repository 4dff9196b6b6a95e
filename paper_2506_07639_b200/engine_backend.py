"""`EngineBackend`: the reference `GenerationBackend` served by the B200 engine.

Implements the protocol of `ecot_sched.backends.GenerationBackend`
(`pkg/src/ecot_sched/backends.py:98-110`: `encode`, `begin_step`,
`deterministic`, `supports_prefix_conditioning`) so the reference's own
runners (`ecot_sched.schedulers`) drive the GPU unchanged.

Batching without a runner fork.  `begin_step` does not decode: it prepares the
request on the device (trunk lookup / prefill, copy-on-write fork of the
paged KV at the prefix length) and returns a `StepGenerator` whose `tokens`
is a `DeviceTokens` sequence -- its length (the length oracle) is known at
once, its ids only when the request completes.  The first time any pending
request's ids are read, *every* pending request is submitted and the engine
decodes them as one continuous batch until that request completes.  The
reference `ParallelSyncRunner` issues all N+1 branch requests of a timestep
before it reads any content (`schedulers.py:399-420`), so its branches decode
together on the GPU; `SequentialRunner` reads each step before issuing the
next (`schedulers.py:329-351`), so it decodes one request at a time, as
Alg. A.1 prescribes.

Reuse across timesteps: trunks live in a content-addressed prefix cache keyed
by (vision seed, input ids); a request whose context and prefix extend a
cached trunk forks it at the longest common prefix and prefills only the
remainder (sequential ECoT extends the trunk step by step; repeated contexts
reuse whole trunks).

For Fast ECoT async (`schedulers.py:459-552`) `make_async_engine(slots)`
returns a device engine with the surface of the reference `_MicroEngine`
(`submit(_EngineRequest)`, `tick(timestep) -> (occupied, completed)`,
`in_flight_names()`, `idle()`; `schedulers.py:244-299`), each tick being one
real decode iteration; `runners.EngineParallelAsyncRunner` plugs it into the
reference runner.

Errors surface as `EngineError`, an `ecot_sched.backends.BackendError`, and
every limit the device would reject at submission (request length, context
length, live requests) is checked in `begin_step`, before the fork, so the
reference failure policies (`schedulers.py:411-434`, `:481-483`,
`:510-517`) see them.
"""

from __future__ import annotations

import contextlib
import threading
import time
from collections.abc import Sequence as _SequenceABC
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np

from .backends import (BackendError, EngineError, StepGenerator, SyntheticProfile, default_profile,
                       encode_context, length_plan)
from .engine import Engine, PRIO_ACTION, PRIO_REASONING
from .model import PAGE_TOKENS, ROPE_MAX_POS, VIS_ID, context_ids, get_config, step_tag, text_ids, vision_seed
from .refapi import batching as _rbatch
from .refapi import trace as _rt

REQUEST_CAP = 1024  # tokens per request (device token arena slot, csrc/engine.cu kRequestCap)


@dataclass(eq=False)   # identity: list.remove must not compare the id arrays
class _Trunk:
    vseed: int
    ids: np.ndarray
    seq: int
    stamp: int


class DeviceRequest:
    """One branch request on the device."""

    __slots__ = ("name", "length", "truncated", "tag", "branch", "priority", "lane", "req", "tokens",
                 "error", "log", "on_complete", "waiter", "ids", "vseed", "reserve", "draft", "prefix")

    def __init__(self, name, length, truncated, tag, priority, ids, vseed):
        self.name, self.length, self.truncated = name, length, truncated
        self.tag, self.priority = tag, priority
        self.ids, self.vseed = ids, vseed  # framed input; forked off a trunk when materialised
        self.branch = -1                   # device sequence once materialised
        self.reserve = 0                   # KV pages held for it until it completes
        self.lane = 0
        self.req = -1                      # device request id once submitted
        self.tokens: Optional[tuple] = None
        self.error: Optional[BaseException] = None
        self.log = None
        self.on_complete: Optional[Callable[["DeviceRequest"], None]] = None
        self.waiter = None                 # engine that owns completion (two-stream lane 1)
        self.draft: tuple = ()             # prev_content to verify as a greedy draft (draft_reuse)
        self.prefix: tuple = ()            # tokens already produced by the draft verification

    @property
    def done(self) -> bool:
        return self.tokens is not None


class DeviceTokens(_SequenceABC):
    """Token ids of a device request.  `len()` is known at issue (the length
    oracle); reading any id resolves the request, driving the engine until it
    completes (see the module docstring)."""

    __slots__ = ("handle", "_owner")

    def __init__(self, handle: DeviceRequest, owner: "EngineBackend"):
        self.handle = handle
        self._owner = owner

    def resolve(self) -> tuple:
        h = self.handle
        if h.tokens is None:
            self._owner._resolve(h)
        return h.tokens

    def __len__(self) -> int:
        return self.handle.length

    def __getitem__(self, i):
        return self.resolve()[i]

    def __iter__(self):
        return iter(self.resolve())

    def __eq__(self, other):
        if isinstance(other, (tuple, list, DeviceTokens)):
            return self.resolve() == tuple(other)
        return NotImplemented

    def __hash__(self):
        return hash(self.resolve())

    def __array__(self, dtype=None, copy=None):
        return np.asarray(self.resolve(), dtype=dtype)

    def __repr__(self) -> str:
        h = self.handle
        return f"DeviceTokens({h.tokens!r})" if h.tokens is not None else f"DeviceTokens(<{h.length} pending>)"


class DeviceStepGenerator(StepGenerator):
    """`StepGenerator` (`backends.py:69-95`) over a device request; the base
    constructor is not called because it would materialise the tokens."""

    def __init__(self, handle: DeviceRequest, owner: "EngineBackend"):  # noqa: D107
        self._seq = DeviceTokens(handle, owner)
        self.truncated = handle.truncated
        self.reported_tokens = handle.length
        self._pos = 0

    @property
    def tokens(self):
        return self._seq

    @property
    def handle(self) -> DeviceRequest:
        return self._seq.handle


def device_handle(tokens) -> Optional[DeviceRequest]:
    return tokens.handle if isinstance(tokens, DeviceTokens) else None


class EngineBackend:
    deterministic = True
    supports_prefix_conditioning = True

    def __init__(self, config="tiny", dtype: str = "f32", seed: int = 0,
                 profile: SyntheticProfile | None = None, device: int = 0,
                 engine: Engine | None = None, trunk_cache: int = 64, async_mode: str = "lockstep",
                 request_log: list | None = None, draft_reuse: bool = False, background_depth: int = 1,
                 tag_in_prefill: bool | None = None, **engine_kw):
        """`async_mode="lockstep"`: the async runner's device engine advances
        exactly as many decode iterations as each control step's action needs
        (the reference landing order, byte-comparable traces);
        `"background"`: a background ticker keeps the reasoning refresh decoding
        between and during control steps, the action joins its ticks at high
        priority (`BackgroundAsyncEngine`).  `request_log`: if a list,
        every completed request appends (context, prefix, step name,
        prev_content, tokens) -- used by per-request parity checks.
        `draft_reuse`: verify each synchronous request's `prev_content` as a
        greedy draft in one batched forward before decoding (SURVEY §8(f)
        rank 1; `_verify_drafts`); the tokens are those of plain greedy
        decoding, only the decode iterations for the accepted prefix are
        skipped."""
        self.cfg = get_config(config)
        if async_mode not in ("lockstep", "background"):
            raise ValueError(f"async_mode must be 'lockstep' or 'background', got {async_mode!r}")
        self.async_mode = async_mode
        self.request_log = request_log
        self._owns_engine = engine is None   # a passed-in engine may be shared: close() leaves it open
        self.engine = engine or Engine(self.cfg, dtype=dtype, device=device, seed=seed, **engine_kw)
        self.profile = profile or default_profile(seed)
        self._trunks: list[_Trunk] = []
        self._trunk_cap = trunk_cache
        self._clock = 0
        self._lock = threading.RLock()
        self._fg = 0                                    # foreground threads waiting for / holding the lock
        self._fg_cv = threading.Condition()
        self._pending: list[DeviceRequest] = []
        self._owners: dict[int, DeviceRequest] = {}
        self._live = 0                                  # prepared, not yet released
        self._reserved = 0                              # KV pages held by live requests
        self._live_cap = max(4 * self.engine.max_slots, 256)   # device token arena slots
        self._async_engines: list = []
        self._slots = 8
        self._fixed_slots = False    # an async engine fixes the batcher to the runner's slots
        self.requests = 0
        self.draft_reuse = draft_reuse
        self.background_depth = background_depth   # decode ticks the background ticker keeps queued
        # the request owning a new trunk (the longest: an async action) gets its
        # first token from the trunk prefill itself -- its TAG row rides along
        # with the trunk rows -- saving one decode tick; exact greedy (same
        # token), but it moves completions one tick earlier, so the lockstep
        # mode (the reference landing order) keeps it off
        self.tag_in_prefill = (async_mode == "background") if tag_in_prefill is None else tag_in_prefill
        self.tag_in_prefill &= getattr(self.engine, "supports_prefill_heads", True)
        self.draft_stats = {"requests": 0, "drafted": 0, "draft_tokens": 0, "accepted_tokens": 0,
                            "verified_tokens": 0, "resolved_by_verify": 0, "verify_forwards": 0,
                            "verify_rows": 0}

    @contextlib.contextmanager
    def _foreground(self):
        """The backend lock for a runner-thread operation.  A background
        ticker (BackgroundAsyncEngine) only takes the lock between ticks when
        no foreground operation is waiting, so control steps never starve
        behind a stream of decode ticks."""
        with self._fg_cv:
            self._fg += 1
        try:
            with self._lock:
                yield
        finally:
            with self._fg_cv:
                self._fg -= 1
                self._fg_cv.notify_all()

    def _background_turn(self):
        """Acquire the lock for one background tick (after any waiting
        foreground operation); use as `with be._background_turn():`."""
        with self._fg_cv:
            while self._fg:
                self._fg_cv.wait(0.01)
        return self._lock

    # -- protocol --------------------------------------------------------------
    def encode(self, instruction: str, observation: bytes) -> _rt.Context:
        return encode_context(instruction, observation)

    def begin_step(self, context: _rt.Context, prefix, step: _rt.StepSpec,
                   prev_content) -> StepGenerator:
        with self._foreground():
            h = self._prepare(context, prefix, step, prev_content, PRIO_REASONING)
            self._pending.append(h)
            self._ensure_slots(len(self._pending) + len(self._owners))
        return DeviceStepGenerator(h, self)

    def make_async_engine(self, slots: int):
        if self.async_mode == "background":
            return BackgroundAsyncEngine(self, slots)
        return AsyncDeviceEngine(self, slots)

    # -- batching ----------------------------------------------------------------
    def flush(self) -> None:
        """Materialise and submit every pending request, in issue order (they
        join the next decode tick)."""
        with self._foreground():
            self._materialize()
            pending, self._pending = self._pending, []
            if self.draft_reuse:
                self._verify_drafts(pending)
            for h in pending:
                if h.tokens is None:
                    self._submit(h, 0)

    def _verify_drafts(self, hs: list[DeviceRequest]) -> None:
        """Reuse-as-draft (anchor: the reference's reuse
        draw returns prev_content verbatim, `backends.py:202-204`, and the
        runners pass it at `schedulers.py:404`, `:478`).  For every request
        with a draft d (its prev_content, cut to length - 1): one batched
        forward over all of them feeds [TAG, d_0 .. d_m-1] after the branch
        and returns the greedy tokens g_0 .. g_m; the accepted prefix is the
        longest a with g_i == d_i (i < a), so g_0 .. g_a are exactly the
        tokens greedy decoding would emit (each was computed from the true
        prefix).  The branch keeps the KV of those a + 1 inputs (the rest is
        truncated) and decodes only the remaining length - a - 1 tokens,
        starting from g_a -- or completes with no decode at all."""
        st = self.draft_stats
        todo = []
        for h in hs:
            if h.error is not None or h.tokens is not None or h.branch < 0:
                continue
            st["requests"] += 1
            d = h.draft[: max(0, h.length - 1)]
            if not d:
                continue
            todo.append((h, d))
        if not todo:
            return
        inputs = [[h.tag] + text_ids(d) for h, d in todo]
        eng = self.engine
        try:
            outs = eng.verify([h.branch for h, _ in todo], inputs)
        except EngineError as exc:
            for h, _ in todo:
                h.error = exc
                self._release(h)
            return
        st["verify_forwards"] += 1
        st["verify_rows"] += sum(len(x) for x in inputs)
        for (h, d), g in zip(todo, outs):
            g = [int(x) for x in g]
            a = 0
            while a < len(d) and g[a] == int(d[a]):
                a += 1
            verified = tuple(g[: a + 1])
            base = h.ids.size
            eng.seq_truncate(h.branch, base + len(verified))
            st["drafted"] += 1
            st["draft_tokens"] += len(d)
            st["accepted_tokens"] += a
            st["verified_tokens"] += len(verified)
            if len(verified) >= h.length:
                h.tokens = verified[: h.length]
                st["resolved_by_verify"] += 1
                if self.request_log is not None and h.log is not None:
                    self.request_log.append(h.log + (h.tokens,))
                if h.on_complete is not None:
                    h.on_complete(h)
                self._release(h)
            else:
                h.prefix = verified

    def _resolve(self, h: DeviceRequest) -> None:
        if h.waiter is not None:
            h.waiter.wait_for(h)
            return
        with self._foreground():
            if h.tokens is not None:
                return
            if h.req < 0 and h.error is None:
                self.flush()
            if h.error is not None:
                raise EngineError(f"request {h.name!r} failed: {h.error}") from h.error
            self._run(h.req)
            if h.tokens is None:
                raise EngineError(f"request {h.name!r} did not complete")

    def _ensure_slots(self, n: int) -> None:
        """Grow the batcher so every request issued together decodes in one batch."""
        if n > self._slots and not self._fixed_slots:
            self._slots = min(max(n, 2 * self._slots), self.engine.max_slots)
            self.engine.set_slots(self._slots)

    # -- trunks & branches -------------------------------------------------------
    def _prepare(self, ctx: _rt.Context, prefix, spec: _rt.StepSpec, prev, priority: int) -> DeviceRequest:
        """Plan a request and check every limit the device could reject later
        (request cap, max_pos, live requests, KV pages); nothing on the device
        changes yet -- the trunk prefill and the fork happen when the request
        is materialised (`_materialize`), longest input first."""
        plan = length_plan(self.profile, ctx, spec, prev)  # BackendError on unknown step
        h = self._new_request(ctx, prefix, spec, plan.length, plan.truncated, priority)
        if self.draft_reuse and priority == PRIO_REASONING:
            h.draft = tuple(int(x) for x in prev)
        if self.request_log is not None:
            h.log = (ctx, tuple(prefix), spec.name, tuple(prev))
        return h

    def _new_request(self, ctx: _rt.Context, prefix, spec: _rt.StepSpec, length: int, truncated: bool,
                     priority: int) -> DeviceRequest:
        ids = np.asarray(context_ids(ctx, self.cfg) + text_ids(prefix), dtype=np.int32)
        if not 1 <= length <= REQUEST_CAP:
            raise EngineError(f"step {spec.name!r}: {length} tokens outside the request cap [1, {REQUEST_CAP}]")
        if ids.size + 1 + length > ROPE_MAX_POS:
            raise EngineError(f"step {spec.name!r}: context {ids.size} + {length} tokens exceed "
                              f"max_pos {ROPE_MAX_POS}")
        if self._live >= self._live_cap:
            raise EngineError(f"too many live requests ({self._live})")
        h = DeviceRequest(spec.name, length, truncated, step_tag(spec), priority, ids,
                          vision_seed(ctx.observation))
        self._reserve_pages(h)
        self._live += 1
        return h

    def begin_completion(self, context: _rt.Context, prefix, step_name: str, length: int) -> StepGenerator:
        """A plain completion of exactly `length` greedy tokens (no length
        oracle, no draft): the request the `/v1/completions` front serves
        (server.py).  Deferred like `begin_step`: requests prepared together
        decode as one batch when the first is read."""
        spec = _rt.StepSpec(step_name, _rt.LOW, max(1, int(length)))
        with self._foreground():
            h = self._new_request(context, prefix, spec, int(length), False, PRIO_REASONING)
            self._pending.append(h)
            self._ensure_slots(len(self._pending) + len(self._owners))
        return DeviceStepGenerator(h, self)

    def _covered(self, vseed: int, ids: np.ndarray) -> int:
        """Longest prefix of `ids` whose KV exists (a cached trunk) or will
        exist once the pending requests are materialised."""
        best = 0
        cands = [t.ids for t in self._trunks if t.vseed == vseed]
        cands += [h.ids for h in self._pending if h.branch < 0 and h.vseed == vseed]
        for other in cands:
            m = min(ids.size, other.size)
            neq = np.flatnonzero(other[:m] != ids[:m])
            best = max(best, int(neq[0]) if neq.size else m)
        return best

    def _reserve_pages(self, h: DeviceRequest) -> None:
        """Hold the KV pages the request can need (trunk extension beyond what
        is cached or pending, the copy-on-write page, its decode pages) so
        that materialising and decoding it cannot exhaust the pool; LRU trunks
        are evicted to make room.  EngineError (a BackendError) otherwise."""
        new_trunk = h.ids.size - self._covered(h.vseed, h.ids)
        need = -(-max(0, new_trunk) // PAGE_TOKENS) + 1 + -(-(h.length + 1) // PAGE_TOKENS) + 1
        while True:
            st = self.engine.stats()
            free = st["pages_total"] - st["pages_used"] - self._reserved
            if free >= need or not self._trunks:
                break
            victim = min(self._trunks, key=lambda t: t.stamp)
            self._trunks.remove(victim)
            self.engine.seq_free(victim.seq)
        if free < need:
            raise EngineError(f"KV pool exhausted: step {h.name!r} needs {need} pages, {free} free")
        h.reserve = need
        self._reserved += need

    def _materialize(self, extra=()) -> None:
        """Fork every pending request (and `extra`) off its trunk.  Trunks are
        planned longest input first, so nested branch prefixes share one
        prefill; every new trunk of the group (e.g. one per episode of a
        batched-episode timestep) is then prefilled by ONE batched engine call
        whose forwards pack the rows of all of them."""
        todo = [h for h in [*self._pending, *extra] if h.branch < 0 and h.error is None and h.ids is not None]
        if not todo:
            return
        todo.sort(key=lambda h: -h.ids.size)
        eng = self.engine
        planned: list[tuple[_Trunk, int, DeviceRequest]] = []   # new trunk, prefilled from lcp, its owner
        for h in todo:
            if self._covering(h.vseed, h.ids, [t for t, _, _ in planned]) is not None:
                continue
            best, lcp = self._best_trunk(h.vseed, h.ids)
            try:
                seq = eng.seq_fork(best.seq, lcp) if best is not None and lcp > 0 else eng.seq_create()
            except EngineError as exc:
                h.error = exc
                self._release(h)
                continue
            self._clock += 1
            planned.append((_Trunk(h.vseed, h.ids.copy(), seq, self._clock), lcp, h))
        first: dict[int, int] = {}   # id(owner) -> its first token, computed by the trunk prefill
        if planned:
            want = [self.tag_in_prefill and not h.draft and not h.prefix and h.length >= 2 for _, _, h in planned]
            ids_list = [np.concatenate([t.ids[lcp:], np.asarray([h.tag] if w else [], np.int32)])
                        for (t, lcp, h), w in zip(planned, want)]
            try:
                toks = eng.prefill_batch([t.seq for t, _, _ in planned], ids_list,
                                         [t.vseed for t, _, _ in planned], VIS_ID, want=want if any(want) else None)
            except EngineError as exc:
                for t, _, _ in planned:
                    eng.seq_free(t.seq)
                for h in todo:
                    if h.error is None and self._covering(h.vseed, h.ids, []) is None:
                        h.error = exc
                        self._release(h)
                planned, toks = [], None
            if toks is not None:
                for (t, _, h), w, tok in zip(planned, want, toks):
                    if w:
                        first[id(h)] = int(tok)
            self._trunks.extend(t for t, _, _ in planned)
        for h in todo:
            if h.error is not None:
                continue
            tr = self._covering(h.vseed, h.ids, [])
            try:
                if tr is None:
                    raise EngineError(f"no trunk covers request {h.name!r}")
                tr.stamp = self._clock
                if id(h) in first:   # its TAG row is in the trunk: fork past it, decode from token 1
                    h.branch = eng.seq_fork(tr.seq, h.ids.size + 1)
                    h.prefix = (first[id(h)],)
                else:
                    h.branch = eng.seq_fork(tr.seq, h.ids.size)
            except EngineError as exc:
                h.error = exc
                self._release(h)
        while len(self._trunks) > self._trunk_cap:
            victim = min(self._trunks, key=lambda t: t.stamp)
            self._trunks.remove(victim)
            eng.seq_free(victim.seq)

    def _best_trunk(self, vseed: int, ids: np.ndarray):
        """Cached trunk with the longest common prefix with ids (ties: the shorter trunk)."""
        best, best_lcp = None, 0
        for tr in self._trunks:
            if tr.vseed != vseed:
                continue
            m = min(ids.size, tr.ids.size)
            neq = np.flatnonzero(tr.ids[:m] != ids[:m])
            lcp = int(neq[0]) if neq.size else m
            if lcp > best_lcp or (lcp == best_lcp and best is not None and tr.ids.size < best.ids.size):
                best, best_lcp = tr, lcp
        return best, best_lcp

    def _covering(self, vseed: int, ids: np.ndarray, extra) -> Optional[_Trunk]:
        """A cached (or `extra`) trunk whose ids start with all of ids."""
        for tr in [*self._trunks, *extra]:
            if tr.vseed == vseed and tr.ids.size >= ids.size and np.array_equal(tr.ids[: ids.size], ids):
                return tr
        return None

    def _submit(self, h: DeviceRequest, lane: int) -> None:
        """Hand a materialised request to the device batcher; a rejection is
        kept on the handle (raised when its tokens are read) and frees it."""
        if h.error is None and h.branch < 0:
            self._materialize(extra=(h,))
        if h.error is not None:
            return
        try:
            h.lane = lane
            first = h.prefix[-1] if h.prefix else h.tag
            h.req = self.engine.submit_lane(lane, h.branch, first, h.length - len(h.prefix), h.priority)
        except EngineError as exc:
            h.error = exc
            self._release(h)
            return
        if lane == 0:
            self._owners[h.req] = h
        self.requests += 1

    def _release(self, h: DeviceRequest) -> None:
        """Free a request's fork and its page reservation (failed or done)."""
        if h.branch >= 0:
            self.engine.seq_free(h.branch)
            h.branch = -1
        if h.reserve:
            self._reserved -= h.reserve
            h.reserve = 0
        if h.ids is not None:
            h.ids = None
            self._live -= 1

    def discard(self, h: DeviceRequest) -> None:
        """Abandon a prepared, never-submitted request."""
        with self._foreground():
            if h in self._pending:
                self._pending.remove(h)
            if h.req < 0:
                self._release(h)

    def _run(self, stop_req: int, max_ticks: int = 0) -> list[int]:
        """Lane-0 decode until `stop_req` completes (-1: idle) or `max_ticks`.
        Per completed request: read its tokens, notify its owner (`on_complete`:
        bookkeeping only, no user callbacks), then release the device id -- in
        that order, because a released id can be reused by the very next
        submit (e.g. from a landing callback)."""
        occupancy, done = self.engine.run(stop_req, lane=0, max_ticks=max_ticks)
        eng = self.engine
        for req, _tick in done:
            h = self._owners.pop(req, None)
            if h is None:
                raise EngineError(f"request {req} completed without an owner")
            h.tokens = h.prefix + tuple(eng.request_tokens(h.req, h.length - len(h.prefix)))
            if self.request_log is not None and h.log is not None:
                self.request_log.append(h.log + (h.tokens,))
            if h.on_complete is not None:
                h.on_complete(h)
            eng.request_release(h.req)
            self._release(h)
        return occupancy

    def close(self) -> None:
        """Stop this backend's async engines; close the device engine if this
        backend created it.  A shared engine (passed in) stays open for its
        other users; requests this backend still has in flight on it must be
        drained by the caller first (`make_async_engine(...).drain()`), since
        the engine completes requests in batches across backends."""
        for eng in list(self._async_engines):
            eng.close()
        if self._owns_engine:
            self.engine.close()


def _device_priority(priority: str) -> int:
    return PRIO_ACTION if priority == _rbatch.ACTION else PRIO_REASONING


class AsyncDeviceEngine:
    """Lockstep Fast-ECoT async engine: the reference `_MicroEngine` surface
    (`schedulers.py:244-299`) over the device batcher.  Admission is the
    reference's (action first, then FIFO; a slot freed at tick k is reused at
    k+1 -- csrc/engine.cu `tick()`), each `tick` is one decode iteration of
    every admitted row, and completions fire the requests' `on_complete`
    after the tick, as the reference does."""

    def __init__(self, backend: EngineBackend, slots: int):
        self.backend = backend
        backend.engine.set_slots(slots)
        backend._slots = slots
        backend._fixed_slots = True
        self._inflight: dict[int, object] = {}   # device request id -> reference _EngineRequest
        self._now = 0
        backend._async_engines.append(self)

    def _take(self, req) -> DeviceRequest:
        h = device_handle(req.tokens)
        if h is None:
            raise EngineError(f"request {req.name!r} was not issued by this engine's backend")
        be = self.backend
        be._materialize()            # every request issued so far: one trunk prefill, longest first
        if h in be._pending:
            be._pending.remove(h)
        h.priority = _device_priority(req.priority)
        return h

    def submit(self, req) -> None:
        be = self.backend
        with be._lock:
            h = self._take(req)
            be._submit(h, 0)
            if h.error is not None:
                raise EngineError(f"request {req.name!r} rejected: {h.error}") from h.error
            self._inflight[h.req] = req
            h.on_complete = self._landed

    def _landed(self, h: DeviceRequest) -> None:
        self._completed.append(self._inflight.pop(h.req))

    def in_flight_names(self) -> set[str]:
        return {r.name for r in self._inflight.values()}

    def idle(self) -> bool:
        return not self._inflight

    def tick(self, timestep: int) -> tuple[int, list]:
        self._now = timestep
        be = self.backend
        with be._lock:
            if be._pending:
                be.flush()
            self._completed = []
            occ = be._run(-1, max_ticks=1)
            completed, self._completed = self._completed, []
        for req in completed:
            req.remaining = 0
            if req.on_complete is not None:
                req.on_complete(req, timestep)
        return (occ[0] if occ else 0), completed

    def drain(self) -> None:
        """Decode every request still in flight (they land at the last control
        timestep) so the engine is idle before it is handed to another runner."""
        while self._inflight:
            self.tick(self._now)

    def wait_for(self, h: DeviceRequest) -> None:  # lane 0 requests resolve through the backend
        self.backend._resolve(h)

    def close(self) -> None:
        if self in self.backend._async_engines:
            self.backend._async_engines.remove(self)


class BackgroundAsyncEngine:
    """Fast ECoT async with the reasoning refresh running in the background
    (north_star item 4; reference `ParallelAsyncRunner`, Alg. 1).

    A host thread ticks the device batcher whenever anything is in flight, so
    reasoning requests keep decoding between and during control steps.  The
    action of a control step is a high-priority request on the same batcher:
    it is admitted ahead of queued reasoning (the reference's admission,
    `schedulers.py:263-273`) and decodes in the same ticks as the in-flight
    reasoning rows.  A decode tick streams every weight once whatever its row
    count, so merging costs the action nothing, whereas a second stream with
    its own ticks would stream the weights twice (measured in round 1: the
    two-lane variant's action p50 was 11 % above lockstep).
    Requests land through the reference runner's own `on_complete`
    (`cache.write`, `schedulers.py:485-486`) at the control timestep current
    when they complete; landing order is real-time, so parity is checked per
    request (identical (context, prefix, step) -> identical tokens)."""

    def __init__(self, backend: EngineBackend, slots: int):
        self.backend = backend
        backend.engine.set_slots(slots)
        backend._slots = slots
        backend._fixed_slots = True
        self._cv = threading.Condition()
        self._inflight: dict[int, tuple[DeviceRequest, object]] = {}   # device id -> (handle, request)
        self._landing: set[str] = set()   # completed, on_complete still running
        self._landed: list = []
        self._ticks = 0
        self._last_occ = 0
        self._now = 0
        self._errors: list[BaseException] = []
        self._stop = False
        self._held = False               # a control step is issuing its requests
        # the ticker enqueues one tick per call and would run arbitrarily far
        # ahead of the GPU; pacing keeps <= 2 ticks queued, so an action waits
        # behind at most those
        self._set_pace(backend.background_depth)
        self._thread = threading.Thread(target=self._loop, name="fastecot-background-ticker", daemon=True)
        self._thread.start()
        backend._async_engines.append(self)

    # -- control-step bracket (EngineParallelAsyncRunner.step) -------------------
    def hold(self) -> None:
        """Pause the ticker while a control step issues its requests (trunk
        prefill, forks, submissions), so the action joins the very next tick
        instead of queueing behind ticks slipped in between those calls."""
        with self._cv:
            self._held = True

    def release(self) -> None:
        with self._cv:
            self._held = False
            self._cv.notify_all()

    # -- runner surface (the reference _MicroEngine's) -------------------------
    def submit(self, req) -> None:
        be = self.backend
        h = device_handle(req.tokens)
        if h is None:
            raise EngineError(f"request {req.name!r} was not issued by this engine's backend")
        if req.priority == _rbatch.ACTION:
            self.release()           # the action is the control step's last submission
        with be._foreground():
            be._materialize()        # every request issued so far: one trunk prefill, longest first
            if h in be._pending:
                be._pending.remove(h)
            h.priority = _device_priority(req.priority)
            be._submit(h, 0)
            if h.error is None:
                h.on_complete = self._on_device_complete
                with self._cv:
                    self._inflight[h.req] = (h, req)
                    self._cv.notify_all()
        if h.error is not None:
            raise EngineError(f"request {req.name!r} rejected: {h.error}") from h.error

    def _on_device_complete(self, h: DeviceRequest) -> None:   # under the backend lock
        with self._cv:
            _, req = self._inflight.pop(h.req)
            self._landing.add(req.name)
            self._landed.append(req)

    def in_flight_names(self) -> set[str]:
        with self._cv:
            names = {r.name for _, r in self._inflight.values()}
            names.update(self._landing)
        return names

    def idle(self) -> bool:
        with self._cv:
            return not self._inflight and not self._landing

    def tick(self, timestep: int) -> tuple[int, list]:
        """Wait for the background ticker's next decode iteration (returns its
        occupancy); completions have already landed through their callbacks."""
        self._raise_background_error()
        self._now = timestep
        with self._cv:
            start = self._ticks
            while self._ticks == start and (self._inflight or self._landing) and not self._errors:
                self._cv.wait(1.0)
            occ = self._last_occ if self._ticks != start else 0
        self._raise_background_error()
        return occ, []

    def set_timestep(self, timestep: int) -> None:
        self._now = timestep

    # -- background ticker ---------------------------------------------------------
    def _loop(self) -> None:
        be = self.backend
        while True:
            with self._cv:
                while (not self._inflight or self._held) and not self._stop:
                    self._cv.wait(0.05)
                if self._stop:
                    return
            try:
                with be._background_turn():   # one tick; waiting runner operations go first
                    occ = be._run(-1, max_ticks=1)
                with self._cv:
                    landed, self._landed = self._landed, []
                for req in landed:
                    try:
                        req.remaining = 0
                        if req.on_complete is not None:
                            req.on_complete(req, self._now)
                    finally:
                        with self._cv:
                            self._landing.discard(req.name)
                with self._cv:
                    self._ticks += 1
                    self._last_occ = occ[0] if occ else 0
                    self._cv.notify_all()
            except BaseException as exc:  # surfaced on the runner thread
                with self._cv:
                    self._errors.append(exc)
                    self._stop = True
                    self._cv.notify_all()
                return

    def wait_for(self, h: DeviceRequest) -> None:
        self.backend._resolve(h)

    def _raise_background_error(self) -> None:
        if self._errors:
            raise EngineError(f"background decode ticker failed: {self._errors[0]!r}")

    def drain(self, timeout: float = 120.0) -> None:
        """Wait until every in-flight request has landed."""
        end = time.monotonic() + timeout
        with self._cv:
            while (self._inflight or self._landing) and not self._errors and time.monotonic() < end:
                self._cv.wait(0.05)
        self._raise_background_error()

    def _set_pace(self, on: int) -> None:
        setter = getattr(self.backend.engine, "set_option", None)
        if setter is not None:   # (the CPU stand-in engine has no options)
            setter("lane0_pace", on)

    def close(self) -> None:
        with self._cv:
            self._stop = True
            self._cv.notify_all()
        self._thread.join(timeout=10.0)
        self._set_pace(0)
        if self in self.backend._async_engines:
            self.backend._async_engines.remove(self)
