"""Host logic of the two-stream async engine (`TwoStreamAsyncEngine`) on CPU,
driven by a fake device engine: request ids are recycled by the engine as soon
as they are released, exactly as `fe_request_release` does, so a submit on the
runner thread can reuse the id of a request the background lane is still
landing (the race the round-1 GPU suite hit)."""

import threading

from paper_2506_07639_b200.engine_backend import EngineRequest, TwoStreamAsyncEngine


class FakeEngine:
    """Lane 1 completes every queued request on the next run() call; ids come
    from a free list (lowest first), like the engine's request table."""

    def __init__(self):
        self.lock = threading.Lock()
        self.free = list(range(4))
        self.queued: list[int] = []
        self.length: dict[int, int] = {}
        self.on_release = None  # hook: runs inside request_release (after the id is free)

    def set_slots(self, n):
        pass

    def set_slots_lane(self, lane, n):
        pass

    def submit_lane(self, lane, seq, tag, length, prio):
        with self.lock:
            r = self.free.pop(0)
            self.queued.append(r)
            self.length[r] = length
        return r

    def run(self, stop_req, lane=0, max_ticks=0):
        with self.lock:
            done, self.queued = self.queued, []
        return [], [(r, 0) for r in done]

    def request_tokens(self, r, n):
        return [r] * n

    def request_release(self, r):
        with self.lock:
            self.free.insert(0, r)
        if self.on_release is not None:
            hook, self.on_release = self.on_release, None
            hook()

    def seq_free(self, seq):
        pass


class FakeBackend:
    def __init__(self):
        self.engine = FakeEngine()
        self._async_engines = []
        self._slots = 0
        self.logged: list[EngineRequest] = []

    def _log(self, h):
        self.logged.append(h)


def _req(name, length=3):
    return EngineRequest(name=name, step=None, length=length, truncated=False, tag=0, branch=0, priority=1, lane=1)


def test_released_id_reused_while_landing():
    be = FakeBackend()
    eng = TwoStreamAsyncEngine(be, slots=4)
    landed = []
    try:
        first, second = _req("plan"), _req("subtask")
        # while the background lane lands `first`, the runner submits `second`,
        # which gets the id `first` just released
        be.engine.on_release = lambda: eng.submit(second, lambda h, t: landed.append(h.name))
        eng.submit(first, lambda h, t: landed.append(h.name))
        eng.drain(timeout=10.0)
        assert sorted(landed) == ["plan", "subtask"]
        assert first.req == second.req  # the id really was reused
        assert first.tokens == (first.req,) * 3 and second.done
        assert eng.idle()
    finally:
        eng.close()
