"""A CPU stand-in for the device engine (`paper_2506_07639_b200.engine.Engine`)
-- test infrastructure for the host logic only.

It keeps the engine's observable contract (csrc/engine.cu): sequences with
copy-on-write forks and prefill, per-lane continuous batchers whose admission
is the reference `_MicroEngine`'s (action first, then FIFO by submission
order; a slot freed at tick k admits at k+1 -- `schedulers.py:263-287`),
request ids recycled from a free list on release, and per-request outputs
that depend only on the request's input ids (sequence content + first id), as
greedy decode does.  The outputs are a hash, not a model: `hash_tokens` is
shared with `HashBackend`, a synchronous `GenerationBackend` computing the
same tokens for the same framed request, so traces produced through the
engine's deferred/batched path can be compared byte for byte with traces
produced one request at a time.
"""

from __future__ import annotations

import hashlib
import threading
import time

import numpy as np

from paper_2506_07639_b200 import backends as B
from paper_2506_07639_b200 import model as M
from paper_2506_07639_b200.engine import PRIO_ACTION


def hash_tokens(vseed: int, ids, first_id: int, n: int) -> tuple:
    h = hashlib.blake2b(digest_size=8)
    h.update(int(vseed).to_bytes(8, "little"))
    h.update(np.asarray(ids, dtype=np.int32).tobytes())
    h.update(int(first_id).to_bytes(4, "little"))
    rng = np.random.default_rng(int.from_bytes(h.digest(), "little"))
    return tuple(int(t) for t in rng.integers(0, M.TEXT_VOCAB, size=n))


def ar_token(vseed: int, ids) -> int:
    """Autoregressive stand-in for one greedy step: the next token is a hash
    of everything the sequence holds (vision seed + every input so far)."""
    h = hashlib.blake2b(digest_size=8)
    h.update(int(vseed).to_bytes(8, "little"))
    h.update(np.asarray(ids, dtype=np.int32).tobytes())
    return int.from_bytes(h.digest(), "little") % M.TEXT_VOCAB


def ar_tokens(vseed: int, ids, first_id: int, n: int) -> tuple:
    seq = [int(i) for i in ids] + [int(first_id)]
    out = []
    for _ in range(n):
        t = ar_token(vseed, seq)
        out.append(t)
        seq.append(t)
    return tuple(out)


class _Lane:
    def __init__(self):
        self.slots: list = [None] * 8
        self.waiting: list[int] = []


class FakeEngine:
    def __init__(self, cfg="tiny", max_slots: int = 512, autoregressive: bool = False):
        self.cfg = M.get_config(cfg)
        self.autoregressive = autoregressive   # outputs from ar_tokens (draft verification tests)
        self.verify_calls = 0
        self.max_slots = max_slots
        self.lock = threading.RLock()
        self.seqs: dict[int, tuple[int, list]] = {}     # seq -> (vseed, ids)
        self._next_seq = 0
        self.lanes = [_Lane(), _Lane()]
        self.reqs: dict[int, dict] = {}
        self.free_ids = list(range(4 * max_slots))
        self._seqno = 0
        self.occupancy_log: list[tuple[int, int]] = []  # (lane, occupied) per tick
        self.prefilled_tokens = 0
        self.prefill_calls = 0
        self.on_release = None                          # hook run inside request_release
        self.pages_total = 1 << 20
        self.tick_delay = 0.0

    # sequences
    def seq_create(self) -> int:
        with self.lock:
            s = self._next_seq
            self._next_seq += 1
            self.seqs[s] = (0, [])
            return s

    def seq_fork(self, parent: int, length: int) -> int:
        with self.lock:
            vseed, ids = self.seqs[parent]
            if length > len(ids):
                raise B.EngineError("fork beyond parent length")
            s = self.seq_create()
            self.seqs[s] = (vseed, list(ids[:length]))
            return s

    def seq_free(self, seq: int) -> None:
        with self.lock:
            del self.seqs[seq]

    def prefill(self, seq: int, ids, vision_seed: int, vis_id: int) -> None:
        with self.lock:
            _, cur = self.seqs[seq]
            self.seqs[seq] = (vision_seed, cur + [int(i) for i in ids])
            self.prefilled_tokens += len(ids)
            self.prefill_calls += 1

    def verify(self, seqs, inputs) -> list:
        """fe_verify: extend each sequence by its inputs; the token after each."""
        if not self.autoregressive:
            raise B.EngineError("verify needs the autoregressive fake engine")
        with self.lock:
            self.verify_calls += 1
            outs = []
            for s, xs in zip(seqs, inputs):
                vseed, ids = self.seqs[s]
                g = []
                for x in xs:
                    ids.append(int(x))
                    g.append(ar_token(vseed, ids))
                outs.append(np.asarray(g, dtype=np.int32))
            return outs

    def seq_truncate(self, seq: int, n: int) -> None:
        with self.lock:
            vseed, ids = self.seqs[seq]
            if n > len(ids):
                raise B.EngineError("truncate beyond the sequence")
            self.seqs[seq] = (vseed, ids[:n])

    def prefill_batch(self, seqs, ids_list, vision_seeds, vis_id: int, want=None):
        with self.lock:
            self.prefill_batch_calls = getattr(self, "prefill_batch_calls", 0) + 1
        out = []
        for i, (s, ids, v) in enumerate(zip(seqs, ids_list, vision_seeds)):
            if len(ids):
                self.prefill(s, ids, v, vis_id)
            if want is not None:   # greedy token after the last id (autoregressive mode only)
                if want[i] and not self.autoregressive:
                    raise B.EngineError("prefill heads need the autoregressive fake engine")
                out.append(ar_token(self.seqs[s][0], self.seqs[s][1]) if want[i] else -1)
        return out if want is not None else None

    @property
    def supports_prefill_heads(self) -> bool:
        return self.autoregressive

    # batcher
    def set_slots(self, n: int) -> None:
        self.set_slots_lane(0, n)

    def set_slots_lane(self, lane: int, n: int) -> None:
        with self.lock:
            ln = self.lanes[lane]
            if any(ln.slots[n:]):
                raise B.EngineError("shrinking over busy slots")
            ln.slots = (ln.slots + [None] * n)[:n]

    def submit_lane(self, lane, seq, first_id, length, priority) -> int:
        with self.lock:
            if length < 1 or length > 1024:
                raise B.EngineError("request length outside [1, 1024]")
            vseed, ids = self.seqs[seq]
            r = self.free_ids.pop(0)
            self.reqs[r] = dict(lane=lane, remaining=length, state=0, seqno=self._seqno,
                                prio=0 if priority == PRIO_ACTION else 1,
                                out=(ar_tokens if self.autoregressive else hash_tokens)(vseed, ids, first_id,
                                                                                       length))
            self._seqno += 1
            self.lanes[lane].waiting.append(r)
            return r

    def submit(self, seq, first_id, length, priority) -> int:
        return self.submit_lane(0, seq, first_id, length, priority)

    def _tick(self, lane: int):
        ln = self.lanes[lane]
        if ln.waiting:
            ln.waiting.sort(key=lambda r: (self.reqs[r]["prio"], self.reqs[r]["seqno"]))
            for s in range(len(ln.slots)):
                if not ln.waiting:
                    break
                if ln.slots[s] is None:
                    ln.slots[s] = ln.waiting.pop(0)
        occupied, done = 0, []
        for s, r in enumerate(ln.slots):
            if r is None:
                continue
            occupied += 1
            q = self.reqs[r]
            q["remaining"] -= 1
            if q["remaining"] == 0:
                q["state"] = 2
                done.append(r)
                ln.slots[s] = None
        self.occupancy_log.append((lane, occupied))
        return occupied, done

    def run(self, stop_req: int = -1, lane: int = 0, max_ticks: int = 0):
        occ, done = [], []
        while True:
            with self.lock:
                ln = self.lanes[lane]
                if stop_req >= 0 and self.reqs[stop_req]["state"] == 2:
                    break
                if not ln.waiting and not any(x is not None for x in ln.slots):
                    if stop_req >= 0:
                        raise B.EngineError("stop request is not in flight on this lane")
                    break
                if max_ticks and len(occ) >= max_ticks:
                    break
                o, d = self._tick(lane)
            if self.tick_delay:
                time.sleep(self.tick_delay)   # a device tick takes time (background-ticker tests)
            occ.append(o)
            done.extend((r, len(occ) - 1) for r in d)
        return occ, done

    def request_tokens(self, r: int, n: int) -> list:
        with self.lock:
            q = self.reqs[r]
            if q["state"] != 2:
                raise B.EngineError("request not complete")
            return list(q["out"][:n])

    def request_release(self, r: int) -> None:
        with self.lock:
            del self.reqs[r]
            self.free_ids.insert(0, r)
        if self.on_release is not None:
            hook, self.on_release = self.on_release, None
            hook()

    def stats(self) -> dict:
        with self.lock:
            used = sum(-(-len(ids) // M.PAGE_TOKENS) for _, ids in self.seqs.values())
        return {"pages_total": self.pages_total, "pages_used": used}

    def close(self) -> None:
        pass


class HashBackend:
    """Synchronous `GenerationBackend` with FakeEngine's outputs: the same
    framing and length oracle as `EngineBackend`, one request at a time."""

    deterministic = True
    supports_prefix_conditioning = True

    def __init__(self, cfg="tiny", profile=None):
        self.cfg = M.get_config(cfg)
        self.profile = profile or B.default_profile(0)

    def encode(self, instruction, observation):
        return B.encode_context(instruction, observation)

    def begin_step(self, context, prefix, step, prev_content):
        plan = B.length_plan(self.profile, context, step, prev_content)
        ids = M.context_ids(context, self.cfg) + M.text_ids(prefix)
        toks = hash_tokens(M.vision_seed(context.observation), ids, M.step_tag(step), plan.length)
        return B.StepGenerator(toks, truncated=plan.truncated)


def fake_backend(profile=None, autoregressive=False, **kw):
    from paper_2506_07639_b200.engine_backend import EngineBackend
    eng = FakeEngine(autoregressive=autoregressive)
    return EngineBackend("tiny", engine=eng, profile=profile, **kw), eng
