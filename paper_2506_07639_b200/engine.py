"""ctypes binding of the B200 engine's C ABI (include/fastecot.h).

The shared library is built in-tree (`_build/libfastecot.so`, see build.py).
There is deliberately no fallback: if the library or a GPU is missing the
constructor raises, so a test or benchmark can never silently run on a CPU
path.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .backends import EngineError
from .model import ModelConfig, ROPE_MAX_POS, TEXT_VOCAB, get_config, rope_table

# FASTECOT_LIB: another build of the library (A/B timing of two builds on one box)
LIB_PATH = Path(os.environ.get("FASTECOT_LIB", Path(__file__).resolve().parent / "_build" / "libfastecot.so"))

F32, BF16 = 0, 1
PRIO_ACTION, PRIO_REASONING = 0, 1

_c_int_p = ctypes.POINTER(ctypes.c_int32)


class FeVisionConfig(ctypes.Structure):
    _fields_ = [("img", ctypes.c_int32), ("patch", ctypes.c_int32), ("d", ctypes.c_int32), ("layers", ctypes.c_int32),
                ("heads", ctypes.c_int32), ("mlp", ctypes.c_int32), ("proj_hidden", ctypes.c_int32),
                ("eps", ctypes.c_float)]


class FeConfig(ctypes.Structure):
    _fields_ = [
        ("d_model", ctypes.c_int32), ("n_layers", ctypes.c_int32), ("n_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32), ("d_ffn", ctypes.c_int32), ("vocab", ctypes.c_int32),
        ("n_text", ctypes.c_int32), ("max_pos", ctypes.c_int32), ("rms_eps", ctypes.c_float),
        ("attn_scale", ctypes.c_float), ("dtype", ctypes.c_int32), ("max_rows", ctypes.c_int32),
        ("kv_pages", ctypes.c_int32), ("max_slots", ctypes.c_int32),
    ]


EXPORTS = (
    "fe_engine_create", "fe_engine_destroy", "fe_weights_init_random", "fe_last_error",
    "fe_seq_create", "fe_seq_fork", "fe_seq_free", "fe_seq_len", "fe_prefill", "fe_prefill_batch", "fe_prefill_batch_heads", "fe_vision_enable", "fe_vision_encode", "fe_verify", "fe_seq_truncate",
    "fe_set_slots",
    "fe_set_slots_lane", "fe_submit_lane", "fe_run_lane", "fe_stream_lane",
    "fe_submit", "fe_run", "fe_request_tokens", "fe_request_release", "fe_request_capture_logits",
    "fe_request_logits", "fe_in_flight", "fe_synchronize", "fe_stream", "fe_stats", "fe_profile",
    "fe_profile_read",
    "fe_weight_ptr", "fe_memcpy", "fe_op_gemv", "fe_op_rmsnorm", "fe_op_gemm_tc", "fe_op_skinny_tc",
    "fe_set_option", "fe_debug_trace",
)

_lib = None


def load_library(path: Path = LIB_PATH) -> ctypes.CDLL:
    """Load libfastecot.so and declare every exported signature."""
    global _lib
    if _lib is not None:
        return _lib
    if not path.exists():
        raise EngineError(f"engine library missing: {path} (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(path))
    vp, i32, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64
    sig = {
        "fe_engine_create": [ctypes.POINTER(FeConfig), i32, vp, ctypes.POINTER(vp)],
        "fe_engine_destroy": [vp],
        "fe_weights_init_random": [vp, u64],
        "fe_seq_create": [vp, _c_int_p],
        "fe_seq_fork": [vp, i32, i32, _c_int_p],
        "fe_seq_free": [vp, i32],
        "fe_seq_len": [vp, i32, _c_int_p],
        "fe_prefill": [vp, i32, vp, i32, u64, i32],
        "fe_verify": [vp, i32, vp, vp, vp, vp],
        "fe_prefill_batch": [vp, i32, vp, vp, vp, vp, i32],
        "fe_prefill_batch_heads": [vp, i32, vp, vp, vp, vp, i32, vp, vp],
        "fe_vision_enable": [vp, vp, u64, i32],
        "fe_vision_encode": [vp, u64, vp],
        "fe_seq_truncate": [vp, i32, i32],
        "fe_set_slots": [vp, i32],
        "fe_set_slots_lane": [vp, i32, i32],
        "fe_submit_lane": [vp, i32, i32, i32, i32, i32, _c_int_p],
        "fe_run_lane": [vp, i32, i32, i32, i32, _c_int_p, vp, vp, vp, _c_int_p],
        "fe_stream_lane": [vp, i32, ctypes.POINTER(vp)],
        "fe_submit": [vp, i32, i32, i32, i32, _c_int_p],
        "fe_run": [vp, i32, i32, _c_int_p, vp, vp, vp, _c_int_p],
        "fe_request_tokens": [vp, i32, vp, i32],
        "fe_request_release": [vp, i32],
        "fe_request_capture_logits": [vp, i32],
        "fe_request_logits": [vp, i32, vp, i32],
        "fe_in_flight": [vp, _c_int_p],
        "fe_synchronize": [vp],
        "fe_stream": [vp, ctypes.POINTER(vp)],
        "fe_stats": [vp, vp, i32],
        "fe_profile": [vp, i32],
        "fe_profile_read": [vp, vp, i32],
        "fe_weight_ptr": [vp, i32, i32, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_size_t)],
        "fe_memcpy": [vp, vp, vp, ctypes.c_size_t],
        "fe_op_gemv": [vp, vp, i32, i32, vp, i32, vp],
        "fe_op_rmsnorm": [vp, vp, vp, vp, i32, i32],
        "fe_op_gemm_tc": [vp, vp, vp, i32, i32, i32, vp],
        "fe_op_skinny_tc": [vp, vp, vp, i32, i32, i32, vp],
        "fe_set_option": [vp, ctypes.c_char_p, ctypes.c_int64],
        "fe_debug_trace": [vp, vp, i32, _c_int_p, _c_int_p],
    }
    for name, argtypes in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = ctypes.c_int
    lib.fe_last_error.restype = ctypes.c_char_p
    lib.fe_last_error.argtypes = []
    _lib = lib
    return lib


def _np_ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


class Engine:
    """One engine per GPU: weights, paged KV pool, continuous batcher."""

    def __init__(self, config: str | ModelConfig = "tiny", dtype: str = "f32", device: int = 0,
                 seed: int = 0, max_rows: int = 1024, kv_pages: int = 0, max_slots: int = 512,
                 vision=None):
        """`vision`: None (synthetic VIS embeddings), True (the LLM's default
        tower, model.DEFAULT_VISION) or a tower preset / VisionConfig."""
        self.cfg = get_config(config)
        self.vision = None
        self.lib = load_library()
        self.dtype = dtype
        self.max_slots = max_slots
        c = self.cfg
        fc = FeConfig(c.d_model, c.n_layers, c.n_heads, c.head_dim, c.d_ffn, c.vocab, TEXT_VOCAB,
                      ROPE_MAX_POS, c.rms_eps, float(np.float32(1.0) / np.sqrt(np.float32(c.head_dim))),
                      F32 if dtype == "f32" else BF16, max_rows, kv_pages, max_slots)
        self._rope = rope_table(c)
        h = ctypes.c_void_p()
        self._h = None
        self._check(self.lib.fe_engine_create(ctypes.byref(fc), device, _np_ptr(self._rope), ctypes.byref(h)))
        self._h = h
        self.seed = seed
        self._check(self.lib.fe_weights_init_random(self._h, seed))
        self._cap = 8192
        self._occ = np.zeros(self._cap, dtype=np.int32)
        self._done = np.zeros(self._cap, dtype=np.int32)
        self._done_tick = np.zeros(self._cap, dtype=np.int32)
        if vision:
            self.enable_vision(vision)

    # -- plumbing ----------------------------------------------------------
    def _check(self, rc: int) -> None:
        if rc != 0:
            raise EngineError(self.lib.fe_last_error().decode(errors="replace"))

    def close(self) -> None:
        if self._h is not None:
            self.lib.fe_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- sequences ---------------------------------------------------------
    def seq_create(self) -> int:
        s = ctypes.c_int32()
        self._check(self.lib.fe_seq_create(self._h, ctypes.byref(s)))
        return s.value

    def seq_fork(self, parent: int, length: int) -> int:
        s = ctypes.c_int32()
        self._check(self.lib.fe_seq_fork(self._h, parent, length, ctypes.byref(s)))
        return s.value

    def seq_free(self, seq: int) -> None:
        self._check(self.lib.fe_seq_free(self._h, seq))

    def seq_len(self, seq: int) -> int:
        n = ctypes.c_int32()
        self._check(self.lib.fe_seq_len(self._h, seq, ctypes.byref(n)))
        return n.value

    def prefill(self, seq: int, ids, vision_seed: int, vis_id: int) -> None:
        a = np.ascontiguousarray(np.asarray(ids, dtype=np.int32))
        if a.size:
            self._check(self.lib.fe_prefill(self._h, seq, _np_ptr(a), int(a.size),
                                            ctypes.c_uint64(vision_seed & 0xFFFFFFFFFFFFFFFF), vis_id))

    def enable_vision(self, vision=True, seed: int | None = None, slots: int = 64) -> None:
        """VIS rows from the vision tower + projector (csrc/vision.cu) instead of
        the synthetic embeddings; `vision`: preset name, VisionConfig or True."""
        from .model import get_vision
        v = get_vision(vision, self.cfg)
        vc = FeVisionConfig(v.img, v.patch, v.d, v.layers, v.heads, v.mlp, v.proj_hidden, v.eps)
        self._check(self.lib.fe_vision_enable(self._h, ctypes.byref(vc),
                                              ctypes.c_uint64(self.seed if seed is None else seed), slots))
        self.vision = v

    def vision_encode(self, vision_seed: int) -> np.ndarray:
        out = np.empty((self.vision.patches, self.cfg.d_model), dtype=np.float32)
        self._check(self.lib.fe_vision_encode(self._h, ctypes.c_uint64(vision_seed & 0xFFFFFFFFFFFFFFFF),
                                              _np_ptr(out)))
        return out

    def prefill_batch(self, seqs, ids_list, vision_seeds, vis_id: int, want=None):
        """Prefill several sequences in as few forwards as the engine holds
        (rows of all of them packed; one GEMM pass per forward).  `want`: per
        sequence, run the lm_head on its last row and return the greedy token
        after it (list, -1 where not wanted); else None."""
        counts = np.asarray([len(x) for x in ids_list], dtype=np.int32)
        if counts.sum() == 0 and not want:
            return None
        flat = np.ascontiguousarray(np.concatenate([np.asarray(x, dtype=np.int32) for x in ids_list]
                                                   + [np.zeros(0, np.int32)]))
        sq = np.ascontiguousarray(np.asarray(seqs, dtype=np.int32))
        vs = np.ascontiguousarray(np.asarray([v & 0xFFFFFFFFFFFFFFFF for v in vision_seeds], dtype=np.uint64))
        if want is None:
            self._check(self.lib.fe_prefill_batch(self._h, int(sq.size), _np_ptr(sq), _np_ptr(counts),
                                                  _np_ptr(flat), _np_ptr(vs), vis_id))
            return None
        w = np.ascontiguousarray(np.asarray([1 if x else 0 for x in want], dtype=np.int32))
        out = np.empty(sq.size, dtype=np.int32)
        self._check(self.lib.fe_prefill_batch_heads(self._h, int(sq.size), _np_ptr(sq), _np_ptr(counts),
                                                    _np_ptr(flat), _np_ptr(vs), vis_id, _np_ptr(w), _np_ptr(out)))
        return out.tolist()

    def verify(self, seqs, inputs) -> list[np.ndarray]:
        """Reuse-as-draft verification: extend every `seqs[i]` by `inputs[i]`
        in one batched forward; returns, per sequence, the greedy token after
        each input (the caller truncates what it rejects)."""
        counts = np.asarray([len(x) for x in inputs], dtype=np.int32)
        flat = np.ascontiguousarray(np.concatenate([np.asarray(x, dtype=np.int32) for x in inputs]))
        sq = np.ascontiguousarray(np.asarray(seqs, dtype=np.int32))
        out = np.empty(flat.size, dtype=np.int32)
        self._check(self.lib.fe_verify(self._h, int(sq.size), _np_ptr(sq), _np_ptr(counts), _np_ptr(flat),
                                       _np_ptr(out)))
        return np.split(out, np.cumsum(counts)[:-1])

    def seq_truncate(self, seq: int, length: int) -> None:
        self._check(self.lib.fe_seq_truncate(self._h, seq, length))

    # -- batcher -------------------------------------------------------------
    def set_slots(self, slots: int) -> None:
        self._check(self.lib.fe_set_slots(self._h, slots))

    def submit(self, seq: int, first_id: int, length: int, priority: int) -> int:
        r = ctypes.c_int32()
        self._check(self.lib.fe_submit(self._h, seq, first_id, length, priority, ctypes.byref(r)))
        return r.value

    def run(self, stop_req: int = -1, lane: int = 0, max_ticks: int = 0) -> tuple[list[int], list[tuple[int, int]]]:
        """Decode on a lane until `stop_req` completes (-1: until idle) or
        `max_ticks` ticks (0: unbounded).
        Returns (occupancy per tick, [(request, tick)] in completion order)."""
        nt, nc = ctypes.c_int32(), ctypes.c_int32()
        occ_buf, done_buf, tick_buf = self._run_bufs(lane)
        self._check(self.lib.fe_run_lane(self._h, lane, stop_req, max_ticks, self._cap, ctypes.byref(nt),
                                         _np_ptr(occ_buf), _np_ptr(done_buf), _np_ptr(tick_buf), ctypes.byref(nc)))
        occ = occ_buf[: nt.value].tolist()
        done = list(zip(done_buf[: nc.value].tolist(), tick_buf[: nc.value].tolist()))
        return occ, done

    def _run_bufs(self, lane: int):
        # per-lane output arrays: the two lanes may be driven from two threads
        if lane == 0:
            return self._occ, self._done, self._done_tick
        if not hasattr(self, "_bufs1"):
            self._bufs1 = tuple(np.zeros(self._cap, dtype=np.int32) for _ in range(3))
        return self._bufs1

    def submit_lane(self, lane: int, seq: int, first_id: int, length: int, priority: int) -> int:
        r = ctypes.c_int32()
        self._check(self.lib.fe_submit_lane(self._h, lane, seq, first_id, length, priority, ctypes.byref(r)))
        return r.value

    def set_slots_lane(self, lane: int, slots: int) -> None:
        self._check(self.lib.fe_set_slots_lane(self._h, lane, slots))

    def stream_handle_lane(self, lane: int) -> int:
        p = ctypes.c_void_p()
        self._check(self.lib.fe_stream_lane(self._h, lane, ctypes.byref(p)))
        return p.value or 0

    def request_tokens(self, req: int, length: int) -> list[int]:
        out = np.zeros(max(length, 1), dtype=np.int32)
        self._check(self.lib.fe_request_tokens(self._h, req, _np_ptr(out), out.size))
        return out[:length].tolist()

    def request_release(self, req: int) -> None:
        self._check(self.lib.fe_request_release(self._h, req))

    def capture_logits(self, req: int) -> None:
        self._check(self.lib.fe_request_capture_logits(self._h, req))

    def request_logits(self, req: int, rows: int) -> np.ndarray:
        out = np.zeros((rows, self.cfg.vocab), dtype=np.float32)
        self._check(self.lib.fe_request_logits(self._h, req, _np_ptr(out), rows))
        return out

    def in_flight(self) -> int:
        n = ctypes.c_int32()
        self._check(self.lib.fe_in_flight(self._h, ctypes.byref(n)))
        return n.value

    def synchronize(self) -> None:
        self._check(self.lib.fe_synchronize(self._h))

    def stream_handle(self) -> int:
        p = ctypes.c_void_p()
        self._check(self.lib.fe_stream(self._h, ctypes.byref(p)))
        return p.value or 0

    def stats(self) -> dict:
        out = np.zeros(9, dtype=np.int64)
        self._check(self.lib.fe_stats(self._h, _np_ptr(out), out.size))
        keys = ("ticks", "forwards", "rows", "pages_used", "pages_total", "page_bytes", "h2d_bytes", "d2h_bytes",
                "launches")
        return dict(zip(keys, out.tolist()))

    PROFILE_CATEGORIES = ("decode_gemv", "decode_attention", "decode_forward", "prefill_forward", "decode_tick")

    def profile(self, enable: bool) -> None:
        """Start (and reset) or stop CUDA-event timing of engine launches."""
        self._check(self.lib.fe_profile(self._h, int(enable)))

    def profile_read(self) -> dict:
        out = np.zeros(3 * len(self.PROFILE_CATEGORIES), dtype=np.float64)
        self._check(self.lib.fe_profile_read(self._h, _np_ptr(out), out.size))
        return {c: {"ms": out[3 * i], "launches": int(out[3 * i + 1]), "bytes": out[3 * i + 2]}
                for i, c in enumerate(self.PROFILE_CATEGORIES)}

    # -- kernel-level hooks (device pointers) ----------------------------------
    def weight_ptr(self, tensor: int, layer: int = 0) -> tuple[int, int]:
        p, n = ctypes.c_void_p(), ctypes.c_size_t()
        self._check(self.lib.fe_weight_ptr(self._h, tensor, layer, ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def memcpy(self, dst: int, src: int, nbytes: int) -> None:
        self._check(self.lib.fe_memcpy(self._h, ctypes.c_void_p(dst), ctypes.c_void_p(src), nbytes))

    def weight_host(self, tensor: int, layer: int = 0) -> np.ndarray:
        """Host copy of a weight tensor (fp32 view; bf16 returned as uint16 bits)."""
        ptr, nbytes = self.weight_ptr(tensor, layer)
        is_norm = tensor in (3,) or (tensor >= 16 and (tensor - 16) % 16 in (0, 5))
        dt = np.float32 if (self.dtype == "f32" or is_norm) else np.uint16
        out = np.empty(nbytes // np.dtype(dt).itemsize, dtype=dt)
        self.memcpy(out.ctypes.data, ptr, nbytes)
        return out

    def op_gemv(self, w_ptr: int, N: int, K: int, x_ptr: int, rows: int, y_ptr: int) -> None:
        self._check(self.lib.fe_op_gemv(self._h, ctypes.c_void_p(w_ptr), N, K, ctypes.c_void_p(x_ptr), rows,
                                        ctypes.c_void_p(y_ptr)))

    def op_gemm_tc(self, x_ptr: int, w_ptr: int, M: int, N: int, K: int, y_ptr: int) -> None:
        self._check(self.lib.fe_op_gemm_tc(self._h, ctypes.c_void_p(x_ptr), ctypes.c_void_p(w_ptr), M, N, K,
                                           ctypes.c_void_p(y_ptr)))

    def op_skinny_tc(self, x_ptr: int, w_ptr: int, M: int, N: int, K: int, y_ptr: int) -> None:
        self._check(self.lib.fe_op_skinny_tc(self._h, ctypes.c_void_p(x_ptr), ctypes.c_void_p(w_ptr), M, N, K,
                                             ctypes.c_void_p(y_ptr)))

    def debug_trace(self) -> np.ndarray:
        """Persistent-tick phase timestamps [phases][6][grid] (ns) of the last tick:
        barrier passed, phase done, last weight load issued, first / last
        accumulator ready, segments drained."""
        n = 4 * 1024 * 1024
        out = np.zeros(n, dtype=np.uint64)
        ph, g = ctypes.c_int(), ctypes.c_int()
        self._check(self.lib.fe_debug_trace(self._h, _np_ptr(out), n, ctypes.byref(ph), ctypes.byref(g)))
        return out[: ph.value * 6 * g.value].reshape(ph.value, 6, g.value)

    def set_option(self, key: str, value: int) -> None:
        self._check(self.lib.fe_set_option(self._h, key.encode(), int(value)))

    def op_rmsnorm(self, x_ptr: int, w_ptr: int, out_ptr: int, rows: int, d: int) -> None:
        self._check(self.lib.fe_op_rmsnorm(self._h, ctypes.c_void_p(x_ptr), ctypes.c_void_p(w_ptr),
                                           ctypes.c_void_p(out_ptr), rows, d))
