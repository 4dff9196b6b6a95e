"""CPU ORACLE BACKEND -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
`--impl reference`) may import this module; the product package never does.

`OracleBackend` implements the reference `GenerationBackend` protocol
(`pkg/src/ecot_sched/backends.py:98-110`) over the C model of oracle.c, so
the *reference's own runners* (`schedulers.py:329-552`) can drive it to
produce golden traces.  The request framing and the length decision are
restated here independently of the product package:

* framing: ``[BOS] + [VIS]*n_vision + ctx.encoded%32000 + prefix%32000 + [TAG]``
  (tag after the prefix);
* length: the reference `SyntheticBackend.begin_step` draw order
  (backends.py:181-207) -- Bernoulli reuse keeps len(prev_content), else a
  rounded Gaussian clamped to [1, max_tokens]; `truncated` when the budget
  binds.  The emitted *tokens* are the oracle model's greedy decode.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liboracle.so"

TEXT_VOCAB, VOCAB, BOS, VIS, TAG_BASE = 32000, 32064, 32000, 32001, 32002

# (d, layers, heads, head_dim, ffn, n_vision) -- must match model.PRESETS
SHAPES = {
    "tiny": (256, 4, 4, 64, 688, 16),
    "small": (1024, 4, 8, 128, 2752, 64),
    "7b_2layer": (4096, 2, 32, 128, 11008, 256),
    "7b": (4096, 32, 32, 128, 11008, 256),
}


def _digest(*parts) -> int:
    # blake2b-64 over parts joined by 0x1f (reference backends.py:56-66)
    h = hashlib.blake2b(digest_size=8)
    for p in parts:
        if isinstance(p, str):
            p = p.encode("utf-8")
        elif isinstance(p, int):
            p = p.to_bytes(16, "little", signed=True)
        h.update(p)
        h.update(b"\x1f")
    return int.from_bytes(h.digest(), "little")


def rope_table(head_dim: int, max_pos: int, theta: float = 10000.0) -> np.ndarray:
    half = head_dim // 2
    inv = theta ** (-np.arange(half, dtype=np.float64) * 2.0 / head_dim)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.ascontiguousarray(np.stack([np.cos(ang), np.sin(ang)], axis=1).astype(np.float32))


def load_library() -> ctypes.CDLL:
    if not _LIB_PATH.exists():
        raise RuntimeError(f"oracle library missing: {_LIB_PATH} (run `make -C oracle`)")
    lib = ctypes.CDLL(str(_LIB_PATH))
    lib.or_create.restype = ctypes.c_void_p
    lib.or_create.argtypes = [ctypes.c_int] * 7 + [ctypes.c_float, ctypes.c_float, ctypes.c_uint64,
                                                   ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    lib.or_destroy.argtypes = [ctypes.c_void_p]
    lib.or_generate.restype = ctypes.c_int
    lib.or_generate.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64,
                                ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    lib.or_cdot.restype = ctypes.c_float
    lib.or_cdot.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    lib.or_exp.restype = ctypes.c_float
    lib.or_exp.argtypes = [ctypes.c_float]
    lib.or_rmsnorm.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_float]
    lib.or_matmul.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3
    lib.or_attention.argtypes = [ctypes.c_void_p] * 6 + [ctypes.c_int]
    lib.or_vision_create.restype = ctypes.c_void_p
    lib.or_vision_create.argtypes = [ctypes.c_int] * 8 + [ctypes.c_float, ctypes.c_uint64]
    lib.or_vision_destroy.argtypes = [ctypes.c_void_p]
    lib.or_vision_encode.restype = ctypes.c_int
    lib.or_vision_encode.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
    lib.or_set_vision.restype = ctypes.c_int
    lib.or_set_vision.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    lib.or_tensor.restype = ctypes.c_void_p
    lib.or_tensor.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    return lib


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


class OracleModel:
    """Handle on the C model; weights are generated at construction."""

    def __init__(self, config: str = "tiny", seed: int = 0, threads: int = 0, max_pos: int = 8192,
                 vision=None):
        self.lib = load_library()
        self._vh = None
        self.config = config
        d, L, H, hd, F, nv = SHAPES[config]
        self.d, self.L, self.H, self.hd, self.F, self.n_vision = d, L, H, hd, F, nv
        self.seed = seed
        self.max_pos = max_pos
        self.rope = rope_table(hd, max_pos)
        self.attn_scale = np.float32(1.0) / np.sqrt(np.float32(hd))
        self._h = self.lib.or_create(d, L, H, hd, F, VOCAB, TEXT_VOCAB, ctypes.c_float(1e-5),
                                     ctypes.c_float(self.attn_scale), ctypes.c_uint64(seed),
                                     _ptr(self.rope), max_pos, threads or (os.cpu_count() or 1))
        if not self._h:
            raise RuntimeError("or_create failed")
        self.vision = None
        if vision:   # VIS rows from the vision tower + projector (oracle.c or_vision_encode)
            from paper_2506_07639_b200.model import get_vision
            v = get_vision(vision, config)
            self._vh = self.lib.or_vision_create(v.img, v.patch, v.d, v.layers, v.heads, v.mlp, v.proj_hidden, d,
                                                 ctypes.c_float(v.eps), ctypes.c_uint64(seed))
            if not self._vh or self.lib.or_set_vision(self._h, self._vh) != 0:
                raise RuntimeError("or_vision_create / or_set_vision failed")
            self.vision = v

    def vision_encode(self, vseed: int) -> np.ndarray:
        out = np.empty((self.vision.patches, self.d), dtype=np.float32)
        self.lib.or_vision_encode(self._vh, ctypes.c_uint64(vseed & 0xFFFFFFFFFFFFFFFF), _ptr(out))
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self.lib.or_destroy(h)
            self._h = None
        vh = getattr(self, "_vh", None)
        if vh:
            self.lib.or_vision_destroy(vh)
            self._vh = None

    def generate(self, ids, vseed: int, n_out: int, want_logits: bool = False):
        ids = np.ascontiguousarray(np.asarray(ids, dtype=np.int32))
        out = np.zeros(n_out, dtype=np.int32)
        logits = np.zeros((n_out, VOCAB), dtype=np.float32) if want_logits else None
        rc = self.lib.or_generate(self._h, _ptr(ids), int(ids.size), ctypes.c_uint64(vseed), VIS,
                                  int(n_out), _ptr(out), _ptr(logits) if want_logits else None)
        if rc != 0:
            raise RuntimeError(f"or_generate failed ({rc})")
        return [int(t) for t in out], logits

    def tensor(self, which: int, layer: int, shape) -> np.ndarray:
        p = self.lib.or_tensor(self._h, which, layer)
        n = int(np.prod(shape))
        return np.ctypeslib.as_array((ctypes.c_float * n).from_address(p)).reshape(shape).copy()


def frame(config: str, encoded, prefix, step_name: str) -> list[int]:
    nv = SHAPES[config][5]
    tag = TAG_BASE + _digest("tag", step_name) % (VOCAB - TAG_BASE)
    return ([BOS] + [VIS] * nv + [int(e) % TEXT_VOCAB for e in encoded]
            + [int(t) % TEXT_VOCAB for t in prefix] + [tag])


def planned_length(profile, context, step, prev_content) -> tuple[int, bool]:
    """Length decision of the reference SyntheticBackend (backends.py:181-207)."""
    prof = profile.steps.get(step.name)
    if prof is None:
        return -1, False
    ctx_part = _digest(context.instruction, context.observation) if profile.vary_with_context else 0
    rng = np.random.default_rng(_digest("step", profile.seed, ctx_part, step.name))
    if rng.random() < prof.change_probability or not prev_content:
        raw = int(round(rng.normal(prof.mean_tokens, prof.stddev_tokens)))
        return min(max(raw, 1), step.max_tokens), raw > step.max_tokens
    return len(prev_content), False


class OracleBackend:
    """GenerationBackend over the CPU oracle model (fp32, canonical arithmetic)."""

    deterministic = True
    supports_prefix_conditioning = True

    def __init__(self, config: str = "tiny", seed: int = 0, profile=None, threads: int = 0,
                 model: OracleModel | None = None, vision=None):
        from paper_2506_07639_b200.refapi import backends as rb  # the reference API (profile is data)
        default_profile = rb.default_profile
        self.model = model or OracleModel(config, seed, threads, vision=vision)
        self.config = config
        self.profile = profile or default_profile(seed)
        self.requests = 0

    def encode(self, instruction: str, observation: bytes):
        from paper_2506_07639_b200.refapi import trace as rt
        Context = rt.Context
        if not instruction and not observation:
            return Context(instruction, observation, ())
        rng = np.random.default_rng(_digest("encode", instruction, observation))
        return Context(instruction, observation, tuple(int(t) for t in rng.integers(0, 2**32, size=16)))

    def begin_step(self, context, prefix, step, prev_content):
        from paper_2506_07639_b200.refapi import backends as rb
        BackendError, StepGenerator = rb.BackendError, rb.StepGenerator
        n, truncated = planned_length(self.profile, context, step, prev_content)
        if n < 0:
            raise BackendError(f"no synthetic profile for step {step.name!r}")
        ids = frame(self.config, context.encoded, prefix, step.name)
        tokens, _ = self.model.generate(ids, _digest("vision", context.observation), n)
        self.requests += 1
        return StepGenerator(tokens, truncated=truncated)
