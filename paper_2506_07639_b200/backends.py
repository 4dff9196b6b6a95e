"""The generation-backend boundary and the workload length oracle.

Mirror of the reference plugin boundary (`pkg/src/ecot_sched/backends.py`):

* `GenerationBackend` protocol and `StepGenerator` result type
  (`backends.py:69-110`) -- the B200 `EngineBackend` implements this verbatim;
* typed errors (`backends.py:32-53`) -- engine failures surface as
  `BackendError` so the runners' failure policies apply unchanged;
* `stable_digest` / context encoding (`backends.py:56-66`, `:113-117`);
* `SyntheticBackend` and its profiles (`backends.py:120-209`).  On the engine
  path the synthetic draw is *not* the generator: the engine decodes tokens
  greedily from the decoder and only borrows the synthetic backend's length
  decision (`length_plan`), so random-init weights reproduce the calibrated
  per-step workload ("model-input framing").
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, replace
from typing import NamedTuple, Optional, Protocol, Sequence

import numpy as np

from .trace import Context, StepSpec, TokenSeq

TOKEN_SPACE = 2**32           # backends.py:28
ENCODED_CONTEXT_TOKENS = 16   # backends.py:29


class BackendError(Exception):
    """Base class of generation failures (backends.py:32-33)."""


class RemoteError(BackendError):
    def __init__(self, message: str, endpoint: str):
        super().__init__(f"{message} [endpoint {endpoint}]")
        self.endpoint = endpoint


class RemoteStatusError(RemoteError):
    def __init__(self, status: int, endpoint: str):
        super().__init__(f"unexpected HTTP status {status}", endpoint)
        self.status = status


class RemoteTimeoutError(RemoteError):
    pass


class RemoteProtocolError(RemoteError):
    pass


class EngineError(BackendError):
    """Raised when the B200 engine (C-ABI) reports a non-zero status."""


def stable_digest(*parts: bytes | str | int) -> int:
    """64-bit blake2b digest, process-stable (backends.py:56-66)."""
    h = hashlib.blake2b(digest_size=8)
    for part in parts:
        if isinstance(part, str):
            part = part.encode("utf-8")
        elif isinstance(part, int):
            part = part.to_bytes(16, "little", signed=True)
        h.update(part)
        h.update(b"\x1f")
    return int.from_bytes(h.digest(), "little")


class StepGenerator:
    """Hands out a finished token sequence one token per call (backends.py:69-95)."""

    def __init__(self, tokens: Sequence[int], truncated: bool = False,
                 reported_tokens: int | None = None):
        self.tokens: TokenSeq = tuple(int(t) for t in tokens)
        self.truncated = truncated
        self.reported_tokens = len(self.tokens) if reported_tokens is None else reported_tokens
        self._pos = 0

    @property
    def done(self) -> bool:
        return self._pos >= len(self.tokens)

    def next_token(self) -> Optional[int]:
        if self.done:
            return None
        self._pos += 1
        return self.tokens[self._pos - 1]

    def drain(self) -> TokenSeq:
        self._pos = len(self.tokens)
        return self.tokens


class GenerationBackend(Protocol):
    """Plugin boundary (backends.py:98-110)."""

    deterministic: bool
    supports_prefix_conditioning: bool

    def encode(self, instruction: str, observation: bytes) -> Context: ...

    def begin_step(self, context: Context, prefix: TokenSeq, step: StepSpec,
                   prev_content: TokenSeq) -> StepGenerator: ...


def encode_tokens(instruction: str, observation: bytes) -> TokenSeq:
    """The 16 hash-seeded context ids of `backends.py:113-117`."""
    if not instruction and not observation:
        return ()
    rng = np.random.default_rng(stable_digest("encode", instruction, observation))
    return tuple(int(t) for t in rng.integers(0, TOKEN_SPACE, size=ENCODED_CONTEXT_TOKENS))


_encode_tokens = encode_tokens  # reference spelling, used by its test fixtures


@dataclass(frozen=True)
class StepProfile:
    """Truncated-Gaussian length + per-timestep change probability (backends.py:120-134)."""

    mean_tokens: float
    stddev_tokens: float = 0.0
    change_probability: float = 1.0

    def __post_init__(self):
        if self.mean_tokens <= 0 or self.stddev_tokens < 0:
            raise ValueError("mean_tokens must be positive, stddev non-negative")
        if not 0.0 <= self.change_probability <= 1.0:
            raise ValueError("change_probability must lie in [0, 1]")


@dataclass(frozen=True)
class SyntheticProfile:
    steps: dict[str, StepProfile]
    seed: int = 0
    vary_with_context: bool = True

    def with_seed(self, seed: int) -> "SyntheticProfile":
        return replace(self, seed=seed)


def default_profile(seed: int = 0) -> SyntheticProfile:
    """Calibrated profile of `backends.py:149-164`."""
    table = {
        "task": (50, 4, 0.03), "plan": (75, 6, 0.084), "subtask": (70, 6, 0.15),
        "move": (18, 2, 0.45), "gripper": (15, 2, 0.30),
        "visible_objects": (120, 8, 0.60), "action": (7, 0, 1.0),
    }
    return SyntheticProfile({k: StepProfile(*v) for k, v in table.items()}, seed=seed)


class LengthPlan(NamedTuple):
    """Outcome of the synthetic draw for one request.

    `reuse` -- the Bernoulli kept `prev_content` (the reference then emits it
    verbatim); `length` -- emitted token count; `truncated` -- budget bound.
    """

    reuse: bool
    length: int
    truncated: bool
    rng: np.random.Generator


def _step_rng(profile: SyntheticProfile, context: Context, step: StepSpec) -> np.random.Generator:
    ctx_part = (stable_digest(context.instruction, context.observation)
                if profile.vary_with_context else 0)
    return np.random.default_rng(stable_digest("step", profile.seed, ctx_part, step.name))


def length_plan(profile: SyntheticProfile, context: Context, step: StepSpec,
                prev_content: TokenSeq) -> LengthPlan:
    """Replays the draw order of `SyntheticBackend.begin_step`
    (backends.py:197-207): Bernoulli, then rounded Gaussian, then clamp."""
    try:
        prof = profile.steps[step.name]
    except KeyError:
        raise BackendError(f"no synthetic profile for step {step.name!r}") from None
    rng = _step_rng(profile, context, step)
    changed = rng.random() < prof.change_probability
    if not changed and prev_content:
        return LengthPlan(True, len(prev_content), False, rng)
    raw = int(round(rng.normal(prof.mean_tokens, prof.stddev_tokens)))
    return LengthPlan(False, min(max(raw, 1), step.max_tokens), raw > step.max_tokens, rng)


class SyntheticBackend:
    """Seeded synthetic generator (backends.py:167-209)."""

    deterministic = True
    supports_prefix_conditioning = True

    def __init__(self, profile: SyntheticProfile):
        self.profile = profile

    def encode(self, instruction: str, observation: bytes) -> Context:
        return Context(instruction, observation, encode_tokens(instruction, observation))

    def begin_step(self, context: Context, prefix: TokenSeq, step: StepSpec,
                   prev_content: TokenSeq) -> StepGenerator:
        plan = length_plan(self.profile, context, step, prev_content)
        if plan.reuse:
            return StepGenerator(prev_content)
        ids = plan.rng.integers(0, TOKEN_SPACE, size=plan.length)
        return StepGenerator(ids, truncated=plan.truncated)
