"""Engine-side additions to the reference backend boundary.

The boundary itself is the reference's (`ecot_sched.backends`,
`pkg/src/ecot_sched/backends.py:98-110`); this module only adds

* `EngineError` -- a `ecot_sched.backends.BackendError`, so the reference
  runners' `reuse_stale` / `abort_episode` policies apply to engine
  failures unchanged (`schedulers.py:411-434`, `:481-483`, `:510-517`);
* `length_plan` -- the workload length oracle: the length
  and `truncated` flag the reference `SyntheticBackend.begin_step` would
  emit for the request (`backends.py:190-209`).  Random-init weights never
  emit a meaningful stop token, so the engine decodes greedily for exactly
  this many tokens and the calibrated makespan distribution is kept;
* `encode_context` -- the reference context encoding
  (`SyntheticBackend.encode`, `backends.py:178-179`, `:113-117`).
"""

from __future__ import annotations

from typing import NamedTuple

from .refapi import backends as _rb
from .refapi import trace as _rt

BackendError = _rb.BackendError
StepGenerator = _rb.StepGenerator
SyntheticBackend = _rb.SyntheticBackend
SyntheticProfile = _rb.SyntheticProfile
StepProfile = _rb.StepProfile
default_profile = _rb.default_profile
stable_digest = _rb.stable_digest


class EngineError(BackendError):
    """Raised when the B200 engine (C ABI) reports a non-zero status."""


class LengthPlan(NamedTuple):
    length: int
    truncated: bool


def length_plan(profile: SyntheticProfile, context: _rt.Context, step: _rt.StepSpec,
                prev_content) -> LengthPlan:
    """Length decision of the reference synthetic backend for this request,
    taken from the reference implementation itself (so the draw order --
    reuse Bernoulli, rounded Gaussian, clamp -- cannot drift).  Raises the
    reference `BackendError` for a step without a profile."""
    gen = SyntheticBackend(profile).begin_step(context, (), step, tuple(prev_content))
    return LengthPlan(len(gen.tokens), bool(gen.truncated))


def encode_context(instruction: str, observation: bytes) -> _rt.Context:
    """The reference context encoding (`backends.py:113-117`, `:178-179`)."""
    return SyntheticBackend(default_profile()).encode(instruction, observation)
