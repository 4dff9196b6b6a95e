"""The reference experiments harness (`ecot_sched.experiments`) over the B200
engine -- SURVEY §8(f) rank 4, harness plumbing.

The reference builds each repetition's backend in `_make_backend`
(`/root/reference/pkg/src/ecot_sched/experiments.py:267-270`) and its spec
only admits `"synthetic"` / `"remote"` (`:66-67`).  `run_engine_experiment`
runs the unmodified `run_experiment` (`:292ff`: every mode cell, the
traces.jsonl / timesteps.csv outputs, the comparison rows and latency ratios)
with that factory swapped for one that serves the spec's calibrated profile
(seeded per repetition, exactly as the synthetic factory seeds it) from one
`EngineBackend` -- so a reference experiment preset runs on the GPU
unchanged.  The swap is scoped to the call.
"""

from __future__ import annotations

import contextlib
from pathlib import Path
from typing import Callable, Optional

from .refapi import experiments as _rx  # noqa: F401  (ecot_sched.experiments)


@contextlib.contextmanager
def engine_backends(factory: Callable[[object, int], object]):
    """Within the block, the reference harness builds backends with
    `factory(spec, rep)` instead of `_make_backend`."""
    orig = _rx._make_backend
    _rx._make_backend = factory
    try:
        yield
    finally:
        _rx._make_backend = orig


def run_engine_experiment(spec, out_root, wall_clock: bool = False, backend=None, config: str = "7b",
                          dtype: str = "bf16", **engine_kw):
    """`ecot_sched.experiments.run_experiment(spec, out_root, wall_clock)` with
    every repetition served by the engine: `backend` (an `EngineBackend`,
    reused across cells; its profile is reseeded per repetition), or one
    built from `config` / `dtype` / `engine_kw`."""
    owned = backend is None
    if owned:
        from .engine_backend import EngineBackend
        backend = EngineBackend(config, dtype=dtype, profile=spec.profile, **engine_kw)

    def factory(sp, rep: int):
        backend.profile = sp.profile.with_seed(sp.profile.seed + rep)   # experiments.py:270
        return backend

    try:
        with engine_backends(factory):
            return _rx.run_experiment(spec, Path(out_root), wall_clock=wall_clock)
    finally:
        if owned:
            backend.close()
