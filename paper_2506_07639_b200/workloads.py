"""BASELINE.json workloads as data (schema + length profile).

The reference keeps the step schema and profile as data, not code
(`SPEC.md:86`; `experiments.py:88-117`), so the stress configuration is just
a custom schema and profile.
"""

from __future__ import annotations

from .refapi import backends as _rb
from .refapi import trace as _rt

StepProfile, SyntheticProfile, default_profile = _rb.StepProfile, _rb.SyntheticProfile, _rb.default_profile
HIGH, LOW, StepSchema, StepSpec, default_schema = _rt.HIGH, _rt.LOW, _rt.StepSchema, _rt.StepSpec, _rt.default_schema

STRESS_STEPS = ("task", "plan", "subtask", "move", "gripper", "visible_objects", "scene")


def stress_schema(action_dim: int = 7) -> StepSchema:
    """Config 5: 7 reasoning steps + action (8-way branch fan-out), budgets
    raised so ~292-token steps fit (~2048 cached reasoning tokens)."""
    levels = (HIGH, HIGH, HIGH, LOW, LOW, LOW, LOW)
    steps = tuple(StepSpec(n, lv, 384) for n, lv in zip(STRESS_STEPS, levels))
    return StepSchema(steps + (StepSpec("action", LOW, 16),), action_dim=action_dim)


def stress_profile(seed: int = 0) -> SyntheticProfile:
    """Every step regenerated every timestep (change_probability 1.0:
    frequent cache invalidation), mean 292 tokens per reasoning step."""
    steps = {n: StepProfile(292, 16, 1.0) for n in STRESS_STEPS}
    steps["action"] = StepProfile(7, 0, 1.0)
    return SyntheticProfile(steps, seed=seed)


WORKLOADS = {
    "config2": (default_schema, default_profile),
    "stress": (stress_schema, stress_profile),
}
