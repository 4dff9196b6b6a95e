"""Host-side mirror of the reference API vs vectors produced by the reference
itself (tests/golden/make_golden.py).  CPU only."""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2506_07639_b200 import backends as B
from paper_2506_07639_b200 import batching as BA
from paper_2506_07639_b200 import schedulers as S
from paper_2506_07639_b200 import trace as T

V = json.loads((GOLDEN / "mirror_vectors.json").read_text())


def _part(p):
    return bytes.fromhex(p[2:]) if isinstance(p, str) and p.startswith("b:") else p


def test_stable_digest_matches_reference():
    for case in V["stable_digest"]:
        assert B.stable_digest(*[_part(p) for p in case["parts"]]) == case["digest"]


def test_observation_for_matches_reference():
    for case in V["observation_for"]:
        assert S.observation_for(case["seed"], case["t"]).hex() == case["hex"]


def test_context_encoding_matches_reference():
    for case in V["encode"]:
        got = B.encode_tokens(case["instruction"], bytes.fromhex(case["observation"]))
        assert list(got) == case["encoded"]


def test_synthetic_draws_match_reference(schema):
    spec_of = {s.name: s for s in schema.steps}
    for d in V["synthetic_draws"]:
        if d.get("profile") == "truncation":
            be = B.SyntheticBackend(B.SyntheticProfile({"task": B.StepProfile(500, 0, 1.0)}, seed=1))
            ctx = be.encode("i", b"o")
        else:
            be = B.SyntheticBackend(B.default_profile(d["seed"]))
            ctx = be.encode("pick up the object and place it on the target", S.observation_for(d["seed"], d["t"]))
        g = be.begin_step(ctx, (1, 2, 3), spec_of[d["step"]], tuple(d["prev"]))
        assert list(g.tokens) == d["tokens"]
        assert g.truncated == d["truncated"]
        plan = B.length_plan(be.profile, ctx, spec_of[d["step"]], tuple(d["prev"]))
        assert plan.length == len(d["tokens"]) and plan.truncated == d["truncated"]


def test_decode_action_matches_reference():
    for case in V["decode_action"]:
        assert list(S.decode_action(tuple(case["tokens"]), case["dim"]).components) == case["components"]


def test_trace_bytes_match_reference(schema):
    tr = T.ReasoningTrace(3, (("task", (1, 2)), ("plan", ()), ("action", (5, 6, 7))),
                          T.ActionVector((0.5, -0.25, 1e-7)))
    assert T.trace_content_bytes(tr, schema).decode() == V["trace_bytes"]["content"]
    assert T.serialize_trace(tr, schema, wall_ms=12.5).decode() == V["trace_bytes"]["serialized"]
    back = T.deserialize_trace(V["trace_bytes"]["serialized"].encode())
    assert back == tr


def test_trace_parse_error_carries_offset():
    with pytest.raises(T.TraceParseError) as exc:
        T.parse_log_line(b'{"timestep": 1, "steps": [', base_offset=100)
    assert exc.value.offset >= 100


def test_fig5_known_answers():
    # PAPER Fig. 5: 44 vs 26 tokens, waste 0.409 (reference tests/test_batching.py:34-67)
    b = V["batching"]
    reqs = [BA.GenerationRequest(i, i, 0, L) for i, L in enumerate((3, 6, 8, 9))]
    cb = BA.continuous_batch(reqs, 4)
    sb = BA.static_batch(reqs, 4, pad_to=11)
    lm = BA.LatencyModel(c_iter=10, c_slot=1, c_encode=20, c_decode=5)
    assert cb.busy_slot_iterations == b["fig5_continuous_busy"] == 26
    assert sb.occupied_slot_iterations == b["fig5_static_occupied"] == 44
    assert BA.padding_waste(sb) == pytest.approx(b["fig5_waste"])
    assert BA.schedule_cost(cb, lm) == b["fig5_cost"]
    assert cb.makespan == b["fig5_makespan"]
    assert cb.grid.tolist() == b["fig5_grid"]


def test_continuous_batch_priority_and_arrivals_match_reference():
    mixed = [BA.GenerationRequest(0, 0, 0, 5), BA.GenerationRequest(1, 1, 0, 7, priority=BA.ACTION),
             BA.GenerationRequest(2, 2, 0, 3, arrival_iteration=2), BA.GenerationRequest(3, 3, 0, 4)]
    assert BA.continuous_batch(mixed, 2).grid.tolist() == V["batching"]["mixed_grid"]


def test_step_generator_one_token_per_call(schema):
    # reference tests/test_backends.py:59-66
    be = B.SyntheticBackend(B.default_profile(42))
    gen = be.begin_step(be.encode("pick", b"obs"), (), schema.steps[0], ())
    out = []
    while not gen.done:
        out.append(gen.next_token())
    assert tuple(out) == gen.tokens
    assert gen.next_token() is None


def test_unknown_step_raises_backend_error(schema):
    be = B.SyntheticBackend(B.SyntheticProfile(steps={}, seed=0))
    with pytest.raises(B.BackendError):
        be.begin_step(be.encode("i", b"o"), (), schema.steps[0], ())
