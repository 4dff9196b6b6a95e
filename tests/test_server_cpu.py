"""The `/v1/completions` front (server.py) driven by the UNMODIFIED reference
client (`ecot_sched.backends.remote_complete` / `RemoteBackend`, backends.py:
285-379) -- the contract the reference's own stub tests pin
(`pkg/tests/test_remote.py`) -- over the CPU fake engine."""

import json
import threading

import pytest
import requests
from fake_engine import ar_tokens, fake_backend

import ecot_sched
from ecot_sched.backends import (RemoteBackend, RemoteEndpoint, RemoteStatusError, default_prompt_builder,
                                 remote_complete)
from ecot_sched.schedulers import ParallelSyncRunner, SchedulerConfig
from ecot_sched.trace import default_schema
from paper_2506_07639_b200 import model as M
from paper_2506_07639_b200.backends import encode_context
from paper_2506_07639_b200.server import CompletionServer, parse_prompt


@pytest.fixture()
def served():
    be, eng = fake_backend(autoregressive=True)
    with CompletionServer(be, observation=b"frame-0") as srv:
        yield srv, be, eng


def test_parse_reference_default_prompt():
    ctx = encode_context("pick up the cup", b"")
    step = default_schema().steps[2]
    prompt = default_prompt_builder(ctx, (5, 17, 123456789), step)
    assert parse_prompt(prompt) == ("pick up the cup", step.name, (5, 17, 123456789))
    assert parse_prompt("free text") == ("free text", "completion", ())
    assert parse_prompt(default_prompt_builder(ctx, (), step)) == ("pick up the cup", step.name, ())


def test_completion_contract_with_reference_client(served):
    srv, _, _ = served
    res = remote_complete(RemoteEndpoint(srv.url), "lift the cup", 12)
    assert res.tokens_reported == 12
    assert len(res.text.split()) == 12
    assert res.retries == 0
    assert remote_complete(RemoteEndpoint(srv.url), "go", 0).tokens_reported == 0


def test_tokens_are_the_engines_greedy_tokens(served):
    """The reply is exactly the request EngineBackend.begin_step would decode:
    context + prefix framing, the step's tag, greedy continuation."""
    srv, be, _ = served
    step = default_schema().steps[1]
    ctx = encode_context("open the drawer", b"frame-0")
    prompt = default_prompt_builder(ctx, (7, 8, 9), step)
    res = remote_complete(RemoteEndpoint(srv.url), prompt, 20)
    ids = M.context_ids(ctx, be.cfg) + M.text_ids((7, 8, 9))
    want = ar_tokens(M.vision_seed(b"frame-0"), ids, M.step_tag(step), 20)
    assert tuple(int(t) for t in res.text.split()) == want


def test_observation_field_overrides_the_default(served):
    srv, _, _ = served
    body = {"prompt": "x", "max_tokens": 6, "stream": False}
    a = requests.post(srv.url + "/v1/completions", json=body).json()["choices"][0]["text"]
    b = requests.post(srv.url + "/v1/completions", json={**body, "observation": b"other".hex()}).json()
    assert a != b["choices"][0]["text"]


def test_reference_runner_over_the_wire(served):
    """A full reference ParallelSyncRunner timestep through RemoteBackend
    (test_remote.py:88-103 analogue, against the engine instead of a stub)."""
    srv, _, _ = served
    schema = default_schema()
    backend = RemoteBackend(RemoteEndpoint(srv.url, max_retries=2))
    runner = ParallelSyncRunner(backend, schema, SchedulerConfig(mode="parallel_sync", slots=8, wall_clock=True))
    r0 = runner.step(backend.encode("pick", b"obs-0"), 0)
    r1 = runner.step(backend.encode("pick", b"obs-1"), 1)
    want = sum(s.max_tokens for s in schema.steps)
    assert r0.generated_tokens == want and r1.generated_tokens == want
    assert backend.metrics["requests"] == 2 * len(schema.steps)
    assert backend.metrics["failures"] == 0


def test_concurrent_requests_decode_as_one_batch(served):
    srv, _, eng = served
    out = [None] * 8

    def call(i):
        out[i] = remote_complete(RemoteEndpoint(srv.url), f"task {i}", 10).text

    ts = [threading.Thread(target=call, args=(i,)) for i in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert all(o is not None and len(o.split()) == 10 for o in out)
    assert srv.stats["max_batch"] > 1
    assert max(o for lane, o in eng.occupancy_log) > 1


def test_bad_requests_are_not_retried(served):
    srv, _, _ = served
    for body in (b"not json", json.dumps({"prompt": 3}).encode(),
                 json.dumps({"prompt": "x", "max_tokens": -1}).encode(),
                 json.dumps({"prompt": "x", "max_tokens": 4, "stream": True}).encode()):
        r = requests.post(srv.url + "/v1/completions", data=body)
        assert r.status_code == 400
    with pytest.raises(RemoteStatusError) as exc:
        remote_complete(RemoteEndpoint(srv.url, max_retries=3), "x", 5000)
    assert exc.value.status == 400
    assert requests.get(srv.url + "/health").status_code == 200


def test_engine_rejection_is_retryable_503():
    be, eng = fake_backend(autoregressive=True)
    eng.pages_total = 0                     # every request fails its KV reservation
    with CompletionServer(be) as srv:
        with pytest.raises(RemoteStatusError) as exc:
            remote_complete(RemoteEndpoint(srv.url, max_retries=1), "x", 8)
    assert exc.value.status == 503
    assert isinstance(exc.value, ecot_sched.BackendError)
