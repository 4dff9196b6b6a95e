"""The reference's backend laws (`/root/reference/pkg/tests/test_backends.py`)
applied to the device backend: the same calls and assertions, with
`EngineBackend` in place of `SyntheticBackend` and the tokens checked against
the CPU oracle backend (tiny, fp32: bit-exact).

Reference tests mirrored (file:line of the reference test):
  test_encode_degenerate_input           test_backends.py:23
  test_encode_deterministic              test_backends.py:28
  test_begin_step_deterministic          test_backends.py:51
  test_step_generator_yields_one_token_per_call  test_backends.py:59
  test_truncation_flag                   test_backends.py:90
  test_missing_profile_step_raises       test_backends.py:99
"""

import pytest

from ecot_sched.backends import BackendError, StepProfile, SyntheticProfile, default_profile
from paper_2506_07639_b200.engine_backend import EngineBackend

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def backend():
    be = EngineBackend("tiny", dtype="f32", seed=0, kv_pages=512, profile=default_profile(seed=42))
    yield be
    be.close()


@pytest.fixture(scope="module")
def oracle():
    from oracle.backend import OracleBackend
    return OracleBackend("tiny", seed=0, profile=default_profile(seed=42))


def test_encode_degenerate_input(backend, oracle, schema):
    ctx = backend.encode("", b"")
    assert ctx.encoded == ()
    # and the empty context still frames and decodes (BOS + VIS rows + TAG only)
    got = backend.begin_step(ctx, (), schema.steps[0], ()).drain()
    want = oracle.begin_step(oracle.encode("", b""), (), schema.steps[0], ()).drain()
    assert got == want


def test_encode_deterministic(backend):
    a = backend.encode("lift the cup", b"\x01\x02")
    b = backend.encode("lift the cup", b"\x01\x02")
    assert a == b
    assert len(a.encoded) > 0


def test_begin_step_deterministic(backend, oracle, schema):
    ctx = backend.encode("pick", b"obs")
    spec = schema.steps[1]
    prev = (7, 8, 9)
    runs = [backend.begin_step(ctx, (1, 2), spec, prev).drain() for _ in range(3)]
    assert runs[0] == runs[1] == runs[2]
    assert runs[0] == oracle.begin_step(oracle.encode("pick", b"obs"), (1, 2), spec, prev).drain()


def test_step_generator_yields_one_token_per_call(backend, schema):
    ctx = backend.encode("pick", b"obs")
    gen = backend.begin_step(ctx, (), schema.steps[0], ())
    out = []
    while not gen.done:
        out.append(gen.next_token())
    assert tuple(out) == gen.tokens
    assert gen.next_token() is None


def test_truncation_flag(schema):
    profile = SyntheticProfile(steps={"task": StepProfile(500, 0, 1.0)}, seed=1)
    be = EngineBackend("tiny", dtype="f32", seed=0, kv_pages=256, profile=profile)
    try:
        spec = schema.steps[0]
        gen = be.begin_step(be.encode("i", b"o"), (), spec, ())
        assert gen.truncated
        assert len(gen.drain()) == spec.max_tokens
    finally:
        be.close()


def test_missing_profile_step_raises(schema):
    be = EngineBackend("tiny", dtype="f32", seed=0, kv_pages=64, profile=SyntheticProfile(steps={}, seed=0))
    try:
        with pytest.raises(BackendError):
            be.begin_step(be.encode("i", b"o"), (), schema.steps[0], ())
        assert be.engine.stats()["pages_used"] == 0   # rejected before any trunk or branch exists
    finally:
        be.close()
