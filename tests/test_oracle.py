"""The CPU oracle pinned before it is trusted (CPU only):

* its weights equal the numpy restatement of the counter-based init;
* its logits agree with an independent plain-PyTorch fp32 model (standard
  ops, not the canonical arithmetic) within the north-star 1e-3 relative
  tolerance, with identical greedy tokens;
* it reproduces the committed golden request vectors exactly;
* its canonical primitives behave as specified (exp accuracy, dot order).
"""

import json
import math

import numpy as np
import pytest
import torch

import torch_ref
from conftest import GOLDEN
from oracle.backend import OracleModel, frame
from paper_2506_07639_b200 import model as M

LOGIT_RTOL = 1e-3  # north_star: logits within 1e-3 relative in fp32


@pytest.fixture(scope="module")
def tiny():
    return OracleModel("tiny", seed=0)


def test_weights_match_numpy_init(tiny):
    cfg = M.PRESETS["tiny"]
    assert np.array_equal(tiny.tensor(M.T_EMBED, 0, (cfg.vocab, cfg.d_model)),
                          M.init_linear(0, M.T_EMBED, cfg.vocab, cfg.d_model))
    assert np.array_equal(tiny.tensor(M.layer_tensor(2, M.L_WDOWN), 2, (cfg.d_model, cfg.d_ffn)),
                          M.init_linear(0, M.layer_tensor(2, M.L_WDOWN), cfg.d_model, cfg.d_ffn))
    assert np.array_equal(tiny.tensor(M.layer_tensor(3, M.L_ATTN_NORM), 3, (cfg.d_model,)),
                          M.init_norm(0, M.layer_tensor(3, M.L_ATTN_NORM), cfg.d_model))


@pytest.mark.parametrize("prefix_len", [0, 37, 150])
def test_logits_match_torch_fp32(tiny, prefix_len):
    cfg = M.PRESETS["tiny"]
    rng = np.random.default_rng(prefix_len)
    ids = frame("tiny", rng.integers(0, 2**32, 16).tolist(), rng.integers(0, 32000, prefix_len).tolist(), "plan")
    toks, logits = tiny.generate(ids, 99 + prefix_len, 6, want_logits=True)
    ref = torch_ref.forward_logits(cfg, torch_ref.build_weights(cfg, 0), ids + toks[:-1], 99 + prefix_len)
    ref = ref[len(ids) - 1:].numpy()
    assert np.abs(ref - logits).max() / np.abs(ref).max() < LOGIT_RTOL
    assert ref[:, : M.TEXT_VOCAB].argmax(-1).tolist() == toks


@pytest.mark.parametrize("name", ["small"])
def test_golden_requests(name):
    g = json.loads((GOLDEN / f"requests_{name}.json").read_text())
    om = OracleModel(name, seed=g["seed"])
    for case in g["cases"][:2]:
        toks, logits = om.generate(case["ids"], case["vseed"], case["n_out"], want_logits=True)
        assert toks == case["tokens"]
        assert logits[:, :8].tolist() == case["logits_head"]


def test_prefix_cache_is_exact(tiny):
    ids = frame("tiny", list(range(16)), list(range(200, 290)), "task")
    a, la = tiny.generate(ids, 5, 4, want_logits=True)       # fills the cache
    b, lb = tiny.generate(ids, 5, 4, want_logits=True)       # reuses the whole prefix
    fresh = OracleModel("tiny", seed=0)
    c, lc = fresh.generate(ids, 5, 4, want_logits=True)
    assert a == b == c
    assert np.array_equal(la, lb) and np.array_equal(la, lc)


def test_deterministic_exp_accuracy():
    lib = OracleModel("tiny", seed=0).lib
    xs = np.concatenate([np.linspace(-86.9, 0.0, 5000), np.linspace(0.0, 20.0, 200)]).astype(np.float32)
    for x in xs:
        got = lib.or_exp(float(x))
        want = math.exp(float(x))
        assert abs(got - want) <= 4e-6 * want + 1e-38
    assert lib.or_exp(-1000.0) == 0.0
    assert lib.or_exp(0.0) == 1.0


def test_canonical_dot_order():
    lib = OracleModel("tiny", seed=0).lib
    rng = np.random.default_rng(3)
    for K in (4, 64, 128, 256, 688, 4096):
        w = rng.standard_normal(K).astype(np.float32)
        x = rng.standard_normal(K).astype(np.float32)
        a = np.zeros(32, dtype=np.float64)
        # exact emulation with float32 rounding at every step
        acc = np.zeros(32, dtype=np.float32)
        for j in range(0, K, 128):
            for l in range(32):
                k = j + 4 * l
                if k < K:
                    for c in range(4):
                        acc[l] = np.float32(np.float64(w[k + c]) * np.float64(x[k + c]) + np.float64(acc[l]))
        off = 16
        while off:
            acc[:off] = acc[:off] + acc[off:2 * off]
            off //= 2
        got = lib.or_cdot(w.ctypes.data, x.ctypes.data, K)
        assert np.float32(got) == acc[0]
        del a


def test_reference_runners_over_oracle_reproduce_golden(schema, golden_traces):
    """The golden lines were produced by the reference runners over the CPU
    oracle (tests/golden/make_golden.py); re-running them here pins the
    oracle (and the runners' simulated accounting) for the GPU parity tests."""
    import ecot_sched
    from ecot_sched.trace import trace_content_bytes

    from oracle.backend import OracleBackend, OracleModel
    model = OracleModel("tiny", seed=0)
    for mode in ("sequential", "parallel_sync", "parallel_async", "k_step", "two_track"):
        g = golden_traces["modes"][mode]
        cfg = ecot_sched.SchedulerConfig(mode=mode, slots=8)
        res, _ = ecot_sched.run_episode(cfg, golden_traces["T"], OracleBackend("tiny", seed=0, model=model),
                                        schema, seed=0)
        assert [trace_content_bytes(r.trace, schema).decode() for r in res] == g["lines"], mode
        assert [r.latency_ms for r in res] == g["latency_ms"]
        assert [r.staleness for r in res] == g["staleness"]
        assert [r.generated_tokens for r in res] == g["generated_tokens"]


def test_vision_oracle_matches_float64_restatement():
    """oracle/oracle.c's vision tower + projector (canonical fp32) against an
    independent float64 numpy restatement of the same definition."""
    from vision_ref import vision_rows

    from oracle.backend import OracleModel
    m = OracleModel("tiny", seed=3, vision="vit_tiny")
    for vseed in (1, 987654321):
        got = m.vision_encode(vseed)
        want = vision_rows("tiny", "vit_tiny", 3, vseed)
        assert got.shape == want.shape == (16, 256)
        rel = np.abs(got - want).max() / np.abs(want).max()
        assert rel < 1e-4, rel


def test_vision_rows_feed_the_oracle_model():
    """With a tower, the oracle's VIS rows are the tower's output: the greedy
    continuation changes with the observation's image."""
    from oracle.backend import OracleModel, frame
    m = OracleModel("tiny", seed=0, vision="vit_tiny")
    ids = frame("tiny", list(range(16)), [5, 6, 7], "plan")
    a, _ = m.generate(ids, 11, 6)
    b, _ = m.generate(ids, 12, 6)
    plain = OracleModel("tiny", seed=0)
    c, _ = plain.generate(ids, 11, 6)
    assert a != b and a != c
