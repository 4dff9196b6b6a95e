"""The benchmarked bf16 path pinned to the fp32 CPU oracle (needs a GPU).

Golden vectors: tests/golden/make_bf16_golden.py (the oracle, fp32, and the
reference runners over it).  The bf16 engine is not bit-exact by design
(bf16 weights/KV, tensor-core and split-K reduction orders); what is asserted
is the agreement the north star asks to be stated:

* teacher-forced logits at the benchmark's shapes (7B width, ~600-token
  Fast-ECoT branch inputs): every generated position is decoded from the
  oracle's own prefix, through the trunk prefill (tcgen05 GEMMs + prefill
  attention) and ONE decode tick of all positions as forked branches -- the
  persistent tick kernel for <= 16 rows, the per-matrix kernel chain above;
  bounds: relative logit error and greedy-argmax agreement;
* free-running token-match rate of whole Fast-ECoT episodes (reference
  `run_episode`, and `BatchedEpisodes` for the > 16-row config-4 path) vs the
  oracle's golden traces.

Measured numbers are written to $BF16_PARITY_OUT (json) when set, which is
how profiles/bf16_parity.json is produced.
"""

import json
import os

import numpy as np
import pytest

import ecot_sched
from conftest import GOLDEN
from ecot_sched import schedulers as RS
from paper_2506_07639_b200 import BatchedEpisodes
from paper_2506_07639_b200 import model as M
from paper_2506_07639_b200.engine import Engine
from paper_2506_07639_b200.engine_backend import EngineBackend

pytestmark = pytest.mark.gpu

# bounds (set from the measured values below with margin)
TF_LOGIT_RTOL = {"7b_2layer": 3e-2, "7b": 1e-1}   # max |dlogit| / max |logit| (stored columns)
# teacher-forced greedy agreement, all positions.  The full-7B golden file has
# 24 positions (one position = 4.2 %): measured 0.83-0.92 across kernel
# revisions, every bf16 argmax inside the oracle's top 5; 7b_2layer (24 and,
# in the episode test, 3160 positions) measures 0.96-1.0
TF_ARGMAX_MIN = {"7b_2layer": 0.85, "7b": 0.79}
TF_EPISODE_MIN = 0.90       # teacher-forced agreement over every golden-episode position
FREE_RUN_MIN = 0.04         # free-running whole-episode token match (chaotic after the first near-tie)
RESULTS: dict = {}


def _record(key, value):
    RESULTS[key] = value
    out = os.environ.get("BF16_PARITY_OUT")
    if out:
        path = os.path.abspath(out)
        prev = json.loads(open(path).read()) if os.path.exists(path) else {}
        prev[key] = value
        with open(path, "w") as fh:
            json.dump(prev, fh, indent=1, sort_keys=True)


def _load(config):
    p = GOLDEN / f"tf_{config}.npz"
    if not p.exists():
        pytest.skip(f"{p.name} not generated")
    return dict(np.load(p))


def teacher_forced(eng: Engine, g: dict, cases, mk: int) -> dict:
    """All positions of `cases` as forked one-token requests in one tick."""
    eng.set_option("mk", mk)
    rows, seqs = [], []
    for c in cases:
        ids = [int(x) for x in g["ids"][c][: g["n_ids"][c]]]
        toks = [int(x) for x in g["tokens"][c]]
        full = ids + toks
        n0 = len(ids) - 1
        trunk = eng.seq_create()
        eng.prefill(trunk, full[: n0 + len(toks) - 1], int(g["vseed"][c]), M.VIS_ID)
        seqs.append(trunk)
        for i in range(len(toks)):
            b = eng.seq_fork(trunk, n0 + i)
            seqs.append(b)
            r = eng.submit(b, full[n0 + i], 1, 1)
            eng.capture_logits(r)
            rows.append((c, i, r))
    eng.set_slots(len(rows))
    eng.run(-1)
    out = {}
    for c, i, r in rows:
        out[(c, i)] = eng.request_logits(r, 1)[0]
        eng.request_release(r)
    for s in seqs:
        eng.seq_free(s)
    return out


def _compare(g, got) -> dict:
    rel, agree, in_top5, n = 0.0, 0, 0, 0
    for (c, i), lg in got.items():
        ref = g["logits_head"][c, i]
        rel = max(rel, float(np.abs(lg[: ref.size] - ref).max() / np.abs(ref).max()))
        tok = int(np.argmax(lg[:32000]))
        agree += tok == int(g["tokens"][c, i])
        in_top5 += tok in set(int(x) for x in g["top5_ids"][c, i])
        n += 1
    return {"positions": n, "max_rel_logit_err": rel, "argmax_agreement": agree / n, "argmax_in_oracle_top5": in_top5 / n}


@pytest.mark.parametrize("config", ["7b_2layer", "7b"])
@pytest.mark.parametrize("path", ["tick", "chain"])
def test_bf16_teacher_forced_vs_fp32_oracle(config, path):
    g = _load(config)
    cases = range(g["tokens"].shape[0])
    eng = Engine(config, dtype="bf16", seed=0, kv_pages=256, max_rows=512)
    try:
        eng.profile(True)
        if path == "tick":    # <= 16 rows: one case (8 positions) per tick -> persistent tick kernel
            got = {}
            for c in cases:
                got.update(teacher_forced(eng, g, [c], mk=1))
        else:                 # all cases at once (24 rows) -> the per-matrix kernel chain
            got = teacher_forced(eng, g, list(cases), mk=0)
        ticks = eng.profile_read()["decode_tick"]["launches"]
        eng.profile(False)
        assert (ticks > 0) == (path == "tick"), ticks
    finally:
        eng.close()
    stats = _compare(g, got)
    _record(f"teacher_forced_{config}_{path}", stats)
    print(config, path, stats)
    assert stats["max_rel_logit_err"] < TF_LOGIT_RTOL[config], stats
    assert stats["argmax_agreement"] >= TF_ARGMAX_MIN[config], stats


def _token_match(got_lines, want_lines):
    """(matching tokens, total tokens, first-divergence index per request)."""
    same = total = 0
    first_div = []
    for a, b in zip(got_lines, want_lines):
        ja, jb = json.loads(a), json.loads(b)
        for sa, sb in zip(ja["steps"], jb["steps"]):
            total += len(sb["tokens"])
            eq = [x == y for x, y in zip(sa["tokens"], sb["tokens"])]
            same += sum(eq)
            first_div.append(eq.index(False) if False in eq else len(eq))
    return same, total, first_div


def _traces():
    p = GOLDEN / "traces_7b_2layer.json"
    if not p.exists():
        pytest.skip("traces_7b_2layer.json not generated")
    return json.loads(p.read_text())


def _golden_requests(g):
    """Every request of the golden episodes, rebuilt the way the reference
    runners issued it: (framed ids, vision seed, oracle tokens).  t = 0 is
    the sequential warm-up (prefix = this timestep's earlier steps,
    schedulers.py:329-351); t >= 1 are Fast-ECoT branches (prefix = the
    previous trace's earlier steps, schedulers.py:399-404)."""
    from ecot_sched.backends import SyntheticBackend, default_profile, stable_digest

    from oracle.backend import frame
    enc = SyntheticBackend(default_profile(0))
    out = []
    for seed, lines in g["episodes"].items():
        traces = [json.loads(l) for l in lines]
        for t, tr in enumerate(traces):
            obs = RS.observation_for(int(seed), t)
            ctx = enc.encode("pick up the object and place it on the target", obs)
            src = tr if t == 0 else traces[t - 1]
            prefix = []
            for i, st in enumerate(tr["steps"]):
                out.append((frame(g["config"], ctx.encoded, prefix, st["name"]), stable_digest("vision", obs),
                            st["tokens"]))
                prefix = prefix + src["steps"][i]["tokens"]
    return out


def _teacher_force_all(eng, reqs, max_rows):
    """Greedy token at every position of every request given the oracle's
    own prefix: the positions of a request are forked off one trunk and
    decoded as one-token branches, `max_rows` per tick."""
    agree = total = 0
    for ids, vseed, toks in reqs:
        full = list(ids) + list(toks)
        n0 = len(ids) - 1
        trunk = eng.seq_create()
        eng.prefill(trunk, full[: n0 + len(toks) - 1], vseed, M.VIS_ID)
        for c0 in range(0, len(toks), max_rows):
            pos = range(c0, min(len(toks), c0 + max_rows))
            forks = [eng.seq_fork(trunk, n0 + i) for i in pos]
            reqs_ = [eng.submit(b, full[n0 + i], 1, 1) for b, i in zip(forks, pos)]
            eng.set_slots(max(8, len(reqs_)))
            eng.run(-1)
            for r, i in zip(reqs_, pos):
                agree += eng.request_tokens(r, 1)[0] == toks[i]
                total += 1
                eng.request_release(r)
            for b in forks:
                eng.seq_free(b)
        eng.seq_free(trunk)
    return agree, total


@pytest.mark.parametrize("path", ["tick", "chain"])
def test_bf16_teacher_forced_golden_episodes(path):
    """bf16 token-match rate, teacher-forced, over every token of the golden
    7b_2layer episodes (~3k positions): the tick kernel (16 rows per tick)
    and the kernel chain (a request's positions in one wide tick)."""
    g = _traces()
    reqs = _golden_requests(g)
    eng = Engine("7b_2layer", dtype="bf16", seed=0, kv_pages=1024, max_rows=512)
    try:
        eng.set_option("mk", 1 if path == "tick" else 0)
        agree, total = _teacher_force_all(eng, reqs, 16 if path == "tick" else 128)
    finally:
        eng.close()
    rate = agree / total
    _record(f"teacher_forced_7b_2layer_episodes_{path}", {"positions": total, "argmax_agreement": rate})
    print("bf16 teacher-forced token-match", path, rate, total)
    assert rate >= TF_EPISODE_MIN, rate


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_7b_2layer_episodes_vs_oracle_traces(schema, dtype):
    """Reference `run_episode` (parallel_sync) over the engine vs the reference
    runners over the fp32 oracle: fp32 bit-exact; bf16 free-running
    token-match rate (greedy decode of a random-init model diverges at the
    first near-tie and never re-converges, so this rate is dominated by where
    the first divergence falls; the teacher-forced rate above is the
    per-position agreement)."""
    from ecot_sched.trace import trace_content_bytes
    g = _traces()
    be = EngineBackend("7b_2layer", dtype=dtype, seed=0, kv_pages=1024)
    same = total = 0
    first = []
    try:
        for seed, want in g["episodes"].items():
            res, _ = ecot_sched.run_episode(RS.SchedulerConfig(mode="parallel_sync", slots=8), g["T"], be,
                                            schema, seed=int(seed))
            got = [trace_content_bytes(r.trace, schema).decode() for r in res]
            if dtype == "f32":
                assert got == want, seed
            s, t, fd = _token_match(got, want)
            same, total, first = same + s, total + t, first + fd
    finally:
        be.close()
    if dtype == "bf16":
        rate = same / total
        _record("free_running_7b_2layer_episodes", {"tokens": total, "match_rate": rate, "rows_per_tick": "<= 7",
                                                      "median_first_divergence": float(np.median(first)),
                                                      "requests": len(first)})
        print("bf16 free-running token-match rate", rate, total, "median first divergence", np.median(first))
        assert rate >= FREE_RUN_MIN


def test_7b_2layer_batched_episodes_wide_rows_vs_oracle_traces(schema):
    """Config-4 path: every episode's branches in one batch (21 rows > 16: the
    kernel chain), bf16, free-running token-match rate vs the oracle traces."""
    from ecot_sched.trace import trace_content_bytes
    g = _traces()
    seeds = sorted(g["episodes"], key=int)
    be = EngineBackend("7b_2layer", dtype="bf16", seed=0, kv_pages=2048)
    try:
        drv = BatchedEpisodes(RS.SchedulerConfig(mode="parallel_sync", slots=8), be, schema, [int(s) for s in seeds])
        steps = [drv.step(t) for t in range(g["T"])]
    finally:
        be.close()
    same = total = 0
    first = []
    for e, seed in enumerate(seeds):
        got = [trace_content_bytes(steps[t][e].trace, schema).decode() for t in range(g["T"])]
        s, t, fd = _token_match(got, g["episodes"][seed])
        same, total, first = same + s, total + t, first + fd
    rate = same / total
    _record("free_running_7b_2layer_batched", {"tokens": total, "match_rate": rate, "rows_per_tick": len(seeds) * 7,
                                               "median_first_divergence": float(np.median(first))})
    print("bf16 batched free-running token-match rate", rate, total)
    assert rate >= FREE_RUN_MIN
