"""Generate the committed golden fixtures from the REFERENCE (run in the
build container, where /root/reference exists; the GPU box only reads the
JSON outputs).

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py --quick    # skip the 7b_2layer requests

Fixtures:
  mirror_vectors.json   reference outputs for the host-side mirror
                        (stable_digest, context encoding, SyntheticBackend draws,
                        decode_action, trace bytes, continuous_batch / Fig. 5 KATs)
  traces_tiny.json      golden ECoT traces: the reference's own runners
                        (SequentialRunner, ParallelSyncRunner, ParallelAsyncRunner;
                        schedulers.py:363-552) over the CPU oracle model (`tiny`,
                        fp32), BASELINE config 1: T=10, seed 0, default schema and
                        profile, 8 slots.  Lines are `trace_content_bytes`.
  requests_<cfg>.json   per-request greedy tokens of the oracle model for
                        `small` and `7b_2layer` shapes (framed ids + vision seed)
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
REF_SRC = Path("/root/reference/pkg/src")

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402
from ecot_sched import backends as rb  # noqa: E402  (the reference)
from ecot_sched import batching as rbat  # noqa: E402
from ecot_sched import schedulers as rs  # noqa: E402
from ecot_sched import trace as rt  # noqa: E402

from oracle.backend import OracleBackend, OracleModel, frame  # noqa: E402


def mirror_vectors() -> dict:
    out: dict = {}
    out["stable_digest"] = [
        {"parts": ["encode", "task", "b:0102"], "digest": rb.stable_digest("encode", "task", b"\x01\x02")},
        {"parts": ["step", 7, 123456789, "plan"], "digest": rb.stable_digest("step", 7, 123456789, "plan")},
        {"parts": ["vision", "b:" + "ab" * 24], "digest": rb.stable_digest("vision", bytes.fromhex("ab" * 24))},
    ]
    out["observation_for"] = [{"seed": s, "t": t, "hex": rs.observation_for(s, t).hex()}
                              for s in (0, 7, 63) for t in (0, 1, 99)]
    enc = []
    for instr, obs in [("pick up the object and place it on the target", rs.observation_for(0, 3)),
                       ("", b""), ("lift the cup", b"\x01\x02")]:
        enc.append({"instruction": instr, "observation": obs.hex(), "encoded": list(rb._encode_tokens(instr, obs))})
    out["encode"] = enc
    # SyntheticBackend draws (lengths, truncation, reuse and token ids)
    schema = rt.default_schema()
    draws = []
    for seed in (0, 5):
        be = rb.SyntheticBackend(rb.default_profile(seed))
        for t in range(4):
            ctx = be.encode("pick up the object and place it on the target", rs.observation_for(seed, t))
            for spec in schema.steps:
                prev = tuple(range(3 + t)) if t % 2 else ()
                g = be.begin_step(ctx, (1, 2, 3), spec, prev)
                draws.append({"seed": seed, "t": t, "step": spec.name, "prev": list(prev),
                              "tokens": list(g.tokens), "truncated": g.truncated})
    trunc = rb.SyntheticBackend(rb.SyntheticProfile({"task": rb.StepProfile(500, 0, 1.0)}, seed=1))
    g = trunc.begin_step(trunc.encode("i", b"o"), (), schema.steps[0], ())
    draws.append({"seed": -1, "t": 0, "step": "task", "prev": [], "tokens": list(g.tokens),
                  "truncated": g.truncated, "profile": "truncation"})
    out["synthetic_draws"] = draws
    out["decode_action"] = [{"tokens": toks, "dim": dim,
                             "components": list(rs.decode_action(tuple(toks), dim).components)}
                            for toks, dim in [([0, 1, 65535, 65536, 32768, 12345, 4294967295], 7),
                                              ([100, 200], 7), ([31999, 0, 17], 3)]]
    tr = rt.ReasoningTrace(3, (("task", (1, 2)), ("plan", ()), ("action", (5, 6, 7))),
                           rt.ActionVector((0.5, -0.25, 1e-7)))
    out["trace_bytes"] = {"content": rt.trace_content_bytes(tr, schema).decode(),
                          "serialized": rt.serialize_trace(tr, schema, wall_ms=12.5).decode()}
    reqs = [rbat.GenerationRequest(i, i, 0, L) for i, L in enumerate((3, 6, 8, 9))]
    cb = rbat.continuous_batch(reqs, 4)
    sb = rbat.static_batch(reqs, 4, pad_to=11)
    lm = rbat.LatencyModel(c_iter=10, c_slot=1, c_encode=20, c_decode=5)
    out["batching"] = {
        "fig5_continuous_busy": cb.busy_slot_iterations, "fig5_static_occupied": sb.occupied_slot_iterations,
        "fig5_waste": rbat.padding_waste(sb), "fig5_cost": rbat.schedule_cost(cb, lm),
        "fig5_makespan": cb.makespan, "fig5_grid": cb.grid.tolist(),
    }
    mixed = [rbat.GenerationRequest(0, 0, 0, 5), rbat.GenerationRequest(1, 1, 0, 7, priority=rbat.ACTION),
             rbat.GenerationRequest(2, 2, 0, 3, arrival_iteration=2), rbat.GenerationRequest(3, 3, 0, 4)]
    out["batching"]["mixed_grid"] = rbat.continuous_batch(mixed, 2).grid.tolist()
    return out


def golden_traces(T: int = 10) -> dict:
    schema = rt.default_schema()
    model = OracleModel("tiny", seed=0)
    out = {"config": "tiny", "seed": 0, "T": T, "slots": 8, "modes": {}}
    for mode in ("sequential", "parallel_sync", "parallel_async"):
        backend = OracleBackend("tiny", seed=0, model=model)
        cfg = rs.SchedulerConfig(mode=mode, slots=8)
        results, summary = rs.run_episode(cfg, T, backend, schema, seed=0)
        out["modes"][mode] = {
            "lines": [rt.trace_content_bytes(r.trace, schema).decode() for r in results],
            "latency_ms": [r.latency_ms for r in results],
            "staleness": [r.staleness for r in results],
            "generated_tokens": [r.generated_tokens for r in results],
            "failures": [list(r.failures) for r in results],
            "requests": backend.requests,
        }
        print(f"  {mode}: {backend.requests} oracle requests", file=sys.stderr)
    return out


def golden_requests(config: str, n_out: int, cases: int) -> dict:
    model = OracleModel(config, seed=0)
    rng = np.random.default_rng(11)
    out = {"config": config, "seed": 0, "cases": []}
    for c in range(cases):
        obs = rs.observation_for(c, c + 1)
        encoded = rb._encode_tokens("pick up the object and place it on the target", obs)
        prefix = [int(t) for t in rng.integers(0, 32000, size=int(rng.integers(0, 90)))]
        step = ("task", "plan", "action")[c % 3]
        ids = frame(config, encoded, prefix, step)
        vseed = rb.stable_digest("vision", obs)
        toks, logits = model.generate(ids, vseed, n_out, want_logits=True)
        out["cases"].append({"ids": ids, "vseed": vseed, "n_out": n_out, "tokens": toks,
                             "logits_head": logits[:, :8].tolist(),
                             "logits_argmax_value": [float(logits[i, t]) for i, t in enumerate(toks)]})
        print(f"  {config} case {c}: {len(ids)} ids -> {toks}", file=sys.stderr)
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    (HERE / "mirror_vectors.json").write_text(json.dumps(mirror_vectors()))
    print("mirror_vectors.json", file=sys.stderr)
    (HERE / "traces_tiny.json").write_text(json.dumps(golden_traces()))
    print("traces_tiny.json", file=sys.stderr)
    (HERE / "requests_small.json").write_text(json.dumps(golden_requests("small", 12, 4)))
    if not args.quick:
        (HERE / "requests_7b_2layer.json").write_text(json.dumps(golden_requests("7b_2layer", 6, 2)))


if __name__ == "__main__":
    main()
