"""Generate the committed golden fixtures from the REFERENCE (run in the
build container, where /root/reference exists; the GPU box only reads the
JSON outputs).

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py --quick    # skip the 7b_2layer requests
    python tests/golden/make_golden.py --traces   # traces_tiny.json only

Fixtures:
  traces_tiny.json      golden ECoT traces: the reference's own runners
                        (SequentialRunner, ParallelSyncRunner, ParallelAsyncRunner,
                        KStepRunner, TwoTrackRunner; schedulers.py:363-716) over
                        the CPU oracle model (`tiny`,
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
from ecot_sched import schedulers as rs  # noqa: E402
from ecot_sched import trace as rt  # noqa: E402

from oracle.backend import OracleBackend, OracleModel, frame  # noqa: E402


def golden_traces(T: int = 10) -> dict:
    schema = rt.default_schema()
    model = OracleModel("tiny", seed=0)
    out = {"config": "tiny", "seed": 0, "T": T, "slots": 8, "modes": {}}
    for mode in ("sequential", "parallel_sync", "parallel_async", "k_step", "two_track"):
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
    ap.add_argument("--traces", action="store_true")
    args = ap.parse_args()
    (HERE / "traces_tiny.json").write_text(json.dumps(golden_traces()))
    print("traces_tiny.json", file=sys.stderr)
    if args.traces:
        return
    (HERE / "requests_small.json").write_text(json.dumps(golden_requests("small", 12, 4)))
    if not args.quick:
        (HERE / "requests_7b_2layer.json").write_text(json.dumps(golden_requests("7b_2layer", 6, 2)))


if __name__ == "__main__":
    main()
