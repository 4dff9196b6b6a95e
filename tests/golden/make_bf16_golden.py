"""fp32 CPU-oracle golden vectors that pin the benchmarked bf16 path
(run in the build container; the GPU box only reads the outputs).

    python tests/golden/make_bf16_golden.py [--configs 7b_2layer 7b] [--traces]

tf_<config>.npz -- teacher-forced requests at the benchmark's shapes: a framed
    Fast-ECoT branch input (BOS + 256 vision rows + 16 context ids + a
    ~300-token reasoning prefix + step tag) and the oracle's first N greedy
    tokens; for every generated position the oracle logits of the first
    LOGIT_COLS vocabulary columns and its top-5 (ids, values).  The GPU test
    feeds the oracle's tokens (teacher forcing), so every position is
    compared on identical inputs.
traces_<config>.json -- free-running golden traces from the REFERENCE runners
    (`ecot_sched` run_episode, parallel_sync, 8 slots) over the oracle for a
    few seeds: the bf16 token-match rate of whole episodes is measured
    against these.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402
from ecot_sched import backends as rb  # noqa: E402  (the reference)
from ecot_sched import schedulers as rs  # noqa: E402
from ecot_sched import trace as rt  # noqa: E402

from oracle.backend import OracleBackend, OracleModel, frame  # noqa: E402

LOGIT_COLS = 2048
INSTR = "pick up the object and place it on the target"


def teacher_forced(config: str, cases: int, n_out: int) -> dict:
    model = OracleModel(config, seed=0)
    rng = np.random.default_rng(2025)
    out = {"ids": [], "vseed": [], "tokens": [], "logits_head": [], "top5_ids": [], "top5_val": []}
    for c in range(cases):
        obs = rs.observation_for(100 + c, c)
        ctx = rb.SyntheticBackend(rb.default_profile(0)).encode(INSTR, obs)
        prefix = [int(t) for t in rng.integers(0, 2**32, size=int(rng.integers(250, 350)))]
        step = ("visible_objects", "plan", "action")[c % 3]
        ids = frame(config, ctx.encoded, prefix, step)
        vseed = rb.stable_digest("vision", obs)
        t0 = time.time()
        toks, logits = model.generate(ids, vseed, n_out, want_logits=True)
        top = np.argsort(-logits[:, :32000], axis=1, kind="stable")[:, :5]
        out["ids"].append(np.asarray(ids, np.int32))
        out["vseed"].append(vseed)
        out["tokens"].append(np.asarray(toks, np.int32))
        out["logits_head"].append(logits[:, :LOGIT_COLS].astype(np.float32))
        out["top5_ids"].append(top.astype(np.int32))
        out["top5_val"].append(np.take_along_axis(logits, top, axis=1).astype(np.float32))
        print(f"  {config} case {c}: {len(ids)} ids -> {toks} ({time.time() - t0:.0f} s)", file=sys.stderr)
    L = max(len(i) for i in out["ids"])
    ids = np.full((cases, L), -1, np.int32)
    for c, i in enumerate(out["ids"]):
        ids[c, : len(i)] = i
    return {"ids": ids, "n_ids": np.asarray([len(i) for i in out["ids"]], np.int32),
            "vseed": np.asarray(out["vseed"], np.uint64), "tokens": np.stack(out["tokens"]),
            "logits_head": np.stack(out["logits_head"]), "top5_ids": np.stack(out["top5_ids"]),
            "top5_val": np.stack(out["top5_val"])}


def traces(config: str, seeds, T: int) -> dict:
    schema = rt.default_schema()
    model = OracleModel(config, seed=0)
    out = {"config": config, "T": T, "mode": "parallel_sync", "slots": 8, "episodes": {}}
    for s in seeds:
        t0 = time.time()
        be = OracleBackend(config, seed=0, model=model)
        res, _ = rs.run_episode(rs.SchedulerConfig(mode="parallel_sync", slots=8), T, be, schema, seed=s)
        out["episodes"][str(s)] = [rt.trace_content_bytes(r.trace, schema).decode() for r in res]
        print(f"  {config} traces seed {s}: {time.time() - t0:.0f} s", file=sys.stderr)
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["7b_2layer", "7b"])
    ap.add_argument("--cases", type=int, default=3)
    ap.add_argument("--n-out", type=int, default=8)
    ap.add_argument("--traces", action="store_true", help="also the free-running 7b_2layer traces")
    args = ap.parse_args()
    for cfg in args.configs:
        np.savez(HERE / f"tf_{cfg}.npz", **teacher_forced(cfg, args.cases, args.n_out))
    if args.traces:
        (HERE / "traces_7b_2layer.json").write_text(json.dumps(traces("7b_2layer", [0, 1, 2], 3)))


if __name__ == "__main__":
    main()
