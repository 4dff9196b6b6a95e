"""Config-3 action-latency breakdown (diagnostics): the reference
ParallelAsyncRunner (lockstep landing order) over the 7B bf16 engine; per
timestep the device ms, engine decode ticks, forwards, prefill rows and the
CUDA-event time of prefill forwards vs decode ticks."""

import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2506_07639_b200.engine_backend import EngineBackend  # noqa: E402  (resolves ecot_sched)
from paper_2506_07639_b200.workloads import WORKLOADS  # noqa: E402
from ecot_sched import schedulers as RS  # noqa: E402
from ecot_sched.schedulers import observation_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="7b")
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--mode", default="parallel_async")
ap.add_argument("--async-mode", default="lockstep")
args = ap.parse_args()

make_schema, make_profile = WORKLOADS["config2"]
schema = make_schema()
kw = {} if args.async_mode == "lockstep" else {"async_mode": args.async_mode}
be = EngineBackend(args.config, dtype="bf16", seed=0, device=0, profile=make_profile(0), **kw)
eng = be.engine
stream = torch.cuda.ExternalStream(eng.stream_handle())
runner = RS.make_runner(RS.SchedulerConfig(mode=args.mode, slots=8, wall_clock=True), be, schema)
INSTR = "pick up the object and place it on the target"
rows = []
for t in range(args.steps):
    s0 = eng.stats()
    eng.profile(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    runner.step(be.encode(INSTR, observation_for(7, t)), t)
    b.record(stream)
    b.synchronize()
    p = eng.profile_read()
    eng.profile(False)
    s1 = eng.stats()
    d = {k: s1[k] - s0[k] for k in ("ticks", "forwards", "rows")}
    rows.append((a.elapsed_time(b), d, p))
    print(f"t={t}: {a.elapsed_time(b):7.2f} ms  ticks {d['ticks']:3d} forwards {d['forwards']:3d} rows {d['rows']:5d} | "
          + "  ".join(f"{k} {v['ms']:.2f}ms/{v['launches']}" for k, v in p.items() if v["launches"]), flush=True)
print("p50", statistics.median(r[0] for r in rows[1:]))
