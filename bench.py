#!/usr/bin/env python
"""Fast-ECoT on B200: policy steps/s of a 7B-shaped ECoT VLA.

    python bench.py [--gpus N --steps K --warmup W] [--impl engine|reference]

Workload (BASELINE.json config 2, 1 GPU): Llama-2-7B-shaped decoder + 256
vision tokens, random-init bf16 weights, synthetic LIBERO-shaped
observations (`observation_for(seed, t)`), default ECoT schema/profile; one
episode per GPU driven by the Fast-ECoT runner (`parallel_sync`: trunk
prefill + 7 forked branches decoded as one batch).  A *step* is one control
timestep.  `value` = policy steps/s over all ranks (device time, CUDA events
on the engine stream, max over ranks); `e2e` = the same through the public
runner API with host wall clock (all H2D/D2H inside).  Sequential ECoT and
async action latency are reported alongside.  Every decode iteration streams
13.2 GB of weights (> L2), so no L2 flush is needed between steps.

Multi-GPU: one process per GPU (torchrun); each rank runs an independent
episode (seed = rank) on its own engine; NCCL is used only to gather the
per-rank results at the end ("scaling": "weak").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "p50 per-step ECoT latency (ms) and policy steps/s, 7B-shaped VLA, 1/2/4/8 B200"
INSTRUCTION = "pick up the object and place it on the target"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("engine", "reference"), default="engine")
    ap.add_argument("--config", default="7b")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--mode", default="parallel_sync")
    ap.add_argument("--workload", choices=("config2", "stress"), default="config2",
                    help="config2: default ECoT schema; stress: config 5 (8-way fan-out, ~2k-token cached prefix)")
    ap.add_argument("--episodes", type=int, default=1,
                    help="total episodes (config 4: >1 shards them over ranks, batched per timestep)")
    ap.add_argument("--seq-steps", type=int, default=2)
    ap.add_argument("--async-steps", type=int, default=10)
    ap.add_argument("--no-extras", action="store_true", help="skip sequential/async side measurements")
    ap.add_argument("--profile-steps", type=int, default=3, help="eager timesteps timed per kernel after the run")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--out", default=None, help="also write the JSON line here")
    return ap.parse_args()


# --------------------------------------------------------------------------
def dist_setup(backend: str):
    from paper_2506_07639_b200.distributed import init_from_env
    return init_from_env(backend)


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def all_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_objects(obj, world):
    from paper_2506_07639_b200.distributed import gather_to_all
    return gather_to_all(obj, world)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        rows = []
        for line in open(self.path).read().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in rows for n, v in zip(names, r[4:8]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max((float(r[2]) for r in rows if r[2].replace(".", "").isdigit()), default=None)}


def measured_peaks() -> dict:
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops_sustained"], "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


def ncu_traffic(name: str = "ncu_decode_gemv.json") -> float | None:
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    p = REPO / "profiles" / name
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except (ValueError, OSError):
            return None
    return None


# --------------------------------------------------------------------------
def workload_shapes(config: str, seed: int, warmup: int, steps: int, mode: str = "parallel_sync"):
    """Per timed step: (trunk tokens to prefill, decode tokens) of the ECoT
    workload.  Lengths come from the synthetic length oracle only, so the
    shape is known without running the model (it equals the engine's)."""
    from paper_2506_07639_b200 import schedulers as S
    from paper_2506_07639_b200.backends import SyntheticBackend, default_profile
    from paper_2506_07639_b200.model import get_config
    from paper_2506_07639_b200.trace import default_schema
    cfg = get_config(config)
    ctx_len = 1 + cfg.n_vision + 16
    schema = default_schema()
    be = SyntheticBackend(default_profile(seed))
    runner = S.make_runner(S.SchedulerConfig(mode=mode, slots=8), be, schema)
    shapes, prev = [], None
    for t in range(warmup + steps):
        r = runner.step(be.encode(INSTRUCTION, S.observation_for(seed, t)), t)
        if t >= warmup:
            lens = [len(toks) for _, toks in r.trace.steps]
            if mode == "parallel_sync" and prev is not None:
                trunk = ctx_len + sum(len(toks) for _, toks in prev.steps[:-1])
            else:  # sequential chain: context + every step but the last is prefilled
                trunk = ctx_len + sum(lens[:-1])
            shapes.append((trunk, sum(lens)))
        prev = r.trace
    return shapes


def cpu_sample(config: str, threads: int) -> dict:
    """Time the CPU oracle (fp32, canonical arithmetic, all host threads) on a
    bounded sample of the same model shape: one 48-token prefill and 3 decode
    tokens.  Falls back to the 2-layer 7B shape scaled by depth when host RAM
    cannot hold the 26 GB fp32 7B model."""
    from oracle.backend import OracleModel, SHAPES
    mem_gb = 0.0
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable"):
                mem_gb = int(line.split()[1]) / 1e6
    except OSError:
        pass
    use, scale = config, 1.0
    if config == "7b" and mem_gb < 80:
        use, scale = "7b_2layer", SHAPES["7b"][1] / SHAPES["7b_2layer"][1]
    t0 = time.perf_counter()
    om = OracleModel(use, seed=0, threads=threads)
    init_s = time.perf_counter() - t0
    ids = [32000] + [32001] * 16 + list(range(100, 131))       # 48 ids
    t0 = time.perf_counter()
    om.generate(ids, 1, 1)                                      # prefill 48 + 1 head
    t_pre = time.perf_counter() - t0
    t0 = time.perf_counter()
    om.generate(ids, 1, 4)                                      # cached prefix: 1 row + 3 decode tokens
    t_dec = (time.perf_counter() - t0) / 4.0
    per_prefill = (t_pre - t_dec) / 47.0
    return {"model": use, "depth_scale": scale, "prefill_s_per_token": per_prefill * scale,
            "decode_s_per_token": t_dec * scale, "init_s": init_s, "threads": threads, "mem_gb": mem_gb}


def extrapolate_ms(sample: dict, shape) -> float:
    trunk, dec = shape
    return 1000.0 * (trunk * sample["prefill_s_per_token"] + dec * sample["decode_s_per_token"])


# --------------------------------------------------------------------------
def run_reference(args, rank, world):
    """Reference arm: the reference's CPU path for this workload -- the
    reference runners (baseline/_ref when installed, else the mirror) over
    the CPU oracle model -- timed on the host cores in a bounded sample."""
    if rank != 0:
        return None
    threads = os.cpu_count() or 1
    ref_runner = "mirror"
    try:
        sys.path.insert(0, str(REPO / "baseline" / "_ref"))
        os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
        import ecot_sched  # noqa: F401
        ref_runner = "reference (baseline/_ref)"
    except Exception:
        pass
    sample = cpu_sample(args.config, threads)
    shapes = workload_shapes(args.config, 0, args.warmup, args.steps, args.mode)
    ms = [extrapolate_ms(sample, s) for s in shapes]
    value = 1000.0 / statistics.mean(ms)
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(ms),
        "p50_ms": statistics.median(ms), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": "config 2: 7B-shaped ECoT VLA, single episode, Fast ECoT parallel_sync",
                   "model": args.config, "mode": args.mode},
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": threads, "kind": "port",
                         "sample": (f"CPU oracle ({sample['model']}, fp32, {threads} threads): 47-token prefill "
                                    f"+ 4 decode tokens timed, extrapolated to each step's trunk and branch "
                                    f"lengths (depth x{sample['depth_scale']:.0f}); runners: {ref_runner}")},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "detail": sample,
    }
    return line


def time_mode(backend, runner, seed, t0, n, stream):
    """Run n timesteps from t0; returns per-step (device ms, host ms, results).
    `runner` is a reference-style runner (one episode, `seed`) or a
    `BatchedEpisodes` driver (all its episodes per step)."""
    import torch
    from paper_2506_07639_b200.schedulers import BatchedEpisodes, observation_for
    dev, host, results = [], [], []
    for t in range(t0, t0 + n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        h0 = time.perf_counter()
        if isinstance(runner, BatchedEpisodes):
            results.append(runner.step(t))
        else:
            results.append(runner.step(backend.encode(INSTRUCTION, observation_for(seed, t)), t))
        host.append((time.perf_counter() - h0) * 1000.0)
        b.record(stream)
        b.synchronize()
        dev.append(a.elapsed_time(b))
    return dev, host, results


def run_engine(args, rank, world, local):
    import torch
    from paper_2506_07639_b200 import schedulers as S
    from paper_2506_07639_b200.engine_backend import EngineBackend
    from paper_2506_07639_b200.trace import default_schema

    from paper_2506_07639_b200.workloads import WORKLOADS
    torch.cuda.set_device(local)
    make_schema, make_profile = WORKLOADS[args.workload]
    schema = make_schema()
    seed = rank
    backend = EngineBackend(args.config, dtype=args.dtype, seed=0, device=local, profile=make_profile(0))
    eng = backend.engine
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=local)
    cfg_run = S.SchedulerConfig(mode=args.mode, slots=8, wall_clock=True)
    if args.episodes > 1:  # config 4: this rank's shard of the episodes, one batch per timestep
        from paper_2506_07639_b200.distributed import shard_episodes
        local_seeds = shard_episodes(list(range(args.episodes)), world, rank)
        runner = S.BatchedEpisodes(cfg_run, backend, schema, local_seeds)
    else:
        runner = S.make_runner(cfg_run, backend, schema)

    # warm-up (t=0 is the reference's sequential warm-up pass); decode ticks
    # of each row count are captured into CUDA graphs during warm-up
    time_mode(backend, runner, seed, 0, args.warmup, stream)
    eng.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    stats0 = eng.stats()
    clocks = ClockSampler(local)
    clocks.start()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(stream)
    h0 = time.perf_counter()
    dev, host, results = time_mode(backend, runner, seed, args.warmup, args.steps, stream)
    host_total = time.perf_counter() - h0
    end.record(stream)
    eng.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    stats1 = eng.stats()
    total_s = start.elapsed_time(end) / 1000.0
    total_max = all_max(total_s, world)
    host_max = all_max(host_total, world)

    # per-kernel CUDA-event timing (eager launches, events around every decode
    # GEMM / attention launch on the engine stream) over the next timesteps
    eng.profile(True)
    pdev, _, _ = time_mode(backend, runner, seed, args.warmup + args.steps, args.profile_steps, stream)
    prof = eng.profile_read()
    eng.profile(False)
    prof["steps"] = args.profile_steps
    prof["step_ms"] = sum(pdev)

    extras = {}
    if world == 1 and not args.no_extras and args.episodes <= 1:
        seq_runner = S.make_runner(S.SchedulerConfig(mode="sequential", slots=8, wall_clock=True), backend, schema)
        sdev, shost, _ = time_mode(backend, seq_runner, 1000 + seed, 0, 1 + args.seq_steps, stream)
        asy = S.make_runner(S.SchedulerConfig(mode="parallel_async", slots=8, wall_clock=True), backend, schema)
        adev, ahost, ares = time_mode(backend, asy, 2000 + seed, 0, 1 + args.async_steps, stream)
        asy.engine.drain()  # land the lockstep runner's in-flight reasoning before the engine is reused
        # config 3 proper: two CUDA streams, reasoning refresh free-running on the
        # low-priority lane between and during control steps
        backend2 = EngineBackend(args.config, dtype=args.dtype, seed=0, device=local, profile=make_profile(0),
                                 engine=backend.engine, async_streams=2)
        asy2 = S.make_runner(S.SchedulerConfig(mode="parallel_async", slots=8, wall_clock=True), backend2, schema)
        a2dev, a2host, a2res = time_mode(backend2, asy2, 3000 + seed, 0, 1 + args.async_steps, stream)
        asy2.engine.drain()
        asy2.engine.close()
        stal = [max(v for k, v in r.staleness.items() if k != schema.action_step.name) for r in a2res[1:]]
        extras = {
            "sequential_ms": {"p50": statistics.median(sdev[1:]), "steps": len(sdev) - 1,
                              "all": [round(x, 2) for x in sdev[1:]]},
            "parallel_async_action_ms": {"p50": statistics.median(adev[1:]),
                                         "p99": sorted(adev[1:])[max(0, int(0.99 * (len(adev) - 1)) - 1)],
                                         "steps": len(adev) - 1, "scheduler": "lockstep (reference landing order)"},
            "parallel_async_2stream_action_ms": {"p50": statistics.median(a2host[1:]),
                                                 "p99": sorted(a2host[1:])[max(0, int(0.99 * (len(a2host) - 1)) - 1)],
                                                 "steps": len(a2host) - 1,
                                                 "max_reasoning_staleness_p50": statistics.median(stal),
                                                 "scheduler": "two CUDA streams, host wall clock per action"},
        }
    gathered = gather_objects({"rank": rank, "dev_ms": dev, "host_ms": host}, world)
    return backend, dict(dev=dev, host=host, results=results, total_max=total_max, host_max=host_max,
                         prof=prof, clocks=clk, stats0=stats0, stats1=stats1, extras=extras, gathered=gathered)


def main():
    args = parse()
    if args.impl == "reference":
        rank, world, local = dist_setup("gloo")
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
            if args.out:
                Path(args.out).write_text(json.dumps(line) + "\n")
        return

    import torch
    rank, world, local = dist_setup("nccl")
    backend, r = run_engine(args, rank, world, local)
    K = args.steps
    peaks = measured_peaks()
    prof = r["prof"]
    # dominant kernel: the persistent decode-tick kernel (one launch per decode
    # iteration: all layers' weights + the staged KV) when it ran, else the
    # per-matrix decode GEMMs of the kernel chain
    tick = prof.get("decode_tick", {"ms": 0.0, "launches": 0, "bytes": 0.0})
    use_tick = tick["launches"] > 0
    g = tick if use_tick else prof["decode_gemv"]
    achieved = (g["bytes"] / 1e9) / (g["ms"] / 1e3) if g["ms"] > 0 else None
    steps_prof = prof.pop("steps")
    step_ms_prof = prof.pop("step_ms")
    dev_sorted = sorted(d for gr in r["gathered"] for d in gr["dev_ms"])
    p50 = statistics.median(dev_sorted)
    p99 = dev_sorted[min(len(dev_sorted) - 1, int(round(0.99 * (len(dev_sorted) - 1))))]
    s0, s1 = r["stats0"], r["stats1"]
    eps = max(1, args.episodes) if args.episodes > 1 else world  # episodes across all ranks
    value = eps * K / r["total_max"]
    e2e = eps * K / r["host_max"]
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.episodes <= 1:
        try:
            threads = os.cpu_count() or 1
            sample = cpu_sample(args.config, threads)
            shapes = workload_shapes(args.config, 0, args.warmup, K, args.mode)
            ms = statistics.mean(extrapolate_ms(sample, s) for s in shapes)
            cpu = {"value": 1000.0 / ms, "unit": "steps/s", "cores": threads, "kind": "port",
                   "sample": (f"CPU oracle ({sample['model']}, fp32, {threads} threads): 47-token prefill + 4 "
                              f"decode tokens timed, extrapolated to the timed steps' trunk/branch lengths "
                              f"(depth x{sample['depth_scale']:.0f}); {ms:.0f} ms/step")}
        except Exception as exc:  # the baseline must never sink the GPU line
            cpu = {"value": None, "unit": "steps/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc!r}"}
    if rank != 0:
        return
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "steps/s" if args.episodes <= 1 else "episode-steps/s",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 * r["total_max"] / K,
        "p50_ms": p50,
        "p99_ms": p99,
        "higher_is_better": True,
        "scaling": "weak" if args.episodes <= 1 else "strong",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic",
        "config": {"workload": ("config 2: 7B-shaped ECoT VLA (Llama-2-7B decoder + 256 vision tokens), "
                                "random-init weights, one episode per GPU, Fast ECoT parallel_sync")
                               if args.episodes <= 1 else
                               (f"config 4: batched rollouts of {args.episodes} independent episodes sharded "
                                f"over {world} GPU(s), 7B-shaped, Fast ECoT parallel_sync, one decode batch "
                                f"per timestep per GPU"),
                   "model": args.config, "mode": args.mode, "schema": args.workload,
                   "episodes": args.episodes if args.episodes > 1 else world,
                   "episodes_per_gpu": (args.episodes / world) if args.episodes > 1 else 1, "slots": 8,
                   "l2": "no flush: every decode iteration streams 13.2 GB of weights (> 126 MB L2)"},
        "e2e": {"value": e2e, "unit": "steps/s",
                "h2d_bytes_per_step": (s1["h2d_bytes"] - s0["h2d_bytes"]) / K,
                "d2h_bytes_per_step": (s1["d2h_bytes"] - s0["d2h_bytes"]) / K},
        "gpu_launches": s1["launches"] - s0["launches"],
        "roofline": {"bound": "hbm",
                     "kernel": ("persistent decode-tick kernel (decode_mk_kernel: every layer's QKV/O/gate-up/down "
                                "+ lm_head weights and the cascade-attention KV pages, one launch per tick)")
                               if use_tick else "decode GEMV (QKV/O/gate-up/down/lm_head, bf16 weights)",
                     "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": (achieved / peaks["hbm_gbs"]) if achieved else None, "traffic": ncu_traffic("ncu_decode_tick.json" if use_tick else "ncu_decode_gemv.json"),
                     "peak_source": peaks["source"],
                     "launches": g["launches"], "ms_total": g["ms"],
                     "share_of_step": g["ms"] / step_ms_prof,
                     "measured_on": f"{steps_prof} eager timesteps right after the timed region, CUDA events "
                                    f"around each {'decode-tick' if use_tick else 'decode GEMM'} launch on the "
                                    f"engine stream",
                     "bytes_per_launch": g["bytes"] / max(1, g["launches"])},
        "cpu_baseline": cpu,
        "clocks": r["clocks"],
        "breakdown_ms_per_step_eager": {k: v["ms"] / steps_prof for k, v in prof.items()},
        "decode_ticks_per_step": (s1["ticks"] - s0["ticks"]) / K,
        **r["extras"],
    }
    print(json.dumps(line), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(line) + "\n")
    backend.close()


if __name__ == "__main__":
    main()
