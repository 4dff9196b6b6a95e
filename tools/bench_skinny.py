"""Micro-benchmark of the tcgen05 skinny decode GEMM on 7B shapes (warm,
back-to-back launches, CUDA events on the engine stream)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_07639_b200.engine import Engine  # noqa: E402

eng = Engine("small", dtype="bf16", seed=0, kv_pages=8, max_rows=64)
import os
if os.environ.get("PDL"):
    eng.set_option("pdl", int(os.environ["PDL"]))
if os.environ.get("SK_STAGES"):
    eng.set_option("sk_stages", int(os.environ["SK_STAGES"]))
stream = torch.cuda.ExternalStream(eng.stream_handle())
shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "gate_up": (22016, 4096), "down": (4096, 11008),
          "lm_head": (32128, 4096), "big": (262144, 4096)}
for rows in (int(a) for a in (sys.argv[1:] or ["7"])):
    for name, (N, K) in shapes.items():
        w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        x = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
        y = torch.empty(rows, N, device="cuda")
        torch.cuda.synchronize()
        for _ in range(3):
            eng.op_skinny_tc(x.data_ptr(), w.data_ptr(), rows, N, K, y.data_ptr())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        eng.set_option("op_reps", reps)  # back-to-back launches inside one call: device-bound timing
        a.record(stream)
        eng.op_skinny_tc(x.data_ptr(), w.data_ptr(), rows, N, K, y.data_ptr())
        b.record(stream)
        eng.set_option("op_reps", 1)
        b.synchronize()
        us = a.elapsed_time(b) * 1000 / reps
        gbs = N * K * 2 / (us * 1e3)
        ref = x.float() @ w.float().T
        err = ((y - ref).abs().max() / ref.abs().max()).item()
        del w, ref
        print(f"rows {rows:3d} {name:8s} N={N:6d} K={K:6d}: {us:8.2f} us  {gbs:7.0f} GB/s  err {err:.1e}", flush=True)
eng.close()
