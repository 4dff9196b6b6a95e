"""Micro-benchmark of the tcgen05 decode GEMMs on 7B shapes (warm,
back-to-back launches, CUDA events on the engine stream): the persistent
swap-AB skinny GEMM at every K split, and the tile GEMM, per row count.

    python tools/bench_skinny.py ROWS... [--splits 0,1,2,4,8] [--tile]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_07639_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("rows", nargs="*", type=int, default=[7])
ap.add_argument("--splits", default="0")
ap.add_argument("--tile", action="store_true", help="also time the tile GEMM")
ap.add_argument("--shapes", default="qkv,o,gate_up,down,lm_head")
args = ap.parse_args()

eng = Engine("small", dtype="bf16", seed=0, kv_pages=8, max_rows=512)
stream = torch.cuda.ExternalStream(eng.stream_handle())
shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "gate_up": (22016, 4096), "down": (4096, 11008),
          "lm_head": (32128, 4096)}


def timed(fn, reps=30):
    for _ in range(2):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.set_option("op_reps", reps)  # back-to-back launches inside one call: device-bound timing
    a.record(stream)
    fn()
    b.record(stream)
    eng.set_option("op_reps", 1)
    b.synchronize()
    return a.elapsed_time(b) * 1000 / reps


for rows in args.rows:
    for name in args.shapes.split(","):
        N, K = shapes[name]
        w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        x = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
        y = torch.empty(rows, N, device="cuda")
        ref = x.float() @ w.float().T
        torch.cuda.synchronize()
        line = f"rows {rows:3d} {name:8s} N={N:6d} K={K:6d}:"
        for sp in (int(v) for v in args.splits.split(",")):
            eng.set_option("sk_splits", sp)
            us = timed(lambda: eng.op_skinny_tc(x.data_ptr(), w.data_ptr(), rows, N, K, y.data_ptr()))
            err = ((y - ref).abs().max() / ref.abs().max()).item()
            assert err < 1e-4, err
            line += f"  sk{sp}: {us:7.1f}us {N * K * 2 / (us * 1e3):5.0f}GB/s"
        eng.set_option("sk_splits", 0)
        if args.tile:
            us = timed(lambda: eng.op_gemm_tc(x.data_ptr(), w.data_ptr(), rows, N, K, y.data_ptr()))
            err = ((y - ref).abs().max() / ref.abs().max()).item()
            line += f"  tile: {us:7.1f}us {2 * rows * N * K / (us * 1e6):6.0f}TF/s"
        print(line, flush=True)
        del w, ref
eng.close()
