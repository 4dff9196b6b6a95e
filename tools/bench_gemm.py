"""Micro-benchmark of the dense-contraction tcgen05 GEMMs on 7B shapes (warm,
back-to-back launches inside one call, CUDA events on the engine stream):
the CTA-pair persistent GEMM (with and without split-K for one-m-tile
batches)
against the round-1 1-CTA 128 x 128 tile GEMM, per row count.

    python tools/bench_gemm.py [ROWS...] [--shapes qkv,o,gate_up,down]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_07639_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("rows", nargs="*", type=int, default=[33, 48, 96, 168, 256, 448, 625, 1024, 8192])
ap.add_argument("--shapes", default="qkv,o,gate_up,down")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--out", default=None)
ap.add_argument("--sk", type=lambda v: [int(x) for x in v.split(",") if x], default=[],
                help="extra variants with engine option tc_sk = each value")
ap.add_argument("--force-splits", type=lambda v: [int(x) for x in v.split(",") if x], default=[])
args = ap.parse_args()

eng = Engine("7b_2layer", dtype="bf16", seed=0, kv_pages=8, max_rows=64)  # 7B-sized split-K planes
stream = torch.cuda.ExternalStream(eng.stream_handle())
shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "gate_up": (22016, 4096), "down": (4096, 11008)}


def timed(fn, reps):
    for _ in range(2):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.set_option("op_reps", reps)
    a.record(stream)
    fn()
    b.record(stream)
    eng.set_option("op_reps", 1)
    b.synchronize()
    return a.elapsed_time(b) * 1000 / reps


results = []
for rows in args.rows:
    for name in args.shapes.split(","):
        N, K = shapes[name]
        w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        x = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
        y = torch.empty(rows, N, device="cuda")
        ref = x.float() @ w.float().T
        torch.cuda.synchronize()
        line = f"rows {rows:5d} {name:8s} N={N:6d} K={K:6d}:"
        rec = {"rows": rows, "shape": name, "N": N, "K": K}
        variants = [("v1", 0, 0, 0), ("pair_nosplit", 1, 0, 0), ("pair", 1, 1, 0)]
        variants += [(f"split{k}", 1, k, 0) for k in args.force_splits]
        variants += [(f"sk{k}", 1, 1, k) for k in args.sk]
        for label, pair, split, sk in variants:
            eng.set_option("tc_pair", pair)
            eng.set_option("tc_split", split)
            eng.set_option("tc_sk", sk)
            y.fill_(float("nan"))
            us = timed(lambda: eng.op_gemm_tc(x.data_ptr(), w.data_ptr(), rows, N, K, y.data_ptr()), args.reps)
            err = ((y - ref).abs().max() / ref.abs().max()).item()
            assert err < 1e-4, (label, err)
            tf = 2 * rows * N * K / (us * 1e6)
            rec[label] = {"us": us, "tflops": tf}
            line += f"  {label}: {us:8.1f}us {tf:6.0f}TF/s"
        eng.set_option("tc_pair", 1)
        eng.set_option("tc_split", 1)
        eng.set_option("tc_sk", 0)
        print(line, flush=True)
        results.append(rec)
        del w, ref
if args.out:
    Path(args.out).write_text(json.dumps(results, indent=1))
eng.close()
