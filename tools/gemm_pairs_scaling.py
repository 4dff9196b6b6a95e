"""Pair-count scaling of the CTA-pair GEMM (option tc_maxp): per-pair TF/s
when fewer pairs share the GPU -- the measurement behind DESIGN.md 5.2 (L2
operand-traffic bound)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2506_07639_b200.engine import Engine
eng = Engine("7b_2layer", dtype="bf16", seed=0, kv_pages=8, max_rows=64)
stream = torch.cuda.ExternalStream(eng.stream_handle())
for rows, (N, K) in [(8192, (12288, 4096)), (4096, (22016, 4096)), (2048, (12288, 4096))]:
    w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    x = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
    y = torch.empty(rows, N, device="cuda")
    for maxp in (74, 56, 37, 18):
        eng.set_option("tc_maxp", maxp)
        for _ in range(2):
            eng.op_gemm_tc(x.data_ptr(), w.data_ptr(), rows, N, K, y.data_ptr())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eng.set_option("op_reps", 10)
        a.record(stream); eng.op_gemm_tc(x.data_ptr(), w.data_ptr(), rows, N, K, y.data_ptr()); b.record(stream)
        eng.set_option("op_reps", 1)
        b.synchronize()
        us = a.elapsed_time(b) * 100
        tiles = ((rows + 255) // 256) * (N // 256)
        print(f"rows {rows} N {N}: pairs {maxp:3d}: {us:8.1f} us  {2*rows*N*K/us/1e6:6.0f} TF/s  per-pair {2*rows*N*K/us/1e6/maxp:5.1f} TF/s  L2 operand TB/s {tiles*(K//64)*65536/us/1e6:5.2f}", flush=True)
eng.close()
