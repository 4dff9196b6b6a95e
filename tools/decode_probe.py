"""Decode-iteration probe: one trunk prefill + `rows` forked branches decoded
for `ticks` iterations on the 7B-shaped bf16 engine.  Used under ncu for the
per-kernel launch list and alone for host-vs-device tick timing."""

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2506_07639_b200 import model as M  # noqa: E402
from paper_2506_07639_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="7b")
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--rows", type=int, default=7)
ap.add_argument("--max-rows", type=int, default=1024, help="engine rows per forward (prefill chunk)")
ap.add_argument("--trunk", type=int, default=625)
ap.add_argument("--ticks", type=int, default=8)
ap.add_argument("--repeat", type=int, default=3)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--skip", type=int, default=0, help="debug_skip mask (timing attribution only)")
ap.add_argument("--stages", type=int, default=0)
ap.add_argument("--pdl", type=int, default=1)
ap.add_argument("--graphs", type=int, default=1)
ap.add_argument("--mk", type=int, default=1)
ap.add_argument("--mk-flags", type=int, default=0)
ap.add_argument("--pf", type=int, default=0, help="persistent tick: weight stages prefetched across a barrier")
ap.add_argument("--opt", action="append", default=[], help="extra engine option key=value")
ap.add_argument("--trace", action="store_true", help="per-phase barrier timeline of the persistent tick kernel")
args = ap.parse_args()

eng = Engine(args.config, dtype=args.dtype, seed=0, kv_pages=256, max_rows=args.max_rows)
if args.skip:
    eng.set_option("debug_skip", args.skip)
eng.set_option("pdl", args.pdl)
eng.set_option("graphs", args.graphs)
eng.set_option("mk", args.mk)
eng.set_option("mk_flags", args.mk_flags)
eng.set_option("mk_pf", args.pf)
for kv in args.opt:
    k, v = kv.split("=")
    eng.set_option(k, int(v))
if args.trace:
    eng.set_option("mk_trace", 1)
if args.stages:
    eng.set_option("sk_stages", args.stages)
cfg = M.get_config(args.config)
ids = [M.BOS_ID] + [M.VIS_ID] * cfg.n_vision + list(range(100, 100 + args.trunk - 1 - cfg.n_vision))
stream = torch.cuda.ExternalStream(eng.stream_handle())
for rep in range(args.repeat):
    trunk = eng.seq_create()
    t0 = time.perf_counter()
    eng.prefill(trunk, ids, 7, M.VIS_ID)
    eng.synchronize()
    t_pre = time.perf_counter() - t0
    reqs, seqs = [], []
    for j in range(args.rows):
        b = eng.seq_fork(trunk, len(ids) - 40 * (j % 8))
        seqs.append(b)
        reqs.append(eng.submit(b, M.TAG_BASE + j, args.ticks, 1))
    eng.set_slots(max(8, args.rows))
    if args.profile:
        eng.profile(True)
    a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    h0 = time.perf_counter()
    eng.run(-1)
    host = time.perf_counter() - h0
    b_.record(stream)
    eng.synchronize()
    dev = a.elapsed_time(b_)
    prof = eng.profile_read() if args.profile else {}
    if args.profile:
        eng.profile(False)
    for r in reqs:
        eng.request_tokens(r, args.ticks)
        eng.request_release(r)
    for s in seqs + [trunk]:
        eng.seq_free(s)
    print(f"rep {rep}: prefill {t_pre*1e3:.1f} ms | {args.ticks} ticks x {args.rows} rows: device {dev:.2f} ms "
          f"({dev/args.ticks:.3f} ms/tick), host enqueue {host*1e3:.2f} ms  {prof}", flush=True)
if args.trace:
    import numpy as np
    tr = eng.debug_trace().astype(np.int64)  # [P][6][G]
    P = tr.shape[0]
    t0 = tr[0, 0].min()
    fused = int(dict(o.split("=") for o in args.opt).get("mk_fused", 20)) if args.opt else 20
    seq = [("QKV", -1), ("RQKV", 0), ("ATTN", -1), ("AMERGE", -1), ("O", -1), ("RO", 1),
           ("GU", -1), ("RGU", 2), ("DOWN", -1), ("RDOWN", 3)]  # reduction phases exist unless fused
    layer = [n for n, bit in seq if bit < 0 or not (fused >> bit & 1)]
    names = ["EMBED"] + layer * cfg.n_layers + ["LM", "FINAL"]
    agg = {}
    print("phase         start   span | W-issue end   1st acc      last acc     drained  (min/max us from phase start)")
    for ph in range(P):
        start = tr[ph, 0].min()
        last_done = tr[ph, 1].max() if ph + 1 < P else tr[ph, 0].max()
        nxt = tr[ph + 1, 0].min() if ph + 1 < P else last_done
        span = (last_done - start) / 1e3
        bar = (nxt - last_done) / 1e3
        wi = tr[ph, 2] - start
        fa = tr[ph, 3] - start
        la = tr[ph, 4] - start
        dr = tr[ph, 5] - start
        has_w = tr[ph, 2].max() > 0 and tr[ph, 2].max() >= start
        a = agg.setdefault(names[ph], [0, 0.0, 0.0])
        a[0] += 1; a[1] += span; a[2] += bar
        if ph < 22 or ph >= P - 4:
            extra = "".join(f"  {v.min()/1e3:5.1f} {v.max()/1e3:5.1f} " for v in (wi, fa, la, dr)) if has_w else ""
            print(f"{ph:3d} {names[ph]:7s} {(start - t0)/1e3:7.1f} {span:6.1f} |{extra}   bar {bar:5.2f}")
    np.save("gpurun_out/mk_trace.npy", tr)
    for k, (n, sp, b) in agg.items():
        print(f"{k:6s} x{n:3d}: span {sp/n:7.2f} us  barrier {b/n:5.2f} us  total {sp+b:8.1f} us")
eng.close()
