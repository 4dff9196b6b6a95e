"""Prefill-attention timeline (diagnostics): one trunk prefill on the 7B bf16
engine with option pattn_trace, then per query tile (head 0, last layer) the
clock64 stamps of every page: S seen by the softmax, P handed back, P V
issued, S two pages ahead issued -- in cycles from the CTA's start."""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from paper_2506_07639_b200 import model as M  # noqa: E402
from paper_2506_07639_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="7b")
ap.add_argument("--trunk", type=int, default=625)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--no-trace", action="store_true", help="plain prefills (for an ncu launch list)")
args = ap.parse_args()

eng = Engine(args.config, dtype="bf16", seed=0, kv_pages=256, max_rows=1024)
if not args.no_trace:
    eng.set_option("pattn_trace", 1)
for rep in range(args.reps):
    s = eng.seq_create()
    eng.prefill(s, list(range(3, 3 + args.trunk)), 7, M.VIS_ID)
    eng.synchronize()
    eng.seq_free(s)
if args.no_trace:
    eng.close()
    sys.exit(0)
tr = eng.debug_trace().ravel()[: 1 << 14].astype(np.int64)
n_tiles = (args.trunk + 127) // 128
names = ["S seen", "-", "max", "pbuf"] + [f"P w{w}" for w in range(8)] + ["| p_full", "PV", "S+3"]
for t in range(n_tiles):
    row = tr[t * 512:(t + 1) * 512]
    t0 = row[0]
    if t0 == 0:
        continue
    print(f"cta {t} (tile {n_tiles - 1 - t}): start->pdl/Q staged {row[1] - t0:6d}  end {row[15] - t0:6d} cycles")
    print("        " + " ".join(f"{n:>7s}" for n in names))
    j = 0
    while 16 + 16 * j < 512 and row[16 + 16 * j] >= t0 > 0:
        st = [row[16 + 16 * j + k] - t0 if row[16 + 16 * j + k] >= t0 else -1 for k in range(15)]
        print(f"page {j:2d} " + " ".join(f"{v:7d}" for v in st))
        j += 1
eng.close()
