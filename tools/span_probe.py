"""Wide chain decode tick probe for the span attention (debug / timing):
`--branches` forks of one trunk decoded together with mk off."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2506_07639_b200 import model as M  # noqa: E402
from paper_2506_07639_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="small")
ap.add_argument("--branches", type=int, default=7)
ap.add_argument("--episodes", type=int, default=1, help="trunks (each with --branches forks)")
ap.add_argument("--trunk", type=int, default=300)
ap.add_argument("--tokens", type=int, default=3)
ap.add_argument("--opt", action="append", default=[])
args = ap.parse_args()
eng = Engine(args.config, dtype="bf16", seed=0, kv_pages=max(512, 40 * args.episodes), max_rows=1024)
eng.set_option("mk", 0)
for kv in args.opt:
    k, v = kv.split("=")
    eng.set_option(k, int(v))
cfg = M.get_config(args.config)
ids = [M.BOS_ID] + [M.VIS_ID] * cfg.n_vision + list(range(100, 100 + args.trunk))
reqs = []
for ep in range(args.episodes):
    trunk = eng.seq_create()
    eng.prefill(trunk, ids, 7 + ep, M.VIS_ID)
    for j in range(args.branches):   # fork points spread over the trunk like Fast-ECoT's nested prefixes
        b = eng.seq_fork(trunk, len(ids) - (len(ids) - cfg.n_vision) * j // (2 * args.branches))
        reqs.append(eng.submit(b, M.TAG_BASE + j % 32, args.tokens, 1))
eng.synchronize()
print("prefill done", flush=True)
eng.set_slots(max(8, len(reqs)))
t0 = time.perf_counter()
eng.run(-1)
eng.synchronize()
print("decode done", time.perf_counter() - t0, [eng.request_tokens(r, args.tokens)[0] for r in reqs[:8]], flush=True)
