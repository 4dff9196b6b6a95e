"""One bf16 decode through the persistent tick kernel (debug / sanitizer runs)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.backend import frame  # noqa: E402
from paper_2506_07639_b200 import model as M  # noqa: E402
from paper_2506_07639_b200.engine import Engine  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "small"
mk = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ids = frame(config, list(range(16)), list(range(500, 560)), "plan")
eng = Engine(config, dtype="bf16", seed=0, kv_pages=64, max_rows=512)
eng.set_option("mk", mk)
eng.set_option("graphs", 0)
seq = eng.seq_create()
eng.prefill(seq, ids[:-1], 4242, M.VIS_ID)
eng.synchronize()
print("prefill ok", flush=True)
req = eng.submit(seq, ids[-1], 3, 0)
eng.run(req)
print("tokens", eng.request_tokens(req, 3), flush=True)
eng.close()
