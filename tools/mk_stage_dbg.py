"""Per-stage timeline of phase 10 (layer 1 QKV) for CTAs 0-3 (decode_probe --trace --mk-flags 1024):
W issue, X issue and landing (MMA warp past the full barrier) of the first 24 stages, us from the barrier."""
import numpy as np
tr = np.load("gpurun_out/mk_trace.npy").astype(np.int64)
P, K, G = tr.shape
flat = tr[0].reshape(-1)
for c in range(4):
    t0 = tr[10, 0, c]
    d = flat[c * 96: c * 96 + 96]
    f = lambda v: "   .  " if v == 0 or abs(v - t0) > 1e8 else f"{(v - t0) / 1e3:6.2f}"
    print(f"CTA {c}: bar {0:.2f}")
    print("  W  " + " ".join(f(v) for v in d[24:48]))
    print("  X  " + " ".join(f(v) for v in d[48:72]))
    print("  L  " + " ".join(f(v) for v in d[0:24]))
