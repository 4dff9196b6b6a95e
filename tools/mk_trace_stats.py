"""Per-phase percentile summary of a persistent-tick trace (gpurun_out/mk_trace.npy,
written by tools/decode_probe.py --trace): slot times relative to the phase's
first barrier pass, 5th / 50th / max percentile over CTAs."""
import sys

import numpy as np

tr = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/mk_trace.npy").astype(np.int64)
first, last = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (1, 12)
slots = ["bar", "done", "Wiss", "acc1", "accL", "drain"][: tr.shape[1]]
for ph in range(first, min(last, tr.shape[0])):
    t0 = tr[ph, 0].min()
    row = []
    for k, nm in enumerate(slots):
        v = (tr[ph, k] - t0) / 1e3
        v = v[np.abs(v) < 1e5]
        if len(v):
            row.append(f"{nm} {np.percentile(v, 5):6.1f}/{np.median(v):6.1f}/{v.max():6.1f}")
    print(f"{ph:3d} " + " | ".join(row))
