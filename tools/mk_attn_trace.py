"""Summarise the attention phases of a persistent-tick trace (gpurun_out/mk_trace.npy)."""
import numpy as np
tr = np.load("gpurun_out/mk_trace.npy").astype(np.int64)
P = tr.shape[0]
for ph in range(3, P - 3, 10):
    st = tr[ph, 0].min()
    a = (tr[ph, 3] - tr[ph, 2]) / 1e3
    b = (tr[ph, 4] - tr[ph, 3]) / 1e3
    c = (tr[ph, 5] - tr[ph, 4]) / 1e3
    e = (tr[ph, 1] - tr[ph, 5]) / 1e3
    f = lambda x: f"med {np.median(x):5.1f} p90 {np.percentile(x, 90):5.1f} max {x.max():5.1f}"
    print(f"ph {ph:3d} staging {f(a)} | warp2 pairs {f(b)} | other warps {f(c)} | to done {f(e)}")
    ph2 = ph + 1
    st2 = tr[ph2, 2]
    m = (tr[ph2, 3] - st2) / 1e3
    m = m[tr[ph2, 3] > 0]
    e2 = (tr[ph2, 5] - tr[ph2, 2]) / 1e3
    print(f"   amerge: start->first merge done {f(m)} | start->all warps {f(e2)} | span {(tr[ph2,1].max()-tr[ph2,0].min())/1e3:.1f}")
    if ph > 40:
        break
