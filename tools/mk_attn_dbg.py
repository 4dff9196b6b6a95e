import numpy as np
tr = np.load("gpurun_out/mk_trace.npy").astype(np.int64)
P, _, G = tr.shape
d = tr[P - 1, 2]
for l in range(1, 6):
    t = d[8 * l: 8 * l + 4]
    print(f"layer {l}: QK {(t[1]-t[0])/1e3:.2f} us  softmax {(t[2]-t[1])/1e3:.2f} us  PV+stores {(t[3]-t[2])/1e3:.2f} us")
