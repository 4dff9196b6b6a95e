import numpy as np
tr = np.load("gpurun_out/mk_trace.npy").astype(np.int64)
for ph in (6, 8, 10, 16):
    a, b = tr[ph, 3], tr[ph, 4]
    print(ph, "partial ld.cg ns/load: median %d p90 %d | out_tokens ld.cg: median %d p90 %d" % (
        np.median(a), np.percentile(a, 90), np.median(b), np.percentile(b, 90)))
