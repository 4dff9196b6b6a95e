"""Summarise an ncu --csv launch list: per kernel (name, grid) totals, and
for the skinny decode GEMM a per-matrix split by launch order within a layer."""
import collections
import csv
import sys

path = sys.argv[1]
rows = list(csv.reader(open(path)))
hdr, launches = None, {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        key = int(d["ID"])
        L = launches.setdefault(key, {"name": d["Kernel Name"], "grid": d["Grid Size"], "block": d["Block Size"]})
        L[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
order = [launches[k] for k in sorted(launches)]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for L in order:
    k = L["name"].split("(")[0][-42:] + " " + L["grid"]
    agg[k][0] += 1
    agg[k][1] += L.get("gpu__time_duration.sum", 0) / 1000.0
    agg[k][2] += L.get("dram__bytes_read.sum", 0)
print(f"{'total us':>10} {'n':>5} {'us/launch':>9} {'GB/s':>7}  kernel grid")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    gbs = v[2] / (v[1] * 1e3) if v[1] else 0
    print(f"{v[1]:10.1f} {v[0]:5d} {v[1]/v[0]:9.2f} {gbs:7.0f}  {k}")
sk = [L for L in order if "skinny" in L["name"]]
if sk:
    names = ["qkv", "o", "gate_up", "down"]
    per = collections.defaultdict(list)
    body = sk[:-1] if len(sk) % 4 else sk
    for i, L in enumerate(sk):
        per["lm_head" if (len(sk) % 4 == 1 and i == len(sk) - 1) else names[i % 4]].append(L)
    for n, Ls in per.items():
        t = sum(L.get("gpu__time_duration.sum", 0) for L in Ls) / len(Ls) / 1000
        b = sum(L.get("dram__bytes_read.sum", 0) for L in Ls) / len(Ls)
        print(f"skinny {n:8s}: {t:8.2f} us/launch, {b/1e6:8.1f} MB read, {b/(t*1e3):7.0f} GB/s  (n={len(Ls)})")
