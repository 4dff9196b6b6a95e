"""Extract per-launch DRAM traffic of the dominant decode kernel from an ncu
--set full report into profiles/ncu_decode_tick.json (persistent decode-tick
kernel) or profiles/ncu_decode_gemv.json (kernel chain); read by bench.py's
roofline `traffic`.

    python tools/ncu_traffic.py gpurun_out/prof_tick.ncu-rep profiles/ncu_decode_tick.json"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
names = {12288: "qkv", 4096: "o/down", 22016: "gate_up", 32064: "lm_head"}
launches = []
units = dict(zip(hdr, rows[1]))
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3,            # -> MB
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
         "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}                          # -> us
for r in rows[2:]:
    d = dict(zip(hdr, r))

    def f(k, d=d):
        if d.get(k) in (None, ""):
            return None
        return float(d[k].replace(",", "")) * SCALE.get(units.get(k, ""), 1.0)
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    launches.append({
        "kernel": d["Kernel Name"].split("(")[0].split("::")[-1], "grid": d["Grid Size"],
        "duration_us": f("gpu__time_duration.sum"),
        "dram_read_MB": rd, "dram_write_MB": wr,
        "dram_pct_peak": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "sm_active_frac": (f("sm__cycles_active.avg") or 0) / (f("gpc__cycles_elapsed.max") or 1),
        "registers": f("launch__registers_per_thread"),
    })
tot = sum((L["dram_read_MB"] or 0) + (L["dram_write_MB"] or 0) for L in launches)
summary = {"source": rep, "launches": launches,
           "dram_bytes_per_launch": tot * 1e6 / len(launches) if launches else None,
           "note": "ncu --set full, cold cache, clock-control none; bytes in MB per launch"}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary, indent=1)[:1500])
