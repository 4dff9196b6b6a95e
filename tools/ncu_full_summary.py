"""Summarise an `ncu --set full` report (.ncu-rep) into a JSON of the metrics
the roofline needs, per captured launch: duration, DRAM bytes / throughput,
tensor-pipe activity, SM throughput, registers, achieved occupancy.

    python tools/ncu_full_summary.py REPORT.ncu-rep OUT.json [--flops-per-launch F ...]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
}
SCALE = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9, "s": 1.0,
         "second": 1.0, "Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0, "MB": 1e6, "GB": 1e9, "KB": 1e3}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:120], "grid": r[hdr.index("Grid Size")],
             "block": r[hdr.index("Block Size")]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                v = float(r[i].replace(",", "")) if r[i] else None
                u = units[i]
                if v is not None and u in SCALE:
                    v *= SCALE[u]
                d[name] = v
        if d.get("duration") and d.get("dram_read") is not None:
            d["dram_gbs"] = (d["dram_read"] + (d.get("dram_write") or 0)) / d["duration"] / 1e9
        launches.append(d)
    json.dump({"report": rep, "units": "seconds / bytes / percent", "launches": launches}, open(out, "w"), indent=1)
    for d in launches:
        print({k: (round(v, 6) if isinstance(v, float) else v) for k, v in d.items()})


if __name__ == "__main__":
    main()
