#!/bin/bash
# Fresh bench lines for every BASELINE config on one B200 plus the launch list
# of the default bench command (run under gpurun; results in gpurun_out/).
set -u
O=gpurun_out
timeout 900 python bench.py --out $O/bench_c2.json > $O/bench_c2.log 2>&1; echo "c2 rc=$?"
timeout 900 python bench.py --workload stress --no-extras --no-cpu-baseline --out $O/bench_c5.json > $O/bench_c5.log 2>&1; echo "c5 rc=$?"
timeout 900 python bench.py --episodes 64 --steps 3 --warmup 2 --no-cpu-baseline --out $O/bench_c4.json > $O/bench_c4.log 2>&1; echo "c4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --profile-steps 1 > $O/launches_bench.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/launches_bench.csv 2>/dev/null | head -12
