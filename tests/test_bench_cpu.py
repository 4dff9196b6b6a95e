"""bench.py's N-GPU entry point and reference arm on CPU: `--gpus 2` outside
torchrun re-launches itself with two ranks (gloo for the reference arm), rank
0 runs the reference runners over the CPU oracle and prints the one JSON line,
the other rank exits 0 without work."""

import json
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]


def test_reference_arm_self_launches_two_ranks():
    cmd = [sys.executable, str(REPO / "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "2",
           "--warmup", "1", "--config", "small", "--ref-config", "tiny", "--ref-budget-s", "5"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=str(REPO))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["steps"] >= 1 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and "ecot_sched" in line["cpu_baseline"]["sample"] or \
        "reference ParallelSyncRunner" in line["cpu_baseline"]["sample"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["reference_synthetic_backend"]["steps"] == 2
