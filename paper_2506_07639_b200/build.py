"""In-tree build of libfastecot.so for sm_100a (explicit nvcc, no JIT cache).

`python -m paper_2506_07639_b200.build` or `__graft_entry__.build()`.
Every kernel is compiled with --fmad=false: fused multiply-adds are written
explicitly (__fmaf_rn), which is what makes the fp32 mode bit-exact against
the CPU oracle.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "_build" / "libfastecot.so"
SOURCES = ["kernels.cu", "gemm_tc.cu", "decode_mk.cu", "decode_mk_trace.cu", "prefill_attn.cu", "prefill_attn_tc.cu", "attn_span.cu", "vision.cu", "engine.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
         "-Xcompiler", "-fPIC", "-diag-suppress", "1886,177"]


def needs_build() -> bool:
    if not OUT.exists():
        return True
    mtime = OUT.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))
    deps.append(PKG.parent / "include" / "fastecot.h")
    return any(p.stat().st_mtime > mtime for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    tmp = OUT.with_suffix(".so.tmp")
    objs = [OUT.parent / (Path(s).stem + ".o") for s in SOURCES]

    def compile_one(src_obj):
        src, obj = src_obj
        cmd = [NVCC, *FLAGS, "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True, cwd=str(CSRC))

    # one nvcc per translation unit, in parallel (the tick kernel dominates)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(compile_one, zip(SOURCES, objs)))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *map(str, objs), "-o", str(tmp)]
    subprocess.run(cmd, check=True, cwd=str(CSRC))
    tmp.replace(OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
