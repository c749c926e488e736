"""Build libucp_b200.so in-tree for sm_100a.

    python -m paper_2406_18820_b200._build

Flags: -gencode arch=compute_100a,code=sm_100a, -O3, -lineinfo, and no fast
math (the partial-noise and mean epilogues rely on IEEE f64/f32 with
denormals; nvcc defaults keep -ftz=false -prec-div=true).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "ucp_b200.cu")
OUT = os.path.join(HERE, "libucp_b200.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC,-O2", "-ftz=false",
              "-prec-div=true", "-prec-sqrt=true", "-fmad=false"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def build(verbose: bool = False) -> str:
    """Compile if the .so is missing or older than its sources."""
    srcs = [SRC, os.path.join(ROOT, "include", "ucp_b200.h")]
    if os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(s) for s in srcs):
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), SRC, "-o", OUT + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode:
        raise RuntimeError(f"nvcc failed ({res.returncode}): {' '.join(cmd)}")
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose=True))
