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
COMM_SRC = os.path.join(HERE, "csrc", "ucp_comm.cpp")
COMM_OUT = os.path.join(HERE, "libucp_b200_comm.so")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC,-O2", "-ftz=false",
              "-prec-div=true", "-prec-sqrt=true", "-fmad=false"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _fresh(out: str, srcs: list) -> bool:
    return os.path.exists(out) and all(os.path.getmtime(out) >= os.path.getmtime(s) for s in srcs)


def build_comm(verbose: bool = False) -> str:
    """libucp_b200_comm.so: host-only NCCL wrapper (links libnccl.so.2 by
    soname, so a process that already loaded torch's NCCL reuses it)."""
    srcs = [COMM_SRC, os.path.join(ROOT, "include", "ucp_b200_comm.h")]
    if _fresh(COMM_OUT, srcs):
        return COMM_OUT
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA_HOME, "include"), COMM_SRC, "-o", COMM_OUT + ".tmp",
           "-L", os.path.join(CUDA_HOME, "lib64"), "-lnccl", "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode:
        raise RuntimeError(f"g++ failed ({res.returncode}): {' '.join(cmd)}")
    os.replace(COMM_OUT + ".tmp", COMM_OUT)
    return COMM_OUT


def build(verbose: bool = False) -> str:
    """Compile if a .so is missing or older than its sources."""
    build_comm(verbose)
    srcs = [SRC, os.path.join(ROOT, "include", "ucp_b200.h")]
    if _fresh(OUT, srcs):
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
