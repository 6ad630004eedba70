"""Build libgwcp_b200.so in-tree for sm_100a (nvcc; no JIT cache)."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = [os.path.join(HERE, "csrc", "engine.cu"), os.path.join(HERE, "csrc", "parse.cpp"),
       os.path.join(HERE, "csrc", "codec.cpp")]
DEPS = SRC + [os.path.join(HERE, "csrc", f) for f in ("primitives.cuh", "walker.cuh", "walker_warp.cuh", "bucket.cuh", "workloads.cuh", "validate.cuh",
                                                         "access.cuh", "common.h")]
OUT = os.path.join(HERE, "libgwcp_b200.so")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-lpthread",
]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(OUT):
        mt = os.path.getmtime(OUT)
        hdr = os.path.join(os.path.dirname(HERE), "include", "gwcp_b200.h")
        if all(os.path.getmtime(p) <= mt for p in DEPS + [hdr]):
            return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-o", OUT, *SRC]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
