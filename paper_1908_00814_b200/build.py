"""Build libknnm.so in-tree for sm_100a (nvcc; no JIT cache)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "knnm.cu")
OUT = os.path.join(HERE, "libknnm.so")
DEPS = [os.path.join(HERE, "csrc", f) for f in ("knnm.cu", "knnm_kernels.cuh", "knnm_device.cuh", "knnm_bf.cuh",
                                                   "knnm_tcjoin.cuh", "knnm_dense.cuh")]
DEPS.append(os.path.join(os.path.dirname(HERE), "include", "knnm.h"))

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc() -> str:
    for cand in (os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc"), "nvcc"):
        if os.path.sep not in cand or os.path.exists(cand):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(OUT):
        t = os.path.getmtime(OUT)
        if all(os.path.getmtime(d) <= t for d in DEPS):
            return OUT
    # KNNM_NVCC_EXTRA: extra flags for debug builds (e.g. "-DKNNM_DEBUG":
    # device-side bounds asserts on the lazy / batch paths)
    extra = os.environ.get("KNNM_NVCC_EXTRA", "").split()
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", OUT, SRC]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
