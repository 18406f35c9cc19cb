"""Build libgem.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2509_25075_b200.build        # or __graft_entry__.build()

The library is plain CUDA C++ behind the C ABI of include/gem.h, linked
against the shared CUDA runtime and cuFFT (the FFT is the one library call
the hot path makes; the CTF multiply, loss and everything else are ours).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgem.so")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-v", "-Xptxas", "-warn-spills",
    "-shared", "-cudart", "shared",
    "-I" + os.path.join(ROOT, "include"),
]
LINK = ["-L" + os.path.join(CUDA_HOME, "lib64"), "-lcufft", "-Xlinker", "-rpath=" + os.path.join(CUDA_HOME, "lib64")]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "gem.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    extra = os.environ.get("GEM_NVCC_EXTRA", "").split()   # experiment-only -D switches
    cmd = [NVCC, *NVCC_FLAGS, *extra, "-o", tmp, *sources(), *LINK]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libgem.so")
    if verbose:
        sys.stderr.write(res.stderr)
    # resource report (registers, spills) for the kernels; untracked, under build/
    os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
    with open(os.path.join(ROOT, "build", "ptxas.log"), "w") as f:
        f.write(res.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
