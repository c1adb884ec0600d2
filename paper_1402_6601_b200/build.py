"""In-tree build of ``libhetgpu.so`` (sm_100a CUDA kernels + runtime + native planner).

``python -m paper_1402_6601_b200.build`` or ``__graft_entry__.build()``.
nvcc cross-compiles for sm_100a without a GPU; the result lands next to this
file so it travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libhetgpu.so")
OBJ = os.path.join(ROOT, "build", "obj")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
                     "-I", CSRC, "-I", os.path.join(ROOT, "include")]
HOST_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall",
              "-I", os.path.join(ROOT, "include")]

CU_SOURCES = ["tiles_chol.cu", "tiles_lu.cu", "tiles_qr.cu", "runtime.cu", "peak.cu", "devrt.cu"]
CPP_SOURCES = ["planner.cpp"]


def _deps_mtime():
    newest = 0.0
    for d in (CSRC, os.path.join(ROOT, "include")):
        for f in os.listdir(d):
            newest = max(newest, os.path.getmtime(os.path.join(d, f)))
    return newest


def _compile(cmd):
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("compile failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    return res.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every source into ``libhetgpu.so``; returns its path."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps_mtime():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    jobs = []
    objs = []
    for src in CU_SOURCES:
        obj = os.path.join(OBJ, src + ".o")
        objs.append(obj)
        extra = ["-Xptxas", "-v"] if verbose else []
        jobs.append([NVCC] + CUDA_FLAGS + extra + ["-c", os.path.join(CSRC, src), "-o", obj])
    for src in CPP_SOURCES:
        obj = os.path.join(OBJ, src + ".o")
        objs.append(obj)
        jobs.append(["g++"] + HOST_FLAGS + ["-c", os.path.join(CSRC, src), "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as pool:
        for log in pool.map(_compile, jobs):
            if verbose and log:
                sys.stderr.write(log)
    tmp = LIB + ".tmp"
    _compile([NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lpthread"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
