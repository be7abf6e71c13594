"""Builds libpaces_b200.so (hand-written sm_100a CUDA + the C ABI of include/paces_b200.h) with nvcc.

The library is built IN-TREE (paper_2603_07341_b200/libpaces_b200.so) so it travels to the GPU box with the
repo snapshot.  nvcc cross-compiles without a GPU.  -fmad=false: the reference binary contains no FMA
(proj/CMakeLists.txt:6-8) and bit-exact amplitudes need the same (the kernels also use explicit
__dmul_rn/__dadd_rn).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("PB200_LIB_OUT") or os.path.join(HERE, "libpaces_b200.so")
# Separate translation units compiled in parallel (kernels live in headers with internal linkage).  No -split-compile
# anywhere: with it ptxas gave the same source different register allocations from one build to the next (the Taylor
# kernels: 32 or 40 registers, spills or none) -- up to 10 % of a step.
SOURCES = ["engine.cu", "incremental.cu", "histogram.cu", "sharded.cu", "nccl_comm.cu", "capi.cu", "taylor.cu"]
DEPS = SOURCES + ["taylor.cuh", "engine.cuh", "sharded.cuh", "kernels.cuh", "window.cuh", "incremental.cuh", "histogram.cuh",
                  "keys.cuh", "primitives.cuh", "host_model.hpp", "nccl_comm.hpp",
                  os.path.join("..", "..", "include", "paces_b200.h")]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo", "-fmad=false",
              "-Xcompiler", "-fPIC,-O2", "-shared"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.exists(os.path.join(CSRC, d)) and os.path.getmtime(os.path.join(CSRC, d)) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    flags = [f for f in NVCC_FLAGS if f != "-shared"] + ["-diag-suppress", "177"]
    if os.environ.get("PB200_ONLY_W"):  # development / profiling build restricted to one key width
        flags += ["-DPB_ONLY_W=" + str(int(os.environ["PB200_ONLY_W"]))]
    flags += os.environ.get("PB200_EXTRA_NVCC_FLAGS", "").split()  # experiments (e.g. -DTILE_TR=128)
    if verbose:
        flags += ["-Xptxas", "-v"]
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]

    def compile_one(src):
        obj = os.path.join(HERE, "_" + os.path.splitext(src)[0] + ".o")
        r = subprocess.run([_nvcc(), *flags, "-c", "-o", obj, os.path.join(CSRC, src)], cwd=CSRC, capture_output=True,
                           text=True)
        return src, obj, r

    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        results = list(ex.map(compile_one, srcs))
    objs = []
    for src, obj, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed compiling " + src)
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    r = subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs, "-ldl"],
                       cwd=CSRC, capture_output=True, text=True)
    for obj in objs:
        if os.path.exists(obj) and not os.environ.get("PB200_KEEP_OBJS"):  # tools/build_variants.sh relinks them
            os.remove(obj)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libpaces_b200.so")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
