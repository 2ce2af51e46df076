"""Build libshampoo.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python paper_2002_09018_b200/build.py            # incremental
    python paper_2002_09018_b200/build.py --force    # rebuild everything
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libshampoo.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
            "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
CU_FLAGS += os.environ.get("SHAMPOO_NVCC_EXTRA", "").split()  # measurement knobs (e.g. -DOZ_PROBE=...)
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-I", INCLUDE, "-I", CSRC, "-I", "/usr/local/cuda/include"]

SOURCES = ["abi.cpp", "plan.cpp", "stats.cu", "root.cu", "precondition.cu", "tc_gemm.cu", "momentum.cu", "tensor.cu",
           "root_tail.cu", "oz_precondition.cu"]
HEADERS = ["common.cuh", "dmma_gemm.cuh", "internal.h", "tc_common.cuh", "tc_gemm.h", "ozaki.cuh", "oz_precondition.h"]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "shampoo.h")]
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if not force and not _newer(obj, [path] + hdrs):
            continue
        if src.endswith(".cu"):
            cmd = [NVCC] + ARCH + CU_FLAGS + ["-c", path, "-o", obj]
            if verbose:
                cmd += ["-Xptxas", "-v"]
        else:
            cmd = ["g++"] + CXX_FLAGS + ["-c", path, "-o", obj]
        print("[build]", " ".join(cmd[:1] + [src]), flush=True)
        subprocess.check_call(cmd)
    if force or _newer(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "--cudart", "static", "-o", LIB] + objs
        print("[build] link", os.path.basename(LIB), flush=True)
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
