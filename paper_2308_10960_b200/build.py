"""Build libhcmx_gpu.so in-tree (sm_100a only; cross-compiles without a GPU).

    python -m paper_2308_10960_b200.build

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo for the kernels, g++
-ffp-contract=off for the host scalar rules (the reference's Release flags keep
separate FP multiply/add), linked with the static CUDA runtime.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# HCMX_BUILD_TAG (profiling aid): build a variant (e.g. other HCMX_NVCC_DEFS)
# into variants/libhcmx_gpu_<tag>.so instead of the product library
_TAG = os.environ.get("HCMX_BUILD_TAG")
OBJ = os.path.join(HERE, "_build" + (f"_{_TAG}" if _TAG else ""))
LIB = (os.path.join(ROOT, "variants", f"libhcmx_gpu_{_TAG}.so") if _TAG
       else os.path.join(HERE, "libhcmx_gpu.so"))
INC = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", "nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + [*(["-DHCMX_PROF"] if os.environ.get("HCMX_PROF_BUILD") else []),
                  *os.environ.get("HCMX_NVCC_DEFS", "").split(), "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
                  "-I" + INC, "-I" + CSRC]
CUDA_INC = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "include")
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-I" + INC, "-I" + CSRC, "-I" + CUDA_INC]

CU = ["codec_kernels.cu", "hmat.cu", "compress.cu"]
CPP = ["codec_host.cpp", "dist.cpp"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[0]} {cmd[-1]}")
    return r


STAMP = os.path.join(OBJ, "flags.stamp")


def _flags_changed() -> bool:
    """the active compile flags (HCMX_NVCC_DEFS / HCMX_PROF_BUILD included) differ
    from the ones the objects were built with (a profiling build must never be
    kept by a later plain build)"""
    want = " ".join(NVFLAGS + CXXFLAGS)
    have = open(STAMP).read() if os.path.exists(STAMP) else None
    return have != want


def _stale(src, obj, extra=()):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src, os.path.join(CSRC, "internal.h"), os.path.join(INC, "hcmx_gpu.h"), *extra]
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if _flags_changed():
        force = True
    objs = []
    for f in CU:
        src, obj = os.path.join(CSRC, f), os.path.join(OBJ, f + ".o")
        if force or _stale(src, obj):
            r = _run([NVCC, *NVFLAGS, "-Xptxas", "-v", "-c", src, "-o", obj])
            if verbose:
                sys.stderr.write(r.stderr)
        objs.append(obj)
    for f in CPP:
        src, obj = os.path.join(CSRC, f), os.path.join(OBJ, f + ".o")
        if force or _stale(src, obj):
            _run([CXX, *CXXFLAGS, "-c", src, "-o", obj])
        objs.append(obj)
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static", "-lpthread", "-ldl"])
    with open(STAMP, "w") as f:
        f.write(" ".join(NVFLAGS + CXXFLAGS))
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
