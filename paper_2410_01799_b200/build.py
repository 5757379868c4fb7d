"""In-tree build of the native engine: ``libsigcut_b200.so`` (sm_100a).

nvcc compiles the CUDA kernels and the C++ host driver into one shared
library next to this file so it travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsigcut_b200.so")
SOURCES = ["sweep.cu", "ops.cu", "capi.cpp", "ops.cpp"]
HEADERS = ["sweep.h", "rng.h", "ops.h", "ctx.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-cudart", "static",
         "-Xptxas", "-v" if os.environ.get("SCB_PTXAS_VERBOSE") else "-O3"]
if os.environ.get("SCB_PROFILE"):  # clock64 phase breakdown compiled in (tuning builds only)
    FLAGS += ["-DSCB_PROFILE=1"]
FLAGS += [f"-D{d}" for d in os.environ.get("SCB_DEFINES", "").split(",") if d]  # A/B builds only


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "sigcut_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    srcs = [os.path.join(CSRC, f) for f in SOURCES]
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, *FLAGS, "-shared", "-o", tmp, *srcs]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr, file=sys.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
