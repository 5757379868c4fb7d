"""In-tree build of the native engine: ``libsigcut_b200.so`` (sm_100a).

nvcc compiles the CUDA kernels and the C++ host driver into one shared
library next to this file so it travels with the repo snapshot to the GPU box.
Every translation unit is compiled to an object in parallel (the kernel
families live in separate sweep_k_*.cu units), then linked once.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("SCB_LIB_OUT") or os.path.join(HERE, "libsigcut_b200.so")  # SCB_LIB_OUT: A/B and profile builds
SOURCES = ["sweep.cu", "sweep_k_f32m.cu", "sweep_k_f32t.cu", "sweep_k_f64m.cu", "sweep_k_f64t.cu", "sweep_k_vr.cu",
           "ops.cu", "capi.cpp", "ops.cpp"]
HEADERS = ["sweep.h", "sweep_impl.cuh", "rng.h", "ops.h", "ctx.h"]
OBJDIR = os.environ.get("SCB_OBJDIR") or os.path.join(HERE, "build")
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
    os.makedirs(OBJDIR, exist_ok=True)

    def compile_one(f):
        obj = os.path.join(OBJDIR, f + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-c", "-o", obj, os.path.join(CSRC, f)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {f} ({r.returncode}):\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
