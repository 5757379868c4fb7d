"""Run one decomposition with an alternative engine build (SCB_LIB=path, e.g. an
SCB_PROFILE=1 build) with the engine option profile=1 (PROF_CTA=1: per-CTA lines):
prints the kernel's clock64 phase breakdown.
usage: SCB_LIB=ablibs/lib_prof.so python scripts/prof_lib.py W [M N] [f32|f64]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2410_01799_b200 import _native as N  # noqa: E402

if os.environ.get("SCB_LIB"):
    N.LIB_PATH = os.environ["SCB_LIB"]
import paper_2410_01799_b200 as sc  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 64
m = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
n = int(sys.argv[3]) if len(sys.argv) > 3 else m
dt = sys.argv[4] if len(sys.argv) > 4 else "f32"
opts = {k: int(v) for k, v in (x.split("=") for x in os.environ.get("PROF_OPTS", "").split(",") if x)}  # e.g. delta=0
eng = sc.Engine(0, profile=2 if os.environ.get("PROF_CTA") else 1, **opts)
a = sc.fill_normal(1, m * n, np.float32).reshape(m, n)
dec, rep, _ = eng.run(a, sc.DecomposeConfig(width=w, search=sc.SearchConfig(seed=1)), dtype=dt)
print("kernel_ms", rep.kernel_ms, "passes", rep.passes, "dense", rep.dense_passes, "delta", rep.delta_passes,
      "us/pass", rep.kernel_ms * 1e3 / rep.passes)
