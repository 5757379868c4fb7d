"""Same-box A/B: time the 64-cut 4096^2 f32 decomposition with two builds of the
engine (env SCB_LIB_A / SCB_LIB_B = paths to libsigcut_b200.so builds)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2410_01799_b200 import _native as N
import paper_2410_01799_b200 as sc

libs = [os.environ.get("SCB_LIB_A", N.LIB_PATH)] + os.environ["SCB_LIB_B"].split(",")
M, N_ = (int(x) for x in os.environ.get("AB_SHAPE", "4096,4096").split(","))
SEED = int(os.environ.get("AB_SEED", 1))
a = sc.fill_normal(SEED, M * N_, np.float32).reshape(M, N_)
if os.environ.get("AB_C3"):  # config 3: the order-3 blob image, search seed 2
    from paper_2410_01799_b200 import workloads as wl
    a, SEED = wl.c3_blob_image(), 2
cfg = sc.DecomposeConfig(width=int(os.environ.get("AB_W", 64)), search=sc.SearchConfig(seed=SEED))
res = {}
ALL_SIGS = dict(N.SIGNATURES)
for rnd in range(int(os.environ.get("AB_ROUNDS", 3))):
    for path in libs:
        import ctypes
        probe = ctypes.CDLL(path)
        N.SIGNATURES = {k: v for k, v in ALL_SIGS.items() if hasattr(probe, k)}  # older builds: fewer symbols
        N._lib = None
        N.LIB_PATH = path
        eng = sc.Engine(0, **{k: int(v) for k, v in (x.split("=") for x in os.environ.get("AB_ENGINE_OPTS", "").split(",") if x)})
        dec, rep, _ = eng.run(a, cfg, dtype="f32")
        res.setdefault(path, []).append((rep.kernel_ms, rep.passes, tuple(rep.sweeps[:8])))
        del eng
for path, v in res.items():
    ms = [x[0] for x in v]
    print(f"{os.path.basename(path):28s} kernel ms {['%.2f' % m for m in ms]}  min {min(ms):.2f}  us/pass {min(ms) * 1e3 / v[0][1]:.2f}  sweeps {v[0][2]}")
