"""Sweep launch-shape knobs (env overrides read per call) on an f32 matrix."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
eng = sc.Engine(0)
n = int(os.environ.get("TUNE_N", 4096))
m = int(os.environ.get("TUNE_M", n))
dt = os.environ.get("TUNE_DTYPE", "f32")
a = sc.fill_normal(1, m * n, np.float32 if dt == "f32" else np.float64).reshape(m, n)
w = int(os.environ.get("TUNE_W", 16))
cfg = sc.DecomposeConfig(width=w, search=sc.SearchConfig(seed=1))
os.environ["SCB_PROF"] = "1"
grid = json.loads(os.environ.get("TUNE_GRID", '[{}]'))
ref = None
for gd in grid:
    for k in ("SCB_DS", "SCB_STAGES", "SCB_RES_ROWS", "SCB_VARIANT"):
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in gd.items()})
    dec, rep, _ = eng.run(a, cfg, dtype=dt)
    if ref is None:
        ref = (rep.sweeps.copy(), rep._cut_values.copy(), [f.copy() for f in dec.factors])
    same = (rep.sweeps == ref[0]).all() and (rep._cut_values == ref[1]).all() and all((x == y).all() for x, y in zip(dec.factors, ref[2]))
    alg = float(np.sum(2 * rep.sweeps.astype(np.float64) + 1)) * m * n * (4 if dt == "f32" else 8)
    print(gd, f"kernel {rep.kernel_ms:.2f} ms  {w/rep.kernel_ms*1e3:.1f} cuts/s  us/pass {rep.kernel_ms*1e3/rep.passes:.2f}  alg {alg/rep.kernel_ms/1e6:.0f} GB/s bitsame={same}", flush=True)
