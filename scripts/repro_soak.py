"""One soak case against the reference: usage repro_soak.py m n dtype w restarts div seed intdata"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
from oracle.pyoracle import Oracle
m, n, dtype, w, restarts, div, seed, intdata = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), int(sys.argv[5]), int(sys.argv[6]), int(sys.argv[7]), int(sys.argv[8])
ref = Oracle("ref")
eng = sc.Engine(0)
a = sc.fill_normal(seed, m * n, np.float32).reshape(m, n)
if intdata:
    a = np.round(a * 2).astype(np.float32)
a = a if dtype == "f32" else a.astype(np.float64)
cfg = sc.DecomposeConfig(width=w, record_curve=True, search=sc.SearchConfig(seed=seed, restarts=restarts))
od = ref.greedy_decompose(a.astype(np.float64), w, seed=seed, restarts=restarts)
print("ref sweeps", od.iterations.astype(int).tolist())
for mode, dv in ((1, div), (0, div), (1, 32), (0, 32)):
    with eng.options(fast_delta=mode, delta_div=dv):
        dec, rep, _ = eng.run(a, cfg, dtype=dtype)
    same = [bool((dec.factors[0][k] == od.signs[0][k]).all() and (dec.factors[1][k] == od.signs[1][k]).all()) for k in range(w)]
    print("fast" if mode else "barrier", "div", dv, "sweeps", rep.sweeps.tolist(), "identical to ref", same,
          "max rel dc", float(np.max(np.abs(rep._cut_values - od.cut_value) / np.abs(od.cut_value))))
