import os, sys, time
sys.path.insert(0, "/root/repo")
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2410_01799_b200 as sc
from oracle.pyoracle import Oracle
from paper_2410_01799_b200 import workloads as wl
ref = Oracle("ref"); eng = sc.Engine(0)
a3 = wl.c3_blob_image(); w = 10
od = ref.greedy_decompose(a3.astype(np.float64), w, seed=2, flush_width=1)
for dtype in ("f64", "f32"):
    cfg = sc.DecomposeConfig(width=w, flush_width=1, record_curve=True, search=sc.SearchConfig(seed=2))
    dec, rep, _ = eng.run(a3.astype(np.float32) if dtype == "f32" else a3.astype(np.float64), cfg, dtype=dtype)
    same = [all((dec.factors[i][k] == od.signs[i][k]).all() for i in range(3)) for k in range(w)]
    print("C3", dtype, "identical", same, "sweeps", rep.sweeps.tolist(), od.iterations.astype(int).tolist(), "max rel dc", float(np.max(np.abs(rep._cut_values - od.cut_value) / od.cut_value)))
