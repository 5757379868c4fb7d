"""Parity of the wide-row (column-chunk) path against the reference on small row counts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
from oracle.pyoracle import Oracle
ref = Oracle("ref")
eng = sc.Engine(0)
for shape, dtype in [((40, 12000), "f64"), ((40, 12000), "f32"), ((96, 14336), "f32"), ((33, 20000), "f64"), ((150, 8300), "f64")]:
    a = ref.fill_normal(7, shape[0] * shape[1]).reshape(shape)
    if dtype == "f32":
        a = a.astype(np.float32).astype(np.float64)
    cfg = sc.DecomposeConfig(width=6, flush_width=1, record_curve=True, search=sc.SearchConfig(seed=4))
    dec, rep, _ = eng.run(a.astype(np.float32) if dtype == "f32" else a, cfg, dtype=dtype)
    od = ref.greedy_decompose(a, 6, seed=4, flush_width=1)
    same = [all((dec.factors[i][k] == od.signs[i][k]).all() for i in range(2)) for k in range(6)]
    print(shape, dtype, "signs identical per term", same, "gpu sweeps", rep.sweeps.tolist(), "ref", od.iterations.tolist(),
          "c rel", np.max(np.abs(rep._cut_values - od.cut_value) / od.cut_value), flush=True)
