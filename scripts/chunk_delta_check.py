"""Chunked rows with delta passes: parity with the reference on inputs with many sweeps, and C5-like timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
from oracle.pyoracle import Oracle
ref = Oracle("ref")
eng = sc.Engine(0)
for shape, dtype, w in [((1024, 20000), "f32", 3), ((512, 16000), "f32", 3), ((300, 9000), "f64", 3), ((2048, 16384), "f32", 2)]:
    a = ref.fill_normal(8, shape[0] * shape[1]).reshape(shape)
    if dtype == "f32":
        a = a.astype(np.float32).astype(np.float64)
    cfg = sc.DecomposeConfig(width=w, flush_width=1, record_curve=True, search=sc.SearchConfig(seed=4))
    dec, rep, _ = eng.run(a.astype(np.float32) if dtype == "f32" else a, cfg, dtype=dtype)
    od = ref.greedy_decompose(a, w, seed=4, flush_width=1)
    same = [all((dec.factors[i][k] == od.signs[i][k]).all() for i in range(2)) for k in range(w)]
    print(shape, dtype, "identical", same, "sweeps", rep.sweeps.tolist(), od.iterations.tolist(),
          "us/pass", round(rep.kernel_ms * 1e3 / rep.passes, 1), flush=True)
