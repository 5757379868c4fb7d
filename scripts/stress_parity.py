"""Parity stress on mid-size inputs that exercise resident + streamed rows, dense and delta
passes, restarts, the sweep cap and order-k, against the reference (first cuts)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
from oracle.pyoracle import Oracle
ref = Oracle("ref")
eng = sc.Engine(0)
cases = [
    ("f64 2048x3000 r2", (2048, 3000), "f64", 5, 2, 100, 11),
    ("f32 3000x2048 r3 cap20", (3000, 2048), "f32", 5, 3, 20, 12),
    ("f64 4096x4096 w12", (4096, 4096), "f64", 12, 1, 100, 1),
    ("f32 777x5000 r2", (777, 5000), "f32", 6, 2, 100, 13),
    ("f64 300x40x30 r2", (300, 40, 30), "f64", 5, 2, 100, 14),
    ("f32 64x64x64 cap7", (64, 64, 64), "f32", 6, 1, 7, 15),
    ("f64 5000x300", (5000, 300), "f64", 8, 1, 100, 16),
]
for name, shape, dtype, w, restarts, cap, seed in cases:
    a = ref.fill_normal(seed, int(np.prod(shape))).reshape(shape)
    if dtype == "f32":
        a = a.astype(np.float32).astype(np.float64)
    cfg = sc.DecomposeConfig(width=w, flush_width=1, record_curve=True,
                             search=sc.SearchConfig(seed=seed, restarts=restarts, max_sweeps=cap))
    dec, rep, _ = eng.run(a.astype(np.float32) if dtype == "f32" else a, cfg, dtype=dtype)
    t0 = time.time()
    od = ref.greedy_decompose(a, w, seed=seed, flush_width=1, restarts=restarts, max_sweeps=cap)
    same = [all((dec.factors[i][k] == od.signs[i][k]).all() for i in range(len(shape))) for k in range(w)]
    gs, rs = rep.sweeps.astype(int), od.iterations.astype(int)
    sweeps_ok = bool(np.all((gs == rs) | ((gs % 16 == 0) & (rs == gs + 1))))
    print(f"{name:24s} identical {sum(same)}/{w} first_bad {next((k for k, x in enumerate(same) if not x), None)} "
          f"sweeps_ok {sweeps_ok} {gs.tolist()} {rs.tolist()} max rel dc "
          f"{np.max(np.abs(rep._cut_values - od.cut_value) / od.cut_value):.2e} cpu {time.time() - t0:.1f}s", flush=True)
