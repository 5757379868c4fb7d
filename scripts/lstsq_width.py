"""Least-squares decomposition at growing widths (the term loop's host solve is the incremental
factor: O(k^2) per term): terms/s and the relative residual.  usage: lstsq_width.py [n] [w ...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ws = [int(x) for x in sys.argv[2:]] or [64, 256, 1024]
eng = sc.Engine(0)
a = sc.fill_normal(3, n * n, np.float32).reshape(n, n).astype(np.float64)
for w in ws:
    t0 = time.time()
    dec, rep = eng.lstsq_decompose(a, sc.DecomposeConfig(width=w, search=sc.SearchConfig(seed=2)))
    dt = time.time() - t0
    print(f"lstsq {n}x{n} f64 w={w}: {dt:.2f} s, {w / dt:.0f} terms/s, rel residual {rep.final_residual_norm / rep.input_norm:.4f}", flush=True)
