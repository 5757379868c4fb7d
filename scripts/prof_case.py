"""Small fixed case for ncu: 4096^2 f32, width from argv."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
w = int(sys.argv[1]) if len(sys.argv) > 1 else 2
m = n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
eng = sc.Engine(0)
a = sc.fill_normal(1, m * n, np.float32).reshape(m, n)
dec, rep, _ = eng.run(a, sc.DecomposeConfig(width=w, search=sc.SearchConfig(seed=1)), dtype="f32")
print("kernel_ms", rep.kernel_ms, "passes", rep.passes, "sweeps", rep.sweeps.tolist())
