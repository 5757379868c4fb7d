"""Small fixed cases for ncu (one sweep_kernel launch each):
  python scripts/prof_case.py W [M [N]]   M x N f32 N(0,1) (Xoshiro256pp(1)), W cuts, search seed 1
  python scripts/prof_case.py W c5        the C5 matrix (65536^2 f32, block-seeded rows), search seed 4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2410_01799_b200 as sc  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 2
eng = sc.Engine(0)
if len(sys.argv) > 2 and sys.argv[2] == "c5":
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from c5_runs import c5_matrix

    a, seed = c5_matrix(), 4
else:
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    n = int(sys.argv[3]) if len(sys.argv) > 3 else m
    a, seed = sc.fill_normal(1, m * n, np.float32).reshape(m, n), 1
dec, rep, _ = eng.run(a, sc.DecomposeConfig(width=w, search=sc.SearchConfig(seed=seed)), dtype="f32")
print("kernel_ms", rep.kernel_ms, "passes", rep.passes, "dense", rep.dense_passes, "delta", rep.delta_passes,
      "device_bytes", rep.device_bytes, "sweeps", rep.sweeps.tolist())
