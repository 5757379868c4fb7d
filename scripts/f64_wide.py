"""f64 rows of 4097..7168 columns: 16-warp whole rows vs the chunked form (SCB_VARIANT=8,8,1), timing and parity."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
eng = sc.Engine(0)
a = sc.fill_normal(3, 4096 * 6000).reshape(4096, 6000)
for _ in range(2):
    dec, rep, _ = eng.run(a, sc.DecomposeConfig(width=16, search=sc.SearchConfig(seed=3)), dtype="f64")
    print(os.environ.get("SCB_VARIANT", "default"), "kernel_ms", round(rep.kernel_ms, 2), "passes", rep.passes,
          "us/pass", round(rep.kernel_ms * 1e3 / rep.passes, 1), "sweeps", rep.sweeps[:6].tolist(), flush=True)
