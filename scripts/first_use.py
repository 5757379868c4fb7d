"""First-use cost of a kernel variant in a fresh process (lazy module loading / local-memory growth)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
t0 = time.perf_counter()
eng = sc.Engine(0)
print("engine create %.1f ms" % ((time.perf_counter() - t0) * 1e3), flush=True)
for shape in [(4096, 4096), (4096, 14336), (512, 9000)]:
    a = sc.fill_normal(1, shape[0] * shape[1], np.float32).reshape(shape)
    for k in range(2):
        t0 = time.perf_counter()
        dec, rep, _ = eng.run(a, sc.DecomposeConfig(width=2, search=sc.SearchConfig(seed=1)), dtype="f32")
        print(shape, "call", k, "wall %.1f ms" % ((time.perf_counter() - t0) * 1e3), "kernel %.1f ms" % rep.kernel_ms, flush=True)
