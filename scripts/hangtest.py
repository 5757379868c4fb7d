import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
m, n, w = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
os.environ["SCB_VARIANT"] = sys.argv[4]
os.environ["SCB_RES_ROWS"] = sys.argv[5] if len(sys.argv) > 5 else "1000"
eng = sc.Engine(0)
a = sc.fill_normal(1, m * n, np.float32).reshape(m, n)
t = time.time()
dec, rep, _ = eng.run(a, sc.DecomposeConfig(width=w, search=sc.SearchConfig(seed=1)), dtype="f32")
print(sys.argv[1:], "ok", f"{time.time()-t:.2f}s passes", rep.passes, "sweeps", rep.sweeps.tolist(), flush=True)
