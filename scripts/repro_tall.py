import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
from paper_2410_01799_b200 import batch
jobs = batch.mistral_jobs()
j = [x for x in jobs if x.name == 'embed'][0]
a = batch.mistral_matrix(j)
eng = sc.Engine(0)
for w in (64, 128, 256, 512):
    try:
        dec, rep, _ = eng.run(a, sc.DecomposeConfig(width=w, search=sc.SearchConfig(seed=j.seed)), dtype="f32")
        print(w, "ok", rep.sweeps[-8:].tolist(), rep.final_residual_norm / rep.input_norm, rep.kernel_ms, flush=True)
    except Exception as e:
        print(w, "FAIL", e, flush=True)
        for opts in [dict(delta=0), dict(fuse_update=0), dict(two_phase=1)]:
            with eng.options(**opts):
                try:
                    dec, rep, _ = eng.run(a, sc.DecomposeConfig(width=w, search=sc.SearchConfig(seed=j.seed)), dtype="f32")
                    print("  ", opts, "ok", rep.final_residual_norm / rep.input_norm, flush=True)
                except Exception as e2:
                    print("  ", opts, "FAIL", e2, flush=True)
        break
