"""First cuts of every Mistral-shaped C4 job (one of each shape) and of C2 f64 against the
reference on the same input: signs identical, sweeps equal, c within tolerance."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
from oracle.pyoracle import Oracle
from paper_2410_01799_b200.batch import mistral_jobs, mistral_matrix
ref = Oracle("ref")
eng = sc.Engine(0)
jobs = mistral_jobs()
for idx in (0, 1, 4, 6, 224):
    j = jobs[idx]
    a = mistral_matrix(j)
    w = 3
    cfg = sc.DecomposeConfig(width=w, flush_width=1, record_curve=True, search=sc.SearchConfig(seed=j.seed))
    dec, rep, _ = eng.run(a, cfg, dtype="f32")
    t0 = time.time()
    od = ref.greedy_decompose(a.astype(np.float64), w, seed=j.seed, flush_width=1)
    same = [all((dec.factors[i][k] == od.signs[i][k]).all() for i in range(2)) for k in range(w)]
    print(j.name, j.shape, "identical", same, "sweeps", rep.sweeps.tolist(), od.iterations.tolist(),
          "max rel dc %.2e" % np.max(np.abs(rep._cut_values - od.cut_value) / od.cut_value),
          "cpu %.1fs" % (time.time() - t0), flush=True)
