"""Parity of wide rows on shapes with many sweeps: a 1024 x 12000 N(0,1) matrix and the
C4 'down' matrix (4096 x 14336), first cuts against the reference."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
from oracle.pyoracle import Oracle
from paper_2410_01799_b200.batch import mistral_jobs, mistral_matrix
ref = Oracle("ref")
eng = sc.Engine(0)
j = mistral_jobs()[6]
cases = [("n01_1024x12000", ref.fill_normal(8, 1024 * 12000).reshape(1024, 12000).astype(np.float32), 3, 4),
         ("down", mistral_matrix(j), 2, j.seed)]
for name, a32, w, seed in cases:
    cfg = sc.DecomposeConfig(width=w, flush_width=1, record_curve=True, search=sc.SearchConfig(seed=seed))
    dec, rep, _ = eng.run(a32, cfg, dtype="f32")
    od = ref.greedy_decompose(a32.astype(np.float64), w, seed=seed, flush_width=1)
    same = [all((dec.factors[i][k] == od.signs[i][k]).all() for i in range(2)) for k in range(w)]
    print(name, "variant option %d" % eng.get_option("variant"), "identical", same, "gpu sweeps", rep.sweeps.tolist(),
          "ref", od.iterations.tolist(), "c", rep._cut_values.tolist(), od.cut_value.tolist(), flush=True)
