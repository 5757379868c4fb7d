"""Small ragged cases through every kernel, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
from paper_2410_01799_b200 import io as scio
eng = sc.Engine(0)
rng = np.random.default_rng(1)
for shape, dt in [((37, 70), "f32"), ((70, 37), "f64"), ((5, 6, 7), "f64"), ((130,), "f32")]:
    a = rng.standard_normal(shape)
    dec, rep, rem = eng.run(a.astype(np.float32) if dt == "f32" else a,
                            sc.DecomposeConfig(width=5, record_curve=True, search=sc.SearchConfig(seed=3, restarts=2)),
                            dtype=dt, want_remainder=True)
    x = eng.expand(dec)
    g = eng.gram_matrix(dec)
    r = eng.contract_terms(dec, a)
    d2, r2 = eng.lstsq_decompose(a, sc.DecomposeConfig(width=3, search=sc.SearchConfig(seed=2)))
    print(shape, dt, "ok", rep.sweeps.tolist(), float(np.abs(x).max()), g.shape, r.shape, d2.width())
img = rng.random((9, 11, 3))
d3, r3 = eng.rgb_scalars_decompose(img, sc.DecomposeConfig(width=3))
print("rgb ok", d3.coefficients.shape, scio.read_scd(scio.write_scd(d3)).width())
