"""Same-box, same-process A/B of engine options (sc_set_option):
AB_OPTS="fuse_update=1;fuse_update=0|delta=0" alternates the settings (";" between
settings, "|" between options) for AB_ROUNDS rounds on the 4096^2 f32 config-2
matrix (or AB_SHAPE), AB_W cuts per call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2410_01799_b200 as sc  # noqa: E402

M, N = (int(x) for x in os.environ.get("AB_SHAPE", "4096,4096").split(","))
SEED = int(os.environ.get("AB_SEED", 1))
dtype = os.environ.get("AB_DTYPE", "f32")
a = sc.fill_normal(SEED, M * N, np.float32).reshape(M, N)
if dtype == "f64":
    a = a.astype(np.float64)
cfg = sc.DecomposeConfig(width=int(os.environ.get("AB_W", 512)), search=sc.SearchConfig(seed=SEED))
settings = [s for s in os.environ.get("AB_OPTS", "").split(";")]
eng = sc.Engine(0)
eng.run(a, sc.DecomposeConfig(width=4, search=sc.SearchConfig(seed=SEED)), dtype=dtype)
res = {}
for rnd in range(int(os.environ.get("AB_ROUNDS", 3))):
    for st in settings:
        kv = {k: int(v) for k, v in (x.split("=", 1) for x in st.split("|") if x)}
        with eng.options(**kv):
            dec, rep, _ = eng.run(a, cfg, dtype=dtype)
        res.setdefault(st, []).append((rep.kernel_ms, rep.passes, rep.dense_passes, rep.delta_passes,
                                       hash(dec.factors[0].tobytes())))
for st, v in res.items():
    ms = [x[0] for x in v]
    print(f"{st or '(default)':40s} ms {['%.1f' % m for m in ms]} min {min(ms):.1f} cuts/s {cfg.width / min(ms) * 1e3:.1f}"
          f" passes {v[0][1]} dense {v[0][2]} delta {v[0][3]} us/pass {min(ms) * 1e3 / v[0][1]:.2f} sig {v[0][4] & 0xffff}")
