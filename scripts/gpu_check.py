"""Quick GPU parity/timing probe used during development (not a test)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2410_01799_b200 as sc
from oracle.pyoracle import Oracle

ref = Oracle("ref") if os.path.exists(os.path.join("oracle", "_ref", "libsigcut_ref.so")) else Oracle("orc")
eng = sc.Engine(0)


def compare(name, a, w, seed, dtype, flush=1, restarts=1, max_sweeps=100, oracle_input=None):
    cfg = sc.DecomposeConfig(width=w, flush_width=flush, record_curve=True,
                             search=sc.SearchConfig(seed=seed, restarts=restarts, max_sweeps=max_sweeps))
    t = time.time()
    dec, rep, rem = eng.run(a, cfg, dtype=dtype, want_remainder=True)
    tg = time.time() - t
    oa = np.asarray(a, np.float64) if oracle_input is None else oracle_input
    t = time.time()
    od = ref.greedy_decompose(oa, w, seed=seed, flush_width=flush, restarts=restarts, max_sweeps=max_sweeps,
                              want_remainder=True)
    to = time.time() - t
    wd = min(dec.width(), od.width)
    first_div = None
    for k in range(wd):
        if not all((dec.factors[i][k] == od.signs[i][k]).all() for i in range(2)):
            first_div = k
            break
    upto = wd if first_div is None else first_div
    dc = np.max(np.abs(rep._cut_values[:upto] - od.cut_value[:upto]) / np.abs(od.cut_value[:upto])) if upto else 0
    sw = (rep.sweeps[:upto].astype(int) - od.iterations[:upto].astype(int))
    rel_g = rep.final_residual_norm / rep.input_norm
    rel_o = od.final_residual_norm / od.input_norm
    print(f"{name}: w={dec.width()}/{od.width} first_div={first_div} max_rel_dc={dc:.2e} "
          f"sweep_mismatch={np.count_nonzero(sw)} rel_err gpu={rel_g:.10f} ref={rel_o:.10f} "
          f"d={abs(rel_g-rel_o):.2e} kernel_ms={rep.kernel_ms:.2f} total={tg*1e3:.1f}ms cpu={to:.2f}s "
          f"passes={rep.passes} sweeps_mean={rep.sweeps.mean():.1f}", flush=True)
    if rem is not None and od.remainder is not None and first_div is None:
        print(f"   remainder max abs diff {np.max(np.abs(rem.astype(np.float64) - od.remainder)):.3e}")
    return dec, rep


# closed forms
r = eng.greedy_signed_cut(np.array([[1.0, -1.0], [-1.0, 1.0]]), sc.SearchConfig(seed=3, restarts=8))
print("2x2 alternating ->", r.value, r.iterations)
r = eng.greedy_signed_cut(np.ones((3, 3)), sc.SearchConfig(seed=1))
print("ones 3x3 ->", r.value)

for (m, n), w, seed, dt, rs in [((8, 8), 20, 1, "f64", 1), ((37, 29), 30, 3, "f64", 2), ((200, 150), 64, 8, "f64", 1),
                               ((300, 1000), 32, 9, "f64", 1), ((1000, 300), 32, 9, "f32", 3)]:
    a = ref.fill_normal(seed, m * n).reshape(m, n)
    if dt == "f32":
        a = a.astype(np.float32)
    compare(f"{m}x{n} {dt} rs{rs}", a, w, seed, dt, restarts=rs)

a = ref.fill_normal(0, 1024 * 1024).reshape(1024, 1024).astype(np.float32)
compare("C1 1024^2 f32 w256", a, 256, 0, "f32", flush=32)
a64 = ref.fill_normal(0, 1024 * 1024).reshape(1024, 1024)
compare("1024^2 f64 w128", a64, 128, 0, "f64", flush=32)

a = ref.fill_normal(1, 4096 * 4096).reshape(4096, 4096).astype(np.float32)
cfg = sc.DecomposeConfig(width=64, search=sc.SearchConfig(seed=1))
for it in range(3):
    dec, rep, _ = eng.run(a, cfg, dtype="f32")
    bytes_alg = float(np.sum(2 * rep.sweeps.astype(np.float64) + 1)) * 4096 * 4096 * 4
    print(f"4096^2 f32 w64: kernel {rep.kernel_ms:.2f} ms -> {64 / rep.kernel_ms * 1e3:.1f} cuts/s, "
          f"alg {bytes_alg / rep.kernel_ms / 1e6:.0f} GB/s, passes {rep.passes}, sweeps mean {rep.sweeps.mean():.1f}, "
          f"total {rep.total_ms:.1f} ms", flush=True)
od = ref.greedy_decompose(a.astype(np.float64), 4, seed=1)
print("4096 first 4 cuts sweeps gpu", rep.sweeps[:4], "ref", od.iterations, "c", rep._cut_values[:4], od.cut_value)

# sweep-count mismatch detail on the small f64 case
a = ref.fill_normal(1, 64).reshape(8, 8)
cfg = sc.DecomposeConfig(width=20, flush_width=1, search=sc.SearchConfig(seed=1))
dec, rep, _ = eng.run(a, cfg, dtype="f64")
od = ref.greedy_decompose(a, 20, seed=1, flush_width=1)
print("8x8 sweeps gpu", rep.sweeps.tolist())
print("8x8 sweeps ref", od.iterations.tolist())
print("8x8 c diff", (rep._cut_values - od.cut_value).tolist())
