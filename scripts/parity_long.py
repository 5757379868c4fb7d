"""Longer trajectories at full size against the reference: the C4 shapes in f64
storage (the reference's own arithmetic: signs must stay identical cut after cut) and in f32
storage (first divergent cut, then lockstep: the reference's single cut on the GPU's own
remainder must reproduce the GPU's cut), and C3 (order 3).  CPU reference time bounds the cut counts."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
from oracle.pyoracle import Oracle
from paper_2410_01799_b200.batch import mistral_jobs, mistral_matrix
from paper_2410_01799_b200 import workloads as wl

ref = Oracle("ref")
eng = sc.Engine(0)
jobs = mistral_jobs()


def sweeps_ok(gs, rs):
    gs, rs = np.asarray(gs, int), np.asarray(rs, int)
    return bool(np.all((gs == rs) | ((gs % 16 == 0) & (rs == gs + 1))))


def first_bad(dec, od, w, order):
    for k in range(w):
        if not all((dec.factors[i][k] == od.signs[i][k]).all() for i in range(order)):
            return k
    return None


for idx, w in ((0, 48), (1, 48), (4, 12), (6, 12), (224, 6)):
    j = jobs[idx]
    a = mistral_matrix(j)
    t0 = time.time()
    od = ref.greedy_decompose(a.astype(np.float64), w, seed=j.seed, flush_width=1)
    cpu = time.time() - t0
    for dtype in ("f64", "f32"):
        cfg = sc.DecomposeConfig(width=w, flush_width=1, record_curve=True, search=sc.SearchConfig(seed=j.seed))
        dec, rep, _ = eng.run(a if dtype == "f32" else a.astype(np.float64), cfg, dtype=dtype)
        fb = first_bad(dec, od, w, 2)
        upto = w if fb is None else fb
        print(f"{j.name} {j.shape} {dtype} storage, {w} cuts: first divergent cut {fb}; sweeps ok to there "
              f"{sweeps_ok(rep.sweeps[:upto], od.iterations[:upto])}; max rel dc to there "
              f"{(np.max(np.abs(rep._cut_values[:upto] - od.cut_value[:upto]) / od.cut_value[:upto]) if upto else 0):.2e}; "
              f"rel residual gpu {rep.final_residual_norm / rep.input_norm:.6f} ref {od.final_residual_norm / od.input_norm:.6f}; cpu {cpu:.0f}s",
              flush=True)

a3 = wl.c3_blob_image()
w = 12
t0 = time.time()
od = ref.greedy_decompose(a3.astype(np.float64), w, seed=2, flush_width=1)
cpu = time.time() - t0
for dtype in ("f64", "f32"):
    cfg = sc.DecomposeConfig(width=w, flush_width=1, record_curve=True, search=sc.SearchConfig(seed=2))
    dec, rep, _ = eng.run(a3.astype(np.float32) if dtype == "f32" else a3.astype(np.float64), cfg, dtype=dtype)
    fb = first_bad(dec, od, w, 3)
    upto = w if fb is None else fb
    print(f"C3 4000x3000x3 {dtype} storage, {w} cuts: first divergent cut {fb}; sweeps ok to there "
          f"{sweeps_ok(rep.sweeps[:upto], od.iterations[:upto])}; cpu {cpu:.0f}s", flush=True)
