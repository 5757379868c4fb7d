"""BASELINE config 2 width sweep: relative remainder ||R_w||_F / ||A||_F against
the width w on the 4096x4096 matrix (N(0,1) from Xoshiro256pp(1), f32 values),
in f32 storage and again in f64 storage, from w = 512 up to the bf16-equivalent
footprint and beyond it to the paper's Fig. 7 break-even with bf16 round-off
(bf16 rel. error 0.00166 at compression p = 0.2064, i.e.
w ~ 26,844 for f64 coefficients; the reference skips this as a multi-hour run,
proj/tests/acceptance.cpp:367-369).

One greedy_decompose call per dtype runs the whole width on the device; the
per-cut exact remainder norms (CutReport extras) give the whole curve.  The
bf16 / f16 round-off errors of the same matrix are computed on the host with
round-to-nearest-even (quantize_half, metrics.hpp:113-160).

usage: python scripts/width_curve.py [--f32-width 16376] [--f64-width 32640] > curve.jsonl
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_01799_b200 as sc  # noqa: E402
from paper_2410_01799_b200 import workloads as wl  # noqa: E402
from paper_2410_01799_b200.batch import round_bf16  # noqa: E402

M = N = 4096
CHECK = [512, 1024, 2048, 4096, 8192, 12000, 16320, 16376, 20000, 24000, 26844, 28000, 30000, 32640]


def compression(k, coeff_bits=64, source_bits=64):
    # compression_rate (metrics.hpp:46-52) under the f64 coefficient / f64 source model
    return k * (coeff_bits + M + N) / (source_bits * M * N)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--f32-width", type=int, default=16376)
    ap.add_argument("--f64-width", type=int, default=32640)
    args = ap.parse_args()
    a32 = wl.c2(np.float32)
    a64 = a32.astype(np.float64)
    na = float(np.linalg.norm(a64))
    e_bf16 = float(np.linalg.norm(round_bf16(a64) - a64)) / na
    e_f16 = float(np.linalg.norm(a64.astype(np.float16).astype(np.float64) - a64)) / na
    print(json.dumps({"matrix": "C2 4096x4096 N(0,1) seed 1 (f32 values)", "bf16_rel_error": e_bf16,
                      "f16_rel_error": e_f16, "paper_bf16": 0.00166, "paper_f16": 0.000208}), flush=True)
    eng = sc.Engine(0)
    for dtype, width, a in (("f32", args.f32_width, a32), ("f64", args.f64_width, a64)):
        if width <= 0:
            continue
        cfg = sc.DecomposeConfig(width=width, flush_width=32, record_curve=True, search=sc.SearchConfig(seed=1))
        dec, rep, _ = eng.run(a, cfg, dtype=dtype)
        rel = rep.residual_norm_exact / rep.input_norm
        sw = rep.sweeps.astype(np.float64)
        pts = {str(k): float(rel[k - 1]) for k in CHECK if k <= rep.width}
        cross = {}
        for name, e in (("bf16", e_bf16), ("f16", e_f16)):
            idx = np.nonzero(rel <= e)[0]
            if idx.size:
                k = int(idx[0]) + 1
                cross[name] = {"width": k, "compression_f64": compression(k), "rel_error": float(rel[k - 1])}
            else:
                cross[name] = None
        print(json.dumps({"dtype": dtype, "width": int(rep.width), "kernel_s": rep.kernel_ms / 1e3,
                          "cuts_per_s": rep.width / (rep.kernel_ms / 1e3), "sweeps_mean": float(sw.mean()),
                          "sweeps_max": int(sw.max()), "cap_hits": int((sw >= 100).sum()), "passes": rep.passes,
                          "rel_error_at": pts, "crossings": cross,
                          "curve_every_256": [float(x) for x in rel[255::256]]}), flush=True)


if __name__ == "__main__":
    main()
