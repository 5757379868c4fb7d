"""Per-configuration measurements of the decomposition on one B200 (BASELINE.json
configs C1-C4; C5 single-GPU is scripts/c5 in sharded.py), with the reference CPU
implementation (oracle/_ref, headers compiled unchanged, 1 thread) timed beside
it on a bounded sample of the same input.

Each line: cuts/s on the device (CUDA events around the persistent kernel),
mean sweeps per cut, the algorithmic GB/s of SURVEY §8d
(sum_j (2 sweeps_j + 1) m n B, order k: k sweeps_j numel B) against the
measured HBM peak, the relative remainder ||R_w|| / ||A||, and -- where the
CPU can finish -- parity against the reference on the same input.

usage: python scripts/bench_configs.py [--only c1,c2,c2f64,c3,c4] [--no-cpu]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_01799_b200 as sc  # noqa: E402
from paper_2410_01799_b200 import workloads as wl  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6526.5


def run(eng, a, width, seed, dtype, record=True):
    cfg = sc.DecomposeConfig(width=width, flush_width=32, record_curve=record, search=sc.SearchConfig(seed=seed))
    dec, rep, _ = eng.run(a, cfg, dtype=dtype)
    return dec, rep


def line(name, a, dec, rep, dtype, extra=None):
    es = 4 if dtype == "f32" else 8
    numel = float(np.prod(a.shape))
    sw = rep.sweeps.astype(np.float64)
    k = a.ndim
    alg = float(((2 * sw + 1) if k == 2 else k * sw).sum()) * numel * es
    s = rep.kernel_ms * 1e-3
    d = {"config": name, "shape": list(a.shape), "dtype": dtype, "width": int(rep.width),
         "cuts_per_s": rep.width / s, "kernel_s": s, "sweeps_mean": float(sw.mean()), "sweeps_max": int(sw.max()),
         "passes": rep.passes, "algorithmic_GBps": alg / s / 1e9, "hbm_peak_GBps": peak(),
         "frac_algorithmic": alg / s / 1e9 / peak(),
         "physical_GBps": rep.device_bytes / s / 1e9, "frac_physical": rep.device_bytes / s / 1e9 / peak(),
         "dense_passes": rep.dense_passes, "delta_passes": rep.delta_passes,
         "us_per_pass": rep.kernel_ms * 1e3 / max(1, rep.passes),
         "rel_residual": rep.final_residual_norm / rep.input_norm,
         "e2e_s": rep.total_ms * 1e-3, "kernel_launches": rep.kernel_launches}
    if extra:
        d.update(extra)
    print(json.dumps(d), flush=True)


def cpu_ref(a, width, seed):
    from oracle.pyoracle import Oracle

    ref = Oracle("ref")
    t0 = time.perf_counter()
    od = ref.greedy_decompose(np.asarray(a, np.float64), width, seed=seed, want_iterations=False)
    return od, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c2,c2f64,c3,c4")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    eng = sc.Engine(0)
    todo = args.only.split(",")
    if "c1" in todo:
        for dtype in ("f32", "f64"):
            a = wl.c1(np.float32)
            a = a if dtype == "f32" else a.astype(np.float64)
            run(eng, a, 8, 0, dtype)
            dec, rep = run(eng, a, 256, 0, dtype)
            extra = {}
            if not args.no_cpu:
                od, cs = cpu_ref(a, 256, 0)
                same = [all((dec.factors[i][k] == od.signs[i][k]).all() for i in range(2)) for k in range(256)]
                first_div = next((k for k, ok in enumerate(same) if not ok), None)
                extra = {"cpu_baseline": {"value": 256 / cs, "unit": "cuts/s", "cores": 1, "kind": "reference",
                                          "sample": "full C1 decomposition (256 cuts)"},
                         "parity": {"identical_terms": int(sum(same)), "first_divergent_term": first_div,
                                    "rel_residual_ref": od.final_residual_norm / od.input_norm}}
            line(f"C1 1024x1024 w=256 ({dtype} storage)", a, dec, rep, dtype, extra)
    for key, dtype in (("c2", "f32"), ("c2f64", "f64")):
        if key not in todo:
            continue
        a = wl.c2(np.float32 if dtype == "f32" else np.float64)
        run(eng, a, 4, 1, dtype)
        dec, rep = run(eng, a, 512, 1, dtype)
        curve = {str(w): rep.steps[w - 1].residual_norm / rep.input_norm for w in (64, 128, 256, 512)}
        extra = {"rel_error_curve": curve}
        if not args.no_cpu:
            od, cs = cpu_ref(a, 2, 1)
            extra["cpu_baseline"] = {"value": 2 / cs, "unit": "cuts/s", "cores": 1, "kind": "reference",
                                     "sample": "first 2 cuts of the same decomposition"}
            extra["parity_first2"] = bool(all((dec.factors[i][:2] == od.signs[i]).all() for i in range(2)))
        line(f"C2 4096x4096 w=512 ({dtype} storage)", a, dec, rep, dtype, extra)
    if "c3" in todo:
        img = wl.c3_blob_image()
        run(eng, img, 4, 2, "f32")
        dec, rep = run(eng, img, 1024, 2, "f32")
        curve = {str(w): rep.steps[w - 1].residual_norm / rep.input_norm for w in (64, 128, 256, 512, 1024)}
        extra = {"rel_error_curve": curve}
        if not args.no_cpu:
            od, cs = cpu_ref(img, 2, 2)
            extra["cpu_baseline"] = {"value": 2 / cs, "unit": "cuts/s", "cores": 1, "kind": "reference",
                                     "sample": "first 2 cuts of the same decomposition"}
            extra["parity_first2"] = bool(all((dec.factors[i][:2] == od.signs[i]).all() for i in range(3)))
        line("C3 4000x3000x3 blob image f32, widths to 1024", img, dec, rep, "f32", extra)
    if "c4" in todo:
        from paper_2410_01799_b200.batch import mistral_jobs, mistral_matrix

        jobs = mistral_jobs()
        for idx in (0, 1, 4, 6, 224):  # q, k, gate, down, embed shapes
            j = jobs[idx]
            a = mistral_matrix(j)
            run(eng, a, 2, j.seed, "f32")  # warm-up: first use of a kernel variant in the process
            dec, rep = run(eng, a, 64, j.seed, "f32")
            line(f"C4 {j.name} {j.shape[0]}x{j.shape[1]} first 64 of w={j.width}", a, dec, rep, "f32")


if __name__ == "__main__":
    main()
