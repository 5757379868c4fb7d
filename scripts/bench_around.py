"""Measurements of the rows around the path on one B200.

One JSON line per workload (device time from CUDA events inside the C ABI;
e2e = the public call with host buffers, copies included):

  expand   BASELINE C2 at the bf16-equivalent width: 4096 x 4096, w = 16320
           terms (random signs, decaying coefficients) -> 2.74e11 dependent f64
           additions.  Roofline: FP64 pipe (64 DFMA lanes / clk / SM measured,
           scripts/micro/fp64lat.cu) x 148 SMs x the SM clock under load.
  gram     w = 16320 Gram matrix of the same factors (XOR-popcount).
  lstsq    least-squares decomposition, 512 x 512 f64, w = 64.

The reference CPU arm (oracle/_ref, reference headers compiled unchanged) runs
the same arithmetic on a bounded sample (rows of the same matrix), 1 thread.

usage: python scripts/bench_around.py [--no-cpu] [--only expand,gram,lstsq]
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_01799_b200 as sc  # noqa: E402


def rand_factors(shape, w, seed):
    rng = np.random.default_rng(seed)
    fs = []
    for n in shape:
        nw = (n + 63) // 64
        f = rng.integers(0, 1 << 63, size=(w, nw), dtype=np.uint64) * np.uint64(2)
        f ^= rng.integers(0, 2, size=(w, nw), dtype=np.uint64)
        if n % 64:
            f[:, -1] &= np.uint64((1 << (n % 64)) - 1)
        fs.append(f)
    co = 0.04 * np.exp(-np.arange(w) / 8000.0)
    return sc.CutDecomposition(tuple(shape), fs, co)


class Clocks:
    def __init__(self):
        self.samples, self.reasons, self.stop = [], set(), False

    def run(self):
        while not self.stop:
            try:
                out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks_throttle_reasons.active",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip().split(",")
                self.samples.append(float(out[0]))
                mask = int(out[1], 16)
                names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                         0x4: "sw_power_cap"}
                self.reasons |= {v for k, v in names.items() if mask & k}
            except Exception:
                pass
            time.sleep(0.2)

    def __enter__(self):
        self.t = threading.Thread(target=self.run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop = True
        self.t.join()

    def summary(self):
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "reasons": sorted(self.reasons), "samples": len(s)}


def fp64_peak(sm_mhz):
    return 64 * 148 * sm_mhz * 1e6  # DFMA lanes / s


def bench_expand(eng, args):
    m = n = 4096
    w = 16320
    d = rand_factors((m, n), w, 1)
    import torch

    out = torch.zeros((m, n), dtype=torch.float64, device="cuda")
    for _ in range(2):
        eng.accumulate_expansion(d, out, first_term=0)
    times = []
    with Clocks() as ck:
        for _ in range(args.steps):
            out.zero_()
            st = {}
            eng.accumulate_expansion(d, out, stats=st)
            times.append(st["kernel_ms"])
        st = {}
        t0 = time.perf_counter()
        host = eng.expand(d, stats=st)  # public call, host output (D2H of 128 MiB inside)
        e2e_s = time.perf_counter() - t0
    ms = float(np.median(times))
    ops = float(m) * n * w
    clk = ck.summary()
    peak = fp64_peak(clk["sm_mhz"] or 1965.0)
    line = {"metric": "expansion element-terms/s (expand, 4096x4096, w=16320)", "value": ops / (ms * 1e-3),
            "unit": "element-terms/s", "ms": ms, "dtype": "f64",
            "config": {"workload": "expand 4096x4096 w=16320 (BASELINE C2 bf16-equivalent width), random signs"},
            "roofline": {"bound": "fp64", "achieved": ops / (ms * 1e-3) / 1e12, "peak": peak / 1e12,
                         "unit": "TDFMA/s", "frac": ops / (ms * 1e-3) / peak,
                         "peak_source": "64 DFMA lanes/clk/SM (scripts/micro/fp64lat.cu) x 148 SMs x SM clock"},
            "e2e": {"value": ops / e2e_s, "unit": "element-terms/s", "h2d_bytes": st["h2d_bytes"],
                    "d2h_bytes": st["d2h_bytes"]},
            "bit_exact_check": "tests/test_around_gpu.py (reference accumulate_expansion)", "clocks": clk}
    if not args.no_cpu:
        from oracle.pyoracle import Oracle

        ref = Oracle("ref")
        rows = 4
        t0 = time.perf_counter()
        ref.accumulate_expansion((rows, n), [d.factors[0][:, :1] & np.uint64((1 << rows) - 1), d.factors[1]],
                                 d.coefficients)
        cpu_s = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": rows * n * w / cpu_s, "unit": "element-terms/s", "cores": 1,
                                "kind": "reference", "sample": f"{rows} x {n} rows, same {w} terms"}
    return line


def bench_gram(eng, args):
    d = rand_factors((4096, 4096), 16320, 2)
    eng.gram_matrix(sc.truncated(d, 256))
    st = {}
    t0 = time.perf_counter()
    g = eng.gram_matrix(d, stats=st)
    s = time.perf_counter() - t0
    pairs = float(d.width()) ** 2
    words = 2 * (64 + 64)  # u32 words per pair (two 4096-long axes)
    ms = st["kernel_ms"]
    return {"metric": "Gram entries/s (w=16320, 4096x4096 factors)", "value": pairs / (ms * 1e-3), "unit": "entries/s",
            "kernel_ms": ms, "ms_e2e": s * 1e3, "d2h_bytes": st["d2h_bytes"],
            "popc_per_s": pairs * words / (ms * 1e-3), "diag_ok": bool((np.diag(g) == 4096.0 * 4096.0).all())}


def bench_lstsq(eng, args):
    from oracle.pyoracle import Oracle

    a = Oracle("orc").fill_normal(5, 512 * 512).reshape(512, 512)
    cfg = sc.DecomposeConfig(width=64, search=sc.SearchConfig(seed=5))
    eng.lstsq_decompose(a, sc.DecomposeConfig(width=2, search=sc.SearchConfig(seed=5)))
    t0 = time.perf_counter()
    dec, rep = eng.lstsq_decompose(a, cfg)
    s = time.perf_counter() - t0
    line = {"metric": "lstsq_decompose terms/s (512x512 f64, w=64)", "value": 64 / s, "unit": "terms/s",
            "rel_err": rep.final_residual_norm / rep.input_norm, "kernel_ms": rep.kernel_ms}
    if not args.no_cpu:
        ref = Oracle("ref")
        t0 = time.perf_counter()
        r = ref.lstsq_decompose(a, 16, seed=5)
        cs = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": 16 / cs, "unit": "terms/s", "cores": 1, "kind": "reference",
                                "sample": "first 16 terms of the same decomposition"}
        line["signs_match_first16"] = bool(all((x[:16] == y).all() for x, y in zip(dec.factors, r.signs)))
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--only", default="expand,gram,lstsq")
    args = ap.parse_args()
    eng = sc.Engine(0)
    for name in args.only.split(","):
        line = {"expand": bench_expand, "gram": bench_gram, "lstsq": bench_lstsq}[name](eng, args)
        line["workload"] = name
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
