#!/usr/bin/env python
"""Benchmark: greedy signed cuts/sec on the 4096x4096 f32 matrix (BASELINE.json
config 2: i.i.d. N(0,1) from Xoshiro256pp seed 1, f32 storage, search seed 1).

One step = one greedy decomposition of `--width` cuts from the original matrix
(sigcut::greedy_decompose semantics, default 64 cuts) through the C ABI.
  value : cuts / device time, inputs resident in HBM (torch tensor, no H2D)
  e2e   : cuts / host wall time of the same call with a pinned HOST input
          (H2D of A, per-cut start vectors and D2H of S, T, c inside the step)
Multi-GPU (torchrun): every rank decomposes its own copy of the matrix (independent
units, no data-path collective) -> weak scaling; times are the max over ranks.

--impl reference times the reference's own CPU implementation (oracle/_ref, the
reference headers compiled unchanged) on all host cores: each step every worker
runs `--ref-cuts` cuts of the same decomposition (a bounded sample)."""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M = N = 4096
SEED = 1
METRIC = "signed cuts/sec at 4096x4096 f32; achieved HBM GB/s vs B200 peak"


def bench_config(width, world):
    """The workload description both arms print (the reference arm times a bounded
    sample of the same decomposition; its cpu_baseline.sample says which)."""
    return {"workload": "4096x4096 f32 N(0,1) seed 1 (BASELINE config 2, one copy per rank), greedy_decompose, "
                        f"{width} cuts per step from the original matrix",
            "cuts_per_step": width, "l2": "flushed (256 MB write) before every step; R (64 MiB) "
                                          "stays L2/SMEM-resident within a step",
            "parallelism": f"independent matrices x{world}"}


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """dram bytes per launch of the sweep kernel from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "latest_kernel_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


# ----------------------------------------------------------------- reference
_REF = {}


def _ref_worker_init():
    from oracle.pyoracle import Oracle

    o = Oracle("ref") if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libsigcut_ref.so")) else Oracle("orc")
    a = o.fill_normal(SEED, M * N).reshape(M, N).astype("float32").astype("float64")
    _REF["o"], _REF["a"] = o, a


def _ref_step(cuts):
    t = time.perf_counter()
    _REF["o"].greedy_decompose(_REF["a"], cuts, seed=SEED, want_iterations=False)
    return time.perf_counter() - t


def cpu_reference(steps, warmup, cuts, workers):
    import multiprocessing as mp

    from oracle.pyoracle import LIBS

    kind = "reference" if os.path.exists(LIBS["ref"]) else "port"
    ctx = mp.get_context("fork")
    with ctx.Pool(workers, initializer=_ref_worker_init) as pool:
        for _ in range(warmup):
            pool.map(_ref_step, [cuts] * workers)
        t0 = time.perf_counter()
        for _ in range(steps):
            pool.map(_ref_step, [cuts] * workers)
        dt = time.perf_counter() - t0
    return {"value": steps * workers * cuts / dt, "seconds": dt, "kind": kind, "cores": workers,
            "sample": f"{cuts} cuts of the 4096^2 decomposition (seed {SEED}, f32 data widened to f64) "
                      f"per worker per step, {workers} workers x {steps} steps"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    workers = args.ref_workers or os.cpu_count() or 1
    r = cpu_reference(args.steps, args.warmup, args.ref_cuts, workers)
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": "cuts/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["seconds"] / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args.width, world),
            "cpu_baseline": {"value": r["value"], "unit": "cuts/s", "cores": r["cores"], "kind": r["kind"],
                             "sample": r["sample"]},
            "e2e": {"value": r["value"], "unit": "cuts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------- ours
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--width", type=int, default=64, help="cuts per step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-cuts", type=int, default=2)
    ap.add_argument("--ref-workers", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    import paper_2410_01799_b200 as sc

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = local if world > 1 else 0
    torch.cuda.set_device(dev)
    eng = sc.Engine(dev)

    # each rank: its own copy of the BASELINE config-2 matrix (the same seed, so the
    # per-GPU work -- sweeps per cut -- is identical and N GPUs is pure weak scaling)
    seed = SEED
    a_host = torch.from_numpy(sc.fill_normal(seed, M * N, np.float32).reshape(M, N)).pin_memory()
    a_dev = a_host.cuda()
    cfg = sc.DecomposeConfig(width=args.width, search=sc.SearchConfig(seed=seed))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > L2 (126 MB)

    def step(src):
        flush.zero_()  # evict L2 between steps (outside the kernel's timed span)
        torch.cuda.synchronize()
        dec, rep, _ = eng.run(src, cfg, dtype="f32")
        return dec, rep

    for _ in range(args.warmup):
        step(a_dev)
    sampler = ClockSampler(dev)
    sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    kernel_ms, launches, alg_bytes, sweeps, passes = [], 0, 0.0, [], 0
    for _ in range(args.steps):
        dec, rep = step(a_dev)
        kernel_ms.append(rep.kernel_ms)
        launches += rep.kernel_launches
        alg_bytes += float(np.sum(2.0 * rep.sweeps.astype(np.float64) + 1.0)) * M * N * 4
        sweeps.extend(rep.sweeps.tolist())
        passes += rep.passes
    torch.cuda.synchronize()
    # end-to-end through the public API with a pinned host input
    e2e_ms, h2d, d2h = [], 0, 0
    for _ in range(max(2, args.steps // 2)):
        dec, rep = step(a_host.numpy())
        e2e_ms.append(rep.total_ms)
        h2d, d2h = rep.h2d_bytes, rep.d2h_bytes
    clocks = sampler.stop()
    dev_s = sum(kernel_ms) / 1e3
    e2e_s = sum(e2e_ms) / 1e3
    if world > 1:
        t = torch.tensor([dev_s, e2e_s / len(e2e_ms)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s, e2e_step_s = float(t[0]), float(t[1])
        dist.barrier()
    else:
        e2e_step_s = e2e_s / len(e2e_ms)
    total_cuts = args.steps * args.width * world
    value = total_cuts / dev_s
    peak, peak_src = measured_peak()
    achieved = alg_bytes / args.steps / (dev_s / args.steps) / 1e9  # algorithmic GB/s per launch
    traffic = ncu_traffic()
    line = {
        "metric": METRIC, "value": value, "unit": "cuts/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_s / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args.width, world),
        "e2e": {"value": args.width * world / e2e_step_s, "unit": "cuts/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": (traffic or {}).get("dram_bytes_per_launch"),
                     "l2_traffic": (traffic or {}).get("l2_bytes_per_launch"),
                     "peak_source": peak_src,
                     "algorithmic_bytes": "sum_j (2*sweeps_j+1)*m*n*4 per launch (SURVEY 8d)",
                     "passes_per_launch": passes / args.steps,
                     "physical_stream_bytes_per_launch": passes / args.steps * M * N * 4,
                     "note": "algorithmic bytes count every half-iteration as a full read of R (the "
                             "BASELINE formula); the engine reads less: one pass per sweep, R resident in "
                             "SMEM/L2, and sparse delta passes (flipped t columns / s rows only) between "
                             "dense refreshes, so frac can exceed 1; physical DRAM traffic is 'traffic', L2 traffic "
                             "(lts__t_sectors x 32 B, same ncu capture) is 'l2_traffic'"},
        "sweeps_per_cut_mean": float(np.mean(sweeps)),
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = cpu_reference(1, 0, 1, min(os.cpu_count() or 1, 16))
            line["cpu_baseline"] = {"value": r["value"], "unit": "cuts/s", "cores": r["cores"], "kind": r["kind"],
                                    "sample": r["sample"]}
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "unit": "cuts/s", "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
