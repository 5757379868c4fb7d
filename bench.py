#!/usr/bin/env python
"""Benchmark: greedy signed cuts/sec on the 4096x4096 f32 matrix (BASELINE.json
config 2: i.i.d. N(0,1) from Xoshiro256pp seed 1, f32 storage, search seed 1).

One step = one greedy decomposition of `--width` cuts (default 512, config 2's
smallest width) from the original matrix (sigcut::greedy_decompose semantics)
through the C ABI.
  value : cuts / device time of the decomposition kernel (CUDA events on the
          engine's stream), input already resident in HBM (torch tensor)
  e2e   : cuts / host wall time of the same public call with a pinned HOST input
          (H2D of A, per-cut start vectors, D2H of S, T, c inside the step)
  roofline.frac : PHYSICAL bytes the kernel moved through L2 / HBM (counted in the
          kernel: streamed rows, delta-pass gathers, rank-1 write-backs, column
          partial exchange) / launch time / measured HBM peak.  The BASELINE
          accounting ((2 sweeps + 1) m n 4 bytes per cut) is algorithmic_frac.
Multi-GPU: `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks (and fails loudly if fewer GPUs are visible).
Every rank decomposes its own copy of the matrix (independent units, no
data-path collective) -> weak scaling; times are the max over ranks.  At N > 1
the C4 batch prefix (Mistral-shaped jobs, LPT over the ranks) is reported too.

--impl reference times the reference's own CPU implementation (oracle/_ref, the
reference headers compiled unchanged; loaded in this process, then forked) on
all host cores: each step every worker runs the first `--ref-cuts` cuts of the
same decomposition (a bounded sample)."""
import argparse
import json
import os
import socket
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
SYNC_FLOOR_US = 1.25  # flat grid barrier over 148 CTAs on this B200 (scripts/micro/barrier3.cu): ends every dense pass
# Latency floor of one barrier-free delta pass: six dependent L2 trips -- the t words'
# store and poll, the column gather, the records' store and poll, the flipped-row gather -- at the
# ~250-cycle L2 hit latency of the microarchitecture guide, 1.965 GHz
DELTA_FLOOR_US = 6 * 250 / 1965.0


def bench_config(width, world):
    """The workload description both arms print (the reference arm times a bounded
    sample of the same decomposition; its cpu_baseline.sample says which)."""
    return {"workload": "4096x4096 f32 N(0,1) Xoshiro256pp(1) (BASELINE config 2), greedy_decompose from the "
                        f"original matrix, {width} cuts per step, search seed 1, one copy per rank",
            "cuts_per_step": width,
            "l2": "a 256 MB write flushes L2 before every step; the call's device copy of A into the engine "
                  "arena (before the kernel's timed span) leaves R L2-resident, and R (64 MiB) then stays "
                  "SMEM/L2-resident for the whole decomposition",
            "parallelism": f"independent matrices x{world}"}


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def spawn(args):
    """`--gpus N` outside torchrun: re-launch under torch.distributed.run (one rank per GPU)."""
    try:
        import torch

        have = torch.cuda.device_count()
    except Exception:
        have = 0
    if args.impl == "ours" and have < args.gpus:
        print(f"bench.py --gpus {args.gpus}: only {have} GPU(s) visible; refusing to run fewer ranks",
              file=sys.stderr)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


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
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(width):
    """DRAM / L2 bytes per launch of the sweep kernel from the committed ncu --set full
    capture of this same bench workload (profiles/latest_kernel_traffic.json), if the
    capture's cuts per launch match."""
    p = os.path.join(ROOT, "profiles", "latest_kernel_traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        return t if int(t.get("cuts_per_launch", -1)) == width else None
    except Exception:
        return None


# ----------------------------------------------------------------- reference
_REF = {}


def _ref_load():
    """Load the reference library and the matrix in THIS process (forked workers inherit both)."""
    from oracle.pyoracle import LIBS, Oracle

    kind = "reference" if os.path.exists(LIBS["ref"]) else "port"
    o = Oracle("ref") if kind == "reference" else Oracle("orc")
    a = o.fill_normal(SEED, M * N).reshape(M, N).astype("float32").astype("float64")
    _REF["o"], _REF["a"], _REF["kind"] = o, a, kind


def _ref_step(cuts):
    t = time.perf_counter()
    d = _REF["o"].greedy_decompose(_REF["a"], cuts, seed=SEED, want_iterations=True)
    return time.perf_counter() - t, [int(x) for x in d.iterations]


def cpu_reference(steps, warmup, cuts, workers):
    import multiprocessing as mp

    if "o" not in _REF:
        _ref_load()
    ctx = mp.get_context("fork")
    sweeps = []
    with ctx.Pool(workers) as pool:
        for _ in range(warmup):
            pool.map(_ref_step, [cuts] * workers)
        t0 = time.perf_counter()
        for _ in range(steps):
            for _, it in pool.map(_ref_step, [cuts] * workers):
                sweeps.extend(it)
        dt = time.perf_counter() - t0
    return {"value": steps * workers * cuts / dt, "seconds": dt, "kind": _REF["kind"], "cores": workers,
            "sweeps_mean": float(sum(sweeps) / max(1, len(sweeps))),
            "sample": f"the first {cuts} cuts of the same 4096^2 decomposition (seed {SEED}, f32 data widened "
                      f"to f64, the reference's own arithmetic) per worker per step, {workers} single-threaded "
                      f"workers x {steps} steps"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    workers = args.ref_workers or min(os.cpu_count() or 1, 64)
    _ref_load()  # in the parent: the reference library is loaded by the process the driver watches
    r = cpu_reference(args.steps, args.warmup, args.ref_cuts, workers)
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": "cuts/s",
            "n_gpus": max(args.gpus, world), "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["seconds"] / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": bench_config(args.width, world),
            "cpu_baseline": {"value": r["value"], "unit": "cuts/s", "cores": r["cores"], "kind": r["kind"],
                             "sample": r["sample"], "sweeps_per_cut_mean": r["sweeps_mean"]},
            "e2e": {"value": r["value"], "unit": "cuts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------- ours
def batch_prefix(local, world, rank, jobs_n, cuts, gather):
    """C4 prefix: the first `jobs_n` Mistral-shaped jobs x `cuts` cuts, LPT over the ranks."""
    import numpy as np

    from paper_2410_01799_b200 import batch
    from paper_2410_01799_b200.api import DecomposeConfig, Engine, SearchConfig

    eng = Engine(local)
    jobs = [batch.Job(j.index, j.name, j.shape, min(j.width, cuts), j.seed) for j in batch.mistral_jobs()[:jobs_n]]

    def execute(job, a):
        dec, rep, _ = eng.run(a, DecomposeConfig(width=job.width, search=SearchConfig(seed=job.seed)), dtype="f32")
        return {"cuts": dec.width(), "device_s": rep.kernel_ms / 1e3,
                "sweeps_mean": float(np.mean(rep.sweeps)) if len(rep.sweeps) else 0.0}

    res = batch.run_batch(jobs, rank, world, execute, gather, prepare=batch.mistral_matrix)
    eng.close()
    return {"jobs": jobs_n, "cuts_per_job": cuts, "cuts": res["cuts"], "device_s_max_rank": res["device_s"],
            "value": res["cuts"] / res["device_s"], "unit": "cuts/s", "scaling": "strong (fixed job set, LPT)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--width", type=int, default=512, help="cuts per step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-cuts", type=int, default=4, help="reference arm: cuts per worker per step")
    ap.add_argument("--ref-workers", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch-jobs", type=int, default=14, help="N > 1: C4 prefix jobs reported beside the line")
    ap.add_argument("--batch-cuts", type=int, default=32)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
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
    a_host = torch.from_numpy(sc.fill_normal(SEED, M * N, np.float32).reshape(M, N)).pin_memory()
    a_dev = a_host.cuda()
    cfg = sc.DecomposeConfig(width=args.width, search=sc.SearchConfig(seed=SEED))
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
    kernel_ms, launches, alg_bytes, sweeps, passes, dense, delta, phys = [], 0, 0.0, [], 0, 0, 0, 0
    for _ in range(args.steps):
        dec, rep = step(a_dev)
        kernel_ms.append(rep.kernel_ms)
        launches += rep.kernel_launches
        alg_bytes += float(np.sum(2.0 * rep.sweeps.astype(np.float64) + 1.0)) * M * N * 4
        sweeps.extend(rep.sweeps.tolist())
        passes += rep.passes
        dense += rep.dense_passes
        delta += rep.delta_passes
        phys += rep.device_bytes
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
    launch_s = dev_s / args.steps
    alg_gbs = alg_bytes / args.steps / launch_s / 1e9  # BASELINE accounting
    phys_per_launch = phys / args.steps
    phys_gbs = phys_per_launch / launch_s / 1e9
    traffic = ncu_traffic(args.width)
    passes_l = passes / args.steps
    us_per_pass = launch_s * 1e6 / max(1.0, passes_l)
    line = {
        "metric": METRIC, "value": value, "unit": "cuts/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": launch_s * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args.width, world),
        "e2e": {"value": args.width * world / e2e_step_s, "unit": "cuts/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": launches,
        "roofline": {
            "bound": "hbm", "achieved": phys_gbs, "peak": peak, "unit": "GB/s", "frac": phys_gbs / peak,
            "traffic": (traffic or {}).get("dram_bytes_per_launch"),
            "l2_traffic": (traffic or {}).get("l2_bytes_per_launch"),
            "traffic_source": (traffic or {}).get("source"),
            "peak_source": peak_src,
            "achieved_is": "physical bytes the kernel moved through L2/HBM per launch (sc_result.device_bytes, "
                           "counted in the kernel: streamed rows of R, delta-pass gathers at 32 B sectors, "
                           "rank-1 write-backs, column-partial exchange; SMEM-resident rows excluded) / launch "
                           "time",
            "physical_bytes_per_launch": phys_per_launch,
            "algorithmic_achieved": alg_gbs, "algorithmic_frac": alg_gbs / peak,
            "algorithmic_bytes": "sum_j (2*sweeps_j+1)*m*n*4 per launch (SURVEY 8d / BASELINE); counts every "
                                 "half-iteration as a full read of R, so it exceeds 1 when R is on chip",
            "binding": "per-pass exchange latency: R is on chip; a delta pass (95% of the passes) is a chain "
                       "of two publish->poll exchanges and two L2 gathers with no grid barrier in it, a dense "
                       "pass streams R from SMEM/L2 and ends in one grid barrier (DESIGN.md 4.6, 5)",
            "latency_model": {"passes_per_launch": passes_l, "dense_passes_per_launch": dense / args.steps,
                              "delta_passes_per_launch": delta / args.steps, "us_per_pass": us_per_pass,
                              "delta_pass_floor_us": DELTA_FLOOR_US, "grid_sync_floor_us": SYNC_FLOOR_US,
                              "floor_is": "six dependent L2 trips per delta pass at the 250-cycle L2 hit latency",
                              "floor_frac": DELTA_FLOOR_US / us_per_pass},
        },
        "sweeps_per_cut_mean": float(np.mean(sweeps)),
        "clocks": clocks,
    }
    if world > 1:
        def gather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out

        try:
            line["batch_c4_prefix"] = batch_prefix(local, world, rank, args.batch_jobs, args.batch_cuts, gather)
        except Exception as e:  # reported beside the line, never required
            line["batch_c4_prefix"] = {"error": repr(e)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = cpu_reference(1, 0, args.ref_cuts, min(os.cpu_count() or 1, 16))
            line["cpu_baseline"] = {"value": r["value"], "unit": "cuts/s", "cores": r["cores"], "kind": r["kind"],
                                    "sample": r["sample"], "sweeps_per_cut_mean": r["sweeps_mean"]}
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
