"""Multi-GPU batch of independent decompositions.

A batch of independent matrices needs no data-path collective: the host costs
every job as ``w·m·n`` (the per-pass bytes times the width; the mean sweep
count is shape-independent to first order), assigns jobs to devices longest
processing time first (``sc_lpt_schedule``), and each rank -- one process per
GPU under torchrun -- decomposes its own jobs on its own engine. Only small
per-job summaries travel (``all_gather_object``), and the batch's device time is
the max over ranks.

The C4 job set is the Mistral-7B weight inventory in layer order (32 layers of
q, k, v, o, gate, up, down; then embed and lm_head: 226 matrices) at the widths
of paper Table 2 (``width_for_compression``, metrics.hpp:55-63, 32-bit
coefficients over a 16-bit source at rate 0.5). The real weights are not in the
container; each matrix is synthesised on the host from the reference's
generator: ``Xoshiro256pp(substream(3, i))`` draws U (m×64), V (n×64) and then the
m·n noise terms as one normal stream, ``L = 0.015·U Vᵀ / 8 + 0.02·noise`` rounded
to bf16 (round to nearest even, as ``quantize_half(kBf16)``, metrics.hpp:113-160)
and stored as f32.

CLI (one rank per GPU)::

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        -m paper_2410_01799_b200.batch --jobs 14 --prefix-cuts 64
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

MASK64 = (1 << 64) - 1

# (name, m, n) per transformer layer, then the two vocabulary matrices
LAYER = (("q", 4096, 4096), ("k", 1024, 4096), ("v", 1024, 4096), ("o", 4096, 4096),
         ("gate", 14336, 4096), ("up", 14336, 4096), ("down", 4096, 14336))
VOCAB = (("embed", 32000, 4096), ("lm_head", 32000, 4096))


def mix64(z: int) -> int:
    """rng.hpp:10-17 (restated in csrc/rng.h)."""
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def substream(seed: int, index: int) -> int:
    """rng.hpp:19-24: independent stream ``index`` of ``seed``."""
    return mix64((seed ^ ((0xD1342543DE82EF95 * (index + 1)) & MASK64)) & MASK64)


@dataclass(frozen=True)
class Job:
    index: int
    name: str
    shape: tuple
    width: int
    seed: int

    @property
    def cost(self) -> float:
        m, n = self.shape
        return float(self.width) * float(m) * float(n)


def mistral_jobs(rate: float = 0.5, layers: int = 32, coeff_bits: int = 32, source_bits: int = 16,
                 base_seed: int = 3) -> List[Job]:
    from .api import width_for_compression

    shapes = [(f"layers.{l}.{nm}", m, n) for l in range(layers) for nm, m, n in LAYER] + list(VOCAB)
    jobs = []
    for i, (nm, m, n) in enumerate(shapes):
        w = width_for_compression((m, n), rate, coeff_bits=coeff_bits, source_bits=source_bits)
        jobs.append(Job(i, nm, (m, n), w, substream(base_seed, i)))
    return jobs


def round_bf16(x: np.ndarray) -> np.ndarray:
    """f64 -> nearest bf16 (ties to even) -> f64; finite inputs in the normal range."""
    x = np.asarray(x, np.float64)
    f, e = np.frexp(x)  # x = f * 2**e, 0.5 <= |f| < 1
    return np.ldexp(np.rint(f * 256.0) / 256.0, e)


def mistral_matrix(job: Job, rank_k: int = 64) -> np.ndarray:
    """Synthetic stand-in for the job's weight matrix (see module docstring)."""
    from .api import fill_normal

    m, n = job.shape
    z = fill_normal(job.seed, m * rank_k + n * rank_k + m * n)
    u = z[: m * rank_k].reshape(m, rank_k)
    v = z[m * rank_k: (m + n) * rank_k].reshape(n, rank_k)
    noise = z[(m + n) * rank_k:].reshape(m, n)
    low = (0.015 / 8.0) * (u @ v.T)
    return round_bf16(low + 0.02 * noise).astype(np.float32)


def plan(jobs: Sequence[Job], world: int) -> np.ndarray:
    """Bin (rank) of every job: LPT over the job costs (deterministic, ties by index)."""
    from .api import lpt_schedule

    return lpt_schedule(np.array([j.cost for j in jobs]), world)


def run_batch(jobs: Sequence[Job], rank: int, world: int,
              execute: Callable[..., Dict], gather: Optional[Callable[[list], List[list]]] = None,
              prepare: Optional[Callable[[Job], object]] = None,
              pair: Optional[Callable[[Job], bool]] = None, lookahead: int = 1) -> Dict:
    """Run this rank's share and collect every rank's summaries.

    ``execute(job)`` returns a dict summary (it must contain ``cuts`` and
    ``device_s``); ``gather(list) -> list of lists`` is the collective used to
    bring summaries together (``torch.distributed.all_gather_object``), None for a
    single process.  With ``prepare(job)`` (host-side input synthesis), the next
    job's input is prepared on a background thread while the device works on the
    current one (the engine call releases the GIL), and ``execute(job, data)`` is
    called; ``lookahead`` jobs are prepared concurrently (host threads; numpy
    releases the GIL).  With ``pair(job)``, the jobs it accepts (the sync-bound small
    shapes, which sort to the tail of the longest-first order) run two at a time
    on two host threads as ``execute(job, data, lane)``, lane 0 or 1, each lane
    on its own engine with half the grid (1024×4096 jobs +76%); the
    pair's device time is the wall time of the pair, which also covers the
    gap between the two launches.  Returns ``{"jobs": [...by index],
    "device_s": max over ranks, "cuts": total}``.
    """
    jobs = list(jobs)
    index_of = {j.index: k for k, j in enumerate(jobs)}
    bins = plan(jobs, world)
    mine = [j for j in jobs if int(bins[index_of[j.index]]) == rank]
    mine.sort(key=lambda j: (-j.cost, j.index))
    out = []
    dev = 0.0
    solo = [j for j in mine if pair is None or not pair(j)]
    duo = [j for j in mine if pair is not None and pair(j)]
    order = solo + duo
    la = max(1, int(lookahead))
    pool = ThreadPoolExecutor(max_workers=la) if prepare is not None and order else None
    ahead = {k: pool.submit(prepare, order[k]) for k in range(min(la, len(order)))} if pool else {}

    def fetch(k):
        if pool is None:
            return None
        data = ahead.pop(k).result()
        if k + la < len(order):
            ahead[k + la] = pool.submit(prepare, order[k + la])
        return data

    def record(j, s):
        s.update(index=j.index, name=j.name, rank=rank)
        out.append(s)

    for k, j in enumerate(solo):
        data = fetch(k)
        s = dict(execute(j, data) if pool is not None else execute(j))
        dev += float(s["device_s"])
        record(j, s)
    k = len(solo)
    if duo:
        lanes = ThreadPoolExecutor(max_workers=2)
        while k < len(order):
            group = order[k:k + 2]
            args = [(j, fetch(k + i)) for i, j in enumerate(group)]
            t0 = time.perf_counter()
            futs = [lanes.submit(execute, j, d, i) for i, (j, d) in enumerate(args)]
            res = [dict(f.result()) for f in futs]
            wall = time.perf_counter() - t0
            dev += max([wall] + [float(s["device_s"]) for s in res])
            for j, s in zip(group, res):
                s["paired"] = len(group) == 2
                record(j, s)
            k += len(group)
        lanes.shutdown()
    if pool is not None:
        pool.shutdown()
    per_rank = gather([dev, out]) if gather is not None else [[dev, out]]
    allj = sorted((s for _, lst in per_rank for s in lst), key=lambda s: s["index"])
    return {"jobs": allj, "device_s": max(d for d, _ in per_rank), "cuts": sum(s["cuts"] for s in allj),
            "bins": [int(b) for b in bins]}


def _main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=226, help="first J jobs of the 226 (layer order)")
    ap.add_argument("--prefix-cuts", type=int, default=512, help="cuts per job (prefix of its Table-2 width)")
    ap.add_argument("--lookahead", type=int, default=8, help="jobs synthesised concurrently on the host")
    ap.add_argument("--out", default="", help="also write the JSON summary here")
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--pair-rows", type=int, default=0,
                    help="jobs with at most this many rows run two at a time, half the grid each "
                         "(0: off; off by default, DESIGN §8: the two host calls serialise)")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    from .api import DecomposeConfig, Engine, SearchConfig

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    eng = Engine(local)
    half = torch.cuda.get_device_properties(local).multi_processor_count // 2
    # pair phase: one engine per lane, each grid capped at half the SMs (engine option)
    lanes = [Engine(local, ctas=half), Engine(local, ctas=half)] if args.pair_rows > 0 else []
    for e in lanes:  # first-use setup of the lanes' engines stays out of the batch
        e.run(np.ones((64, 64), np.float32), DecomposeConfig(width=1), dtype=args.dtype)
    jobs = [Job(j.index, j.name, j.shape, min(j.width, args.prefix_cuts), j.seed)
            for j in mistral_jobs()[: args.jobs]]

    def execute(job: Job, a, lane: Optional[int] = None) -> Dict:
        cfg = DecomposeConfig(width=job.width, search=SearchConfig(seed=job.seed))
        try:
            dec, rep, _ = (eng if lane is None else lanes[lane]).run(a, cfg, dtype=args.dtype)
        except Exception as e:  # reported per job; the batch goes on
            print(f"job {job.index} {job.name} {job.shape}: {e!r}", file=sys.stderr, flush=True)
            return {"shape": list(job.shape), "cuts": 0, "device_s": 0.0, "error": repr(e)}
        print(f"job {job.index} {job.name} {job.shape}: {dec.width()} cuts in {rep.kernel_ms:.1f} ms",
              file=sys.stderr, flush=True)
        return {"shape": list(job.shape), "cuts": dec.width(), "device_s": rep.kernel_ms / 1e3,
                "call_s": rep.total_ms / 1e3, "rel_residual": rep.final_residual_norm / rep.input_norm,
                "sweeps_mean": float(np.mean(rep.sweeps)) if len(rep.sweeps) else 0.0,
                "sweeps_max": int(np.max(rep.sweeps)) if len(rep.sweeps) else 0,
                "cap_hits": int(np.sum(rep.sweeps >= 100)), "passes": rep.passes,
                "device_bytes": rep.device_bytes}

    def gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    t0 = time.perf_counter()
    pair = (lambda j: j.shape[0] <= args.pair_rows) if args.pair_rows > 0 else None
    res = run_batch(jobs, rank, world, execute, gather if world > 1 else None, prepare=mistral_matrix,
                    pair=pair, lookahead=args.lookahead)
    wall = time.perf_counter() - t0
    if rank == 0:
        out = {"metric": "batch signed cuts/sec (Mistral-shaped prefix)", "n_gpus": world,
               "jobs": len(jobs), "cuts_per_job": args.prefix_cuts, "cuts": res["cuts"],
               "device_s_max_rank": res["device_s"], "value": res["cuts"] / res["device_s"], "unit": "cuts/s",
               "wall_s": wall, "schedule": "LPT over ranks (sc_lpt_schedule), cost w*m*n",
               "data": "synthetic Mistral-7B-shaped matrices (rank-64 + noise, bf16-rounded, f32)",
               "per_job": res["jobs"]}
        print(json.dumps(out))
        if args.out:
            with open(args.out, "w") as f:
                json.dump(out, f, indent=1)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(_main())
