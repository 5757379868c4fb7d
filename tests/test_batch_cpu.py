"""Multi-GPU batch path host logic on CPU: the Mistral-shaped
job set, its seeded inputs, LPT assignment, and a world_size-2 gloo run of the
batch driver (stub executor: no GPU work, the scheduling/gather logic is real)."""
import json
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2410_01799_b200 import batch


def test_mistral_job_set_and_table2_widths(orc):
    jobs = batch.mistral_jobs()
    assert len(jobs) == 226
    widths = {j.shape: j.width for j in jobs}
    # paper Table 2 at 50% of the bf16 footprint (metrics.hpp:55-63)
    assert widths[(4096, 4096)] == 16320 and widths[(1024, 4096)] == 6512
    assert widths[(14336, 4096)] == 25442 and widths[(4096, 14336)] == 25442
    assert widths[(32000, 4096)] == 29023
    assert [j.name for j in jobs[:7]] == [f"layers.0.{n}" for n in ("q", "k", "v", "o", "gate", "up", "down")]
    assert jobs[-2].name == "embed" and jobs[-1].name == "lm_head"
    for j in jobs[:5] + jobs[-2:]:
        assert j.seed == orc.substream(3, j.index)


def test_round_bf16_is_reference_quantize_half(orc):
    x = orc.fill_normal(9, 20000) * 0.02
    x[:4] = [1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -1.0 - 2 ** -9, 0.0]  # ties to even
    assert np.array_equal(batch.round_bf16(x), orc.quantize_bf16(x))


def test_mistral_matrix_is_seeded_stream(orc):
    job = batch.Job(7, "t", (24, 40), 3, orc.substream(3, 7))
    a = batch.mistral_matrix(job, rank_k=5)
    z = orc.fill_normal(job.seed, 24 * 5 + 40 * 5 + 24 * 40)
    u, v, nz = z[:120].reshape(24, 5), z[120:320].reshape(40, 5), z[320:].reshape(24, 40)
    want = orc.quantize_bf16(0.015 / 8.0 * (u @ v.T) + 0.02 * nz).astype(np.float32)
    assert a.dtype == np.float32 and np.array_equal(a, want)
    assert not np.any(a.view(np.uint32) & 0xFFFF)  # bf16-representable


def test_lpt_plan_of_the_full_batch_is_balanced():
    jobs = batch.mistral_jobs()
    for world in (2, 4, 8):
        bins = batch.plan(jobs, world)
        loads = np.bincount(bins, weights=[j.cost for j in jobs], minlength=world)
        assert loads.max() <= loads.mean() + max(j.cost for j in jobs)  # LPT makespan bound
        assert loads.max() / loads.mean() < 1.05


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, jobs, out_path):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

    def execute(job):
        return {"cuts": job.width, "device_s": job.cost * 1e-12, "ran_on": rank}

    def gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    res = batch.run_batch(jobs, rank, world, execute, gather)
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


def test_batch_driver_world2_gloo():
    jobs = [batch.Job(j.index, j.name, j.shape, min(j.width, 50), j.seed) for j in batch.mistral_jobs()[:23]]
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "res.json")
        mp.spawn(_worker, args=(2, _free_port(), jobs, out), nprocs=2, join=True)
        res = json.load(open(out))
    idx = [s["index"] for s in res["jobs"]]
    assert idx == list(range(23))  # every job exactly once, gathered in job order
    bins = batch.plan(jobs, 2)
    assert all(s["ran_on"] == s["rank"] == int(bins[s["index"]]) for s in res["jobs"])
    per_rank = [sum(j.cost for j in jobs if bins[j.index] == r) * 1e-12 for r in range(2)]
    assert abs(res["device_s"] - max(per_rank)) <= 1e-9 * max(per_rank)
    assert res["cuts"] == sum(j.width for j in jobs)


def test_run_batch_prefetches_inputs_in_order():
    """prepare(job) runs one job ahead on a helper thread; execute(job, data) sees
    exactly that job's data, in the rank's longest-first order."""
    from paper_2410_01799_b200.batch import Job, run_batch

    jobs = [Job(i, f"j{i}", (4 + i, 8), 3 + (i % 4), 100 + i) for i in range(9)]
    seen = []

    def prepare(job):
        return ("data", job.index)

    def execute(job, data):
        assert data == ("data", job.index)
        seen.append(job.index)
        return {"cuts": job.width, "device_s": 0.001}

    res = run_batch(jobs, 0, 1, execute, prepare=prepare)
    assert sorted(seen) == list(range(9))
    assert seen == [j.index for j in sorted(jobs, key=lambda j: (-j.cost, j.index))]
    assert res["cuts"] == sum(j.width for j in jobs)


def test_run_batch_pairs_small_jobs_two_lanes():
    """pair(job) jobs run after every solo job, two at a time on lanes 0 and 1, each
    with its own prefetched data; the pair's device time is counted once."""
    import threading
    import time as _time

    from paper_2410_01799_b200.batch import Job, run_batch

    jobs = [Job(i, f"j{i}", (64 if i < 3 else 8, 8), 4, 100 + i) for i in range(8)]
    lock = threading.Lock()
    calls = []

    def prepare(job):
        return ("data", job.index)

    def execute(job, data, lane=None):
        assert data == ("data", job.index)
        with lock:
            calls.append((job.index, lane))
        if lane is not None:
            _time.sleep(0.1)
        return {"cuts": job.width, "device_s": 0.1 if lane is not None else 0.001}

    small = lambda j: j.shape[0] <= 8
    res = run_batch(jobs, 0, 1, execute, prepare=prepare, pair=small)
    solo = [c for c in calls if c[1] is None]
    duo = [c for c in calls if c[1] is not None]
    assert sorted(c[0] for c in solo) == [0, 1, 2]
    assert calls[:3] == solo  # every solo job runs before the pair phase
    assert sorted(c[0] for c in duo) == [3, 4, 5, 6, 7]
    assert sorted(c[1] for c in duo) == [0, 0, 0, 1, 1]
    assert res["cuts"] == sum(j.width for j in jobs)
    assert [s["index"] for s in res["jobs"]] == list(range(8))
    assert sum(1 for s in res["jobs"] if s.get("paired")) == 4
    # two pairs and a single of ~100 ms each: concurrent lanes, not 5 x 100 ms
    assert 0.3 <= res["device_s"] < 0.45
