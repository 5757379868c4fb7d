"""Row-sharded multi-GPU path: host logic on CPU -- balanced
bands, the gather of each rank's row signs into the global SignVector words
(band edges not on 64-row boundaries), per-rank C5 input generation, and a
world_size-2 gloo run of the gather protocol the driver uses."""
import os
import socket
import tempfile

import numpy as np
import torch.multiprocessing as mp

from paper_2410_01799_b200 import sharded


def test_bands_are_balanced_and_contiguous():
    for m, w in [(65536, 8), (200, 3), (7, 7), (1000, 2)]:
        b = sharded.bands(m, w)
        assert b[0][0] == 0 and sum(r for _, r in b) == m
        assert all(b[i][0] + b[i][1] == b[i + 1][0] for i in range(w - 1))
        assert max(r for _, r in b) - min(r for _, r in b) <= 1


def test_assemble_signs_ragged_bands():
    rng = np.random.default_rng(1)
    m, width, w = 203, 4, 3
    bits = rng.integers(0, 2, (width, m)).astype(np.uint8)
    bl = sharded.bands(m, w)
    local = [np.stack([sharded.pack_rows(bits[k, r0:r0 + rows]) for k in range(width)]) for r0, rows in bl]
    glob = sharded.assemble_signs(local, bl)
    for k in range(width):
        assert np.array_equal(glob[k], sharded.pack_rows(bits[k]))
        assert int(glob[k][-1]) >> (m % 64) == 0  # pad bits zero


def test_c5_rows_are_the_block_seeded_stream(orc):
    """One C5 generator (workloads.c5_rows, 1024-row blocks), any row range."""
    from paper_2410_01799_b200 import workloads

    n, B = 40, workloads.C5_BLOCK
    full = np.concatenate([orc.fill_normal(orc.substream(4, b), B * n).astype(np.float32)
                           .reshape(B, n) for b in range(3)])
    for r0, rows in [(0, 10), (250, 20), (300, 1400), (1023, 1025), (2047, 1)]:
        assert np.array_equal(sharded.c5_rows(r0, rows, n), full[r0:r0 + rows])
        assert np.array_equal(workloads.c5_rows(r0, rows, n), full[r0:r0 + rows])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m, width, out):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

    def allgather(x):
        o = [None] * world
        dist.all_gather_object(o, x)
        return o

    r0, rows = sharded.bands(m, world)[rank]
    rng = np.random.default_rng(7)
    bits = rng.integers(0, 2, (width, m)).astype(np.uint8)  # same on every rank
    mine = np.stack([sharded.pack_rows(bits[k, r0:r0 + rows]) for k in range(width)])
    glob = sharded.assemble_signs(allgather(mine), sharded.bands(m, world))
    handles = allgather(bytes([rank]) * 64)  # the IPC-handle exchange: rank order
    ok = all(np.array_equal(glob[k], sharded.pack_rows(bits[k])) for k in range(width))
    ok = ok and [h[0] for h in handles] == list(range(world))
    if rank == 0:
        with open(out, "w") as f:
            f.write("ok" if ok else "bad")
    dist.barrier()
    dist.destroy_process_group()


def test_gather_protocol_world2_gloo():
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "r")
        mp.spawn(_worker, args=(2, _free_port(), 333, 5, out), nprocs=2, join=True)
        assert open(out).read() == "ok"
