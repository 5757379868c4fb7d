"""Row-sharded decomposition of ONE matrix over several GPUs.

Rank r (one process per GPU) owns the contiguous row band ``bands(m, world)[r]``
of the m×n matrix and runs the persistent kernel on it.  The kernels of all
ranks form one grid: their z partials and c / ||R||² partials are reduced in
the same fixed order through peer-mapped exchange buffers (CUDA IPC over
NVLink), owner CTAs publish the next t to every rank, and one system-scope
barrier separates the passes -- the per-half-iteration allreduce of Rᵀs and of
the objective happens inside the kernel, over peer memory, instead of as NCCL
calls between kernel launches.  Every rank therefore holds the same t, α and
curve; the row signs s are distributed like the rows and gathered at the end.

C5 input (65536² f32): row block b of ``workloads.C5_BLOCK`` (1024) rows is drawn
from ``Xoshiro256pp(substream(4, b))`` so every rank generates only its own rows
(workloads.c5_rows, the single C5 generator).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        -m paper_2410_01799_b200.sharded --m 65536 --n 65536 --cuts 4
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import time
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N

def bands(m: int, world: int) -> List[Tuple[int, int]]:
    """(row0, rows) of every rank: balanced contiguous bands (floor / ceil of m / world)."""
    return [(r * m // world, (r + 1) * m // world - r * m // world) for r in range(world)]


def pack_rows(bits: np.ndarray) -> np.ndarray:
    """Sign bits (1 = negative) of consecutive rows -> SignVector words (LSB first, pad 0)."""
    bits = np.asarray(bits, np.uint8)
    pad = (-len(bits)) % 64
    b = np.concatenate([bits, np.zeros(pad, np.uint8)])
    return np.packbits(b, bitorder="little").view(np.uint64)


def unpack_rows(words: np.ndarray, rows: int) -> np.ndarray:
    return np.unpackbits(np.asarray(words, np.uint64).view(np.uint8), bitorder="little")[:rows]


def assemble_signs(local_words: Sequence[np.ndarray], band_list: Sequence[Tuple[int, int]]) -> np.ndarray:
    """Global term-major row-sign words from every rank's local words (rank order)."""
    width = local_words[0].shape[0]
    m = sum(r for _, r in band_list)
    out = np.zeros((width, (m + 63) // 64), np.uint64)
    for k in range(width):
        bits = np.concatenate([unpack_rows(w[k], rows) for w, (_, rows) in zip(local_words, band_list)])
        out[k] = pack_rows(bits)
    return out


def c5_rows(row0: int, rows: int, n: int = 65536, base_seed: int = 4) -> np.ndarray:
    """Rows [row0, row0+rows) of the C5 matrix (f32): the one generator, workloads.c5_rows."""
    from .workloads import c5_rows as _c5

    return _c5(row0, rows, n, seed=base_seed)


def emulated(a, cfg, world: int, dtype: Optional[str] = None, ctas: int = 0, timeout_ms: int = 0,
             dead_rank: int = -1, engine=None, want_remainder: bool = False):
    """The row-sharded protocol with ``world`` virtual ranks on ONE GPU (one
    cooperative launch over all ranks' bands; sc_greedy_decompose_sharded_emulated).
    ``a`` is the whole matrix; returns the gathered (CutDecomposition, CutReport,
    remainder) like Engine.run.  For testing the multi-rank exchange where fewer
    GPUs than ranks are available."""
    from .api import Engine

    eng = engine or Engine(0)
    opt = N.ScShardEmulation(world, ctas, timeout_ms, dead_rank)
    return eng.run(a, cfg, dtype=dtype, emulate=opt, want_remainder=want_remainder)


class ShardedEngine:
    """One rank of a row-sharded decomposition.  ``allgather(obj) -> list`` and
    ``barrier()`` are the host collectives (torch.distributed when world > 1)."""

    def __init__(self, m_global: int, n: int, dtype: str = "f32", rank: int = 0, world: int = 1,
                 device: Optional[int] = None, allgather: Optional[Callable] = None,
                 barrier: Optional[Callable] = None, ctas: int = 0, timeout_ms: int = 0):
        from .api import Engine

        self.m_global, self.n, self.dtype, self.rank, self.world = m_global, n, dtype, rank, world
        self.band = bands(m_global, world)[rank]
        self.eng = Engine(rank if device is None else device)
        self._allgather = allgather or (lambda x: [x])
        self._barrier = barrier or (lambda: None)
        self.cfg = N.ScShardConfig(rank, world, m_global, self.band[0], n,
                                   N.SC_F32 if dtype == "f32" else N.SC_F64, ctas, timeout_ms)
        h = C.create_string_buffer(N.SC_IPC_HANDLE_BYTES)
        self.eng._check(self.eng.lib.sc_shard_open(self.eng.handle, C.byref(self.cfg), h))
        handles = self._allgather(h.raw)  # rank order
        if world > 1:
            buf = C.create_string_buffer(b"".join(handles), N.SC_IPC_HANDLE_BYTES * world)
            self.eng._check(self.eng.lib.sc_shard_connect(self.eng.handle, buf))
        else:
            self.eng._check(self.eng.lib.sc_shard_connect(self.eng.handle, h))

    def decompose(self, a_local, cfg, want_remainder: bool = False):
        """This rank's rows -> (local CutDecomposition, CutReport, remainder rows)."""
        self.eng._check(self.eng.lib.sc_shard_reset(self.eng.handle))
        self._barrier()  # every rank's exchange region is reset before any kernel starts
        out = self.eng.run(a_local, cfg, dtype=self.dtype, want_remainder=want_remainder, shard=self.cfg)
        self._barrier()
        return out

    def gather_signs(self, dec) -> Optional[np.ndarray]:
        """Global row-sign words (term-major) on every rank."""
        return assemble_signs(self._allgather(dec.factors[0]), bands(self.m_global, self.world))

    def close(self):
        self.eng.lib.sc_shard_close(self.eng.handle)


def _main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=65536)
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--cuts", type=int, default=4)
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    from .api import DecomposeConfig, SearchConfig

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")  # host collectives only; the data path is peer memory

    def allgather(x):
        out = [None] * world
        dist.all_gather_object(out, x)
        return out

    se = ShardedEngine(args.m, args.n, args.dtype, rank, world, device=local,
                       allgather=allgather if world > 1 else None, barrier=dist.barrier if world > 1 else None)
    row0, rows = se.band
    a = c5_rows(row0, rows, args.n)
    if args.dtype == "f64":
        a = a.astype(np.float64)
    cfg = DecomposeConfig(width=args.cuts, search=SearchConfig(seed=4))
    t0 = time.perf_counter()
    dec, rep, _ = se.decompose(a, cfg)
    wall = time.perf_counter() - t0
    dev = rep.kernel_ms / 1e3
    devs = allgather(dev) if world > 1 else [dev]
    S = se.gather_signs(dec)
    if rank == 0:
        print(json.dumps({"metric": "row-sharded signed cuts/sec", "shape": [args.m, args.n], "n_gpus": world,
                          "cuts": dec.width(), "device_s_max_rank": max(devs), "value": dec.width() / max(devs),
                          "unit": "cuts/s", "wall_s": wall, "sweeps": rep.sweeps.tolist(),
                          "rel_residual": rep.final_residual_norm / rep.input_norm,
                          "row_sign_words": int(S.size)}))
    se.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(_main())
