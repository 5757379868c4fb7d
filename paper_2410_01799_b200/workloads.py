"""Synthetic inputs of the BASELINE.json configurations (host-side input
synthesis; not on the device path).

No public dataset is involved: the paper's Mistral weights and photograph are
not in the container, so seeded streams of the reference's generator
(Xoshiro256pp, rng.hpp) stand in with the configs' shapes and distributions.

  C1  1024 x 1024, N(0,1) from Xoshiro256pp(0), row-major, stored f32; w = 256.
  C2  4096 x 4096, N(0,1) from Xoshiro256pp(1) (f32, and the same values in f64).
  C3  4000 x 3000 x 3 "RGB image": per channel c, 8 Gaussian blobs with
      cx = 3000 u, cy = 4000 u, amp = u, sigma = 100 + 700 u (u = next_f64 of
      Xoshiro256pp(2), drawn in that order, channel-major), value
      sum amp exp(-((x - cx)^2 + (y - cy)^2) / (2 sigma^2)), plus 0.02 N(0,1)
      noise drawn from Xoshiro256pp(substream(2, 1)) in row-major order, clipped
      to [0, 1], stored f32.  (Recipe of SURVEY §8d with the noise on its own
      substream so the uniforms and the noise can be drawn independently.)
  C4  Mistral-7B-shaped batch (batch.mistral_jobs / batch.mistral_matrix).
  C5  65536 x 65536 N(0,1): row block b of 1024 rows from
      Xoshiro256pp(substream(4, b)) (parallel generation rule).
"""
from __future__ import annotations

import numpy as np

from .api import fill_normal
from .batch import MASK64, mix64, substream


class Xoshiro256pp:
    """rng.hpp:26-56 (seeding by four SplitMix64 steps, xoshiro256++, 53-bit f64)."""

    def __init__(self, seed: int):
        s = []
        z = seed & MASK64
        for _ in range(4):
            z = (z + 0x9E3779B97F4A7C15) & MASK64
            x = z
            x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
            x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
            s.append(x ^ (x >> 31))
        self.s = s

    @staticmethod
    def _rotl(v, k):
        return ((v << k) | (v >> (64 - k))) & MASK64

    def next_u64(self) -> int:
        s = self.s
        result = (self._rotl((s[0] + s[3]) & MASK64, 23) + s[0]) & MASK64
        t = (s[1] << 17) & MASK64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = self._rotl(s[3], 45)
        return result

    def next_f64(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)


def c1(dtype=np.float32) -> np.ndarray:
    return fill_normal(0, 1024 * 1024, np.float32 if dtype == np.float32 else np.float64).reshape(1024, 1024)


def c2(dtype=np.float32) -> np.ndarray:
    """C2; the f64 variant holds the same (f32-rounded) values as the f32 one."""
    a = fill_normal(1, 4096 * 4096, np.float32).reshape(4096, 4096)
    return a if dtype == np.float32 else a.astype(np.float64)


def c3_blob_image(height: int = 4000, width: int = 3000, blobs: int = 8, seed: int = 2) -> np.ndarray:
    rng = Xoshiro256pp(seed)
    params = [[(width * rng.next_f64(), height * rng.next_f64(), rng.next_f64(), 100.0 + 700.0 * rng.next_f64())
               for _ in range(blobs)] for _ in range(3)]
    y = np.arange(height, dtype=np.float64)[:, None]
    x = np.arange(width, dtype=np.float64)[None, :]
    img = np.zeros((height, width, 3))
    for c in range(3):
        acc = np.zeros((height, width))
        for cx, cy, amp, sig in params[c]:
            acc += amp * np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2.0 * sig * sig))
        img[:, :, c] = acc
    img += 0.02 * fill_normal(substream(seed, 1), height * width * 3).reshape(height, width, 3)
    return np.clip(img, 0.0, 1.0).astype(np.float32)


C5_BLOCK = 1024


def c5_rows(row0: int, rows: int, n: int = 65536, block: int = C5_BLOCK, seed: int = 4) -> np.ndarray:
    """Rows [row0, row0 + rows) of C5 (any range): row block b of ``block`` rows is
    fill_normal(substream(seed, b)), so ranks generate only their own bands."""
    out = np.empty((rows, n), np.float32)
    if rows <= 0:
        return out
    b0, b1 = row0 // block, (row0 + rows - 1) // block
    for b in range(b0, b1 + 1):
        lo, hi = max(row0, b * block), min(row0 + rows, (b + 1) * block)
        blk = fill_normal(substream(seed, b), (hi - b * block) * n, np.float32).reshape(-1, n)
        out[lo - row0: hi - row0] = blk[lo - b * block:]
    return out


__all__ = ["C5_BLOCK", "Xoshiro256pp", "c1", "c2", "c3_blob_image", "c5_rows", "mix64", "substream"]
