"""C2 f64 whole-trajectory golden (BASELINE config 2 repeated with f64 storage):
the 4096x4096 matrix of N(0,1) values from Xoshiro256pp(1), rounded to f32 and
stored as f64, decomposed by the REFERENCE compiled unchanged (oracle/_ref,
greedy_decompose, decompose.hpp:314-361) to width 512, search seed 1,
flush_width 32.  Stored per term: an 8-byte digest (blake2b) of the packed row
and column sign words (S_k || T_k, SignVector layout), c_k, the sweep count, the
reference curve residual_norm and alpha -- the full words would be 512 KiB of
incompressible bits; the digest pins them exactly.

    python tests/golden/make_c2_f64.py   # ~10 min on one core (0.4-1.2 s per cut)
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import LIBS, Oracle  # noqa: E402

WIDTH = 512


def term_digest(s_words: np.ndarray, t_words: np.ndarray) -> np.uint64:
    h = hashlib.blake2b(np.ascontiguousarray(s_words, np.uint64).tobytes() +
                        np.ascontiguousarray(t_words, np.uint64).tobytes(), digest_size=8).digest()
    return np.frombuffer(h, np.uint64)[0]


def main():
    assert os.path.exists(LIBS["ref"]), "build oracle/_ref first (make -C oracle)"
    o = Oracle("ref")
    a = o.fill_normal(1, 4096 * 4096).astype(np.float32).astype(np.float64).reshape(4096, 4096)
    t0 = time.time()
    d = o.greedy_decompose(a, WIDTH, seed=1, flush_width=32)
    dig = np.array([term_digest(d.signs[0][k], d.signs[1][k]) for k in range(WIDTH)], np.uint64)
    np.savez_compressed(os.path.join(HERE, "c2_f64_w512.npz"), digest=dig, cut_value=d.cut_value,
                        alpha=d.alpha, iterations=np.asarray(d.iterations, np.uint32),
                        resid_norm=d.resid_norm, input_norm=d.input_norm,
                        final_residual_norm=d.final_residual_norm, width=WIDTH, seed=1, flush=32,
                        generator="oracle/_ref (reference headers compiled unchanged)",
                        seconds=time.time() - t0)
    print(f"wrote c2_f64_w512.npz in {time.time() - t0:.0f} s; rel_err {d.final_residual_norm / d.input_norm:.9f}")


if __name__ == "__main__":
    main()
