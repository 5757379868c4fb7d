"""Loader for tests/golden/*.npz (fixtures generated from the compiled reference
by tests/golden/make_golden.py).  Inputs that are not stored verbatim are
regenerated from the same Xoshiro256pp normal streams (pinned by rng.npz)."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# name -> (seed, dtype roundtrip) for decompositions stored without the input
_RECIPES = {
    "rect_200x150": (8, None),
    "tall_300x7": (21, None),
    "f32in_256_w64": (0, np.float32),
}


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def normal_stream(seed, count):
    """Xoshiro256pp(seed).next_normal() -- restated here in numpy-free C via the oracle."""
    from oracle.pyoracle import Oracle

    return Oracle("orc").fill_normal(seed, count)


def dec_input(name, d):
    if "a" in d:
        return d["a"]
    seed, rt = _RECIPES[name]
    shape = tuple(int(x) for x in d["shape"])
    a = normal_stream(seed, int(np.prod(shape))).reshape(shape)
    if rt is not None:
        a = a.astype(rt).astype(np.float64)
    return a


def dec_names():
    return sorted(os.path.basename(p)[4:-4] for p in glob.glob(os.path.join(GOLDEN, "dec_*.npz")))


def cut_names():
    return sorted(os.path.basename(p)[4:-4] for p in glob.glob(os.path.join(GOLDEN, "cut_*.npz")))


def names(prefix):
    return sorted(os.path.basename(p)[len(prefix) + 1:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "_*.npz")))


def factors_of(d):
    """(shape, channel_axis, factors, coeffs) of a fixture written by fac_dict()."""
    shape = tuple(int(x) for x in d["shape"])
    ch = int(d["channel_axis"])
    k = len(shape) - (1 if ch >= 0 else 0)
    return shape, ch, [d[f"fac{i}"] for i in range(k)], d["coeffs"]
