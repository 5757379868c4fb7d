"""ctypes front-end of the CPU parity oracle -- TEST INFRASTRUCTURE ONLY.

Loads either the plain-C restatement (``oracle/liboracle.so``, prefix ``orc_``)
or the reference compiled unchanged (``oracle/_ref/libsigcut_ref.so``, prefix
``ref_``); both implement ``oracle/oracle.h``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg import this
module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "orc": os.path.join(HERE, "liboracle.so"),
    "ref": os.path.join(HERE, "_ref", "libsigcut_ref.so"),
}

u64 = C.c_uint64
P = C.POINTER


class OracleConfig(C.Structure):
    _fields_ = [
        ("width", u64),
        ("flush_width", u64),
        ("seed", u64),
        ("restarts", u64),
        ("max_sweeps", u64),
        ("min_value_fraction", C.c_double),
        ("max_factor_bytes", u64),
    ]


class OracleOutput(C.Structure):
    _fields_ = [
        ("signs", P(u64) * 8),
        ("alpha", P(C.c_double)),
        ("cut_value", P(C.c_double)),
        ("resid_norm", P(C.c_double)),
        ("iterations", P(u64)),
        ("remainder", P(C.c_double)),
        ("width_done", u64),
        ("input_norm", C.c_double),
        ("final_residual_norm", C.c_double),
    ]


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def words(n: int) -> int:
    return (n + 63) // 64


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(P(ctype))


@dataclass
class Decomposition:
    shape: tuple
    signs: list            # per axis: (width, words) uint64
    alpha: np.ndarray
    cut_value: np.ndarray
    resid_norm: np.ndarray  # CutStep::residual_norm curve
    iterations: np.ndarray | None
    remainder: np.ndarray | None
    input_norm: float
    final_residual_norm: float
    width: int = 0
    extra: dict = field(default_factory=dict)


class Oracle:
    def __init__(self, which: str = "orc"):
        path = LIBS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (make -C oracle)")
        self.which = which
        self.lib = C.CDLL(path)
        p = which + "_"
        L = self.lib
        self._f = {}
        sig = {
            "last_error": (C.c_char_p, []),
            "mix64": (u64, [u64]),
            "substream": (u64, [u64, u64]),
            "fill_u64": (None, [u64, u64, P(u64)]),
            "fill_normal": (None, [u64, u64, P(C.c_double)]),
            "fill_f64": (None, [u64, u64, P(C.c_double)]),
            "greedy_decompose": (C.c_int, [P(C.c_double), C.c_int, P(u64), P(OracleConfig), P(OracleOutput)]),
            "signed_cut": (C.c_int, [P(C.c_double), C.c_int, P(u64), u64, u64, u64, P(C.c_double),
                                     P(P(u64)), P(u64), P(C.c_double), P(u64)]),
            "width_for_compression": (u64, [C.c_int, C.c_int, C.c_int, P(u64), C.c_double]),
            "compression_rate": (C.c_double, [u64, C.c_int, C.c_int, C.c_int, P(u64)]),
            "quantize_bf16": (None, [u64, P(C.c_double), P(C.c_double)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, p + name)
            f.restype = res
            f.argtypes = args
            self._f[name] = f

    # -- rng / metrics --------------------------------------------------------
    def mix64(self, z: int) -> int:
        return self._f["mix64"](z)

    def substream(self, seed: int, index: int) -> int:
        return self._f["substream"](seed, index)

    def fill_u64(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        self._f["fill_u64"](seed, count, _ptr(out, u64))
        return out

    def fill_normal(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.float64)
        self._f["fill_normal"](seed, count, _ptr(out, C.c_double))
        return out

    def fill_f64(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.float64)
        self._f["fill_f64"](seed, count, _ptr(out, C.c_double))
        return out

    def width_for_compression(self, shape, rate, coeff_bits=64, source_bits=64) -> int:
        sh = np.asarray(shape, np.uint64)
        return self._f["width_for_compression"](coeff_bits, source_bits, len(sh), _ptr(sh, u64), rate)

    def compression_rate(self, k, shape, coeff_bits=64, source_bits=64) -> float:
        sh = np.asarray(shape, np.uint64)
        return self._f["compression_rate"](k, coeff_bits, source_bits, len(sh), _ptr(sh, u64))

    def quantize_bf16(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty_like(x)
        self._f["quantize_bf16"](x.size, _ptr(x, C.c_double), _ptr(out, C.c_double))
        return out

    def _err(self, rc):
        if rc != 0:
            raise OracleError(rc, self._f["last_error"]().decode())

    # -- the path ------------------------------------------------------------
    def greedy_decompose(self, a: np.ndarray, width: int, seed: int = 0, flush_width: int = 32,
                         restarts: int = 1, max_sweeps: int = 100, min_value_fraction: float = 0.0,
                         max_factor_bytes: int = 1 << 30, want_iterations: bool = True,
                         want_remainder: bool = False) -> Decomposition:
        a = np.ascontiguousarray(a, np.float64)
        shape = tuple(int(d) for d in a.shape)
        sh = np.asarray(shape, np.uint64)
        cfg = OracleConfig(width, flush_width, seed, restarts, max_sweeps, min_value_fraction,
                           max_factor_bytes)
        out = OracleOutput()
        alloc_w = max(width, 1)
        signs = [np.zeros((alloc_w, words(d)), np.uint64) for d in shape]
        for i, s in enumerate(signs):
            out.signs[i] = _ptr(s, u64)
        alpha = np.zeros(alloc_w)
        cut = np.zeros(alloc_w)
        rn = np.zeros(alloc_w)
        it = np.zeros(alloc_w, np.uint64) if want_iterations else None
        rem = np.zeros(a.size) if want_remainder else None
        out.alpha, out.cut_value, out.resid_norm = _ptr(alpha, C.c_double), _ptr(cut, C.c_double), _ptr(rn, C.c_double)
        out.iterations = _ptr(it, u64) if it is not None else None
        out.remainder = _ptr(rem, C.c_double) if rem is not None else None
        self._err(self._f["greedy_decompose"](_ptr(a, C.c_double), len(shape), _ptr(sh, u64),
                                              C.byref(cfg), C.byref(out)))
        w = int(out.width_done)
        return Decomposition(shape, [s[:w] for s in signs], alpha[:w], cut[:w], rn[:w],
                             it[:w] if it is not None else None,
                             rem.reshape(shape) if rem is not None else None,
                             out.input_norm, out.final_residual_norm, w)

    def signed_cut(self, a: np.ndarray, seed: int = 0, restarts: int = 1, max_sweeps: int = 100):
        a = np.ascontiguousarray(a, np.float64)
        shape = tuple(int(d) for d in a.shape)
        sh = np.asarray(shape, np.uint64)
        signs = [np.zeros(words(d), np.uint64) for d in shape]
        arr = (P(u64) * len(shape))(*[_ptr(s, u64) for s in signs])
        value = C.c_double()
        iters = u64()
        sv = np.zeros(max_sweeps)
        nsv = u64()
        self._err(self._f["signed_cut"](_ptr(a, C.c_double), len(shape), _ptr(sh, u64), seed, restarts,
                                        max_sweeps, C.byref(value), arr, C.byref(iters),
                                        _ptr(sv, C.c_double), C.byref(nsv)))
        return dict(value=value.value, signs=signs, iterations=int(iters.value),
                    sweep_values=sv[: nsv.value].copy())


def normal_matrix(seed: int, shape, oracle: Oracle | None = None) -> np.ndarray:
    """Row-major Xoshiro256pp(seed).next_normal() stream (inc/rng.hpp:58-71)."""
    o = oracle or Oracle("orc")
    n = int(np.prod(shape))
    return o.fill_normal(seed, n).reshape(shape)
