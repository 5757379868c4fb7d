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
            "accumulate_expansion": (C.c_int, [C.c_int, P(u64), C.c_int, u64, P(P(u64)), P(C.c_double),
                                               C.c_double, u64, P(C.c_double)]),
            "build_gram": (C.c_int, [P(C.c_double), C.c_int, P(u64), C.c_int, u64, P(P(u64)), P(C.c_double),
                                     P(C.c_double)]),
            "solve_gram": (C.c_int, [u64, u64, P(C.c_double), P(C.c_double), P(C.c_double)]),
            "correct_coefficients": (C.c_int, [P(C.c_double), C.c_int, P(u64), C.c_int, u64, P(P(u64)),
                                               P(C.c_double), P(C.c_double)]),
            "lstsq_decompose": (C.c_int, [P(C.c_double), C.c_int, P(u64), C.c_int, P(OracleConfig),
                                          P(OracleOutput)]),
            "write_scd": (C.c_int, [C.c_int, P(u64), C.c_int, u64, P(P(u64)), P(C.c_double), C.c_int,
                                    P(C.c_uint8), u64, P(u64)]),
            "read_scd": (C.c_int, [P(C.c_uint8), u64, P(C.c_int), P(u64), P(C.c_int), P(u64), P(P(u64)),
                                   P(C.c_double)]),
            "write_raw": (C.c_int, [C.c_int, P(u64), P(C.c_double), C.c_int, P(C.c_uint8), u64, P(u64)]),
            "read_raw": (C.c_int, [P(C.c_uint8), u64, P(C.c_int), P(u64), P(C.c_double)]),
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


    # -- around the path -------------------------------------
    @staticmethod
    def _fac(factors):
        fs = [np.ascontiguousarray(f, np.uint64) for f in factors]
        arr = (P(u64) * max(1, len(fs)))(*[_ptr(f, u64) for f in fs])
        return fs, arr

    def accumulate_expansion(self, shape, factors, coeffs, data=None, scale=1.0, first_term=0,
                             channel_axis=-1) -> np.ndarray:
        """data (f64, shape) += sum_{j >= first_term} flip(scale coef_j, parity); zeros if None."""
        shape = tuple(int(d) for d in shape)
        sh = np.asarray(shape, np.uint64)
        out = np.zeros(shape) if data is None else np.array(data, np.float64, copy=True)
        co = np.ascontiguousarray(coeffs, np.float64)
        width = co.shape[0] if co.ndim else 0
        fs, arr = self._fac(factors)
        self._err(self._f["accumulate_expansion"](len(shape), _ptr(sh, u64), channel_axis, width, arr,
                                                  _ptr(co, C.c_double), scale, first_term, _ptr(out, C.c_double)))
        return out

    def build_gram(self, a, factors, width, channel_axis=-1):
        a = np.ascontiguousarray(a, np.float64)
        sh = np.asarray(a.shape, np.uint64)
        q = a.shape[channel_axis] if channel_axis >= 0 else 1
        gram = np.zeros((width, width))
        rhs = np.zeros((width, q))
        fs, arr = self._fac(factors)
        self._err(self._f["build_gram"](_ptr(a, C.c_double), a.ndim, _ptr(sh, u64), channel_axis, width, arr,
                                        _ptr(gram, C.c_double), _ptr(rhs, C.c_double)))
        return gram, rhs

    def solve_gram(self, gram, rhs):
        gram = np.ascontiguousarray(gram, np.float64)
        rhs = np.ascontiguousarray(rhs, np.float64)
        w = gram.shape[0]
        ch = rhs.size // max(w, 1)
        out = np.zeros_like(rhs)
        self._err(self._f["solve_gram"](w, ch, _ptr(gram, C.c_double), _ptr(rhs, C.c_double), _ptr(out, C.c_double)))
        return out

    def correct_coefficients(self, a, factors, coeffs, channel_axis=-1):
        a = np.ascontiguousarray(a, np.float64)
        sh = np.asarray(a.shape, np.uint64)
        co = np.ascontiguousarray(coeffs, np.float64)
        out = np.zeros_like(co)
        fs, arr = self._fac(factors)
        self._err(self._f["correct_coefficients"](_ptr(a, C.c_double), a.ndim, _ptr(sh, u64), channel_axis,
                                                  co.shape[0], arr, _ptr(co, C.c_double), _ptr(out, C.c_double)))
        return out

    def lstsq_decompose(self, a, width, seed=0, channel_axis=-1, restarts=1, max_sweeps=100,
                        min_value_fraction=0.0, max_factor_bytes=1 << 30) -> Decomposition:
        a = np.ascontiguousarray(a, np.float64)
        shape = tuple(int(d) for d in a.shape)
        sh = np.asarray(shape, np.uint64)
        cfg = OracleConfig(width, 32, seed, restarts, max_sweeps, min_value_fraction, max_factor_bytes)
        q = shape[channel_axis] if channel_axis >= 0 else 1
        axes = [i for i in range(len(shape)) if i != channel_axis]
        alloc_w = max(width, 1)
        signs = [np.zeros((alloc_w, words(shape[i])), np.uint64) for i in axes]
        out = OracleOutput()
        for i, s in enumerate(signs):
            out.signs[i] = _ptr(s, u64)
        alpha = np.zeros((alloc_w, q))
        cut, rn = np.zeros(alloc_w), np.zeros(alloc_w)
        it = np.zeros(alloc_w, np.uint64)
        out.alpha, out.cut_value, out.resid_norm = _ptr(alpha, C.c_double), _ptr(cut, C.c_double), _ptr(rn, C.c_double)
        out.iterations = _ptr(it, u64) if self.which == "orc" else None
        out.remainder = None
        self._err(self._f["lstsq_decompose"](_ptr(a, C.c_double), len(shape), _ptr(sh, u64), channel_axis,
                                             C.byref(cfg), C.byref(out)))
        w = int(out.width_done)
        return Decomposition(shape, [s[:w] for s in signs], alpha[:w] if channel_axis >= 0 else alpha[:w, 0],
                             cut[:w], rn[:w], it[:w] if self.which == "orc" else None, None,
                             out.input_norm, out.final_residual_norm, w)

    def write_scd(self, shape, factors, coeffs, channel_axis=-1, coeff_bits=64) -> bytes:
        sh = np.asarray(shape, np.uint64)
        co = np.ascontiguousarray(coeffs, np.float64)
        fs, arr = self._fac(factors)
        size = u64()
        cap = 64 + 8 * len(shape) + co.size * 8 + sum(f.size * 8 for f in fs) + 1024
        buf = np.zeros(cap, np.uint8)
        self._err(self._f["write_scd"](len(shape), _ptr(sh, u64), channel_axis, co.shape[0] if co.ndim else 0, arr,
                                       _ptr(co, C.c_double), coeff_bits, _ptr(buf, C.c_uint8), cap, C.byref(size)))
        return bytes(buf[: size.value])

    def read_scd(self, data: bytes):
        buf = np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
        order, chax, width = C.c_int(), C.c_int(), u64()
        shape = np.zeros(8, np.uint64)
        self._err(self._f["read_scd"](_ptr(buf, C.c_uint8), len(data), C.byref(order), _ptr(shape, u64),
                                      C.byref(chax), C.byref(width), None, None))
        k, ca, w = order.value, chax.value, int(width.value)
        shp = tuple(int(x) for x in shape[:k])
        q = shp[ca] if ca >= 0 else 1
        axes = [i for i in range(k) if i != ca]
        fs = [np.zeros((max(w, 1), words(shp[i])), np.uint64) for i in axes]
        co = np.zeros((max(w, 1), q))
        _, arr = self._fac(fs)
        self._err(self._f["read_scd"](_ptr(buf, C.c_uint8), len(data), C.byref(order), _ptr(shape, u64),
                                      C.byref(chax), C.byref(width), arr, _ptr(co, C.c_double)))
        return shp, ca, [f[:w] for f in fs], (co[:w] if ca >= 0 else co[:w, 0])

    def write_raw(self, a, dtype=0) -> bytes:
        a = np.ascontiguousarray(a, np.float64)
        sh = np.asarray(a.shape, np.uint64)
        cap = 16 + 8 * a.ndim + a.size * 8
        buf = np.zeros(cap, np.uint8)
        size = u64()
        self._err(self._f["write_raw"](a.ndim, _ptr(sh, u64), _ptr(a, C.c_double), dtype, _ptr(buf, C.c_uint8), cap,
                                       C.byref(size)))
        return bytes(buf[: size.value])

    def read_raw(self, data: bytes) -> np.ndarray:
        buf = np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
        order = C.c_int()
        shape = np.zeros(8, np.uint64)
        self._err(self._f["read_raw"](_ptr(buf, C.c_uint8), len(data), C.byref(order), _ptr(shape, u64), None))
        shp = tuple(int(x) for x in shape[: order.value])
        out = np.zeros(shp)
        self._err(self._f["read_raw"](_ptr(buf, C.c_uint8), len(data), C.byref(order), _ptr(shape, u64),
                                      _ptr(out, C.c_double)))
        return out


# -- reference-only PPM / CSV helpers (io.hpp:294-396) --------------------------
def _ref_extra(oracle):
    L = oracle.lib
    sig = {
        "ref_write_ppm": (C.c_int, [u64, u64, P(C.c_double), P(C.c_uint8), u64, P(u64)]),
        "ref_read_ppm": (C.c_int, [P(C.c_uint8), u64, P(u64), P(u64), P(C.c_double)]),
        "ref_write_curve_csv": (C.c_int, [u64, P(u64), P(C.c_double), P(C.c_double), C.c_char_p, u64, P(u64)]),
        "ref_read_curve_csv": (C.c_int, [C.c_char_p, u64, P(u64), P(u64), P(C.c_double), P(C.c_double)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    return L


def ref_write_ppm(oracle, a) -> bytes:
    L = _ref_extra(oracle)
    a = np.ascontiguousarray(a, np.float64)
    cap = 64 + a.size
    buf = np.zeros(cap, np.uint8)
    size = u64()
    oracle._err(L.ref_write_ppm(a.shape[0], a.shape[1], _ptr(a, C.c_double), _ptr(buf, C.c_uint8), cap, C.byref(size)))
    return bytes(buf[: size.value])


def ref_read_ppm(oracle, data: bytes) -> np.ndarray:
    L = _ref_extra(oracle)
    buf = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
    h, w = u64(), u64()
    oracle._err(L.ref_read_ppm(_ptr(buf, C.c_uint8), len(data), C.byref(h), C.byref(w), None))
    out = np.zeros((h.value, w.value, 3))
    oracle._err(L.ref_read_ppm(_ptr(buf, C.c_uint8), len(data), C.byref(h), C.byref(w), _ptr(out, C.c_double)))
    return out


def ref_write_curve_csv(oracle, points) -> str:
    L = _ref_extra(oracle)
    w = np.array([p[0] for p in points], np.uint64)
    r = np.array([p[1] for p in points], np.float64)
    e = np.array([p[2] for p in points], np.float64)
    cap = 64 + 80 * len(points)
    buf = C.create_string_buffer(cap)
    size = u64()
    oracle._err(L.ref_write_curve_csv(len(points), _ptr(w, u64), _ptr(r, C.c_double), _ptr(e, C.c_double), buf, cap,
                                      C.byref(size)))
    return buf.raw[: size.value].decode()


def ref_read_curve_csv(oracle, text: str):
    L = _ref_extra(oracle)
    b = text.encode()
    n = u64()
    oracle._err(L.ref_read_curve_csv(b, len(b), C.byref(n), None, None, None))
    w, r, e = np.zeros(n.value, np.uint64), np.zeros(n.value), np.zeros(n.value)
    oracle._err(L.ref_read_curve_csv(b, len(b), C.byref(n), _ptr(w, u64), _ptr(r, C.c_double), _ptr(e, C.c_double)))
    return [(int(a), float(x), float(y)) for a, x, y in zip(w, r, e)]


def normal_matrix(seed: int, shape, oracle: Oracle | None = None) -> np.ndarray:
    """Row-major Xoshiro256pp(seed).next_normal() stream (inc/rng.hpp:58-71)."""
    o = oracle or Oracle("orc")
    n = int(np.prod(shape))
    return o.fill_normal(seed, n).reshape(shape)
