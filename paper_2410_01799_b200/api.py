"""Host-side mirror of the reference's public decomposition API.

Same names, argument meaning and error behaviour as the reference's C++ API
(``/root/reference/proj/include/sigcut``):

=============================  ==========================================
this module                    reference
=============================  ==========================================
``SearchConfig``               ``sigcut::SearchConfig``     search.hpp:20-24
``DecomposeConfig``            ``sigcut::DecomposeConfig``  decompose.hpp:273-286
``CutResult``                  ``sigcut::CutResult``        search.hpp:28-32
``CutStep`` / ``CutReport``    metrics.hpp:85-97
``CutDecomposition``           decompose.hpp:30-100
``greedy_decompose``           decompose.hpp:314-361
``decompose`` (greedy)         decompose.hpp:472-476
``greedy_signed_cut``          search.hpp:259-263
``axial_greedy_cut`` (order 2) search.hpp:269-272
``width_for_compression``      metrics.hpp:55-63
``InvalidArgument``            ``std::invalid_argument``
=============================  ==========================================

Every call goes through the C ABI into the sm_100a kernels; nothing here
computes the decomposition on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N


class InvalidArgument(ValueError):
    """std::invalid_argument analogue (bad shape / config / non-finite data)."""


class SigcutRuntimeError(RuntimeError):
    """std::runtime_error analogue."""


class DeviceError(RuntimeError):
    """CUDA failure or no usable sm_100 device (there is no CPU fallback)."""


class NotSupported(RuntimeError):
    """Shape outside the kernels' envelope."""


_ERRORS = {
    N.SC_INVALID_ARGUMENT: InvalidArgument,
    N.SC_RUNTIME_ERROR: SigcutRuntimeError,
    N.SC_CUDA_ERROR: DeviceError,
    N.SC_NOT_SUPPORTED: NotSupported,
}


@dataclass
class SearchConfig:
    seed: int = 0
    restarts: int = 1
    max_sweeps: int = 100


@dataclass
class DecomposeConfig:
    width: int = 0
    flush_width: int = 32
    method: str = "greedy"
    search: SearchConfig = field(default_factory=SearchConfig)
    record_curve: bool = False
    min_value_fraction: float = 0.0
    max_factor_bytes: int = 1 << 30


@dataclass
class CutResult:
    value: float
    signs: List[np.ndarray]  # one packed uint64 word array per axis
    iterations: int


@dataclass
class CutStep:
    k: int
    cut_value: float
    residual_norm: float
    compression: float


@dataclass
class CutReport:
    steps: List[CutStep] = field(default_factory=list)
    input_norm: float = 0.0
    final_residual_norm: float = 0.0
    width: int = 0
    # engine extras (not in the reference struct)
    residual_norm_exact: Optional[np.ndarray] = None
    sweeps: Optional[np.ndarray] = None
    passes: int = 0
    kernel_ms: float = 0.0
    total_ms: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    kernel_launches: int = 0


@dataclass
class CutDecomposition:
    shape: tuple
    factors: List[np.ndarray]  # per axis: (width, words) uint64, SignMatrix columns
    coefficients: np.ndarray   # alpha_k = c_k / numel
    channel_axis: int = -1

    def width(self) -> int:
        return int(self.coefficients.shape[0])

    def order(self) -> int:
        return len(self.shape)


def unpack_signs(words: np.ndarray, n: int) -> np.ndarray:
    """Packed SignVector words -> +-1.0 vector (set bit = -1, LSB first)."""
    w = np.ascontiguousarray(words, dtype="<u8")
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")[:n]
    return 1.0 - 2.0 * bits.astype(np.float64)


def expand(d: CutDecomposition, first: int = 0, last: Optional[int] = None) -> np.ndarray:
    """Host reconstruction sum_k alpha_k s_k t_k^T (reference expand(), decompose.hpp:266-270).

    Test/analysis helper for matrices; not on the hot path."""
    last = d.width() if last is None else last
    m, n = d.shape
    S = np.stack([unpack_signs(d.factors[0][k], m) for k in range(first, last)], 1) if last > first else np.zeros((m, 0))
    T = np.stack([unpack_signs(d.factors[1][k], n) for k in range(first, last)], 1) if last > first else np.zeros((n, 0))
    return (S * d.coefficients[first:last]) @ T.T


def _shape_array(shape):
    return (N.u64 * len(shape))(*[int(x) for x in shape])


class Engine:
    """One device context (reference calls are reentrant; one Engine per device)."""

    def __init__(self, device: int = 0):
        self.lib = N.lib()
        h = C.c_void_p()
        st = self.lib.sc_create(C.byref(h), device)
        if st != N.SC_OK:
            raise DeviceError(f"sc_create(device={device}) failed: no usable sm_100 device")
        self.handle = h
        self.device = device

    def close(self):
        if getattr(self, "handle", None):
            self.lib.sc_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != N.SC_OK:
            msg = self.lib.sc_last_error(self.handle).decode()
            raise _ERRORS.get(st, SigcutRuntimeError)(msg)

    # -- core call -----------------------------------------------------------
    def run(self, a, cfg: DecomposeConfig, *, dtype: Optional[str] = None, seed_mode: int = N.SC_SEED_PER_TERM,
            want_remainder: bool = False, shard=None):
        """Runs the device decomposition; returns (CutDecomposition, CutReport, remainder|None).

        ``a`` is a numpy array (host path) or a CUDA torch tensor (device path,
        no host copy of the input).  ``dtype`` ('f32'/'f64') selects the storage
        type of the remainder; default: float32 input -> f32, else f64."""
        if cfg.method not in ("greedy", 0):
            raise InvalidArgument("only the greedy method runs on this engine")
        on_device = hasattr(a, "data_ptr") and getattr(a, "is_cuda", False)
        if on_device:
            import torch

            if dtype is None:
                dtype = "f32" if a.dtype == torch.float32 else "f64"
            want = torch.float32 if dtype == "f32" else torch.float64
            if a.dtype != want:
                a = a.to(want)
            a = a.contiguous()
            shape = tuple(a.shape)
            ptr = a.data_ptr()
            keep = a
        else:
            arr = np.asarray(a)
            if dtype is None:
                dtype = "f32" if arr.dtype == np.float32 else "f64"
            arr = np.ascontiguousarray(arr, dtype=np.float32 if dtype == "f32" else np.float64)
            shape = arr.shape
            ptr = arr.ctypes.data
            keep = arr
        sh = _shape_array(shape)
        prob = N.ScProblem()
        prob.dtype = N.SC_F32 if dtype == "f32" else N.SC_F64
        prob.order = len(shape)
        prob.shape = C.cast(sh, C.POINTER(N.u64))
        prob.data = ptr
        prob.data_on_device = 1 if on_device else 0
        prob.seed_mode = seed_mode
        prob.width = int(cfg.width)
        prob.flush_width = int(cfg.flush_width)
        prob.seed = int(cfg.search.seed) & ((1 << 64) - 1)
        prob.restarts = int(cfg.search.restarts)
        prob.max_sweeps = int(cfg.search.max_sweeps)
        prob.min_value_fraction = float(cfg.min_value_fraction)
        prob.max_factor_bytes = int(cfg.max_factor_bytes)
        msg = C.create_string_buffer(256)
        st = self.lib.sc_validate_problem(C.byref(prob), msg, 256)
        if st != N.SC_OK:
            raise _ERRORS.get(st, InvalidArgument)(msg.value.decode())
        w = max(int(cfg.width), 1)
        words = [(int(d) + 63) // 64 for d in shape]
        signs = [np.zeros((w, wd), np.uint64) for wd in words]
        alpha, cut = np.zeros(w), np.zeros(w)
        rn, rne = np.zeros(w), np.zeros(w)
        sweeps = np.zeros(w, np.uint32)
        rem = np.zeros(shape, np.float32 if dtype == "f32" else np.float64) if want_remainder else None
        res = N.ScResult()
        for i, s in enumerate(signs):
            res.sign_words[i] = s.ctypes.data_as(C.POINTER(N.u64))
        res.alpha = alpha.ctypes.data_as(C.POINTER(C.c_double))
        res.cut_value = cut.ctypes.data_as(C.POINTER(C.c_double))
        res.resid_norm = rn.ctypes.data_as(C.POINTER(C.c_double))
        res.resid_norm_exact = rne.ctypes.data_as(C.POINTER(C.c_double))
        res.sweeps = sweeps.ctypes.data_as(C.POINTER(C.c_uint32))
        res.remainder = rem.ctypes.data if rem is not None else None
        if shard is None:
            self._check(self.lib.sc_greedy_decompose(self.handle, C.byref(prob), C.byref(res)))
        else:  # this rank's band of a row-sharded matrix (sharded.py)
            self._check(self.lib.sc_greedy_decompose_sharded(self.handle, C.byref(prob), C.byref(shard), C.byref(res)))
        del keep
        wd = int(res.width_done)
        numel = float(np.prod([float(d) for d in shape])) if shard is None else float(shard.m_global) * shape[1]
        bits_per_term = 64 + sum(int(d) for d in shape)
        steps = []
        if cfg.record_curve:
            steps = [CutStep(k + 1, float(cut[k]), float(rn[k]), (k + 1) * bits_per_term / (64.0 * numel))
                     for k in range(wd)]
        dec = CutDecomposition(tuple(int(d) for d in shape), [s[:wd].copy() for s in signs], alpha[:wd].copy())
        rep = CutReport(steps, float(res.input_norm), float(res.final_residual_norm), wd,
                        residual_norm_exact=rne[:wd].copy(), sweeps=sweeps[:wd].copy(), passes=int(res.passes),
                        kernel_ms=float(res.kernel_ms), total_ms=float(res.total_ms),
                        h2d_bytes=int(res.h2d_bytes), d2h_bytes=int(res.d2h_bytes),
                        kernel_launches=int(res.kernel_launches))
        rep._cut_values = cut[:wd].copy()
        return dec, rep, rem

    def greedy_decompose(self, a, cfg: DecomposeConfig, dtype: Optional[str] = None):
        dec, rep, _ = self.run(a, cfg, dtype=dtype)
        return dec, rep

    def greedy_signed_cut(self, a, cfg: Optional[SearchConfig] = None, dtype: Optional[str] = None) -> CutResult:
        """One cut searched with cfg.seed itself: order 2 is greedy_signed_cut
        (search.hpp:259-263), any other order axial_greedy_cut (:269-272)."""
        cfg = cfg or SearchConfig()
        dc = DecomposeConfig(width=1, search=cfg)
        dec, rep, _ = self.run(a, dc, dtype=dtype, seed_mode=N.SC_SEED_DIRECT)
        return CutResult(float(rep._cut_values[0]), [f[0] for f in dec.factors], int(rep.sweeps[0]))


_default: Optional[Engine] = None


def default_engine() -> Engine:
    global _default
    if _default is None:
        _default = Engine(0)
    return _default


def greedy_decompose(a, cfg: DecomposeConfig, dtype: Optional[str] = None):
    """Reference ``greedy_decompose``: returns ``(CutDecomposition, CutReport)``."""
    return default_engine().greedy_decompose(a, cfg, dtype=dtype)


def decompose(a, cfg: DecomposeConfig, dtype: Optional[str] = None):
    if cfg.method not in ("greedy", 0):
        raise InvalidArgument("only DecomposeConfig.method == greedy is on the B200 path")
    return greedy_decompose(a, cfg, dtype=dtype)


def greedy_signed_cut(a, cfg: Optional[SearchConfig] = None, dtype: Optional[str] = None) -> CutResult:
    return default_engine().greedy_signed_cut(a, cfg, dtype=dtype)


def axial_greedy_cut(a, cfg: Optional[SearchConfig] = None, dtype: Optional[str] = None) -> CutResult:
    """Order-k cut (axial_run, search.hpp:191-213); order 2 routes to the matrix
    alternation exactly as the reference does (search.hpp:247, :269-272)."""
    return greedy_signed_cut(a, cfg, dtype=dtype)


def width_for_compression(shape, rate: float, coeff_bits: int = 64, source_bits: int = 64) -> int:
    if not (rate > 0.0) or rate > 1.0:
        raise InvalidArgument("width_for_compression: rate must be in (0, 1]")
    sh = _shape_array(shape)
    return int(N.lib().sc_width_for_compression(coeff_bits, source_bits, len(shape),
                                                C.cast(sh, C.POINTER(N.u64)), rate))


def start_vectors(shape, seed: int, term: int, restart: int = 0, seed_mode: int = N.SC_SEED_PER_TERM) -> np.ndarray:
    """Host start words of (term, restart) -- the reference's draw order."""
    sh = _shape_array(shape)
    prob = N.ScProblem()
    prob.dtype, prob.order = N.SC_F64, len(shape)
    prob.shape = C.cast(sh, C.POINTER(N.u64))
    prob.data = 1  # non-null placeholder: validation only
    prob.seed_mode = seed_mode
    prob.width, prob.flush_width, prob.seed, prob.restarts, prob.max_sweeps = 1, 1, seed, restart + 1, 1
    prob.max_factor_bytes = 1 << 62
    out = np.zeros(sum((int(d) + 63) // 64 for d in shape) + 1, np.uint64)
    k = N.lib().sc_start_vectors(C.byref(prob), term, restart, out.ctypes.data_as(C.POINTER(N.u64)))
    return out[:k]


def fill_normal(seed: int, count: int, dtype=np.float64) -> np.ndarray:
    """Xoshiro256pp(seed).next_normal() stream (rng.hpp:58-71), optionally narrowed to f32."""
    if dtype == np.float32:
        out = np.empty(count, np.float32)
        N.lib().sc_fill_normal_f32(seed, count, out.ctypes.data_as(C.POINTER(C.c_float)))
    else:
        out = np.empty(count, np.float64)
        N.lib().sc_fill_normal_f64(seed, count, out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def lpt_schedule(costs, bins: int) -> np.ndarray:
    c = np.ascontiguousarray(costs, np.float64)
    out = np.zeros(len(c), np.uint32)
    N.lib().sc_lpt_schedule(c.ctypes.data_as(C.POINTER(C.c_double)), len(c), bins,
                            out.ctypes.data_as(C.POINTER(C.c_uint32)))
    return out
