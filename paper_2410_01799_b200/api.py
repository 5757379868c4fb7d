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
``expand`` / ``truncated``     decompose.hpp:266-270 / :103-115
``accumulate_expansion``       decompose.hpp:182-197
``build_gram``/``solve_gram``  decompose.hpp:383-393 / gram.hpp:83-107
``correct_coefficients``       decompose.hpp:418-428
``lstsq_decompose``            decompose.hpp:434-469
``rgb_scalars_decompose``      decompose.hpp:485-536
``InvalidArgument``            ``std::invalid_argument``
=============================  ==========================================

Every call goes through the C ABI into the sm_100a kernels; nothing here
computes the decomposition on the CPU.
"""
from __future__ import annotations

import contextlib
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


class IOError_(SigcutRuntimeError):
    """sigcut::io_error analogue (io.hpp:22-24; derives from std::runtime_error)."""


_ERRORS = {
    N.SC_INVALID_ARGUMENT: InvalidArgument,
    N.SC_RUNTIME_ERROR: SigcutRuntimeError,
    N.SC_CUDA_ERROR: DeviceError,
    N.SC_NOT_SUPPORTED: NotSupported,
    N.SC_IO_ERROR: IOError_,
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
class SearchDiagnostics:
    """search.hpp:37-40.  sweep_values: c after every sweep of the winning restart.
    The engine recomputes its products (dense refresh) instead of checking a CPU
    delta cache, so max_cache_rel_error is always 0."""
    sweep_values: List[float] = field(default_factory=list)
    max_cache_rel_error: float = 0.0


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
    dense_passes: int = 0
    delta_passes: int = 0
    device_bytes: int = 0  # bytes the kernel moved through L2 / HBM (sc_result::device_bytes)


@dataclass
class CutDecomposition:
    shape: tuple
    factors: List[np.ndarray]  # per SIGN axis (ascending): (width, words) uint64, SignMatrix columns
    coefficients: np.ndarray   # (width,) alpha_k = c_k / numel; (width, channels) when channel_axis >= 0
    channel_axis: int = -1

    def width(self) -> int:
        return int(self.coefficients.shape[0])

    def order(self) -> int:
        return len(self.shape)

    def channels(self) -> int:
        return int(self.shape[self.channel_axis]) if self.channel_axis >= 0 else 1

    def sign_axes(self) -> List[int]:
        return [i for i in range(len(self.shape)) if i != self.channel_axis]

    def _c_struct(self):
        """(ScFactors, keep-alive list) for the C ABI."""
        sh = _shape_array(self.shape)
        fs = [np.ascontiguousarray(f, np.uint64) for f in self.factors]
        co = np.ascontiguousarray(self.coefficients, np.float64)
        f = N.ScFactors()
        f.order = len(self.shape)
        f.shape = C.cast(sh, C.POINTER(N.u64))
        f.channel_axis = self.channel_axis
        f.width = self.width()
        for i, a in enumerate(fs):
            f.sign_words[i] = a.ctypes.data_as(C.POINTER(N.u64))
        f.coefficients = co.ctypes.data_as(C.POINTER(C.c_double))
        return f, [sh, fs, co]


def truncated(d: CutDecomposition, new_width: int) -> CutDecomposition:
    """First ``new_width`` terms (decompose.hpp:103-115)."""
    if new_width > d.width():
        raise InvalidArgument("truncated: width exceeds stored width")
    return CutDecomposition(d.shape, [f[:new_width].copy() for f in d.factors],
                            d.coefficients[:new_width].copy(), d.channel_axis)


def unpack_signs(words: np.ndarray, n: int) -> np.ndarray:
    """Packed SignVector words -> +-1.0 vector (set bit = -1, LSB first)."""
    w = np.ascontiguousarray(words, dtype="<u8")
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")[:n]
    return 1.0 - 2.0 * bits.astype(np.float64)


def _shape_array(shape):
    return (N.u64 * len(shape))(*[int(x) for x in shape])


class Engine:
    """One device context (reference calls are reentrant; one Engine per device)."""

    def __init__(self, device: int = 0, **options):
        self.lib = N.lib()
        h = C.c_void_p()
        st = self.lib.sc_create(C.byref(h), device)
        if st != N.SC_OK:
            raise DeviceError(f"sc_create(device={device}) failed: no usable sm_100 device")
        self.handle = h
        self.device = device
        for k, v in options.items():
            self.set_option(k, v)

    def set_option(self, name: str, value: int) -> None:
        """Engine option of this context (sc_set_option): ctas, delta, delta_div,
        delta_refresh, two_phase, stages, res_rows, fuse_update, variant, fast_delta,
        l2_persist, profile, poison."""
        self._check(self.lib.sc_set_option(self.handle, name.encode(), int(value)))

    def get_option(self, name: str) -> int:
        v = C.c_int64()
        self._check(self.lib.sc_get_option(self.handle, name.encode(), C.byref(v)))
        return int(v.value)

    @contextlib.contextmanager
    def options(self, **kv):
        """Temporarily set engine options (restored on exit)."""
        old = {k: self.get_option(k) for k in kv}
        try:
            for k, v in kv.items():
                self.set_option(k, v)
            yield self
        finally:
            for k, v in old.items():
                self.set_option(k, v)

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
            want_remainder: bool = False, shard=None, diag: Optional[SearchDiagnostics] = None,
            emulate=None):
        """Runs the device decomposition; returns (CutDecomposition, CutReport, remainder|None).

        ``a`` is a numpy array (host path) or a CUDA torch tensor (device path,
        no host copy of the input).  ``dtype`` ('f32'/'f64') selects the storage
        type of the remainder; default: float32 input -> f32, else f64."""
        if cfg.method not in ("greedy", 0):
            raise InvalidArgument("Engine.run is the greedy driver; use lstsq_decompose for least squares")
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
        sv = np.zeros(max(int(cfg.search.max_sweeps), 1)) if diag is not None else None
        if sv is not None:
            res.sweep_values = sv.ctypes.data_as(C.POINTER(C.c_double))
        if emulate is not None:  # row sharding over virtual ranks on this device (sharded.emulated)
            self._check(self.lib.sc_greedy_decompose_sharded_emulated(self.handle, C.byref(prob), C.byref(emulate),
                                                                      C.byref(res)))
        elif shard is None:
            self._check(self.lib.sc_greedy_decompose(self.handle, C.byref(prob), C.byref(res)))
        else:  # this rank's band of a row-sharded matrix (sharded.py)
            self._check(self.lib.sc_greedy_decompose_sharded(self.handle, C.byref(prob), C.byref(shard), C.byref(res)))
        del keep
        wd = int(res.width_done)
        # the global shape: a row-sharded rank holds only its band of the m_global rows
        gshape = tuple(int(d) for d in shape) if shard is None else (int(shard.m_global), int(shape[1]))
        numel = float(np.prod([float(d) for d in gshape]))
        bits_per_term = 64 + sum(gshape)
        steps = []
        if cfg.record_curve:
            steps = [CutStep(k + 1, float(cut[k]), float(rn[k]), (k + 1) * bits_per_term / (64.0 * numel))
                     for k in range(wd)]
        dec = CutDecomposition(tuple(int(d) for d in shape), [s[:wd].copy() for s in signs], alpha[:wd].copy())
        rep = CutReport(steps, float(res.input_norm), float(res.final_residual_norm), wd,
                        residual_norm_exact=rne[:wd].copy(), sweeps=sweeps[:wd].copy(), passes=int(res.passes),
                        kernel_ms=float(res.kernel_ms), total_ms=float(res.total_ms),
                        h2d_bytes=int(res.h2d_bytes), d2h_bytes=int(res.d2h_bytes),
                        kernel_launches=int(res.kernel_launches), dense_passes=int(res.dense_passes),
                        delta_passes=int(res.delta_passes), device_bytes=int(res.device_bytes))
        rep._cut_values = cut[:wd].copy()
        if diag is not None:
            diag.sweep_values = sv[: int(res.n_sweep_values)].tolist()
            diag.max_cache_rel_error = 0.0
        return dec, rep, rem

    def greedy_decompose(self, a, cfg: DecomposeConfig, dtype: Optional[str] = None):
        dec, rep, _ = self.run(a, cfg, dtype=dtype)
        return dec, rep

    # -- around the path: expansion, Gram system, least squares ----------------
    def accumulate_expansion(self, d: CutDecomposition, data=None, scale: float = 1.0, first_term: int = 0,
                             last_term: Optional[int] = None, stats: Optional[dict] = None):
        """``data += sum_{first <= j < last} flip(scale coef_j, parity_j)`` on the device,
        bit-identical to detail::accumulate_expansion (decompose.hpp:182-197).

        ``data``: None (zeros: expand), a numpy array (copied, returned) or a CUDA
        float64 torch tensor (updated in place, no host copy)."""
        f, keep = d._c_struct()
        last = d.width() if last_term is None else int(last_term)
        st = N.ScOpStats()
        if data is not None and hasattr(data, "data_ptr") and getattr(data, "is_cuda", False):
            import torch

            if data.dtype != torch.float64 or not data.is_contiguous():
                raise InvalidArgument("accumulate_expansion: device data must be contiguous float64")
            self._check(self.lib.sc_accumulate_expansion(self.handle, C.byref(f), float(scale), int(first_term), last,
                                                         C.c_void_p(data.data_ptr()), 1, 0, C.byref(st)))
            out = data
        else:
            zero = data is None
            out = np.zeros(d.shape) if zero else np.array(data, np.float64, copy=True).reshape(d.shape)
            self._check(self.lib.sc_accumulate_expansion(self.handle, C.byref(f), float(scale), int(first_term), last,
                                                         C.c_void_p(out.ctypes.data), 0, 1 if zero else 0, C.byref(st)))
        del keep
        if stats is not None:
            stats.update(kernel_ms=st.kernel_ms, total_ms=st.total_ms, h2d_bytes=st.h2d_bytes,
                         d2h_bytes=st.d2h_bytes, kernel_launches=st.kernel_launches)
        return out

    def expand(self, d: CutDecomposition, stats: Optional[dict] = None):
        """Reconstruction sum_j coef_j (outer product of term j's signs) (decompose.hpp:266-270)."""
        return self.accumulate_expansion(d, None, 1.0, 0, None, stats)

    def gram_matrix(self, d: CutDecomposition, stats: Optional[dict] = None) -> np.ndarray:
        """G[i, j] = prod over sign axes of sign_dot (gram_column, decompose.hpp:367-381)."""
        f, keep = d._c_struct()
        w = d.width()
        g = np.zeros((w, w))
        st = N.ScOpStats()
        self._check(self.lib.sc_gram_matrix(self.handle, C.byref(f), g.ctypes.data_as(C.POINTER(C.c_double)),
                                            C.byref(st)))
        del keep
        if stats is not None:
            stats.update(kernel_ms=st.kernel_ms, total_ms=st.total_ms, h2d_bytes=st.h2d_bytes,
                         d2h_bytes=st.d2h_bytes, kernel_launches=st.kernel_launches)
        return g

    def _input(self, a, dtype=None):
        on_device = hasattr(a, "data_ptr") and getattr(a, "is_cuda", False)
        if on_device:
            import torch

            if dtype is None:
                dtype = "f32" if a.dtype == torch.float32 else "f64"
            a = a.to(torch.float32 if dtype == "f32" else torch.float64).contiguous()
            return a, a.data_ptr(), 1, dtype
        arr = np.asarray(a)
        if dtype is None:
            dtype = "f32" if arr.dtype == np.float32 else "f64"
        arr = np.ascontiguousarray(arr, np.float32 if dtype == "f32" else np.float64)
        return arr, arr.ctypes.data, 0, dtype

    def contract_terms(self, d: CutDecomposition, a, first_term: int = 0, count: Optional[int] = None,
                       dtype: Optional[str] = None) -> np.ndarray:
        """<sign outer product of term j, A> per channel (contract_term, decompose.hpp:218-260)."""
        f, keep = d._c_struct()
        count = d.width() - first_term if count is None else count
        arr, ptr, on_dev, dtype = self._input(a, dtype)
        out = np.zeros((max(count, 0), d.channels()))
        self._check(self.lib.sc_contract_terms(self.handle, C.byref(f), N.SC_F32 if dtype == "f32" else N.SC_F64,
                                               C.c_void_p(ptr), on_dev, first_term, count,
                                               out.ctypes.data_as(C.POINTER(C.c_double)), None))
        del keep, arr
        return out if d.channel_axis >= 0 else out[:, 0]

    def correct_coefficients(self, a, d: CutDecomposition, dtype: Optional[str] = None) -> CutDecomposition:
        """Refit the coefficients with the signs fixed (decompose.hpp:418-428)."""
        if tuple(np.shape(a)) != tuple(d.shape):
            raise InvalidArgument("correct_coefficients: shape mismatch")
        if d.width() == 0:
            return d
        f, keep = d._c_struct()
        arr, ptr, on_dev, dtype = self._input(a, dtype)
        out = np.zeros_like(np.asarray(d.coefficients, np.float64))
        self._check(self.lib.sc_correct_coefficients(self.handle, C.byref(f), N.SC_F32 if dtype == "f32" else N.SC_F64,
                                                     C.c_void_p(ptr), on_dev,
                                                     out.ctypes.data_as(C.POINTER(C.c_double)), None))
        del keep, arr
        return CutDecomposition(d.shape, [x.copy() for x in d.factors], out, d.channel_axis)

    def lstsq_decompose(self, a, cfg: DecomposeConfig, dtype: Optional[str] = None, channel_axis: int = -1):
        """Least-squares decomposition (decompose.hpp:434-469); with channel_axis >= 0 the
        scalar-channel variant rgb_scalars_decompose (:485-536).  The term search, the
        Gram column, the contraction and the residual re-expansion run on the device;
        the w x w Cholesky solve runs on the host like the reference's."""
        arr, ptr, on_dev, dtype = self._input(a, dtype)
        shape = tuple(int(x) for x in arr.shape)
        if channel_axis is None:
            channel_axis = len(shape) - 1
        sh = _shape_array(shape)
        prob = N.ScProblem()
        prob.dtype = N.SC_F32 if dtype == "f32" else N.SC_F64
        prob.order = len(shape)
        prob.shape = C.cast(sh, C.POINTER(N.u64))
        prob.data = ptr
        prob.data_on_device = on_dev
        prob.seed_mode = N.SC_SEED_PER_TERM
        prob.width = int(cfg.width)
        prob.flush_width = int(cfg.flush_width)
        prob.seed = int(cfg.search.seed) & ((1 << 64) - 1)
        prob.restarts = int(cfg.search.restarts)
        prob.max_sweeps = int(cfg.search.max_sweeps)
        prob.min_value_fraction = float(cfg.min_value_fraction)
        prob.max_factor_bytes = int(cfg.max_factor_bytes)
        q = shape[channel_axis] if channel_axis >= 0 else 1
        axes = [i for i in range(len(shape)) if i != channel_axis]
        w = max(int(cfg.width), 1)
        signs = [np.zeros((w, (shape[i] + 63) // 64), np.uint64) for i in axes]
        alpha = np.zeros((w, q))
        cut, rn, rne = np.zeros(w), np.zeros(w), np.zeros(w)
        sweeps = np.zeros(w, np.uint32)
        res = N.ScResult()
        for i, sgn in enumerate(signs):
            res.sign_words[i] = sgn.ctypes.data_as(C.POINTER(N.u64))
        res.alpha = alpha.ctypes.data_as(C.POINTER(C.c_double))
        res.cut_value = cut.ctypes.data_as(C.POINTER(C.c_double))
        res.resid_norm = rn.ctypes.data_as(C.POINTER(C.c_double))
        res.resid_norm_exact = rne.ctypes.data_as(C.POINTER(C.c_double))
        res.sweeps = sweeps.ctypes.data_as(C.POINTER(C.c_uint32))
        self._check(self.lib.sc_lstsq_decompose(self.handle, C.byref(prob), int(channel_axis), C.byref(res)))
        del arr
        wd = int(res.width_done)
        numel = float(np.prod([float(x) for x in shape]))
        bits_per_term = 64 * q + sum(int(shape[i]) for i in axes)
        steps = []
        if cfg.record_curve:
            steps = [CutStep(k + 1, float(cut[k]), float(rn[k]), (k + 1) * bits_per_term / (64.0 * numel))
                     for k in range(wd)]
        coef = alpha[:wd].copy() if channel_axis >= 0 else alpha[:wd, 0].copy()
        dec = CutDecomposition(shape, [sgn[:wd].copy() for sgn in signs], coef, channel_axis)
        rep = CutReport(steps, float(res.input_norm), float(res.final_residual_norm), wd,
                        residual_norm_exact=rne[:wd].copy(), sweeps=sweeps[:wd].copy(), passes=int(res.passes),
                        kernel_ms=float(res.kernel_ms), total_ms=float(res.total_ms),
                        h2d_bytes=int(res.h2d_bytes), d2h_bytes=int(res.d2h_bytes),
                        kernel_launches=int(res.kernel_launches), dense_passes=int(res.dense_passes),
                        delta_passes=int(res.delta_passes), device_bytes=int(res.device_bytes))
        rep._cut_values = cut[:wd].copy()
        return dec, rep

    def rgb_scalars_decompose(self, a, cfg: DecomposeConfig, channel_axis: Optional[int] = None,
                              dtype: Optional[str] = None):
        return self.lstsq_decompose(a, cfg, dtype=dtype,
                                    channel_axis=(np.ndim(a) - 1) if channel_axis is None else channel_axis)

    def greedy_signed_cut(self, a, cfg: Optional[SearchConfig] = None, dtype: Optional[str] = None,
                          diag: Optional[SearchDiagnostics] = None) -> CutResult:
        """One cut searched with cfg.seed itself: order 2 is greedy_signed_cut
        (search.hpp:259-263), any other order axial_greedy_cut (:269-272).  With
        ``diag`` the winning restart's per-sweep values are returned like
        SearchDiagnostics."""
        cfg = cfg or SearchConfig()
        dc = DecomposeConfig(width=1, search=cfg)
        dec, rep, _ = self.run(a, dc, dtype=dtype, seed_mode=N.SC_SEED_DIRECT, diag=diag)
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
    """Dispatch on the configured method (decompose.hpp:472-476)."""
    if cfg.method in ("least_squares", "lstsq", 1):
        return default_engine().lstsq_decompose(a, cfg, dtype=dtype)
    return greedy_decompose(a, cfg, dtype=dtype)


def lstsq_decompose(a, cfg: DecomposeConfig, dtype: Optional[str] = None):
    return default_engine().lstsq_decompose(a, cfg, dtype=dtype)


def rgb_scalars_decompose(a, cfg: DecomposeConfig, channel_axis: Optional[int] = None, dtype: Optional[str] = None):
    return default_engine().rgb_scalars_decompose(a, cfg, channel_axis=channel_axis, dtype=dtype)


def expand(d: CutDecomposition) -> np.ndarray:
    """Reconstruction on the device (decompose.hpp:266-270); width 0 gives zeros."""
    return default_engine().expand(d)


def correct_coefficients(a, d: CutDecomposition) -> CutDecomposition:
    return default_engine().correct_coefficients(a, d)


def solve_gram(gram, rhs) -> np.ndarray:
    """Host Cholesky with the reference's ridge retry (gram.hpp:83-107)."""
    g = np.ascontiguousarray(gram, np.float64)
    r = np.ascontiguousarray(rhs, np.float64)
    w = g.shape[0] if g.ndim == 2 else 0
    out = np.zeros_like(r)
    if w == 0:
        return out
    msg = C.create_string_buffer(256)
    st = N.lib().sc_solve_gram(w, r.size // w, g.ctypes.data_as(C.POINTER(C.c_double)),
                               r.ctypes.data_as(C.POINTER(C.c_double)), out.ctypes.data_as(C.POINTER(C.c_double)),
                               msg, 256)
    if st != N.SC_OK:
        raise _ERRORS.get(st, SigcutRuntimeError)(msg.value.decode())
    return out


def solve_gram_leading(gram, rhs) -> List[np.ndarray]:
    """solve_gram of every leading block k = 1..w of one system (what lstsq_decompose solves term
    by term, decompose.hpp:434-469), with the factor grown one row per block: O(k^2) per block,
    each result bit-identical to solve_gram(gram[:k, :k], rhs[:k])."""
    g = np.ascontiguousarray(gram, np.float64)
    w = g.shape[0] if g.ndim == 2 else 0
    r = np.ascontiguousarray(rhs, np.float64).reshape(w, -1) if w else np.zeros((0, 1))
    ch = r.shape[1]
    out = np.zeros((w * (w + 1) // 2, ch))
    if w == 0:
        return []
    msg = C.create_string_buffer(256)
    st = N.lib().sc_solve_gram_leading(w, ch, g.ctypes.data_as(C.POINTER(C.c_double)),
                                       r.ctypes.data_as(C.POINTER(C.c_double)),
                                       out.ctypes.data_as(C.POINTER(C.c_double)), msg, 256)
    if st != N.SC_OK:
        raise _ERRORS.get(st, SigcutRuntimeError)(msg.value.decode())
    res, off = [], 0
    for k in range(1, w + 1):
        res.append(out[off:off + k].copy())
        off += k
    return res


def greedy_signed_cut(a, cfg: Optional[SearchConfig] = None, dtype: Optional[str] = None,
                      diag: Optional[SearchDiagnostics] = None) -> CutResult:
    return default_engine().greedy_signed_cut(a, cfg, dtype=dtype, diag=diag)


def axial_greedy_cut(a, cfg: Optional[SearchConfig] = None, dtype: Optional[str] = None,
                     diag: Optional[SearchDiagnostics] = None) -> CutResult:
    """Order-k cut (axial_run, search.hpp:191-213); order 2 routes to the matrix
    alternation exactly as the reference does (search.hpp:247, :269-272)."""
    return greedy_signed_cut(a, cfg, dtype=dtype, diag=diag)


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


def batch_decompose(inputs, cfgs, dtype: Optional[str] = None, devices=(0,)):
    """Independent greedy decompositions over several devices (sc_batch_decompose:
    LPT by width x numel, one host thread and context per device, no data-path
    communication).  Returns [(CutDecomposition, CutReport, device)] in input order;
    each equals Engine.run of that input.  Raises the first failing job's error."""
    inputs = [np.ascontiguousarray(a) for a in inputs]
    cfgs = list(cfgs)
    if len(inputs) != len(cfgs):
        raise InvalidArgument("batch_decompose: inputs and configs differ in count")
    keep, calls = [], []
    jobs = (N.ScBatchJob * max(1, len(inputs)))()
    for i, (a0, cfg) in enumerate(zip(inputs, cfgs)):
        dt = dtype or ("f32" if a0.dtype == np.float32 else "f64")
        a = np.ascontiguousarray(a0, dtype=np.float32 if dt == "f32" else np.float64)
        shape = a.shape
        sh = _shape_array(shape)
        p = jobs[i].problem
        p.dtype = N.SC_F32 if dt == "f32" else N.SC_F64
        p.order = len(shape)
        p.shape = C.cast(sh, C.POINTER(N.u64))
        p.data = a.ctypes.data
        p.data_on_device = 0
        p.seed_mode = N.SC_SEED_PER_TERM
        p.width = int(cfg.width)
        p.flush_width = int(cfg.flush_width)
        p.seed = int(cfg.search.seed) & ((1 << 64) - 1)
        p.restarts = int(cfg.search.restarts)
        p.max_sweeps = int(cfg.search.max_sweeps)
        p.min_value_fraction = float(cfg.min_value_fraction)
        p.max_factor_bytes = int(cfg.max_factor_bytes)
        w = max(int(cfg.width), 1)
        bufs = {"signs": [np.zeros((w, (int(d) + 63) // 64), np.uint64) for d in shape],
                "alpha": np.zeros(w), "cut": np.zeros(w), "rn": np.zeros(w), "rne": np.zeros(w),
                "sweeps": np.zeros(w, np.uint32)}
        res = N.ScResult()
        for k, sg in enumerate(bufs["signs"]):
            res.sign_words[k] = sg.ctypes.data_as(C.POINTER(N.u64))
        res.alpha = bufs["alpha"].ctypes.data_as(C.POINTER(C.c_double))
        res.cut_value = bufs["cut"].ctypes.data_as(C.POINTER(C.c_double))
        res.resid_norm = bufs["rn"].ctypes.data_as(C.POINTER(C.c_double))
        res.resid_norm_exact = bufs["rne"].ctypes.data_as(C.POINTER(C.c_double))
        res.sweeps = bufs["sweeps"].ctypes.data_as(C.POINTER(C.c_uint32))
        jobs[i].result = C.pointer(res)
        keep.append((a, sh, res))
        calls.append((shape, cfg, bufs, res))
    devs = (C.c_int32 * len(devices))(*devices)
    msg = C.create_string_buffer(512)
    st = N.lib().sc_batch_decompose(devs, len(devices), jobs, len(inputs), msg, 512)
    if st != N.SC_OK:
        raise _ERRORS.get(st, SigcutRuntimeError)(msg.value.decode())
    out = []
    for i, (shape, cfg, b, res) in enumerate(calls):
        wd = int(res.width_done)
        numel = float(np.prod([float(d) for d in shape]))
        bpt = 64 + sum(int(d) for d in shape)
        steps = [CutStep(k + 1, float(b["cut"][k]), float(b["rn"][k]), (k + 1) * bpt / (64.0 * numel))
                 for k in range(wd)] if cfg.record_curve else []
        dec = CutDecomposition(tuple(int(d) for d in shape), [sg[:wd].copy() for sg in b["signs"]],
                               b["alpha"][:wd].copy())
        rep = CutReport(steps, float(res.input_norm), float(res.final_residual_norm), wd,
                        residual_norm_exact=b["rne"][:wd].copy(), sweeps=b["sweeps"][:wd].copy(),
                        passes=int(res.passes), kernel_ms=float(res.kernel_ms), total_ms=float(res.total_ms),
                        h2d_bytes=int(res.h2d_bytes), d2h_bytes=int(res.d2h_bytes),
                        kernel_launches=int(res.kernel_launches), dense_passes=int(res.dense_passes),
                        delta_passes=int(res.delta_passes), device_bytes=int(res.device_bytes))
        rep._cut_values = b["cut"][:wd].copy()
        out.append((dec, rep, int(jobs[i].device)))
    del keep
    return out
