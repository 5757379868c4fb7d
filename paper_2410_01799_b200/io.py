"""SCD / DTEN containers over the C ABI (reference ``io.hpp``).

=========================  =====================================
this module                reference (proj/include/sigcut/io.hpp)
=========================  =====================================
``scd_file_size``          ``scd_file_size``        :135-140
``write_scd``              ``write_scd``            :142-166
``read_scd``               ``read_scd``             :168-213
``write_raw``              ``write_raw``            :226-246
``read_raw``               ``read_raw``             :250-292
``write_ppm`` / ``read_ppm`` ``write_ppm`` / ``read_ppm`` :324-356
``write_curve_csv`` etc.   ``write_curve_csv`` / ``read_curve_csv`` :363-396
``emit_curve``             ``emit_curve``   (metrics.hpp:101-111)
``IOError_``               ``sigcut::io_error``     :22-24
=========================  =====================================

Bytes are identical to the reference's streams, so a decomposition computed
on the GPU is a drop-in for ``sigcut decompose ... out.scd``.
The encoders are host C++ in the engine library (byte layout work, no device
compute).
"""
from __future__ import annotations

import ctypes as C
import re

import numpy as np

from . import _native as N
from .api import _ERRORS, CutDecomposition, IOError_, InvalidArgument, SigcutRuntimeError

RAW_DTYPES = {"f64": 0, "f32": 1, "u8": 2, 0: 0, 1: 1, 2: 2}


def _raise(st: int, msg) -> None:
    if st != N.SC_OK:
        raise _ERRORS.get(st, SigcutRuntimeError)(msg.value.decode())


def _buf(data: bytes):
    arr = np.frombuffer(bytes(data), np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
    return arr, arr.ctypes.data_as(C.POINTER(C.c_uint8))


def scd_file_size(d: CutDecomposition, coeff_bits: int = 64) -> int:
    f, keep = d._c_struct()
    n = int(N.lib().sc_scd_size(C.byref(f), coeff_bits))
    del keep
    return n


def write_scd(d: CutDecomposition, coeff_bits: int = 64) -> bytes:
    if coeff_bits not in (32, 64):
        raise InvalidArgument("write_scd: coeff_bits must be 32 or 64")
    f, keep = d._c_struct()
    cap = int(N.lib().sc_scd_size(C.byref(f), coeff_bits))
    out = np.zeros(max(cap, 1), np.uint8)
    written = N.u64()
    msg = C.create_string_buffer(256)
    st = N.lib().sc_write_scd(C.byref(f), coeff_bits, out.ctypes.data_as(C.POINTER(C.c_uint8)), cap,
                              C.byref(written), msg, 256)
    del keep
    _raise(st, msg)
    return bytes(out[: written.value])


def read_scd(data: bytes) -> CutDecomposition:
    arr, p = _buf(data)
    order, chax, cbits = C.c_int32(), C.c_int32(), C.c_int32()
    width = N.u64()
    shape = (N.u64 * N.SC_MAX_ORDER)()
    msg = C.create_string_buffer(256)
    _raise(N.lib().sc_read_scd_header(p, len(data), C.byref(order), shape, C.byref(chax), C.byref(width),
                                      C.byref(cbits), msg, 256), msg)
    k, ca, w = order.value, chax.value, int(width.value)
    shp = tuple(int(shape[i]) for i in range(k))
    q = shp[ca] if ca >= 0 else 1
    axes = [i for i in range(k) if i != ca]
    # allocation guard: the payload must hold every record (read_scd would hit EOF)
    per_term = q * cbits.value // 8 + sum((shp[i] + 7) // 8 for i in axes)
    if w and per_term and w > len(data) // per_term + 1:
        raise IOError_("truncated payload")
    fs = [np.zeros((max(w, 1), (shp[i] + 63) // 64), np.uint64) for i in axes]
    co = np.zeros((max(w, 1), q))
    ptrs = (C.POINTER(N.u64) * max(1, len(fs)))(*[f.ctypes.data_as(C.POINTER(N.u64)) for f in fs])
    _raise(N.lib().sc_read_scd(p, len(data), ptrs, co.ctypes.data_as(C.POINTER(C.c_double)), msg, 256), msg)
    del arr
    return CutDecomposition(shp, [f[:w] for f in fs], co[:w] if ca >= 0 else co[:w, 0], ca)


def write_raw(a, dtype="f64") -> bytes:
    a = np.ascontiguousarray(a, np.float64)
    dt = RAW_DTYPES[dtype]
    sh = (N.u64 * a.ndim)(*a.shape)
    cap = int(N.lib().sc_dten_size(a.ndim, sh, dt))
    out = np.zeros(max(cap, 1), np.uint8)
    written = N.u64()
    msg = C.create_string_buffer(256)
    st = N.lib().sc_write_dten(a.ndim, sh, a.ctypes.data_as(C.POINTER(C.c_double)), dt,
                               out.ctypes.data_as(C.POINTER(C.c_uint8)), cap, C.byref(written), msg, 256)
    _raise(st, msg)
    return bytes(out[: written.value])


def read_raw(data: bytes, return_source_bits: bool = False):
    arr, p = _buf(data)
    order, dt = C.c_int32(), C.c_int32()
    shape = (N.u64 * N.SC_MAX_ORDER)()
    msg = C.create_string_buffer(256)
    _raise(N.lib().sc_read_dten_header(p, len(data), C.byref(order), shape, C.byref(dt), msg, 256), msg)
    shp = tuple(int(shape[i]) for i in range(order.value))
    es = {0: 8, 1: 4, 2: 1}[dt.value]
    numel = int(np.prod(shp))
    if numel * es > len(data):
        raise IOError_("truncated payload")
    out = np.zeros(shp)
    _raise(N.lib().sc_read_dten(p, len(data), out.ctypes.data_as(C.POINTER(C.c_double)), msg, 256), msg)
    del arr
    if return_source_bits:
        return out, {0: 64, 1: 32, 2: 8}[dt.value]
    return out


# ---------------------------------------------------------------------------
# PPM (io.hpp:294-356) and CSV curve reports (io.hpp:358-396), with the curve
# helper emit_curve (metrics.hpp:99-111).  Plain byte/text formats on the host.
# ---------------------------------------------------------------------------
def write_ppm(a) -> bytes:
    """Binary P6, maxval 255; values clamped to [0, 255], halves rounded away from zero."""
    a = np.asarray(a, np.float64)
    if a.ndim != 3 or a.shape[2] != 3:
        raise InvalidArgument("write_ppm: tensor must have shape m x n x 3")
    h, w = a.shape[0], a.shape[1]
    body = np.floor(np.clip(a, 0.0, 255.0) + 0.5).astype(np.uint8)  # lround on [0, 255]
    return f"P6\n{w} {h}\n255\n".encode() + body.tobytes()


def _isspace(c) -> bool:  # C isspace in the "C" locale
    return c is not None and c in b" \t\n\v\f\r"


def _isdigit(c) -> bool:
    return c is not None and 48 <= c <= 57


def _ppm_token(data: bytes, pos: int):
    n = len(data)
    c = data[pos] if pos < n else None
    pos += 1
    while c is not None and (_isspace(c) or c == ord("#")):
        if c == ord("#"):
            while c is not None and c != ord("\n"):
                c = data[pos] if pos < n else None
                pos += 1
        c = data[pos] if pos < n else None
        pos += 1
    if not _isdigit(c):
        raise IOError_("malformed PPM header")
    value = 0
    while _isdigit(c):
        value = value * 10 + (c - ord("0"))
        if value > (1 << 32):
            raise IOError_("PPM dimension overflow")
        c = data[pos] if pos < n else None
        pos += 1
    if c is not None:
        pos -= 1  # unget
    return value, pos


def read_ppm(data: bytes) -> np.ndarray:
    """height x width x 3 float64 in [0, 255] (read_ppm, io.hpp:324-340)."""
    data = bytes(data)
    if len(data) < 2:
        raise IOError_("truncated payload")
    if data[:2] != b"P6":
        raise IOError_("not a binary P6 PPM")
    pos = 2
    width, pos = _ppm_token(data, pos)
    height, pos = _ppm_token(data, pos)
    maxval, pos = _ppm_token(data, pos)
    if maxval != 255:
        raise IOError_("PPM maxval must be 255")
    if pos >= len(data) or not _isspace(data[pos]):
        raise IOError_("malformed PPM header")
    pos += 1
    if width == 0 or height == 0:
        raise IOError_("PPM with empty dimensions")
    count = height * width * 3
    if len(data) - pos < count:
        raise IOError_("truncated payload")
    px = np.frombuffer(data, np.uint8, count=count, offset=pos)
    return px.astype(np.float64).reshape(height, width, 3)


def emit_curve(report, shape, coeff_bits: int = 64, source_bits: int = 64, channel_axis: int = -1):
    """(width, compression_rate, relative_error) rows from the width-0 point (0, 0, 1)."""
    if report.input_norm == 0.0:
        raise InvalidArgument("emit_curve: zero input norm")
    shape = tuple(int(x) for x in shape)
    channels = shape[channel_axis] if channel_axis >= 0 else 1
    bits = coeff_bits * channels + sum(n for i, n in enumerate(shape) if i != channel_axis)
    src = float(source_bits) * float(np.prod([float(x) for x in shape]))
    pts = [(0, 0.0, 1.0)]
    for st in report.steps:
        pts.append((int(st.k), st.k * float(bits) / src, st.residual_norm / report.input_norm))
    return pts


def write_curve_csv(points) -> str:
    """`width,compression_rate,relative_error`, full-precision decimals (%.17g)."""
    out = ["width,compression_rate,relative_error\n"]
    for w, rate, err in points:
        out.append(f"{int(w)},{'%.17g' % rate},{'%.17g' % err}\n")
    return "".join(out)


_CSV_NUM = re.compile(r"-?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][-+]?\d+)?|inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?)",
                      re.IGNORECASE)


def read_curve_csv(text: str):
    lines = text.split("\n")
    if not lines or lines[0] != "width,compression_rate,relative_error":
        raise IOError_("bad CSV header")
    pts = []
    for line in lines[1:]:
        if not line:
            continue
        parts = line.split(",")
        if len(parts) != 3 or not re.fullmatch(r"[0-9]+", parts[0]) or not _CSV_NUM.fullmatch(parts[1]) \
                or not _CSV_NUM.fullmatch(parts[2]):
            raise IOError_("bad CSV row")
        pts.append((int(parts[0]), float(parts[1]), float(parts[2])))
    return pts
