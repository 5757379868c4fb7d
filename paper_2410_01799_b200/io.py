"""SCD / DTEN containers over the C ABI (reference ``io.hpp``).

=========================  =====================================
this module                reference (proj/include/sigcut/io.hpp)
=========================  =====================================
``scd_file_size``          ``scd_file_size``        :135-140
``write_scd``              ``write_scd``            :142-166
``read_scd``               ``read_scd``             :168-213
``write_raw``              ``write_raw``            :226-246
``read_raw``               ``read_raw``             :250-292
``IOError_``               ``sigcut::io_error``     :22-24
=========================  =====================================

Bytes are identical to the reference's streams, so a decomposition computed
on the GPU is a drop-in for ``sigcut decompose ... out.scd``.
The encoders are host C++ in the engine library (byte layout work, no device
compute).
"""
from __future__ import annotations

import ctypes as C

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
