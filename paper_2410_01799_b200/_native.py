"""ctypes binding of the C ABI declared in ``include/sigcut_b200.h``.

Loads the in-tree ``libsigcut_b200.so`` (built by ``build.py`` for sm_100a).
There is no fallback: if the library is missing or no B200 is visible the
product calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsigcut_b200.so")

SC_OK, SC_INVALID_ARGUMENT, SC_RUNTIME_ERROR, SC_CUDA_ERROR, SC_NOT_SUPPORTED, SC_IO_ERROR = 0, 1, 2, 3, 4, 5
SC_F32, SC_F64 = 0, 1
SC_SEED_PER_TERM, SC_SEED_DIRECT = 0, 1
SC_MAX_ORDER = 8

u64 = C.c_uint64
P = C.POINTER


class ScProblem(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32),
        ("order", C.c_int32),
        ("shape", P(u64)),
        ("data", C.c_void_p),
        ("data_on_device", C.c_int32),
        ("seed_mode", C.c_int32),
        ("width", u64),
        ("flush_width", u64),
        ("seed", u64),
        ("restarts", u64),
        ("max_sweeps", u64),
        ("min_value_fraction", C.c_double),
        ("max_factor_bytes", u64),
    ]


class ScResult(C.Structure):
    _fields_ = [
        ("sign_words", P(u64) * SC_MAX_ORDER),
        ("alpha", P(C.c_double)),
        ("cut_value", P(C.c_double)),
        ("resid_norm", P(C.c_double)),
        ("resid_norm_exact", P(C.c_double)),
        ("sweeps", P(C.c_uint32)),
        ("remainder", C.c_void_p),
        ("width_done", u64),
        ("input_norm", C.c_double),
        ("final_residual_norm", C.c_double),
        ("passes", u64),
        ("kernel_ms", C.c_double),
        ("total_ms", C.c_double),
        ("h2d_bytes", u64),
        ("d2h_bytes", u64),
        ("kernel_launches", C.c_int32),
        ("sweep_values", P(C.c_double)),
        ("n_sweep_values", u64),
        ("dense_passes", u64),
        ("delta_passes", u64),
        ("device_bytes", u64),
    ]


class ScShardConfig(C.Structure):
    _fields_ = [
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("m_global", u64),
        ("row0", u64),
        ("n", u64),
        ("dtype", C.c_int32),
        ("ctas", C.c_int32),
        ("timeout_ms", C.c_uint32),
    ]


class ScBatchJob(C.Structure):
    _fields_ = [
        ("problem", ScProblem),
        ("result", C.POINTER(ScResult)),
        ("status", C.c_int32),
        ("device", C.c_int32),
    ]


class ScShardEmulation(C.Structure):
    _fields_ = [
        ("world", C.c_int32),
        ("ctas", C.c_int32),
        ("timeout_ms", C.c_uint32),
        ("dead_rank", C.c_int32),
    ]


class ScFactors(C.Structure):
    _fields_ = [
        ("order", C.c_int32),
        ("shape", P(u64)),
        ("channel_axis", C.c_int32),
        ("width", u64),
        ("sign_words", P(u64) * SC_MAX_ORDER),
        ("coefficients", P(C.c_double)),
    ]


class ScOpStats(C.Structure):
    _fields_ = [
        ("kernel_ms", C.c_double),
        ("total_ms", C.c_double),
        ("h2d_bytes", u64),
        ("d2h_bytes", u64),
        ("kernel_launches", C.c_int32),
    ]


SC_IPC_HANDLE_BYTES = 64
B = P(C.c_uint8)

# every symbol the header declares, with its ctypes signature
SIGNATURES = {
    "sc_version": (C.c_char_p, []),
    "sc_abi_version": (C.c_int, []),
    "sc_create": (C.c_int, [P(C.c_void_p), C.c_int]),
    "sc_destroy": (None, [C.c_void_p]),
    "sc_last_error": (C.c_char_p, [C.c_void_p]),
    "sc_set_option": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64]),
    "sc_get_option": (C.c_int, [C.c_void_p, C.c_char_p, P(C.c_int64)]),
    "sc_greedy_decompose": (C.c_int, [C.c_void_p, P(ScProblem), P(ScResult)]),
    "sc_validate_problem": (C.c_int, [P(ScProblem), C.c_char_p, C.c_size_t]),
    "sc_start_vectors": (u64, [P(ScProblem), u64, u64, P(u64)]),
    "sc_fill_normal_f64": (None, [u64, u64, P(C.c_double)]),
    "sc_fill_normal_f32": (None, [u64, u64, P(C.c_float)]),
    "sc_width_for_compression": (u64, [C.c_int, C.c_int, C.c_int, P(u64), C.c_double]),
    "sc_lpt_schedule": (None, [P(C.c_double), u64, C.c_uint32, P(C.c_uint32)]),
    "sc_batch_decompose": (C.c_int, [P(C.c_int32), C.c_int32, P(ScBatchJob), u64, C.c_char_p, C.c_size_t]),
    "sc_shard_open": (C.c_int, [C.c_void_p, P(ScShardConfig), C.c_void_p]),
    "sc_shard_connect": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sc_shard_reset": (C.c_int, [C.c_void_p]),
    "sc_greedy_decompose_sharded": (C.c_int, [C.c_void_p, P(ScProblem), P(ScShardConfig), P(ScResult)]),
    "sc_shard_close": (None, [C.c_void_p]),
    "sc_greedy_decompose_sharded_emulated": (C.c_int, [C.c_void_p, P(ScProblem), P(ScShardEmulation), P(ScResult)]),
    "sc_accumulate_expansion": (C.c_int, [C.c_void_p, P(ScFactors), C.c_double, u64, u64, C.c_void_p, C.c_int32,
                                          C.c_int32, P(ScOpStats)]),
    "sc_gram_matrix": (C.c_int, [C.c_void_p, P(ScFactors), P(C.c_double), P(ScOpStats)]),
    "sc_contract_terms": (C.c_int, [C.c_void_p, P(ScFactors), C.c_int32, C.c_void_p, C.c_int32, u64, u64,
                                    P(C.c_double), P(ScOpStats)]),
    "sc_solve_gram": (C.c_int, [u64, u64, P(C.c_double), P(C.c_double), P(C.c_double), C.c_char_p, C.c_size_t]),
    "sc_solve_gram_leading": (C.c_int, [u64, u64, P(C.c_double), P(C.c_double), P(C.c_double), C.c_char_p, C.c_size_t]),
    "sc_correct_coefficients": (C.c_int, [C.c_void_p, P(ScFactors), C.c_int32, C.c_void_p, C.c_int32,
                                          P(C.c_double), P(ScOpStats)]),
    "sc_lstsq_decompose": (C.c_int, [C.c_void_p, P(ScProblem), C.c_int32, P(ScResult)]),
    "sc_scd_size": (u64, [P(ScFactors), C.c_int]),
    "sc_write_scd": (C.c_int, [P(ScFactors), C.c_int, B, u64, P(u64), C.c_char_p, C.c_size_t]),
    "sc_read_scd_header": (C.c_int, [B, u64, P(C.c_int32), P(u64), P(C.c_int32), P(u64), P(C.c_int32),
                                     C.c_char_p, C.c_size_t]),
    "sc_read_scd": (C.c_int, [B, u64, P(P(u64)), P(C.c_double), C.c_char_p, C.c_size_t]),
    "sc_dten_size": (u64, [C.c_int32, P(u64), C.c_int32]),
    "sc_write_dten": (C.c_int, [C.c_int32, P(u64), P(C.c_double), C.c_int32, B, u64, P(u64), C.c_char_p,
                                C.c_size_t]),
    "sc_read_dten_header": (C.c_int, [B, u64, P(C.c_int32), P(u64), P(C.c_int32), C.c_char_p, C.c_size_t]),
    "sc_read_dten": (C.c_int, [B, u64, P(C.c_double), C.c_char_p, C.c_size_t]),
}

_lib = None


def lib():
    """The loaded native library (built on first use if absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from . import build as _b

            _b.build()
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
