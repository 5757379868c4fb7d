"""sigcut-b200: B200-native greedy signed-cut decomposition (arXiv 2410.01799).

The hot path (greedy_decompose -> greedy_matrix_run) runs as one persistent
sm_100a kernel behind the C ABI in ``include/sigcut_b200.h``; this package is
the host-side mirror of the reference's public API over that ABI.
"""
from .api import (  # noqa: F401
    CutDecomposition,
    CutReport,
    CutResult,
    CutStep,
    DecomposeConfig,
    DeviceError,
    Engine,
    InvalidArgument,
    IOError_,
    NotSupported,
    SearchConfig,
    SearchDiagnostics,
    SigcutRuntimeError,
    axial_greedy_cut,
    batch_decompose,
    correct_coefficients,
    decompose,
    default_engine,
    expand,
    fill_normal,
    greedy_decompose,
    greedy_signed_cut,
    lpt_schedule,
    lstsq_decompose,
    rgb_scalars_decompose,
    solve_gram,
    solve_gram_leading,
    start_vectors,
    truncated,
    unpack_signs,
    width_for_compression,
)

from . import io  # noqa: F401,E402  (SCD / DTEN containers)

__all__ = [n for n in dir() if not n.startswith("_")]
