"""CPU tests of the native library's host side (no kernel launches): the C ABI
exports every symbol declared in include/sigcut_b200.h, host validation has
the reference's error semantics, and the host-drawn start vectors / synthetic
streams are the reference generator's."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2410_01799_b200 as sc
from paper_2410_01799_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "sigcut_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = N.lib()
    names = header_functions()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(N.SIGNATURES), "ctypes table and header disagree"
    assert lib.sc_abi_version() == 1
    assert b"sm_100a" in lib.sc_version()


def test_library_is_sm100a_only():
    # the fatbinary carries sm_100a SASS only (no PTX / other archs to JIT)
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def _problem(shape, **kw):
    sh = (N.u64 * len(shape))(*shape)
    p = N.ScProblem()
    p.dtype, p.order, p.shape, p.data = N.SC_F32, len(shape), C.cast(sh, C.POINTER(N.u64)), 1
    p.width, p.flush_width, p.seed, p.restarts, p.max_sweeps = 4, 32, 0, 1, 100
    p.max_factor_bytes = 1 << 30
    for k, v in kw.items():
        setattr(p, k, v)
    p._keep = sh
    return p


@pytest.mark.parametrize("shape,kw,msg", [
    ((4, 0), {}, "zero-length axis"),
    ((4, 4), {"flush_width": 0}, "flush_width must be >= 1"),
    ((4, 4), {"restarts": 0}, "restarts must be >= 1"),
    ((4, 4), {"max_sweeps": 0}, "max_sweeps must be >= 1"),
    ((4, 4), {"width": 1_000_000_000, "max_factor_bytes": 1 << 20}, "factor memory budget"),
    ((4, 4), {"dtype": 7}, "dtype"),
])
def test_validation_matches_reference_errors(shape, kw, msg):
    p = _problem(shape, **kw)
    buf = C.create_string_buffer(256)
    st = N.lib().sc_validate_problem(C.byref(p), buf, 256)
    assert st == N.SC_INVALID_ARGUMENT
    assert msg in buf.value.decode()


def test_validation_accepts_good_problem():
    p = _problem((4096, 4096))
    assert N.lib().sc_validate_problem(C.byref(p), None, 0) == N.SC_OK


def test_validation_budget_boundary_like_reference(orc):
    # per-term bytes = 8 + 8*ceil(m/64) + 8*ceil(n/64) vs max_factor_bytes / width (decompose.hpp:290-298)
    shape, width = (64, 64), 1000
    per_term = 8 + 8 + 8
    ok = _problem(shape, width=width, max_factor_bytes=per_term * width)
    bad = _problem(shape, width=width, max_factor_bytes=per_term * width - 1)
    assert N.lib().sc_validate_problem(C.byref(ok), None, 0) == N.SC_OK
    assert N.lib().sc_validate_problem(C.byref(bad), None, 0) == N.SC_INVALID_ARGUMENT


@pytest.mark.parametrize("shape,seed,term,restart", [((1024, 1024), 0, 0, 0), ((37, 29), 5, 3, 1),
                                                     ((100, 130), 7, 11, 2), ((1, 65), 9, 0, 0),
                                                     ((4096, 4096), 1, 16375, 0)])
def test_start_vectors_are_reference_draws(orc, shape, seed, term, restart):
    # best_of_restarts rng = Xoshiro256pp(substream(substream(seed, term), r)); s0 then t0 (search.hpp:149-150)
    words = sc.start_vectors(shape, seed, term, restart)
    m, n = shape
    wm, wn = (m + 63) // 64, (n + 63) // 64
    raw = orc.fill_u64(orc.substream(orc.substream(seed, term), restart), wm + wn)[wm:]
    if n % 64:
        raw[-1] &= np.uint64((1 << (n % 64)) - 1)
    assert (words == raw).all()


def test_start_vectors_order_k_draw_every_axis(orc):
    shape = (5, 70, 3)
    words = sc.start_vectors(shape, 2, 4, 0)
    raw = orc.fill_u64(orc.substream(orc.substream(2, 4), 0), 1 + 2 + 1)
    raw[0] &= np.uint64(0b11111)
    raw[2] &= np.uint64((1 << 6) - 1)
    raw[3] &= np.uint64(0b111)
    assert (words == raw).all()


def test_direct_seed_mode_for_single_cut(orc):
    w = sc.start_vectors((8, 8), 42, 0, 0, seed_mode=N.SC_SEED_DIRECT)
    raw = orc.fill_u64(orc.substream(42, 0), 2)[1:] & np.uint64(0xFF)
    assert (w == raw).all()


def test_synthetic_streams_are_reference_streams(orc):
    assert np.array_equal(sc.fill_normal(1, 4097), orc.fill_normal(1, 4097))
    assert np.array_equal(sc.fill_normal(3, 999, np.float32), orc.fill_normal(3, 999).astype(np.float32))


def test_width_for_compression_table2():
    assert sc.width_for_compression((4096, 4096), 0.5, 32, 16) == 16320
    assert sc.width_for_compression((1024, 4096), 0.5, 32, 16) == 6512
    assert sc.width_for_compression((14336, 4096), 0.5, 32, 16) == 25442
    assert sc.width_for_compression((32000, 4096), 0.5, 32, 16) == 29023
    with pytest.raises(sc.InvalidArgument):
        sc.width_for_compression((4, 4), 1.5)


def test_lpt_schedule_longest_first():
    costs = np.array([5.0, 3.0, 8.0, 1.0, 2.0, 8.0, 7.0])
    b = sc.lpt_schedule(costs, 3)
    loads = np.bincount(b, weights=costs, minlength=3)
    assert loads.max() - loads.min() <= costs.max()
    # deterministic: same plan twice, ties broken by job index
    assert (sc.lpt_schedule(costs, 3) == b).all()
    assert b[2] == 0 and b[5] == 1  # the two 8s go to the first two empty bins in job order


def test_no_cpu_fallback_without_gpu():
    from conftest import gpu_available

    if gpu_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(sc.DeviceError):
        sc.Engine(0)


def test_host_path_rejects_bad_input_before_device():
    # validation errors surface as the reference's invalid_argument even without a device
    with pytest.raises((sc.InvalidArgument, sc.DeviceError)):
        sc.greedy_decompose(np.zeros((4, 0)), sc.DecomposeConfig(width=1))


def test_cpp_shim_compiles_against_reference_headers(tmp_path):
    """include/sigcut_b200.hpp type-checks against the reference's unchanged
    headers (the drop-in a maintainer would include); skipped where the
    reference tree is absent (the GPU box)."""
    import subprocess

    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc):
        pytest.skip("reference headers absent")
    src = tmp_path / "t.cpp"
    src.write_text('#include <sigcut/sigcut.hpp>\n#include "sigcut_b200.hpp"\n'
                   "int main() { sigcut::DenseTensor a({2, 2}, {1, 2, 3, 4}); sigcut::DecomposeConfig c; c.width = 1;\n"
                   "  auto r = sigcut::b200::greedy_decompose(a, c); return (int)r.first.width(); }\n")
    r = subprocess.run(["g++", "-std=gnu++20", "-fsyntax-only", f"-I{ref_inc}", f"-I{ROOT}/include", str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
