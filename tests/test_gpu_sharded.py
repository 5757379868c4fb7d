"""Row-sharded path at world 2 and 4 on ONE B200.

The pool gives one GPU per call, and ranks whose kernels wait on one another
must not run as separate launches on one device.  So the ranks are emulated as
ONE cooperative launch over all ranks' bands (sc_greedy_decompose_sharded_emulated):
CTA block r runs rank r's band with rank r's parameters and exchange region,
through the same multi-rank code as the IPC path -- rank partials of R^T s and
of the objective, bounded rank-local and cross-rank barriers, owners publishing
the next t to every rank.  The host checks that every rank took identical
decisions (t words, c, sweeps) before gathering.

Parity: against the single-GPU engine (world 1) on the same input -- row and
column signs bit-identical, sweeps equal, c within 1e-12 (the rank partials add
the same f64 terms in a different order) -- and against the reference.
alpha = c / (m_global * n) (the advisor's round-1 finding: the local row count
was used)."""
import numpy as np
import pytest

import paper_2410_01799_b200 as sc
from paper_2410_01799_b200 import sharded

pytestmark = pytest.mark.gpu

CASES = [((1024, 1024), "f32", 24), ((600, 777), "f64", 16), ((512, 16384), "f32", 5), ((2000, 300), "f32", 30),
         ((1500, 2048), "f64", 12)]


def _cfg(width, seed):
    return sc.DecomposeConfig(width=width, flush_width=8, record_curve=True, search=sc.SearchConfig(seed=seed))


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("shape,dtype,width", CASES)
def test_emulated_ranks_equal_world1(engine, ref, world, shape, dtype, width):
    m, n = shape
    a = ref.fill_normal(31 * m + n, m * n).reshape(m, n)
    a = a.astype(np.float32) if dtype == "f32" else a
    cfg = _cfg(width, 7)
    dec, rep, rem = engine.run(a, cfg, dtype=dtype, want_remainder=True)
    sdec, srep, srem = sharded.emulated(a, cfg, world, dtype=dtype, engine=engine, want_remainder=True)
    assert sdec.width() == dec.width() == width
    assert (sdec.factors[0] == dec.factors[0]).all(), "row signs"
    assert (sdec.factors[1] == dec.factors[1]).all(), "column signs"
    assert np.array_equal(srep.sweeps, rep.sweeps)
    c, sc_ = rep._cut_values, srep._cut_values
    assert np.max(np.abs(sc_ - c) / np.abs(c)) <= 1e-12
    # alpha uses the GLOBAL element count
    assert np.array_equal(sdec.coefficients, sc_ / (float(m) * n))
    assert np.max(np.abs(srep.residual_norm_exact - rep.residual_norm_exact) / rep.residual_norm_exact) <= 1e-10
    assert np.max(np.abs(np.array([s.residual_norm for s in srep.steps]) -
                         np.array([s.residual_norm for s in rep.steps])) / rep.input_norm) <= 1e-10
    # compression p_k of the global shape (CutStep::compression, metrics.hpp:46-52)
    assert srep.steps[-1].compression == rep.steps[-1].compression
    assert np.max(np.abs(srem.astype(np.float64) - rem.astype(np.float64))) <= (1e-5 if dtype == "f32" else 1e-12)
    if dtype == "f64":  # and the reference itself
        od = ref.greedy_decompose(a, width, seed=7, flush_width=8)
        assert (sdec.factors[0] == od.signs[0]).all() and (sdec.factors[1] == od.signs[1]).all()
        assert np.max(np.abs(sc_ - od.cut_value) / np.abs(od.cut_value)) <= 1e-10


def test_emulated_world1_is_the_engine(engine, ref):
    a = ref.fill_normal(3, 700 * 513).reshape(700, 513).astype(np.float32)
    cfg = _cfg(10, 2)
    with engine.options(fast_delta=0, delta_div=32):  # the barrier passes the row-sharded path runs
        dec, rep, _ = engine.run(a, cfg, dtype="f32")
    sdec, srep, _ = sharded.emulated(a, cfg, 1, dtype="f32", engine=engine)
    assert all((x == y).all() for x, y in zip(dec.factors, sdec.factors))
    assert np.array_equal(rep._cut_values, srep._cut_values)


@pytest.mark.parametrize("world", [2, 8])
def test_emulated_dense_only_and_delta_agree(engine, ref, world):
    """Delta passes over the rank partials (only ranks with a flipped row send a
    partial) against dense-only passes, both sharded."""
    a = ref.fill_normal(17, 2048 * 1024).reshape(2048, 1024).astype(np.float32)
    cfg = _cfg(20, 9)
    out = {}
    for mode in (0, 1):
        with engine.options(delta=mode):
            out[mode] = sharded.emulated(a, cfg, world, dtype="f32", engine=engine)
    (d0, r0, _), (d1, r1, _) = out[0], out[1]
    assert all((x == y).all() for x, y in zip(d0.factors, d1.factors))
    assert np.array_equal(r0.sweeps, r1.sweeps)
    assert np.max(np.abs(r1._cut_values - r0._cut_values) / np.abs(r0._cut_values)) <= 1e-12


def test_dead_rank_times_out_instead_of_hanging(engine, ref):
    """A rank whose kernel never joins: the other ranks' bounded spins time out,
    set the shared abort word, and the call raises (runtime_error), instead of
    hanging the GPU.  The context stays usable."""
    a = ref.fill_normal(5, 512 * 256).reshape(512, 256).astype(np.float32)
    for dead in (0, 1):
        with pytest.raises(sc.SigcutRuntimeError, match="did not arrive"):
            sharded.emulated(a, _cfg(4, 1), 2, dtype="f32", engine=engine, timeout_ms=200, dead_rank=dead)
    dec, rep, _ = engine.run(a, _cfg(4, 1), dtype="f32")
    od = ref.greedy_decompose(a.astype(np.float64), 4, seed=1, flush_width=8)
    assert (dec.factors[0] == od.signs[0]).all()


def test_emulation_rejects_bad_layouts(engine):
    a = np.ones((100, 64), np.float32)
    with pytest.raises(sc.NotSupported):
        sharded.emulated(a, _cfg(2, 0), 4, dtype="f32", engine=engine)  # 25-row bands < 37 CTAs
    with pytest.raises(sc.InvalidArgument):
        sharded.emulated(a, _cfg(2, 0), 9, dtype="f32", engine=engine)


# ------------------------------------------------ batch over devices (C ABI)
def test_batch_decompose_equals_single_runs(engine, ref):
    """sc_batch_decompose (LPT over the listed devices, one context and host thread per
    device): every job's result equals Engine.run of that input; device list [0, 0]
    runs two contexts on the one GPU concurrently."""
    shapes = [(300, 200), (64, 1024), (1000, 96), (33, 33), (512, 512)]
    arrs = [ref.fill_normal(40 + i, m * n).reshape(m, n).astype(np.float32) for i, (m, n) in enumerate(shapes)]
    cfgs = [_cfg(6 + i, 3 * i + 1) for i in range(len(shapes))]
    for devices in ((0,), (0, 0)):
        out = sc.batch_decompose(arrs, cfgs, dtype="f32", devices=devices)
        for a, cfg, (dec, rep, dev) in zip(arrs, cfgs, out):
            d1, r1, _ = engine.run(a, cfg, dtype="f32")
            assert dev == 0
            assert all((x == y).all() for x, y in zip(dec.factors, d1.factors))
            assert np.array_equal(rep.sweeps, r1.sweeps)
            assert np.array_equal(rep._cut_values, r1._cut_values)
    bad = list(cfgs)
    bad[1] = sc.DecomposeConfig(width=2, search=sc.SearchConfig(restarts=0))
    with pytest.raises(sc.InvalidArgument):
        sc.batch_decompose(arrs, bad, dtype="f32")
