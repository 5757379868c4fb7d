"""CPU tests: pin the C restatement (oracle/liboracle.so) against the reference's
own outputs (golden fixtures from the compiled reference) and, when the
reference build oracle/_ref is present, against it directly; plus the
reference's closed-form known answers (proj/tests/test_search.cpp,
test_decompose.cpp)."""
import os

import numpy as np
import pytest

from golden_cases import cut_names, dec_input, dec_names, load
from oracle.pyoracle import LIBS, Oracle

HAVE_REF = os.path.exists(LIBS["ref"])


def test_rng_streams_match_golden(orc):
    g = load("rng")
    for i, s in enumerate(g["seeds"]):
        s = int(s)
        assert (orc.fill_u64(s, 16) == g["u64"][i]).all()
        assert (orc.fill_normal(s, 17) == g["normal"][i]).all()  # bit-exact Box-Muller
        assert (orc.fill_f64(s, 8) == g["f64"][i]).all()
        assert [orc.substream(s, k) for k in range(6)] == [int(x) for x in g["substream"][i]]
        assert orc.mix64(s) == int(g["mix64"][i])


def test_metrics_table2_and_bf16(orc):
    g = load("metrics")
    for i, s in enumerate(g["shapes"]):
        for j, r in enumerate(g["rates"]):
            assert orc.width_for_compression(tuple(s), float(r), 32, 16) == g["widths"][i, j]
    # Table 2 of the paper: 50% widths
    assert list(g["widths"][:, 0]) == [6512, 16320, 25442, 25442, 29023]
    q = orc.quantize_bf16(g["bf16_in"])
    assert np.array_equal(q, g["bf16_out"]) or np.allclose(q, g["bf16_out"], rtol=0, atol=0)


@pytest.mark.parametrize("name", cut_names())
def test_single_cut_matches_golden(orc, name):
    d = load("cut_" + name)
    r = orc.signed_cut(d["a"], seed=int(d["seed"]), restarts=int(d["restarts"]), max_sweeps=int(d["max_sweeps"]))
    assert r["value"] == float(d["value"])
    assert r["iterations"] == int(d["iterations"])
    for i, s in enumerate(r["signs"]):
        assert (s == d[f"signs{i}"]).all()
    assert np.array_equal(r["sweep_values"], d["sweep_values"])


def test_single_cut_known_answers(orc):
    # test_search.cpp:46-73, :90-136
    assert load("cut_rank1_5x7")["value"] == 35.0
    assert orc.signed_cut(np.array([[1.0, -1.0], [-1.0, 1.0]]), seed=3, restarts=8)["value"] == 4.0
    assert orc.signed_cut(np.ones((3, 3)), seed=1)["value"] == 9.0
    assert orc.signed_cut(np.ones((2, 2, 2)), seed=9)["value"] == 8.0
    r = orc.signed_cut(np.array([1.5, -2.0, 0.25, -0.5]), seed=3)
    assert r["value"] == 4.25 and int(r["signs"][0][0]) == 0b1010


@pytest.mark.parametrize("name", dec_names())
def test_decomposition_matches_golden(orc, name):
    d = load("dec_" + name)
    a = dec_input(name, d)
    o = orc.greedy_decompose(a, int(d["width"]), seed=int(d["seed"]), flush_width=int(d["flush"]),
                             restarts=int(d["restarts"]), max_sweeps=int(d["max_sweeps"]),
                             min_value_fraction=float(d["mvf"]), want_remainder="remainder" in d)
    assert o.width == int(d["width_done"])
    for i in range(len(o.signs)):
        assert (o.signs[i] == d[f"signs{i}"]).all()
    assert np.array_equal(o.cut_value, d["cut_value"])
    assert np.array_equal(o.alpha, d["alpha"])
    assert np.array_equal(o.resid_norm, d["resid_norm"])
    assert np.array_equal(o.iterations, d["iterations"])
    assert o.input_norm == float(d["input_norm"]) and o.final_residual_norm == float(d["final_residual_norm"])
    if "remainder" in d:
        assert np.array_equal(o.remainder.ravel(), d["remainder"].ravel())


def test_decompose_known_answers(orc):
    # width-1 on 3 s t^T -> alpha = 3, R = 0 (test_decompose.cpp:63-77)
    d = load("dec_rank1x3_4x4")
    assert d["alpha"][0] == 3.0 and d["final_residual_norm"] == 0.0
    # 2*I: c1 = 4, alpha1 = 1, ||R1||^2 = 4, R2 = 0 (:79-101)
    d = load("dec_twoI_2x2")
    assert d["cut_value"][0] == 4.0 and d["alpha"][0] == 1.0
    assert abs(d["resid_norm"][0] ** 2 - 4.0) < 1e-12 and d["resid_norm"][1] == 0.0
    # min_value_fraction stop after an exact first term (:344-357)
    assert int(load("dec_mvf_6x6")["width_done"]) == 1


def test_pythagoras_chain(orc):
    # ||R_{k+1}||^2 = ||R_k||^2 - c^2/mn against residuals recomputed from scratch (:103-122)
    for n in (8, 13, 16):
        a = orc.fill_normal(2000 + n, n * n).reshape(n, n)
        prev = float((a * a).sum())
        for k in range(1, 21):
            d = orc.greedy_decompose(a, k, seed=0, flush_width=7, want_remainder=True)
            fresh = float((d.remainder ** 2).sum())
            expect = prev - d.cut_value[-1] ** 2 / (n * n)
            assert abs(fresh - expect) <= 1e-9 * max(1.0, abs(expect))
            prev = fresh


def test_errors_mirror_reference(orc):
    from oracle.pyoracle import OracleError

    with pytest.raises(OracleError):
        orc.greedy_decompose(np.ones((4, 4)), 1, flush_width=0)
    with pytest.raises(OracleError):
        orc.greedy_decompose(np.ones((4, 4)), 1, restarts=0)
    with pytest.raises(OracleError):
        orc.greedy_decompose(np.ones((4, 4)), 1_000_000_000, max_factor_bytes=1 << 20)
    with pytest.raises(OracleError):
        orc.greedy_decompose(np.array([[1.0, np.nan]]), 1)


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (needs /root/reference at build time)")
@pytest.mark.parametrize("seed,shape,w,fw,rs", [(11, (23, 31), 25, 32, 1), (12, (50, 17), 30, 5, 2),
                                                (13, (3, 4, 5), 10, 3, 1), (14, (129, 65), 20, 1, 1),
                                                (15, (6, 7, 2, 3), 6, 2, 2)])
def test_restatement_bit_exact_vs_reference(seed, shape, w, fw, rs):
    o, r = Oracle("orc"), Oracle("ref")
    a = o.fill_normal(seed, int(np.prod(shape))).reshape(shape)
    A = o.greedy_decompose(a, w, seed=seed, flush_width=fw, restarts=rs, want_remainder=True)
    B = r.greedy_decompose(a, w, seed=seed, flush_width=fw, restarts=rs, want_remainder=True)
    assert all((x == y).all() for x, y in zip(A.signs, B.signs))
    assert np.array_equal(A.cut_value, B.cut_value) and np.array_equal(A.resid_norm, B.resid_norm)
    assert np.array_equal(A.iterations, B.iterations) and np.array_equal(A.remainder, B.remainder)
