"""CPU tests of the rows around the path that need no GPU:

* the oracle's C restatement (oracle/sigcut_oracle.c) of expansion, Gram
  system, least squares and the SCD / DTEN containers against fixtures
  generated from the reference itself (tests/golden/make_golden.py);
* the product's host-side containers and Cholesky solve (libsigcut_b200.so,
  no kernel launch) against the same fixtures and the reference's malformed-
  input behaviour (proj/tests/test_io.cpp:109-196).
"""
import numpy as np
import pytest

import paper_2410_01799_b200 as sc
from golden_cases import factors_of, load, names
from paper_2410_01799_b200 import io as scio


def dec_of(d):
    shape, ch, fs, co = factors_of(d)
    return sc.CutDecomposition(shape, fs, co, ch)


def bits(x):
    return np.ascontiguousarray(x, np.float64).view(np.uint64)


# ---------------------------------------------------------------- oracle pins
@pytest.mark.parametrize("name", names("expand"))
def test_oracle_expansion_matches_reference(orc, name):
    d = load("expand_" + name)
    shape, ch, fs, co = factors_of(d)
    out = orc.accumulate_expansion(shape, fs, co, data=d["base"], scale=float(d["scale"]),
                                   first_term=int(d["first_term"]), channel_axis=ch)
    assert (bits(out) == bits(d["out"])).all()


@pytest.mark.parametrize("name", names("gram"))
def test_oracle_gram_matches_reference(orc, name):
    d = load("gram_" + name)
    shape, ch, fs, co = factors_of(d)
    g, r = orc.build_gram(d["a"], fs, len(co), ch)
    assert (g == d["gram"]).all()
    assert (bits(r) == bits(d["rhs"])).all()
    assert (bits(orc.correct_coefficients(d["a"], fs, co, ch)) == bits(d["corrected"])).all()


@pytest.mark.parametrize("name", names("lsq"))
def test_oracle_lstsq_matches_reference(orc, name):
    d = load("lsq_" + name)
    r = orc.lstsq_decompose(d["a"], int(d["width"]), seed=int(d["seed"]), channel_axis=int(d["channel_axis"]))
    assert r.width == int(d["width_done"])
    for i, s in enumerate(r.signs):
        assert (s == d[f"signs{i}"]).all()
    assert (bits(r.alpha) == bits(d["alpha"])).all()
    assert (bits(r.resid_norm) == bits(d["resid_norm"])).all()


@pytest.mark.parametrize("name", names("scd"))
def test_oracle_scd_bytes_match_reference(orc, name):
    d = load("scd_" + name)
    shape, ch, fs, co = factors_of(d)
    assert orc.write_scd(shape, fs, co, ch, 64) == d["scd64"].tobytes()
    assert orc.write_scd(shape, fs, co, ch, 32) == d["scd32"].tobytes()


def test_oracle_dten_bytes_match_reference(orc):
    d = load("dten")
    for dt, key in enumerate(("f64", "f32", "u8")):
        assert orc.write_raw(d["a"], dt) == d[key].tobytes()


# ---------------------------------------------------------------- product: SCD
@pytest.mark.parametrize("name", names("scd"))
def test_scd_bytes_identical_to_reference(name):
    d = load("scd_" + name)
    dec = dec_of(d)
    assert scio.write_scd(dec, 64) == d["scd64"].tobytes()
    assert scio.write_scd(dec, 32) == d["scd32"].tobytes()
    assert scio.scd_file_size(dec, 64) == len(d["scd64"])


@pytest.mark.parametrize("name", names("scd"))
def test_scd_round_trip(name):
    d = load("scd_" + name)
    dec = dec_of(d)
    back = scio.read_scd(d["scd64"].tobytes())
    assert back.shape == dec.shape and back.channel_axis == dec.channel_axis
    assert all((x == y).all() for x, y in zip(back.factors, dec.factors))
    assert (bits(back.coefficients) == bits(dec.coefficients)).all()
    # 32-bit coefficients round-trip through f32 rounding (test_io.cpp:89-96)
    b32 = scio.read_scd(d["scd32"].tobytes())
    assert (b32.coefficients == np.asarray(dec.coefficients).astype(np.float32).astype(np.float64)).all()


def test_scd_prefix_truncation_equals_truncated():
    # term-major records: the first k records + patched width = truncated(d, k) (test_io.cpp:98-107)
    d = load("scd_sample_4x4")
    dec = dec_of(d)
    full = d["scd64"].tobytes()
    header = 4 + 1 + 1 + 8 * 2 + 8 + 1
    per = 8 + 1 + 1
    for keep in (0, 1, 3, 6):
        cut = bytearray(full[: header + keep * per])
        cut[4 + 1 + 1 + 16: 4 + 1 + 1 + 16 + 8] = keep.to_bytes(8, "little")
        assert bytes(cut) == scio.write_scd(sc.truncated(dec, keep), 64)


def _scd_error(data):
    with pytest.raises(sc.SigcutRuntimeError) as e:
        scio.read_scd(data)
    assert isinstance(e.value, scio.IOError_)
    return str(e.value)


def test_scd_malformed_inputs_like_reference(ref):
    from oracle.pyoracle import OracleError

    good = load("scd_sample_4x4")["scd64"].tobytes()
    bad_magic = b"X" + good[1:]
    bad_width = bytearray(good)
    bad_width[4 + 1 + 1 + 16 + 8] = 16
    pad = bytearray(good)
    pad[-1] = 0xF0
    overflow = b"SCD1" + bytes([2, 0]) + b"\xff" * 16 + b"\x00" * 8 + bytes([64])
    for blob in (bad_magic, good[:-1], bytes(bad_width), bytes(pad), overflow, b"", b"SCD1\x00"):
        msg = _scd_error(blob)
        with pytest.raises(OracleError) as e:
            ref.read_scd(blob)
        assert e.value.code == 3  # io_error
        assert msg == str(e.value), (msg, str(e.value))


def test_write_scd_rejects_bad_arguments():
    dec = dec_of(load("scd_sample_4x4"))
    with pytest.raises(sc.InvalidArgument):
        scio.write_scd(dec, 16)
    bad = sc.CutDecomposition(dec.shape, dec.factors, np.where(np.arange(dec.width()) == 3, np.inf, dec.coefficients))
    with pytest.raises(sc.InvalidArgument, match="non-finite coefficient"):
        scio.write_scd(bad)


# ---------------------------------------------------------------- product: DTEN
def test_dten_bytes_identical_to_reference():
    d = load("dten")
    for key in ("f64", "f32", "u8"):
        assert scio.write_raw(d["a"], key) == d[key].tobytes()
    assert (bits(scio.read_raw(d["f64"].tobytes())) == bits(d["a"])).all()
    x32, sb = scio.read_raw(d["f32"].tobytes(), return_source_bits=True)
    assert sb == 32 and (x32 == d["a"].astype(np.float32).astype(np.float64)).all()
    x8 = scio.read_raw(d["u8"].tobytes())
    assert (x8 == np.array([[0, 0, 2, 0], [0, 255, 255, 255], [0, 1, 2, 3]])).all()


def test_dten_malformed_inputs_like_reference(ref):
    from oracle.pyoracle import OracleError

    good = load("dten")["f64"].tobytes()
    zero_axis = good[:5] + b"\x00" * 8 + good[13:]
    bad_dtype = bytearray(good)
    bad_dtype[4 + 1 + 16] = 9
    nonfinite = scio.write_raw(np.array([1.0, np.inf]), "f64")
    for blob in (b"XTEN" + good[4:], zero_axis, bytes(bad_dtype), good[:-3], nonfinite, b"DTEN\x00"):
        with pytest.raises(scio.IOError_) as mine:
            scio.read_raw(blob)
        with pytest.raises(OracleError) as theirs:
            ref.read_raw(blob)
        assert theirs.value.code == 3
        assert str(mine.value) == str(theirs.value)


# ---------------------------------------------------------------- product: Cholesky
@pytest.mark.parametrize("name", names("gram"))
def test_solve_gram_bit_identical_to_reference(ref, name):
    d = load("gram_" + name)
    mine = sc.solve_gram(d["gram"], d["rhs"])
    theirs = ref.solve_gram(d["gram"], d["rhs"])
    assert (bits(mine) == bits(theirs)).all()


def test_solve_gram_ridge_and_failure_like_reference(ref):
    # duplicate terms make G singular: the ridge retry (gram.hpp:83-97) still solves
    g = np.array([[4.0, 4.0], [4.0, 4.0]])
    r = np.array([1.0, 1.0])
    assert (bits(sc.solve_gram(g, r)) == bits(ref.solve_gram(g, r))).all()
    with pytest.raises(sc.SigcutRuntimeError, match="factorization failed"):
        sc.solve_gram(np.array([[-1.0]]), np.array([1.0]))


@pytest.mark.parametrize("w,nbits,ch,dup", [(1, 8, 1, None), (12, 64, 1, None), (40, 256, 3, None), (24, 96, 2, 9)])
def test_solve_gram_leading_blocks_bit_identical(ref, w, nbits, ch, dup):
    """The incremental factor of lstsq's term loop (one row per term, O(k^2)): every leading
    block's solution equals the reference's solve_gram of that block bit for bit -- also after
    a duplicated term made a pivot fail and the ridge retry took over (dup)."""
    rng = np.random.default_rng(100 + w)
    f = np.where(rng.standard_normal((w, nbits)) < 0, -1.0, 1.0)
    if dup is not None:
        f[dup] = f[dup - 3]  # term dup repeats an earlier one: singular from block dup + 1 on
    gram = f @ f.T
    rhs = rng.standard_normal((w, ch)) * nbits
    blocks = sc.solve_gram_leading(gram, rhs)
    assert len(blocks) == w
    for k in range(1, w + 1):
        theirs = ref.solve_gram(np.ascontiguousarray(gram[:k, :k]), np.ascontiguousarray(rhs[:k]))
        assert blocks[k - 1].shape == (k, ch)
        assert (bits(blocks[k - 1].reshape(-1)) == bits(np.asarray(theirs).reshape(-1))).all(), k


def test_workload_generator_is_reference_stream(orc):
    from paper_2410_01799_b200.workloads import Xoshiro256pp

    r = Xoshiro256pp(2)
    assert (np.array([r.next_u64() for _ in range(9)], np.uint64) == orc.fill_u64(2, 9)).all()
    r = Xoshiro256pp(0x5CD15EED)
    assert (np.array([r.next_f64() for _ in range(9)]) == orc.fill_f64(0x5CD15EED, 9)).all()


def test_c3_blob_image_recipe():
    from paper_2410_01799_b200.workloads import c3_blob_image

    img = c3_blob_image(40, 30)
    assert img.shape == (40, 30, 3) and img.dtype == np.float32
    assert img.min() >= 0.0 and img.max() <= 1.0
    assert (c3_blob_image(40, 30) == img).all()  # seeded, deterministic


# ---------------------------------------------------------------- PPM / CSV (io.hpp:294-396)
def _ref_only(ref):
    if ref.which != "ref":
        pytest.skip("reference library (oracle/_ref) not built")


def test_ppm_bytes_identical_to_reference(ref):
    from oracle.pyoracle import ref_read_ppm, ref_write_ppm

    _ref_only(ref)
    rng = np.random.default_rng(3)
    for shape in [(1, 1, 3), (7, 5, 3), (16, 33, 3)]:
        a = rng.uniform(-20, 275, size=shape)
        a.flat[:6] = [255.7, -3.2, 100.5, 99.4, 0.0, 254.5][: a.size]
        blob = scio.write_ppm(a)
        assert blob == ref_write_ppm(ref, a)
        assert (scio.read_ppm(blob) == ref_read_ppm(ref, blob)).all()
    with pytest.raises(sc.InvalidArgument, match="m x n x 3"):
        scio.write_ppm(np.zeros((2, 2)))


def test_ppm_reader_like_reference(ref):
    from oracle.pyoracle import OracleError, ref_read_ppm

    _ref_only(ref)
    good = b"P6 # comment\n# another\n2 1\n255\n" + bytes([0x7F] * 6)
    assert (scio.read_ppm(good) == ref_read_ppm(ref, good)).all()
    for blob in (b"P5\n2 2\n255\n....", b"P6\n1 1\n65535\n......", b"P6\n2 2\n255\nxx", b"P6\n0 2\n255\n",
                 b"P6\n99999999999 1\n255\n", b"P6\n2 1\n255", b"P6\n2x1", b"P"):
        with pytest.raises(scio.IOError_) as mine:
            scio.read_ppm(blob)
        with pytest.raises(OracleError) as theirs:
            ref_read_ppm(ref, blob)
        assert str(mine.value) == str(theirs.value), blob


def test_curve_csv_like_reference(ref):
    from oracle.pyoracle import OracleError, ref_read_curve_csv, ref_write_curve_csv

    _ref_only(ref)
    pts = [(0, 0.0, 1.0), (1, 0.03125, 0.9876543210987654), (17, 1.0 / 3.0, 1e-300), (4096, 2.5e-7, 0.1)]
    text = scio.write_curve_csv(pts)
    assert text == ref_write_curve_csv(ref, pts)
    assert scio.read_curve_csv(text) == ref_read_curve_csv(ref, text) == pts
    for bad in ("width,rate\n1,2,3\n", "width,compression_rate,relative_error\n1,2\n",
                "width,compression_rate,relative_error\n-1,0.5,0.5\n", "width,compression_rate,relative_error\nx,1,1\n"):
        with pytest.raises(scio.IOError_) as mine:
            scio.read_curve_csv(bad)
        with pytest.raises(OracleError) as theirs:
            ref_read_curve_csv(ref, bad)
        assert str(mine.value) == str(theirs.value)


def test_emit_curve_uses_the_storage_model(ref):
    rep = sc.CutReport(steps=[sc.CutStep(k, 1.0, 0.5 / k, 0.0) for k in (1, 2, 3)], input_norm=2.0)
    pts = scio.emit_curve(rep, (37, 29), coeff_bits=32, source_bits=16)
    assert pts[0] == (0, 0.0, 1.0)
    for k, (w, rate, err) in zip((1, 2, 3), pts[1:]):
        assert w == k and rate == ref.compression_rate(k, (37, 29), 32, 16) and err == 0.25 / k
