"""GPU parity of the rows around the path, through the C ABI:

* expansion / accumulate_expansion (decompose.hpp:128-197, :266-270): the
  device result is BIT-IDENTICAL to the reference (same per-element term
  order, exact sign flips);
* Gram matrix (gram_column, decompose.hpp:367-381): integers, bit-identical;
* contract_term (decompose.hpp:218-260): f64 sums in a parallel order, so
  within 1e-12 of sum|a| (the reference sums sequentially);
* correct_coefficients / lstsq_decompose / rgb_scalars_decompose: signs
  bit-identical to the reference, coefficients and residual norms within
  1e-9 relative (they inherit the contraction's last-bit differences);
* SCD bytes of a device decomposition identical to the reference's file.
"""
import numpy as np
import pytest

import paper_2410_01799_b200 as sc
from golden_cases import factors_of, load, names
from paper_2410_01799_b200 import io as scio

pytestmark = pytest.mark.gpu


def bits(x):
    return np.ascontiguousarray(x, np.float64).view(np.uint64)


def dec_of(d):
    shape, ch, fs, co = factors_of(d)
    return sc.CutDecomposition(shape, fs, co, ch)


@pytest.mark.parametrize("name", names("expand"))
def test_expansion_bit_identical_golden(engine, name):
    d = load("expand_" + name)
    dec = dec_of(d)
    base = d["base"]
    st = {}
    out = engine.accumulate_expansion(dec, None if not base.any() else base, scale=float(d["scale"]),
                                      first_term=int(d["first_term"]), stats=st)
    assert (bits(out) == bits(d["out"])).all()
    assert st["kernel_launches"] >= 1


def test_expand_width0_and_truncated(engine, ref):
    d = dec_of(load("expand_mat_37x70"))
    z = engine.expand(sc.truncated(d, 0))
    assert z.shape == (37, 70) and not z.any()
    t = sc.truncated(d, 17)
    assert (bits(engine.expand(t)) == bits(ref.accumulate_expansion(t.shape, t.factors, t.coefficients))).all()
    with pytest.raises(sc.InvalidArgument):
        sc.truncated(d, 41)


def test_expansion_in_place_on_device_tensor(engine, ref):
    import torch

    d = dec_of(load("expand_resid_37x70"))
    base = load("expand_resid_37x70")["base"]
    t = torch.tensor(base, dtype=torch.float64, device="cuda")
    engine.accumulate_expansion(d, t, scale=-1.0, first_term=5)
    assert (bits(t.cpu().numpy()) == bits(load("expand_resid_37x70")["out"])).all()


@pytest.mark.parametrize("shape,w,ragged", [((1024, 1024), 256, False), ((333, 517), 1000, True),
                                            ((4096, 64), 65, True)])
def test_expansion_of_device_decomposition_matches_reference(engine, ref, shape, w, ragged):
    a = ref.fill_normal(41, shape[0] * shape[1]).reshape(shape)
    cfg = sc.DecomposeConfig(width=min(w, 64), flush_width=1, search=sc.SearchConfig(seed=3))
    dec, rep, rem = engine.run(a, cfg, dtype="f64", want_remainder=True)
    if ragged:  # a longer synthetic term list (random signs, decaying coefficients) on the same shape
        rng = np.random.default_rng(5)
        fs = []
        for n in shape:
            nw = (n + 63) // 64
            f = rng.integers(0, 1 << 63, size=(w, nw), dtype=np.uint64) * np.uint64(2)
            f ^= rng.integers(0, 2, size=(w, nw), dtype=np.uint64)
            if n % 64:
                f[:, -1] &= np.uint64((1 << (n % 64)) - 1)
            fs.append(f)
        dec = sc.CutDecomposition(shape, fs, np.exp(-np.arange(w) / 300.0) * rng.uniform(0.5, 1.0, w))
    mine = engine.expand(dec)
    theirs = ref.accumulate_expansion(shape, dec.factors, dec.coefficients)
    assert (bits(mine) == bits(theirs)).all()
    if not ragged:  # A - expand(d) is the remainder up to rounding of the deflation order
        assert np.abs(a - mine - rem).max() <= 1e-12 * np.abs(a).max()


@pytest.mark.parametrize("name", names("gram"))
def test_gram_bit_identical_and_contraction(engine, name):
    d = load("gram_" + name)
    dec = dec_of(d)
    assert (engine.gram_matrix(dec) == d["gram"]).all()
    rhs = engine.contract_terms(dec, d["a"])
    scale = np.abs(d["a"]).sum()
    assert np.abs(rhs - d["rhs"].reshape(rhs.shape)).max() <= 1e-12 * scale
    # f32 storage of A: the contraction widens exactly (DTEN f32 semantics)
    a32 = d["a"].astype(np.float32)
    r32 = engine.contract_terms(dec, a32)
    assert np.abs(r32 - engine.contract_terms(dec, a32.astype(np.float64))).max() == 0.0
    corr = engine.correct_coefficients(d["a"], dec)
    np.testing.assert_allclose(corr.coefficients, d["corrected"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("name", names("lsq"))
def test_lstsq_matches_reference(engine, name):
    d = load("lsq_" + name)
    ch = int(d["channel_axis"])
    cfg = sc.DecomposeConfig(width=int(d["width"]), record_curve=True, search=sc.SearchConfig(seed=int(d["seed"])))
    dec, rep = engine.lstsq_decompose(d["a"], cfg, channel_axis=ch)
    assert dec.width() == int(d["width_done"])
    for i, f in enumerate(dec.factors):
        assert (f == d[f"signs{i}"]).all(), f"axis slot {i}"
    np.testing.assert_allclose(dec.coefficients, d["alpha"], rtol=1e-9, atol=1e-13)
    np.testing.assert_allclose([s.residual_norm for s in rep.steps], d["resid_norm"], rtol=1e-10)
    assert abs(rep.input_norm - float(d["input_norm"])) <= 1e-12 * float(d["input_norm"])
    # least squares never does worse than greedy's coefficients on the same signs
    assert rep.final_residual_norm <= rep.input_norm


def test_lstsq_dispatch_and_validation(engine, ref):
    a = load("lsq_mat_24x20")["a"]
    cfg = sc.DecomposeConfig(width=3, method="least_squares", search=sc.SearchConfig(seed=7))
    dec, rep = sc.decompose(a, cfg)
    assert (dec.factors[0] == load("lsq_mat_24x20")["signs0"][:3]).all()
    with pytest.raises(sc.InvalidArgument, match="channel axis too long"):
        engine.rgb_scalars_decompose(np.ones((4, 4, 9)), sc.DecomposeConfig(width=1))
    with pytest.raises(sc.InvalidArgument, match="order >= 2"):
        engine.rgb_scalars_decompose(np.ones(5), sc.DecomposeConfig(width=1), channel_axis=0)


def test_device_decomposition_scd_is_reference_file(engine, ref):
    # sigcut decompose -> write_scd: the GPU decomposition's container bytes equal
    # the reference's for the same input (f64 storage, bit-exact trajectory)
    a = ref.fill_normal(77, 96 * 80).reshape(96, 80)
    dec, rep = engine.greedy_decompose(a, sc.DecomposeConfig(width=24, search=sc.SearchConfig(seed=0x5CD15EED)),
                                       dtype="f64")
    od = ref.greedy_decompose(a, 24, seed=0x5CD15EED)
    mine = scio.write_scd(dec, 64)
    theirs = ref.write_scd(a.shape, od.signs, od.alpha, -1, 64)
    assert len(mine) == len(theirs)
    # sign columns byte-identical; coefficients agree to the f64 tolerance (the
    # reference defers rank-1 updates by flush_width, the engine applies them eagerly)
    back, rback = scio.read_scd(mine), scio.read_scd(theirs)
    assert all((x == y).all() for x, y in zip(back.factors, rback.factors))
    np.testing.assert_allclose(back.coefficients, rback.coefficients, rtol=1e-12)
    header, per = 4 + 1 + 1 + 16 + 8 + 1, 8 + 12 + 10
    for j in range(24):
        r0 = header + j * per + 8
        assert mine[r0: r0 + 22] == theirs[r0: r0 + 22]
    assert (bits(engine.expand(back)) == bits(ref.accumulate_expansion(a.shape, back.factors, back.coefficients))).all()


def test_lstsq_f32_and_device_inputs(engine, ref):
    import torch

    a = ref.fill_normal(505, 30 * 22).reshape(30, 22)
    a32 = a.astype(np.float32)
    cfg = sc.DecomposeConfig(width=5, search=sc.SearchConfig(seed=9))
    d_host, r_host = engine.lstsq_decompose(a32, cfg)
    d_dev, r_dev = engine.lstsq_decompose(torch.tensor(a32, device="cuda"), cfg)
    od = ref.lstsq_decompose(a32.astype(np.float64), 5, seed=9)
    for x, y, z in zip(d_host.factors, d_dev.factors, od.signs):
        assert (x == z).all() and (y == z).all()
    np.testing.assert_allclose(d_host.coefficients, od.alpha, rtol=1e-9, atol=1e-13)
    assert (d_host.coefficients == d_dev.coefficients).all()
    # width 0: nothing appended, the residual is the input
    d0, r0 = engine.lstsq_decompose(a, sc.DecomposeConfig(width=0))
    assert d0.width() == 0 and abs(r0.final_residual_norm - np.linalg.norm(a)) <= 1e-12 * np.linalg.norm(a)


def test_lstsq_min_value_fraction_and_budget(engine, ref):
    a = load("lsq_mat_40x33")["a"]
    cfg = sc.DecomposeConfig(width=12, min_value_fraction=0.9, search=sc.SearchConfig(seed=3))
    dec, rep = engine.lstsq_decompose(a, cfg)
    od = ref.lstsq_decompose(a, 12, seed=3, min_value_fraction=0.9)
    assert dec.width() == od.width < 12
    with pytest.raises(sc.InvalidArgument, match="factor memory budget"):
        engine.lstsq_decompose(a, sc.DecomposeConfig(width=1000, max_factor_bytes=1024))


def test_tensor_decomposition_scd_round_trip(engine, ref):
    a = ref.fill_normal(606, 6 * 7 * 5).reshape(6, 7, 5)
    dec, rep = engine.greedy_decompose(a, sc.DecomposeConfig(width=9, search=sc.SearchConfig(seed=1)), dtype="f64")
    blob = scio.write_scd(dec)
    assert blob == ref.write_scd(a.shape, dec.factors, dec.coefficients, -1, 64)
    back = scio.read_scd(blob)
    assert (bits(engine.expand(back)) == bits(ref.accumulate_expansion(a.shape, dec.factors, dec.coefficients))).all()


def test_around_edge_cases(engine, ref):
    # 1 x 1 and single-row / single-column shapes through expansion, Gram and least squares
    for shape in [(1, 1), (1, 9), (9, 1), (1,)]:
        a = ref.fill_normal(9, int(np.prod(shape))).reshape(shape) + 0.5
        dec, rep = engine.greedy_decompose(a, sc.DecomposeConfig(width=3, search=sc.SearchConfig(seed=2)), dtype="f64")
        assert (bits(engine.expand(dec)) == bits(ref.accumulate_expansion(shape, dec.factors, dec.coefficients))).all()
        g = engine.gram_matrix(dec)
        gr, _ = ref.build_gram(a, dec.factors, dec.width())
        assert (g == gr).all()
        ld, lr = engine.lstsq_decompose(a, sc.DecomposeConfig(width=2, search=sc.SearchConfig(seed=2)))
        od = ref.lstsq_decompose(a, 2, seed=2)
        assert ld.width() == od.width
        for x, y in zip(ld.factors, od.signs):
            assert (x == y).all()
    # non-finite input is rejected like the reference's DenseTensor
    bad = np.ones((4, 5))
    bad[2, 3] = np.nan
    with pytest.raises(sc.InvalidArgument, match="non-finite"):
        engine.lstsq_decompose(bad, sc.DecomposeConfig(width=1))
    # correct_coefficients: shape mismatch like the reference
    d = dec_of(load("gram_mat_37x70"))
    with pytest.raises(sc.InvalidArgument, match="shape mismatch"):
        engine.correct_coefficients(np.ones((3, 3)), d)
