"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the
reference headers compiled unchanged).  Run here, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

The fixtures are small and committed; the GPU box never needs the reference.
Inputs are Xoshiro256pp streams (inc/rng.hpp) so they are stored by seed and
also verbatim for the small cases.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.pyoracle import Oracle  # noqa: E402

ref = Oracle("ref")


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)


# ---- RNG streams (inc/rng.hpp) ----
seeds = np.array([0, 1, 2, 3, 4, 5, 0x5CD15EED, 2**63 + 11], dtype=np.uint64)
save("rng",
     seeds=seeds,
     u64=np.stack([ref.fill_u64(int(s), 16) for s in seeds]),
     normal=np.stack([ref.fill_normal(int(s), 17) for s in seeds]),
     f64=np.stack([ref.fill_f64(int(s), 8) for s in seeds]),
     substream=np.array([[ref.substream(int(s), i) for i in range(6)] for s in seeds], dtype=np.uint64),
     mix64=np.array([ref.mix64(int(s)) for s in seeds], dtype=np.uint64))

# ---- metrics: Table 2 widths and bf16 rounding ----
shapes = [(1024, 4096), (4096, 4096), (14336, 4096), (4096, 14336), (32000, 4096)]
rates = [0.5, 0.45, 0.4, 0.35, 0.3, 0.25]
widths = np.array([[ref.width_for_compression(s, r, 32, 16) for r in rates] for s in shapes], dtype=np.int64)
xq = np.concatenate([ref.fill_normal(9, 64) * 3.0, [0.0, -0.0, 1e-40, 3.3895313892515355e38, 1e39, -1e39]])
save("metrics", shapes=np.array(shapes), rates=np.array(rates), widths=widths, bf16_in=xq, bf16_out=ref.quantize_bf16(xq))


# ---- single cuts (greedy_signed_cut / axial_greedy_cut) ----
def cut_case(name, a, seed, restarts=1, max_sweeps=100):
    r = ref.signed_cut(a, seed=seed, restarts=restarts, max_sweeps=max_sweeps)
    d = dict(a=np.asarray(a, np.float64), seed=np.uint64(seed), restarts=restarts, max_sweeps=max_sweeps,
             value=r["value"], iterations=r["iterations"], sweep_values=r["sweep_values"])
    for i, s in enumerate(r["signs"]):
        d[f"signs{i}"] = s
    return name, d


cuts = []
w = ref.fill_u64(5, 2)  # random_sign_vector(Xoshiro256pp(5), 5), then (.., 7)
s5 = np.array([-1.0 if (int(w[0]) >> i) & 1 else 1.0 for i in range(5)])
t7 = np.array([-1.0 if (int(w[1]) >> i) & 1 else 1.0 for i in range(7)])
cuts.append(cut_case("rank1_5x7", np.outer(s5, t7), 42))                            # test_search.cpp:46-59
cuts.append(cut_case("alt_2x2", np.array([[1.0, -1.0], [-1.0, 1.0]]), 3, restarts=8))  # :61-68
cuts.append(cut_case("ones_3x3", np.ones((3, 3)), 1))                                 # :70-73
cuts.append(cut_case("ones_2x2x2", np.ones((2, 2, 2)), 9))                            # :90-99
cuts.append(cut_case("order1", np.array([1.5, -2.0, 0.25, -0.5]), 3))                 # :128-136
cuts.append(cut_case("rand_9x6_r3", ref.fill_f64(77, 54).reshape(9, 6) * 2 - 1, 123, restarts=3))
cuts.append(cut_case("rand_15x11_cap", ref.fill_f64(300, 165).reshape(15, 11) * 2 - 1, 987, restarts=5, max_sweeps=2))
for name, d in cuts:
    save("cut_" + name, **d)


# ---- whole greedy decompositions (greedy_decompose) ----
def dec_case(name, a, width, seed, flush=32, restarts=1, max_sweeps=100, mvf=0.0, store_input=True):
    d = ref.greedy_decompose(a, width, seed=seed, flush_width=flush, restarts=restarts, max_sweeps=max_sweeps,
                             min_value_fraction=mvf, want_remainder=a.size <= 20000)
    out = dict(shape=np.array(a.shape), width=width, seed=np.uint64(seed), flush=flush, restarts=restarts,
               max_sweeps=max_sweeps, mvf=mvf, alpha=d.alpha, cut_value=d.cut_value, resid_norm=d.resid_norm,
               iterations=d.iterations, input_norm=d.input_norm, final_residual_norm=d.final_residual_norm,
               width_done=d.width)
    for i, s in enumerate(d.signs):
        out[f"signs{i}"] = s
    if store_input:
        out["a"] = np.asarray(a, np.float64)
    if d.remainder is not None:
        out["remainder"] = d.remainder
    save("dec_" + name, **out)


sv = ref.fill_u64(12, 2)
s4 = np.array([-1.0 if (int(sv[0]) >> i) & 1 else 1.0 for i in range(4)])
t4 = np.array([-1.0 if (int(sv[1]) >> i) & 1 else 1.0 for i in range(4)])
dec_case("rank1x3_4x4", 3.0 * np.outer(s4, t4), 1, 0)                                 # test_decompose.cpp:63-77
dec_case("twoI_2x2", np.array([[2.0, 0.0], [0.0, 2.0]]), 2, 5, restarts=8)            # :79-101
for n in (8, 13, 16):                                                                  # :103-122
    dec_case(f"pyth_{n}", ref.fill_normal(2000 + n, n * n).reshape(n, n), 20, 0, flush=7)
dec_case("flush1_16", ref.fill_normal(2600, 256).reshape(16, 16), 20, 0, flush=1)      # :154-166
sv = ref.fill_u64(4300, 2)
s6 = np.array([-1.0 if (int(sv[0]) >> i) & 1 else 1.0 for i in range(6)])
t6 = np.array([-1.0 if (int(sv[1]) >> i) & 1 else 1.0 for i in range(6)])
dec_case("mvf_6x6", 2.0 * np.outer(s6, t6), 5, 0, mvf=0.5)                            # :344-357
dec_case("rect_37x29_r2", ref.fill_normal(3, 37 * 29).reshape(37, 29), 30, 3, flush=1, restarts=2)
dec_case("rect_64x100", ref.fill_normal(4, 6400).reshape(64, 100), 40, 4, flush=1)
dec_case("rect_200x150", ref.fill_normal(8, 30000).reshape(200, 150), 64, 8, flush=1, store_input=False)
dec_case("tall_300x7", ref.fill_normal(21, 2100).reshape(300, 7), 12, 21, flush=1, store_input=False)
dec_case("cap2_40x33", ref.fill_normal(22, 40 * 33).reshape(40, 33), 10, 22, flush=1, max_sweeps=2)
a32 = ref.fill_normal(0, 256 * 256).reshape(256, 256).astype(np.float32).astype(np.float64)
dec_case("f32in_256_w64", a32, 64, 0, flush=32, store_input=False)
dec_case("order3_4x5x3", ref.fill_normal(404, 60).reshape(4, 5, 3), 12, 0, flush=4)    # :124-140


# ---- around the path: expansion, Gram, least squares, SCD/DTEN ----
def rand_factors(seed, shape, channel_axis, width):
    axes = [i for i in range(len(shape)) if i != channel_axis]
    fs = []
    for k, i in enumerate(axes):
        n = shape[i]
        nw = (n + 63) // 64
        f = ref.fill_u64(seed * 100 + k, max(width * nw, 1))[: width * nw].reshape(width, nw)
        if n % 64:
            f[:, -1] &= np.uint64((1 << (n % 64)) - 1)
        fs.append(f)
    q = shape[channel_axis] if channel_axis >= 0 else 1
    co = ref.fill_normal(seed * 100 + 50, max(width * q, 1))[: width * q].reshape(width, q)
    return fs, (co if channel_axis >= 0 else co[:, 0])


def fac_dict(fs, co, shape, ch):
    d = dict(shape=np.array(shape), channel_axis=ch, coeffs=co)
    for i, f in enumerate(fs):
        d[f"fac{i}"] = f
    return d


scd_cases = [("sample_4x4", (4, 4), -1, 16), ("order3_5x7x3", (5, 7, 3), -1, 9), ("rgb_6x10x3", (6, 10, 3), 2, 5),
             ("chw_3x9x8", (3, 9, 8), 0, 4), ("vec_130", (130,), -1, 3), ("empty_7x9", (7, 9), -1, 0),
             ("wide_3x200", (3, 200), -1, 7)]
for i, (name, shape, ch, w) in enumerate(scd_cases):
    fs, co = rand_factors(700 + i, shape, ch, w)
    d = fac_dict(fs, co, shape, ch)
    d["scd64"] = np.frombuffer(ref.write_scd(shape, fs, co, ch, 64), np.uint8)
    d["scd32"] = np.frombuffer(ref.write_scd(shape, fs, co, ch, 32), np.uint8)
    save("scd_" + name, **d)

exp_cases = [("mat_37x70", (37, 70), -1, 40, 1.0, 0, False), ("resid_37x70", (37, 70), -1, 40, -1.0, 5, True),
             ("order3_5x7x3", (5, 7, 3), -1, 33, 1.0, 0, True), ("rgb_6x10x3", (6, 10, 3), 2, 12, -1.0, 0, True),
             ("chw_3x9x8", (3, 9, 8), 0, 9, 1.0, 2, False), ("vec_130", (130,), -1, 70, 1.0, 0, True),
             ("wide_5x300", (5, 300), -1, 64, 1.0, 0, False), ("tall_150x3", (150, 3), -1, 31, -1.0, 0, True),
             ("manych_6x20", (6, 20), 1, 40, -1.0, 3, True), ("manych_rows_12x9", (12, 9), 0, 33, 1.0, 0, True)]
for i, (name, shape, ch, w, scale, first, base) in enumerate(exp_cases):
    fs, co = rand_factors(800 + i, shape, ch, w)
    d = fac_dict(fs, co, shape, ch)
    a = ref.fill_normal(900 + i, int(np.prod(shape))).reshape(shape) if base else np.zeros(shape)
    d.update(base=a, scale=scale, first_term=first,
             out=ref.accumulate_expansion(shape, fs, co, data=a, scale=scale, first_term=first, channel_axis=ch))
    save("expand_" + name, **d)

gram_cases = [("mat_37x70", (37, 70), -1, 20), ("rgb_6x10x3", (6, 10, 3), 2, 9), ("order3_5x7x3", (5, 7, 3), -1, 11)]
for i, (name, shape, ch, w) in enumerate(gram_cases):
    fs, co = rand_factors(1000 + i, shape, ch, w)
    d = fac_dict(fs, co, shape, ch)
    a = ref.fill_normal(1100 + i, int(np.prod(shape))).reshape(shape)
    g, r = ref.build_gram(a, fs, w, ch)
    d.update(a=a, gram=g, rhs=r, corrected=ref.correct_coefficients(a, fs, co, ch))
    save("gram_" + name, **d)

lsq_cases = [("mat_24x20", (24, 20), -1, 6, 7), ("mat_40x33", (40, 33), -1, 12, 3), ("rgb_12x10x3", (12, 10, 3), 2, 5, 2),
             ("order3_5x6x4", (5, 6, 4), -1, 5, 11), ("chw_3x8x7", (3, 8, 7), 0, 4, 5)]
for i, (name, shape, ch, w, seed) in enumerate(lsq_cases):
    a = ref.fill_normal(1200 + i, int(np.prod(shape))).reshape(shape)
    r = ref.lstsq_decompose(a, w, seed=seed, channel_axis=ch)
    d = dict(a=a, shape=np.array(shape), channel_axis=ch, width=w, seed=np.uint64(seed), alpha=r.alpha,
             cut_value=r.cut_value, resid_norm=r.resid_norm, input_norm=r.input_norm,
             final_residual_norm=r.final_residual_norm, width_done=r.width)
    for k, f in enumerate(r.signs):
        d[f"signs{k}"] = f
    save("lsq_" + name, **d)

x = np.array([[0.0, -0.0, 1.5, -2.25], [1e-300, 3.4e38, 255.4, 255.6], [-7.5, 0.5, 1.5, 2.5]])
save("dten", a=x, f64=np.frombuffer(ref.write_raw(x, 0), np.uint8), f32=np.frombuffer(ref.write_raw(x, 1), np.uint8),
     u8=np.frombuffer(ref.write_raw(x, 2), np.uint8))
print("golden fixtures written to", HERE)
