// Integration check of include/sigcut_b200.hpp: the reference's own
// sigcut::greedy_decompose / greedy_signed_cut (headers compiled unchanged, the
// checker) against sigcut::b200::* (the device engine behind the C ABI) on the
// same DenseTensor.  Built by __graft_entry__.build() when the reference tree
// is present; run by tests/test_gpu_parity.py::test_cpp_shim_matches_reference.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <stdexcept>

#include <sigcut/sigcut.hpp>

#include "sigcut_b200.hpp"

using namespace sigcut;

static DenseTensor randn(std::vector<std::size_t> shape, std::uint64_t seed) {
  std::size_t n = 1;
  for (auto d : shape) n *= d;
  Xoshiro256pp g(seed);
  std::vector<double> v(n);
  for (auto& x : v) x = g.next_normal();
  return DenseTensor(std::move(shape), std::move(v));
}

static int fails = 0;
#define CHECK(c, ...)                 \
  do {                                \
    if (!(c)) {                       \
      std::printf("FAIL: " __VA_ARGS__); \
      std::printf("\n");              \
      ++fails;                        \
    }                                 \
  } while (0)

int main() {
  b200::Engine eng(0);
  {  // decomposition, f64: bit-identical factors, coefficients to 1e-12 relative
    const DenseTensor a = randn({96, 130}, 11);
    DecomposeConfig cfg;
    cfg.width = 12;
    cfg.flush_width = 1;
    cfg.record_curve = true;
    cfg.search.seed = 5;
    auto [rd, rr] = greedy_decompose(a, cfg);
    auto [gd, gr] = b200::greedy_decompose(a, cfg, b200::DType::kF64, eng);
    CHECK(rd.width() == gd.width(), "width %zu vs %zu", rd.width(), gd.width());
    for (std::size_t i = 0; i < rd.factors.size(); ++i) CHECK(rd.factors[i] == gd.factors[i], "factor %zu differs", i);
    for (std::size_t k = 0; k < rd.coefficients.size() && k < gd.coefficients.size(); ++k)
      CHECK(std::fabs(rd.coefficients[k] - gd.coefficients[k]) <= 1e-12 * std::fabs(rd.coefficients[k]),
            "alpha %zu", k);
    CHECK(rr.steps.size() == gr.steps.size(), "curve length");
    for (std::size_t k = 0; k < rr.steps.size() && k < gr.steps.size(); ++k) {
      CHECK(rr.steps[k].k == gr.steps[k].k, "step k");
      CHECK(std::fabs(rr.steps[k].residual_norm - gr.steps[k].residual_norm) <= 1e-10 * rr.input_norm, "resid %zu", k);
      CHECK(rr.steps[k].compression == gr.steps[k].compression, "compression %zu", k);
    }
    CHECK(std::fabs(rr.input_norm - gr.input_norm) <= 1e-12 * rr.input_norm, "input norm");
    CHECK(std::fabs(rr.final_residual_norm - gr.final_residual_norm) <= 1e-10 * rr.input_norm, "final norm");
  }
  {  // single cut with the search seed used directly
    const DenseTensor a = randn({40, 33}, 3);
    SearchConfig sc;
    sc.seed = 9;
    const CutResult r = greedy_signed_cut(a, sc);
    const CutResult g = b200::greedy_signed_cut(a, sc, b200::DType::kF64, eng);
    CHECK(r.signs.size() == g.signs.size(), "axes");
    for (std::size_t i = 0; i < r.signs.size() && i < g.signs.size(); ++i)
      CHECK(r.signs[i] == g.signs[i], "cut signs axis %zu", i);
    CHECK(std::fabs(r.value - g.value) <= 1e-12 * std::fabs(r.value), "cut value %.17g vs %.17g", r.value, g.value);
    CHECK(r.iterations == g.iterations, "iterations %zu vs %zu", r.iterations, g.iterations);
    SearchDiagnostics rd, gd;
    greedy_signed_cut(a, sc, &rd);
    b200::greedy_signed_cut(a, sc, &gd, b200::DType::kF64, eng);
    CHECK(rd.sweep_values.size() == gd.sweep_values.size(), "sweep value count");
    for (std::size_t k = 0; k < rd.sweep_values.size() && k < gd.sweep_values.size(); ++k)
      CHECK(std::fabs(rd.sweep_values[k] - gd.sweep_values[k]) <= 1e-12 * std::fabs(rd.sweep_values[k]) + 1e-12,
            "sweep value %zu", k);
  }
  {  // error semantics: same exception type as the reference
    const DenseTensor a = randn({4, 4}, 1);
    DecomposeConfig bad;
    bad.width = 2;
    bad.flush_width = 0;
    bool ref_threw = false, b200_threw = false;
    try { greedy_decompose(a, bad); } catch (const std::invalid_argument&) { ref_threw = true; }
    try { b200::greedy_decompose(a, bad, b200::DType::kF64, eng); } catch (const std::invalid_argument&) { b200_threw = true; }
    CHECK(ref_threw && b200_threw, "invalid_argument mapping (%d, %d)", ref_threw, b200_threw);
  }
  {  // expansion: bit-identical DenseTensor (decompose.hpp:266-270)
    const DenseTensor a = randn({77, 150}, 21);
    DecomposeConfig cfg;
    cfg.width = 40;
    auto [rd, rr] = greedy_decompose(a, cfg);
    CHECK(expand(rd) == b200::expand(rd, eng), "expand differs");
    DenseTensor r1 = a, r2 = a;
    detail::accumulate_expansion(r1, rd, -1.0, 3);
    b200::accumulate_expansion(r2, rd, -1.0, 3, eng);
    CHECK(r1 == r2, "accumulate_expansion differs");
    // SCD: the drop-in writer emits the reference's bytes; its reader round-trips
    for (int bits : {64, 32}) {
      std::ostringstream o1(std::ios::binary), o2(std::ios::binary);
      write_scd(o1, rd, bits);
      b200::write_scd(o2, rd, bits);
      CHECK(o1.str() == o2.str(), "scd bytes (%d-bit)", bits);
      std::istringstream i1(o1.str(), std::ios::binary);
      CHECK(b200::read_scd(i1) == [&] { std::istringstream i(o1.str(), std::ios::binary); return read_scd(i); }(),
            "read_scd (%d-bit)", bits);
    }
    bool io_ref = false, io_b200 = false;
    std::string junk = "SCD1\x02";
    try { std::istringstream i(junk, std::ios::binary); read_scd(i); } catch (const io_error&) { io_ref = true; }
    try { std::istringstream i(junk, std::ios::binary); b200::read_scd(i); } catch (const io_error&) { io_b200 = true; }
    CHECK(io_ref && io_b200, "io_error mapping (%d, %d)", io_ref, io_b200);
  }
  {  // least squares and scalar channels: same signs, coefficients to 1e-9
    const DenseTensor a = randn({30, 26}, 31);
    DecomposeConfig cfg;
    cfg.width = 6;
    cfg.record_curve = true;
    cfg.search.seed = 4;
    auto [rd, rr] = lstsq_decompose(a, cfg);
    auto [gd, gr] = b200::lstsq_decompose(a, cfg, eng);
    CHECK(rd.width() == gd.width(), "lstsq width");
    for (std::size_t i = 0; i < rd.factors.size(); ++i) CHECK(rd.factors[i] == gd.factors[i], "lstsq factor %zu", i);
    for (std::size_t k = 0; k < rd.coefficients.size() && k < gd.coefficients.size(); ++k)
      CHECK(std::fabs(rd.coefficients[k] - gd.coefficients[k]) <= 1e-9 * std::fabs(rd.coefficients[k]) + 1e-13,
            "lstsq coef %zu", k);
    CHECK(std::fabs(rr.final_residual_norm - gr.final_residual_norm) <= 1e-10 * rr.input_norm, "lstsq norm");
    const DenseTensor img = randn({14, 11, 3}, 32);
    auto [rg, rgr] = rgb_scalars_decompose(img, cfg);
    auto [gg, ggr] = b200::rgb_scalars_decompose(img, cfg, {}, eng);
    CHECK(rg.channel_axis == gg.channel_axis && rg.width() == gg.width(), "rgb layout");
    for (std::size_t i = 0; i < rg.factors.size(); ++i) CHECK(rg.factors[i] == gg.factors[i], "rgb factor %zu", i);
    for (std::size_t k = 0; k < rg.coefficients.size() && k < gg.coefficients.size(); ++k)
      CHECK(std::fabs(rg.coefficients[k] - gg.coefficients[k]) <= 1e-9 * std::fabs(rg.coefficients[k]) + 1e-13,
            "rgb coef %zu", k);
    const CutDecomposition rc = correct_coefficients(a, rd);
    const CutDecomposition gc = b200::correct_coefficients(a, rd, eng);
    for (std::size_t k = 0; k < rc.coefficients.size(); ++k)
      CHECK(std::fabs(rc.coefficients[k] - gc.coefficients[k]) <= 1e-9 * std::fabs(rc.coefficients[k]) + 1e-13,
            "correct_coefficients %zu", k);
  }
  {  // batch_decompose (sc_batch_decompose, LPT over devices): every job equals the reference's
    std::vector<DenseTensor> ins;
    std::vector<DecomposeConfig> cfgs;
    const std::size_t shapes[][2] = {{40, 70}, {128, 33}, {9, 9}, {300, 64}, {64, 257}};
    for (std::size_t i = 0; i < 5; ++i) {
      ins.push_back(randn({shapes[i][0], shapes[i][1]}, 100 + i));
      DecomposeConfig c;
      c.width = 4 + i;
      c.record_curve = true;
      c.search.seed = 7 * i + 1;
      cfgs.push_back(c);
    }
    const auto out = b200::batch_decompose(ins, cfgs, b200::DType::kF64, {0});
    CHECK(out.size() == ins.size(), "batch size");
    for (std::size_t i = 0; i < out.size() && i < ins.size(); ++i) {
      auto [rd, rr] = greedy_decompose(ins[i], cfgs[i]);
      const auto& [gd, gr] = out[i];
      CHECK(rd.width() == gd.width(), "batch job %zu width", i);
      for (std::size_t f = 0; f < rd.factors.size(); ++f) CHECK(rd.factors[f] == gd.factors[f], "batch job %zu factor %zu", i, f);
      for (std::size_t k = 0; k < rd.coefficients.size() && k < gd.coefficients.size(); ++k)
        CHECK(std::fabs(rd.coefficients[k] - gd.coefficients[k]) <= 1e-10 * std::fabs(rd.coefficients[k]),
              "batch job %zu coef %zu", i, k);
    }
    bool threw = false;
    try {
      std::vector<DecomposeConfig> bad = cfgs;
      bad[2].search.restarts = 0;
      b200::batch_decompose(ins, bad, b200::DType::kF64, {0});
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw, "batch: invalid config must throw invalid_argument");
  }
  std::printf(fails ? "SHIM FAILED (%d)\n" : "SHIM OK\n", fails);
  return fails ? 1 : 0;
}
