// Integration check of include/sigcut_b200.hpp: the reference's own
// sigcut::greedy_decompose / greedy_signed_cut (headers compiled unchanged, the
// checker) against sigcut::b200::* (the device engine behind the C ABI) on the
// same DenseTensor.  Built by __graft_entry__.build() when the reference tree
// is present; run by tests/test_gpu_parity.py::test_cpp_shim_matches_reference.
#include <cmath>
#include <cstdio>
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
  std::printf(fails ? "SHIM FAILED (%d)\n" : "SHIM OK\n", fails);
  return fails ? 1 : 0;
}
