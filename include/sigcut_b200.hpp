// sigcut_b200.hpp -- C++ drop-in over the C ABI (sigcut_b200.h) for code built
// against the reference library (proj/include/sigcut/, header-only C++20).
//
// A maintainer switches a call site by replacing
//     auto [dec, rep] = sigcut::greedy_decompose(a, cfg);        // decompose.hpp:314-361
// with
//     auto [dec, rep] = sigcut::b200::greedy_decompose(a, cfg);  // same types, same errors
// and links libsigcut_b200.so.  The result types are the reference's own
// (CutDecomposition decompose.hpp:30-100, CutReport metrics.hpp:92-97,
// CutResult search.hpp:28-32); status codes map back onto the reference's
// exceptions (std::invalid_argument / std::runtime_error).
//
// Include after <sigcut/sigcut.hpp>.  No CPU fallback: without a usable sm_100
// device the Engine constructor throws std::runtime_error.
#ifndef SIGCUT_B200_HPP
#define SIGCUT_B200_HPP

#include <sigcut/sigcut.hpp>

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sigcut_b200.h"

namespace sigcut::b200 {

/// Storage / streaming type of the device remainder.  kF64 reproduces the
/// reference arithmetic (f64 DenseTensor); kF32 keeps R in f32 (half the HBM
/// traffic) with f64 accumulation of every product.
enum class DType : std::int32_t { kF32 = SC_F32, kF64 = SC_F64 };

namespace detail {
[[noreturn]] inline void raise(sc_status st, const std::string& msg) {
  if (st == SC_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);  // SC_RUNTIME_ERROR, SC_CUDA_ERROR, SC_NOT_SUPPORTED
}
}  // namespace detail

/// One device context (sc_create / sc_destroy).  Calls on one Engine are
/// serialised by the caller; distinct Engines are independent.
class Engine {
 public:
  explicit Engine(int device = 0) {
    sc_ctx* c = nullptr;
    const sc_status st = sc_create(&c, device);
    if (st != SC_OK) detail::raise(st, "sigcut_b200: no usable sm_100 device " + std::to_string(device));
    ctx_.reset(c);
  }
  sc_ctx* get() const noexcept { return ctx_.get(); }
  void check(sc_status st) const {
    if (st != SC_OK) detail::raise(st, sc_last_error(ctx_.get()));
  }

  static Engine& default_engine() {
    static Engine e(0);
    return e;
  }

 private:
  struct Del {
    void operator()(sc_ctx* c) const noexcept { sc_destroy(c); }
  };
  std::unique_ptr<sc_ctx, Del> ctx_;
};

struct RunOutput {
  std::pair<CutDecomposition, CutReport> result;
  std::vector<std::uint32_t> sweeps;       // CutResult::iterations per term
  std::vector<double> resid_norm_exact;    // device-exact ||R_k||_F per term
  DenseTensor remainder;                   // R_w when requested (else empty)
  double kernel_ms = 0.0;
};

/// Greedy width-w decomposition on the device; fills the reference's result
/// types exactly as sigcut::greedy_decompose does (decompose.hpp:314-361).
inline RunOutput run(const DenseTensor& a, const DecomposeConfig& cfg, DType dtype, Engine& eng,
                     bool want_remainder, sc_seed_mode seed_mode = SC_SEED_PER_TERM) {
  if (cfg.method != DecomposeConfig::Method::kGreedy)
    throw std::invalid_argument("sigcut_b200: only the greedy method runs on the device");
  const std::vector<std::size_t>& shape = a.shape();
  std::vector<std::uint64_t> shp(shape.begin(), shape.end());
  std::vector<float> a32;
  sc_problem p{};
  p.dtype = static_cast<std::int32_t>(dtype);
  p.order = static_cast<std::int32_t>(shape.size());
  p.shape = shp.data();
  if (dtype == DType::kF32) {
    a32.assign(a.data().begin(), a.data().end());  // same rounding as the DTEN f32 path
    p.data = a32.data();
  } else {
    p.data = a.data().data();
  }
  p.data_on_device = 0;
  p.seed_mode = seed_mode;
  p.width = cfg.width;
  p.flush_width = cfg.flush_width;
  p.seed = cfg.search.seed;
  p.restarts = cfg.search.restarts;
  p.max_sweeps = cfg.search.max_sweeps;
  p.min_value_fraction = cfg.min_value_fraction;
  p.max_factor_bytes = cfg.max_factor_bytes;

  char msg[256];
  const sc_status vst = sc_validate_problem(&p, msg, sizeof msg);
  if (vst != SC_OK) detail::raise(vst, msg);

  const std::size_t w = cfg.width;
  sc_result r{};
  std::vector<std::vector<std::uint64_t>> words(shape.size());
  for (std::size_t ax = 0; ax < shape.size(); ++ax) {
    words[ax].assign(w * SignVector::word_count(shape[ax]), 0);
    r.sign_words[ax] = words[ax].data();
  }
  std::vector<double> alpha(w), cut(w), rn(w), rne(w);
  std::vector<std::uint32_t> sweeps(w);
  std::vector<double> rem64;
  std::vector<float> rem32;
  r.alpha = alpha.data();
  r.cut_value = cut.data();
  r.resid_norm = rn.data();
  r.resid_norm_exact = rne.data();
  r.sweeps = sweeps.data();
  if (want_remainder) {
    if (dtype == DType::kF32) {
      rem32.resize(a.numel());
      r.remainder = rem32.data();
    } else {
      rem64.resize(a.numel());
      r.remainder = rem64.data();
    }
  }
  eng.check(sc_greedy_decompose(eng.get(), &p, &r));

  RunOutput out;
  CutDecomposition d = CutDecomposition::with_shape(shape);
  CutReport rep;
  rep.input_norm = r.input_norm;
  const StorageModel model{64, 64, shape, -1};
  for (std::size_t k = 0; k < r.width_done; ++k) {
    std::vector<SignVector> signs;
    for (std::size_t ax = 0; ax < shape.size(); ++ax) {
      const std::size_t nw = SignVector::word_count(shape[ax]);
      signs.push_back(SignVector::from_words(
          shape[ax], std::vector<std::uint64_t>(words[ax].begin() + k * nw, words[ax].begin() + (k + 1) * nw)));
    }
    d.append_term(signs, std::span<const double>(&alpha[k], 1));
    if (cfg.record_curve) rep.steps.push_back(CutStep{k + 1, cut[k], rn[k], compression_rate(k + 1, model)});
  }
  rep.width = d.width();
  rep.final_residual_norm = r.final_residual_norm;
  out.sweeps.assign(sweeps.begin(), sweeps.begin() + r.width_done);
  out.resid_norm_exact.assign(rne.begin(), rne.begin() + r.width_done);
  if (want_remainder) {
    std::vector<double> v = dtype == DType::kF32 ? std::vector<double>(rem32.begin(), rem32.end()) : rem64;
    out.remainder = DenseTensor::from_raw(shape, std::move(v));
  }
  out.kernel_ms = r.kernel_ms;
  out.result = {std::move(d), std::move(rep)};
  return out;
}

/// Drop-in for sigcut::greedy_decompose (decompose.hpp:314-361).
inline std::pair<CutDecomposition, CutReport> greedy_decompose(const DenseTensor& a, const DecomposeConfig& cfg,
                                                               DType dtype = DType::kF64,
                                                               Engine& eng = Engine::default_engine()) {
  return run(a, cfg, dtype, eng, false).result;
}

/// Drop-in for sigcut::decompose (decompose.hpp:472-476), greedy method.
inline std::pair<CutDecomposition, CutReport> decompose(const DenseTensor& a, const DecomposeConfig& cfg,
                                                        DType dtype = DType::kF64,
                                                        Engine& eng = Engine::default_engine()) {
  return greedy_decompose(a, cfg, dtype, eng);
}

/// Drop-in for sigcut::greedy_signed_cut / axial_greedy_cut (search.hpp:259-272):
/// one cut searched with `cfg.seed` itself (restart r uses substream(seed, r)).
inline CutResult greedy_signed_cut(const DenseTensor& a, const SearchConfig& cfg = {}, DType dtype = DType::kF64,
                                   Engine& eng = Engine::default_engine()) {
  DecomposeConfig dc;
  dc.width = 1;
  dc.search = cfg;
  dc.record_curve = true;
  RunOutput o = run(a, dc, dtype, eng, false, SC_SEED_DIRECT);
  CutResult res;
  const CutDecomposition& d = o.result.first;
  for (const SignMatrix& f : d.factors) res.signs.push_back(f.column(0));
  res.value = o.result.second.steps.empty() ? 0.0 : o.result.second.steps[0].cut_value;
  res.iterations = o.sweeps.empty() ? 0 : o.sweeps[0];
  return res;
}

}  // namespace sigcut::b200

#endif  // SIGCUT_B200_HPP
