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
#include <istream>
#include <iterator>
#include <ostream>
#include <memory>
#include <optional>
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
  if (st == SC_IO_ERROR) throw io_error(msg);
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

namespace detail {
/// One decomposition call's C-ABI problem and caller-owned output buffers, and the
/// conversion of the outputs to the reference's result types.
struct Call {
  std::vector<std::size_t> shape;
  std::vector<std::uint64_t> shp;
  std::vector<float> a32;
  sc_problem p{};
  sc_result r{};
  std::size_t w = 0;
  bool record_curve = true, want_remainder = false;
  DType dtype = DType::kF64;
  std::vector<std::vector<std::uint64_t>> words;
  std::vector<double> alpha, cut, rn, rne, rem64, sv;
  std::vector<float> rem32;
  std::vector<std::uint32_t> sweeps;

  Call(const DenseTensor& a, const DecomposeConfig& cfg, DType dt, bool want_rem, sc_seed_mode seed_mode,
       bool want_diag)
      : shape(a.shape()), shp(shape.begin(), shape.end()), w(cfg.width), record_curve(cfg.record_curve),
        want_remainder(want_rem), dtype(dt) {
    if (cfg.method != DecomposeConfig::Method::kGreedy)
      throw std::invalid_argument("sigcut_b200: only the greedy method runs on the device");
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
    if (vst != SC_OK) raise(vst, msg);
    words.resize(shape.size());
    for (std::size_t ax = 0; ax < shape.size(); ++ax) {
      words[ax].assign(w * SignVector::word_count(shape[ax]), 0);
      r.sign_words[ax] = words[ax].data();
    }
    alpha.assign(w, 0.0);
    cut.assign(w, 0.0);
    rn.assign(w, 0.0);
    rne.assign(w, 0.0);
    sweeps.assign(w, 0);
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
    if (want_diag) {
      sv.assign(std::max<std::size_t>(cfg.search.max_sweeps, 1), 0.0);
      r.sweep_values = sv.data();
    }
  }

  RunOutput finish(SearchDiagnostics* diag) {
    if (diag != nullptr) {  // SearchDiagnostics (search.hpp:37-40); no CPU delta cache to check
      diag->sweep_values.assign(sv.begin(), sv.begin() + static_cast<std::ptrdiff_t>(r.n_sweep_values));
      diag->max_cache_rel_error = 0.0;
    }
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
      if (record_curve) rep.steps.push_back(CutStep{k + 1, cut[k], rn[k], compression_rate(k + 1, model)});
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
};
}  // namespace detail

/// Greedy width-w decomposition on the device; fills the reference's result
/// types exactly as sigcut::greedy_decompose does (decompose.hpp:314-361).
inline RunOutput run(const DenseTensor& a, const DecomposeConfig& cfg, DType dtype, Engine& eng,
                     bool want_remainder, sc_seed_mode seed_mode = SC_SEED_PER_TERM,
                     SearchDiagnostics* diag = nullptr) {
  detail::Call c(a, cfg, dtype, want_remainder, seed_mode, diag != nullptr);
  eng.check(sc_greedy_decompose(eng.get(), &c.p, &c.r));
  return c.finish(diag);
}

/// A batch of independent decompositions over several devices:
/// longest-processing-time-first assignment (cost width x numel), one host thread
/// and one context per device, no data-path communication.  Each result equals
/// the single-device greedy_decompose of that input.  The reference's contract
/// for this is "concurrent calls on distinct inputs are safe".
inline std::vector<std::pair<CutDecomposition, CutReport>> batch_decompose(
    const std::vector<DenseTensor>& inputs, const std::vector<DecomposeConfig>& cfgs, DType dtype = DType::kF64,
    const std::vector<int>& devices = {0}) {
  if (inputs.size() != cfgs.size()) throw std::invalid_argument("batch_decompose: inputs and configs differ in count");
  std::vector<std::unique_ptr<detail::Call>> calls;
  std::vector<sc_batch_job> jobs(inputs.size());
  for (std::size_t i = 0; i < inputs.size(); ++i) {
    calls.push_back(std::make_unique<detail::Call>(inputs[i], cfgs[i], dtype, false, SC_SEED_PER_TERM, false));
    jobs[i].problem = calls[i]->p;
    jobs[i].result = &calls[i]->r;
  }
  std::vector<std::int32_t> devs(devices.begin(), devices.end());
  char msg[512];
  const sc_status st = sc_batch_decompose(devs.data(), static_cast<std::int32_t>(devs.size()), jobs.data(),
                                          jobs.size(), msg, sizeof msg);
  if (st != SC_OK) detail::raise(st, msg);
  std::vector<std::pair<CutDecomposition, CutReport>> out;
  for (auto& c : calls) out.push_back(c->finish(nullptr).result);
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
inline CutResult greedy_signed_cut(const DenseTensor& a, const SearchConfig& cfg, SearchDiagnostics* diag,
                                   DType dtype = DType::kF64, Engine& eng = Engine::default_engine()) {
  DecomposeConfig dc;
  dc.width = 1;
  dc.search = cfg;
  dc.record_curve = true;
  RunOutput o = run(a, dc, dtype, eng, false, SC_SEED_DIRECT, diag);
  CutResult res;
  const CutDecomposition& d = o.result.first;
  for (const SignMatrix& f : d.factors) res.signs.push_back(f.column(0));
  res.value = o.result.second.steps.empty() ? 0.0 : o.result.second.steps[0].cut_value;
  res.iterations = o.sweeps.empty() ? 0 : o.sweeps[0];
  return res;
}

inline CutResult greedy_signed_cut(const DenseTensor& a, const SearchConfig& cfg = {}, DType dtype = DType::kF64,
                                   Engine& eng = Engine::default_engine()) {
  return greedy_signed_cut(a, cfg, nullptr, dtype, eng);
}

// ---------------------------------------------------------------------------
// Around the path: reconstruction, least squares, containers.
// ---------------------------------------------------------------------------
namespace detail {

/// Flat views of a CutDecomposition for the C ABI (sc_factors).
struct FactorView {
  std::vector<std::uint64_t> shape;
  std::vector<std::vector<std::uint64_t>> words;  // per sign axis, term-major
  sc_factors f{};

  explicit FactorView(const CutDecomposition& d) : shape(d.shape.begin(), d.shape.end()) {
    const std::size_t w = d.width();
    for (const SignMatrix& m : d.factors) {
      const std::size_t nw = SignVector::word_count(m.rows());
      std::vector<std::uint64_t> v(w * nw);
      for (std::size_t j = 0; j < w; ++j) {
        const auto cw = m.column(j).words();
        std::copy(cw.begin(), cw.end(), v.begin() + j * nw);
      }
      words.push_back(std::move(v));
    }
    f.order = static_cast<std::int32_t>(shape.size());
    f.shape = shape.data();
    f.channel_axis = d.channel_axis;
    f.width = w;
    for (std::size_t i = 0; i < words.size(); ++i) f.sign_words[i] = words[i].data();
    f.coefficients = d.coefficients.data();
  }
};

inline CutDecomposition from_words(const std::vector<std::size_t>& shape, int channel_axis, std::size_t width,
                                   const std::vector<std::vector<std::uint64_t>>& words,
                                   const std::vector<double>& coefficients) {
  CutDecomposition d = CutDecomposition::with_shape(shape, channel_axis);
  const auto axes = d.sign_axes();
  for (std::size_t j = 0; j < width; ++j) {
    std::vector<SignVector> signs;
    for (std::size_t i = 0; i < axes.size(); ++i) {
      const std::size_t n = shape[axes[i]], nw = SignVector::word_count(n);
      signs.push_back(SignVector::from_words(
          n, std::vector<std::uint64_t>(words[i].begin() + j * nw, words[i].begin() + (j + 1) * nw)));
    }
    d.append_term(signs, std::span<const double>(coefficients.data() + j * d.channels(), d.channels()));
  }
  return d;
}

}  // namespace detail

/// Drop-in for sigcut::expand (decompose.hpp:266-270): bit-identical, on the device.
inline DenseTensor expand(const CutDecomposition& d, Engine& eng = Engine::default_engine()) {
  detail::FactorView v(d);
  std::vector<double> out(DenseTensor::checked_numel(d.shape));
  eng.check(sc_accumulate_expansion(eng.get(), &v.f, 1.0, 0, d.width(), out.data(), 0, 1, nullptr));
  return DenseTensor::from_raw(d.shape, std::move(out));
}

/// Drop-in for detail::accumulate_expansion (decompose.hpp:182-197).
inline void accumulate_expansion(DenseTensor& out, const CutDecomposition& d, double scale,
                                 std::size_t first_term = 0, Engine& eng = Engine::default_engine()) {
  detail::FactorView v(d);
  eng.check(sc_accumulate_expansion(eng.get(), &v.f, scale, first_term, d.width(), out.data().data(), 0, 0, nullptr));
}

/// Drop-in for sigcut::correct_coefficients (decompose.hpp:418-428).
inline CutDecomposition correct_coefficients(const DenseTensor& a, const CutDecomposition& d,
                                             Engine& eng = Engine::default_engine()) {
  if (a.shape() != d.shape) throw std::invalid_argument("correct_coefficients: shape mismatch");
  if (d.width() == 0) return d;
  detail::FactorView v(d);
  CutDecomposition out = d;
  eng.check(sc_correct_coefficients(eng.get(), &v.f, SC_F64, a.data().data(), 0, out.coefficients.data(), nullptr));
  return out;
}

namespace detail {
inline std::pair<CutDecomposition, CutReport> lstsq_run(const DenseTensor& a, const DecomposeConfig& cfg,
                                                        int channel_axis, Engine& eng) {
  std::vector<std::uint64_t> shp(a.shape().begin(), a.shape().end());
  sc_problem p{};
  p.dtype = SC_F64;
  p.order = static_cast<std::int32_t>(shp.size());
  p.shape = shp.data();
  p.data = a.data().data();
  p.seed_mode = SC_SEED_PER_TERM;
  p.width = cfg.width;
  p.flush_width = cfg.flush_width;
  p.seed = cfg.search.seed;
  p.restarts = cfg.search.restarts;
  p.max_sweeps = cfg.search.max_sweeps;
  p.min_value_fraction = cfg.min_value_fraction;
  p.max_factor_bytes = cfg.max_factor_bytes;
  const std::size_t w = cfg.width, k = shp.size();
  const std::size_t q = channel_axis >= 0 && static_cast<std::size_t>(channel_axis) < k ? shp[channel_axis] : 1;
  sc_result r{};
  std::vector<std::vector<std::uint64_t>> words;
  for (std::size_t i = 0; i < k; ++i)
    if (static_cast<int>(i) != channel_axis) words.emplace_back(std::max<std::size_t>(w, 1) * SignVector::word_count(shp[i]));
  for (std::size_t i = 0; i < words.size(); ++i) r.sign_words[i] = words[i].data();
  std::vector<double> alpha(std::max<std::size_t>(w, 1) * q), cut(std::max<std::size_t>(w, 1)), rn(cut.size());
  r.alpha = alpha.data();
  r.cut_value = cut.data();
  r.resid_norm = rn.data();
  eng.check(sc_lstsq_decompose(eng.get(), &p, channel_axis, &r));
  const std::size_t wd = r.width_done;
  alpha.resize(wd * q);
  CutDecomposition d = from_words(a.shape(), channel_axis, wd, words, alpha);
  CutReport rep;
  rep.input_norm = r.input_norm;
  rep.final_residual_norm = r.final_residual_norm;
  const StorageModel model{64, 64, a.shape(), channel_axis};
  if (cfg.record_curve)
    for (std::size_t j = 0; j < wd; ++j) rep.steps.push_back(CutStep{j + 1, cut[j], rn[j], compression_rate(j + 1, model)});
  rep.width = wd;
  return {std::move(d), std::move(rep)};
}
}  // namespace detail

/// Drop-in for sigcut::lstsq_decompose (decompose.hpp:434-469).
inline std::pair<CutDecomposition, CutReport> lstsq_decompose(const DenseTensor& a, const DecomposeConfig& cfg,
                                                              Engine& eng = Engine::default_engine()) {
  return detail::lstsq_run(a, cfg, -1, eng);
}

/// Drop-in for sigcut::rgb_scalars_decompose (decompose.hpp:485-536).
inline std::pair<CutDecomposition, CutReport> rgb_scalars_decompose(const DenseTensor& a, const DecomposeConfig& cfg,
                                                                    std::optional<std::size_t> channel_axis = {},
                                                                    Engine& eng = Engine::default_engine()) {
  if (a.order() < 2) throw std::invalid_argument("rgb_scalars_decompose: order >= 2 required");
  return detail::lstsq_run(a, cfg, static_cast<int>(channel_axis.value_or(a.order() - 1)), eng);
}

/// Drop-in for sigcut::write_scd (io.hpp:142-166): byte-identical stream.
inline void write_scd(std::ostream& os, const CutDecomposition& d, int coeff_bits = 64) {
  detail::FactorView v(d);
  std::vector<std::uint8_t> buf(sc_scd_size(&v.f, coeff_bits) + 1);
  std::uint64_t n = 0;
  char msg[256];
  const sc_status st = sc_write_scd(&v.f, coeff_bits, buf.data(), buf.size(), &n, msg, sizeof msg);
  if (st != SC_OK) detail::raise(st, msg);
  os.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(n));
  if (!os) throw io_error("write failed");
}

/// Drop-in for sigcut::read_scd (io.hpp:168-213) over the rest of the stream.
inline CutDecomposition read_scd(std::istream& is) {
  const std::string bytes((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
  const auto* p = reinterpret_cast<const std::uint8_t*>(bytes.data());
  std::int32_t order = 0, chax = -1, cbits = 0;
  std::uint64_t shape[SC_MAX_ORDER] = {}, width = 0;
  char msg[256];
  sc_status st = sc_read_scd_header(p, bytes.size(), &order, shape, &chax, &width, &cbits, msg, sizeof msg);
  if (st != SC_OK) detail::raise(st, msg);
  std::vector<std::size_t> shp(shape, shape + order);
  const std::size_t q = chax >= 0 ? shp[chax] : 1;
  std::size_t per_term = q * static_cast<std::size_t>(cbits) / 8;
  for (int i = 0; i < order; ++i)
    if (i != chax) per_term += (shp[i] + 7) / 8;
  if (width > 0 && per_term > 0 && width > bytes.size() / per_term + 1) throw io_error("truncated payload");
  std::vector<std::vector<std::uint64_t>> words;
  std::vector<std::uint64_t*> ptrs;
  for (int i = 0; i < order; ++i)
    if (i != chax) words.emplace_back(std::max<std::uint64_t>(width, 1) * SignVector::word_count(shp[i]));
  for (auto& w : words) ptrs.push_back(w.data());
  std::vector<double> co(std::max<std::uint64_t>(width, 1) * q);
  st = sc_read_scd(p, bytes.size(), ptrs.data(), co.data(), msg, sizeof msg);
  if (st != SC_OK) detail::raise(st, msg);
  co.resize(width * q);
  CutDecomposition d = detail::from_words(shp, chax, width, words, co);
  d.validate();
  return d;
}

}  // namespace sigcut::b200

#endif  // SIGCUT_B200_HPP
