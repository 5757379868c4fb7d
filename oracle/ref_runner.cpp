// ref_runner.cpp -- C-ABI wrapper around the REFERENCE library itself (test
// infrastructure only).  It #includes the reference's unchanged header-only
// sources from /root/reference/proj/include (nothing is copied into this repo)
// and is compiled by oracle/Makefile with the reference's Release flags
// (-std=gnu++20 -O3 -DNDEBUG, proj/CMakeLists.txt:8-10) into
// oracle/_ref/libsigcut_ref.so.  Tests use it to pin oracle/sigcut_oracle.c and
// to generate tests/golden/ fixtures; bench.py --impl reference times it.
#include <cstring>
#include <sstream>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "sigcut/sigcut.hpp"

#include "oracle.h"

namespace {
std::string g_err;

int map_exc(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const sigcut::io_error*>(&e) != nullptr) return 3;
  return dynamic_cast<const std::invalid_argument*>(&e) != nullptr ? 1 : 2;
}

// A CutDecomposition assembled from raw factor words (per sign axis) and coefficients.
sigcut::CutDecomposition make_dec(int order, const uint64_t* shape, int channel_axis, uint64_t width,
                                  const uint64_t* const* factors, const double* coeffs) {
  auto d = sigcut::CutDecomposition::with_shape(std::vector<std::size_t>(shape, shape + order), channel_axis);
  const auto axes = d.sign_axes();
  for (uint64_t j = 0; j < width; ++j) {
    std::vector<sigcut::SignVector> signs;
    for (std::size_t i = 0; i < axes.size(); ++i) {
      const std::size_t n = shape[axes[i]];
      const std::size_t nw = sigcut::SignVector::word_count(n);
      signs.push_back(sigcut::SignVector::from_words(
          n, std::vector<std::uint64_t>(factors[i] + j * nw, factors[i] + (j + 1) * nw)));
    }
    d.append_term(signs, std::span<const double>(coeffs + j * d.channels(), d.channels()));
  }
  return d;
}

void put_dec(const sigcut::CutDecomposition& d, uint64_t** factors, double* coeffs) {
  const auto axes = d.sign_axes();
  for (std::size_t i = 0; i < axes.size(); ++i) {
    const std::size_t nw = sigcut::SignVector::word_count(d.shape[axes[i]]);
    for (std::size_t j = 0; j < d.width(); ++j) {
      const auto w = d.factors[i].column(j).words();
      std::memcpy(factors[i] + j * nw, w.data(), nw * 8);
    }
  }
  std::memcpy(coeffs, d.coefficients.data(), d.coefficients.size() * 8);
}

std::vector<std::size_t> to_shape(int order, const uint64_t* shape) {
  return std::vector<std::size_t>(shape, shape + order);
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint64_t ref_mix64(uint64_t z) { return sigcut::mix64(z); }
uint64_t ref_substream(uint64_t seed, uint64_t index) { return sigcut::substream(seed, index); }

void ref_fill_u64(uint64_t seed, uint64_t count, uint64_t* out) {
  sigcut::Xoshiro256pp rng(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng.next_u64();
}

void ref_fill_normal(uint64_t seed, uint64_t count, double* out) {
  sigcut::Xoshiro256pp rng(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng.next_normal();
}

void ref_fill_f64(uint64_t seed, uint64_t count, double* out) {
  sigcut::Xoshiro256pp rng(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng.next_f64();
}

int ref_greedy_decompose(const double* a, int order, const uint64_t* shape,
                         const oracle_config* cfg, oracle_output* out) {
  try {
    const auto sh = to_shape(order, shape);
    const std::size_t numel = sigcut::DenseTensor::checked_numel(sh);
    sigcut::DenseTensor t(sh, std::vector<double>(a, a + numel));
    sigcut::DecomposeConfig dc;
    dc.width = cfg->width;
    dc.flush_width = cfg->flush_width;
    dc.search.seed = cfg->seed;
    dc.search.restarts = cfg->restarts;
    dc.search.max_sweeps = cfg->max_sweeps;
    dc.record_curve = true;
    dc.min_value_fraction = cfg->min_value_fraction;
    dc.max_factor_bytes = cfg->max_factor_bytes;
    auto [d, report] = sigcut::greedy_decompose(t, dc);
    const std::size_t w = d.width();
    for (std::size_t ax = 0; ax < d.factors.size(); ++ax) {
      const std::size_t nw = sigcut::SignVector::word_count(sh[ax]);
      for (std::size_t j = 0; j < w; ++j) {
        const auto words = d.factors[ax].column(j).words();
        std::memcpy(out->signs[ax] + j * nw, words.data(), nw * sizeof(uint64_t));
      }
    }
    for (std::size_t j = 0; j < w; ++j) {
      out->alpha[j] = d.coefficients[j];
      out->cut_value[j] = report.steps[j].cut_value;
      out->resid_norm[j] = report.steps[j].residual_norm;
    }
    out->width_done = w;
    out->input_norm = report.input_norm;
    out->final_residual_norm = report.final_residual_norm;
    if (out->iterations != nullptr || out->remainder != nullptr) {
      // The public driver does not expose per-term sweep counts or R_w; replay the
      // identical term loop (decompose.hpp:332-347) on the reference internals.
      sigcut::DenseTensor base = t;
      std::vector<sigcut::detail::PendingTerm> pending;
      std::vector<std::size_t> axes(sh.size());
      for (std::size_t i = 0; i < axes.size(); ++i) axes[i] = i;
      for (std::size_t term = 0; term < w; ++term) {
        const auto scfg = sigcut::detail::term_search_config(dc.search, term);
        sigcut::CutResult res = sigcut::detail::search_tensor_residual(base, pending, scfg, nullptr);
        if (res.value != out->cut_value[term]) throw std::runtime_error("replay diverged");
        if (out->iterations != nullptr) out->iterations[term] = res.iterations;
        pending.push_back(sigcut::detail::PendingTerm{std::move(res.signs), res.value / double(numel)});
        if (pending.size() >= dc.flush_width) sigcut::detail::flush_pending(base, pending, axes);
      }
      sigcut::detail::flush_pending(base, pending, axes);
      if (out->remainder != nullptr) std::memcpy(out->remainder, base.data().data(), numel * 8);
    }
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

int ref_signed_cut(const double* a, int order, const uint64_t* shape, uint64_t seed,
                   uint64_t restarts, uint64_t max_sweeps, double* value, uint64_t** signs,
                   uint64_t* iterations, double* sweep_values, uint64_t* n_sweep_values) {
  try {
    const auto sh = to_shape(order, shape);
    const std::size_t numel = sigcut::DenseTensor::checked_numel(sh);
    sigcut::DenseTensor t(sh, std::vector<double>(a, a + numel));
    sigcut::SearchConfig sc{seed, restarts, max_sweeps};
    sigcut::SearchDiagnostics diag;
    const sigcut::CutResult res = sigcut::axial_greedy_cut(t, sc, &diag);
    *value = res.value;
    *iterations = res.iterations;
    for (std::size_t ax = 0; ax < res.signs.size(); ++ax) {
      const auto words = res.signs[ax].words();
      std::memcpy(signs[ax], words.data(), words.size() * sizeof(uint64_t));
    }
    if (sweep_values != nullptr) {
      for (std::size_t i = 0; i < diag.sweep_values.size(); ++i) sweep_values[i] = diag.sweep_values[i];
    }
    if (n_sweep_values != nullptr) *n_sweep_values = diag.sweep_values.size();
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

uint64_t ref_width_for_compression(int coeff_bits, int source_bits, int order,
                                   const uint64_t* shape, double rate) {
  try {
    sigcut::StorageModel m{coeff_bits, source_bits, to_shape(order, shape), -1};
    return sigcut::width_for_compression(m, rate);
  } catch (const std::exception& e) {
    map_exc(e);
    return 0;
  }
}

double ref_compression_rate(uint64_t k, int coeff_bits, int source_bits, int order,
                            const uint64_t* shape) {
  sigcut::StorageModel m{coeff_bits, source_bits, to_shape(order, shape), -1};
  return sigcut::compression_rate(k, m);
}

void ref_quantize_bf16(uint64_t count, const double* in, double* out) {
  auto t = sigcut::DenseTensor::from_raw({count}, std::vector<double>(in, in + count));
  const auto q = sigcut::quantize_half(t, sigcut::HalfFormat::kBf16);
  std::memcpy(out, q.data().data(), count * sizeof(double));
}

int ref_accumulate_expansion(int order, const uint64_t* shape, int channel_axis, uint64_t width,
                             const uint64_t* const* factors, const double* coeffs, double scale,
                             uint64_t first_term, double* data) {
  try {
    const auto d = make_dec(order, shape, channel_axis, width, factors, coeffs);
    const std::size_t numel = sigcut::DenseTensor::checked_numel(d.shape);
    auto t = sigcut::DenseTensor::from_raw(d.shape, std::vector<double>(data, data + numel));
    sigcut::detail::accumulate_expansion(t, d, scale, first_term);
    std::memcpy(data, t.data().data(), numel * 8);
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

int ref_build_gram(const double* a, int order, const uint64_t* shape, int channel_axis, uint64_t width,
                   const uint64_t* const* factors, double* gram, double* rhs) {
  try {
    std::vector<double> zero(width * (channel_axis >= 0 ? shape[channel_axis] : 1), 0.0);
    const auto d = make_dec(order, shape, channel_axis, width, factors, zero.data());
    const std::size_t numel = sigcut::DenseTensor::checked_numel(d.shape);
    sigcut::DenseTensor t(d.shape, std::vector<double>(a, a + numel));
    const sigcut::GramSystem sys = sigcut::detail::build_gram(t, d);
    std::memcpy(gram, sys.gram.data(), sys.gram.size() * 8);
    std::memcpy(rhs, sys.rhs.data(), sys.rhs.size() * 8);
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

int ref_solve_gram(uint64_t width, uint64_t channels, const double* gram, const double* rhs, double* out) {
  try {
    sigcut::GramSystem sys;
    sys.width = width;
    sys.channels = channels;
    sys.gram.assign(gram, gram + width * width);
    sys.rhs.assign(rhs, rhs + width * channels);
    const auto x = sigcut::solve_gram(sys);
    std::memcpy(out, x.data(), x.size() * 8);
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

int ref_correct_coefficients(const double* a, int order, const uint64_t* shape, int channel_axis, uint64_t width,
                             const uint64_t* const* factors, const double* coeffs, double* out) {
  try {
    const auto d = make_dec(order, shape, channel_axis, width, factors, coeffs);
    const std::size_t numel = sigcut::DenseTensor::checked_numel(d.shape);
    sigcut::DenseTensor t(d.shape, std::vector<double>(a, a + numel));
    const auto c = sigcut::correct_coefficients(t, d);
    std::memcpy(out, c.coefficients.data(), c.coefficients.size() * 8);
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

int ref_lstsq_decompose(const double* a, int order, const uint64_t* shape, int channel_axis,
                        const oracle_config* cfg, oracle_output* out) {
  try {
    const auto sh = to_shape(order, shape);
    const std::size_t numel = sigcut::DenseTensor::checked_numel(sh);
    sigcut::DenseTensor t(sh, std::vector<double>(a, a + numel));
    sigcut::DecomposeConfig dc;
    dc.width = cfg->width;
    dc.flush_width = cfg->flush_width;
    dc.search.seed = cfg->seed;
    dc.search.restarts = cfg->restarts;
    dc.search.max_sweeps = cfg->max_sweeps;
    dc.record_curve = true;
    dc.min_value_fraction = cfg->min_value_fraction;
    dc.max_factor_bytes = cfg->max_factor_bytes;
    dc.method = sigcut::DecomposeConfig::Method::kLeastSquares;
    auto [d, report] = channel_axis >= 0
                           ? sigcut::rgb_scalars_decompose(t, dc, static_cast<std::size_t>(channel_axis))
                           : sigcut::decompose(t, dc);
    put_dec(d, out->signs, out->alpha);
    for (std::size_t j = 0; j < d.width(); ++j) {
      out->cut_value[j] = report.steps[j].cut_value;
      out->resid_norm[j] = report.steps[j].residual_norm;
    }
    out->width_done = d.width();
    out->input_norm = report.input_norm;
    out->final_residual_norm = report.final_residual_norm;
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

int ref_write_scd(int order, const uint64_t* shape, int channel_axis, uint64_t width, const uint64_t* const* factors,
                  const double* coeffs, int coeff_bits, uint8_t* buf, uint64_t cap, uint64_t* size) {
  try {
    const auto d = make_dec(order, shape, channel_axis, width, factors, coeffs);
    std::ostringstream os(std::ios::binary);
    sigcut::write_scd(os, d, coeff_bits);
    const std::string b = os.str();
    *size = b.size();
    if (b.size() > cap) throw std::invalid_argument("buffer too small");
    std::memcpy(buf, b.data(), b.size());
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

int ref_read_scd(const uint8_t* buf, uint64_t size, int* order, uint64_t* shape, int* channel_axis, uint64_t* width,
                 uint64_t** factors, double* coeffs) {
  try {
    std::istringstream is(std::string(reinterpret_cast<const char*>(buf), size), std::ios::binary);
    const auto d = sigcut::read_scd(is);
    *order = static_cast<int>(d.order());
    for (std::size_t i = 0; i < d.order(); ++i) shape[i] = d.shape[i];
    *channel_axis = d.channel_axis;
    *width = d.width();
    if (factors != nullptr && coeffs != nullptr) put_dec(d, factors, coeffs);
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

int ref_write_raw(int order, const uint64_t* shape, const double* data, int dtype, uint8_t* buf, uint64_t cap,
                  uint64_t* size) {
  try {
    const auto sh = to_shape(order, shape);
    const std::size_t numel = sigcut::DenseTensor::checked_numel(sh);
    auto t = sigcut::DenseTensor::from_raw(sh, std::vector<double>(data, data + numel));
    std::ostringstream os(std::ios::binary);
    sigcut::write_raw(os, t, static_cast<sigcut::RawDType>(dtype));
    const std::string b = os.str();
    *size = b.size();
    if (b.size() > cap) throw std::invalid_argument("buffer too small");
    std::memcpy(buf, b.data(), b.size());
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

int ref_read_raw(const uint8_t* buf, uint64_t size, int* order, uint64_t* shape, double* data) {
  try {
    std::istringstream is(std::string(reinterpret_cast<const char*>(buf), size), std::ios::binary);
    const auto t = sigcut::read_raw(is);
    *order = static_cast<int>(t.order());
    for (std::size_t i = 0; i < t.order(); ++i) shape[i] = t.shape()[i];
    if (data != nullptr) std::memcpy(data, t.data().data(), t.numel() * 8);
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

int ref_write_ppm(uint64_t height, uint64_t width, const double* data, uint8_t* buf, uint64_t cap, uint64_t* size) {
  try {
    auto t = sigcut::DenseTensor::from_raw({height, width, 3}, std::vector<double>(data, data + height * width * 3));
    std::ostringstream os(std::ios::binary);
    sigcut::write_ppm(os, t);
    const std::string b = os.str();
    *size = b.size();
    if (b.size() > cap) throw std::invalid_argument("buffer too small");
    std::memcpy(buf, b.data(), b.size());
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

int ref_read_ppm(const uint8_t* buf, uint64_t size, uint64_t* height, uint64_t* width, double* data) {
  try {
    std::istringstream is(std::string(reinterpret_cast<const char*>(buf), size), std::ios::binary);
    const auto t = sigcut::read_ppm(is);
    *height = t.shape()[0];
    *width = t.shape()[1];
    if (data != nullptr) std::memcpy(data, t.data().data(), t.numel() * 8);
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

int ref_write_curve_csv(uint64_t n, const uint64_t* widths, const double* rates, const double* errors, char* buf,
                        uint64_t cap, uint64_t* size) {
  try {
    std::vector<sigcut::CurvePoint> pts(n);
    for (uint64_t i = 0; i < n; ++i) pts[i] = sigcut::CurvePoint{widths[i], rates[i], errors[i]};
    std::ostringstream os;
    sigcut::write_curve_csv(os, pts);
    const std::string b = os.str();
    *size = b.size();
    if (b.size() > cap) throw std::invalid_argument("buffer too small");
    std::memcpy(buf, b.data(), b.size());
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

int ref_read_curve_csv(const char* buf, uint64_t size, uint64_t* n, uint64_t* widths, double* rates,
                       double* errors) {
  try {
    std::istringstream is(std::string(buf, size));
    const auto pts = sigcut::read_curve_csv(is);
    *n = pts.size();
    if (widths != nullptr)
      for (std::size_t i = 0; i < pts.size(); ++i) {
        widths[i] = pts[i].width;
        rates[i] = pts[i].compression_rate;
        errors[i] = pts[i].relative_error;
      }
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

}  // extern "C"
