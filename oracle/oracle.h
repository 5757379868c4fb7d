/*
 * oracle.h -- C interface of the CPU parity oracle.  TEST INFRASTRUCTURE ONLY.
 *
 * Two libraries implement this header:
 *   oracle/liboracle.so        (prefix orc_) -- plain-C restatement of the
 *                               reference greedy signed-cut path
 *                               (oracle/sigcut_oracle.c).
 *   oracle/_ref/libsigcut_ref.so (prefix ref_) -- the reference's own
 *                               header-only C++ library compiled unchanged from
 *                               /root/reference/proj/include by
 *                               oracle/ref_runner.cpp (Makefile recipe).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may load
 * either library.  The product (paper_2410_01799_b200/) never links them.
 *
 * Status codes: 0 ok, 1 invalid_argument, 2 runtime_error.  The message of the
 * last failure is available from <prefix>last_error().
 */
#ifndef SIGCUT_ORACLE_H
#define SIGCUT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors sigcut::DecomposeConfig + SearchConfig (inc/decompose.hpp:273-286,
 * inc/search.hpp:20-24).  method is always greedy here. */
typedef struct oracle_config {
  uint64_t width;
  uint64_t flush_width;
  uint64_t seed;
  uint64_t restarts;
  uint64_t max_sweeps;
  double min_value_fraction;
  uint64_t max_factor_bytes;
} oracle_config;

/* Caller-owned output buffers, sized for cfg.width terms.
 *   signs[axis]   : width x words(shape[axis]) u64, term-major
 *   alpha, cut_value, resid_norm (CutStep::residual_norm), iterations: width
 *   remainder     : numel doubles (R_w after the final flush) or NULL
 */
typedef struct oracle_output {
  uint64_t* signs[8];
  double* alpha;
  double* cut_value;
  double* resid_norm;
  uint64_t* iterations; /* may be NULL */
  double* remainder;    /* may be NULL */
  uint64_t width_done;
  double input_norm;
  double final_residual_norm;
} oracle_output;

#define ORACLE_DECLARE(P)                                                              \
  const char* P##last_error(void);                                                     \
  uint64_t P##mix64(uint64_t z);                                                       \
  uint64_t P##substream(uint64_t seed, uint64_t index);                                \
  void P##fill_u64(uint64_t seed, uint64_t count, uint64_t* out);                      \
  void P##fill_normal(uint64_t seed, uint64_t count, double* out);                     \
  void P##fill_f64(uint64_t seed, uint64_t count, double* out);                        \
  int P##greedy_decompose(const double* a, int order, const uint64_t* shape,           \
                          const oracle_config* cfg, oracle_output* out);               \
  /* single cut on a residual, seed used as given (greedy_signed_cut /                 \
   * axial_greedy_cut).  signs[axis] words(shape[axis]) each.  sweep_values may be     \
   * NULL; if not, receives up to max_sweeps values of the winning restart and         \
   * *n_sweep_values their count. */                                                   \
  int P##signed_cut(const double* a, int order, const uint64_t* shape, uint64_t seed,  \
                    uint64_t restarts, uint64_t max_sweeps, double* value,             \
                    uint64_t** signs, uint64_t* iterations, double* sweep_values,      \
                    uint64_t* n_sweep_values);                                         \
  uint64_t P##width_for_compression(int coeff_bits, int source_bits, int order,        \
                                    const uint64_t* shape, double rate);               \
  double P##compression_rate(uint64_t k, int coeff_bits, int source_bits, int order,   \
                             const uint64_t* shape);                                   \
  void P##quantize_bf16(uint64_t count, const double* in, double* out);                \
  /* --- around the path ---------------------------------------- */ \
  /* factors[i]: i-th SIGN axis (ascending), width x words(n) u64; coeffs: width x    \
   * channels.  data[numel] += sum_{j >= first_term} flip(scale coef, parity)        \
   * (detail::accumulate_expansion, decompose.hpp:182-197). */                        \
  int P##accumulate_expansion(int order, const uint64_t* shape, int channel_axis,      \
                              uint64_t width, const uint64_t* const* factors,          \
                              const double* coeffs, double scale, uint64_t first_term, \
                              double* data);                                           \
  /* build_gram (decompose.hpp:383-393): gram width x width, rhs width x channels */ \
  int P##build_gram(const double* a, int order, const uint64_t* shape, int channel_axis, \
                    uint64_t width, const uint64_t* const* factors, double* gram,      \
                    double* rhs);                                                      \
  /* solve_gram (gram.hpp:83-107) */                                                  \
  int P##solve_gram(uint64_t width, uint64_t channels, const double* gram,             \
                    const double* rhs, double* out);                                   \
  /* correct_coefficients (decompose.hpp:418-428) */                                  \
  int P##correct_coefficients(const double* a, int order, const uint64_t* shape,       \
                              int channel_axis, uint64_t width,                        \
                              const uint64_t* const* factors, const double* coeffs,    \
                              double* out);                                            \
  /* lstsq_decompose (channel_axis == -1, decompose.hpp:434-469) or                   \
   * rgb_scalars_decompose (:485-536): out->signs per SIGN axis, out->alpha width x   \
   * channels, resid_norm = CutStep::residual_norm. */                                \
  int P##lstsq_decompose(const double* a, int order, const uint64_t* shape,            \
                         int channel_axis, const oracle_config* cfg, oracle_output* out); \
  /* write_scd (io.hpp:142-166) into buf (capacity cap); *size = bytes */             \
  int P##write_scd(int order, const uint64_t* shape, int channel_axis, uint64_t width, \
                   const uint64_t* const* factors, const double* coeffs, int coeff_bits, \
                   uint8_t* buf, uint64_t cap, uint64_t* size);                        \
  /* read_scd (io.hpp:168-213): header fields, then factors / coeffs if non-NULL */   \
  int P##read_scd(const uint8_t* buf, uint64_t size, int* order, uint64_t* shape,      \
                  int* channel_axis, uint64_t* width, uint64_t** factors, double* coeffs); \
  /* write_raw / read_raw (io.hpp:226-292) */                                         \
  int P##write_raw(int order, const uint64_t* shape, const double* data, int dtype,    \
                   uint8_t* buf, uint64_t cap, uint64_t* size);                        \
  int P##read_raw(const uint8_t* buf, uint64_t size, int* order, uint64_t* shape,      \
                  double* data);

ORACLE_DECLARE(orc_)
ORACLE_DECLARE(ref_)

/* Reference-only checkers of the PPM / CSV helpers (io.hpp:294-396): the product's
 * byte formats are compared with the reference's own streams (no restatement). */
int ref_write_ppm(uint64_t height, uint64_t width, const double* data, uint8_t* buf, uint64_t cap, uint64_t* size);
int ref_read_ppm(const uint8_t* buf, uint64_t size, uint64_t* height, uint64_t* width, double* data);
int ref_write_curve_csv(uint64_t n, const uint64_t* widths, const double* rates, const double* errors, char* buf,
                        uint64_t cap, uint64_t* size);
int ref_read_curve_csv(const char* buf, uint64_t size, uint64_t* n, uint64_t* widths, double* rates,
                       double* errors);

#ifdef __cplusplus
}
#endif

#endif /* SIGCUT_ORACLE_H */
