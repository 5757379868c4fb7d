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
  void P##quantize_bf16(uint64_t count, const double* in, double* out);

ORACLE_DECLARE(orc_)
ORACLE_DECLARE(ref_)

#ifdef __cplusplus
}
#endif

#endif /* SIGCUT_ORACLE_H */
