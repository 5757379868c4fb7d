/*
 * sigcut_oracle.c -- CPU PARITY ORACLE (test infrastructure, never shipped).
 *
 * A plain-C restatement of the reference greedy signed-cut decomposition
 * (arXiv 2410.01799, reference tree /root/reference/proj/include/sigcut/).
 * Every function cites the reference file:line it follows; the arithmetic
 * order is kept identical so results are bit-for-bit equal to the reference
 * compiled with its Release flags (pinned by tests/test_oracle.py against
 * oracle/_ref/libsigcut_ref.so and tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library.  Build: oracle/Makefile  (gcc -O3 -ffp-contract=off).
 */
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

#define WORD_BITS 64u

static char g_err[256];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* orc_last_error(void) { return g_err; }

/* ---- RNG: inc/rng.hpp:10-71 ------------------------------------------- */

uint64_t orc_mix64(uint64_t z) { /* inc/rng.hpp:10-15 */
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t orc_substream(uint64_t seed, uint64_t index) { /* inc/rng.hpp:22-24 */
  return orc_mix64(seed ^ (0xd1342543de82ef95ULL * (index + 1)));
}

typedef struct {
  uint64_t s[4];
  double spare;
  int have_spare;
} xoshiro;

static void xo_seed(xoshiro* x, uint64_t seed) { /* inc/rng.hpp:30-40 */
  uint64_t sm = seed;
  for (int i = 0; i < 4; ++i) {
    sm += 0x9e3779b97f4a7c15ULL;
    uint64_t z = sm;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    x->s[i] = z ^ (z >> 31);
  }
  x->spare = 0.0;
  x->have_spare = 0;
}

static uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

static uint64_t xo_next(xoshiro* x) { /* inc/rng.hpp:42-52 */
  uint64_t* s = x->s;
  const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

static double xo_f64(xoshiro* x) { /* inc/rng.hpp:55 */
  return (double)(xo_next(x) >> 11) * 0x1.0p-53;
}

static double xo_normal(xoshiro* x) { /* inc/rng.hpp:58-71, Box-Muller cos then sin */
  if (x->have_spare) {
    x->have_spare = 0;
    return x->spare;
  }
  double u1 = xo_f64(x);
  while (u1 <= 0.0) u1 = xo_f64(x);
  const double u2 = xo_f64(x);
  const double r = sqrt(-2.0 * log(u1));
  const double two_pi = 6.283185307179586476925286766559;
  x->spare = r * sin(two_pi * u2);
  x->have_spare = 1;
  return r * cos(two_pi * u2);
}

void orc_fill_u64(uint64_t seed, uint64_t count, uint64_t* out) {
  xoshiro x;
  xo_seed(&x, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = xo_next(&x);
}

void orc_fill_normal(uint64_t seed, uint64_t count, double* out) {
  xoshiro x;
  xo_seed(&x, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = xo_normal(&x);
}

void orc_fill_f64(uint64_t seed, uint64_t count, double* out) {
  xoshiro x;
  xo_seed(&x, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = xo_f64(&x);
}

/* ---- sign vectors: inc/sign_vector.hpp -------------------------------- */

static size_t nwords(size_t len) { return (len + WORD_BITS - 1) / WORD_BITS; }

static int bit_at(const uint64_t* w, size_t i) { return (int)((w[i / WORD_BITS] >> (i % WORD_BITS)) & 1u); }

/* random_sign_vector, inc/sign_vector.hpp:130-137 */
static void random_signs(xoshiro* x, size_t n, uint64_t* w) {
  const size_t nw = nwords(n);
  for (size_t u = 0; u < nw; ++u) w[u] = xo_next(x);
  const size_t tail = n % WORD_BITS;
  if (tail != 0 && nw != 0) w[nw - 1] &= (((uint64_t)1) << tail) - 1;
}

/* sgn_vector, inc/sign_vector.hpp:107-114: x < 0 -> set bit; rejects non-finite */
static int sgn_vec(const double* x, size_t n, uint64_t* w) {
  memset(w, 0, nwords(n) * sizeof(uint64_t));
  for (size_t i = 0; i < n; ++i) {
    if (!isfinite(x[i])) return fail(1, "sgn_vector: non-finite entry");
    if (x[i] < 0.0) w[i / WORD_BITS] |= ((uint64_t)1) << (i % WORD_BITS);
  }
  return 0;
}

/* sign_dot, inc/sign_vector.hpp:118-127 */
static int64_t sign_dot(const uint64_t* a, const uint64_t* b, size_t n) {
  int64_t disagree = 0;
  for (size_t u = 0; u < nwords(n); ++u) disagree += __builtin_popcountll(a[u] ^ b[u]);
  return (int64_t)n - 2 * disagree;
}

/* ---- kernels: inc/kernels.hpp ------------------------------------------ */

/* flip_sign_if, inc/kernels.hpp:18-20 */
static double flip(double x, uint64_t neg) {
  uint64_t u;
  memcpy(&u, &x, 8);
  u ^= neg << 63;
  memcpy(&x, &u, 8);
  return x;
}

/* signed_dot, inc/kernels.hpp:24-39: 64-entry block partials summed in order */
static double signed_dot(const uint64_t* s, const double* x, size_t n) {
  double total = 0.0;
  size_t i = 0;
  for (size_t u = 0; u < nwords(n); ++u) {
    const uint64_t w = s[u];
    const size_t end = (i + WORD_BITS < n) ? i + WORD_BITS : n;
    double block = 0.0;
    for (size_t b = 0; i < end; ++i, ++b) block += flip(x[i], (w >> b) & 1u);
    total += block;
  }
  return total;
}

/* matvec_signed, inc/kernels.hpp:61-71 */
static void matvec(const double* a, size_t m, size_t n, const uint64_t* t, double* y) {
  for (size_t i = 0; i < m; ++i) y[i] = signed_dot(t, a + i * n, n);
}

/* matvec_signed_t, inc/kernels.hpp:74-88: row-by-row accumulation */
static void matvec_t(const double* a, size_t m, size_t n, const uint64_t* s, double* z) {
  for (size_t j = 0; j < n; ++j) z[j] = 0.0;
  for (size_t i = 0; i < m; ++i) {
    const uint64_t neg = (uint64_t)bit_at(s, i);
    const double* row = a + i * n;
    for (size_t j = 0; j < n; ++j) z[j] += flip(row[j], neg);
  }
}

/* delta_matvec_inplace, inc/kernels.hpp:92-115 (flipped columns, stride n) */
static void delta_matvec(const double* a, size_t m, size_t n, double* y, const uint64_t* tn,
                         const uint64_t* to) {
  for (size_t u = 0; u < nwords(n); ++u) {
    uint64_t diff = tn[u] ^ to[u];
    while (diff != 0) {
      const int b = __builtin_ctzll(diff);
      diff &= diff - 1;
      const size_t j = u * WORD_BITS + (size_t)b;
      const uint64_t neg = (tn[u] >> b) & 1u;
      for (size_t i = 0; i < m; ++i) {
        const double col = a[i * n + j];
        y[i] += flip(col + col, neg);
      }
    }
  }
}

/* delta_matvec_t_inplace, inc/kernels.hpp:126-149 (flipped rows) */
static void delta_matvec_t(const double* a, size_t m, size_t n, double* z, const uint64_t* sn,
                           const uint64_t* so) {
  for (size_t u = 0; u < nwords(m); ++u) {
    uint64_t diff = sn[u] ^ so[u];
    while (diff != 0) {
      const int b = __builtin_ctzll(diff);
      diff &= diff - 1;
      const size_t i = u * WORD_BITS + (size_t)b;
      const uint64_t neg = (sn[u] >> b) & 1u;
      const double* row = a + i * n;
      for (size_t j = 0; j < n; ++j) z[j] += flip(row[j] + row[j], neg);
    }
  }
}

/* axial_contract, inc/kernels.hpp:180-211: out[idx[axis]] += flip(a[e], XOR of the
 * other axes' sign bits), elements visited in row-major order. */
static void axial_contract(const double* a, int k, const size_t* shape, size_t numel, int axis,
                           uint64_t* const* signs, double* out) {
  size_t idx[8] = {0};
  for (size_t q = 0; q < shape[axis]; ++q) out[q] = 0.0;
  for (size_t e = 0; e < numel; ++e) {
    uint64_t xb = 0;
    for (int d = 0; d < k; ++d)
      if (d != axis) xb ^= (uint64_t)bit_at(signs[d], idx[d]);
    out[idx[axis]] += flip(a[e], xb);
    for (int d = k - 1; d >= 0; --d) {
      if (++idx[d] < shape[d]) break;
      idx[d] = 0;
    }
  }
}

/* ---- residual operators with pending terms: inc/search.hpp:53-127 ---------- */

typedef struct {
  uint64_t* signs[8]; /* one per axis */
  double alpha;
} pending_term;

/* MatrixResidualOp::apply_col_correction, inc/search.hpp:74-82 */
static void col_correction(const pending_term* p, size_t np, size_t m, size_t n, double* y,
                           const uint64_t* t) {
  for (size_t q = 0; q < np; ++q) {
    const double g = p[q].alpha * (double)sign_dot(p[q].signs[1], t, n);
    for (size_t i = 0; i < m; ++i) y[i] -= flip(g, (uint64_t)bit_at(p[q].signs[0], i));
  }
}

/* MatrixResidualOp::apply_row_correction, inc/search.hpp:85-93 */
static void row_correction(const pending_term* p, size_t np, size_t m, size_t n, double* z,
                           const uint64_t* s) {
  for (size_t q = 0; q < np; ++q) {
    const double g = p[q].alpha * (double)sign_dot(p[q].signs[0], s, m);
    for (size_t j = 0; j < n; ++j) z[j] -= flip(g, (uint64_t)bit_at(p[q].signs[1], j));
  }
}

typedef struct {
  double value;
  uint64_t* signs[8];
  size_t iterations;
} cut_result;

typedef struct {
  double* values;
  size_t count;
} sweep_log;

/* greedy_matrix_run, inc/search.hpp:145-186 (delta cache, fresh refresh every 16) */
static int greedy_matrix_run(const double* base, size_t m, size_t n, const pending_term* pend,
                             size_t np, xoshiro* rng, size_t max_sweeps, cut_result* res,
                             sweep_log* log) {
  const size_t wm = nwords(m), wn = nwords(n);
  int rc = 0;
  uint64_t* s = calloc(wm, 8);
  uint64_t* t = calloc(wn, 8);
  uint64_t* s_new = calloc(wm, 8);
  uint64_t* t_new = calloc(wn, 8);
  double* y_base = malloc(m * sizeof(double));
  double* z_base = malloc(n * sizeof(double));
  double* y = malloc(m * sizeof(double));
  double* z = malloc(n * sizeof(double));
  random_signs(rng, m, s); /* drawn first, overwritten at sweep 1 (:149) */
  random_signs(rng, n, t); /* effective start vector (:150) */
  matvec(base, m, n, t, y_base);
  double c_prev = -INFINITY;
  size_t sweep;
  for (sweep = 1; sweep <= max_sweeps; ++sweep) {
    memcpy(y, y_base, m * sizeof(double));
    col_correction(pend, np, m, n, y, t);
    if ((rc = sgn_vec(y, m, s_new))) goto done;
    if (sweep == 1) {
      matvec_t(base, m, n, s_new, z_base);
    } else {
      delta_matvec_t(base, m, n, z_base, s_new, s);
    }
    memcpy(z, z_base, n * sizeof(double));
    row_correction(pend, np, m, n, z, s_new);
    if ((rc = sgn_vec(z, n, t_new))) goto done;
    delta_matvec(base, m, n, y_base, t_new, t);
    if (sweep % 16 == 0) { /* kCacheRefreshSweeps, :129, :167-169 */
      matvec(base, m, n, t_new, y_base);
      matvec_t(base, m, n, s_new, z_base);
    }
    memcpy(y, y_base, m * sizeof(double));
    col_correction(pend, np, m, n, y, t_new);
    const double c = signed_dot(s_new, y, m);
    if (log && log->values) log->values[log->count++] = c;
    if (c <= c_prev) {
      res->value = c;
      memcpy(res->signs[0], s_new, wm * 8);
      memcpy(res->signs[1], t_new, wn * 8);
      res->iterations = sweep;
      goto done;
    }
    c_prev = c;
    memcpy(s, s_new, wm * 8);
    memcpy(t, t_new, wn * 8);
  }
  res->value = c_prev; /* cap reached: last sweep's triple (:185) */
  memcpy(res->signs[0], s, wm * 8);
  memcpy(res->signs[1], t, wn * 8);
  res->iterations = max_sweeps;
done:
  free(s); free(t); free(s_new); free(t_new);
  free(y_base); free(z_base); free(y); free(z);
  return rc;
}

/* TensorResidualOp::axial, inc/search.hpp:109-122 */
static void tensor_axial(const double* base, int k, const size_t* shape, size_t numel,
                         const pending_term* pend, size_t np, int axis, uint64_t* const* signs,
                         double* v) {
  axial_contract(base, k, shape, numel, axis, signs, v);
  for (size_t q = 0; q < np; ++q) {
    double g = pend[q].alpha;
    for (int i = 0; i < k; ++i)
      if (i != axis) g *= (double)sign_dot(pend[q].signs[i], signs[i], shape[i]);
    for (size_t e = 0; e < shape[axis]; ++e)
      v[e] -= flip(g, (uint64_t)bit_at(pend[q].signs[axis], e));
  }
}

/* axial_run, inc/search.hpp:191-213 (Gauss-Seidel over axes) */
static int axial_run(const double* base, int k, const size_t* shape, size_t numel,
                     const pending_term* pend, size_t np, xoshiro* rng, size_t max_sweeps,
                     cut_result* res, sweep_log* log) {
  int rc = 0;
  size_t maxlen = 0;
  for (int i = 0; i < k; ++i) maxlen = shape[i] > maxlen ? shape[i] : maxlen;
  double* v = malloc(maxlen * sizeof(double));
  uint64_t* sg[8];
  for (int i = 0; i < k; ++i) {
    sg[i] = calloc(nwords(shape[i]), 8);
    random_signs(rng, shape[i], sg[i]);
  }
  double c_prev = -INFINITY;
  size_t last_sweep = 0;
  for (size_t sweep = 1; sweep <= max_sweeps; ++sweep) {
    for (int axis = 0; axis < k; ++axis) {
      tensor_axial(base, k, shape, numel, pend, np, axis, sg, v);
      if ((rc = sgn_vec(v, shape[axis], sg[axis]))) goto done;
    }
    const double c = signed_dot(sg[k - 1], v, shape[k - 1]);
    if (log && log->values) log->values[log->count++] = c;
    if (c <= c_prev) {
      res->value = c;
      for (int i = 0; i < k; ++i) memcpy(res->signs[i], sg[i], nwords(shape[i]) * 8);
      res->iterations = sweep;
      goto done;
    }
    c_prev = c;
    last_sweep = sweep;
  }
  res->value = c_prev;
  for (int i = 0; i < k; ++i) memcpy(res->signs[i], sg[i], nwords(shape[i]) * 8);
  res->iterations = last_sweep;
done:
  for (int i = 0; i < k; ++i) free(sg[i]);
  free(v);
  return rc;
}

/* best_of_restarts + search_tensor_residual, inc/search.hpp:215-252 */
static int search_residual(const double* base, int k, const size_t* shape, size_t numel,
                           const pending_term* pend, size_t np, uint64_t seed, size_t restarts,
                           size_t max_sweeps, cut_result* best, sweep_log* log) {
  if (restarts < 1) return fail(1, "SearchConfig: restarts must be >= 1");
  if (max_sweeps < 1) return fail(1, "SearchConfig: max_sweeps must be >= 1");
  cut_result cur;
  double* cur_log = log && log->values ? malloc(max_sweeps * sizeof(double)) : NULL;
  for (int i = 0; i < k; ++i) cur.signs[i] = calloc(nwords(shape[i]), 8);
  int have = 0, rc = 0;
  for (size_t r = 0; r < restarts; ++r) {
    xoshiro rng;
    xo_seed(&rng, orc_substream(seed, r));
    sweep_log cl = {cur_log, 0};
    if (k == 2)
      rc = greedy_matrix_run(base, shape[0], shape[1], pend, np, &rng, max_sweeps, &cur, &cl);
    else
      rc = axial_run(base, k, shape, numel, pend, np, &rng, max_sweeps, &cur, &cl);
    if (rc) break;
    if (!have || cur.value > best->value) { /* strict: earliest restart wins ties (:226) */
      best->value = cur.value;
      best->iterations = cur.iterations;
      for (int i = 0; i < k; ++i) memcpy(best->signs[i], cur.signs[i], nwords(shape[i]) * 8);
      if (log && log->values) {
        memcpy(log->values, cur_log, cl.count * sizeof(double));
        log->count = cl.count;
      }
      have = 1;
    }
  }
  for (int i = 0; i < k; ++i) free(cur.signs[i]);
  free(cur_log);
  return rc;
}

/* ---- decomposition driver: inc/decompose.hpp:128-214, 290-361 ------------- */

/* accumulate_terms(base, all_axes, -1, 1, views, -1.0), inc/decompose.hpp:128-180 and
 * flush_pending :200-214.  Per element: acc = sum_j flip(-alpha_j, parity_j) in term
 * order starting from 0.0, then data[e] += acc. */
static void flush_pending(double* base, int k, const size_t* shape, size_t numel,
                          pending_term* pend, size_t np) {
  if (np == 0) return;
  double* scaled = malloc(np * sizeof(double));
  for (size_t j = 0; j < np; ++j) scaled[j] = -1.0 * pend[j].alpha;
  size_t idx[8] = {0};
  for (size_t e = 0; e < numel; ++e) {
    double acc = 0.0;
    for (size_t j = 0; j < np; ++j) {
      uint64_t xb = 0;
      for (int d = 0; d < k; ++d) xb ^= (uint64_t)bit_at(pend[j].signs[d], idx[d]);
      acc += flip(scaled[j], xb);
    }
    base[e] += acc;
    for (int d = k - 1; d >= 0; --d) {
      if (++idx[d] < shape[d]) break;
      idx[d] = 0;
    }
  }
  free(scaled);
}

/* DenseTensor::squared_norm, inc/dense_tensor.hpp:47-51 */
static double squared_norm(const double* a, size_t numel) {
  double acc = 0.0;
  for (size_t i = 0; i < numel; ++i) acc += a[i] * a[i];
  return acc;
}

static int check_shape(int order, const uint64_t* shape, size_t* sh, size_t* numel) {
  if (order < 1 || order > 8) return fail(1, "DenseTensor: order must be >= 1");
  size_t n = 1;
  for (int i = 0; i < order; ++i) {
    if (shape[i] == 0) return fail(1, "DenseTensor: zero-length axis");
    sh[i] = (size_t)shape[i];
    n *= sh[i];
  }
  *numel = n;
  return 0;
}

/* metrics: inc/metrics.hpp:18-63 */
static size_t bits_per_term(int coeff_bits, int order, const size_t* shape) {
  size_t sb = 0;
  for (int i = 0; i < order; ++i) sb += shape[i];
  return (size_t)coeff_bits + sb;
}

double orc_compression_rate(uint64_t k, int coeff_bits, int source_bits, int order,
                            const uint64_t* shape) {
  size_t sh[8], numel;
  if (check_shape(order, shape, sh, &numel)) return NAN;
  const double term_bits = (double)bits_per_term(coeff_bits, order, sh);
  const double src = (double)source_bits * (double)numel;
  return (double)k * term_bits / src;
}

uint64_t orc_width_for_compression(int coeff_bits, int source_bits, int order,
                                   const uint64_t* shape, double rate) {
  size_t sh[8], numel;
  if (check_shape(order, shape, sh, &numel)) return 0;
  if (!(rate > 0.0) || rate > 1.0) return 0;
  const double src = (double)source_bits * (double)numel;
  return (uint64_t)floor(rate * src / (double)bits_per_term(coeff_bits, order, sh));
}

/* quantize_half(kBf16), inc/metrics.hpp:120-160: RNE onto 8-bit exp / 7-bit frac */
void orc_quantize_bf16(uint64_t count, const double* in, double* out) {
  const int exp_bits = 8, frac_bits = 7;
  const int bias = (1 << (exp_bits - 1)) - 1;
  const int emax = bias, emin = 1 - bias;
  for (uint64_t i = 0; i < count; ++i) {
    const double x = in[i];
    if (x == 0.0) {
      out[i] = x;
      continue;
    }
    int e = ilogb(fabs(x));
    if (e < emin) e = emin;
    const double ulp = ldexp(1.0, e - frac_bits);
    const double r = nearbyint(x / ulp) * ulp;
    const double max_finite = (2.0 - ldexp(1.0, -frac_bits)) * ldexp(1.0, emax);
    out[i] = fabs(r) > max_finite ? copysign(max_finite, x) : r;
  }
}

/* greedy_decompose, inc/decompose.hpp:314-361 */
int orc_greedy_decompose(const double* a, int order, const uint64_t* shape,
                         const oracle_config* cfg, oracle_output* out) {
  size_t sh[8], numel;
  int rc = check_shape(order, shape, sh, &numel);
  if (rc) return rc;
  for (size_t i = 0; i < numel; ++i)
    if (!isfinite(a[i])) return fail(1, "DenseTensor: non-finite value");
  /* check_decompose_config, :290-298 */
  if (cfg->flush_width < 1) return fail(1, "DecomposeConfig: flush_width must be >= 1");
  size_t per_term = sizeof(double);
  for (int i = 0; i < order; ++i) per_term += nwords(sh[i]) * sizeof(uint64_t);
  if (cfg->width > 0 && per_term > cfg->max_factor_bytes / cfg->width)
    return fail(1, "DecomposeConfig: width exceeds the factor memory budget");
  if (cfg->restarts < 1) return fail(1, "SearchConfig: restarts must be >= 1");
  if (cfg->max_sweeps < 1) return fail(1, "SearchConfig: max_sweeps must be >= 1");

  const double n_entries = (double)numel;
  double* base = malloc(numel * sizeof(double));
  memcpy(base, a, numel * sizeof(double));
  out->input_norm = sqrt(squared_norm(a, numel));
  double resid_sq = squared_norm(a, numel);
  double first_value = 0.0;
  const size_t fw = (size_t)cfg->flush_width;
  pending_term* pend = calloc(fw, sizeof(pending_term));
  for (size_t j = 0; j < fw; ++j)
    for (int i = 0; i < order; ++i) pend[j].signs[i] = calloc(nwords(sh[i]), 8);
  size_t np = 0;
  cut_result res;
  for (int i = 0; i < order; ++i) res.signs[i] = calloc(nwords(sh[i]), 8);
  size_t done = 0;
  for (size_t term = 0; term < cfg->width; ++term) {
    const uint64_t tseed = orc_substream(cfg->seed, term); /* term_search_config :300-304 */
    rc = search_residual(base, order, sh, numel, pend, np, tseed, cfg->restarts,
                         cfg->max_sweeps, &res, NULL);
    if (rc) break;
    if (term == 0) {
      first_value = res.value;
    } else if (res.value < cfg->min_value_fraction * first_value) {
      break;
    }
    const double alpha = res.value / n_entries;
    for (int i = 0; i < order; ++i)
      memcpy(out->signs[i] + term * nwords(sh[i]), res.signs[i], nwords(sh[i]) * 8);
    out->alpha[term] = alpha;
    out->cut_value[term] = res.value;
    if (out->iterations) out->iterations[term] = res.iterations;
    {
      const double r2 = resid_sq - res.value * res.value / n_entries;
      resid_sq = (0.0 < r2) ? r2 : 0.0; /* std::max(0.0, r2) */
    }
    for (int i = 0; i < order; ++i) memcpy(pend[np].signs[i], res.signs[i], nwords(sh[i]) * 8);
    pend[np].alpha = alpha;
    ++np;
    if (np >= fw) {
      flush_pending(base, order, sh, numel, pend, np);
      np = 0;
      resid_sq = squared_norm(base, numel); /* exact re-anchor */
    }
    out->resid_norm[term] = sqrt(resid_sq);
    done = term + 1;
  }
  if (!rc) {
    flush_pending(base, order, sh, numel, pend, np);
    resid_sq = squared_norm(base, numel);
    if (done > 0) out->resid_norm[done - 1] = sqrt(resid_sq);
    out->width_done = done;
    out->final_residual_norm = sqrt(resid_sq);
    if (out->remainder) memcpy(out->remainder, base, numel * sizeof(double));
  }
  for (size_t j = 0; j < fw; ++j)
    for (int i = 0; i < order; ++i) free(pend[j].signs[i]);
  for (int i = 0; i < order; ++i) free(res.signs[i]);
  free(pend);
  free(base);
  return rc;
}

/* greedy_signed_cut / axial_greedy_cut, inc/search.hpp:259-272 */
int orc_signed_cut(const double* a, int order, const uint64_t* shape, uint64_t seed,
                   uint64_t restarts, uint64_t max_sweeps, double* value, uint64_t** signs,
                   uint64_t* iterations, double* sweep_values, uint64_t* n_sweep_values) {
  size_t sh[8], numel;
  int rc = check_shape(order, shape, sh, &numel);
  if (rc) return rc;
  cut_result res;
  for (int i = 0; i < order; ++i) res.signs[i] = signs[i];
  sweep_log log = {sweep_values, 0};
  rc = search_residual(a, order, sh, numel, NULL, 0, seed, (size_t)restarts, (size_t)max_sweeps,
                       &res, &log);
  if (rc) return rc;
  *value = res.value;
  *iterations = res.iterations;
  if (n_sweep_values) *n_sweep_values = log.count;
  return 0;
}

/* ======================================================================== *
 * Around the path: expansion, Gram system, least squares,
 * SCD / DTEN containers.
 * ======================================================================== */

/* sign slot of every axis (-1 for the channel axis) */
static int sign_slots(int order, int channel_axis, int* slot_of) {
  int s = 0;
  for (int i = 0; i < order; ++i) slot_of[i] = i == channel_axis ? -1 : s++;
  return s;
}

/* accumulate_terms (decompose.hpp:128-180) via accumulate_expansion (:182-197):
 * per element, acc = sum over terms j >= first of flip(scale*coef_j(ch), parity_j)
 * in term order from 0.0, then data[e] += acc. */
int orc_accumulate_expansion(int order, const uint64_t* shape, int channel_axis, uint64_t width,
                             const uint64_t* const* factors, const double* coeffs, double scale,
                             uint64_t first_term, double* data) {
  size_t sh[8], numel;
  int rc = check_shape(order, shape, sh, &numel);
  if (rc) return rc;
  if (channel_axis < -1 || channel_axis >= order) return fail(1, "CutDecomposition: channel axis out of range");
  if (first_term >= width) return 0;
  int slot_of[8];
  sign_slots(order, channel_axis, slot_of);
  const size_t q = channel_axis >= 0 ? sh[channel_axis] : 1;
  const size_t w = (size_t)(width - first_term);
  double* scaled = malloc(w * q * sizeof(double));
  for (size_t j = 0; j < w; ++j)
    for (size_t c = 0; c < q; ++c) scaled[j * q + c] = scale * coeffs[(first_term + j) * q + c];
  size_t idx[8] = {0};
  for (size_t e = 0; e < numel; ++e) {
    const size_t ch = channel_axis >= 0 ? idx[channel_axis] : 0;
    double acc = 0.0;
    for (size_t j = 0; j < w; ++j) {
      uint64_t xb = 0;
      for (int d = 0; d < order; ++d)
        if (slot_of[d] >= 0) xb ^= (uint64_t)bit_at(factors[slot_of[d]] + (first_term + j) * nwords(sh[d]), idx[d]);
      acc += flip(scaled[j * q + ch], xb);
    }
    data[e] += acc;
    for (int d = order - 1; d >= 0; --d) {
      if (++idx[d] < sh[d]) break;
      idx[d] = 0;
    }
  }
  free(scaled);
  return 0;
}

/* contract_term (decompose.hpp:218-260): out[ch] += flip(a[e], parity) in element order */
static void contract_term(const double* a, int order, const size_t* sh, size_t numel, int channel_axis,
                          const int* slot_of, const uint64_t* const* signs, double* out) {
  const size_t q = channel_axis >= 0 ? sh[channel_axis] : 1;
  for (size_t c = 0; c < q; ++c) out[c] = 0.0;
  size_t idx[8] = {0};
  for (size_t e = 0; e < numel; ++e) {
    uint64_t xb = 0;
    for (int d = 0; d < order; ++d)
      if (slot_of[d] >= 0) xb ^= (uint64_t)bit_at(signs[slot_of[d]], idx[d]);
    out[channel_axis >= 0 ? idx[channel_axis] : 0] += flip(a[e], xb);
    for (int d = order - 1; d >= 0; --d) {
      if (++idx[d] < sh[d]) break;
      idx[d] = 0;
    }
  }
}

/* gram_column (decompose.hpp:367-381): products of per-axis sign dots, diag = prod n */
static void gram_column(int order, const size_t* sh, const int* slot_of, const uint64_t* const* factors,
                        size_t count, const uint64_t* const* new_signs, double* col) {
  for (size_t j = 0; j < count; ++j) {
    double g = 1.0;
    for (int d = 0; d < order; ++d) {
      if (slot_of[d] < 0) continue;
      g *= (double)sign_dot(factors[slot_of[d]] + j * nwords(sh[d]), new_signs[slot_of[d]], sh[d]);
    }
    col[j] = g;
  }
  double diag = 1.0;
  for (int d = 0; d < order; ++d)
    if (slot_of[d] >= 0) diag *= (double)sh[d];
  col[count] = diag;
}

int orc_build_gram(const double* a, int order, const uint64_t* shape, int channel_axis, uint64_t width,
                   const uint64_t* const* factors, double* gram, double* rhs) {
  size_t sh[8], numel;
  int rc = check_shape(order, shape, sh, &numel);
  if (rc) return rc;
  int slot_of[8];
  const int ns = sign_slots(order, channel_axis, slot_of);
  const size_t q = channel_axis >= 0 ? sh[channel_axis] : 1;
  double* col = malloc((width + 1) * sizeof(double));
  const uint64_t* sig[8];
  for (size_t j = 0; j < width; ++j) {
    for (int s = 0, d = 0; d < order; ++d)
      if (slot_of[d] >= 0) {
        sig[s] = factors[s] + j * nwords(sh[d]);
        ++s;
      }
    gram_column(order, sh, slot_of, factors, j, sig, col);
    for (size_t i = 0; i < j; ++i) gram[i * width + j] = gram[j * width + i] = col[i];
    gram[j * width + j] = col[j];
    contract_term(a, order, sh, numel, channel_axis, slot_of, sig, rhs + j * q);
  }
  (void)ns;
  free(col);
  return 0;
}

/* cholesky / cholesky_solve / solve_gram (gram.hpp:48-107) */
static int cholesky(double* m, size_t n) {
  for (size_t j = 0; j < n; ++j) {
    double d = m[j * n + j];
    for (size_t p = 0; p < j; ++p) d -= m[j * n + p] * m[j * n + p];
    if (!(d > 0.0) || !isfinite(d)) return 0;
    const double l = sqrt(d);
    m[j * n + j] = l;
    for (size_t i = j + 1; i < n; ++i) {
      double v = m[i * n + j];
      for (size_t p = 0; p < j; ++p) v -= m[i * n + p] * m[j * n + p];
      m[i * n + j] = v / l;
    }
  }
  return 1;
}

static void cholesky_solve(const double* l, size_t n, double* x) {
  for (size_t i = 0; i < n; ++i) {
    double v = x[i];
    for (size_t p = 0; p < i; ++p) v -= l[i * n + p] * x[p];
    x[i] = v / l[i * n + i];
  }
  for (size_t i = n; i-- > 0;) {
    double v = x[i];
    for (size_t p = i + 1; p < n; ++p) v -= l[p * n + i] * x[p];
    x[i] = v / l[i * n + i];
  }
}

int orc_solve_gram(uint64_t width, uint64_t channels, const double* gram, const double* rhs, double* out) {
  const size_t w = (size_t)width;
  if (w == 0) return 0;
  const double base_ridge = 1e-10 * gram[0];
  double* factor = malloc(w * w * sizeof(double));
  int ok = 0;
  for (int attempt = 0; attempt < 5 && !ok; ++attempt) {
    memcpy(factor, gram, w * w * sizeof(double));
    if (attempt > 0) {
      const double ridge = base_ridge * (double)(1 << (attempt - 1));
      for (size_t j = 0; j < w; ++j) factor[j * w + j] += ridge;
    }
    ok = cholesky(factor, w);
  }
  if (!ok) {
    free(factor);
    return fail(2, "solve_gram: factorization failed");
  }
  double* x = malloc(w * sizeof(double));
  for (size_t c = 0; c < channels; ++c) {
    for (size_t j = 0; j < w; ++j) x[j] = rhs[j * channels + c];
    cholesky_solve(factor, w, x);
    for (size_t j = 0; j < w; ++j) out[j * channels + c] = x[j];
  }
  free(x);
  free(factor);
  return 0;
}

/* gram_quadratic (decompose.hpp:397-410) */
static double gram_quadratic(size_t w, size_t ch, const double* gram, const double* rhs, const double* c) {
  double value = 0.0;
  for (size_t k = 0; k < ch; ++k) {
    for (size_t i = 0; i < w; ++i) {
      const double ci = c[i * ch + k];
      value -= 2.0 * ci * rhs[i * ch + k];
      double row = 0.0;
      for (size_t j = 0; j < w; ++j) row += gram[i * w + j] * c[j * ch + k];
      value += ci * row;
    }
  }
  return value;
}

/* correct_coefficients (decompose.hpp:418-428) */
int orc_correct_coefficients(const double* a, int order, const uint64_t* shape, int channel_axis, uint64_t width,
                             const uint64_t* const* factors, const double* coeffs, double* out) {
  size_t sh[8], numel;
  int rc = check_shape(order, shape, sh, &numel);
  if (rc) return rc;
  const size_t q = channel_axis >= 0 ? sh[channel_axis] : 1;
  const size_t w = (size_t)width;
  if (w == 0) return 0;
  double* gram = malloc(w * w * sizeof(double));
  double* rhs = malloc(w * q * sizeof(double));
  double* solved = malloc(w * q * sizeof(double));
  rc = orc_build_gram(a, order, shape, channel_axis, width, factors, gram, rhs);
  if (!rc) rc = orc_solve_gram(width, q, gram, rhs, solved);
  if (!rc) {
    const int better = gram_quadratic(w, q, gram, rhs, solved) <= gram_quadratic(w, q, gram, rhs, coeffs);
    memcpy(out, better ? solved : coeffs, w * q * sizeof(double));
  }
  free(gram);
  free(rhs);
  free(solved);
  return rc;
}

/* lstsq_decompose (decompose.hpp:434-469) and rgb_scalars_decompose (:485-536) */
int orc_lstsq_decompose(const double* a, int order, const uint64_t* shape, int channel_axis,
                        const oracle_config* cfg, oracle_output* out) {
  size_t sh[8], numel;
  int rc = check_shape(order, shape, sh, &numel);
  if (rc) return rc;
  for (size_t i = 0; i < numel; ++i)
    if (!isfinite(a[i])) return fail(1, "DenseTensor: non-finite value");
  size_t q = 1;
  if (channel_axis >= 0) {
    if (order < 2) return fail(1, "rgb_scalars_decompose: order >= 2 required");
    if (channel_axis >= order) return fail(1, "rgb_scalars_decompose: channel axis out of range");
    q = sh[channel_axis];
    if (q > 8) return fail(1, "rgb_scalars_decompose: channel axis too long");
  }
  if (cfg->flush_width < 1) return fail(1, "DecomposeConfig: flush_width must be >= 1");
  size_t per_term = q * sizeof(double);
  for (int i = 0; i < order; ++i) per_term += nwords(sh[i]) * sizeof(uint64_t);
  if (cfg->width > 0 && per_term > cfg->max_factor_bytes / cfg->width)
    return fail(1, "DecomposeConfig: width exceeds the factor memory budget");
  int slot_of[8];
  sign_slots(order, channel_axis, slot_of);
  const size_t w = (size_t)cfg->width;
  double* residual = malloc(numel * sizeof(double));
  memcpy(residual, a, numel * sizeof(double));
  double* gram = NULL;
  double* rhs = malloc((w ? w : 1) * q * sizeof(double));
  double* col = malloc((w + 1) * sizeof(double));
  double* coef = calloc((w ? w : 1) * q, sizeof(double));
  out->input_norm = sqrt(squared_norm(a, numel));
  out->final_residual_norm = out->input_norm;
  cut_result res;
  for (int i = 0; i < order; ++i) res.signs[i] = calloc(nwords(sh[i]), 8);
  double first_value = 0.0;
  size_t gw = 0;
  for (size_t term = 0; term < w; ++term) {
    rc = search_residual(residual, order, sh, numel, NULL, 0, orc_substream(cfg->seed, term), cfg->restarts,
                         cfg->max_sweeps, &res, NULL);
    if (rc) break;
    if (term == 0) first_value = res.value;
    else if (res.value < cfg->min_value_fraction * first_value) break;
    const uint64_t* sig[8];
    for (int d = 0; d < order; ++d)
      if (slot_of[d] >= 0) sig[slot_of[d]] = res.signs[d];
    gram_column(order, sh, slot_of, (const uint64_t* const*)out->signs, gw, sig, col);
    double* grown = malloc((gw + 1) * (gw + 1) * sizeof(double));
    for (size_t i = 0; i < gw; ++i) {
      for (size_t j = 0; j < gw; ++j) grown[i * (gw + 1) + j] = gram[i * gw + j];
      grown[i * (gw + 1) + gw] = col[i];
      grown[gw * (gw + 1) + i] = col[i];
    }
    grown[gw * (gw + 1) + gw] = col[gw];
    free(gram);
    gram = grown;
    contract_term(a, order, sh, numel, channel_axis, slot_of, sig, rhs + gw * q);
    for (int d = 0; d < order; ++d)
      if (slot_of[d] >= 0) memcpy(out->signs[slot_of[d]] + gw * nwords(sh[d]), res.signs[d], nwords(sh[d]) * 8);
    ++gw;
    rc = orc_solve_gram(gw, q, gram, rhs, coef);
    if (rc) break;
    memcpy(residual, a, numel * sizeof(double));
    orc_accumulate_expansion(order, shape, channel_axis, gw, (const uint64_t* const*)out->signs, coef, -1.0, 0,
                             residual);
    out->final_residual_norm = sqrt(squared_norm(residual, numel));
    out->cut_value[term] = res.value;
    out->resid_norm[term] = out->final_residual_norm;
    if (out->iterations) out->iterations[term] = res.iterations;
  }
  if (!rc) {
    memcpy(out->alpha, coef, gw * q * sizeof(double));
    out->width_done = gw;
  }
  for (int i = 0; i < order; ++i) free(res.signs[i]);
  free(residual);
  free(gram);
  free(rhs);
  free(col);
  free(coef);
  return rc;
}

/* ---- SCD / DTEN containers: inc/io.hpp -------------------------------- */

typedef struct {
  uint8_t* buf;
  uint64_t cap, pos;
} bytes_out;

static void put(bytes_out* o, const void* p, size_t n) {
  if (o->pos + n <= o->cap) memcpy(o->buf + o->pos, p, n);
  o->pos += n;
}
static void put_u64le(bytes_out* o, uint64_t v) {
  uint8_t b[8];
  for (int i = 0; i < 8; ++i) b[i] = (uint8_t)(v >> (8 * i));
  put(o, b, 8);
}
static void put_u8(bytes_out* o, uint8_t v) { put(o, &v, 1); }

/* write_scd (io.hpp:142-166) */
int orc_write_scd(int order, const uint64_t* shape, int channel_axis, uint64_t width, const uint64_t* const* factors,
                  const double* coeffs, int coeff_bits, uint8_t* buf, uint64_t cap, uint64_t* size) {
  if (coeff_bits != 32 && coeff_bits != 64) return fail(1, "write_scd: coeff_bits must be 32 or 64");
  size_t sh[8], numel;
  int rc = check_shape(order, shape, sh, &numel);
  if (rc) return rc;
  const size_t q = channel_axis >= 0 ? sh[channel_axis] : 1;
  for (size_t i = 0; i < width * q; ++i)
    if (!isfinite(coeffs[i])) return fail(1, "CutDecomposition: non-finite coefficient");
  int slot_of[8];
  sign_slots(order, channel_axis, slot_of);
  bytes_out o = {buf, cap, 0};
  put(&o, "SCD1", 4);
  put_u8(&o, (uint8_t)order);
  put_u8(&o, channel_axis >= 0 ? 1 : 0);
  if (channel_axis >= 0) put_u8(&o, (uint8_t)channel_axis);
  for (int i = 0; i < order; ++i) put_u64le(&o, shape[i]);
  put_u64le(&o, width);
  put_u8(&o, (uint8_t)coeff_bits);
  for (uint64_t j = 0; j < width; ++j) {
    for (size_t c = 0; c < q; ++c) {
      uint64_t u;
      if (coeff_bits == 64) {
        memcpy(&u, &coeffs[j * q + c], 8);
        put_u64le(&o, u);
      } else {
        const float f = (float)coeffs[j * q + c];
        uint32_t v;
        memcpy(&v, &f, 4);
        uint8_t b[4];
        for (int i = 0; i < 4; ++i) b[i] = (uint8_t)(v >> (8 * i));
        put(&o, b, 4);
      }
    }
    for (int d = 0; d < order; ++d) { /* put_sign_column, io.hpp:82-92 */
      if (slot_of[d] < 0) continue;
      const uint64_t* wds = factors[slot_of[d]] + j * nwords(sh[d]);
      for (size_t byte = 0; byte < (sh[d] + 7) / 8; ++byte) put_u8(&o, (uint8_t)(wds[byte / 8] >> (8 * (byte % 8))));
    }
  }
  *size = o.pos;
  if (o.pos > cap) return fail(1, "buffer too small");
  return 0;
}

typedef struct {
  const uint8_t* buf;
  uint64_t size, pos;
} bytes_in;

static int get(bytes_in* in, void* p, size_t n) {
  if (in->pos + n > in->size) return fail(3, "truncated payload");
  memcpy(p, in->buf + in->pos, n);
  in->pos += n;
  return 0;
}
static int get_u64le(bytes_in* in, uint64_t* v) {
  uint8_t b[8];
  if (get(in, b, 8)) return 3;
  *v = 0;
  for (int i = 0; i < 8; ++i) *v |= (uint64_t)b[i] << (8 * i);
  return 0;
}

/* read_scd (io.hpp:168-213) */
int orc_read_scd(const uint8_t* buf, uint64_t size, int* order, uint64_t* shape, int* channel_axis, uint64_t* width,
                 uint64_t** factors, double* coeffs) {
  bytes_in in = {buf, size, 0};
  char magic[4];
  uint8_t k, mode, cb, ca = 0;
  if (get(&in, magic, 4)) return 3;
  if (memcmp(magic, "SCD1", 4) != 0) return fail(3, "bad SCD magic");
  if (get(&in, &k, 1)) return 3;
  if (k == 0) return fail(3, "SCD order must be >= 1");
  if (get(&in, &mode, 1)) return 3;
  if (mode > 1) return fail(3, "bad SCD channel mode");
  int chax = -1;
  if (mode == 1) {
    if (get(&in, &ca, 1)) return 3;
    if (ca >= k) return fail(3, "SCD channel axis out of range");
    chax = ca;
  }
  if (k > 8) return fail(3, "SCD order above the oracle's limit");
  uint64_t numel = 1;
  for (int i = 0; i < k; ++i) {
    if (get_u64le(&in, &shape[i])) return 3;
    if (shape[i] == 0) return fail(3, "bad SCD shape");
    if (shape[i] > UINT64_MAX / numel) return fail(3, "SCD shape overflow");
    numel *= shape[i];
  }
  uint64_t w;
  if (get_u64le(&in, &w)) return 3;
  if (get(&in, &cb, 1)) return 3;
  if (cb != 32 && cb != 64) return fail(3, "bad SCD coefficient width");
  *order = k;
  *channel_axis = chax;
  *width = w;
  if (factors == NULL || coeffs == NULL) return 0;
  const uint64_t q = chax >= 0 ? shape[chax] : 1;
  for (uint64_t j = 0; j < w; ++j) {
    for (uint64_t c = 0; c < q; ++c) {
      double v;
      if (cb == 64) {
        uint64_t u;
        if (get_u64le(&in, &u)) return 3;
        memcpy(&v, &u, 8);
      } else {
        uint8_t b[4];
        if (get(&in, b, 4)) return 3;
        uint32_t u = 0;
        for (int i = 0; i < 4; ++i) u |= (uint32_t)b[i] << (8 * i);
        float f;
        memcpy(&f, &u, 4);
        v = (double)f;
      }
      if (!isfinite(v)) return fail(3, "non-finite SCD coefficient");
      coeffs[j * q + c] = v;
    }
    for (int d = 0, s = 0; d < k; ++d) { /* get_sign_column, io.hpp:94-109 */
      if (d == chax) continue;
      const size_t nw = nwords(shape[d]);
      uint64_t* wds = factors[s] + j * nw;
      memset(wds, 0, nw * 8);
      for (size_t byte = 0; byte < (shape[d] + 7) / 8; ++byte) {
        uint8_t b;
        if (get(&in, &b, 1)) return 3;
        wds[byte / 8] |= (uint64_t)b << (8 * (byte % 8));
      }
      const size_t tail = shape[d] % 64;
      if (tail != 0 && (wds[nw - 1] >> tail) != 0) return fail(3, "sign column has nonzero pad bits");
      ++s;
    }
  }
  return 0;
}

/* write_raw (io.hpp:226-246) */
int orc_write_raw(int order, const uint64_t* shape, const double* data, int dtype, uint8_t* buf, uint64_t cap,
                  uint64_t* size) {
  size_t sh[8], numel;
  int rc = check_shape(order, shape, sh, &numel);
  if (rc) return rc;
  bytes_out o = {buf, cap, 0};
  put(&o, "DTEN", 4);
  put_u8(&o, (uint8_t)order);
  for (int i = 0; i < order; ++i) put_u64le(&o, shape[i]);
  put_u8(&o, (uint8_t)dtype);
  for (size_t e = 0; e < numel; ++e) {
    if (dtype == 0) {
      uint64_t u;
      memcpy(&u, &data[e], 8);
      put_u64le(&o, u);
    } else if (dtype == 1) {
      const float f = (float)data[e];
      uint32_t v;
      memcpy(&v, &f, 4);
      uint8_t b[4];
      for (int i = 0; i < 4; ++i) b[i] = (uint8_t)(v >> (8 * i));
      put(&o, b, 4);
    } else {
      double v = data[e] < 0.0 ? 0.0 : (data[e] > 255.0 ? 255.0 : data[e]);
      put_u8(&o, (uint8_t)lround(v));
    }
  }
  *size = o.pos;
  if (o.pos > cap) return fail(1, "buffer too small");
  return 0;
}

/* read_raw (io.hpp:250-292) */
int orc_read_raw(const uint8_t* buf, uint64_t size, int* order, uint64_t* shape, double* data) {
  bytes_in in = {buf, size, 0};
  char magic[4];
  uint8_t k, dt;
  if (get(&in, magic, 4)) return 3;
  if (memcmp(magic, "DTEN", 4) != 0) return fail(3, "bad DTEN magic");
  if (get(&in, &k, 1)) return 3;
  if (k == 0) return fail(3, "DTEN order must be >= 1");
  if (k > 8) return fail(3, "DTEN order above the oracle's limit");
  uint64_t numel = 1;
  for (int i = 0; i < k; ++i) {
    if (get_u64le(&in, &shape[i])) return 3;
    if (shape[i] == 0) return fail(3, "DTEN zero-length axis");
    if (shape[i] > UINT64_MAX / numel) return fail(3, "DTEN shape overflow");
    numel *= shape[i];
  }
  if (get(&in, &dt, 1)) return 3;
  if (dt > 2) return fail(3, "bad DTEN dtype");
  *order = k;
  if (data == NULL) return 0;
  for (uint64_t e = 0; e < numel; ++e) {
    if (dt == 0) {
      uint64_t u;
      if (get_u64le(&in, &u)) return 3;
      memcpy(&data[e], &u, 8);
    } else if (dt == 1) {
      uint8_t b[4];
      if (get(&in, b, 4)) return 3;
      uint32_t u = 0;
      for (int i = 0; i < 4; ++i) u |= (uint32_t)b[i] << (8 * i);
      float f;
      memcpy(&f, &u, 4);
      data[e] = (double)f;
    } else {
      uint8_t b;
      if (get(&in, &b, 1)) return 3;
      data[e] = (double)b;
    }
  }
  for (uint64_t e = 0; e < numel; ++e)
    if (!isfinite(data[e])) return fail(3, "invalid DTEN payload: DenseTensor: non-finite value");
  return 0;
}
