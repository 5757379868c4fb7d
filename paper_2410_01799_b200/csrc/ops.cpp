// ops.cpp -- C ABI of the operations around the decomposition:
// expansion / residual accumulation, the Gram system, signed contractions, the
// least-squares and scalar-channel drivers, and the SCD / DTEN containers.
//
// Device work goes to the kernels in ops.cu (and, for the term search, to the
// persistent sweep kernel through sc_greedy_decompose).  Host work is control,
// the w x w Cholesky solve (gram.hpp:48-107) and byte-level container
// encoding -- the reference's own host-side responsibilities.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/sigcut_b200.h"
#include "ctx.h"
#include "ops.h"
#include "rng.h"

namespace {

using scb::set_err;

uint64_t words64(uint64_t n) { return (n + 63) / 64; }

sc_status put_msg(char* msg, size_t len, sc_status st, const std::string& s) {
  if (msg && len) {
    std::strncpy(msg, s.c_str(), len - 1);
    msg[len - 1] = 0;
  }
  return st;
}

// Accumulates one call's accounting into the caller's (optional) stats.
void add_stats(sc_op_stats* out, const sc_op_stats& st) {
  if (out == nullptr) return;
  out->kernel_ms += st.kernel_ms;
  out->total_ms += st.total_ms;
  out->h2d_bytes += st.h2d_bytes;
  out->d2h_bytes += st.d2h_bytes;
  out->kernel_launches += st.kernel_launches;
}

struct Timer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double ms() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
};

// ---------------------------------------------------------------------------
// the tensor as P x Q (rows = axis 0, columns = the trailing axes; order 1:
// P = 1) with the sign slots and channel placement of a CutDecomposition
// ---------------------------------------------------------------------------
struct Layout {
  int order = 0, channel_axis = -1, nsign = 0;
  uint64_t shape[SC_MAX_ORDER] = {};
  uint64_t numel = 1;
  long long P = 1, Q = 1;
  int row_slot = -1;  // sign slot of axis 0 when it is a row sign axis
  int chan = 0;       // 0 none, 1 channel = row, 2 channel from the column index
  long long cstride = 1;
  int nch = 1;
  uint64_t aw[SC_MAX_ORDER] = {};  // u64 words per term of each sign slot
  int ntr = 0;                     // trailing sign axes (column bits)
  int tr_slot[SC_MAX_ORDER] = {};
  long long tr_n[SC_MAX_ORDER] = {}, tr_stride[SC_MAX_ORDER] = {};
  bool v_direct() const { return ntr == 1 && tr_stride[0] == 1 && tr_n[0] == Q; }
  long long v_stride_kron() const { return ((Q + 63) / 64) * 2; }
};

sc_status make_layout(int order, const uint64_t* shape, int channel_axis, Layout* L, std::string* msg) {
  if (shape == nullptr) {
    *msg = "sc_factors: null shape";
    return SC_INVALID_ARGUMENT;
  }
  if (order < 1 || order > SC_MAX_ORDER) {
    *msg = "DenseTensor: order must be >= 1";
    return SC_INVALID_ARGUMENT;
  }
  if (channel_axis < -1 || channel_axis >= order) {
    *msg = "CutDecomposition: channel axis out of range";
    return SC_INVALID_ARGUMENT;
  }
  L->order = order;
  L->channel_axis = channel_axis;
  for (int i = 0; i < order; ++i) {
    if (shape[i] == 0) {
      *msg = "DenseTensor: zero-length axis";
      return SC_INVALID_ARGUMENT;
    }
    if (shape[i] > UINT64_MAX / L->numel) {
      *msg = "DenseTensor: shape overflow";
      return SC_INVALID_ARGUMENT;
    }
    L->shape[i] = shape[i];
    L->numel *= shape[i];
  }
  if (L->numel > (1ull << 40)) {
    *msg = "tensor too large for this build";
    return SC_NOT_SUPPORTED;
  }
  L->nsign = order - (channel_axis >= 0 ? 1 : 0);
  L->nch = channel_axis >= 0 ? static_cast<int>(shape[channel_axis]) : 1;
  int slot_of[SC_MAX_ORDER];
  for (int i = 0, s = 0; i < order; ++i) {
    slot_of[i] = i == channel_axis ? -1 : s++;
    if (slot_of[i] >= 0) L->aw[slot_of[i]] = words64(shape[i]);
  }
  const int first_col = order == 1 ? 0 : 1;
  if (order >= 2) {
    L->P = static_cast<long long>(shape[0]);
    L->row_slot = slot_of[0];
  }
  L->Q = 1;
  for (int i = first_col; i < order; ++i) L->Q *= static_cast<long long>(shape[i]);
  if (channel_axis >= 0) {
    if (order >= 2 && channel_axis == 0) {
      L->chan = 1;
    } else {
      L->chan = 2;
      long long cs = 1;
      for (int i = channel_axis + 1; i < order; ++i) cs *= static_cast<long long>(shape[i]);
      L->cstride = cs;
    }
  }
  long long stride = 1;
  for (int i = order - 1; i >= first_col; --i) {
    if (slot_of[i] >= 0) {
      L->tr_slot[L->ntr] = slot_of[i];
      L->tr_n[L->ntr] = static_cast<long long>(shape[i]);
      L->tr_stride[L->ntr] = stride;
      ++L->ntr;
    }
    stride *= static_cast<long long>(shape[i]);
  }
  return SC_OK;
}

sc_status check_factors(sc_ctx* ctx, const sc_factors* d, Layout* L) {
  if (d == nullptr) return set_err(ctx, SC_INVALID_ARGUMENT, "sc_factors: null");
  std::string msg;
  if (sc_status s = make_layout(d->order, d->shape, d->channel_axis, L, &msg); s != SC_OK)
    return set_err(ctx, s, "%s", msg.c_str());
  if (d->width > 0 && d->coefficients == nullptr)
    return set_err(ctx, SC_INVALID_ARGUMENT, "sc_factors: null coefficients");
  for (int s = 0; s < L->nsign; ++s)
    if (d->width > 0 && d->sign_words[s] == nullptr)
      return set_err(ctx, SC_INVALID_ARGUMENT, "sc_factors: sign_words[%d] missing", s);
  return SC_OK;
}

// ---------------------------------------------------------------------------
// device copies of the sign words of `cap` terms per sign slot, plus the column
// bit rows V (a view of the trailing factor, or Kronecker rows built on device)
// ---------------------------------------------------------------------------
struct DevFactors {
  uint64_t* fac[SC_MAX_ORDER] = {};
  uint32_t* V = nullptr;
  long long v_stride = 0, v_words = 0;
  const uint32_t* U = nullptr;
  long long u_stride = 0;
};

sc_status alloc_factors(sc_ctx* ctx, const Layout& L, uint64_t cap, const std::string& tag, DevFactors* F) {
  for (int s = 0; s < L.nsign; ++s) {
    void* p = nullptr;
    if (sc_status st = scb::pool_get(ctx, tag + ".fac" + std::to_string(s), std::max<uint64_t>(1, cap * L.aw[s]) * 8, &p);
        st != SC_OK)
      return st;
    F->fac[s] = static_cast<uint64_t*>(p);
  }
  if (L.row_slot >= 0) {
    F->U = reinterpret_cast<const uint32_t*>(F->fac[L.row_slot]);
    F->u_stride = static_cast<long long>(2 * L.aw[L.row_slot]);
  }
  if (L.ntr > 0) {
    F->v_words = (L.Q + 31) / 32;
    if (L.v_direct()) {
      F->V = reinterpret_cast<uint32_t*>(F->fac[L.tr_slot[0]]);
      F->v_stride = static_cast<long long>(2 * L.aw[L.tr_slot[0]]);
    } else {
      F->v_stride = L.v_stride_kron();
      void* p = nullptr;
      if (sc_status st = scb::pool_get(ctx, tag + ".V", std::max<uint64_t>(1, cap) * F->v_stride * 4, &p); st != SC_OK)
        return st;
      F->V = static_cast<uint32_t*>(p);
    }
  }
  return SC_OK;
}

// Uploads the words of `count` terms (host rows starting at term `src_first` of
// each slot's array) into device rows [dst_first, dst_first + count), then
// builds their Kronecker column rows.
sc_status upload_factors(sc_ctx* ctx, const Layout& L, const uint64_t* const* host_words, uint64_t src_first,
                         uint64_t dst_first, uint64_t count, const DevFactors& F, sc_op_stats* st) {
  if (count == 0) return SC_OK;
  for (int s = 0; s < L.nsign; ++s) {
    const size_t bytes = count * L.aw[s] * 8;
    SC_CUDA(ctx, cudaMemcpyAsync(F.fac[s] + dst_first * L.aw[s], host_words[s] + src_first * L.aw[s], bytes,
                                 cudaMemcpyHostToDevice, ctx->stream));
    st->h2d_bytes += bytes;
  }
  if (L.ntr > 0 && !L.v_direct()) {
    scb::KronParams kp{};
    kp.V = F.V + dst_first * F.v_stride;
    kp.v_stride = F.v_stride;
    kp.Q = L.Q;
    kp.nterms = static_cast<long long>(count);
    kp.nax = L.ntr;
    for (int a = 0; a < L.ntr; ++a) {
      kp.ax_n[a] = L.tr_n[a];
      kp.ax_stride[a] = L.tr_stride[a];
      kp.fac[a] = F.fac[L.tr_slot[a]] + dst_first * L.aw[L.tr_slot[a]];
      kp.fac_words[a] = static_cast<long long>(L.aw[L.tr_slot[a]]);
    }
    SC_CUDA(ctx, scb::launch_kron(kp, ctx->stream));
    st->kernel_launches += 1;
  }
  return SC_OK;
}

scb::ExpandParams expand_params(const Layout& L, const DevFactors& F, uint64_t first, uint64_t nterms,
                                const double* dcoef, double scale, double* ddata) {
  scb::ExpandParams ep{};
  ep.data = ddata;
  ep.P = L.P;
  ep.Q = L.Q;
  ep.U = F.U ? F.U + first * F.u_stride : nullptr;
  ep.u_stride = F.u_stride;
  ep.V = F.V ? F.V + first * F.v_stride : nullptr;
  ep.v_stride = F.v_stride;
  ep.v_words = F.v_words;
  ep.coef = dcoef + first * L.nch;
  ep.nch = L.nch;
  ep.chan = L.chan;
  ep.cstride = L.cstride;
  ep.nterms = static_cast<long long>(nterms);
  ep.scale = scale;
  return ep;
}

// contraction of device terms [first, first + count) against device A (a_dtype)
sc_status contract(sc_ctx* ctx, const Layout& L, const DevFactors& F, uint64_t first, uint64_t count, int a_dtype,
                   const void* dA, double* rhs_host, sc_op_stats* st) {
  if (count == 0) return SC_OK;
  const int per = L.chan == 0 ? scb::kContractTerms : 1;
  const int slots = L.chan == 0 ? 1 : 8;
  void *part = nullptr, *out = nullptr;
  if (sc_status s = scb::pool_get(ctx, "contract.part", sizeof(double) * scb::kContractCtas * scb::kContractTerms * 8, &part);
      s != SC_OK)
    return s;
  // every batch writes its outputs at its own offset; one copy back at the end
  const uint64_t nbatch = (count + per - 1) / per;
  if (sc_status s = scb::pool_get(ctx, "contract.out", sizeof(double) * nbatch * per * slots, &out); s != SC_OK) return s;
  for (uint64_t b = 0; b < count; b += per) {
    const uint64_t nt = std::min<uint64_t>(per, count - b);
    const uint64_t j = first + b;
    scb::ContractParams cp{};
    cp.A = dA;
    cp.a_f32 = a_dtype == SC_F32;
    cp.P = L.P;
    cp.Q = L.Q;
    cp.U = F.U ? F.U + j * F.u_stride : nullptr;
    cp.u_stride = F.u_stride;
    cp.V = F.V ? F.V + j * F.v_stride : nullptr;
    cp.v_stride = F.v_stride;
    cp.nterms = static_cast<long long>(nt);
    cp.nch = L.nch;
    cp.chan = L.chan;
    cp.cstride = L.cstride;
    cp.part = static_cast<double*>(part);
    cp.out = static_cast<double*>(out) + b * slots;
    SC_CUDA(ctx, scb::launch_contract(cp, ctx->stream));
    st->kernel_launches += 2;
  }
  std::vector<double> tmp(count * slots);
  SC_CUDA(ctx, cudaMemcpyAsync(tmp.data(), out, count * slots * 8, cudaMemcpyDeviceToHost, ctx->stream));
  SC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  st->d2h_bytes += count * slots * 8;
  for (uint64_t t = 0; t < count; ++t)
    for (int c = 0; c < L.nch; ++c) rhs_host[t * L.nch + c] = tmp[t * slots + c];
  return SC_OK;
}

sc_status gram_block(sc_ctx* ctx, const Layout& L, const DevFactors& F, uint64_t i0, uint64_t rows, uint64_t j0,
                     uint64_t cols, double* dG, long long ldg, sc_op_stats* st) {
  scb::GramParams gp{};
  gp.G = dG;
  gp.ldg = ldg;
  gp.rows = static_cast<long long>(rows);
  gp.cols = static_cast<long long>(cols);
  gp.nax = L.nsign;
  for (int s = 0, i = 0; i < L.order; ++i) {
    if (i == L.channel_axis) continue;
    gp.Fi[s] = reinterpret_cast<const uint32_t*>(F.fac[s] + i0 * L.aw[s]);
    gp.Fj[s] = reinterpret_cast<const uint32_t*>(F.fac[s] + j0 * L.aw[s]);
    gp.fw[s] = static_cast<long long>(2 * L.aw[s]);
    gp.n[s] = static_cast<long long>(L.shape[i]);
    ++s;
  }
  SC_CUDA(ctx, scb::launch_gram(gp, ctx->stream));
  st->kernel_launches += 1;
  return SC_OK;
}

sc_status sqnorm(sc_ctx* ctx, const double* dx, uint64_t n, double* out, sc_op_stats* st) {
  void *part = nullptr, *res = nullptr;
  if (sc_status s = scb::pool_get(ctx, "sqnorm.part", 8 * 600, &part); s != SC_OK) return s;
  if (sc_status s = scb::pool_get(ctx, "sqnorm.out", 8, &res); s != SC_OK) return s;
  SC_CUDA(ctx, scb::launch_sqnorm(dx, static_cast<long long>(n), static_cast<double*>(part), static_cast<double*>(res),
                                  ctx->stream));
  st->kernel_launches += 2;
  SC_CUDA(ctx, cudaMemcpyAsync(out, res, 8, cudaMemcpyDeviceToHost, ctx->stream));
  SC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  st->d2h_bytes += 8;
  return SC_OK;
}

// Device copy of A (numel values of dtype) widened into f64 `dst`.
sc_status widen_into(sc_ctx* ctx, int dtype, const void* dA, uint64_t n, double* dst, sc_op_stats* st) {
  if (dtype == SC_F64) {
    SC_CUDA(ctx, cudaMemcpyAsync(dst, dA, n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    SC_CUDA(ctx, scb::launch_widen(static_cast<const float*>(dA), dst, static_cast<long long>(n), ctx->stream));
    st->kernel_launches += 1;
  }
  return SC_OK;
}

// ---------------------------------------------------------------------------
// Cholesky (gram.hpp:48-107), restated with the same loop order so the
// coefficients are bit-identical for an identical system
// ---------------------------------------------------------------------------
bool cholesky(std::vector<double>& m, size_t n) {
  for (size_t j = 0; j < n; ++j) {
    double d = m[j * n + j];
    for (size_t p = 0; p < j; ++p) d -= m[j * n + p] * m[j * n + p];
    if (!(d > 0.0) || !std::isfinite(d)) return false;
    const double l = std::sqrt(d);
    m[j * n + j] = l;
    for (size_t i = j + 1; i < n; ++i) {
      double v = m[i * n + j];
      for (size_t p = 0; p < j; ++p) v -= m[i * n + p] * m[j * n + p];
      m[i * n + j] = v / l;
    }
  }
  return true;
}

void cholesky_solve(const std::vector<double>& l, size_t n, double* x) {
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

bool solve_gram(size_t w, size_t ch, const double* gram, const double* rhs, double* out) {
  if (w == 0) return true;
  const double base_ridge = 1e-10 * gram[0];
  std::vector<double> factor;
  bool ok = false;
  for (int attempt = 0; attempt < 5 && !ok; ++attempt) {
    factor.assign(gram, gram + w * w);
    if (attempt > 0) {
      const double ridge = base_ridge * static_cast<double>(1 << (attempt - 1));
      for (size_t j = 0; j < w; ++j) factor[j * w + j] += ridge;
    }
    ok = cholesky(factor, w);
  }
  if (!ok) return false;
  std::vector<double> x(w);
  for (size_t c = 0; c < ch; ++c) {
    for (size_t j = 0; j < w; ++j) x[j] = rhs[j * ch + c];
    cholesky_solve(factor, w, x.data());
    for (size_t j = 0; j < w; ++j) out[j * ch + c] = x[j];
  }
  return true;
}

// ---------------------------------------------------------------------------
// Incremental form of the same factorisation for the term-by-term solves of
// lstsq_decompose (decompose.hpp:434-469 calls solve_gram afresh for every leading
// block: O(k^3) per term).  In the reference's left-looking column order, entry
// L[i][j] depends only on G[i][j] and on rows i and j of L to the left of column j,
// so the factor of the bordered system keeps every earlier row bit for bit and gains
// one row, computed here by the very same operations in the very same order: O(k^2)
// per term, identical coefficients.  Lower triangle packed by rows.  A failed pivot
// (ridge retry needed) hands the system back to solve_gram.
struct IncCholesky {
  std::vector<double> l;  // packed rows: row i at i (i + 1) / 2
  size_t n = 0;
  bool valid = true;
  static size_t at(size_t i) { return i * (i + 1) / 2; }
  // col: Gram column of the new term against terms 0..n (col[n] = its diagonal)
  bool append(const double* col) {
    const size_t i = n;
    l.resize(at(i + 1));
    double* ri = l.data() + at(i);
    for (size_t j = 0; j < i; ++j) {
      const double* rj = l.data() + at(j);
      double v = col[j];
      for (size_t p = 0; p < j; ++p) v -= ri[p] * rj[p];
      ri[j] = v / rj[j];
    }
    double d = col[i];
    for (size_t p = 0; p < i; ++p) d -= ri[p] * ri[p];
    if (!(d > 0.0) || !std::isfinite(d)) {
      l.resize(at(i));
      valid = false;
      return false;
    }
    ri[i] = std::sqrt(d);
    n = i + 1;
    return true;
  }
  void solve(double* x) const {  // cholesky_solve on the packed factor
    for (size_t i = 0; i < n; ++i) {
      const double* ri = l.data() + at(i);
      double v = x[i];
      for (size_t p = 0; p < i; ++p) v -= ri[p] * x[p];
      x[i] = v / ri[i];
    }
    for (size_t i = n; i-- > 0;) {
      double v = x[i];
      for (size_t p = i + 1; p < n; ++p) v -= l[at(p) + i] * x[p];
      x[i] = v / l[at(i) + i];
    }
  }
};

// gram_quadratic (decompose.hpp:397-410)
double gram_quadratic(size_t w, size_t ch, const double* gram, const double* rhs, const double* c) {
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

// A on the device in its own dtype (uploaded when it is host memory)
sc_status device_input(sc_ctx* ctx, int dtype, const void* a, int on_device, uint64_t numel, const void** dA,
                       sc_op_stats* st) {
  if (on_device) {
    *dA = a;
    return SC_OK;
  }
  const size_t bytes = numel * (dtype == SC_F32 ? 4 : 8);
  void* p = nullptr;
  if (sc_status s = scb::pool_get(ctx, "input.A", bytes, &p); s != SC_OK) return s;
  SC_CUDA(ctx, cudaMemcpyAsync(p, a, bytes, cudaMemcpyHostToDevice, ctx->stream));
  st->h2d_bytes += bytes;
  *dA = p;
  return SC_OK;
}

// ---------------------------------------------------------------------------
// byte containers (io.hpp)
// ---------------------------------------------------------------------------
struct Writer {
  uint8_t* out;
  uint64_t cap, pos = 0;
  bool ok = true;
  void bytes(const void* p, size_t n) {
    if (pos + n > cap) {
      ok = false;
      return;
    }
    std::memcpy(out + pos, p, n);
    pos += n;
  }
  void u8(uint8_t v) { bytes(&v, 1); }
  void u64le(uint64_t v) {
    uint8_t b[8];
    for (int i = 0; i < 8; ++i) b[i] = static_cast<uint8_t>(v >> (8 * i));
    bytes(b, 8);
  }
  void u32le(uint32_t v) {
    uint8_t b[4];
    for (int i = 0; i < 4; ++i) b[i] = static_cast<uint8_t>(v >> (8 * i));
    bytes(b, 4);
  }
  void f64le(double v) {
    uint64_t u;
    std::memcpy(&u, &v, 8);
    u64le(u);
  }
  void f32le(float v) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    u32le(u);
  }
};

struct io_fail {
  std::string what;
};

struct Reader {
  const uint8_t* in;
  uint64_t size, pos = 0;
  void bytes(void* p, size_t n) {  // get_bytes, io.hpp:33-36
    if (pos + n > size) throw io_fail{"truncated payload"};
    std::memcpy(p, in + pos, n);
    pos += n;
  }
  uint8_t u8() {
    uint8_t v;
    bytes(&v, 1);
    return v;
  }
  uint64_t u64le() {
    uint8_t b[8];
    bytes(b, 8);
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
    return v;
  }
  uint32_t u32le() {
    uint8_t b[4];
    bytes(b, 4);
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(b[i]) << (8 * i);
    return v;
  }
  double f64le() {
    const uint64_t u = u64le();
    double v;
    std::memcpy(&v, &u, 8);
    return v;
  }
  float f32le() {
    const uint32_t u = u32le();
    float v;
    std::memcpy(&v, &u, 4);
    return v;
  }
};

uint64_t column_bytes(uint64_t len) { return (len + 7) / 8; }

// put_sign_column, io.hpp:82-92
void put_sign_column(Writer& w, const uint64_t* words, uint64_t len) {
  uint64_t remaining = column_bytes(len);
  for (uint64_t u = 0; remaining > 0; ++u) {
    const uint64_t take = std::min<uint64_t>(8, remaining);
    uint8_t b[8];
    for (uint64_t i = 0; i < take; ++i) b[i] = static_cast<uint8_t>(words[u] >> (8 * i));
    w.bytes(b, take);
    remaining -= take;
  }
}

// get_sign_column, io.hpp:94-109 (pad bits beyond len must be zero)
void get_sign_column(Reader& r, uint64_t len, uint64_t* words) {
  const uint64_t nw = words64(len);
  std::fill(words, words + nw, 0);
  uint64_t remaining = column_bytes(len);
  for (uint64_t u = 0; u < nw && remaining > 0; ++u) {
    const uint64_t take = std::min<uint64_t>(8, remaining);
    uint8_t b[8] = {};
    r.bytes(b, take);
    for (uint64_t i = 0; i < take; ++i) words[u] |= static_cast<uint64_t>(b[i]) << (8 * i);
    remaining -= take;
  }
  const uint64_t tail = len % 64;
  if (tail != 0 && (words[nw - 1] >> tail) != 0) throw io_fail{"sign column has nonzero pad bits"};
}

struct ScdHeader {
  int order = 0, channel_axis = -1, coeff_bits = 64;
  uint64_t shape[SC_MAX_ORDER] = {};
  uint64_t width = 0;
};

// read_scd header part, io.hpp:168-194
ScdHeader read_scd_header(Reader& r) {
  char magic[4];
  r.bytes(magic, 4);
  if (std::memcmp(magic, "SCD1", 4) != 0) throw io_fail{"bad SCD magic"};
  ScdHeader h;
  const int k = r.u8();
  if (k == 0) throw io_fail{"SCD order must be >= 1"};
  const uint8_t mode = r.u8();
  if (mode > 1) throw io_fail{"bad SCD channel mode"};
  if (mode == 1) {
    h.channel_axis = r.u8();
    if (h.channel_axis >= k) throw io_fail{"SCD channel axis out of range"};
  }
  if (k > SC_MAX_ORDER) throw io_fail{"SCD order above this build's limit (8)"};
  h.order = k;
  uint64_t numel = 1;
  bool overflow = false;
  for (int i = 0; i < k; ++i) {
    h.shape[i] = r.u64le();
    if (h.shape[i] == 0) throw io_fail{"bad SCD shape"};
    if (h.shape[i] > UINT64_MAX / numel) overflow = true;
    else numel *= h.shape[i];
  }
  if (overflow) throw io_fail{"SCD shape overflow"};
  h.width = r.u64le();
  h.coeff_bits = r.u8();
  if (h.coeff_bits != 32 && h.coeff_bits != 64) throw io_fail{"bad SCD coefficient width"};
  return h;
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------------------
// expansion
// ---------------------------------------------------------------------------
sc_status sc_accumulate_expansion(sc_ctx* ctx, const sc_factors* d, double scale, uint64_t first_term,
                                  uint64_t last_term, double* data, int32_t data_on_device, int32_t zero_fill,
                                  sc_op_stats* stats) {
  if (ctx == nullptr) return SC_INVALID_ARGUMENT;
  Timer tm;
  Layout L;
  if (sc_status s = check_factors(ctx, d, &L); s != SC_OK) return s;
  if (data == nullptr) return set_err(ctx, SC_INVALID_ARGUMENT, "sc_accumulate_expansion: null data");
  last_term = std::min<uint64_t>(last_term, d->width);
  const uint64_t nterms = last_term > first_term ? last_term - first_term : 0;
  SC_CUDA(ctx, cudaSetDevice(ctx->device));
  sc_op_stats st{};
  DevFactors F;
  if (sc_status s = alloc_factors(ctx, L, nterms, "exp", &F); s != SC_OK) return s;
  void *dcoef = nullptr, *dd = data;
  if (sc_status s = scb::pool_get(ctx, "exp.coef", std::max<uint64_t>(1, nterms * L.nch) * 8, &dcoef); s != SC_OK)
    return s;
  const size_t dbytes = L.numel * 8;
  if (!data_on_device)
    if (sc_status s = scb::pool_get(ctx, "exp.data", dbytes, &dd); s != SC_OK) return s;
  double* ddata = static_cast<double*>(dd);
  if (zero_fill) {
    SC_CUDA(ctx, cudaMemsetAsync(ddata, 0, dbytes, ctx->stream));
  } else if (!data_on_device) {
    SC_CUDA(ctx, cudaMemcpyAsync(ddata, data, dbytes, cudaMemcpyHostToDevice, ctx->stream));
    st.h2d_bytes += dbytes;
  }
  if (nterms) {
    if (sc_status s = upload_factors(ctx, L, d->sign_words, first_term, 0, nterms, F, &st); s != SC_OK) return s;
    const size_t cb = nterms * L.nch * 8;
    SC_CUDA(ctx, cudaMemcpyAsync(dcoef, d->coefficients + first_term * L.nch, cb, cudaMemcpyHostToDevice,
                                 ctx->stream));
    st.h2d_bytes += cb;
    const scb::ExpandParams ep = expand_params(L, F, 0, nterms, static_cast<double*>(dcoef), scale, ddata);
    SC_CUDA(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    SC_CUDA(ctx, scb::launch_expand(ep, ctx->stream));
    SC_CUDA(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
    st.kernel_launches += 1;
  }
  if (!data_on_device) {
    SC_CUDA(ctx, cudaMemcpyAsync(data, ddata, dbytes, cudaMemcpyDeviceToHost, ctx->stream));
    st.d2h_bytes += dbytes;
  }
  SC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (nterms) {
    float ms = 0.f;
    SC_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    st.kernel_ms = ms;
  }
  st.total_ms = tm.ms();
  add_stats(stats, st);
  return SC_OK;
}

// ---------------------------------------------------------------------------
// Gram system and contractions
// ---------------------------------------------------------------------------
sc_status sc_gram_matrix(sc_ctx* ctx, const sc_factors* d, double* gram, sc_op_stats* stats) {
  if (ctx == nullptr) return SC_INVALID_ARGUMENT;
  Timer tm;
  Layout L;
  if (sc_status s = check_factors(ctx, d, &L); s != SC_OK) return s;
  if (gram == nullptr && d->width > 0) return set_err(ctx, SC_INVALID_ARGUMENT, "sc_gram_matrix: null output");
  const uint64_t w = d->width;
  if (w == 0) return SC_OK;
  SC_CUDA(ctx, cudaSetDevice(ctx->device));
  sc_op_stats st{};
  DevFactors F;
  if (sc_status s = alloc_factors(ctx, L, w, "gram", &F); s != SC_OK) return s;
  void* dG = nullptr;
  if (sc_status s = scb::pool_get(ctx, "gram.G", w * w * 8, &dG); s != SC_OK) return s;
  if (sc_status s = upload_factors(ctx, L, d->sign_words, 0, 0, w, F, &st); s != SC_OK) return s;
  SC_CUDA(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
  if (sc_status s = gram_block(ctx, L, F, 0, w, 0, w, static_cast<double*>(dG), static_cast<long long>(w), &st);
      s != SC_OK)
    return s;
  SC_CUDA(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
  SC_CUDA(ctx, cudaMemcpyAsync(gram, dG, w * w * 8, cudaMemcpyDeviceToHost, ctx->stream));
  st.d2h_bytes += w * w * 8;
  SC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  float ms = 0.f;
  SC_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  st.kernel_ms = ms;
  st.total_ms = tm.ms();
  add_stats(stats, st);
  return SC_OK;
}

sc_status sc_contract_terms(sc_ctx* ctx, const sc_factors* d, int32_t a_dtype, const void* a, int32_t a_on_device,
                            uint64_t first_term, uint64_t count, double* rhs, sc_op_stats* stats) {
  if (ctx == nullptr) return SC_INVALID_ARGUMENT;
  Timer tm;
  Layout L;
  if (sc_status s = check_factors(ctx, d, &L); s != SC_OK) return s;
  if (a == nullptr || (rhs == nullptr && count > 0))
    return set_err(ctx, SC_INVALID_ARGUMENT, "sc_contract_terms: null input or output");
  if (a_dtype != SC_F32 && a_dtype != SC_F64) return set_err(ctx, SC_INVALID_ARGUMENT, "sc_contract_terms: bad dtype");
  if (first_term + count > d->width) return set_err(ctx, SC_INVALID_ARGUMENT, "sc_contract_terms: term range");
  if (L.chan != 0 && L.nch > 8)
    return set_err(ctx, SC_NOT_SUPPORTED, "sc_contract_terms: at most 8 channel slices");
  if (count == 0) return SC_OK;
  SC_CUDA(ctx, cudaSetDevice(ctx->device));
  sc_op_stats st{};
  DevFactors F;
  if (sc_status s = alloc_factors(ctx, L, count, "ctr", &F); s != SC_OK) return s;
  if (sc_status s = upload_factors(ctx, L, d->sign_words, first_term, 0, count, F, &st); s != SC_OK) return s;
  const void* dA = nullptr;
  if (sc_status s = device_input(ctx, a_dtype, a, a_on_device, L.numel, &dA, &st); s != SC_OK) return s;
  SC_CUDA(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
  if (sc_status s = contract(ctx, L, F, 0, count, a_dtype, dA, rhs, &st); s != SC_OK) return s;
  SC_CUDA(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
  SC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  float ms = 0.f;
  SC_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  st.kernel_ms = ms;
  st.total_ms = tm.ms();
  add_stats(stats, st);
  return SC_OK;
}

sc_status sc_solve_gram_leading(uint64_t width, uint64_t channels, const double* gram, const double* rhs, double* out,
                                char* msg, size_t msg_len) {
  if ((width > 0 && (gram == nullptr || rhs == nullptr || out == nullptr)) || channels == 0)
    return put_msg(msg, msg_len, SC_INVALID_ARGUMENT, "sc_solve_gram_leading: null argument");
  IncCholesky chol;
  std::vector<double> col(width), x(width), blk;
  size_t off = 0;
  for (uint64_t k = 1; k <= width; ++k) {
    for (uint64_t j = 0; j < k; ++j) col[j] = gram[(k - 1) * width + j];
    double* o = out + off * channels;
    if (chol.valid && chol.append(col.data())) {
      for (uint64_t c = 0; c < channels; ++c) {
        for (uint64_t j = 0; j < k; ++j) x[j] = rhs[j * channels + c];
        chol.solve(x.data());
        for (uint64_t j = 0; j < k; ++j) o[j * channels + c] = x[j];
      }
    } else {
      blk.resize(k * k);
      for (uint64_t i = 0; i < k; ++i)
        for (uint64_t j = 0; j < k; ++j) blk[i * k + j] = gram[i * width + j];
      if (!solve_gram(k, channels, blk.data(), rhs, o))
        return put_msg(msg, msg_len, SC_RUNTIME_ERROR, "solve_gram: factorization failed");
    }
    off += k;
  }
  return SC_OK;
}

sc_status sc_solve_gram(uint64_t width, uint64_t channels, const double* gram, const double* rhs, double* out,
                        char* msg, size_t msg_len) {
  if (width == 0) return SC_OK;
  if (gram == nullptr || rhs == nullptr || out == nullptr || channels == 0)
    return put_msg(msg, msg_len, SC_INVALID_ARGUMENT, "sc_solve_gram: null argument");
  if (!solve_gram(width, channels, gram, rhs, out))
    return put_msg(msg, msg_len, SC_RUNTIME_ERROR, "solve_gram: factorization failed");
  return SC_OK;
}

sc_status sc_correct_coefficients(sc_ctx* ctx, const sc_factors* d, int32_t a_dtype, const void* a,
                                  int32_t a_on_device, double* coeffs_out, sc_op_stats* stats) {
  if (ctx == nullptr) return SC_INVALID_ARGUMENT;
  Layout L;
  if (sc_status s = check_factors(ctx, d, &L); s != SC_OK) return s;
  if (coeffs_out == nullptr) return set_err(ctx, SC_INVALID_ARGUMENT, "sc_correct_coefficients: null output");
  const uint64_t w = d->width;
  if (w == 0) return SC_OK;
  std::vector<double> gram(w * w), rhs(w * L.nch), solved(w * L.nch);
  if (sc_status s = sc_gram_matrix(ctx, d, gram.data(), stats); s != SC_OK) return s;
  if (sc_status s = sc_contract_terms(ctx, d, a_dtype, a, a_on_device, 0, w, rhs.data(), stats); s != SC_OK) return s;
  // correct_coefficients (decompose.hpp:418-428)
  if (!solve_gram(w, L.nch, gram.data(), rhs.data(), solved.data()))
    return set_err(ctx, SC_RUNTIME_ERROR, "solve_gram: factorization failed");
  const double q_new = gram_quadratic(w, L.nch, gram.data(), rhs.data(), solved.data());
  const double q_old = gram_quadratic(w, L.nch, gram.data(), rhs.data(), d->coefficients);
  const double* src = q_new <= q_old ? solved.data() : d->coefficients;
  std::copy(src, src + w * L.nch, coeffs_out);
  return SC_OK;
}

// ---------------------------------------------------------------------------
// least squares / scalar channels (decompose.hpp:434-469, :485-536)
// ---------------------------------------------------------------------------
sc_status sc_lstsq_decompose(sc_ctx* ctx, const sc_problem* p, int32_t channel_axis, sc_result* res) {
  if (ctx == nullptr) return SC_INVALID_ARGUMENT;
  Timer tm;
  if (res == nullptr) return set_err(ctx, SC_INVALID_ARGUMENT, "sc_result: null");
  // validation: DenseTensor / SearchConfig as sc_validate_problem, then the
  // driver's own checks with channels = q (check_decompose_config :290-298)
  {
    char m[256];
    sc_problem q = *p;
    q.max_factor_bytes = UINT64_MAX;  // the budget is re-checked below with the channel count
    if (sc_status s = sc_validate_problem(&q, m, sizeof m); s != SC_OK) return set_err(ctx, s, "%s", m);
  }
  const int k = p->order;
  int nch = 1;
  if (channel_axis >= 0) {
    if (k < 2) return set_err(ctx, SC_INVALID_ARGUMENT, "rgb_scalars_decompose: order >= 2 required");
    if (channel_axis >= k) return set_err(ctx, SC_INVALID_ARGUMENT, "rgb_scalars_decompose: channel axis out of range");
    if (p->shape[channel_axis] > 8) return set_err(ctx, SC_INVALID_ARGUMENT, "rgb_scalars_decompose: channel axis too long");
    nch = static_cast<int>(p->shape[channel_axis]);
  } else if (channel_axis != -1) {
    return set_err(ctx, SC_INVALID_ARGUMENT, "sc_lstsq_decompose: channel axis out of range");
  }
  {
    uint64_t per_term = static_cast<uint64_t>(nch) * sizeof(double);
    for (int i = 0; i < k; ++i) per_term += words64(p->shape[i]) * sizeof(uint64_t);
    if (p->width > 0 && per_term > p->max_factor_bytes / p->width)
      return set_err(ctx, SC_INVALID_ARGUMENT, "DecomposeConfig: width exceeds the factor memory budget");
  }
  Layout L;
  {
    std::string msg;
    if (sc_status s = make_layout(k, p->shape, channel_axis, &L, &msg); s != SC_OK)
      return set_err(ctx, s, "%s", msg.c_str());
  }
  for (int s = 0; s < L.nsign; ++s)
    if (res->sign_words[s] == nullptr)
      return set_err(ctx, SC_INVALID_ARGUMENT, "sc_result: sign_words of every sign axis are required");
  if (res->cut_value == nullptr || (res->alpha == nullptr && p->width > 0))
    return set_err(ctx, SC_INVALID_ARGUMENT, "sc_result: alpha and cut_value are required");
  SC_CUDA(ctx, cudaSetDevice(ctx->device));
  sc_op_stats st{};
  const uint64_t w = p->width;
  const uint64_t n = L.numel;

  const void* dA = nullptr;
  if (sc_status s = device_input(ctx, p->dtype, p->data, p->data_on_device, n, &dA, &st); s != SC_OK) return s;
  void *vR = nullptr, *vcoef = nullptr;
  if (sc_status s = scb::pool_get(ctx, "lsq.R", n * 8, &vR); s != SC_OK) return s;
  if (sc_status s = scb::pool_get(ctx, "lsq.coef", std::max<uint64_t>(1, w * nch) * 8, &vcoef); s != SC_OK) return s;
  double* dR = static_cast<double*>(vR);
  double* dcoef = static_cast<double*>(vcoef);
  DevFactors F;
  if (sc_status s = alloc_factors(ctx, L, std::max<uint64_t>(w, 1), "lsq", &F); s != SC_OK) return s;
  void* vcol = nullptr;
  if (sc_status s = scb::pool_get(ctx, "lsq.gcol", std::max<uint64_t>(w, 1) * 8, &vcol); s != SC_OK) return s;
  double* dcol = static_cast<double*>(vcol);

  // residual = a; input norm (frobenius_norm)
  if (sc_status s = widen_into(ctx, p->dtype, dA, n, dR, &st); s != SC_OK) return s;
  double sq = 0.0;
  if (sc_status s = sqnorm(ctx, dR, n, &sq, &st); s != SC_OK) return s;
  res->input_norm = std::sqrt(sq);
  res->final_residual_norm = res->input_norm;

  // the single-cut search of every term runs on the engine's persistent kernel
  std::vector<std::vector<uint64_t>> cut_words(k);
  for (int i = 0; i < k; ++i) cut_words[i].assign(words64(p->shape[i]), 0);
  std::vector<double> gram, rhs;  // GramSystem (gram.hpp:17-43)
  std::vector<double> coef;
  IncCholesky chol;
  size_t gw = 0;
  double first_value = 0.0;
  uint64_t done = 0;
  uint64_t passes = 0;
  double kernel_ms = 0.0;
  int launches = 0;  // search kernels (the aux kernels count in st)
  for (uint64_t term = 0; term < w; ++term) {
    sc_problem q{};
    q.dtype = SC_F64;
    q.order = k;
    q.shape = p->shape;
    q.data = dR;
    q.data_on_device = 1;
    q.seed_mode = SC_SEED_DIRECT;
    q.width = 1;
    q.flush_width = 1;
    q.seed = scb::substream(p->seed, term);  // term_search_config, decompose.hpp:300-304
    q.restarts = p->restarts;
    q.max_sweeps = p->max_sweeps;
    q.min_value_fraction = 0.0;
    q.max_factor_bytes = UINT64_MAX;
    sc_result r{};
    for (int i = 0; i < k; ++i) r.sign_words[i] = cut_words[i].data();
    double cv = 0.0, al = 0.0;
    uint32_t sw = 0;
    r.cut_value = &cv;
    r.alpha = &al;
    r.sweeps = &sw;
    if (sc_status s = sc_greedy_decompose(ctx, &q, &r); s != SC_OK) return s;
    kernel_ms += r.kernel_ms;
    launches += r.kernel_launches;
    passes += r.passes;
    st.h2d_bytes += r.h2d_bytes;
    st.d2h_bytes += r.d2h_bytes;
    if (term == 0) {
      first_value = cv;
    } else if (cv < p->min_value_fraction * first_value) {
      break;
    }
    // keep the signs of the sign axes (the channel sign is dropped, :516-520)
    std::vector<const uint64_t*> host_new(SC_MAX_ORDER, nullptr);
    for (int i = 0, s = 0; i < k; ++i) {
      if (i == channel_axis) continue;
      std::memcpy(res->sign_words[s] + term * L.aw[s], cut_words[i].data(), L.aw[s] * 8);
      host_new[s] = cut_words[i].data();
      ++s;
    }
    if (sc_status s = upload_factors(ctx, L, host_new.data(), 0, term, 1, F, &st); s != SC_OK) return s;
    // Gram column of the new term against every kept term + diagonal (gram_column)
    if (sc_status s = gram_block(ctx, L, F, 0, term + 1, term, 1, dcol, 1, &st); s != SC_OK) return s;
    std::vector<double> col(term + 1), rb(nch);
    SC_CUDA(ctx, cudaMemcpyAsync(col.data(), dcol, (term + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    st.d2h_bytes += (term + 1) * 8;
    // rhs block: contract_term(a, channel_axis, signs)
    if (sc_status s = contract(ctx, L, F, term, 1, p->dtype, dA, rb.data(), &st); s != SC_OK) return s;
    // GramSystem::extend (gram.hpp:28-42); rows at a fixed stride w, so a term costs O(k)
    // here (the compact k x k copy is made only if the ridge retry is needed)
    if (gram.empty()) gram.assign(static_cast<size_t>(w) * w, 0.0);
    for (size_t i = 0; i < gw; ++i) {
      gram[i * w + gw] = col[i];
      gram[gw * w + i] = col[i];
    }
    gram[gw * w + gw] = col[gw];
    rhs.insert(rhs.end(), rb.begin(), rb.end());
    ++gw;
    coef.assign(gw * nch, 0.0);
    // the factor grows by one row per term (identical to solve_gram of the whole system);
    // once a pivot fails, solve_gram with its ridge retries takes over for good
    if (chol.valid && chol.append(col.data())) {
      std::vector<double> x(gw);
      for (int c = 0; c < nch; ++c) {
        for (size_t j = 0; j < gw; ++j) x[j] = rhs[j * nch + c];
        chol.solve(x.data());
        for (size_t j = 0; j < gw; ++j) coef[j * nch + c] = x[j];
      }
    } else {
      std::vector<double> blk(gw * gw);
      for (size_t i = 0; i < gw; ++i)
        for (size_t j = 0; j < gw; ++j) blk[i * gw + j] = gram[i * w + j];
      if (!solve_gram(gw, nch, blk.data(), rhs.data(), coef.data()))
        return set_err(ctx, SC_RUNTIME_ERROR, "solve_gram: factorization failed");
    }
    // residual = a - expand(d) with the re-solved coefficients
    SC_CUDA(ctx, cudaMemcpyAsync(dcoef, coef.data(), gw * nch * 8, cudaMemcpyHostToDevice, ctx->stream));
    st.h2d_bytes += gw * nch * 8;
    if (sc_status s = widen_into(ctx, p->dtype, dA, n, dR, &st); s != SC_OK) return s;
    const scb::ExpandParams ep = expand_params(L, F, 0, gw, dcoef, -1.0, dR);
    SC_CUDA(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    SC_CUDA(ctx, scb::launch_expand(ep, ctx->stream));
    SC_CUDA(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
    st.kernel_launches += 1;
    if (sc_status s = sqnorm(ctx, dR, n, &sq, &st); s != SC_OK) return s;
    float ms = 0.f;
    SC_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    kernel_ms += ms;
    res->final_residual_norm = std::sqrt(sq);
    res->cut_value[term] = cv;
    if (res->resid_norm) res->resid_norm[term] = res->final_residual_norm;
    if (res->resid_norm_exact) res->resid_norm_exact[term] = res->final_residual_norm;
    if (res->sweeps) res->sweeps[term] = sw;
    done = term + 1;
  }
  if (done > 0) std::memcpy(res->alpha, coef.data(), done * nch * 8);
  if (res->remainder) {
    if (p->dtype == SC_F64) {
      SC_CUDA(ctx, cudaMemcpyAsync(res->remainder, dR, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
      SC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    } else {
      std::vector<double> tmp(n);
      SC_CUDA(ctx, cudaMemcpyAsync(tmp.data(), dR, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
      SC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      float* o = static_cast<float*>(res->remainder);
      for (uint64_t i = 0; i < n; ++i) o[i] = static_cast<float>(tmp[i]);
    }
    st.d2h_bytes += n * 8;
  }
  res->width_done = done;
  res->passes = passes;
  res->kernel_ms = kernel_ms;
  res->kernel_launches = launches + st.kernel_launches;
  res->h2d_bytes = st.h2d_bytes;
  res->d2h_bytes = st.d2h_bytes;
  res->total_ms = tm.ms();
  return SC_OK;
}

// ---------------------------------------------------------------------------
// SCD (io.hpp:113-213)
// ---------------------------------------------------------------------------
uint64_t sc_scd_size(const sc_factors* d, int coeff_bits) {
  if (d == nullptr || d->shape == nullptr || d->order < 1 || d->order > SC_MAX_ORDER) return 0;
  // scd_file_size, io.hpp:135-140
  uint64_t header = 4 + 1 + 1 + (d->channel_axis >= 0 ? 1 : 0) + 8 * static_cast<uint64_t>(d->order) + 8 + 1;
  const uint64_t ch = d->channel_axis >= 0 ? d->shape[d->channel_axis] : 1;
  uint64_t per_term = ch * static_cast<uint64_t>(coeff_bits) / 8;
  for (int i = 0; i < d->order; ++i)
    if (i != d->channel_axis) per_term += column_bytes(d->shape[i]);
  return header + d->width * per_term;
}

sc_status sc_write_scd(const sc_factors* d, int coeff_bits, uint8_t* out, uint64_t capacity, uint64_t* written,
                       char* msg, size_t msg_len) {
  if (coeff_bits != 32 && coeff_bits != 64)
    return put_msg(msg, msg_len, SC_INVALID_ARGUMENT, "write_scd: coeff_bits must be 32 or 64");
  Layout L;
  std::string m;
  if (d == nullptr) return put_msg(msg, msg_len, SC_INVALID_ARGUMENT, "sc_factors: null");
  if (sc_status s = make_layout(d->order, d->shape, d->channel_axis, &L, &m); s != SC_OK)
    return put_msg(msg, msg_len, s, m);
  // CutDecomposition::validate (decompose.hpp:79-97)
  for (uint64_t i = 0; i < d->width * L.nch; ++i)
    if (!std::isfinite(d->coefficients[i]))
      return put_msg(msg, msg_len, SC_INVALID_ARGUMENT, "CutDecomposition: non-finite coefficient");
  if (out == nullptr || capacity < sc_scd_size(d, coeff_bits))
    return put_msg(msg, msg_len, SC_INVALID_ARGUMENT, "sc_write_scd: output buffer too small");
  Writer wr{out, capacity};
  wr.bytes("SCD1", 4);
  wr.u8(static_cast<uint8_t>(d->order));
  wr.u8(d->channel_axis >= 0 ? 1 : 0);
  if (d->channel_axis >= 0) wr.u8(static_cast<uint8_t>(d->channel_axis));
  for (int i = 0; i < d->order; ++i) wr.u64le(d->shape[i]);
  wr.u64le(d->width);
  wr.u8(static_cast<uint8_t>(coeff_bits));
  for (uint64_t j = 0; j < d->width; ++j) {
    const double* c = d->coefficients + j * L.nch;
    for (int ch = 0; ch < L.nch; ++ch) {
      if (coeff_bits == 64)
        wr.f64le(c[ch]);
      else
        wr.f32le(static_cast<float>(c[ch]));  // documented lossy narrowing (io.hpp:161)
    }
    for (int i = 0, s = 0; i < d->order; ++i) {
      if (i == d->channel_axis) continue;
      put_sign_column(wr, d->sign_words[s] + j * L.aw[s], d->shape[i]);
      ++s;
    }
  }
  if (!wr.ok) return put_msg(msg, msg_len, SC_IO_ERROR, "write failed");
  if (written) *written = wr.pos;
  return SC_OK;
}

sc_status sc_read_scd_header(const uint8_t* in, uint64_t size, int32_t* order, uint64_t* shape,
                             int32_t* channel_axis, uint64_t* width, int32_t* coeff_bits, char* msg, size_t msg_len) {
  if (in == nullptr && size > 0) return put_msg(msg, msg_len, SC_INVALID_ARGUMENT, "sc_read_scd_header: null input");
  try {
    Reader r{in, size};
    const ScdHeader h = read_scd_header(r);
    if (order) *order = h.order;
    if (shape)
      for (int i = 0; i < h.order; ++i) shape[i] = h.shape[i];
    if (channel_axis) *channel_axis = h.channel_axis;
    if (width) *width = h.width;
    if (coeff_bits) *coeff_bits = h.coeff_bits;
  } catch (const io_fail& e) {
    return put_msg(msg, msg_len, SC_IO_ERROR, e.what);
  }
  return SC_OK;
}

sc_status sc_read_scd(const uint8_t* in, uint64_t size, uint64_t** sign_words, double* coefficients, char* msg,
                      size_t msg_len) {
  try {
    Reader r{in, size};
    const ScdHeader h = read_scd_header(r);
    const uint64_t q = h.channel_axis >= 0 ? h.shape[h.channel_axis] : 1;
    for (uint64_t j = 0; j < h.width; ++j) {
      for (uint64_t ch = 0; ch < q; ++ch) {
        const double c = h.coeff_bits == 64 ? r.f64le() : static_cast<double>(r.f32le());
        if (!std::isfinite(c)) throw io_fail{"non-finite SCD coefficient"};
        coefficients[j * q + ch] = c;
      }
      for (int i = 0, s = 0; i < h.order; ++i) {
        if (i == h.channel_axis) continue;
        get_sign_column(r, h.shape[i], sign_words[s] + j * words64(h.shape[i]));
        ++s;
      }
    }
  } catch (const io_fail& e) {
    return put_msg(msg, msg_len, SC_IO_ERROR, e.what);
  }
  return SC_OK;
}

// ---------------------------------------------------------------------------
// DTEN (io.hpp:215-292)
// ---------------------------------------------------------------------------
uint64_t sc_dten_size(int32_t order, const uint64_t* shape, int32_t raw_dtype) {
  if (order < 1 || shape == nullptr) return 0;
  uint64_t numel = 1;
  for (int i = 0; i < order; ++i) numel *= shape[i];
  const uint64_t es = raw_dtype == 0 ? 8 : raw_dtype == 1 ? 4 : 1;
  return 4 + 1 + 8 * static_cast<uint64_t>(order) + 1 + numel * es;
}

sc_status sc_write_dten(int32_t order, const uint64_t* shape, const double* data, int32_t raw_dtype, uint8_t* out,
                        uint64_t capacity, uint64_t* written, char* msg, size_t msg_len) {
  if (order < 1 || order > 255 || shape == nullptr || data == nullptr)
    return put_msg(msg, msg_len, SC_INVALID_ARGUMENT, "sc_write_dten: bad tensor");
  if (raw_dtype < 0 || raw_dtype > 2) return put_msg(msg, msg_len, SC_INVALID_ARGUMENT, "sc_write_dten: bad dtype");
  if (out == nullptr || capacity < sc_dten_size(order, shape, raw_dtype))
    return put_msg(msg, msg_len, SC_INVALID_ARGUMENT, "sc_write_dten: output buffer too small");
  Writer wr{out, capacity};
  wr.bytes("DTEN", 4);
  wr.u8(static_cast<uint8_t>(order));
  uint64_t numel = 1;
  for (int i = 0; i < order; ++i) {
    wr.u64le(shape[i]);
    numel *= shape[i];
  }
  wr.u8(static_cast<uint8_t>(raw_dtype));
  for (uint64_t e = 0; e < numel; ++e) {
    const double v = data[e];
    if (raw_dtype == 0) {
      wr.f64le(v);
    } else if (raw_dtype == 1) {
      wr.f32le(static_cast<float>(v));
    } else {
      const long rr = std::lround(std::clamp(v, 0.0, 255.0));
      wr.u8(static_cast<uint8_t>(rr));
    }
  }
  if (!wr.ok) return put_msg(msg, msg_len, SC_IO_ERROR, "write failed");
  if (written) *written = wr.pos;
  return SC_OK;
}

namespace {
struct DtenHeader {
  int order = 0, dtype = 0;
  uint64_t shape[SC_MAX_ORDER] = {};
  uint64_t numel = 1;
};
DtenHeader read_dten_header(Reader& r) {
  char magic[4];
  r.bytes(magic, 4);
  if (std::memcmp(magic, "DTEN", 4) != 0) throw io_fail{"bad DTEN magic"};
  DtenHeader h;
  const int k = r.u8();
  if (k == 0) throw io_fail{"DTEN order must be >= 1"};
  if (k > SC_MAX_ORDER) throw io_fail{"DTEN order above this build's limit (8)"};
  h.order = k;
  bool overflow = false;
  for (int i = 0; i < k; ++i) {
    h.shape[i] = r.u64le();
    if (h.shape[i] == 0) throw io_fail{"DTEN zero-length axis"};
    if (h.shape[i] > UINT64_MAX / h.numel) overflow = true;
    else h.numel *= h.shape[i];
  }
  if (overflow) throw io_fail{"DTEN shape overflow"};
  h.dtype = r.u8();
  if (h.dtype > 2) throw io_fail{"bad DTEN dtype"};
  return h;
}
}  // namespace

sc_status sc_read_dten_header(const uint8_t* in, uint64_t size, int32_t* order, uint64_t* shape, int32_t* raw_dtype,
                              char* msg, size_t msg_len) {
  try {
    Reader r{in, size};
    const DtenHeader h = read_dten_header(r);
    if (order) *order = h.order;
    if (shape)
      for (int i = 0; i < h.order; ++i) shape[i] = h.shape[i];
    if (raw_dtype) *raw_dtype = h.dtype;
  } catch (const io_fail& e) {
    return put_msg(msg, msg_len, SC_IO_ERROR, e.what);
  }
  return SC_OK;
}

sc_status sc_read_dten(const uint8_t* in, uint64_t size, double* data, char* msg, size_t msg_len) {
  try {
    Reader r{in, size};
    const DtenHeader h = read_dten_header(r);
    for (uint64_t e = 0; e < h.numel; ++e) {
      if (h.dtype == 0)
        data[e] = r.f64le();
      else if (h.dtype == 1)
        data[e] = static_cast<double>(r.f32le());
      else
        data[e] = static_cast<double>(r.u8());
    }
    for (uint64_t e = 0; e < h.numel; ++e)
      if (!std::isfinite(data[e])) throw io_fail{"invalid DTEN payload: DenseTensor: non-finite value"};
  } catch (const io_fail& e) {
    return put_msg(msg, msg_len, SC_IO_ERROR, e.what);
  }
  return SC_OK;
}

}  // extern "C"
