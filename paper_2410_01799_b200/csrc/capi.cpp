// capi.cpp -- host driver behind the C ABI (include/sigcut_b200.h).
//
// Owns the CUDA context/stream, validates problems with the reference's error
// semantics, draws the per-cut start vectors with the reference's generator,
// lays the remainder out in HBM (row pitch padded to 32 elements, pad zero),
// sizes the shared-memory residency / TMA ring for the persistent kernel,
// launches it cooperatively and rebuilds the reference's CutReport curve.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <thread>
#include <string>
#include <vector>

#include "../../include/sigcut_b200.h"
#include "ctx.h"
#include "rng.h"
#include "sweep.h"


namespace {

using scb::set_err;

constexpr const char* kVersion = "sigcut-b200 0.1 (sm_100a)";


uint64_t words64(uint64_t n) { return (n + 63) / 64; }

sc_status validate(const sc_problem* p, std::string* msg) {
  auto bad = [&](const char* m) {
    if (msg) *msg = m;
    return SC_INVALID_ARGUMENT;
  };
  if (p == nullptr) return bad("sc_problem: null");
  if (p->dtype != SC_F32 && p->dtype != SC_F64) return bad("sc_problem: dtype must be F32 or F64");
  // DenseTensor::checked_numel, dense_tensor.hpp:57-67
  if (p->order < 1 || p->order > SC_MAX_ORDER) return bad("DenseTensor: order must be >= 1");
  if (p->shape == nullptr) return bad("sc_problem: null shape");
  uint64_t numel = 1;
  for (int i = 0; i < p->order; ++i) {
    if (p->shape[i] == 0) return bad("DenseTensor: zero-length axis");
    if (p->shape[i] > UINT64_MAX / numel) return bad("DenseTensor: shape overflow");
    numel *= p->shape[i];
  }
  if (p->data == nullptr) return bad("sc_problem: null data");
  // check_decompose_config, decompose.hpp:290-298
  if (p->flush_width < 1) return bad("DecomposeConfig: flush_width must be >= 1");
  uint64_t per_term = sizeof(double);
  for (int i = 0; i < p->order; ++i) per_term += words64(p->shape[i]) * sizeof(uint64_t);
  if (p->width > 0 && per_term > p->max_factor_bytes / p->width)
    return bad("DecomposeConfig: width exceeds the factor memory budget");
  // best_of_restarts, search.hpp:217-218
  if (p->restarts < 1) return bad("SearchConfig: restarts must be >= 1");
  if (p->max_sweeps < 1) return bad("SearchConfig: max_sweeps must be >= 1");
  if (p->seed_mode != SC_SEED_PER_TERM && p->seed_mode != SC_SEED_DIRECT)
    return bad("sc_problem: unknown seed_mode");
  return SC_OK;
}

uint64_t term_seed(const sc_problem* p, uint64_t term) {
  // term_search_config (decompose.hpp:300-304); greedy_signed_cut uses the seed as given
  if (p->seed_mode == SC_SEED_DIRECT && term == 0) return p->seed;
  return scb::substream(p->seed, term);
}

// Start vectors of (term, restart): the rng of best_of_restarts (search.hpp:222)
// draws s0 (discarded) then t0 for matrices (search.hpp:149-150), or one vector
// per axis for order k (search.hpp:197).
uint64_t start_vectors(const sc_problem* p, uint64_t term, uint64_t restart, uint64_t* out) {
  scb::Xoshiro rng(scb::substream(term_seed(p, term), restart));
  if (p->order == 2) {
    rng.skip(words64(p->shape[0]));
    rng.sign_words(p->shape[1], out);
    return words64(p->shape[1]);
  }
  uint64_t off = 0;
  for (int i = 0; i < p->order; ++i) {
    rng.sign_words(p->shape[i], out + off);
    off += words64(p->shape[i]);
  }
  return off;
}

template <typename T>
T* carve(char*& cur, size_t count) {
  T* p = reinterpret_cast<T*>(cur);
  cur += (count * sizeof(T) + 255) & ~size_t(255);
  return p;
}


}  // namespace

extern "C" {

const char* sc_version(void) { return kVersion; }
int sc_abi_version(void) { return SC_ABI_VERSION; }

sc_status sc_create(sc_ctx** out, int device) {
  if (out == nullptr) return SC_INVALID_ARGUMENT;
  *out = nullptr;
  auto* ctx = new sc_ctx();
  ctx->device = device;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0 || device < 0 || device >= ndev) {
    delete ctx;
    return SC_CUDA_ERROR;
  }
  cudaDeviceProp prop{};
  if (cudaSetDevice(device) != cudaSuccess || cudaGetDeviceProperties(&prop, device) != cudaSuccess ||
      prop.major != 10) {
    delete ctx;
    return SC_CUDA_ERROR;  // sm_100a kernels only; no fallback
  }
  ctx->num_sms = prop.multiProcessorCount;
  ctx->smem_optin = prop.sharedMemPerBlockOptin;
  ctx->smem_per_sm = prop.sharedMemPerMultiprocessor;
  ctx->l2_persist_max = static_cast<size_t>(prop.persistingL2CacheMaxSize);
  ctx->l2_window_max = static_cast<size_t>(prop.accessPolicyMaxWindowSize);
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess) {
    delete ctx;
    return SC_CUDA_ERROR;
  }
  *out = ctx;
  return SC_OK;
}

void sc_destroy(sc_ctx* ctx) {
  if (!ctx) return;
  sc_shard_close(ctx);
  cudaSetDevice(ctx->device);
  if (ctx->arena) cudaFree(ctx->arena);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  scb::pool_release(ctx);
  if (!ctx->borrowed) {
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
  }
  delete ctx;
}

const char* sc_last_error(const sc_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

sc_status sc_set_option(sc_ctx* ctx, const char* name, int64_t value) {
  if (ctx == nullptr || name == nullptr) return SC_INVALID_ARGUMENT;
  auto& o = ctx->opts;
  struct {
    const char* name;
    long long* field;
  } const table[] = {{"ctas", &o.ctas},           {"delta", &o.delta},         {"delta_div", &o.delta_div},
                     {"delta_refresh", &o.delta_refresh}, {"two_phase", &o.two_phase}, {"stages", &o.stages},
                     {"res_rows", &o.res_rows},   {"fuse_update", &o.fuse_update}, {"variant", &o.variant},
                     {"profile", &o.profile},     {"poison", &o.poison},       {"fast_delta", &o.fast_delta},
                     {"l2_persist", &o.l2_persist}};
  for (const auto& e : table)
    if (std::strcmp(e.name, name) == 0) {
      *e.field = value;
      return SC_OK;
    }
  return set_err(ctx, SC_INVALID_ARGUMENT, "sc_set_option: unknown option '%s'", name);
}

sc_status sc_get_option(const sc_ctx* ctx, const char* name, int64_t* value) {
  if (ctx == nullptr || name == nullptr || value == nullptr) return SC_INVALID_ARGUMENT;
  const auto& o = ctx->opts;
  struct {
    const char* name;
    long long v;
  } const table[] = {{"ctas", o.ctas},           {"delta", o.delta},         {"delta_div", o.delta_div},
                     {"delta_refresh", o.delta_refresh}, {"two_phase", o.two_phase}, {"stages", o.stages},
                     {"res_rows", o.res_rows},   {"fuse_update", o.fuse_update}, {"variant", o.variant},
                     {"profile", o.profile},     {"poison", o.poison},       {"fast_delta", o.fast_delta},
                     {"l2_persist", o.l2_persist}};
  for (const auto& e : table)
    if (std::strcmp(e.name, name) == 0) {
      *value = e.v;
      return SC_OK;
    }
  return SC_INVALID_ARGUMENT;
}

sc_status sc_validate_problem(const sc_problem* problem, char* msg, size_t msg_len) {
  std::string m;
  const sc_status st = validate(problem, &m);
  if (msg && msg_len) {
    std::snprintf(msg, msg_len, "%s", m.c_str());
  }
  return st;
}

uint64_t sc_start_vectors(const sc_problem* problem, uint64_t term, uint64_t restart,
                          uint64_t* out_words) {
  if (validate(problem, nullptr) != SC_OK || out_words == nullptr) return 0;
  return start_vectors(problem, term, restart, out_words);
}

void sc_fill_normal_f64(uint64_t seed, uint64_t count, double* out) {
  scb::Xoshiro rng(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng.next_normal();
}

void sc_fill_normal_f32(uint64_t seed, uint64_t count, float* out) {
  scb::Xoshiro rng(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = static_cast<float>(rng.next_normal());
}

uint64_t sc_width_for_compression(int coeff_bits, int source_bits, int order, const uint64_t* shape,
                                  double rate) {
  // width_for_compression, metrics.hpp:55-63
  if (order < 1 || shape == nullptr || !(rate > 0.0) || rate > 1.0) return 0;
  double numel = 1.0;
  uint64_t sign_bits = 0;
  for (int i = 0; i < order; ++i) {
    numel *= static_cast<double>(shape[i]);
    sign_bits += shape[i];
  }
  const double src = static_cast<double>(source_bits) * numel;
  return static_cast<uint64_t>(std::floor(rate * src / static_cast<double>(coeff_bits + sign_bits)));
}

void sc_lpt_schedule(const double* costs, uint64_t count, uint32_t bins, uint32_t* bin_of_job) {
  if (bins == 0) return;
  std::vector<uint64_t> order(count);
  std::iota(order.begin(), order.end(), uint64_t{0});
  // longest first; ties by job index so every rank computes the same plan
  std::stable_sort(order.begin(), order.end(),
                   [&](uint64_t a, uint64_t b) { return costs[a] > costs[b]; });
  std::vector<double> load(bins, 0.0);
  for (uint64_t j : order) {
    uint32_t best = 0;
    for (uint32_t b = 1; b < bins; ++b)
      if (load[b] < load[best]) best = b;
    bin_of_job[j] = best;
    load[best] += costs[j];
  }
}

sc_status sc_batch_decompose(const int32_t* devices, int32_t ndevices, sc_batch_job* jobs, uint64_t njobs,
                             char* msg, size_t msg_len) {
  auto fail_msg = [&](const char* m) {
    if (msg && msg_len) std::snprintf(msg, msg_len, "%s", m);
  };
  if (msg && msg_len) msg[0] = '\0';
  if (devices == nullptr || ndevices < 1 || (jobs == nullptr && njobs > 0)) {
    fail_msg("sc_batch_decompose: no devices / null jobs");
    return SC_INVALID_ARGUMENT;
  }
  std::vector<double> cost(njobs, 0.0);
  for (uint64_t j = 0; j < njobs; ++j) {
    const sc_problem& p = jobs[j].problem;
    double numel = 1.0;
    for (int i = 0; p.shape != nullptr && i < p.order && i < SC_MAX_ORDER; ++i) numel *= static_cast<double>(p.shape[i]);
    cost[j] = static_cast<double>(std::max<uint64_t>(p.width, 1)) * numel;
    jobs[j].status = SC_OK;
    jobs[j].device = -1;
  }
  std::vector<uint32_t> bin(njobs, 0);
  sc_lpt_schedule(cost.data(), njobs, static_cast<uint32_t>(ndevices), bin.data());
  std::mutex mu;
  sc_status first = SC_OK;
  std::string first_msg;
  auto note = [&](sc_status st, const std::string& m) {
    std::lock_guard<std::mutex> lk(mu);
    if (first == SC_OK) {
      first = st;
      first_msg = m;
    }
  };
  auto worker = [&](int32_t b) {
    std::vector<uint64_t> mine;
    for (uint64_t j = 0; j < njobs; ++j)
      if (bin[j] == static_cast<uint32_t>(b)) mine.push_back(j);
    std::stable_sort(mine.begin(), mine.end(), [&](uint64_t x, uint64_t y) { return cost[x] > cost[y]; });
    sc_ctx* ctx = nullptr;
    const sc_status cst = sc_create(&ctx, devices[b]);
    for (uint64_t j : mine) {
      jobs[j].device = devices[b];
      if (cst != SC_OK) {
        jobs[j].status = cst;
        note(cst, "sc_batch_decompose: sc_create(device " + std::to_string(devices[b]) + ") failed");
        continue;
      }
      const sc_status st = sc_greedy_decompose(ctx, &jobs[j].problem, jobs[j].result);
      jobs[j].status = st;
      if (st != SC_OK) note(st, "job " + std::to_string(j) + ": " + sc_last_error(ctx));
    }
    if (ctx) sc_destroy(ctx);
  };
  std::vector<std::thread> threads;
  for (int32_t b = 1; b < ndevices; ++b) threads.emplace_back(worker, b);
  worker(0);
  for (auto& t : threads) t.join();
  if (first != SC_OK) fail_msg(first_msg.c_str());
  return first;
}

namespace {
// Everything finish_run needs after the launch (prepare_run fills it).
struct RunState {
  std::chrono::steady_clock::time_point t_start;
  scb::Variant var{};
  scb::KParams kp{};
  size_t smem = 0;
  bool tensor = false, prof = false;
  int kax = 0, G = 0, res_rows = 0, stages = 0;
  int ax_off[7] = {0, 0, 0, 0, 0, 0, 0};
  uint64_t axw64 = 0, m = 0, n = 0, w = 0, wm = 0, wn = 0, h2d = 0, d2h = 0;
  size_t es = 0, rowB = 0;
  double numel = 0.0;  // global element count (row-sharded: m_global * n)
  void* dR = nullptr;
  unsigned* ctr_g = nullptr;
  unsigned long long* stats = nullptr;
  double* norm2 = nullptr;
  uint64_t *S_out = nullptr, *T_out = nullptr, *AX_out = nullptr;
  double* c_out = nullptr;
  uint32_t* sweeps_out = nullptr;
  double* dsweeps = nullptr;
  unsigned long long* dprof = nullptr;
};
sc_status prepare_run(sc_ctx* ctx, const sc_problem* p, sc_result* res, const sc_ctx::Shard* sh, RunState& S,
                      bool vr);
sc_status finish_run(sc_ctx* ctx, const sc_problem* p, sc_result* res, RunState& S);
sc_status run_decompose(sc_ctx* ctx, const sc_problem* p, sc_result* res, const sc_ctx::Shard* sh);

// CTAs for m rows (the engine and the sharded path agree, so world-1 sharding is
// bit-identical to the engine)
uint64_t auto_ctas(int num_sms, int cps, uint64_t m) {
  uint64_t g = std::min<uint64_t>(static_cast<uint64_t>(num_sms) * cps, m);
  if (cps == 1 && m <= 8ull * num_sms) {
    const uint64_t k = (m + 127) / 128;
    g = std::min<uint64_t>(g, (m + k - 1) / k);
  }
  return g;
}
}

sc_status sc_greedy_decompose(sc_ctx* ctx, const sc_problem* p, sc_result* res) {
  return run_decompose(ctx, p, res, nullptr);
}

namespace {
sc_status run_decompose(sc_ctx* ctx, const sc_problem* p, sc_result* res, const sc_ctx::Shard* sh) {
  RunState S;
  if (sc_status st = prepare_run(ctx, p, res, sh, S, false); st != SC_OK) return st;
  // the attribute is a per-function maximum shared by every context and thread of
  // the process: always the device's opt-in limit, so concurrent engines never
  // lower it under each other's launches (the launch passes the real size)
  SC_CUDA(ctx, scb::set_smem_limit(S.var, ctx->smem_optin));
  // Option l2_persist: the remainder R as a persisting-L2 access window for the launch, so
  // the delta passes' latency-critical gathers are not evicted to DRAM by the exchange
  // buffers and write-backs (hit ratio scaled down when R exceeds the carve-out).
  const size_t r_bytes = S.m * S.rowB;
  const bool persist = ctx->opts.l2_persist && ctx->l2_persist_max > 0 && ctx->l2_window_max > 0 && r_bytes > 0;
  if (persist) {
    const size_t carve = ctx->l2_persist_max;
    SC_CUDA(ctx, cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
    cudaStreamAttrValue av{};
    av.accessPolicyWindow.base_ptr = S.dR;
    av.accessPolicyWindow.num_bytes = std::min(r_bytes, ctx->l2_window_max);
    av.accessPolicyWindow.hitRatio =
        static_cast<float>(std::min(1.0, static_cast<double>(carve) / static_cast<double>(av.accessPolicyWindow.num_bytes)));
    av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    SC_CUDA(ctx, cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &av));
  }
  SC_CUDA(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
  SC_CUDA(ctx, scb::launch_sweep(S.var, S.kp, S.smem, ctx->stream));
  SC_CUDA(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
  if (persist) {
    cudaStreamAttrValue av{};
    av.accessPolicyWindow.num_bytes = 0;
    SC_CUDA(ctx, cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &av));
  }
  const sc_status fin = finish_run(ctx, p, res, S);
  if (persist) cudaCtxResetPersistingL2Cache();
  return fin;
}

sc_status prepare_run(sc_ctx* ctx, const sc_problem* p, sc_result* res, const sc_ctx::Shard* sh, RunState& S,
                      bool vr) {
  const auto t_start = std::chrono::steady_clock::now();
  if (ctx == nullptr) return SC_INVALID_ARGUMENT;
  if (res == nullptr) return set_err(ctx, SC_INVALID_ARGUMENT, "sc_result: null");
  std::string msg;
  if (validate(p, &msg) != SC_OK) return set_err(ctx, SC_INVALID_ARGUMENT, "%s", msg.c_str());
  for (int i = 0; i < p->order; ++i)
    if (res->sign_words[i] == nullptr)
      return set_err(ctx, SC_INVALID_ARGUMENT, "sc_result: sign_words of every axis are required");
  if (res->cut_value == nullptr) return set_err(ctx, SC_INVALID_ARGUMENT, "sc_result: cut_value is required");
  SC_CUDA(ctx, cudaSetDevice(ctx->device));

  // Order 2: the matrix itself.  Order k (1 or >= 3; axial_run, search.hpp:191-213):
  // the matrix view M = n_0 x (n_1 ... n_{k-1}) with the Kronecker sign of the
  // trailing axes as t; the trailing axes are updated on the device from M^T s_0.
  const bool tensor = p->order != 2;
  const int kax = p->order - 1;
  const uint64_t m = p->shape[0];
  uint64_t n = 1;
  for (int i = 1; i < p->order; ++i) {
    if (p->shape[i] > INT32_MAX / 2 || n > (INT32_MAX / 2) / p->shape[i])
      return set_err(ctx, SC_NOT_SUPPORTED, "tensor trailing size too large for this build");
    n *= p->shape[i];
  }
  uint64_t axw64 = 0;  // u64 words of the trailing axes' signs
  int ax_off[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int i = 1; i < p->order; ++i) {
    ax_off[i - 1] = static_cast<int>(2 * axw64);
    axw64 += words64(p->shape[i]);
  }
  if (!tensor) axw64 = 0;
  const int axw = static_cast<int>(2 * axw64);
  if (m > INT32_MAX / 2 || n > INT32_MAX / 2)
    return set_err(ctx, SC_NOT_SUPPORTED, "matrix dimension too large for this build");
  const int dt = p->dtype;
  const size_t es = dt == SC_F32 ? 4 : 8;
  const long long pitch = static_cast<long long>((n + 31) / 32 * 32);
  scb::Variant var{};
  if (scb::pick_variant(dt, pitch, &var, ctx->opts.variant) != 0)
    return set_err(ctx, SC_NOT_SUPPORTED, "row length %llu exceeds the fused-kernel envelope",
                   static_cast<unsigned long long>(n));
  // One GPU, matrices, f32 rows of 2049..4096 columns: 16 consumer warps x 2 vectors instead of
  // 8 x 4 -- four warps per scheduler hide the per-row latency chain of the dense passes
  // (14336 x 4096: 67.5 -> 53.8 ms per 64 cuts, 32000 x 4096: 76.5 -> 58.9 ms; 4096^2 and
  // 1024 x 4096 unchanged).  Order-k and row-sharded runs keep the 8-warp tile.
  if (!tensor && !sh && ctx->opts.variant == 0 && dt == SC_F32 && var.nw == 8 && var.vpt == 4 && var.rg == 1) {
    var.nw = 16;
    var.vpt = 2;
  }
  // f64 rows of 2049..4096 columns: the same 16-warp tile once R spills to HBM (14336 x 4096 f64:
  // 36.3 -> 34.1 ms per 32 cuts; L2-resident 4096^2 f64 is 3% faster with 8 warps)
  if (!tensor && !sh && ctx->opts.variant == 0 && dt == SC_F64 && var.nw == 8 && var.vpt == 8 && var.rg == 1 &&
      pitch <= 4096 && m * static_cast<uint64_t>(pitch) * 8 > (uint64_t{160} << 20)) {
    var.nw = 16;
    var.vpt = 4;
  }
  var.tensor = tensor ? 1 : 0;  // order-k kernels are separate instantiations
  var.mr = (sh && sh->world > 1 && !vr) ? 1 : 0;  // the multi-rank exchange is compiled in separately
  if (var.mr && !scb::has_vr(var))
    return set_err(ctx, SC_NOT_SUPPORTED, "row sharding: no multi-rank kernel for rows of %llu", static_cast<unsigned long long>(n));
  if (vr && !scb::has_vr(var))
    return set_err(ctx, SC_NOT_SUPPORTED, "emulated row sharding: no virtual-rank kernel for rows of %llu", static_cast<unsigned long long>(n));

  // wide rows: column chunks of one warp-tile pass (var.nw * 32 * var.vpt vectors)
  const long long tile_cols = static_cast<long long>(var.nw) * 32 * var.vpt * (dt == SC_F32 ? 4 : 2);
  const int cpr = pitch > tile_cols ? static_cast<int>((pitch + tile_cols - 1) / tile_cols) : 1;
  if (sh && (tensor || var.cps != 1 || static_cast<uint64_t>(sh->G) > m))
    return set_err(ctx, SC_NOT_SUPPORTED, "row sharding: matrices only, one CTA per SM, band >= %d rows", sh ? sh->G : 0);
  // CTAs: one per SM; small matrices (<= 8 rows per SM) use at most 128 CTAs with
  // equal bands -- the pass is synchronisation-bound there and a smaller, balanced
  // grid is faster (1024^2 f32: 11.5 vs 13.1 us/pass).  SCB_CTAS caps G (tuning).
  const uint64_t g_auto = auto_ctas(ctx->num_sms, var.cps, m);
  const int G = sh ? sh->G
                  : static_cast<int>(ctx->opts.ctas > 0 ? std::min<uint64_t>(g_auto, static_cast<uint64_t>(ctx->opts.ctas))
                                                        : g_auto);
  const int rows_base = static_cast<int>(m / G), rows_rem = static_cast<int>(m % G);
  const int rows_max = rows_base + (rows_rem ? 1 : 0);
  const int Q = static_cast<int>(pitch / 32);
  const int sw = (rows_max + 31) / 32;
  const int zl = std::max(1, std::min(4, (Q + G - 1) / G));
  const size_t rowB = static_cast<size_t>(pitch) * es;
  const size_t stageB = cpr > 1 ? static_cast<size_t>(tile_cols) * es : rowB;  // one row or one chunk
  auto smem_for = [&](int st_, int res_) {
    return scb::make_layout(stageB, st_, res_, var.rg, var.nw, rows_max, Q, zl, sw, axw, G).total;
  };
  // per-CTA shared memory: the opt-in maximum, or an even split of the SM's
  // 228 KB (minus the 1 KB the runtime reserves per CTA) when two CTAs share an SM
  const size_t cap = var.cps == 1 ? ctx->smem_optin : std::min(ctx->smem_optin, (ctx->smem_per_sm / var.cps) - 1024);
  int stages = 0, res_rows = rows_max;
  if (cpr > 1 || smem_for(0, rows_max) > cap) {
    stages = static_cast<int>(ctx->opts.stages > 0 ? ctx->opts.stages : 2 * var.rg + 4);
    stages = std::max(2, std::min(stages, scb::kMaxStages));
    while (stages > 2 && smem_for(stages, 0) > cap) --stages;
    if (smem_for(stages, 0) > cap)
      return set_err(ctx, SC_NOT_SUPPORTED, "row of %zu bytes does not fit the shared-memory ring", rowB);
    res_rows = 0;
    while (cpr == 1 && res_rows < rows_max && smem_for(stages, res_rows + 1) <= cap) ++res_rows;
    if (ctx->opts.res_rows >= 0) res_rows = static_cast<int>(std::min<long long>(ctx->opts.res_rows, res_rows));
  }
  // the cooperative launch needs every CTA co-resident: trim resident rows until
  // the occupancy API confirms var.cps CTAs per SM at this footprint
  while (var.cps > 1 && res_rows > 0 && scb::blocks_per_sm(var, smem_for(stages, res_rows)) < var.cps) --res_rows;
  while (var.cps > 1 && stages > 2 && scb::blocks_per_sm(var, smem_for(stages, res_rows)) < var.cps) --stages;
  const size_t smem = smem_for(stages, res_rows);
  if (scb::blocks_per_sm(var, smem) < var.cps)
    return set_err(ctx, SC_NOT_SUPPORTED, "%d CTAs per SM do not fit (%zu bytes of shared memory each)", var.cps, smem);

  const uint64_t w = p->width;
  const uint64_t wm = words64(m), wn = words64(n);
  const int t_stride = static_cast<int>(2 * wn), s_stride = static_cast<int>(2 * wm);
  const int tw32 = std::max(Q, t_stride);
  const uint64_t nstart = std::max<uint64_t>(w, 1) * p->restarts;

  // ---- device arena ----
  // barrier-free delta passes: one self-tagged record per CTA and pass parity, whole 128-byte lines
  const int rstride = ((2 * (sw + 1) + 15) / 16) * 16;
  const size_t need = ((m * rowB + 255) & ~size_t(255)) + ((2 * G * rowB * 8 / es + 255) & ~size_t(255)) +
                      ((G * sizeof(scb::Slot) + 255) & ~size_t(255)) + 4 * 256 +
                      ((2 * static_cast<size_t>(tw32) * 8 * scb::kTbStride + 255) & ~size_t(255)) +
                      ((tw32 * 8 + 255) & ~size_t(255)) +
                      ((nstart * wn * 8 + 255) & ~size_t(255)) +
                      ((std::max<uint64_t>(w, 1) * (wm + wn) * 8 + 511) & ~size_t(255)) +
                      ((std::max<uint64_t>(w, 1) * 8 + 255) & ~size_t(255)) * 2 +
                      (((w + 1) * 8 + 255) & ~size_t(255)) + 8 * 256 + 4096 +
                      ((nstart * axw64 * 8 + 255) & ~size_t(255)) +
                      ((std::max<uint64_t>(w, 1) * axw64 * 8 + 255) & ~size_t(255)) +
                      2 * ((static_cast<size_t>(pitch) * 8 + 255) & ~size_t(255)) +
                      ((2 * static_cast<size_t>(G) * sw * 8 + 255) & ~size_t(255)) +
                      ((2 * static_cast<size_t>(G) * rstride * 8 + 255) & ~size_t(255));
  if (need > ctx->arena_bytes) {
    if (ctx->arena) cudaFree(ctx->arena);
    ctx->arena = nullptr;
    ctx->arena_bytes = 0;
    SC_CUDA(ctx, cudaMalloc(&ctx->arena, need));
    ctx->arena_bytes = need;
  }
  char* cur = static_cast<char*>(ctx->arena);
  void* dR = carve<char>(cur, m * rowB);
  double* zpart = carve<double>(cur, 2 * static_cast<size_t>(G) * pitch);  // [2][G][pitch] by pass parity
  scb::Slot* slots = carve<scb::Slot>(cur, G);
  unsigned* ctr = carve<unsigned>(cur, 8);  // [0] grid barrier, [1..3] err_pass
  unsigned long long* stats = carve<unsigned long long>(cur, 8);
  unsigned long long* tb64 = carve<unsigned long long>(cur, 2 * static_cast<size_t>(tw32) * scb::kTbStride);
  unsigned* ctr_g = ctr;  // the grid's barrier / error words (rank 0's when sharded)
  if (sh) {  // exchange buffers live in the peer-mapped shard region (reset by sc_shard_reset)
    if (sh->pitch != pitch || sh->dtype != dt || sh->n != n)
      return set_err(ctx, SC_INVALID_ARGUMENT, "sc_greedy_decompose_sharded: problem does not match the shard");
    if (sh->G != G) return set_err(ctx, SC_INVALID_ARGUMENT, "sc_greedy_decompose_sharded: CTA count mismatch");
    char* ex = static_cast<char*>(sh->exch);
    zpart = reinterpret_cast<double*>(ex + sh->off_zpart);
    slots = reinterpret_cast<scb::Slot*>(ex + sh->off_slots);
    tb64 = reinterpret_cast<unsigned long long*>(ex + sh->off_tb64);
    ctr = reinterpret_cast<unsigned*>(ex + sh->off_ctr);
    ctr_g = reinterpret_cast<unsigned*>(static_cast<char*>(sh->peers[0]) + sh->off_ctr);
  }
  uint32_t* tbest = carve<uint32_t>(cur, tw32);
  uint64_t* t0 = carve<uint64_t>(cur, nstart * wn);
  uint64_t* S_out = carve<uint64_t>(cur, std::max<uint64_t>(w, 1) * wm);
  uint64_t* T_out = carve<uint64_t>(cur, std::max<uint64_t>(w, 1) * wn);
  double* c_out = carve<double>(cur, std::max<uint64_t>(w, 1));
  uint32_t* sweeps_out = carve<uint32_t>(cur, std::max<uint64_t>(w, 1) * 2);
  double* norm2 = carve<double>(cur, w + 1);
  uint64_t* ax0 = carve<uint64_t>(cur, std::max<uint64_t>(nstart * axw64, 1));
  uint64_t* AX_out = carve<uint64_t>(cur, std::max<uint64_t>(std::max<uint64_t>(w, 1) * axw64, 1));
  double* zfull = carve<double>(cur, static_cast<size_t>(pitch));
  double* zstate = carve<double>(cur, static_cast<size_t>(pitch));
  unsigned long long* flipw = carve<unsigned long long>(cur, 2 * static_cast<size_t>(G) * sw);
  unsigned long long* drec = carve<unsigned long long>(cur, 2 * static_cast<size_t>(G) * rstride);

  // ---- host staging (pinned) for the start vectors ----
  const size_t t0_bytes = nstart * wn * 8, ax0_bytes = nstart * axw64 * 8;
  if (t0_bytes + ax0_bytes > ctx->pinned_bytes) {
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    ctx->pinned = nullptr;
    ctx->pinned_bytes = 0;
    SC_CUDA(ctx, cudaMallocHost(&ctx->pinned, t0_bytes + ax0_bytes));
    ctx->pinned_bytes = t0_bytes + ax0_bytes;
  }
  uint64_t* ht0 = static_cast<uint64_t*>(ctx->pinned);
  uint64_t* hax0 = ht0 + nstart * wn;
  if (!tensor) {
    // sharded: the draw of s0 skips the words of the GLOBAL row count
    sc_problem pg = *p;
    uint64_t gshape[2] = {sh ? sh->m_global : m, n};
    pg.shape = gshape;
    for (uint64_t term = 0; term < w; ++term)
      for (uint64_t r = 0; r < p->restarts; ++r) start_vectors(&pg, term, r, ht0 + (term * p->restarts + r) * wn);
  } else {
    // all k axes drawn in axis order (search.hpp:197); s_0 is recomputed first,
    // the trailing axes seed the axial step and form the first t = kron(s_1..s_{k-1})
    std::vector<uint64_t> buf(words64(m) + axw64);
    for (uint64_t term = 0; term < w; ++term)
      for (uint64_t r = 0; r < p->restarts; ++r) {
        start_vectors(p, term, r, buf.data());
        const uint64_t* axs = buf.data() + words64(m);
        uint64_t* rec = hax0 + (term * p->restarts + r) * axw64;
        std::copy(axs, axs + axw64, rec);
        uint64_t* tw = ht0 + (term * p->restarts + r) * wn;
        std::fill(tw, tw + wn, uint64_t{0});
        for (uint64_t col = 0; col < n; ++col) {
          uint64_t c = col, xb = 0;
          for (int i = kax - 1; i >= 0; --i) {
            const uint64_t ni = p->shape[i + 1], idx = c % ni;
            c /= ni;
            xb ^= (axs[ax_off[i] / 2 + idx / 64] >> (idx % 64)) & 1u;
          }
          tw[col / 64] |= xb << (col % 64);
        }
      }
  }

  cudaStream_t st = ctx->stream;
  uint64_t h2d = 0, d2h = 0;
  if (ctx->opts.poison) SC_CUDA(ctx, cudaMemsetAsync(ctx->arena, 0xff, ctx->arena_bytes, st));
  const cudaMemcpyKind in_kind = p->data_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (static_cast<uint64_t>(pitch) != n) SC_CUDA(ctx, cudaMemsetAsync(dR, 0, m * rowB, st));
  SC_CUDA(ctx, cudaMemcpy2DAsync(dR, rowB, p->data, n * es, n * es, m, in_kind, st));
  if (!p->data_on_device) h2d += m * n * es;
  if (w > 0) {
    SC_CUDA(ctx, cudaMemcpyAsync(t0, ht0, t0_bytes, cudaMemcpyHostToDevice, st));
    h2d += t0_bytes;
    if (ax0_bytes) {
      SC_CUDA(ctx, cudaMemcpyAsync(ax0, hax0, ax0_bytes, cudaMemcpyHostToDevice, st));
      h2d += ax0_bytes;
    }
  }
  if (!sh) {
    SC_CUDA(ctx, cudaMemsetAsync(ctr, 0, 4, st));
    SC_CUDA(ctx, cudaMemsetAsync(ctr + 1, 0xff, 12, st));
    SC_CUDA(ctx, cudaMemsetAsync(slots, 0, static_cast<size_t>(G) * sizeof(scb::Slot), st));
    SC_CUDA(ctx, cudaMemsetAsync(tb64, 0, 2 * static_cast<size_t>(tw32) * 8 * scb::kTbStride, st));
  }
  SC_CUDA(ctx, cudaMemsetAsync(tbest, 0, static_cast<size_t>(tw32) * 4, st));
  SC_CUDA(ctx, cudaMemsetAsync(drec, 0, 2 * static_cast<size_t>(G) * rstride * 8, st));
  SC_CUDA(ctx, cudaMemsetAsync(stats, 0, 64, st));
  if (!sh) SC_CUDA(ctx, cudaMemsetAsync(ctr + 4, 0xff, 4, st));
  if (w > 0) SC_CUDA(ctx, cudaMemsetAsync(S_out, 0, w * wm * 8, st));

  scb::KParams kp{};
  kp.R = dR;
  kp.pitch = pitch;
  kp.m = static_cast<int>(m);
  kp.n = static_cast<int>(n);
  kp.G = G;
  kp.rows_base = rows_base;
  kp.rows_rem = rows_rem;
  kp.res_rows = res_rows;
  kp.rows_max = rows_max;
  kp.stages = stages;
  kp.Q = Q;
  kp.sw = sw;
  kp.zl = zl;
  kp.t0 = reinterpret_cast<const uint32_t*>(t0);
  kp.t0_stride = t_stride;
  kp.tb64 = tb64;
  kp.tbest = tbest;
  kp.zpart = zpart;
  kp.slots = slots;
  kp.bar = ctr_g;
  kp.err_pass = ctr_g + 1;
  kp.S_out = reinterpret_cast<uint32_t*>(S_out);
  kp.s_stride = s_stride;
  kp.T_out = reinterpret_cast<uint32_t*>(T_out);
  kp.t_stride = t_stride;
  kp.c_out = c_out;
  kp.sweeps_out = sweeps_out;
  kp.norm2_out = norm2;
  kp.stats = stats;
  kp.width = static_cast<long long>(w);
  kp.restarts = static_cast<long long>(p->restarts);
  kp.max_sweeps = static_cast<long long>(std::min<uint64_t>(p->max_sweeps, 1ull << 40));
  kp.min_frac = p->min_value_fraction;
  kp.numel_d = static_cast<double>((sh ? sh->m_global : m) * n);
  kp.widen_mul = 1 << 29;
  kp.tensor = tensor ? 1 : 0;
  kp.kax = tensor ? kax : 0;
  for (int i = 0; i < 7; ++i) {
    kp.ax_n[i] = (tensor && i < kax) ? static_cast<int>(p->shape[i + 1]) : 1;
    kp.ax_off[i] = ax_off[i];
  }
  kp.axw = axw;
  kp.ax0 = reinterpret_cast<const uint32_t*>(ax0);
  kp.AX_out = reinterpret_cast<uint32_t*>(AX_out);
  kp.zfull = zfull;
  kp.zstate = zstate;
  kp.flipw = flipw;
  kp.drec = drec;
  kp.rstride = rstride;
  // one GPU, matrices, whole rows, one record-polling thread per CTA of the grid
  kp.fast_delta = (ctx->opts.fast_delta && !tensor && !sh && !vr && cpr == 1 && var.nw * 32 >= G && G <= 160 && Q <= 4 * G) ? 1 : 0;
  // delta pass only if the last sweep flipped <= n / delta_div columns.  Auto (0): n / 4 with the
  // barrier-free delta pass (4096^2 w=512 on the final kernel: 278.7 ms at 8, 276.7 at 6, 270.8
  // at 4, 271.6 at 3; 2.5 dense passes per cut instead of 3.5), n / 32 for the barrier passes
  // (order-k, row-sharded, chunked rows: measured best in round 1)
  kp.delta_div = static_cast<int>(ctx->opts.delta_div > 0 ? ctx->opts.delta_div : (kp.fast_delta ? 4 : 32));
  // Sparse delta passes between dense refreshes (matrices, any row length: the dz of
  // flipped rows walks every column chunk).
  kp.delta = ctx->opts.delta ? 1 : 0;
  kp.fuse_update = ctx->opts.fuse_update ? 1 : 0;
  kp.delta_refresh = static_cast<int>(std::max<long long>(1, ctx->opts.delta_refresh));
  // Dot-pass form: the two-phase pass reads R twice per sweep but has no per-row
  // serial chain -- the better choice while R stays in SMEM / L2; once R spills
  // to HBM the fused single-read pass wins (14336x4096 f32: 77.6 vs 84 us/pass).
  // Wide rows (cpr > 1) always take the two-phase pass.  SCB_2PH=0/1 overrides.
  const bool l2_resident = m * rowB <= (size_t{160} << 20);  // 4096^2 f64 (128 MB): two-phase 24.0 vs 24.6 us/pass
  // The 16-warp whole-row variants (8193..14336 f32 columns) are faster two-phase
  // even when R spills to HBM (4096 x 14336 f32: 58 vs 97 us/pass; C3: 91 vs 183).
  kp.two_phase = (cpr > 1 || var.nw == 16) ? 1
                 : (ctx->opts.two_phase >= 0 ? (ctx->opts.two_phase ? 1 : 0) : (l2_resident ? 1 : 0));
  kp.cpr = cpr;
  kp.world = sh ? sh->world : 1;
  kp.rank = sh ? sh->rank : 0;
  kp.GT = G * kp.world;
  for (int r = 0; r < kp.world; ++r) {
    char* ex = sh ? static_cast<char*>(sh->peers[r]) : nullptr;
    kp.zr_pe[r] = sh ? reinterpret_cast<double*>(ex + sh->off_zr) : nullptr;
    kp.rslot_pe[r] = sh ? reinterpret_cast<scb::Slot*>(ex + sh->off_rslot) : nullptr;
    kp.tb64_pe[r] = sh ? reinterpret_cast<unsigned long long*>(ex + sh->off_tb64) : tb64;
  }
  kp.zr_own = kp.zr_pe[kp.rank];
  kp.rslot_own = kp.rslot_pe[kp.rank];
  kp.bar_local = ctr + 5;  // this rank's own counter
  kp.abort_word = ctr_g + 6;
  kp.timeout_ns = static_cast<long long>(sh && sh->timeout_ms ? sh->timeout_ms : 30000u) * 1000000ll;
  kp.fault = sh ? sh->fault : 0;
  kp.chunk_cols = cpr > 1 ? static_cast<int>(tile_cols) : static_cast<int>(pitch);

  const bool prof = ctx->opts.profile != 0;
  unsigned long long* dprof = nullptr;
  if (prof) {
    SC_CUDA(ctx, cudaMalloc(&dprof, static_cast<size_t>(G) * 32 * 8));
    SC_CUDA(ctx, cudaMemsetAsync(dprof, 0, static_cast<size_t>(G) * 32 * 8, st));
  }
  kp.prof = dprof;
  // SearchDiagnostics::sweep_values of term 0, every restart (the host keeps the winner's)
  double* dsweeps = nullptr;
  res->n_sweep_values = 0;
  if (res->sweep_values != nullptr && w > 0 && !sh) {
    void* pv = nullptr;
    const size_t nb = static_cast<size_t>(p->restarts) * p->max_sweeps * 8;
    if (sc_status s2 = scb::pool_get(ctx, "diag.sweeps", nb, &pv); s2 != SC_OK) return s2;
    dsweeps = static_cast<double*>(pv);
    SC_CUDA(ctx, cudaMemsetAsync(dsweeps, 0, nb, st));
  }
  kp.sweep_vals = dsweeps;
  S.t_start = t_start;
  S.var = var;
  S.kp = kp;
  S.smem = smem;
  S.tensor = tensor;
  S.prof = prof;
  S.kax = kax;
  S.G = G;
  S.res_rows = res_rows;
  S.stages = stages;
  std::copy(ax_off, ax_off + 7, S.ax_off);
  S.axw64 = axw64;
  S.m = m;
  S.n = n;
  S.w = w;
  S.wm = wm;
  S.wn = wn;
  S.h2d = h2d;
  S.d2h = d2h;
  S.es = es;
  S.rowB = rowB;
  S.numel = kp.numel_d;
  S.dR = dR;
  S.ctr_g = ctr_g;
  S.stats = stats;
  S.norm2 = norm2;
  S.S_out = S_out;
  S.T_out = T_out;
  S.AX_out = AX_out;
  S.c_out = c_out;
  S.sweeps_out = sweeps_out;
  S.dsweeps = dsweeps;
  S.dprof = dprof;
  return SC_OK;
}

sc_status finish_run(sc_ctx* ctx, const sc_problem* p, sc_result* res, RunState& S) {
  const auto t_start = S.t_start;
  const scb::Variant& var = S.var;
  const bool tensor = S.tensor, prof = S.prof;
  const int kax = S.kax, G = S.G, res_rows = S.res_rows, stages = S.stages;
  const int* ax_off = S.ax_off;
  const uint64_t axw64 = S.axw64, m = S.m, n = S.n, w = S.w, wm = S.wm, wn = S.wn;
  uint64_t h2d = S.h2d, d2h = S.d2h;
  const size_t es = S.es, rowB = S.rowB, smem = S.smem;
  void* dR = S.dR;
  unsigned* ctr_g = S.ctr_g;
  unsigned long long* stats = S.stats;
  double* norm2 = S.norm2;
  uint64_t *S_out = S.S_out, *T_out = S.T_out, *AX_out = S.AX_out;
  double* c_out = S.c_out;
  uint32_t* sweeps_out = S.sweeps_out;
  double* dsweeps = S.dsweeps;
  unsigned long long* dprof = S.dprof;
  cudaStream_t st = ctx->stream;
  const long long pitch = S.kp.pitch;
  (void)pitch;

  // ---- results ----
  unsigned h_ctr[8];
  unsigned long long h_stats[8];
  std::vector<double> h_norm2(w + 1);
  SC_CUDA(ctx, cudaMemcpyAsync(h_ctr, ctr_g, 32, cudaMemcpyDeviceToHost, st));
  SC_CUDA(ctx, cudaMemcpyAsync(h_stats, stats, 64, cudaMemcpyDeviceToHost, st));
  SC_CUDA(ctx, cudaMemcpyAsync(h_norm2.data(), norm2, (w + 1) * 8, cudaMemcpyDeviceToHost, st));
  SC_CUDA(ctx, cudaStreamSynchronize(st));
  d2h += 32 + 64 + (w + 1) * 8;
  float kms = 0.f;
  cudaEventElapsedTime(&kms, ctx->ev0, ctx->ev1);
  res->kernel_ms = kms;
  res->kernel_launches = 1;
  if (prof) {
    std::vector<unsigned long long> hp(static_cast<size_t>(G) * 32);
    cudaMemcpy(hp.data(), dprof, hp.size() * 8, cudaMemcpyDeviceToHost);
    {
      double d[16] = {0};
      for (int g = 0; g < G; ++g)
        for (int i = 0; i < 16; ++i) d[i] += static_cast<double>(hp[static_cast<size_t>(G) * 16 + g * 16 + i]);
      const double nd = std::max<double>(1.0, static_cast<double>(h_stats[3])) * G;
      if (S.kp.fast_delta && ctx->opts.profile >= 2) {
        static const int slots[] = {0, 1, 2, 3, 4, 7, 8, 9, 10};
        static const char* nm[] = {"t wait", "list+sync", "gathers+bar", "signs+publish", "c poll", "decision", "flip poll", "gather", "final+publish"};
        const double npd = std::max<double>(1.0, static_cast<double>(h_stats[3]));
        for (int q = 0; q < 9; ++q) {
          std::fprintf(stderr, "[scb cta] %s:", nm[q]);
          for (int g = 0; g < G; ++g) std::fprintf(stderr, " %.0f", static_cast<double>(hp[static_cast<size_t>(G) * 16 + g * 16 + slots[q]]) / npd);
          std::fprintf(stderr, "\n");
        }
      }
      if (S.kp.fast_delta)
        std::fprintf(stderr, "[scb prof fast delta] per delta pass per CTA: thread 0: t wait %.0f list+sync %.0f gathers+bar %.0f signs+publish %.0f c poll %.0f decision %.0f | thread 32: flip poll %.0f rows counted %.0f rows listed %.0f gather %.0f final+publish %.0f\n",
                     d[0] / nd, d[1] / nd, d[2] / nd, d[3] / nd, d[4] / nd, d[7] / nd, d[8] / nd, d[11] / nd, d[12] / nd, d[9] / nd, d[10] / nd);
      else
        std::fprintf(stderr, "[scb prof delta] per delta pass per CTA: fliplists %.0f gathers %.0f sync %.0f signs %.0f dz %.0f | CTAs with dz per pass %.2f | column reduction (thread 32) %.0f decision %.0f\n",
                     d[0] / nd, d[1] / nd, d[2] / nd, d[3] / nd, d[4] / nd, d[5] / std::max<double>(1.0, static_cast<double>(h_stats[3])), d[6] / nd, d[7] / nd);
    }
    cudaFree(dprof);
    double acc[16] = {0};
    for (int g = 0; g < G; ++g)
      for (int i = 0; i < 16; ++i) acc[i] += static_cast<double>(hp[g * 16 + i]) / G;
    if (!tensor)
      std::fprintf(stderr, "[scb prof matrix] dot pass per dense pass %.0f, per delta pass %.0f cycles\n",
                   acc[8] * G / std::max<double>(1.0, static_cast<double>(h_stats[2])) / G,
                   acc[9] * G / std::max<double>(1.0, static_cast<double>(h_stats[3])) / G);
    if (tensor)
      std::fprintf(stderr, "[scb prof tensor] axis1 %.0f axis2 %.0f kron %.0f (slots 15, 8, 9 per dot pass)\n",
                   acc[15] / std::max<double>(1.0, static_cast<double>(h_stats[2])),
                   acc[8] / std::max<double>(1.0, static_cast<double>(h_stats[2])),
                   acc[9] / std::max<double>(1.0, static_cast<double>(h_stats[2])));
    if (tensor)
      std::fprintf(stderr, "[scb prof tensor] per dot pass: Z reduction+barrier %.0f (barrier %.0f), axial step %.0f cycles\n",
                   acc[12] / std::max<double>(1.0, static_cast<double>(h_stats[2])),
                   acc[14] / std::max<double>(1.0, static_cast<double>(h_stats[2])),
                   acc[13] / std::max<double>(1.0, static_cast<double>(h_stats[2])));
    {
      double mn[8], mx[8];
      for (int i = 0; i < 8; ++i) {
        mn[i] = 1e300;
        mx[i] = 0;
      }
      for (int g = 0; g < G; ++g)
        for (int i = 0; i < 8; ++i) {
          mn[i] = std::min(mn[i], static_cast<double>(hp[g * 16 + i]));
          mx[i] = std::max(mx[i], static_cast<double>(hp[g * 16 + i]));
        }
      const double np_ = std::max<double>(1.0, static_cast<double>(h_stats[1]));
      if (ctx->opts.profile >= 2) {
        std::fprintf(stderr, "[scb cta] barrier wait per pass:");
        for (int g = 0; g < G; ++g) std::fprintf(stderr, " %.0f", static_cast<double>(hp[g * 16 + 6]) / np_);
        std::fprintf(stderr, "\n[scb cta] dot pass per pass:");
        for (int g = 0; g < G; ++g) std::fprintf(stderr, " %.0f", static_cast<double>(hp[g * 16 + 1]) / np_);
        std::fprintf(stderr, "\n[scb cta] staging per pass:");
        for (int g = 0; g < G; ++g) std::fprintf(stderr, " %.0f", static_cast<double>(hp[g * 16 + 5]) / np_);
        std::fprintf(stderr, "\n");
      }
      std::fprintf(stderr, "[scb prof3] per pass min/max over CTAs: chunks %.0f/%.0f passend %.0f/%.0f decision %.0f/%.0f reduce %.0f/%.0f staging %.0f/%.0f\n",
                   mn[1] / np_, mx[1] / np_, mn[2] / np_, mx[2] / np_, mn[3] / np_, mx[3] / np_, mn[4] / np_, mx[4] / np_,
                   mn[5] / np_, mx[5] / np_);
    }
    std::fprintf(stderr, "[scb passes] dense dot %llu, delta dot %llu, total %llu | per delta pass: %.1f flipped columns, %.1f flipped rows\n",
                 static_cast<unsigned long long>(h_stats[2]), static_cast<unsigned long long>(h_stats[3]),
                 static_cast<unsigned long long>(h_stats[1]),
                 static_cast<double>(h_stats[7]) / std::max<double>(1.0, static_cast<double>(h_stats[3])),
                 static_cast<double>(h_stats[5]) / std::max<double>(1.0, static_cast<double>(h_stats[3])));
    std::fprintf(stderr, "[scb prof2] per pass: stagewait=%.0f A=%.0f B=%.0f C=%.0f\n",
                 acc[8] / std::max<double>(1.0, static_cast<double>(h_stats[1])),
                 acc[9] / std::max<double>(1.0, static_cast<double>(h_stats[1])),
                 acc[10] / std::max<double>(1.0, static_cast<double>(h_stats[1])),
                 acc[11] / std::max<double>(1.0, static_cast<double>(h_stats[1])));
    std::fprintf(stderr,
                 "[scb prof] G=%d res_rows=%d stages=%d nw=%d vpt=%d rg=%d smem=%zu | cycles/CTA: "
                 "fullwait=%.0f chunks=%.0f passend+bar=%.0f decision=%.0f reduce+bar=%.0f | staging=%.0f ringwait=%.0f | prod emptywait=%.0f  (per pass: chunks %.0f) passes=%llu\n",
                 G, res_rows, stages, var.nw, var.vpt, var.rg, smem, acc[0], acc[1], acc[2], acc[3], acc[4], acc[5], acc[6], acc[7],
                 acc[1] / std::max<double>(1.0, static_cast<double>(h_stats[1])),
                 static_cast<unsigned long long>(h_stats[1]));
  }
  if (S.kp.world > 1 && h_ctr[4] != 0xffffffffu)
    return set_err(ctx, SC_RUNTIME_ERROR,
                   "row-sharded exchange: a rank did not arrive within %lld ms (pass %u); run aborted",
                   S.kp.timeout_ns / 1000000, h_ctr[4]);
  if (h_ctr[3] != 0xffffffffu) return set_err(ctx, SC_INVALID_ARGUMENT, "DenseTensor: non-finite value");
  if (h_ctr[1] != 0xffffffffu || h_ctr[2] != 0xffffffffu)
    return set_err(ctx, SC_INVALID_ARGUMENT, "sgn_vector: non-finite entry");

  const uint64_t wd = h_stats[0];
  res->width_done = wd;
  res->passes = h_stats[1];
  res->dense_passes = h_stats[2];
  res->delta_passes = h_stats[3];
  {
    // Bytes the kernel moved through L2 / HBM, from the pass counts and the kernel's
    // traffic counters (SMEM-resident rows are on chip and not counted): streamed
    // rows per read (two-phase dot passes read twice), rank-1 write-backs, delta
    // gathers at 32-byte sectors (flipped columns x streamed rows) plus the flipped
    // streamed rows, and the column-partial rows written and read by the owners.
    const scb::KParams& kp = S.kp;
    uint64_t srows = 0, rrows = 0;
    for (int g = 0; g < kp.G; ++g) {
      const uint64_t rg = static_cast<uint64_t>(kp.rows_base + (g < kp.rows_rem ? 1 : 0));
      const uint64_t nr = std::min<uint64_t>(rg, static_cast<uint64_t>(kp.res_rows));
      rrows += nr;
      srows += rg - nr;
    }
    const double sb = static_cast<double>(srows) * rowB, zb = static_cast<double>(kp.pitch) * 8.0;
    const uint64_t dense = h_stats[2], delta = h_stats[3], maint = h_stats[1] - dense - delta;
    const uint64_t upd_terms = wd == 0 ? 0 : std::min<uint64_t>(wd, static_cast<uint64_t>(w) - 1);
    const uint64_t fused = kp.fuse_update ? upd_terms : 0;
    const uint64_t maint_upd = (kp.fuse_update ? 0 : upd_terms) + (wd == w && wd > 0 ? 1 : 0);
    double bytes = 0.0;
    bytes += static_cast<double>(dense - fused) * (sb * (kp.two_phase ? 2.0 : 1.0) + 2.0 * zb * kp.G);
    bytes += static_cast<double>(fused) * (sb * 3.0 + 2.0 * zb * kp.G);
    bytes += static_cast<double>(maint) * sb + static_cast<double>(maint_upd) * sb + static_cast<double>(rrows) * rowB;
    // (the barrier-free delta pass gathers every row of the band from L2, resident or not)
    bytes += static_cast<double>(h_stats[7]) * static_cast<double>(kp.fast_delta ? S.m : srows) * 32.0 +
             static_cast<double>(h_stats[5]) * rowB + static_cast<double>(h_stats[6]) * 2.0 * zb;
    if (kp.world > 1) bytes += static_cast<double>(dense + delta) * 2.0 * zb;  // rank partials
    res->device_bytes = static_cast<uint64_t>(bytes);
  }
  if (wd > 0) {
    SC_CUDA(ctx, cudaMemcpyAsync(res->sign_words[0], S_out, wd * wm * 8, cudaMemcpyDeviceToHost, st));
    if (!tensor) {
      SC_CUDA(ctx, cudaMemcpyAsync(res->sign_words[1], T_out, wd * wn * 8, cudaMemcpyDeviceToHost, st));
      d2h += wd * wn * 8;
    } else if (axw64) {  // split the per-term axis records into the per-axis outputs
      for (int i = 0; i < kax; ++i)
        SC_CUDA(ctx, cudaMemcpy2DAsync(res->sign_words[i + 1], words64(p->shape[i + 1]) * 8,
                                       AX_out + ax_off[i] / 2, axw64 * 8, words64(p->shape[i + 1]) * 8, wd,
                                       cudaMemcpyDeviceToHost, st));
      d2h += wd * axw64 * 8;
    }
    SC_CUDA(ctx, cudaMemcpyAsync(res->cut_value, c_out, wd * 8, cudaMemcpyDeviceToHost, st));
    d2h += wd * (wm + 1) * 8;
    if (res->sweeps) {
      SC_CUDA(ctx, cudaMemcpyAsync(res->sweeps, sweeps_out, wd * 4, cudaMemcpyDeviceToHost, st));
      d2h += wd * 4;
    }
  }
  if (res->remainder) {
    SC_CUDA(ctx, cudaMemcpy2DAsync(res->remainder, n * es, dR, rowB, n * es, m, cudaMemcpyDeviceToHost, st));
    d2h += m * n * es;
  }
  if (dsweeps != nullptr && wd > 0) {
    uint32_t n0 = 0;
    SC_CUDA(ctx, cudaMemcpyAsync(&n0, sweeps_out, 4, cudaMemcpyDeviceToHost, st));
    SC_CUDA(ctx, cudaStreamSynchronize(st));
    n0 = static_cast<uint32_t>(std::min<uint64_t>(n0, p->max_sweeps));
    SC_CUDA(ctx, cudaMemcpyAsync(res->sweep_values, dsweeps + h_stats[4] * p->max_sweeps, n0 * 8ull,
                                 cudaMemcpyDeviceToHost, st));
    res->n_sweep_values = n0;
    d2h += 4 + n0 * 8ull;
  }
  SC_CUDA(ctx, cudaStreamSynchronize(st));

  // ---- CutReport reconstruction (decompose.hpp:317-359) ----
  const double N = S.numel;  // m_global * n when row-sharded (the kernel's alpha divisor)
  res->input_norm = std::sqrt(h_norm2[0]);
  double resid_sq = h_norm2[0];
  for (uint64_t k = 0; k < wd; ++k) {
    const double c = res->cut_value[k];
    if (res->alpha) res->alpha[k] = c / N;
    const double r2 = resid_sq - c * c / N;
    resid_sq = (0.0 < r2) ? r2 : 0.0;
    if ((k + 1) % p->flush_width == 0) resid_sq = h_norm2[k + 1];  // exact re-anchor
    if (res->resid_norm) res->resid_norm[k] = std::sqrt(resid_sq);
    if (res->resid_norm_exact) res->resid_norm_exact[k] = std::sqrt(h_norm2[k + 1]);
  }
  res->final_residual_norm = std::sqrt(h_norm2[wd]);
  if (wd > 0 && res->resid_norm) res->resid_norm[wd - 1] = res->final_residual_norm;
  res->h2d_bytes = h2d;
  res->d2h_bytes = d2h;
  res->total_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  return SC_OK;
}
}  // namespace

// ---------------------------------------------------------------------------
// Row-sharded decomposition of one matrix over `world` GPUs.
namespace {
// This rank's exchange region: [zpart (local column partials) | zr (rank partial,
// read by peers) | slots | rank slot (read by peers) | tagged t words (written by
// peers) | counters].  Counters: [0] cross-rank barrier (rank 0's is used),
// [1..3] first failing pass per error class, [4] first pass of a cross-rank
// timeout, [5] this rank's local barrier, [6] abort word (rank 0's is used).
sc_status shard_alloc(sc_ctx* ctx, const sc_shard_config* cfg) {
  auto& S = ctx->shard;
  S.pitch = static_cast<long long>((cfg->n + 31) / 32 * 32);
  const uint64_t min_band = cfg->m_global / cfg->world;  // bands are floor/ceil of m/world
  S.G = cfg->ctas > 0 ? cfg->ctas : static_cast<int>(auto_ctas(ctx->num_sms, 1, min_band));
  const int Q = static_cast<int>(S.pitch / 32);
  S.tw32 = std::max(Q, static_cast<int>(2 * words64(cfg->n)));
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  S.off_zpart = 0;
  S.off_zr = al(2 * static_cast<size_t>(S.G) * S.pitch * 8);
  S.off_slots = S.off_zr + al(2 * static_cast<size_t>(S.pitch) * 8);
  S.off_rslot = S.off_slots + al(static_cast<size_t>(S.G) * sizeof(scb::Slot));
  S.off_tb64 = S.off_rslot + al(sizeof(scb::Slot));
  S.off_ctr = S.off_tb64 + al(2 * static_cast<size_t>(S.tw32) * 8 * scb::kTbStride);
  S.exch_bytes = S.off_ctr + 256;
  SC_CUDA(ctx, cudaMalloc(&S.exch, S.exch_bytes));
  S.peers[S.rank] = S.exch;
  return SC_OK;
}
}  // namespace

sc_status sc_shard_open(sc_ctx* ctx, const sc_shard_config* cfg, void* handle_out) {
  if (!ctx || !cfg || !handle_out) return SC_INVALID_ARGUMENT;
  if (cfg->world < 1 || cfg->world > 8 || cfg->rank < 0 || cfg->rank >= cfg->world || cfg->n == 0 ||
      cfg->m_global < static_cast<uint64_t>(cfg->world) || (cfg->dtype != SC_F32 && cfg->dtype != SC_F64))
    return set_err(ctx, SC_INVALID_ARGUMENT, "sc_shard_config: bad rank/world/shape/dtype");
  SC_CUDA(ctx, cudaSetDevice(ctx->device));
  sc_shard_close(ctx);
  auto& S = ctx->shard;
  S.world = cfg->world;
  S.rank = cfg->rank;
  S.dtype = cfg->dtype;
  S.m_global = cfg->m_global;
  S.row0 = cfg->row0;
  S.n = cfg->n;
  S.timeout_ms = cfg->timeout_ms;
  if (sc_status st = shard_alloc(ctx, cfg); st != SC_OK) return st;
  cudaIpcMemHandle_t h;
  SC_CUDA(ctx, cudaIpcGetMemHandle(&h, S.exch));
  std::memcpy(handle_out, &h, sizeof h);
  return sc_shard_reset(ctx);
}

sc_status sc_shard_connect(sc_ctx* ctx, const void* handles) {
  if (!ctx || !handles || !ctx->shard.exch) return SC_INVALID_ARGUMENT;
  SC_CUDA(ctx, cudaSetDevice(ctx->device));
  auto& S = ctx->shard;
  for (int r = 0; r < S.world; ++r) {
    if (r == S.rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + r * SC_IPC_HANDLE_BYTES, sizeof h);
    SC_CUDA(ctx, cudaIpcOpenMemHandle(&S.peers[r], h, cudaIpcMemLazyEnablePeerAccess));
  }
  S.connected = true;
  return SC_OK;
}

sc_status sc_shard_reset(sc_ctx* ctx) {
  if (!ctx || !ctx->shard.exch) return SC_INVALID_ARGUMENT;
  SC_CUDA(ctx, cudaSetDevice(ctx->device));
  auto& S = ctx->shard;
  char* ex = static_cast<char*>(S.exch);
  SC_CUDA(ctx, cudaMemset(ex + S.off_slots, 0, S.off_ctr - S.off_slots));  // slots, rank slot, tagged t words
  SC_CUDA(ctx, cudaMemset(ex + S.off_ctr, 0, 32));                         // barrier counters, abort word
  SC_CUDA(ctx, cudaMemset(ex + S.off_ctr + 4, 0xff, 16));                  // no error / timeout seen
  SC_CUDA(ctx, cudaDeviceSynchronize());
  return SC_OK;
}

sc_status sc_greedy_decompose_sharded(sc_ctx* ctx, const sc_problem* local, const sc_shard_config* cfg,
                                      sc_result* res) {
  if (!ctx || !local || !cfg || !res) return SC_INVALID_ARGUMENT;
  const auto& S = ctx->shard;
  if (!S.exch || !(S.connected || S.world == 1))
    return set_err(ctx, SC_INVALID_ARGUMENT, "sc_greedy_decompose_sharded: sc_shard_open/connect first");
  if (local->order != 2 || cfg->rank != S.rank || cfg->world != S.world || cfg->m_global != S.m_global ||
      cfg->n != S.n || local->shape[1] != S.n)
    return set_err(ctx, SC_INVALID_ARGUMENT, "sc_greedy_decompose_sharded: problem/config do not match the shard");
  return run_decompose(ctx, local, res, &S);
}

// Row sharding emulated on one device: `world` virtual ranks, each with its own
// child context (arena, exchange region, band of rows), launched as ONE
// cooperative kernel (sweep_kernel_vr) so that ranks that wait on one another are
// co-resident.  The peer pointers are the siblings' exchange regions.
sc_status sc_greedy_decompose_sharded_emulated(sc_ctx* ctx, const sc_problem* p, const sc_shard_emulation* opt,
                                               sc_result* res) {
  const auto t_start = std::chrono::steady_clock::now();
  if (ctx == nullptr) return SC_INVALID_ARGUMENT;
  if (res == nullptr) return set_err(ctx, SC_INVALID_ARGUMENT, "sc_result: null");
  std::string msg;
  if (validate(p, &msg) != SC_OK) return set_err(ctx, SC_INVALID_ARGUMENT, "%s", msg.c_str());
  if (p->order != 2) return set_err(ctx, SC_NOT_SUPPORTED, "emulated row sharding: matrices only");
  if (res->sign_words[0] == nullptr || res->sign_words[1] == nullptr || res->cut_value == nullptr)
    return set_err(ctx, SC_INVALID_ARGUMENT, "sc_result: sign_words of every axis and cut_value are required");
  const int world = opt ? opt->world : 1;
  if (world < 1 || world > scb::kMaxVRanks)
    return set_err(ctx, SC_INVALID_ARGUMENT, "sc_shard_emulation: world must be in [1, %d]", scb::kMaxVRanks);
  SC_CUDA(ctx, cudaSetDevice(ctx->device));
  const uint64_t m = p->shape[0], n = p->shape[1];
  const int G = (opt && opt->ctas > 0) ? opt->ctas : ctx->num_sms / world;
  if (G < 1 || static_cast<long long>(G) * world > ctx->num_sms)
    return set_err(ctx, SC_NOT_SUPPORTED, "emulated row sharding: %d ranks x %d CTAs exceed %d SMs", world, G,
                   ctx->num_sms);
  if (m / world < static_cast<uint64_t>(G))
    return set_err(ctx, SC_NOT_SUPPORTED, "emulated row sharding: bands of %llu rows are smaller than %d CTAs",
                   static_cast<unsigned long long>(m / world), G);
  const size_t es = p->dtype == SC_F32 ? 4 : 8;
  const uint64_t wmax = std::max<uint64_t>(p->width, 1), wn = words64(n);

  struct Rank {
    sc_ctx* kid = nullptr;
    uint64_t row0 = 0, rows = 0;
    uint64_t shape[2] = {0, 0};
    sc_problem prob{};
    sc_result res{};
    std::vector<uint64_t> s_words, t_words;
    std::vector<double> alpha, cut, rn, rne;
    std::vector<uint32_t> sweeps;
    RunState S;
  };
  std::vector<Rank> R(world);
  auto cleanup = [&]() {
    for (auto& r : R) {
      if (!r.kid) continue;
      sc_destroy(r.kid);  // borrowed stream/events survive; arena, pinned, exchange region freed
      r.kid = nullptr;
    }
  };
  auto fail = [&](sc_status st) {
    const std::string e = ctx->err;
    cleanup();
    ctx->err = e;
    return st;
  };
  for (int r = 0; r < world; ++r) {
    Rank& k = R[r];
    k.kid = new sc_ctx();
    sc_ctx* c = k.kid;
    c->device = ctx->device;
    c->num_sms = ctx->num_sms;
    c->smem_optin = ctx->smem_optin;
    c->smem_per_sm = ctx->smem_per_sm;
    c->stream = ctx->stream;
    c->ev0 = ctx->ev0;
    c->ev1 = ctx->ev1;
    c->borrowed = true;
    c->opts = ctx->opts;  // the parent's engine options apply to every rank
    k.row0 = static_cast<uint64_t>(r) * m / world;
    k.rows = static_cast<uint64_t>(r + 1) * m / world - k.row0;
    sc_shard_config cfg{};
    cfg.rank = r;
    cfg.world = world;
    cfg.m_global = m;
    cfg.row0 = k.row0;
    cfg.n = n;
    cfg.dtype = p->dtype;
    cfg.ctas = G;
    auto& S = c->shard;
    S.world = world;
    S.rank = r;
    S.dtype = p->dtype;
    S.m_global = m;
    S.row0 = k.row0;
    S.n = n;
    S.ipc = false;
    S.timeout_ms = opt ? opt->timeout_ms : 0;
    S.fault = (opt && opt->dead_rank == r) ? 1 : 0;
    if (sc_status st = shard_alloc(c, &cfg); st != SC_OK) {
      ctx->err = c->err;
      return fail(st);
    }
  }
  for (int r = 0; r < world; ++r) {
    auto& S = R[r].kid->shard;
    for (int q = 0; q < world; ++q) S.peers[q] = R[q].kid->shard.exch;
    S.connected = true;
    if (sc_status st = sc_shard_reset(R[r].kid); st != SC_OK) {
      ctx->err = R[r].kid->err;
      return fail(st);
    }
  }
  for (int r = 0; r < world; ++r) {
    Rank& k = R[r];
    k.shape[0] = k.rows;
    k.shape[1] = n;
    k.prob = *p;
    k.prob.shape = k.shape;
    k.prob.data = static_cast<const char*>(p->data) + k.row0 * n * es;
    k.s_words.assign(wmax * words64(k.rows), 0);
    k.t_words.assign(wmax * wn, 0);
    k.alpha.assign(wmax, 0.0);
    k.cut.assign(wmax, 0.0);
    k.rn.assign(wmax, 0.0);
    k.rne.assign(wmax, 0.0);
    k.sweeps.assign(wmax, 0);
    k.res.sign_words[0] = k.s_words.data();
    k.res.sign_words[1] = k.t_words.data();
    k.res.alpha = k.alpha.data();
    k.res.cut_value = k.cut.data();
    k.res.resid_norm = k.rn.data();
    k.res.resid_norm_exact = k.rne.data();
    k.res.sweeps = k.sweeps.data();
    k.res.remainder = res->remainder ? static_cast<char*>(res->remainder) + k.row0 * n * es : nullptr;
    if (sc_status st = prepare_run(k.kid, &k.prob, &k.res, &k.kid->shard, k.S, true); st != SC_OK) {
      ctx->err = k.kid->err;
      return fail(st);
    }
  }
  scb::KParamsVR pv{};
  pv.world = world;
  size_t smem = 0;
  for (int r = 0; r < world; ++r) {
    if (R[r].S.var.nw != R[0].S.var.nw || R[r].S.var.vpt != R[0].S.var.vpt || R[r].S.var.rg != R[0].S.var.rg ||
        R[r].S.G != G)
      return fail(set_err(ctx, SC_RUNTIME_ERROR, "emulated row sharding: ranks chose different kernels"));
    pv.r[r] = R[r].S.kp;
    smem = std::max(smem, R[r].S.smem);
  }
  if (static_cast<size_t>(smem) > ctx->smem_optin)
    return fail(set_err(ctx, SC_NOT_SUPPORTED, "emulated row sharding: %zu bytes of shared memory", smem));
  if (cudaError_t e = scb::set_smem_limit_vr(R[0].S.var, ctx->smem_optin); e != cudaSuccess)
    return fail(set_err(ctx, SC_CUDA_ERROR, "set_smem_limit_vr: %s", cudaGetErrorString(e)));
  cudaEventRecord(ctx->ev0, ctx->stream);
  if (cudaError_t e = scb::launch_sweep_vr(R[0].S.var, pv, G, smem, ctx->stream); e != cudaSuccess)
    return fail(set_err(ctx, SC_CUDA_ERROR, "launch_sweep_vr: %s", cudaGetErrorString(e)));
  cudaEventRecord(ctx->ev1, ctx->stream);
  for (int r = 0; r < world; ++r) {
    if (sc_status st = finish_run(R[r].kid, &R[r].prob, &R[r].res, R[r].S); st != SC_OK) {
      ctx->err = R[r].kid->err;
      return fail(st);
    }
  }
  // gather: every rank must hold the same t, c and sweeps (one decision everywhere)
  const uint64_t wd = R[0].res.width_done;
  for (int r = 1; r < world; ++r) {
    const Rank& k = R[r];
    if (k.res.width_done != wd || std::memcmp(k.t_words.data(), R[0].t_words.data(), wd * wn * 8) != 0 ||
        std::memcmp(k.cut.data(), R[0].cut.data(), wd * 8) != 0 ||
        std::memcmp(k.sweeps.data(), R[0].sweeps.data(), wd * 4) != 0)
      return fail(set_err(ctx, SC_RUNTIME_ERROR, "emulated row sharding: rank %d disagrees with rank 0", r));
  }
  const uint64_t wm = words64(m);
  for (uint64_t t = 0; t < wd; ++t) {
    uint64_t* dst = res->sign_words[0] + t * wm;
    std::fill(dst, dst + wm, uint64_t{0});
    for (int r = 0; r < world; ++r) {
      const Rank& k = R[r];
      const uint64_t* src = k.s_words.data() + t * words64(k.rows);
      for (uint64_t i = 0; i < k.rows; ++i)
        if ((src[i / 64] >> (i % 64)) & 1u) dst[(k.row0 + i) / 64] |= uint64_t{1} << ((k.row0 + i) % 64);
    }
  }
  std::memcpy(res->sign_words[1], R[0].t_words.data(), wd * wn * 8);
  std::memcpy(res->cut_value, R[0].cut.data(), wd * 8);
  if (res->alpha) std::memcpy(res->alpha, R[0].alpha.data(), wd * 8);
  if (res->resid_norm) std::memcpy(res->resid_norm, R[0].rn.data(), wd * 8);
  if (res->resid_norm_exact) std::memcpy(res->resid_norm_exact, R[0].rne.data(), wd * 8);
  if (res->sweeps) std::memcpy(res->sweeps, R[0].sweeps.data(), wd * 4);
  res->width_done = wd;
  res->input_norm = R[0].res.input_norm;
  res->final_residual_norm = R[0].res.final_residual_norm;
  res->passes = R[0].res.passes;
  res->dense_passes = R[0].res.dense_passes;
  res->delta_passes = R[0].res.delta_passes;
  res->device_bytes = 0;
  for (const auto& k : R) res->device_bytes += k.res.device_bytes;
  res->kernel_ms = R[0].res.kernel_ms;
  res->kernel_launches = 1;
  res->n_sweep_values = 0;
  res->h2d_bytes = 0;
  res->d2h_bytes = 0;
  for (const auto& k : R) {
    res->h2d_bytes += k.res.h2d_bytes;
    res->d2h_bytes += k.res.d2h_bytes;
  }
  cleanup();
  res->total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  return SC_OK;
}

void sc_shard_close(sc_ctx* ctx) {
  if (!ctx) return;
  auto& S = ctx->shard;
  cudaSetDevice(ctx->device);
  for (int r = 0; r < 8; ++r)
    if (S.ipc && S.peers[r] && r != S.rank) cudaIpcCloseMemHandle(S.peers[r]);
  if (S.exch) cudaFree(S.exch);
  S = sc_ctx::Shard{};
}

}  // extern "C"
