// ctx.h -- the engine context behind the opaque sc_ctx handle, shared by the
// C-ABI translation units (capi.cpp: decomposition; ops.cpp: expansion, Gram
// system, containers).  Internal: not part of the public headers.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <map>
#include <string>
#include <utility>

#include "../../include/sigcut_b200.h"

struct sc_ctx {
  int device = 0;
  int num_sms = 0;
  size_t smem_optin = 0;
  size_t smem_per_sm = 0;
  size_t l2_persist_max = 0, l2_window_max = 0;  // persisting-L2 carve-out and access-window limits
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool borrowed = false;  // stream / events belong to a parent context (emulated ranks)
  // Engine options (sc_set_option): tuning and test knobs of the decomposition
  // kernel, per context -- never read from the environment on the product path.
  struct Options {
    long long ctas = 0;           // cap on the CTA count (0: auto)
    long long delta = 1;          // sparse delta passes between dense refreshes
    long long delta_div = 0;      // delta pass only if <= n / delta_div columns flipped (0: auto, 8 or 32 by path)
    long long delta_refresh = 64; // dense refresh every delta_refresh sweeps
    long long two_phase = -1;     // dot-pass form: -1 auto (by residency), 0 fused single read, 1 two-phase
    long long stages = 0;         // TMA ring depth (0: auto)
    long long res_rows = -1;      // cap on SMEM-resident rows per CTA (-1: as many as fit)
    long long fuse_update = 1;    // rank-1 update fused into the next term's first dot pass
    long long variant = 0;        // kernel tile override nw*1000000 + vpt*10000 + rg*100 + cps (0: auto)
    long long profile = 0;        // print the clock64 breakdown (SCB_PROFILE builds; 2: per CTA)
    long long fast_delta = 1;     // delta passes exchange self-tagged records instead of meeting at a grid barrier
    long long l2_persist = 0;     // R as a persisting-L2 access window during the launch
    long long poison = 0;         // test hook: fill the device arena with NaN bytes before each call
                                  // (any read of a never-written exchange word then shows up)
  } opts;
  std::string err;
  // cached device arena and pinned staging
  void* arena = nullptr;
  size_t arena_bytes = 0;
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  // row-sharded mode (sc_shard_*): this rank's exchange region and the peers'
  struct Shard {
    int world = 0, rank = 0, G = 0, dtype = 0;
    long long pitch = 0;
    int tw32 = 0;
    uint64_t m_global = 0, row0 = 0, n = 0;
    void* exch = nullptr;
    size_t exch_bytes = 0, off_zpart = 0, off_zr = 0, off_slots = 0, off_rslot = 0, off_tb64 = 0, off_ctr = 0;
    void* peers[8] = {};
    bool connected = false;
    bool ipc = true;          // peers opened with cudaIpcOpenMemHandle (false: emulated ranks, same device)
    uint32_t timeout_ms = 0;  // bound of the kernel's cross-rank spins (0 = 30 s)
    int fault = 0;            // test hook (emulation): this rank's CTAs exit at once
  } shard;
  // auxiliary ops (expansion, Gram system, least squares): named grow-only
  // device buffers, so a driver can hold several at once
  std::map<std::string, std::pair<void*, size_t>> pool;
};

namespace scb {

inline sc_status set_err(sc_ctx* ctx, sc_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return st;
}

// Named device buffer of at least `bytes` (contents kept unless it must grow).
inline sc_status pool_get(sc_ctx* ctx, const std::string& name, size_t bytes, void** out) {
  auto& e = ctx->pool[name];
  if (e.second < bytes || e.first == nullptr) {
    if (e.first) cudaFree(e.first);
    e = {nullptr, 0};
    const size_t want = bytes < 256 ? 256 : bytes;
    cudaError_t err = cudaMalloc(&e.first, want);
    if (err != cudaSuccess) {
      e = {nullptr, 0};
      return set_err(ctx, SC_CUDA_ERROR, "cudaMalloc(%zu) for %s failed: %s", want, name.c_str(),
                     cudaGetErrorString(err));
    }
    e.second = want;
  }
  *out = e.first;
  return SC_OK;
}

inline void pool_release(sc_ctx* ctx) {
  for (auto& kv : ctx->pool)
    if (kv.second.first) cudaFree(kv.second.first);
  ctx->pool.clear();
}

}  // namespace scb

#define SC_CUDA(ctx, call)                                                                      \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      return ::scb::set_err(ctx, SC_CUDA_ERROR, "%s failed: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
