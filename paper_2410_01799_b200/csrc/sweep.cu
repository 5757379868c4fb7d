// sweep.cu -- persistent fused signed-cut kernel for sm_100a.
//
// One cooperative launch runs the whole greedy decomposition
// (reference: sigcut::greedy_decompose, inc/decompose.hpp:314-361, with the
// sweep loop of greedy_matrix_run, inc/search.hpp:145-186, and the restart
// loop of best_of_restarts, inc/search.hpp:215-233).
//
// Data layout: CTA g (one per SM) owns a contiguous band of rows of the
// remainder R (m x pitch, row-major, f32 or f64, pad columns zero).  The
// first `res_rows` rows of the band stay in shared memory for the whole run;
// the rest are streamed every pass, one row per stage, by a TMA bulk-copy
// producer thread (cp.async.bulk + mbarrier ring).
//
// Warp roles inside a CTA (no block-wide barrier inside the row loop):
//   * dot warps: `ds` of them share a row, each summing its column segment
//     of y_i = sum_j t_j R_ij (matvec_signed, inc/kernels.hpp:61-71) in f64;
//     the last segment to finish (shared-memory counter) adds the segment
//     partials in a fixed order, records y_i, s'_i = [y_i < 0] (sgn_vector,
//     sign_vector.hpp:107-114) and signals the row ready.  In the first pass
//     of a term they also apply the previous term's rank-1 deflation
//     R -= alpha s t^T (flush_pending with one term, decompose.hpp:200-214)
//     in place and accumulate ||R||_F^2.
//   * z warps: take rows in sequence order and accumulate z += s'_i R_i
//     (matvec_signed_t, inc/kernels.hpp:74-88) into f64 registers, then hand
//     the stage back to the producer.
//
// Cross-CTA exchange per pass (no float atomics, deterministic):
//   * every CTA stores its column partials and its c / ||R||^2 partials
//     (double-buffered by pass parity), then one flat counter grid barrier;
//     every CTA reduces the G scalar partials in one fixed order, so all CTAs
//     take the identical decision (stop rule c <= c_prev, max_sweeps cap,
//     restart / term bookkeeping);
//   * column slices are reduced in a fixed order by their owner CTA and
//     t' = sgn(z) is packed with __ballot_sync into the reference's LSB-first
//     words (stored with the pass index in the high half as a sanity tag);
//     a second barrier publishes them.
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "sweep.h"

namespace scb {
namespace {

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(saddr(b)), "r"(parity), "r"(0x989680u)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  while (!mbar_try_wait(b, parity)) {
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Flat counter barrier over all CTAs (fastest of the measured designs on B200,
// scripts/micro/barrier3.cu): release-add, relaxed poll, one acquire fence.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
  while (static_cast<int>(ld_relaxed(bar) - target) < 0) {
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ double flipd(double x, uint32_t m) {
  // flip_sign_if (inc/kernels.hpp:18-20): XOR of the sign bit, m in {0, 0x80000000}
  return __hiloint2double(__double2hiint(x) ^ static_cast<int>(m), __double2loint(x));
}
__device__ __forceinline__ double warp_sum(double v) {
  // butterfly: every lane ends with the same, order-fixed sum
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename E>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int N = 4;
  using T = float4;
  __device__ static void split(const float4& v, float* e) {
    e[0] = v.x; e[1] = v.y; e[2] = v.z; e[3] = v.w;
  }
  __device__ static float4 join(const float* e) { return make_float4(e[0], e[1], e[2], e[3]); }
  __device__ static float narrow(double d) { return __double2float_rn(d); }
};
template <>
struct Vec<double> {
  static constexpr int N = 2;
  using T = double2;
  __device__ static void split(const double2& v, double* e) { e[0] = v.x; e[1] = v.y; }
  __device__ static double2 join(const double* e) { return make_double2(e[0], e[1]); }
  __device__ static double narrow(double d) { return d; }
};

// sign bit (0 / 0x80000000) of column element e of vector v from packed words
template <int EPV>
__device__ __forceinline__ uint32_t vec_bits(const uint32_t* words, int v) {
  const int col0 = v * EPV;
  return (words[col0 >> 5] >> (col0 & 31)) & ((1u << EPV) - 1u);
}
__device__ __forceinline__ uint32_t bitmask(uint32_t bits, int e) { return (bits << (31 - e)) & 0x80000000u; }

// ---------------------------------------------------------------------------
template <typename E, int ND, int NZ, int ZV>
__global__ void __launch_bounds__((ND + NZ + 1) * 32, 1) sweep_kernel(const KParams p) {
  constexpr int EPV = Vec<E>::N;
  constexpr int CW = ND + NZ;  // consumer warps
  constexpr int CT = CW * 32;  // consumer threads
  constexpr int ZE = ZV * EPV; // f64 column accumulators per z thread
  static_assert(CW <= 32, "controller arrays hold 32 warps");
  using VT = typename Vec<E>::T;

  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int g = blockIdx.x;
  const int G = p.G;
  const long long pitch = p.pitch;
  const size_t rowB = static_cast<size_t>(pitch) * sizeof(E);
  const int NV = static_cast<int>(pitch / EPV);
  const int rows_g = p.rows_base + (g < p.rows_rem ? 1 : 0);
  const int r0 = g * p.rows_base + min(g, p.rows_rem);
  const int nres = min(rows_g, p.res_rows);
  const int nstream = rows_g - nres;
  const int D = p.stages;
  const int DS = p.ds;

  const Layout L = make_layout(rowB, D, p.res_rows, DS, p.rows_max, p.Q, p.zl, CW, p.sw);
  unsigned char* stage_base = smem + L.stage;
  unsigned char* res_base = smem + L.res;
  Ctl* ctl = reinterpret_cast<Ctl*>(smem + L.ctl);
  volatile double* red = reinterpret_cast<volatile double*>(smem + L.red);  // [slot][ds]
  double* yrow = reinterpret_cast<double*>(smem + L.yrow);                  // [rows_max]
  uint32_t* tws = reinterpret_cast<uint32_t*>(smem + L.tws);                // [Q] t of this pass
  uint32_t* uws = reinterpret_cast<uint32_t*>(smem + L.uws);                // [Q] t of the update
  int* cnt = reinterpret_cast<int*>(smem + L.cnt);                          // [slot]
  volatile int* negf = reinterpret_cast<volatile int*>(smem + L.negf);      // [slot]
  unsigned long long* ready = reinterpret_cast<unsigned long long*>(smem + L.ready);  // [slot]
  double* zseg = reinterpret_cast<double*>(smem + L.zseg);                  // [zl][CW][32]
  uint32_t* sb = reinterpret_cast<uint32_t*>(smem + L.sb);                  // [3][sw]
  E* R = static_cast<E*>(p.R);

  if (tid == 0) {
    for (int s = 0; s < D; ++s) {
      mbar_init(&ctl->full[s], 1);
      mbar_init(&ctl->empty[s], NZ);
    }
    for (int s = 0; s < D + p.res_rows; ++s) mbar_init(&ready[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int k0 = p.width == 0 ? (F_NORM | F_WB | F_CHECK) : (F_DOT | F_NORM | F_CHECK);
    ctl->kind = k0;
    ctl->kind_ring[0] = k0;
    ctl->decided = 1;
    ctl->stored = 0;
    ctl->abort = 0;
    ctl->pp = 0;
    ctl->term = 0;
    ctl->restart = 0;
    ctl->tsel = -1;
    ctl->utsel = 0;
    ctl->best_tsel = 0;
    ctl->best_sweeps = 0;
    ctl->cur = 0;
    ctl->nxt = 1;
    ctl->best = 2;
    ctl->need_reduce = 0;
    ctl->norm_idx = 0;
    ctl->alpha = 0.0;
    ctl->c_prev = -INFINITY;
    ctl->best_c = 0.0;
    ctl->first_value = 0.0;
  }
  for (int i = tid; i < 3 * p.sw; i += blockDim.x) sb[i] = 0u;
  for (int i = tid; i < D + p.res_rows; i += blockDim.x) cnt[i] = 0;
  // resident rows: loaded once for the whole decomposition
  for (int l = 0; l < nres; ++l) {
    const VT* src = reinterpret_cast<const VT*>(R + static_cast<size_t>(r0 + l) * pitch);
    VT* dst = reinterpret_cast<VT*>(res_base + static_cast<size_t>(l) * rowB);
    for (int v = tid; v < NV; v += blockDim.x) dst[v] = __ldcg(src + v);
  }
  __syncthreads();

  // ======================= TMA producer (one thread) =======================
  if (warp == CW) {
    if (lane != 0 || nstream == 0) return;
    unsigned q = 0;
    int prev_kind = 0;
    long long pwait = 0;
    for (int P = 0;; ++P) {
      while (ctl->decided <= P) {
        if (ctl->abort) goto drain;
        __nanosleep(32);
      }
      {
        const int kind = ctl->kind_ring[P & 3];
        if (kind & K_TERM) break;
        if (prev_kind & F_UPD) {  // streamed rows were rewritten in pass P-1
          while (ctl->stored < P) {
            if (ctl->abort) goto drain;
            __nanosleep(32);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (int j = 0; j < nstream; ++j, ++q) {
          const int s = static_cast<int>(q % D);
          if (q >= static_cast<unsigned>(D)) {
            const uint32_t ph = ((q / D) & 1u) ^ 1u;
            const long long tw0 = p.prof ? clock64() : 0;
            while (!mbar_try_wait(&ctl->empty[s], ph)) {
              if (ctl->abort) goto drain;
            }
            if (p.prof) pwait += clock64() - tw0;
          }
          mbar_expect_tx(&ctl->full[s], static_cast<uint32_t>(rowB));
          bulk_g2s(stage_base + static_cast<size_t>(s) * rowB,
                   R + static_cast<size_t>(r0 + nres + j) * pitch, static_cast<uint32_t>(rowB), &ctl->full[s]);
        }
        prev_kind = kind;
      }
    }
  drain:
    for (unsigned k = (q > static_cast<unsigned>(D) ? q - D : 0u); k < q; ++k)
      mbar_wait(&ctl->full[k % D], (k / D) & 1u);
    if (p.prof) p.prof[g * 16 + 7] = static_cast<unsigned long long>(pwait);
    return;
  }

  // ========================= consumers (CT threads) ========================
  unsigned long long* prof = p.prof;  // optional clock64 breakdown (SCB_PROF=1)
  long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const unsigned* errp = p.err_pass;
  const bool is_dot = warp < ND;
  const int nrf = ND / DS;                    // rows in flight in the dot stage
  const int rgrp = warp / DS, part = warp % DS;
  const int vb = (part * NV) / DS, ve = ((part + 1) * NV) / DS;
  const int zt = tid - ND * 32;               // z thread index (z warps)
  int qs = 0, qph = 0;                        // stage / phase of this pass's first streamed row
  unsigned epoch = 0;                         // grid barriers passed (thread 0)

  for (int P = 0;; ++P) {
    const int kind = ctl->kind;
    if (kind & K_TERM) break;
    const int pp = ctl->pp;
    long long t_pass0 = prof ? clock64() : 0;
    const uint32_t* s_cur = sb + ctl->cur * p.sw;
    uint32_t* s_nxt = sb + ctl->nxt * p.sw;
    const uint32_t* s_upd = sb + ctl->best * p.sw;
    const double alpha = ctl->alpha;

    // ---- stage the sign words of this pass in shared memory ----
    if (kind & F_DOT) {
      if (ctl->tsel < 0) {
        const uint32_t* tw =
            p.t0 + (static_cast<size_t>(ctl->term) * p.restarts + ctl->restart) * p.t0_stride;
        for (int i = tid; i < p.Q; i += CT) tws[i] = __ldg(tw + i);
      } else {
        // t words tagged with the pass index: poll the data itself
        const unsigned long long* tw = p.tb64 + static_cast<size_t>(ctl->tsel) * p.Q;
        for (int i = tid; i < p.Q; i += CT) {
          unsigned long long x;
          do {
            x = ld_relaxed64(tw + i);
          } while (static_cast<int>(static_cast<unsigned>(x >> 32) - static_cast<unsigned>(P)) < 0);
          tws[i] = static_cast<uint32_t>(x);
        }
      }
      if (tid == 0)
        for (int i = 0; i < p.sw; ++i) s_nxt[i] = 0u;
    }
    if (kind & F_UPD) {
      for (int i = tid; i < p.Q; i += CT)
        uws[i] = ctl->utsel == 2 ? __ldcg(p.tbest + i)
                                 : static_cast<uint32_t>(__ldcg(p.tb64 + static_cast<size_t>(ctl->utsel) * p.Q + i));
    }
    consumer_sync(CT);

    double zacc[ZE];
#pragma unroll
    for (int i = 0; i < ZE; ++i) zacc[i] = 0.0;
    double nacc = 0.0;
    bool bad = false;

    if (is_dot) {
      // ========================= dot warps =========================
      // streamed row k of this pass lives in stage (qs + k) % D, phase qph ^ ...
      int js = rgrp < nres ? rgrp : rgrp;  // first row of this group
      int sslot = 0, sph = 0;               // stage / phase of this group's next streamed row
      {
        int j0 = rgrp;
        while (j0 < nres) j0 += nrf;
        const int t = qs + (j0 - nres);
        sslot = t % (D > 0 ? D : 1);
        sph = qph ^ ((t / (D > 0 ? D : 1)) & 1);
      }
      for (int j = js; j < rows_g; j += nrf) {
        const bool streamed = j >= nres;
        int slot;
        unsigned char* rowp;
        if (!streamed) {
          slot = D + j;
          rowp = res_base + static_cast<size_t>(j) * rowB;
        } else {
          slot = sslot;
          if (prof && tid == 0) {
            const long long tw0 = clock64();
            mbar_wait(&ctl->full[slot], static_cast<uint32_t>(sph));
            pacc[0] += clock64() - tw0;
          } else {
            mbar_wait(&ctl->full[slot], static_cast<uint32_t>(sph));
          }
          rowp = stage_base + static_cast<size_t>(slot) * rowB;
          sslot += nrf;
          while (sslot >= D) {
            sslot -= D;
            sph ^= 1;
          }
        }
        VT* rv = reinterpret_cast<VT*>(rowp);
        if (kind & (F_UPD | F_WB)) {
          const uint32_t sneg = ((s_upd[j >> 5] >> (j & 31)) & 1u) << 31;
          VT* grow = reinterpret_cast<VT*>(R + static_cast<size_t>(r0 + j) * pitch);
          for (int v = vb + lane; v < ve; v += 32) {
            E x[EPV];
            Vec<E>::split(rv[v], x);
            if (kind & F_UPD) {
              const uint32_t ub = vec_bits<EPV>(uws, v);
#pragma unroll
              for (int e = 0; e < EPV; ++e)
                if (v * EPV + e < p.n)  // flush_pending with one term: data += flip(-alpha, s_i ^ t_j)
                  x[e] = Vec<E>::narrow(static_cast<double>(x[e]) + flipd(-alpha, sneg ^ bitmask(ub, e)));
              rv[v] = Vec<E>::join(x);
            }
            if (streamed || (kind & F_WB)) grow[v] = Vec<E>::join(x);
          }
        }
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        if (kind == F_DOT) {
          // hot loop: 4 vectors in flight per lane, one f64 chain per vector slot
          int v = vb + lane;
          for (; v + 96 < ve; v += 128) {
            E x[4][EPV];
            uint32_t bb[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) Vec<E>::split(rv[v + 32 * u], x[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) bb[u] = vec_bits<EPV>(tws, v + 32 * u);
#pragma unroll
            for (int e = 0; e < EPV; ++e) {
              a0 += flipd(static_cast<double>(x[0][e]), bitmask(bb[0], e));
              a1 += flipd(static_cast<double>(x[1][e]), bitmask(bb[1], e));
              a2 += flipd(static_cast<double>(x[2][e]), bitmask(bb[2], e));
              a3 += flipd(static_cast<double>(x[3][e]), bitmask(bb[3], e));
            }
          }
          for (; v < ve; v += 32) {
            E x[EPV];
            Vec<E>::split(rv[v], x);
            const uint32_t b = vec_bits<EPV>(tws, v);
#pragma unroll
            for (int e = 0; e < EPV; ++e) a0 += flipd(static_cast<double>(x[e]), bitmask(b, e));
          }
        } else if (kind & (F_DOT | F_NORM)) {
          for (int v = vb + lane; v < ve; v += 32) {
            E x[EPV];
            Vec<E>::split(rv[v], x);
            const uint32_t b = (kind & F_DOT) ? vec_bits<EPV>(tws, v) : 0u;
#pragma unroll
            for (int e = 0; e < EPV; ++e) {
              const double d = static_cast<double>(x[e]);
              if (kind & F_NORM) {
                nacc += d * d;
                if (kind & F_CHECK) bad |= !isfinite(d);
              }
              const double f = flipd(d, bitmask(b, e));
              if (e & 1) a1 += f; else a0 += f;
            }
          }
        }
        const double part_y = warp_sum((a0 + a1) + (a2 + a3));
        if (lane == 0) {
          red[slot * DS + part] = part_y;
          __threadfence_block();
          if (atomicAdd(&cnt[slot], 1) == DS - 1) {
            __threadfence_block();
            double y = 0.0;
            for (int q = 0; q < DS; ++q) y += red[slot * DS + q];
            cnt[slot] = 0;
            if (kind & F_DOT) {
              yrow[j] = y;
              negf[slot] = y < 0.0 ? 1 : 0;
              if (!isfinite(y)) atomicMin(const_cast<unsigned*>(errp) + ERR_Y, static_cast<unsigned>(P));
              if (y < 0.0) atomicOr(&s_nxt[j >> 5], 1u << (j & 31));
            }
            __threadfence_block();
            mbar_arrive(&ready[slot]);
          }
        }
      }
    } else {
      // ========================== z warps ==========================
      int sslot = qs, sph = qph;
      bool zvalid[ZV];
      int zv_idx[ZV];
#pragma unroll
      for (int k = 0; k < ZV; ++k) {
        const int v = zt + k * NZ * 32;
        zvalid[k] = v < NV;
        zv_idx[k] = v < NV ? v : 0;  // always a valid address; contribution masked
      }
      for (int j = 0; j < rows_g; ++j) {
        const bool streamed = j >= nres;
        int slot;
        uint32_t par;
        const VT* rv;
        if (!streamed) {
          slot = D + j;
          par = static_cast<uint32_t>(P & 1);
          rv = reinterpret_cast<const VT*>(res_base + static_cast<size_t>(j) * rowB);
        } else {
          slot = sslot;
          par = static_cast<uint32_t>(sph);
          rv = reinterpret_cast<const VT*>(stage_base + static_cast<size_t>(slot) * rowB);
          if (++sslot == D) {
            sslot = 0;
            sph ^= 1;
          }
        }
        if (prof && zt == 0) {
          const long long tw0 = clock64();
          mbar_wait(&ready[slot], par);
          pacc[5] += clock64() - tw0;
        } else {
          mbar_wait(&ready[slot], par);
        }
        if (kind & F_DOT) {
          const uint32_t negm = negf[slot] ? 0x80000000u : 0u;
          constexpr int ZH = ZV > 4 ? 4 : ZV;  // loads in flight per group (register budget)
#pragma unroll
          for (int k0 = 0; k0 < ZV; k0 += ZH) {
            E x[ZH][EPV];
#pragma unroll
            for (int k = 0; k < ZH; ++k) Vec<E>::split(rv[zv_idx[k0 + k]], x[k]);
#pragma unroll
            for (int k = 0; k < ZH; ++k)
#pragma unroll
              for (int e = 0; e < EPV; ++e)
                if (zvalid[k0 + k]) zacc[(k0 + k) * EPV + e] += flipd(static_cast<double>(x[k][e]), negm);
          }
        }
        if (streamed) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&ctl->empty[slot]);
        }
      }
    }
    if (D > 0) {  // advance the stage ring past this pass's streamed rows
      const int t = qs + nstream;
      qph ^= (t / D) & 1;
      qs = t % D;
    }
    if (prof && zt == 0) pacc[6] += clock64() - t_pass0;

    // ------------------------------ pass end ------------------------------
    if (prof && tid == 0) {
      const long long t = clock64();
      pacc[1] += t - t_pass0;
      t_pass0 = t;
    }
    if (kind & (F_UPD | F_WB)) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __threadfence();
    }
    if (!is_dot && (kind & F_DOT)) {
      double* zrow = p.zpart + static_cast<size_t>(g) * pitch;
#pragma unroll
      for (int k = 0; k < ZV; ++k) {
        const int v = zt + k * NZ * 32;
        if (v < NV) {
#pragma unroll
          for (int e = 0; e < EPV; e += 2)
            __stcg(reinterpret_cast<double2*>(zrow + v * EPV + e),
                   make_double2(zacc[k * EPV + e], zacc[k * EPV + e + 1]));
        }
      }
    }
    if (is_dot && (kind & F_NORM)) {
      const double ws = warp_sum(nacc);
      if (lane == 0) ctl->nred[warp] = ws;
      if (bad) atomicMin(const_cast<unsigned*>(errp) + ERR_INPUT, static_cast<unsigned>(P));
    }
    consumer_sync(CT);
    if (warp == 0) {
      // this CTA's c partial: sum_i s_i y_i in row order (lane-strided, fixed tree)
      double cl = 0.0;
      if ((kind & F_DOT) && pp >= 1)
        for (int j = lane; j < rows_g; j += 32)
          cl += flipd(yrow[j], ((s_cur[j >> 5] >> (j & 31)) & 1u) << 31);
      cl = warp_sum(cl);
      if (lane == 0) {
        if (kind & (F_UPD | F_WB)) {
          __threadfence_block();
          ctl->stored = P + 1;
        }
        double nsum = 0.0;
        if (kind & F_NORM)
          for (int w = 0; w < ND; ++w) nsum += ctl->nred[w];
        Slot* my = p.slots + g;
        __stcg(&my->c[P & 1], cl);
        __stcg(&my->n[P & 1], nsum);
      }
    }
    consumer_sync(CT);
    if (tid == 0) grid_barrier(p.bar, ++epoch * static_cast<unsigned>(G));
    consumer_sync(CT);
    {
      // every CTA reduces the G partials in the same fixed order
      double cs = 0.0, ns = 0.0;
      for (int i = tid; i < G; i += CT) {
        const Slot* s = p.slots + i;
        cs += __ldcg(&s->c[P & 1]);
        ns += __ldcg(&s->n[P & 1]);
      }
      cs = warp_sum(cs);
      ns = warp_sum(ns);
      consumer_sync(CT);  // thread 0 is done reading ctl->nred of the norm step
      if (lane == 0) {
        ctl->cred[warp] = cs;
        ctl->nred[warp] = ns;
      }
    }
    consumer_sync(CT);
    if (prof && tid == 0) {
      const long long t = clock64();
      pacc[2] += t - t_pass0;
      t_pass0 = t;
    }

    // ------------------------------ decision ------------------------------
    if (tid == 0) {
      double cs = 0.0, ns = 0.0;
      for (int w = 0; w < CW; ++w) {
        cs += ctl->cred[w];
        ns += ctl->nred[w];
      }
      int next;
      int need_reduce = 0;
      const unsigned ey = __ldcg(errp + ERR_Y), ei = __ldcg(errp + ERR_INPUT), ez = __ldcg(errp + ERR_Z);
      if (ey <= static_cast<unsigned>(P) || ei <= static_cast<unsigned>(P) ||
          ez < static_cast<unsigned>(P)) {
        next = K_TERM;
      } else {
        if ((kind & F_NORM) && g == 0) p.norm2_out[ctl->norm_idx] = ns;
        if (!(kind & F_DOT)) {
          next = K_TERM;
        } else if (pp == 0) {
          const int t = ctl->cur;  // s_1 (just computed) becomes current
          ctl->cur = ctl->nxt;
          ctl->nxt = t;
          ctl->pp = 1;
          ctl->tsel = 1;
          need_reduce = 1;
          next = F_DOT;
        } else {
          const double c = cs;
          const bool stop = (c <= ctl->c_prev) || (pp >= p.max_sweeps);
          if (!stop) {
            ctl->c_prev = c;
            const int t = ctl->cur;
            ctl->cur = ctl->nxt;
            ctl->nxt = t;
            ctl->pp = pp + 1;
            ctl->tsel = (pp + 1) & 1;
            need_reduce = 1;
            next = F_DOT;
          } else {
            // restart result (c, s_pp, t_pp, pp): search.hpp:178-180 / :185
            const bool better = (ctl->restart == 0) || (c > ctl->best_c);
            if (better) {
              ctl->best_c = c;
              ctl->best_sweeps = pp;
              uint32_t* sbest = sb + ctl->best * p.sw;
              for (int i = 0; i < p.sw; ++i) sbest[i] = s_cur[i];
              if (ctl->restart + 1 < p.restarts) {
                if (g == 0) {
                  const unsigned long long* src = p.tb64 + static_cast<size_t>(pp & 1) * p.Q;
                  for (int i = 0; i < p.Q; ++i) p.tbest[i] = static_cast<uint32_t>(__ldcg(src + i));
                }
                ctl->best_tsel = 2;
              } else {
                ctl->best_tsel = pp & 1;
              }
            }
            ctl->restart += 1;
            if (ctl->restart < p.restarts) {
              ctl->pp = 0;
              ctl->tsel = -1;
              ctl->c_prev = -INFINITY;
              next = F_DOT;
            } else {
              const long long term = ctl->term;
              const double bc = ctl->best_c;
              const bool accept = (term == 0) || !(bc < p.min_frac * ctl->first_value);
              if (accept) {
                if (term == 0) ctl->first_value = bc;
                // record term (CutDecomposition::append_term, decompose.hpp:341)
                const uint32_t* sbest = sb + ctl->best * p.sw;
                uint32_t* srow = p.S_out + static_cast<size_t>(term) * p.s_stride;
                for (int l = 0; l < rows_g; ++l)
                  if ((sbest[l >> 5] >> (l & 31)) & 1u) {
                    const int i = r0 + l;
                    atomicOr(srow + (i >> 5), 1u << (i & 31));
                  }
                if (g == 0) {
                  uint32_t* trow = p.T_out + static_cast<size_t>(term) * p.t_stride;
                  const int nw = min(p.t_stride, p.Q);  // words past Q are pad (zero)
                  if (ctl->best_tsel == 2) {
                    for (int i = 0; i < nw; ++i) trow[i] = __ldcg(p.tbest + i);
                  } else {
                    const unsigned long long* src = p.tb64 + static_cast<size_t>(ctl->best_tsel) * p.Q;
                    for (int i = 0; i < nw; ++i) trow[i] = static_cast<uint32_t>(__ldcg(src + i));
                  }
                  for (int i = nw; i < p.t_stride; ++i) trow[i] = 0u;
                  p.c_out[term] = bc;
                  p.sweeps_out[term] = static_cast<uint32_t>(ctl->best_sweeps);
                  p.stats[0] = static_cast<unsigned long long>(term + 1);
                }
                ctl->alpha = bc / p.numel_d;  // alpha = c / numel (decompose.hpp:340)
                ctl->utsel = ctl->best_tsel;
                ctl->term = static_cast<int>(term + 1);
                ctl->norm_idx = static_cast<int>(term + 1);
                if (term + 1 >= p.width) {
                  next = F_UPD | F_NORM | F_WB;
                } else {
                  next = F_DOT | F_UPD | F_NORM;
                  ctl->pp = 0;
                  ctl->restart = 0;
                  ctl->tsel = -1;
                  ctl->c_prev = -INFINITY;
                }
              } else {
                // min_value_fraction stop (decompose.hpp:337-338): nothing appended
                ctl->norm_idx = static_cast<int>(term);
                next = F_NORM | F_WB;
              }
            }
          }
        }
      }
      ctl->kind = next;
      ctl->need_reduce = need_reduce;
      ctl->kind_ring[(P + 1) & 3] = next;
      __threadfence_block();
      ctl->decided = P + 2;
      if ((next & K_TERM) && g == 0) p.stats[1] = static_cast<unsigned long long>(P + 1);
    }
    consumer_sync(CT);
    if (prof && tid == 0) {
      const long long t = clock64();
      pacc[3] += t - t_pass0;
      t_pass0 = t;
    }

    // --------------------- column reduction: t' = sgn(z) ---------------------
    if (ctl->need_reduce) {
      unsigned long long* tout = p.tb64 + static_cast<size_t>(ctl->tsel & 1) * p.Q;
      const unsigned long long tag = static_cast<unsigned long long>(P + 1) << 32;
      const int gs = (warp * G) / CW, ge = ((warp + 1) * G) / CW;
      for (int q0 = g; q0 < p.Q; q0 += G * p.zl) {
        int nls = 0;
        for (int j = 0; j < p.zl && q0 + j * G < p.Q; ++j) nls = j + 1;
        for (int j = 0; j < nls; ++j) {
          const int col = (q0 + j * G) * 32 + lane;
          const double* zp = p.zpart + col;
          double a = 0.0;
          for (int g0 = gs; g0 < ge; g0 += 16) {  // 16 independent L2 loads in flight
            double v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = (g0 + u < ge) ? __ldcg(zp + static_cast<size_t>(g0 + u) * pitch) : 0.0;
#pragma unroll
            for (int u = 0; u < 16; ++u) a += v[u];
          }
          zseg[(j * CW + warp) * 32 + lane] = a;
        }
        consumer_sync(CT);
        for (int j = warp; j < nls; j += CW) {
          const int qq = q0 + j * G;
          const int col = qq * 32 + lane;
          double z = 0.0;
#pragma unroll
          for (int w = 0; w < CW; ++w) z += zseg[(j * CW + w) * 32 + lane];
          const bool valid = col < p.n;
          if (valid && !isfinite(z)) atomicMin(const_cast<unsigned*>(errp) + ERR_Z, static_cast<unsigned>(P));
          const unsigned word = __ballot_sync(0xffffffffu, valid && z < 0.0);
          if (lane == 0) st_relaxed64(tout + qq, tag | word);
        }
        consumer_sync(CT);
      }
      if (tid == 0) grid_barrier(p.bar, ++epoch * static_cast<unsigned>(G));
      consumer_sync(CT);
      if (prof && tid == 0) pacc[4] += clock64() - t_pass0;
    }
  }
  if (tid == 0) ctl->abort = 1;  // release a producer still waiting on an unconsumed stage
  if (prof && tid == 0)
    for (int i = 0; i < 5; ++i) prof[g * 16 + i] = static_cast<unsigned long long>(pacc[i]);
  if (prof && zt == 0)
    for (int i = 5; i < 7; ++i) prof[g * 16 + i] = static_cast<unsigned long long>(pacc[i]);
}

template <typename E, int ND, int NZ, int ZV>
struct Kern {
  static void* fn() { return reinterpret_cast<void*>(&sweep_kernel<E, ND, NZ, ZV>); }
};

void* kernel_for(const Variant& v) {
#define SCB_K(E, ND, NZ, ZV) \
  if (v.nd == ND && v.nz == NZ && v.zv == ZV) return Kern<E, ND, NZ, ZV>::fn();
  if (v.dtype == 0) {
    SCB_K(float, 4, 1, 1)
    SCB_K(float, 4, 1, 4)
    SCB_K(float, 8, 2, 4)
    SCB_K(float, 8, 4, 4)
    SCB_K(float, 8, 4, 8)
    SCB_K(float, 8, 8, 4)
    SCB_K(float, 8, 8, 8)
  } else {
    SCB_K(double, 4, 1, 1)
    SCB_K(double, 4, 1, 4)
    SCB_K(double, 8, 2, 4)
    SCB_K(double, 8, 4, 4)
    SCB_K(double, 8, 4, 8)
    SCB_K(double, 8, 8, 8)
    SCB_K(double, 8, 8, 16)
  }
#undef SCB_K
  return nullptr;
}

}  // namespace

int pick_variant(int dtype, long long pitch, Variant* v) {
  // nd dot warps + nz z warps (+ 1 producer warp); a z thread owns zv 16-byte
  // column vectors (zv * elements-per-vector f64 accumulators in registers).
  const int epv = dtype == 0 ? 4 : 2;
  const long long nv = pitch / epv;
  v->dtype = dtype;
  struct C { int nd, nz, zv; };
  static const C table[] = {{4, 1, 1}, {4, 1, 4}, {8, 2, 4}, {8, 4, 4}, {8, 4, 8}, {8, 8, 8}};
  bool found = false;
  for (const C& c : table) {
    if (static_cast<long long>(c.nz) * 32 * c.zv >= nv) {
      v->nd = c.nd; v->nz = c.nz; v->zv = c.zv;
      found = true;
      break;
    }
  }
  if (!found) {
    if (dtype == 1 && nv <= 8 * 32 * 16) {
      v->nd = 8; v->nz = 8; v->zv = 16;
    } else {
      return 1;
    }
  }
  if (const char* e = std::getenv("SCB_VARIANT")) {  // tuning override "nd,nz,zv"
    Variant t = *v;
    if (std::sscanf(e, "%d,%d,%d", &t.nd, &t.nz, &t.zv) == 3 && kernel_for(t) != nullptr &&
        static_cast<long long>(t.nz) * 32 * t.zv >= nv)
      *v = t;
  }
  return 0;
}

cudaError_t set_smem_limit(const Variant& v, size_t bytes) {
  void* f = kernel_for(v);
  if (!f) return cudaErrorInvalidValue;
  return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}

cudaError_t launch_sweep(const Variant& v, const KParams& p, size_t smem_bytes, cudaStream_t st) {
  void* f = kernel_for(v);
  if (!f) return cudaErrorInvalidValue;
  KParams copy = p;
  void* args[] = {&copy};
  return cudaLaunchCooperativeKernel(f, dim3(p.G), dim3((v.nd + v.nz + 1) * 32), args, smem_bytes, st);
}

}  // namespace scb
