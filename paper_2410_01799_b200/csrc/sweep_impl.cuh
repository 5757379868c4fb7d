// sweep_impl.cuh -- persistent fused signed-cut kernel for sm_100a (included by the
// per-variant translation units sweep_k_*.cu, compiled in parallel).
#pragma once
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
// Passes (one per sweep; SURVEY §3.2 "equivalent GPU sweep schedule"):
//   * dense dot pass: y = R t, s' = sgn(y) (sgn_vector, sign_vector.hpp:107-114),
//     z = R^T s' (matvec_signed / _t, kernels.hpp:61-88), all in f64 from f32 or
//     f64 storage.  Two forms: two-phase (A: per-warp row partials, B: y and s',
//     C: z streaming the rows again -- while R is L2-resident) and fused single
//     read (rows in registers, a one-group lag between the dot of g and the z
//     update of g-1 -- once R spills to HBM).  Wide rows go as column chunks.
//   * delta dot pass (the GPU form of the reference's delta caches,
//     kernels.hpp:92-156): y += 2 t'_c R[:, c] over the flipped columns only; the
//     CTA publishes its flipped rows, and the column owners add 2 s'_i R[i, cols]
//     for them to their z state.  A dense refresh runs every 64 sweeps.
//   * the first dot pass of each term also applies the previous term's rank-1
//     deflation R -= alpha s t^T (flush_pending with one term,
//     decompose.hpp:200-214) to every row as it streams it, writes R back and
//     accumulates ||R||^2 (north-star kernel 3: sweeps + 1 passes per cut).
//   * maintenance passes (norm of the input, the final update and write-back).
//
// Cross-CTA exchange per pass (no float atomics, deterministic):
//   * every CTA stores its c / ||R||^2 partials (pass-parity slots) and, in dense
//     passes, its column partial row (in delta passes its flip words), then one
//     flat counter grid barrier; every CTA reduces the G slots in one fixed
//     order, so all CTAs take the identical decision (stop rule c <= c_prev,
//     max_sweeps cap, restart / term bookkeeping);
//   * the owner CTA of each 32-column word reduces its columns in a fixed order
//     (dense: the G partials; delta: the flipped rows) and publishes
//     t' = sgn(z), packed with __ballot_sync into the reference's LSB-first
//     words, tagged with the pass index; the next pass polls the tags (no second
//     barrier).
//   * row-sharded (MR instantiations, world > 1): the same per rank, then the
//     rank partials cross NVLink behind one bounded system-scope barrier.
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

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
#ifndef SCB_WAIT_HINT_NS
#define SCB_WAIT_HINT_NS 0
#endif
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* b, uint32_t parity) {
  uint32_t ok;
#if SCB_WAIT_HINT_NS > 0
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(saddr(b)), "r"(parity), "r"(SCB_WAIT_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(saddr(b)), "r"(parity)
      : "memory");
#endif
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

// the same across GPUs: the counter lives on rank 0, peers reach it over NVLink
__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Bounded spin of the row-sharded (world > 1) exchange: every 256 polls it checks
// the shared abort word (rank 0's) and the elapsed time; a timeout sets the abort
// word so every other waiting CTA of every rank gives up too.  Returns false then.
struct SpinBound {
  unsigned* abort_word;
  long long timeout_ns;
  unsigned long long t0;
  unsigned it;
  __device__ __forceinline__ bool ok() {
    if ((++it & 255u) != 0u) return true;
    if (ld_relaxed_sys(abort_word) != 0u) return false;
    const unsigned long long t = global_ns();
    if (t0 == 0) {
      t0 = t;
    } else if (static_cast<long long>(t - t0) > timeout_ns) {
      atomicExch_system(abort_word, 1u);
      return false;
    }
    return true;
  }
};
// Cross-rank barrier (counter on rank 0, reached over NVLink) and the rank-local
// one of a sharded run, both bounded by the abort word / timeout.
template <bool SYS>
__device__ __noinline__ bool grid_barrier_bounded(unsigned* bar, unsigned target, unsigned* abort_word,
                                                  long long timeout_ns) {
  if (SYS)
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
  else
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
  SpinBound sb{abort_word, timeout_ns, 0ull, 0u};
  while (static_cast<int>((SYS ? ld_relaxed_sys(bar) : ld_relaxed(bar)) - target) < 0)
    if (!sb.ok()) return false;
  if (SYS)
    asm volatile("fence.acq_rel.sys;" ::: "memory");
  else
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  return true;
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed64_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
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
// Exact f32 -> f64 widening without F2F (which issues on the quarter-rate XU
// pipe): the f32 bits shifted right by 3 (arithmetic, so the sign lands in bit
// 31 after masking bits 28-30) form a double whose exponent field is the f32
// exponent; scaling by 2^(1023-127) in the accumulating DFMA restores the
// value exactly (f32 subnormals become f64 subnormals, which the FP64 pipe
// handles at full precision; zero stays zero).  The t sign flip folds into the
// same LOP3.  Per element: IMAD.HI + LOP3 + SHF/IMAD + DFMA, no XU.
constexpr double kRebias = 0x1p896;
// Same exact widening with 32-bit shifts (SHF + LOP3 + SHL on the full-rate
// ALU / FMA pipes instead of the quarter-rate IMAD.WIDE).
__device__ __forceinline__ double widen_shf(float x, uint32_t m) {
  const uint32_t u = __float_as_uint(x);
  const uint32_t hi = (static_cast<uint32_t>(static_cast<int>(u) >> 3) & 0x8fffffffu) ^ m;
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(u << 29));
}
__device__ __forceinline__ double widen_shf(double x, uint32_t m) { return flipd(x, m); }

template <typename E>
struct Wide;
template <>
struct Wide<float> {
  __device__ static double prep(float x, uint32_t m, int wmul) {
    const long long w = static_cast<long long>(static_cast<int>(__float_as_uint(x))) * static_cast<long long>(wmul);
    const uint32_t hi = (static_cast<uint32_t>(static_cast<unsigned long long>(w) >> 32) & 0x8fffffffu) ^ m;
    return __hiloint2double(static_cast<int>(hi), static_cast<int>(static_cast<uint32_t>(w)));
  }
  __device__ static double dot(double acc, double w) { return fma(w, kRebias, acc); }
  __device__ static double zscale(double sg) { return sg * kRebias; }
};
template <>
struct Wide<double> {
  __device__ static double prep(double x, uint32_t m, int) { return flipd(x, m); }
  __device__ static double dot(double acc, double w) { return acc + w; }
  __device__ static double zscale(double sg) { return sg; }
};


// Sum RG per-lane partials over the warp with a transposed butterfly: the first
// log2(RG) levels exchange whole rows (each lane keeps half of its rows), the
// remaining levels reduce one value.  Row r's total ends up in lane
// holder_lane<RG>(r); the addition order is fixed, so results are reproducible.
template <int RG>
__device__ __forceinline__ double warp_reduce_rows(double (&p)[RG], int lane) {
  if constexpr (RG == 1) {
    double v = p[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  } else if constexpr (RG == 2) {
    const bool up = lane & 16;
    const double keep = up ? p[1] : p[0], send = up ? p[0] : p[1];
    double v = keep + __shfl_xor_sync(0xffffffffu, send, 16);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  } else {
    static_assert(RG == 4, "RG must be 1, 2 or 4");
    const bool up = lane & 16;
    const double k0 = up ? p[2] : p[0], k1 = up ? p[3] : p[1];
    const double s0 = up ? p[0] : p[2], s1 = up ? p[1] : p[3];
    const double q0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 16);
    const double q1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 16);
    const bool b3 = lane & 8;
    double v = (b3 ? q1 : q0) + __shfl_xor_sync(0xffffffffu, b3 ? q0 : q1, 8);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  }
}
template <int RG>
__device__ __forceinline__ int holder_lane(int r) {
  return RG == 1 ? 0 : (RG == 2 ? r * 16 : (r >> 1) * 16 + (r & 1) * 8);
}


// Arguments of one dot pass (kept small: only hot-loop state is live inside).
// Shared-memory regions are passed as 32-bit offsets from the dynamic smem base
// so the callee addresses them with LDS/STS.
struct DotArgs {
  unsigned res, stage, full, empty, ring, rred, yrow, s_nxt, tws, ypart;
  double* zrow;
  unsigned* errp;
  unsigned rowB;
  int rows_g, nres, D, NV, sslot, sph, P;
  unsigned gcount;
  int wmul;  // 1 << 29 (run-time value)
  unsigned long long* prof;  // [4] thread-0 cycle sums (SCB_PROFILE builds): stage waits, A, B, C
  int cpr, chunk_cols;       // wide rows: column chunks per row (stage = one chunk)
  // Fused rank-1 update (the first dot pass of a term, north-star kernel 3): before
  // its dot, every row is deflated R -= alpha s t^T with the previous term's (s, t)
  // (flush_pending with one term, decompose.hpp:200-214) and written back (resident
  // rows in SMEM, streamed rows to global R); ||R_new||^2 is accumulated.  The
  // update's operands sit in shared memory (Ctl::ua; DotArgs stays small enough to
  // be passed in registers).
  int upd;                   // 1: apply the update in phase A
  unsigned ctl;              // smem offset of the Ctl block
#ifdef SCB_TIMING
  unsigned long long* tprof;  // [blocks][warps][8] section cycle sums (dotbench only)
#endif
};

template <bool C, typename X, typename Y>
__device__ __forceinline__ typename std::conditional<C, X, Y>::type& pick(X& x, Y& y) {
  if constexpr (C)
    return x;
  else
    return y;
}

template <typename E, int NW, int VPT, int RG, int CPS = 1>
__device__ __noinline__ void dot_pass(const DotArgs a) {
  constexpr int EPV = Vec<E>::N;
  constexpr int NE = VPT * EPV;
  using VT = typename Vec<E>::T;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows_g = a.rows_g, nres = a.nres, D = a.D, NV = a.NV, P = a.P;
  const unsigned gcount = a.gcount;
  const size_t rowB = a.rowB;
  extern __shared__ __align__(128) unsigned char smem[];
  const unsigned char* res_base = smem + a.res;
  const unsigned char* stage_base = smem + a.stage;
  double* rred = reinterpret_cast<double*>(smem + a.rred);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + a.full);
  unsigned long long* empty = reinterpret_cast<unsigned long long*>(smem + a.empty);
  double* yrow = reinterpret_cast<double*>(smem + a.yrow);
  uint32_t* s_nxt = reinterpret_cast<uint32_t*>(smem + a.s_nxt);
  const uint32_t* tws = reinterpret_cast<const uint32_t*>(smem + a.tws);
  int sslot = a.sslot, sph = a.sph;
  int vidx[VPT];
  bool vok[VPT];
  bool all_ok = true;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int v = (k * NW + warp) * 32 + lane;
    vok[k] = v < NV;
    vidx[k] = vok[k] ? v : 0;
    all_ok = all_ok && vok[k];
  }
  all_ok = __all_sync(0xffffffffu, all_ok);
  const unsigned toff = static_cast<unsigned>((warp * 32 + lane) * sizeof(VT));
  double zacc[NE];
#pragma unroll
  for (int i = 0; i < NE; ++i) zacc[i] = 0.0;
  // per-thread t sign bits of the owned elements (bit i = element i) and the
  // matching sign-flip masks, loop-invariant for the whole pass
  uint32_t tbits = 0;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int col0 = ((k * NW + warp) * 32 + lane) * EPV;
    if (vok[k]) tbits |= ((tws[col0 >> 5] >> (col0 & 31)) & ((1u << EPV) - 1u)) << (k * EPV);
  }
  uint32_t fm[NE];
#pragma unroll
  for (int i = 0; i < NE; ++i) fm[i] = bitmask(tbits, i);
  const int ngroups = (rows_g + RG - 1) / RG;
#ifdef SCB_TIMING
  long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  // Lag buffers: RG == 1 keeps the widened, t-flipped pairs (z is then one
  // DFMA per element); RG >= 2 keeps the raw elements (register budget) and
  // re-widens them in the z update (IMAD.WIDE + LOP3, no XU).
  constexpr bool KW = RG == 1 && CPS == 1;
  using LB = typename std::conditional<KW, double, E>::type;
  const int wmul = a.wmul;

  // rows_of(grp): row pointers of the group; streamed rows wait for their stage
  auto rows_of = [&](int grp, const VT* (&rp)[RG], int (&sl)[RG]) {
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      const int jr = grp * RG + r;
      const int j = jr < rows_g ? jr : rows_g - 1;  // past-the-end rows alias the last row
      sl[r] = -1;
      if (j < nres) {
        rp[r] = reinterpret_cast<const VT*>(res_base + static_cast<size_t>(j) * rowB);
      } else if (jr < rows_g) {
        mbar_wait(&full[sslot], static_cast<uint32_t>(sph));
        rp[r] = reinterpret_cast<const VT*>(stage_base + static_cast<size_t>(sslot) * rowB);
        sl[r] = sslot;
        if (++sslot == D) {
          sslot = 0;
          sph ^= 1;
        }
      } else {
        rp[r] = rp[r > 0 ? r - 1 : 0];
      }
    }
  };
  // ldrows: this thread's segment of the group's rows into registers
  auto ldrows = [&](E (&x)[RG][NE], const VT* const (&rp)[RG], int grp) {
    if (all_ok) {  // warp-uniform: full rows, compile-time vector strides
#pragma unroll
      for (int r = 0; r < RG; ++r)
#pragma unroll
        for (int k = 0; k < VPT; ++k)
          Vec<E>::split(*reinterpret_cast<const VT*>(reinterpret_cast<const unsigned char*>(rp[r]) + toff +
                                                      k * (NW * 32 * sizeof(VT))),
                        &x[r][k * EPV]);
    } else {
#pragma unroll
      for (int r = 0; r < RG; ++r)
#pragma unroll
        for (int k = 0; k < VPT; ++k) Vec<E>::split(rp[r][vidx[k]], &x[r][k * EPV]);
    }
    if (!all_ok || grp * RG + RG > rows_g) {  // rare: ragged row tail / past-the-end rows
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        const bool rok = grp * RG + r < rows_g;
#pragma unroll
        for (int k = 0; k < VPT; ++k)
          if (!(vok[k] && rok)) {
#pragma unroll
            for (int e = 0; e < EPV; ++e) x[r][k * EPV + e] = E(0);
          }
      }
    }
  };
  // stages whose rows are in registers go back to the producer (after a
  // barrier or __syncwarp has ordered every lane's reads)
  auto release = [&](const int (&sl)[RG]) {
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < RG; ++r)
        if (sl[r] >= 0) mbar_arrive(&empty[sl[r]]);
    }
  };
  // widen + per-row partials of <R_j, t> over this thread's columns
  auto widen_dot = [&](const E (&x)[RG][NE], LB (&keep)[RG][NE], double (&part)[RG]) {
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      double ac[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < NE; ++i) {
        const double w = Wide<E>::prep(x[r][i], fm[i], wmul);
        if constexpr (KW) keep[r][i] = w;
        ac[i & 3] = Wide<E>::dot(ac[i & 3], w);
      }
      part[r] = (ac[0] + ac[1]) + (ac[2] + ac[3]);
    }
  };
  // z' += s'_j (t o R_j) for the group's rows (exact: the product with +-1 is
  // exact); z = t o z' is applied when the pass ends
  auto zupd = [&](const LB (&pw)[RG][NE], unsigned negb) {
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      const double sg = Wide<E>::zscale(((negb >> r) & 1u) ? -1.0 : 1.0);
#pragma unroll
      for (int i = 0; i < NE; ++i) {
        if constexpr (KW)
          zacc[i] = fma(pw[r][i], sg, zacc[i]);
        else
          zacc[i] = fma(Wide<E>::prep(pw[r][i], fm[i], wmul), sg, zacc[i]);
      }
    }
  };
  auto slot = [&](int grp) {
    return rred + static_cast<size_t>((gcount + static_cast<unsigned>(grp)) & (kRing - 1)) * RG * NW;
  };
  // y of the group's rows (lane r < RG holds row r) in fixed warp order, two
  // interleaved chains, branch-free (every lane reads; only lanes < RG matter)
  auto combine = [&](int grp) -> double {
    static_assert(NW % 2 == 0, "two combine chains");
    const double* pr = slot(grp) + (lane < RG ? lane : 0) * NW;
    double y0 = pr[0], y1 = pr[1];
#pragma unroll
    for (int w = 2; w < NW; w += 2) {
      y0 += pr[w];
      y1 += pr[w + 1];
    }
    return y0 + y1;
  };
  // warp 0 records y; every warp tracks the s' word, warp 0 stores it
  uint32_t sword = 0;
  auto record = [&](int grp, double y, unsigned negb) {
    const int j0 = grp * RG, jend = j0 + RG;
    sword |= negb << (j0 & 31);
    if (warp == 0) {
      if (lane < RG && j0 + lane < rows_g) {
        yrow[j0 + lane] = y;
        if (!isfinite(y)) atomicMin(a.errp + ERR_Y, static_cast<unsigned>(P));
      }
      if (lane == 0 && ((jend & 31) == 0 || jend >= rows_g)) s_nxt[j0 >> 5] = sword;
    }
    if ((jend & 31) == 0) sword = 0;
  };
  // One iteration per group g, one CTA barrier: [stage wait for g+1] then a
  // single barrier-free block (y and z update of g-1, widen + dot + reduction
  // of g, the loads of g+1) the scheduler interleaves, then the partials of g
  // are published and the barrier makes them visible.
  //   dx: raw rows of g;  kc: widened keep buffer of g (KW);  kl: lag buffer of g-1
  auto iter = [&](auto wz, auto hn, int grp, const E (&dx)[RG][NE], LB (&kc)[RG][NE], LB (&kl)[RG][NE],
                  E (&ld)[RG][NE]) {
    constexpr bool WZ = decltype(wz)::value, HN = decltype(hn)::value;
#ifdef SCB_TIMING
    long long tt0 = clock64();
#define SCB_T(k) do { const long long t1_ = clock64(); tacc[k] += t1_ - tt0; tt0 = t1_; } while (0)
#else
#define SCB_T(k) do {} while (0)
#endif
    const VT* rpn[RG];
    int sln[RG];
    if constexpr (HN) rows_of(grp + 1, rpn, sln);
    SCB_T(0);
    // (a) the previous group's partials are loaded first (latency hidden by
    // the dot arithmetic), (b) widen + dot of g, (c) y of g-1 and its signs,
    // (d) next group's loads, (e) the reduction of g with the z update of g-1
    // in chunks between its shuffle levels (shuffles and votes are scheduling
    // barriers for ptxas, so the interleave is written out in source order)
    double q[NW];
    if constexpr (WZ) {
      const double* pq = slot(grp - 1) + (lane < RG ? lane : 0) * NW;
#pragma unroll
      for (int w = 0; w < NW; ++w) q[w] = pq[w];
    }
    double part[RG];
    widen_dot(dx, kc, part);
    SCB_T(1);
    double y = 0.0;
    unsigned negb = 0;
    if constexpr (WZ) {
      static_assert(NW % 2 == 0, "two combine chains");
      double y0 = q[0], y1 = q[1];
#pragma unroll
      for (int w = 2; w < NW; w += 2) {
        y0 += q[w];
        y1 += q[w + 1];
      }
      y = y0 + y1;
      negb = __ballot_sync(0xffffffffu, lane < RG && y < 0.0);
    }
    SCB_T(2);
    if constexpr (HN && KW) ldrows(ld, rpn, grp + 1);
    double v;
    if constexpr (RG == 1 && WZ) {
      const double sg = Wide<E>::zscale((negb & 1u) ? -1.0 : 1.0);
      v = part[0];
      constexpr int CH = (NE + 4) / 5;  // z elements per shuffle level
#pragma unroll
      for (int l = 0; l < 5; ++l) {
        const double o = __shfl_xor_sync(0xffffffffu, v, 16 >> l);
#pragma unroll
        for (int i = l * CH; i < (l + 1) * CH && i < NE; ++i) {
          if constexpr (KW)
            zacc[i] = fma(kl[0][i], sg, zacc[i]);
          else
            zacc[i] = fma(Wide<E>::prep(kl[0][i], fm[i], wmul), sg, zacc[i]);
        }
        v += o;
      }
      SCB_T(3);
    } else {
      v = warp_reduce_rows<RG>(part, lane);
      SCB_T(3);
      if constexpr (WZ) zupd(kl, negb);
    }
    if constexpr (HN && !KW) ldrows(ld, rpn, grp + 1);
    SCB_T(4);
    double* pr = slot(grp);
#pragma unroll
    for (int r = 0; r < RG; ++r)
      if (lane == holder_lane<RG>(r)) pr[r * NW + warp] = v;
    SCB_T(5);
    consumer_sync(NW * 32);
    SCB_T(6);
    if constexpr (WZ) record(grp - 1, y, negb);
    if constexpr (HN) release(sln);
    SCB_T(7);
#undef SCB_T
  };
  using F = std::integral_constant<bool, false>;
  using T = std::integral_constant<bool, true>;
  // group k lives in buffer A (k even) or B (k odd)
  E xr[KW ? RG : 1][KW ? NE : 1];  // raw staging (KW only)
  LB A[RG][NE], B[RG][NE];
  // raw rows of a group in A / B: the staging buffer (KW) or the buffer itself
  auto& dxA = pick<KW>(xr, A);
  auto& dxB = pick<KW>(xr, B);
  {
    const VT* rp0[RG];
    int sl0[RG];
    rows_of(0, rp0, sl0);
    ldrows(dxA, rp0, 0);
    __syncwarp();
    release(sl0);
  }
  if (ngroups == 1) {
    iter(F{}, F{}, 0, dxA, A, B, dxB);
  } else {
    iter(F{}, T{}, 0, dxA, A, B, dxB);
    int g = 1;
    for (; g + 2 < ngroups; g += 2) {
      iter(T{}, T{}, g, dxB, B, A, dxA);
      iter(T{}, T{}, g + 1, dxA, A, B, dxB);
    }
    if (g + 1 < ngroups) {
      iter(T{}, T{}, g, dxB, B, A, dxA);
      iter(T{}, F{}, g + 1, dxA, A, B, dxB);
    } else {
      iter(T{}, F{}, g, dxB, B, A, dxA);
    }
  }
  {
    const int last = ngroups - 1;
    const double y = combine(last);
    const unsigned negb = __ballot_sync(0xffffffffu, lane < RG && y < 0.0);
    if (last & 1)
      zupd(B, negb);
    else
      zupd(A, negb);
    record(last, y, negb);
  }

#ifdef SCB_TIMING
  if (lane == 0)
    for (int k = 0; k < 8; ++k) a.tprof[(blockIdx.x * 32 + warp) * 8 + k] += tacc[k];
#endif
#pragma unroll
  for (int i = 0; i < NE; ++i) zacc[i] = flipd(zacc[i], fm[i]);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    if (vok[k]) {
#pragma unroll
      for (int e = 0; e < EPV; e += 2)
        __stcg(reinterpret_cast<double2*>(a.zrow + vidx[k] * EPV + e), make_double2(zacc[k * EPV + e], zacc[k * EPV + e + 1]));
    }
  }
}

// ---------------------------------------------------------------------------
// Two-phase dot pass.  (A) every warp forms the partial <R_j, t> of its column
// segment for each row and reduces it within the warp only (no CTA barrier per
// row; two rows per step for ILP); (B) after ONE barrier the CTA combines the
// per-warp partials of all its rows in fixed warp order (y, s' = sgn(y)); then
// (C) z = R^T s' streams the rows again (SMEM-resident ones from SMEM, the rest
// re-streamed by the producer) as a pure accumulate.  Rows are read twice, but
// they live in SMEM / L2; what this removes is the per-row serial chain.
// Deflation of one loaded row segment by the previous term (fused update): the
// reference's flush arithmetic data += flip(-alpha, s_i ^ t_j), rounded to the
// storage type, on the columns < n; returns the segment's ||.||^2 contribution.
template <typename E, int EPV, int VPT>
__device__ __forceinline__ double deflate(E* x, const uint32_t* um, uint32_t sneg, double alpha, const int* colv,
                                          const bool* vok, int n) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    if (!vok[k]) continue;
#pragma unroll
    for (int e = 0; e < EPV; ++e) {
      const int i = k * EPV + e;
      if (colv[k] + e < n) x[i] = Vec<E>::narrow(static_cast<double>(x[i]) + flipd(-alpha, sneg ^ um[i]));
      const double d = static_cast<double>(x[i]);
      acc += d * d;
    }
  }
  return acc;
}

template <typename E, int NW, int VPT, bool FULL>
__device__ __forceinline__ double dot_pass_2ph_impl(const DotArgs& a) {
  constexpr int EPV = Vec<E>::N;
  constexpr int NE = VPT * EPV;
  using VT = typename Vec<E>::T;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows_g = a.rows_g, nres = a.nres, D = a.D, NV = a.NV, P = a.P;
  const size_t rowB = a.rowB;
  extern __shared__ __align__(128) unsigned char smem[];
  const unsigned char* res_base = smem + a.res;
  const unsigned char* stage_base = smem + a.stage;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + a.full);
  unsigned long long* empty = reinterpret_cast<unsigned long long*>(smem + a.empty);
  double* yrow = reinterpret_cast<double*>(smem + a.yrow);
  double* ypart = reinterpret_cast<double*>(smem + a.ypart);
  uint32_t* s_nxt = reinterpret_cast<uint32_t*>(smem + a.s_nxt);
  const uint32_t* tws = reinterpret_cast<const uint32_t*>(smem + a.tws);
  int sslot = a.sslot, sph = a.sph;
  int vidx[VPT];
  bool vok[VPT];
  bool all_ok = true;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int v = (k * NW + warp) * 32 + lane;
    vok[k] = v < NV;
    vidx[k] = vok[k] ? v : 0;
    all_ok = all_ok && vok[k];
  }
  (void)all_ok;
  const unsigned toff = static_cast<unsigned>((warp * 32 + lane) * sizeof(VT));
  uint32_t tbits = 0;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int col0 = ((k * NW + warp) * 32 + lane) * EPV;
    if (vok[k]) tbits |= ((tws[col0 >> 5] >> (col0 & 31)) & ((1u << EPV) - 1u)) << (k * EPV);
  }
  uint32_t fm[NE];
#pragma unroll
  for (int i = 0; i < NE; ++i) fm[i] = bitmask(tbits, i);
  // fused update: the update's t bits of the owned columns, and their columns
#ifdef SCB_NO_FUSE
  const bool upd = false;
#else
  const bool upd = a.upd != 0;
#endif
  Ctl* ctl = reinterpret_cast<Ctl*>(smem + a.ctl);
  const UpdArgs& ua = ctl->ua;
  uint32_t um[NE];
  int colv[VPT];
  double nacc = 0.0;
  {
    const uint32_t* uws = reinterpret_cast<const uint32_t*>(smem + ua.uws);
    uint32_t ub = 0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      colv[k] = vidx[k] * EPV;
      if (upd && vok[k]) ub |= ((uws[colv[k] >> 5] >> (colv[k] & 31)) & ((1u << EPV) - 1u)) << (k * EPV);
    }
#pragma unroll
    for (int i = 0; i < NE; ++i) um[i] = bitmask(ub, i);
  }
  const uint32_t* s_upd = reinterpret_cast<const uint32_t*>(smem + ua.s_upd);
  // phase A: deflate the loaded row (when fused) and write it back where it lives
  auto upd_row = [&](int j, const VT* rp, E (&x)[NE]) {
    const uint32_t sneg = ((s_upd[j >> 5] >> (j & 31)) & 1u) << 31;
    nacc += deflate<E, EPV, VPT>(x, um, sneg, ua.alpha, colv, vok, ua.n);
    // global R stays current for every row (resident rows too: the owners of a delta
    // pass read flipped rows from global memory); resident rows also in place in SMEM
    VT* dst = reinterpret_cast<VT*>(static_cast<E*>(ua.Rband) + static_cast<size_t>(j) * ua.pitch);
    VT* sdst = const_cast<VT*>(rp);
#pragma unroll
    for (int k = 0; k < VPT; ++k)
      if (vok[k]) {
        dst[vidx[k]] = Vec<E>::join(&x[k * EPV]);
        if (j < nres) sdst[vidx[k]] = Vec<E>::join(&x[k * EPV]);
      }
  };

  long long twait = 0;
  auto rowptr = [&](int j, int& sl) -> const VT* {
    if (j < nres) {
      sl = -1;
      return reinterpret_cast<const VT*>(res_base + static_cast<size_t>(j) * rowB);
    }
#ifdef SCB_PROFILE
    const long long tw0 = clock64();
    mbar_wait(&full[sslot], static_cast<uint32_t>(sph));
    twait += clock64() - tw0;
#else
    mbar_wait(&full[sslot], static_cast<uint32_t>(sph));
#endif
    sl = sslot;
    if (++sslot == D) {
      sslot = 0;
      sph ^= 1;
    }
    return reinterpret_cast<const VT*>(stage_base + static_cast<size_t>(sl) * rowB);
  };
  // FULL: the warp's vectors are all inside the row (warp-uniform; the loops are
  // instantiated per case because ptxas does not unswitch the loop-invariant test)
  auto ld = [&](const VT* rp, E (&x)[NE]) {
    if constexpr (FULL) {
#pragma unroll
      for (int k = 0; k < VPT; ++k)
        Vec<E>::split(*reinterpret_cast<const VT*>(reinterpret_cast<const unsigned char*>(rp) + toff +
                                                    k * (NW * 32 * sizeof(VT))),
                      &x[k * EPV]);
    } else {
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        Vec<E>::split(rp[vidx[k]], &x[k * EPV]);
        if (!vok[k]) {
#pragma unroll
          for (int e = 0; e < EPV; ++e) x[k * EPV + e] = E(0);
        }
      }
    }
  };
  auto release = [&](int sl) {
    if (sl >= 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sl]);
    }
  };
  auto partial = [&](const E (&x)[NE]) -> double {
    double ac[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < NE; ++i) ac[i & 3] = fma(widen_shf(x[i], fm[i]), Wide<E>::zscale(1.0), ac[i & 3]);
    return (ac[0] + ac[1]) + (ac[2] + ac[3]);
  };

  // ---- (A) per-warp row partials ----
  const long long tA = clock64();
  int j = 0;
  for (; j + 1 < rows_g; j += 2) {
    int s0, s1;
    const VT* p0 = rowptr(j, s0);
    const VT* p1 = rowptr(j + 1, s1);
    E x0[NE], x1[NE];
    ld(p0, x0);
    ld(p1, x1);
    if (upd) {
      upd_row(j, p0, x0);
      upd_row(j + 1, p1, x1);
      asm volatile("fence.proxy.async.global;" ::: "memory");  // before the stages go back to the TMA producer
    }
    double v0 = partial(x0), v1 = partial(x1);
    release(s0);
    release(s1);
  #pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double o0 = __shfl_xor_sync(0xffffffffu, v0, o), o1 = __shfl_xor_sync(0xffffffffu, v1, o);
      v0 += o0;
      v1 += o1;
    }
    if (lane == 0) {
      ypart[j * NW + warp] = v0;
      ypart[(j + 1) * NW + warp] = v1;
    }
  }
  if (j < rows_g) {
    int s0;
    const VT* p0 = rowptr(j, s0);
    E x0[NE];
    ld(p0, x0);
    if (upd) {
      upd_row(j, p0, x0);
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    double v0 = partial(x0);
    release(s0);
    v0 = warp_sum(v0);
    if (lane == 0) ypart[j * NW + warp] = v0;
  }
  const long long tB = clock64();
  if (upd) __threadfence();
  consumer_sync(NW * 32);
  if (upd && tid == 0) ctl->upd_done = a.P + 1;  // the producer may now stream the updated rows for (C)
  // ---- (B) y and s' of every row, fixed warp order ----
  for (int jb = 0; jb < rows_g; jb += NW * 32) {
    const int jj = jb + tid;
    const bool ok = jj < rows_g;
    double y = 0.0;
    if (ok) {
      const double* pr = ypart + jj * NW;
      double y0 = pr[0], y1 = pr[1];
  #pragma unroll
      for (int w = 2; w < NW; w += 2) {
        y0 += pr[w];
        y1 += pr[w + 1];
      }
      y = y0 + y1;
      yrow[jj] = y;
      if (!isfinite(y)) atomicMin(a.errp + ERR_Y, static_cast<unsigned>(P));
    }
    const unsigned word = __ballot_sync(0xffffffffu, ok && y < 0.0);
    if (lane == 0 && jb + warp * 32 < rows_g) s_nxt[(jb >> 5) + warp] = word;
  }
  consumer_sync(NW * 32);
  const long long tC = clock64();
  // ---- (C) z = R^T s' ----
  double zacc[NE];
  #pragma unroll
  for (int i = 0; i < NE; ++i) zacc[i] = 0.0;
  auto sgn_of = [&](int r) { return Wide<E>::zscale(((s_nxt[r >> 5] >> (r & 31)) & 1u) ? -1.0 : 1.0); };
  j = 0;
  for (; j + 1 < rows_g; j += 2) {
    int s0, s1;
    const VT* p0 = rowptr(j, s0);
    const VT* p1 = rowptr(j + 1, s1);
    E x0[NE], x1[NE];
    ld(p0, x0);
    ld(p1, x1);
    const double g0 = sgn_of(j), g1 = sgn_of(j + 1);
  #pragma unroll
    for (int i = 0; i < NE; ++i) {
      zacc[i] = fma(widen_shf(x0[i], 0u), g0, zacc[i]);
      zacc[i] = fma(widen_shf(x1[i], 0u), g1, zacc[i]);
    }
    release(s0);
    release(s1);
  }
  if (j < rows_g) {
    int s0;
    const VT* p0 = rowptr(j, s0);
    E x0[NE];
    ld(p0, x0);
    const double g0 = sgn_of(j);
  #pragma unroll
    for (int i = 0; i < NE; ++i) zacc[i] = fma(widen_shf(x0[i], 0u), g0, zacc[i]);
    release(s0);
  }
  #ifdef SCB_PROFILE
  if (a.prof && tid == 0) {
    a.prof[0] += twait;
    a.prof[1] += tB - tA;
    a.prof[2] += tC - tB;
    a.prof[3] += clock64() - tC;
  }
  #else
  (void)tA; (void)tB; (void)tC; (void)twait;
  #endif
  #pragma unroll
  for (int k = 0; k < VPT; ++k) {
    if (vok[k]) {
  #pragma unroll
      for (int e = 0; e < EPV; e += 2)
        __stcg(reinterpret_cast<double2*>(a.zrow + vidx[k] * EPV + e), make_double2(zacc[k * EPV + e], zacc[k * EPV + e + 1]));
    }
  }
  return nacc;
}

// Returns this thread's ||R_new||^2 contribution (fused update passes; else 0).
template <typename E, int NW, int VPT>
__device__ __noinline__ double dot_pass_2ph(const DotArgs a) {
  // warp-uniform: does every vector this warp owns lie inside the row?
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bool full = true;
#pragma unroll
  for (int k = 0; k < VPT; ++k) full = full && ((k * NW + warp) * 32 + lane) < a.NV;
  if (__all_sync(0xffffffffu, full))
    return dot_pass_2ph_impl<E, NW, VPT, true>(a);
  else
    return dot_pass_2ph_impl<E, NW, VPT, false>(a);
}
// ---------------------------------------------------------------------------
// Wide rows (cpr > 1): the two-phase pass over column chunks.  Every (row,
// chunk) piece is one TMA stage; both phases walk the pieces chunk-major, so
// the t-flip masks (phase A) and the z accumulators (phase C) of a chunk stay
// in registers across all rows.  Phase A accumulates the per-warp partial of
// row j over the chunks in ypart[j][warp] (owned by that warp; fixed chunk
// order), then the same combine as the single-chunk pass.  No resident rows.
template <typename E, int NW, int VPT, bool FULL>
__device__ __forceinline__ void ld_piece(const typename Vec<E>::T* rp, unsigned toff, const int (&vloc)[VPT],
                                         const bool (&vok)[VPT], E (&x)[VPT * Vec<E>::N]) {
  using VT = typename Vec<E>::T;
  constexpr int EPV = Vec<E>::N;
  if constexpr (FULL) {
#pragma unroll
    for (int k = 0; k < VPT; ++k)
      Vec<E>::split(*reinterpret_cast<const VT*>(reinterpret_cast<const unsigned char*>(rp) + toff +
                                                  k * (NW * 32 * sizeof(VT))),
                    &x[k * EPV]);
  } else {
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      Vec<E>::split(rp[vok[k] ? vloc[k] : 0], &x[k * EPV]);
      if (!vok[k]) {
#pragma unroll
        for (int e = 0; e < EPV; ++e) x[k * EPV + e] = E(0);
      }
    }
  }
}

struct PieceCursor {
  int sslot, sph, D;
  const unsigned char* stage_base;
  unsigned long long* full;
  unsigned long long* empty;
  size_t stageB;
  __device__ __forceinline__ const unsigned char* next(int& sl) {
    mbar_wait(&full[sslot], static_cast<uint32_t>(sph));
    sl = sslot;
    if (++sslot == D) {
      sslot = 0;
      sph ^= 1;
    }
    return stage_base + static_cast<size_t>(sl) * stageB;
  }
  __device__ __forceinline__ void release(int sl) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[sl]);
  }
};

// phase A over one chunk: every row's partial against this chunk's t, reduced in
// the warp and accumulated into ypart[j][warp]
// Fused update (DotArgs::upd) of the chunk's pieces: deflate, write back to global R.
struct ChunkUpd {
  const uint32_t* s_upd;
  const uint32_t* um;  // [NE] update t masks of this chunk's owned columns
  const int* colv;     // [VPT] first column of each owned vector
  double alpha;
  void* Rband;
  long long pitch;
  int n, vbase;        // vbase: first vector of the chunk within the row
  double nacc;
};

template <typename E, int NW, int VPT, bool FULL, bool UPD>
__device__ __forceinline__ void chunk_dot(PieceCursor& cur, int rows_g, int k, unsigned toff, const int (&vloc)[VPT],
                                          const bool (&vok)[VPT], const uint32_t (&fm)[VPT * Vec<E>::N],
                                          double* ypart, ChunkUpd& cu) {
  using VT = typename Vec<E>::T;
  constexpr int EPV = Vec<E>::N;
  constexpr int NE = VPT * Vec<E>::N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto partial = [&](const E (&x)[NE]) -> double {
    double ac[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < NE; ++i) ac[i & 3] = fma(widen_shf(x[i], fm[i]), Wide<E>::zscale(1.0), ac[i & 3]);
    return (ac[0] + ac[1]) + (ac[2] + ac[3]);
  };
  for (int j = 0; j < rows_g; ++j) {
    int sl;
    const VT* rp = reinterpret_cast<const VT*>(cur.next(sl));
    E x[NE];
    ld_piece<E, NW, VPT, FULL>(rp, toff, vloc, vok, x);
    if constexpr (UPD) {
      const uint32_t sneg = ((cu.s_upd[j >> 5] >> (j & 31)) & 1u) << 31;
      cu.nacc += deflate<E, EPV, VPT>(x, cu.um, sneg, cu.alpha, cu.colv, vok, cu.n);
      VT* dst = reinterpret_cast<VT*>(static_cast<E*>(cu.Rband) + static_cast<size_t>(j) * cu.pitch) + cu.vbase;
#pragma unroll
      for (int q = 0; q < VPT; ++q)
        if (vok[q]) dst[vloc[q]] = Vec<E>::join(&x[q * EPV]);
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    double v = partial(x);
    cur.release(sl);
    v = warp_sum(v);
    if (lane == 0) ypart[j * NW + warp] = (k == 0) ? v : ypart[j * NW + warp] + v;
  }
}

// phase C over one chunk: z of the chunk's columns accumulated over all rows
template <typename E, int NW, int VPT, bool FULL>
__device__ __forceinline__ void chunk_z(PieceCursor& cur, int rows_g, unsigned toff, const int (&vloc)[VPT],
                                        const bool (&vok)[VPT], const uint32_t* s_nxt, double* zrow_chunk) {
  using VT = typename Vec<E>::T;
  constexpr int EPV = Vec<E>::N;
  constexpr int NE = VPT * EPV;
  double zacc[NE];
#pragma unroll
  for (int i = 0; i < NE; ++i) zacc[i] = 0.0;
  for (int j = 0; j < rows_g; ++j) {
    int sl;
    const VT* rp = reinterpret_cast<const VT*>(cur.next(sl));
    E x[NE];
    ld_piece<E, NW, VPT, FULL>(rp, toff, vloc, vok, x);
    const double g = Wide<E>::zscale(((s_nxt[j >> 5] >> (j & 31)) & 1u) ? -1.0 : 1.0);
#pragma unroll
    for (int i = 0; i < NE; ++i) zacc[i] = fma(widen_shf(x[i], 0u), g, zacc[i]);
    cur.release(sl);
  }
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    if (vok[k]) {
#pragma unroll
      for (int e = 0; e < EPV; e += 2)
        __stcg(reinterpret_cast<double2*>(zrow_chunk + vloc[k] * EPV + e), make_double2(zacc[k * EPV + e], zacc[k * EPV + e + 1]));
    }
  }
}

template <typename E, int NW, int VPT>
__device__ __noinline__ double dot_pass_chunked(const DotArgs a) {
  constexpr int EPV = Vec<E>::N;
  constexpr int NE = VPT * EPV;
  constexpr int chunkV = NW * 32 * VPT;  // vectors per chunk
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows_g = a.rows_g, NV = a.NV, P = a.P, cpr = a.cpr;
  extern __shared__ __align__(128) unsigned char smem[];
  double* yrow = reinterpret_cast<double*>(smem + a.yrow);
  double* ypart = reinterpret_cast<double*>(smem + a.ypart);
  uint32_t* s_nxt = reinterpret_cast<uint32_t*>(smem + a.s_nxt);
  const uint32_t* tws = reinterpret_cast<const uint32_t*>(smem + a.tws);
  PieceCursor cur{a.sslot, a.sph, a.D, smem + a.stage, reinterpret_cast<unsigned long long*>(smem + a.full),
                  reinterpret_cast<unsigned long long*>(smem + a.empty), a.rowB};
  const unsigned toff = static_cast<unsigned>((warp * 32 + lane) * sizeof(typename Vec<E>::T));
  int vloc[VPT];
  bool vok[VPT];
  auto setup = [&](int k) -> bool {  // this chunk's vectors; returns warp-uniform "all inside"
    bool ok = true;
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      vloc[q] = (q * NW + warp) * 32 + lane;
      vok[q] = k * chunkV + vloc[q] < NV;
      ok = ok && vok[q];
    }
    return __all_sync(0xffffffffu, ok);
  };
  // ---- (A) y partials, chunk-major (fused update: deflate + write back first) ----
  Ctl* ctl = reinterpret_cast<Ctl*>(smem + a.ctl);
  const UpdArgs& ua = ctl->ua;
  const uint32_t* uws = reinterpret_cast<const uint32_t*>(smem + ua.uws);
  ChunkUpd cu{reinterpret_cast<const uint32_t*>(smem + ua.s_upd), nullptr, nullptr, ua.alpha, ua.Rband, ua.pitch,
              ua.n, 0, 0.0};
  for (int k = 0; k < cpr; ++k) {
    const bool full = setup(k);
    uint32_t tbits = 0, ub = 0;
    int colv[VPT];
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const int col0 = (k * chunkV + vloc[q]) * EPV;
      colv[q] = col0;
      if (vok[q]) tbits |= ((tws[col0 >> 5] >> (col0 & 31)) & ((1u << EPV) - 1u)) << (q * EPV);
      if (a.upd && vok[q]) ub |= ((uws[col0 >> 5] >> (col0 & 31)) & ((1u << EPV) - 1u)) << (q * EPV);
    }
    uint32_t fm[NE], um[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      fm[i] = bitmask(tbits, i);
      um[i] = bitmask(ub, i);
    }
    cu.um = um;
    cu.colv = colv;
    cu.vbase = k * chunkV;
    if (a.upd) {
      if (full)
        chunk_dot<E, NW, VPT, true, true>(cur, rows_g, k, toff, vloc, vok, fm, ypart, cu);
      else
        chunk_dot<E, NW, VPT, false, true>(cur, rows_g, k, toff, vloc, vok, fm, ypart, cu);
    } else {
      if (full)
        chunk_dot<E, NW, VPT, true, false>(cur, rows_g, k, toff, vloc, vok, fm, ypart, cu);
      else
        chunk_dot<E, NW, VPT, false, false>(cur, rows_g, k, toff, vloc, vok, fm, ypart, cu);
    }
  }
  if (a.upd) __threadfence();
  consumer_sync(NW * 32);
  if (a.upd && tid == 0) ctl->upd_done = P + 1;  // the producer may now stream the updated pieces for (C)
  // ---- (B) y and s' of every row, fixed warp order ----
  for (int jb = 0; jb < rows_g; jb += NW * 32) {
    const int jj = jb + tid;
    const bool ok = jj < rows_g;
    double y = 0.0;
    if (ok) {
      const double* pr = ypart + jj * NW;
      double y0 = pr[0], y1 = pr[1];
#pragma unroll
      for (int w = 2; w < NW; w += 2) {
        y0 += pr[w];
        y1 += pr[w + 1];
      }
      y = y0 + y1;
      yrow[jj] = y;
      if (!isfinite(y)) atomicMin(a.errp + ERR_Y, static_cast<unsigned>(P));
    }
    const unsigned word = __ballot_sync(0xffffffffu, ok && y < 0.0);
    if (lane == 0 && jb + warp * 32 < rows_g) s_nxt[(jb >> 5) + warp] = word;
  }
  consumer_sync(NW * 32);
  // ---- (C) z, chunk-major ----
  for (int k = 0; k < cpr; ++k) {
    const bool full = setup(k);
    double* zc = a.zrow + static_cast<size_t>(k) * chunkV * EPV;
    if (full)
      chunk_z<E, NW, VPT, true>(cur, rows_g, toff, vloc, vok, s_nxt, zc);
    else
      chunk_z<E, NW, VPT, false>(cur, rows_g, toff, vloc, vok, s_nxt, zc);
  }
  return cu.nacc;
}

// ---------------------------------------------------------------------------
// Sparse delta dot pass (the GPU form of the reference's delta caches,
// kernels.hpp:92-156 / search.hpp:145-186): with y = R t and z = R^T s kept from
// the previous pass, only the columns whose t flipped and the rows whose s flips
// are read --
//   y_j += 2 sum_{c: t flipped} t'_c R[j,c]   (gather; lanes walk the t-XOR words)
//   s'  = sgn(y)
//   dz  = 2 sum_{j: s flipped} s'_j R[j,:]    (this CTA's rows; owners add it to z)
// No rows are streamed.  Dense passes refresh y and z (restart/term start, every
// 64th sweep, or when many columns flipped), bounding the drift of the caches.
struct DeltaArgs {
  unsigned res, yrow, s_cur, s_nxt, tws, txor;
  const void* Rrows;  // global row 0 of this CTA's band
  double* zrow;       // this CTA's z partial row of this pass
  unsigned* errp;
  int* has_dz;
  int* nfrows;        // [2] run totals: flipped rows read (from global), dz partials written
  int local_dz;       // 1: this CTA forms the dz partial of its flipped rows (order-k mode); 0: it
                      //    publishes its flip words and the column owners read the flipped rows
  unsigned long long* flipw;  // [sw_all] this pass's (flip mask | s' << 32) words of the band (local_dz == 0)
  int sw_all;                 // words per CTA record (from the largest band; bands one row shorter leave
                              // their last word empty -- written as 0, never left stale)
#ifdef SCB_PROFILE
  unsigned long long* prof;  // [6] thread-0 cycle sums of the delta pass sections
#endif
  long long pitch;
  unsigned rowB;
  int rows_g, nres, Q, NV, P;
  int cpr;  // column chunks per row (1: whole rows)
};

template <typename E, int NW, int VPT>
__device__ __noinline__ void delta_pass(const DeltaArgs a) {
  using VT = typename Vec<E>::T;
  constexpr int EPV = Vec<E>::N;
  constexpr int NE = VPT * EPV;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows_g = a.rows_g, nres = a.nres, Q = a.Q, NV = a.NV, P = a.P;
  extern __shared__ __align__(128) unsigned char smem[];
  double* yrow = reinterpret_cast<double*>(smem + a.yrow);
  const uint32_t* s_cur = reinterpret_cast<const uint32_t*>(smem + a.s_cur);
  uint32_t* s_nxt = reinterpret_cast<uint32_t*>(smem + a.s_nxt);
  const uint32_t* tws = reinterpret_cast<const uint32_t*>(smem + a.tws);
  const uint32_t* txor = reinterpret_cast<const uint32_t*>(smem + a.txor);
  const E* Rg = static_cast<const E*>(a.Rrows);
#ifdef SCB_PROFILE
  long long dt0 = clock64();
#define SCB_DT(k) do { if (a.prof && tid == 0) { const long long t1_ = clock64(); a.prof[k] += t1_ - dt0; dt0 = t1_; } } while (0)
#else
#define SCB_DT(k) do {} while (0)
#endif
  auto row_ptr = [&](int j) -> const E* {
    return j < nres ? reinterpret_cast<const E*>(smem + a.res + static_cast<size_t>(j) * a.rowB)
                    : Rg + static_cast<size_t>(j) * a.pitch;
  };

  // ---- y update: one warp per row, lanes over the t-XOR words (fixed order) ----
  // Each lane first lists its flipped columns (ascending); with at most kMaxF
  // per lane every load of two rows is issued at once (one L2 round trip per
  // row pair instead of one per column).  Summation order is the same either way.
  constexpr int kMaxF = 8;
  int fc[kMaxF];
  uint32_t fneg = 0;
  int nf = 0;
  bool over = false;
  for (int w = lane; w < Q; w += 32) {
    uint32_t x = txor[w];
    const uint32_t tn = tws[w];
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      if (nf < kMaxF) {
        fc[nf] = w * 32 + b;
        fneg |= ((tn >> b) & 1u) << nf;
        ++nf;
      } else {
        over = true;
      }
    }
  }
  SCB_DT(0);  // flip lists
  // rows per warp per round trip: up to four, no more than the band needs
  const int rpg = rows_g > 2 * NW ? 4 : (rows_g > NW ? 2 : 1);
  const bool any_over = __any_sync(0xffffffffu, over);
  if (!any_over && rpg < 4) {  // short bands (<= 2 rows per warp): one pair per trip
    auto row_sum = [&](int j) -> double {
      const E* row = row_ptr(j);
      const bool res = j < nres;
      double v[kMaxF];
#pragma unroll
      for (int k = 0; k < kMaxF; ++k)
        v[k] = k < nf ? static_cast<double>(res ? row[fc[k]] : __ldcg(row + fc[k])) : 0.0;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < kMaxF; ++k)
        if (k < nf) acc += ((fneg >> k) & 1u) ? -v[k] : v[k];
      return acc;
    };
    int j = warp;
    for (; j + NW < rows_g; j += 2 * NW) {
      double a0 = row_sum(j), a1 = row_sum(j + NW);
      a0 = warp_sum(a0);
      a1 = warp_sum(a1);
      if (lane == 0) {
        yrow[j] += 2.0 * a0;
        yrow[j + NW] += 2.0 * a1;
      }
    }
    if (j < rows_g) {
      const double a0 = warp_sum(row_sum(j));
      if (lane == 0) yrow[j] += 2.0 * a0;
    }
  } else if (!any_over) {
    // up to four rows per warp per L2 round trip (a band of <= 4 NW rows: one trip)
    for (int j = warp; j < rows_g; j += rpg * NW) {
      E v[4][kMaxF];  // every load of the four rows issued before the first use (R may
                      // have been rewritten this launch: __ldcg, no __ldg)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int jr = j + r * NW;
        const bool ok = r < rpg && jr < rows_g;
        const E* row = row_ptr(ok ? jr : j);
        const bool res = jr < nres;
#pragma unroll
        for (int k = 0; k < kMaxF; ++k)
          v[r][k] = (ok && k < nf) ? (res ? row[fc[k]] : __ldcg(row + fc[k])) : E(0);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (r >= rpg) break;  // uniform: short bands reduce only their own rows
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < kMaxF; ++k)
          if (k < nf) acc += ((fneg >> k) & 1u) ? -static_cast<double>(v[r][k]) : static_cast<double>(v[r][k]);
        const double s = warp_sum(acc);
        if (lane == 0 && j + r * NW < rows_g) yrow[j + r * NW] += 2.0 * s;
      }
    }
  } else {
    // more than kMaxF flips in some lane: the same per-lane ascending sums, kMaxF
    // flips per round trip (each lane walks its t-XOR words with a cursor)
    for (int j = warp; j < rows_g; j += rpg * NW) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      int cw = lane;
      uint32_t cx = cw < Q ? txor[cw] : 0u;
      for (;;) {
        nf = 0;
        fneg = 0;
        while (nf < kMaxF) {
          while (!cx && (cw += 32) < Q) cx = txor[cw];
          if (!cx) break;
          const int b = __ffs(cx) - 1;
          cx &= cx - 1;
          fc[nf] = cw * 32 + b;
          fneg |= ((tws[cw] >> b) & 1u) << nf;
          ++nf;
        }
        if (!__any_sync(0xffffffffu, nf > 0)) break;
        E v[4][kMaxF];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int jr = j + r * NW;
          const bool ok = r < rpg && jr < rows_g;
          const E* row = row_ptr(ok ? jr : j);
          const bool res = jr < nres;
#pragma unroll
          for (int k = 0; k < kMaxF; ++k)
            v[r][k] = (ok && k < nf) ? (res ? row[fc[k]] : __ldcg(row + fc[k])) : E(0);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int k = 0; k < kMaxF; ++k)
            if (k < nf) acc[r] += ((fneg >> k) & 1u) ? -static_cast<double>(v[r][k]) : static_cast<double>(v[r][k]);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (r >= rpg) break;
        const double s = warp_sum(acc[r]);
        if (lane == 0 && j + r * NW < rows_g) yrow[j + r * NW] += 2.0 * s;
      }
    }
  }
  SCB_DT(1);  // y gathers
  consumer_sync(NW * 32);
  SCB_DT(2);  // sync
  // ---- s' = sgn(y) ----
  for (int jb = 0; jb < rows_g; jb += NW * 32) {
    const int jj = jb + tid;
    const bool ok = jj < rows_g;
    const double y = ok ? yrow[jj] : 0.0;
    if (ok && !isfinite(y)) atomicMin(a.errp + ERR_Y, static_cast<unsigned>(P));
    const unsigned word = __ballot_sync(0xffffffffu, ok && y < 0.0);
    if (lane == 0 && jb + warp * 32 < rows_g) s_nxt[(jb >> 5) + warp] = word;
  }
  consumer_sync(NW * 32);
  SCB_DT(3);  // signs + sync
  const int sw = (rows_g + 31) / 32;
  if (!a.local_dz) {
    // Matrix mode: publish (flipped rows, new signs) of the band; the owner of each
    // 32-column word reads those rows of R after the grid barrier and adds
    // 2 s'_i R[i, cols] to its z state.  No dz partial row here: the pass costs every
    // CTA the same whatever its rows did (no arrival spread at the barrier).
    int nf = 0;
    for (int w = lane; w < a.sw_all; w += 32) {
      uint32_t f = w < sw ? (s_nxt[w] ^ s_cur[w]) : 0u;
      if (w == sw - 1 && (rows_g & 31)) f &= (1u << (rows_g & 31)) - 1u;
      const uint32_t sn = w < sw ? s_nxt[w] : 0u;
      if (warp == 0) __stcg(a.flipw + w, static_cast<unsigned long long>(f) | (static_cast<unsigned long long>(sn) << 32));
      nf += __popc(f);
    }
    if (warp == 0) {
      nf = static_cast<int>(warp_sum(static_cast<double>(nf)));
      if (lane == 0) a.nfrows[0] += nf;  // flipped rows the owners read (traffic accounting)
    }
    SCB_DT(4);
    return;
  }
  // ---- dz over the rows whose sign flipped (ascending rows) ----
  // Rows wider than one warp tile (column chunks, cpr > 1) are covered chunk by
  // chunk: the flipped rows are read once per chunk, each chunk's partial stored.
  constexpr int chunkV = NW * 32 * VPT;
  bool any = false;
  int nfg = 0;  // flipped streamed rows (read from L2 / HBM), counted once
  for (int ck = 0; ck < a.cpr; ++ck) {
    int vidx[VPT];
    bool vok[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int v = ck * chunkV + (k * NW + warp) * 32 + lane;
      vok[k] = v < NV;
      vidx[k] = vok[k] ? v : 0;
    }
    double zacc[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) zacc[i] = 0.0;
    auto add_row = [&](int j, const VT (&xv)[VPT]) {
      const double g = ((s_nxt[j >> 5] >> (j & 31)) & 1u) ? -2.0 : 2.0;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        E x[EPV];
        Vec<E>::split(xv[k], x);
#pragma unroll
        for (int e = 0; e < EPV; ++e) zacc[k * EPV + e] = fma(static_cast<double>(x[e]), g, zacc[k * EPV + e]);
      }
    };
    auto load_row = [&](int j, VT (&xv)[VPT]) {
      const VT* rv = reinterpret_cast<const VT*>(row_ptr(j));
#pragma unroll
      for (int k = 0; k < VPT; ++k) xv[k] = j < nres ? rv[vidx[k]] : __ldcg(rv + vidx[k]);
    };
    // (four rows per round trip, through a local-memory row list, was 10% slower)
    int pend = -1;  // a flipped row whose loads are waiting for a partner (two rows per round trip)
    for (int w = 0; w < sw; ++w) {
      uint32_t f = s_nxt[w] ^ s_cur[w];
      if (w == sw - 1 && (rows_g & 31)) f &= (1u << (rows_g & 31)) - 1u;
      while (f) {
        const int j = w * 32 + __ffs(f) - 1;
        f &= f - 1;
        any = true;
        if (ck == 0 && j >= nres) ++nfg;
        if (pend < 0) {
          pend = j;
          continue;
        }
        VT x0[VPT], x1[VPT];
        load_row(pend, x0);
        load_row(j, x1);
        add_row(pend, x0);  // ascending row order, as before
        add_row(j, x1);
        pend = -1;
      }
    }
    if (pend >= 0) {
      VT x0[VPT];
      load_row(pend, x0);
      add_row(pend, x0);
    }
    if (any) {  // uniform across the CTA (every thread walks the same bits)
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        if (vok[k]) {
#pragma unroll
          for (int e = 0; e < EPV; e += 2)
            __stcg(reinterpret_cast<double2*>(a.zrow + static_cast<size_t>(vidx[k]) * EPV + e),
                   make_double2(zacc[k * EPV + e], zacc[k * EPV + e + 1]));
        }
      }
    }
  }
  SCB_DT(4);  // dz
  if (tid == 0) {
    *a.has_dz = any ? 1 : 0;
    a.nfrows[0] += nfg;       // totals over the run (traffic accounting)
    a.nfrows[1] += any ? 1 : 0;
#ifdef SCB_PROFILE
    if (a.prof && any) a.prof[5] += 1;
#endif
  }
#undef SCB_DT
}

// ---------------------------------------------------------------------------
// Barrier-free delta pass (one GPU, matrices, whole rows).  The same arithmetic as
// delta_pass + the owners' column reduction, but the exchange is a chain of
// self-tagged words with no grid barrier in it and the CTA meets only twice:
//   1. warp 0 polls the pass-tagged t words the owners published, forms t XOR the
//      previous t and lists the flipped columns in ascending order (prefix scan);
//   2. every warp updates y of its rows from that list (lanes stride the list, one
//      L2 round trip per four rows), y_j += 2 sum_c t'_c R[j, c];
//   3. warp 0 takes s' = sgn(y) and publishes the band's {flip, s'} words, then its
//      objective partial sum_j s_j y_j -- every 64-bit word carries the pass index;
//   4. warps 1.. of the column owners poll every CTA's flip words, list the flipped
//      rows (each warp extracts its own slice of the one ascending list, no CTA-wide
//      step), add 2 s'_i R[i, cols] to their z state and publish t' = sgn(z), tagged
//      for the next pass; meanwhile warp 0 polls the c partials and reduces them in
//      the fixed order of the barrier passes, and thread 0 takes the decision.
// Nobody can run more than one pass ahead: pass P + 1 needs every owner's t word,
// which needs every CTA's record of pass P.  Records and t words are
// double-buffered by parity.  Pass-invariant operands sit in shared memory
// (Ctl::fc), so the call passes four scalars.
__device__ __forceinline__ void ld_relaxed64x2(const unsigned long long* p, unsigned long long& a,
                                               unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_relaxed64x2(unsigned long long* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

#ifdef SCB_POLL_SLEEP
#define SCB_POLL_BACKOFF() __nanosleep(SCB_POLL_SLEEP)
#else
#define SCB_POLL_BACKOFF() do {} while (0)
#endif
template <typename E, int NW>
__device__ __noinline__ void fast_delta(const unsigned ctl_off, const int P, const int tsel, const int cur_nxt) {
  constexpr int CT = NW * 32;
  constexpr int NP = NW - 1;  // owner warps (warp 0 runs the objective reduction and the decision)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(128) unsigned char smem[];
  Ctl* ctl = reinterpret_cast<Ctl*>(smem + ctl_off);
  const FastConst& F = ctl->fc;
  const int rows_g = F.rows_g, nres = F.nres, Q = F.Q, G = F.G, sw = F.sw;
  const unsigned uP = static_cast<unsigned>(P);
  double* yrow = reinterpret_cast<double*>(smem + F.yrow);
  const uint32_t* s_cur = reinterpret_cast<const uint32_t*>(smem + F.sb) + (cur_nxt & 3) * sw;
  uint32_t* s_nxt = reinterpret_cast<uint32_t*>(smem + F.sb) + (cur_nxt >> 2) * sw;
  uint32_t* tws = reinterpret_cast<uint32_t*>(smem + F.tws);
  uint32_t* txor = reinterpret_cast<uint32_t*>(smem + F.txor);
  uint32_t* tprev = txor + Q;
  uint32_t* clist = reinterpret_cast<uint32_t*>(smem + F.clist);
  unsigned long long* fws = reinterpret_cast<unsigned long long*>(smem + F.fws);
  const E* Rg = static_cast<const E*>(F.Rrows);
  const unsigned long long* rec_in = F.drec + static_cast<size_t>(P & 1) * G * F.rstride;
#ifdef SCB_PROFILE
  long long ft0 = clock64();
#define SCB_FT(k) do { if (F.prof && (tid == 0 || tid == 32)) { const long long t1_ = clock64(); if (tid == ((k) >= 8 ? 32 : 0)) ctl->fprof[k] += t1_ - ft0; ft0 = t1_; } } while (0)
#else
#define SCB_FT(k) do {} while (0)
#endif

  // list entries [base, base + kCList) of the flipped columns (ascending): lane l
  // covers words 4l..4l+3 of every block of 128 t words
  auto emit = [&](const uint32_t (&xs)[4], const uint32_t (&tn)[4], int i0, int base, int run) -> int {
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) cnt += __popc(xs[u]);
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    int pos = run + inc - cnt - base;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint32_t x = xs[u];
      const int c0 = (i0 + 4 * lane + u) * 32;
      while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        if (pos >= 0 && pos < kCList) clist[pos] = static_cast<uint32_t>(c0 + b) | (((tn[u] >> b) & 1u) << 31);
        ++pos;
      }
    }
    return run + __shfl_sync(0xffffffffu, inc, 31);
  };

  // ---- 1. this pass's t (warp 0) ----
  if (warp == 0) {
    const unsigned long long* tw = F.tb64 + static_cast<size_t>(tsel) * Q * kTbStride;
    int run = 0;
#pragma unroll 1
    for (int i0 = 0; i0 < Q; i0 += 128) {
      unsigned long long v[4];
      bool need[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        need[u] = i0 + 4 * lane + u < Q;
        v[u] = 0ull;
      }
      for (;;) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (need[u]) v[u] = ld_relaxed64(tw + static_cast<size_t>(i0 + 4 * lane + u) * kTbStride);
        bool pend = false;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (need[u]) {
            if (static_cast<int>(static_cast<unsigned>(v[u] >> 32) - uP) >= 0)
              need[u] = false;
            else
              pend = true;
          }
        if (!pend) break;
      }
      uint32_t xs[4], tn[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 4 * lane + u;
        tn[u] = static_cast<uint32_t>(v[u]);
        xs[u] = i < Q ? (tn[u] ^ tprev[i]) : 0u;
      }
      if (i0 == 0) SCB_FT(0);
      run = emit(xs, tn, i0, 0, run);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 4 * lane + u;
        if (i < Q) {
          txor[i] = xs[u];
          tprev[i] = tn[u];
          tws[i] = tn[u];
        }
      }
    }
    if (lane == 0) {
      ctl->nflip = run;
      ctl->keep = run == 0;
      ctl->err_pre[0] = UINT_MAX;
      ctl->err_pre[1] = UINT_MAX;
      ctl->err_pre[2] = UINT_MAX;
    }
  }
  consumer_sync(CT);
  SCB_FT(1);
  const int nfl = ctl->nflip;

  // ---- 2. y update: warp w takes rows w, w + NW, ... four at a time ----
  for (int base = 0;;) {
    const int cn = min(kCList, nfl - base);
    // rows per warp and round: no more than the band gives every warp (the same per-lane
    // sums and the same butterfly for every RPG, so the choice never changes a bit)
    auto gather = [&](auto rpg_c) {
      constexpr int RPG = decltype(rpg_c)::value;
#pragma unroll 1
      for (int j0 = warp; j0 < rows_g; j0 += RPG * NW) {
        double acc[RPG];
#pragma unroll
        for (int r = 0; r < RPG; ++r) acc[r] = 0.0;
#pragma unroll 1
        for (int k0 = 0; k0 < cn; k0 += 64) {  // two list entries per lane and round: 2 RPG loads in flight
          uint32_t e[2];
          E v[RPG][2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int k = k0 + u * 32 + lane;
            e[u] = k < cn ? clist[k] : 0xffffffffu;
          }
          // (every row is current in global R; SMEM-resident rows are read from L2 like the
          // rest -- one load path keeps this once-per-pass code short)
#pragma unroll
          for (int r = 0; r < RPG; ++r) {
            const int jr = j0 + r * NW;
            const bool ok = jr < rows_g;
            const E* row = Rg + static_cast<size_t>(ok ? jr : j0) * F.pitch;
#pragma unroll
            for (int u = 0; u < 2; ++u)
              v[r][u] = (ok && e[u] != 0xffffffffu) ? __ldcg(row + (e[u] & 0x7fffffffu)) : E(0);
          }
#pragma unroll
          for (int r = 0; r < RPG; ++r)
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const double d = static_cast<double>(v[r][u]);
              acc[r] += (e[u] >> 31) ? -d : d;
            }
        }
        const double s = warp_reduce_rows<RPG>(acc, lane);
#pragma unroll
        for (int r = 0; r < RPG; ++r)
          if (lane == holder_lane<RPG>(r) && j0 + r * NW < rows_g) yrow[j0 + r * NW] += 2.0 * s;
      }
    };
    if (rows_g > 2 * NW)
      gather(std::integral_constant<int, 4>{});
    else if (rows_g > NW)
      gather(std::integral_constant<int, 2>{});
    else
      gather(std::integral_constant<int, 1>{});
    base += kCList;
    if (base >= nfl) break;
    consumer_sync(CT);  // more flips than one list holds: the next chunk of the list
    if (warp == 0) {
      int run = 0;
#pragma unroll 1
      for (int i0 = 0; i0 < Q; i0 += 128) {
        uint32_t xs[4], tn[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + 4 * lane + u;
          xs[u] = i < Q ? txor[i] : 0u;
          tn[u] = i < Q ? tws[i] : 0u;
        }
        run = emit(xs, tn, i0, base, run);
      }
    }
    consumer_sync(CT);
  }
  // only warp 0 waits for every row's y; the other warps go on to the records
  if (warp != 0) {
    asm volatile("bar.arrive 3, %0;" ::"r"(CT) : "memory");
  } else {
    asm volatile("bar.sync 3, %0;" ::"r"(CT) : "memory");
  }
  SCB_FT(2);

  if (warp == 0) {
    // ---- 3. s' = sgn(y), flips, then the objective partial; publish both ----
    unsigned long long* rec_out = const_cast<unsigned long long*>(rec_in) + static_cast<size_t>(F.g) * F.rstride;
    const unsigned long long tag = static_cast<unsigned long long>(uP) << 32;
    bool bad = false;
    int nfr = 0;
#pragma unroll 1
    for (int w = 0; w < sw; ++w) {
      const int j = w * 32 + lane;
      const bool ok = j < rows_g;
      const double y = ok ? yrow[j] : 0.0;
      bad |= ok && !isfinite(y);
      const uint32_t sn = __ballot_sync(0xffffffffu, ok && y < 0.0);
      const uint32_t f = sn ^ s_cur[w];  // bits past rows_g are zero in both
      if (lane == 0) {
        st_relaxed64x2(rec_out + 2 * w, tag | f, tag | sn);
        s_nxt[w] = sn;
      }
      nfr += __popc(f);
    }
    // this CTA's c partial: sum_i s_i y_i in row order (lane-strided, fixed tree)
    double cl = 0.0;
#pragma unroll 1
    for (int j = lane; j < rows_g; j += 32) cl += flipd(yrow[j], ((s_cur[j >> 5] >> (j & 31)) & 1u) << 31);
    cl = warp_sum(cl);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      if (bad) atomicMin(F.errp + ERR_Y, uP);
      const unsigned long long tagc = tag | ((bad || ctl->zerr) ? (1ull << 63) : 0ull);
      st_relaxed64x2(rec_out + 2 * sw, tagc | static_cast<uint32_t>(__double2hiint(cl)),
                     tagc | static_cast<uint32_t>(__double2loint(cl)));
      ctl->nfrows += nfr;  // flipped rows the owners read (traffic accounting)
    }
    SCB_FT(3);
    // ---- 4a. every CTA's c partial, reduced in the order of the barrier passes:
    // CTA 32 k + lane in "warp" k (butterfly), then k ascending (thread 0) ----
    // (all loads in flight together, then the butterflies side by side: this runs ahead
    // of the decision, which the whole CTA waits for at the end of the pass).  In an owner
    // CTA the polling starts once the owner warps hold every CTA's flip words: each CTA
    // publishes its c pair right after its flip pair, so nothing is lost and the c
    // records are not polled while they cannot be complete.
    if (F.nls > 0 && F.cpar) asm volatile("bar.sync 5, %0;" ::"r"(CT) : "memory");
    bool flag = false;
    constexpr int KC = 5;  // G <= 160 (host gate)
    unsigned long long cw0[KC], cw1[KC];
    unsigned need = 0;
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      cw0[k] = 0ull;
      cw1[k] = 0ull;
      if (k * 32 + lane < G) need |= 1u << k;
    }
    const unsigned long long* pc = rec_in + static_cast<size_t>(lane) * F.rstride + 2 * sw;
    while (need) {
#pragma unroll
      for (int k = 0; k < KC; ++k)
        if ((need >> k) & 1u) ld_relaxed64x2(pc + static_cast<size_t>(k) * 32 * F.rstride, cw0[k], cw1[k]);
#pragma unroll
      for (int k = 0; k < KC; ++k)
        if (((need >> k) & 1u) && (static_cast<unsigned>(cw0[k] >> 32) & 0x7fffffffu) == uP &&
            (static_cast<unsigned>(cw1[k] >> 32) & 0x7fffffffu) == uP)
          need &= ~(1u << k);
    }
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      if (k >= NW) break;
      double c = 0.0;
      if (k * 32 + lane < G) {
        c = __hiloint2double(static_cast<int>(static_cast<uint32_t>(cw0[k])), static_cast<int>(static_cast<uint32_t>(cw1[k])));
        flag |= (cw0[k] >> 63) != 0ull;
      }
      if (k * 32 < G) c = warp_sum(c);
      if (lane == 0) {
        ctl->cred[k] = c;
        ctl->nred[k] = 0.0;
      }
    }
    if (lane == 0)
      for (int k = KC; k < NW; ++k) {
        ctl->cred[k] = 0.0;
        ctl->nred[k] = 0.0;
      }
    flag = __any_sync(0xffffffffu, flag);
    if (flag && lane == 0) ctl->err_pre[0] = uP;  // some CTA saw a non-finite value: every CTA stops at this pass
    __syncwarp();
    SCB_FT(4);
    return;
  }

  // ---- 4b. owners (warps 1..): flip words of every CTA, then the column update ----
  const int nls = F.nls;
  if (nls == 0) return;
  const int lw = warp - 1, lt = tid - 32;
  // z state of this warp's column word (final warps only), issued early
  const int colz = (F.g + lw * G) * 32 + lane;
  double zs = 0.0;
  if (lw < nls && colz < F.n) zs = __ldcg(F.zstate + colz);
  const int items = G * sw;
  int cnt = 0, inc, k0, k1;
  int i0 = 0, i1 = 0;          // staged form: this lane's flip-word entries
  uint32_t myf = 0, mysn = 0;  // direct form: this lane's flip word and new signs
  int myrb = 0;                //              and the first row they stand for
  if (F.direct) {
    // Direct form (every warp's share of the flip words fits its lanes): warp lw takes
    // the CTAs [gs, ge) -- lane l polls their l-th flip pair itself, so the warp moves
    // on as soon as ITS CTAs have published, with no staging and no meeting of the
    // owner warps before the final combine.  Rows stay in ascending order per warp.
    const int gs = (lw * G) / NP, ge = ((lw + 1) * G) / NP;
    const int e = gs * sw + lane;
    if (e < ge * sw) {
      const int g2 = sw == 1 ? e : e / sw, w = e - g2 * sw;
      const unsigned long long* q = rec_in + static_cast<size_t>(g2) * F.rstride + 2 * w;
      unsigned long long f0, f1;
      do {
        ld_relaxed64x2(q, f0, f1);
      } while (static_cast<unsigned>(f0 >> 32) != uP || static_cast<unsigned>(f1 >> 32) != uP);
      myf = static_cast<uint32_t>(f0);
      mysn = static_cast<uint32_t>(f1);
      myrb = g2 * F.rows_base + min(g2, F.rows_rem) + w * 32;
    }
    __syncwarp();
    if (F.cpar) asm volatile("bar.arrive 5, %0;" ::"r"(CT) : "memory");  // warp 0 starts polling the c partials
    SCB_FT(8);
    cnt = __popc(myf);
  } else {
#pragma unroll 1
    for (int idx = lt; idx < items; idx += NP * 32) {
      const int g2 = sw == 1 ? idx : idx / sw;
      const unsigned long long* q = rec_in + static_cast<size_t>(g2) * F.rstride + 2 * (idx - g2 * sw);
      unsigned long long f0, f1;
      do {
        ld_relaxed64x2(q, f0, f1);
        SCB_POLL_BACKOFF();
      } while (static_cast<unsigned>(f0 >> 32) != uP || static_cast<unsigned>(f1 >> 32) != uP);
      fws[idx] = static_cast<unsigned long long>(static_cast<uint32_t>(f0)) | (f1 << 32);
    }
    if (F.cpar) asm volatile("bar.arrive 5, %0;" ::"r"(CT) : "memory");  // warp 0 starts polling the c partials
    asm volatile("bar.sync 2, %0;" ::"r"(NP * 32) : "memory");
    SCB_FT(8);
    if (F.shared_list) return;  // many flip words (tall bands): the caller runs col_reduce's shared row list
    // this warp's slice of the one ascending list of flipped rows (every warp scans
    // all flip words; lane l covers entries [l per, (l + 1) per))
    const int per = (items + 31) / 32;
    i0 = min(items, lane * per);
    i1 = min(items, i0 + per);
#pragma unroll 1
    for (int i = i0; i < i1; ++i) cnt += __popc(static_cast<uint32_t>(fws[i]));
  }
  inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  const int total = __shfl_sync(0xffffffffu, inc, 31);
  SCB_FT(11);
  if (F.direct) {
    k0 = 0;
    k1 = total;
  } else {
    k0 = (total * lw) / NP;
    k1 = (total * (lw + 1)) / NP;
  }
  uint32_t* buf = reinterpret_cast<uint32_t*>(smem + F.fbuf) + lw * kFBuf;
  const E* Rc = static_cast<const E*>(F.R) + F.g * 32 + lane;  // column of word 0; word j: + j * G * 32
  // this warp's partial of every owned word accumulates in its own zseg slot
  double* zseg = reinterpret_cast<double*>(smem + F.zseg);
#pragma unroll 1
  for (int j = 0; j < nls; ++j) zseg[(j * NW + lw) * 32 + lane] = 0.0;
#pragma unroll 1
  for (int c0 = k0; c0 < k1; c0 += kFBuf) {
    const int c1 = min(c0 + kFBuf, k1);
    if (F.direct) {
      int pos = inc - cnt;
      uint32_t f = myf;
      while (f) {
        const int b = __ffs(f) - 1;
        f &= f - 1;
        if (pos >= c0 && pos < c1) buf[pos - c0] = static_cast<uint32_t>(myrb + b) | (((mysn >> b) & 1u) << 31);
        ++pos;
      }
    } else {
      int pos = inc - cnt;
      int gp = sw == 1 ? i0 : i0 / sw, w = i0 - gp * sw;
#pragma unroll 1
      for (int i = i0; i < i1; ++i) {
        const unsigned long long fw = fws[i];
        uint32_t f = static_cast<uint32_t>(fw);
        const uint32_t sn = static_cast<uint32_t>(fw >> 32);
        const int rb = gp * F.rows_base + min(gp, F.rows_rem) + w * 32;
        while (f) {
          const int b = __ffs(f) - 1;
          f &= f - 1;
          if (pos >= c0 && pos < c1) buf[pos - c0] = static_cast<uint32_t>(rb + b) | (((sn >> b) & 1u) << 31);
          ++pos;
        }
        if (++w == sw) {
          w = 0;
          ++gp;
        }
      }
    }
    __syncwarp();
    SCB_FT(12);
#pragma unroll 1
    for (int k = 0; k < c1 - c0; k += 8) {
      uint32_t e[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) e[u] = (k + u < c1 - c0) ? buf[k + u] : 0xffffffffu;
#pragma unroll 1
      for (int j = 0; j < nls; ++j) {  // eight row loads of one owned word in flight
        E v[8];
        const E* Rj = Rc + static_cast<size_t>(j) * G * 32;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = e[u] != 0xffffffffu ? __ldcg(Rj + static_cast<size_t>(e[u] & 0x7fffffffu) * F.pitch) : E(0);
        double a = zseg[(j * NW + lw) * 32 + lane];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e[u] != 0xffffffffu) a = fma(static_cast<double>(v[u]), (e[u] >> 31) ? -2.0 : 2.0, a);
        zseg[(j * NW + lw) * 32 + lane] = a;
      }
    }
    __syncwarp();
  }
  SCB_FT(9);
  if (lw >= nls) {  // partial delivered; only the word's final warp waits
    asm volatile("bar.arrive 4, %0;" ::"r"(NP * 32) : "memory");
    return;
  }
  asm volatile("bar.sync 4, %0;" ::"r"(NP * 32) : "memory");
  {
    double z = 0.0;
#pragma unroll
    for (int w = 0; w < NP; ++w) z += zseg[(lw * NW + w) * 32 + lane];
    const bool valid = colz < F.n;
    z = zs + z;
    if (valid) __stcg(F.zstate + colz, z);
    if (valid && !isfinite(z)) {
      atomicMin(F.errp + ERR_Z, uP);
      ctl->zerr = 1;
    }
    const unsigned word = __ballot_sync(0xffffffffu, valid && z < 0.0);
    const int qq = F.g + lw * G;
    if (lane == 0)
      st_relaxed64(F.tb64 + (static_cast<size_t>(tsel ^ 1) * Q + qq) * kTbStride,
                   (static_cast<unsigned long long>(uP + 1u) << 32) | word);
  }
  SCB_FT(10);
#undef SCB_FT
}

// ---------------------------------------------------------------------------
// Order-k tensors (axial_run, search.hpp:191-213) on the matrix view
// M = n_0 x N', N' = n_1 ... n_{k-1} (row-major, last axis fastest).  Axis 0 of
// a sweep is the dot pass (y = M kron(s_1..s_{k-1}), s_0 = sgn(y)); its column
// reduction gives Z = M^T s_0, from which the trailing axes are updated in
// order (Gauss-Seidel: axis i uses the new s_j, j < i, and the old s_j, j > i):
//   v_i[q] = sum over Z entries with index_i = q of Z * prod_{j != i} s_j,
//   s_i = sgn(v_i), and c = <s_{k-1}, v_{k-1}> = sum_q |v_{k-1}[q]|.
// Every CTA runs this redundantly on the same data in the same order, so all
// CTAs hold identical signs and c (deterministic fixed-order sums).
__device__ __forceinline__ uint32_t axbit(const Ctl* ctl, const uint32_t* sax, int j, int idx) {
  return (sax[ctl->axoff[j] + (idx >> 5)] >> (idx & 31)) & 1u;
}
// t word q of kron(s_1, ..., s_{k-1}) over the N' columns: the multi-index of
// the word's first column is decomposed once (32-bit), then advanced as an
// odometer whose running parity is updated incrementally.  Axis extents and
// offsets come from shared memory (ctl), never from the local-memory copy of
// the kernel parameters.
__device__ uint32_t kron_word(const KParams& p, const Ctl* ctl, const uint32_t* sax, int q) {
  const int col0 = q * 32;
  const int n = p.n, kax = p.kax;
  if (col0 >= n) return 0u;
  const int nb = min(32, n - col0);
  uint32_t word = 0;
  if (kax == 2) {  // order 3: two trailing axes, scalar odometer
    const int n2 = ctl->axn[1];
    int i1 = col0 / n2, i2 = col0 - i1 * n2;
    const uint32_t* w1 = sax + ctl->axoff[0];
    const uint32_t* w2 = sax + ctl->axoff[1];
    uint32_t b1 = (w1[i1 >> 5] >> (i1 & 31)) & 1u;
    for (int b = 0; b < nb; ++b) {
      word |= (b1 ^ ((w2[i2 >> 5] >> (i2 & 31)) & 1u)) << b;
      if (++i2 == n2) {
        i2 = 0;
        ++i1;
        b1 = (w1[i1 >> 5] >> (i1 & 31)) & 1u;
      }
    }
    return word;
  }
  int idx[7];
  uint32_t xb = 0;
  int c = col0;
  for (int j = kax - 1; j >= 0; --j) {
    const int nj = ctl->axn[j];
    idx[j] = c % nj;
    c /= nj;
    xb ^= axbit(ctl, sax, j, idx[j]);
  }
  for (int b = 0; b < nb; ++b) {
    word |= xb << b;
    for (int j = kax - 1; j >= 0; --j) {  // advance the odometer by one column
      xb ^= axbit(ctl, sax, j, idx[j]);
      if (++idx[j] < ctl->axn[j]) {
        xb ^= axbit(ctl, sax, j, idx[j]);
        break;
      }
      idx[j] = 0;
      xb ^= axbit(ctl, sax, j, 0);
    }
  }
  return word;
}

// The trailing-axis update of one sweep.  Outputs of axis i are spread over the
// CTA by their count n_i: few outputs (n_i <= CW) use the whole CTA per output,
// otherwise groups of T = 32 / 2^k lanes share one output (T ~ CT / n_i), each
// group summing a strided slice of the other axes' combinations and combining
// with a fixed butterfly -- so thousands of L2 loads are in flight instead of a
// few warps walking the slices serially.  All index arithmetic is 32-bit.
template <int CW>
__device__ __noinline__ void axial_step(const KParams& p, uint32_t* sax, uint32_t* tws, const uint32_t* tpass,
                                      Ctl* ctl, int P, long long* tsplit) {
  constexpr int CT = CW * 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kax = p.kax;
  const double* Z = p.zfull;
  unsigned* errp = p.err_pass;
  int zstride[7];
  {
    int st = 1;
    for (int j = kax - 1; j >= 0; --j) {
      zstride[j] = st;
      st *= ctl->axn[j];
    }
  }
  double csum = 0.0;
  if (tid == 0) ctl->nflip = 0;  // recounted below for the next pass's t
  if (kax == 0 && tid == 0) csum = __ldcg(Z);  // order 1: c = <s_0, a> = Z[0]
  long long tprev = tsplit ? clock64() : 0;
  // Order 3 with a short last axis (an image: n_2 = 3 channels, up to 4): both trailing axes in
  // one walk over Z.  Thread tid takes q = tid, tid + CT, ... of axis 1: it loads Z[q, 0..n_2),
  // forms v_1[q] with the old axis-2 signs (terms in ascending r), ballots the new s_1 word, and
  // at once adds its row, flipped by its own new s_1[q], to the axis-2 sums -- the Gauss-Seidel
  // order and every summation order of the general path below (which this block replaces for
  // these shapes: same partials per thread, same butterflies, same warp order), in a fraction
  // of its code: the step runs once per pass, cold, and was 40% of the C3 pass.
  // (n_1 > 2 CT: where the general path also gives one thread per axis-1 output, so the sums
  // are the same bit for bit)
  const bool fused3 = kax == 2 && ctl->axn[1] <= 4 && ctl->axn[1] <= CW && ctl->axn[0] > 2 * CT;
  if (fused3) {
    const int n1 = ctl->axn[0], n2 = ctl->axn[1];
    uint32_t* w1 = sax + ctl->axoff[0];
    uint32_t* w2 = sax + ctl->axoff[1];
    const uint32_t s2old = w2[0];  // n_2 <= 4 bits
    consumer_sync(CT);
    if (tid == 0) w2[0] = 0u;
    double a2[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
    for (int q = tid; q - tid < n1; q += CT) {  // warp-uniform trip count (ballots inside)
      const bool ok = q < n1;
      double z[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (ok && r < n2) z[r] = __ldcg(Z + q * n2 + r);
      double v = 0.0;
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (r < n2) v += flipd(z[r], ((s2old >> r) & 1u) << 31);
      const bool neg = ok && v < 0.0;
      const unsigned word = __ballot_sync(0xffffffffu, neg);
      if (lane == 0 && ok) w1[q >> 5] = word;
      if (ok) {
        if (!isfinite(v)) atomicMin(errp + ERR_Z, static_cast<unsigned>(P));
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (r < n2) a2[r] += flipd(z[r], neg ? 0x80000000u : 0u);
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const double t = warp_sum(a2[r]);
      if (lane == 0 && r < n2) ctl->cred[r * CW + warp] = t;
    }
    consumer_sync(CT);
    if (tid < n2) {
      double t = 0.0;
      for (int w = 0; w < CW; ++w) t += ctl->cred[tid * CW + w];
      if (!isfinite(t)) atomicMin(errp + ERR_Z, static_cast<unsigned>(P));
      if (t < 0.0) atomicOr(&w2[0], 1u << tid);
      csum += fabs(t);
    }
    consumer_sync(CT);
    if (tsplit && tid == 0) {
      const long long t = clock64();
      tsplit[0] += t - tprev;
      tprev = t;
    }
  }
  for (int i = 0; i < kax && !fused3; ++i) {
    const int ni = ctl->axn[i];
    const int other = p.n / ni;
    uint32_t* wi = sax + ctl->axoff[i];
    const int nwi = (ni + 31) / 32;
    // signed Z entry of (index_i = q, r-th combination of the other axes, last fastest)
    auto term = [&](int q, int r) -> double {
      if (kax == 2) {  // order 3 (the common case): Z is n_1 x n_2, no index arithmetic
        const int j = 1 - i;
        return flipd(__ldcg(Z + (i == 0 ? q * ctl->axn[1] + r : r * ctl->axn[1] + q)), axbit(ctl, sax, j, r) << 31);
      }
      int flat = q * zstride[i];
      uint32_t xb = 0;
      for (int j = kax - 1; j >= 0; --j) {
        if (j == i) continue;
        const int nj = ctl->axn[j];
        const int ij = r % nj;
        r /= nj;
        flat += ij * zstride[j];
        xb ^= axbit(ctl, sax, j, ij);
      }
      return flipd(__ldcg(Z + flat), xb << 31);
    };
    for (int wq = tid; wq < nwi; wq += CT) wi[wq] = 0u;
    consumer_sync(CT);
    if (ni <= 4 && ni <= CW) {  // few outputs: the whole CTA sums all of them at once
      double v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
      for (int r = tid; r < other; r += CT) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q < ni) v[q] += term(q, r);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double t = warp_sum(v[q]);
        if (lane == 0 && q < ni) ctl->cred[q * CW + warp] = t;
      }
      consumer_sync(CT);
      if (tid < ni) {
        const int q = tid;
        double t = 0.0;
        for (int w = 0; w < CW; ++w) t += ctl->cred[q * CW + w];
        if (!isfinite(t)) atomicMin(errp + ERR_Z, static_cast<unsigned>(P));
        if (t < 0.0) atomicOr(&wi[q >> 5], 1u << (q & 31));
        if (i == kax - 1) csum += fabs(t);
      }
      consumer_sync(CT);
    } else {  // T lanes per output
      int T = 32;
      while (T > 1 && ni * T > 2 * CT) T >>= 1;
      const int groups = CT / T, sub = tid & (T - 1);
#pragma unroll 1
      for (int q = tid / T; q - tid / T < ni; q += groups) {
        const bool ok = q < ni;
        double v = 0.0;
        if (ok) {
#pragma unroll 1
          for (int r = sub; r < other; r += T) v += term(q, r);
        }
        for (int o = T >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (T == 1) {  // the warp's 32 consecutive outputs form one word: no atomics
          const unsigned word = __ballot_sync(0xffffffffu, ok && v < 0.0);
          if (lane == 0 && q < ni) wi[q >> 5] = word;
        } else if (ok && sub == 0 && v < 0.0) {
          atomicOr(&wi[q >> 5], 1u << (q & 31));
        }
        if (ok && sub == 0) {
          if (!isfinite(v)) atomicMin(errp + ERR_Z, static_cast<unsigned>(P));
          if (i == kax - 1) csum += fabs(v);
        }
      }
    }
    consumer_sync(CT);
    if (tsplit && tid == 0 && i < 2) {
      const long long t = clock64();
      tsplit[i] += t - tprev;
      tprev = t;
    }
  }
  csum = warp_sum(csum);
  if (lane == 0) ctl->cred[warp] = csum;
  {
    int nf = 0;  // flips of the next pass's t against this pass's (tpass, set at staging)
    for (int q = tid; q < p.Q; q += CT) {
      const uint32_t w = kron_word(p, ctl, sax, q);
      nf += __popc(w ^ tpass[q]);
      tws[q] = w;
    }
    if (nf) atomicAdd(&ctl->nflip, nf);
  }
  consumer_sync(CT);
  if (tsplit && tid == 0) tsplit[2] += clock64() - tprev;
  if (tid == 0) {
    double c = 0.0;
    for (int w = 0; w < CW; ++w) c += ctl->cred[w];
    ctl->ax_c = c;
  }
}

// ---------------------------------------------------------------------------
// Order-k controller step for a sweep that continues (kept out of line: the matrix
// decision path stays compact in the instruction cache).  The next t is kron(new axes),
// already in tws; this sweep's s_0 becomes the delta pass's previous s.
__device__ __noinline__ int tensor_continue(Ctl* ctl, int delta, int refresh, int div, int n) {
  ctl->tsel = 0;
  const int t = ctl->cur;
  ctl->cur = ctl->nxt;
  ctl->nxt = t;
  if (delta && ctl->since_dense + 1 < refresh && static_cast<long long>(ctl->nflip) * div <= n) {
    ctl->since_dense += 1;
    return F_DOT | F_DELTA;
  }
  ctl->since_dense = 0;
  return F_DOT;
}

// Column ownership: consumer thread (warp w, lane l) owns the 16-byte vectors
// v_k = (k * NW + w) * 32 + l, k < VPT, of every row (coalesced LDS.128), i.e.
// NE = VPT * EPV elements per row, and the matching NE f64 column accumulators.
// CPS: CTAs per SM (1, or 2 with a 112-register budget and raw lag buffers).
// MR: the multi-rank (row-sharded, world > 1) exchange is compiled in.  The
// single-GPU kernels carry none of it (smaller code on the per-pass path).
template <typename E, int NW, int VPT, int RG, int CPS, bool TS, bool MR = false>
__device__ __forceinline__ void sweep_body(const KParams& p, const int g) {
  constexpr int EPV = Vec<E>::N;
  constexpr int CW = NW;       // consumer warps
  constexpr int CT = CW * 32;  // consumer threads
  constexpr int NE = VPT * EPV;
  static_assert(NE <= 32, "sign bits of a thread's elements must fit one word");
  static_assert(CW <= 32, "controller arrays hold 32 warps");
  using VT = typename Vec<E>::T;

  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int G = p.G;
  if (p.fault) return;  // test hook: a rank that never joins (the others must time out, not hang)
  const long long pitch = p.pitch;
  const size_t rowB = static_cast<size_t>(pitch) * sizeof(E);
  const int NV = static_cast<int>(pitch / EPV);
  const int rows_g = p.rows_base + (g < p.rows_rem ? 1 : 0);
  const int r0 = g * p.rows_base + min(g, p.rows_rem);
  const int nres = min(rows_g, p.res_rows);
  const int nstream = rows_g - nres;
  const int D = p.stages;

  // stage = one row, or one column chunk of a wide row (then no resident rows)
  const size_t stageB = p.cpr > 1 ? static_cast<size_t>(p.chunk_cols) * sizeof(E) : rowB;
  const int npieces = nstream * p.cpr;  // TMA pieces per streaming sweep over the band
  const Layout L = make_layout(stageB, D, p.res_rows, RG, NW, p.rows_max, p.Q, p.zl, p.sw, p.axw, G);
  unsigned char* stage_base = smem + L.stage;
  unsigned char* res_base = smem + L.res;
  Ctl* ctl = reinterpret_cast<Ctl*>(smem + L.ctl);
  unsigned long long* ring = reinterpret_cast<unsigned long long*>(smem + L.ring);  // [kRing] mbarriers
  double* yrow = reinterpret_cast<double*>(smem + L.yrow);                 // [rows_max]
  uint32_t* tws = reinterpret_cast<uint32_t*>(smem + L.tws);               // [Q] t of this pass
  uint32_t* uws = reinterpret_cast<uint32_t*>(smem + L.uws);               // [Q] t of the update
  double* zseg = reinterpret_cast<double*>(smem + L.zseg);                 // [zl][CW][32]
  double* zst = reinterpret_cast<double*>(smem + L.zst);                   // [zl][32]
  uint32_t* sb = reinterpret_cast<uint32_t*>(smem + L.sb);                 // [3][sw]
  uint32_t* txor = reinterpret_cast<uint32_t*>(smem + L.txor);             // [Q] t ^ previous t
  uint32_t* tprev = txor + p.Q;                                            // [Q] previous pass's t
  uint32_t* dzmask = reinterpret_cast<uint32_t*>(smem + L.dzmask);         // [64] CTAs with a dz partial
  unsigned long long* fws = reinterpret_cast<unsigned long long*>(smem + L.fws);  // [G][sw] flip words of the pass
  uint32_t* fbuf = reinterpret_cast<uint32_t*>(smem + L.fbuf);             // [CW][kFBuf] flipped-row lists
  double* ybak = reinterpret_cast<double*>(smem + L.ybak);                 // [rows_max] cached y
  uint32_t* sax = reinterpret_cast<uint32_t*>(smem + L.ax);                // [axw] axes 1..k-1 (order-k)
  uint32_t* sax_best = sax + p.axw;                                        // [axw] best restart's
  E* R = static_cast<E*>(p.R);

  if (tid == 0) {
    for (int s = 0; s < D; ++s) {
      mbar_init(&ctl->full[s], 1);
      mbar_init(&ctl->empty[s], NW);
    }
    for (int s = 0; s < kRing; ++s) mbar_init(&ring[s], NW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int k0 = p.width == 0 ? (F_NORM | F_WB | F_CHECK) : (F_NORM | F_CHECK);
    ctl->kind = k0;
    ctl->kind_ring[0] = k0;
    ctl->decided = 1;
    ctl->stored = 0;
    ctl->abort = 0;
    ctl->aborted = 0;
    ctl->upd_done = 0;
    ctl->rank_dz = 0;
    ctl->pp = TS ? 1 : 0;  // order-k: pp = sweep of the current pass (1-based)
    for (int j = 0; j < 8; ++j) {  // read by the axial step from shared memory, not the param copy
      ctl->axn[j] = j < 7 ? p.ax_n[j] : 1;
      ctl->axoff[j] = j < 7 ? p.ax_off[j] : 0;
    }
    ctl->kron_upd = 0;
    ctl->nflip = 0;
    ctl->nfrows = 0;
    ctl->ndz = 0;
    ctl->since_dense = 0;
    ctl->has_dz = 0;
    ctl->keep = 0;
    ctl->zerr = 0;
    for (int k = 0; k < 16; ++k) ctl->fprof[k] = 0;
    {  // pass-invariant operands of the barrier-free delta pass
      FastConst& fc = ctl->fc;
      fc.Rrows = R + static_cast<size_t>(r0) * pitch;
      fc.R = R;
      fc.drec = p.drec;
      fc.tb64 = p.tb64;
      fc.zstate = p.zstate;
      fc.errp = p.err_pass;
#ifdef SCB_PROFILE
      fc.prof = p.prof ? p.prof + static_cast<size_t>(p.G) * 16 + g * 16 : nullptr;
#else
      fc.prof = nullptr;
#endif
      fc.pitch = pitch;
      fc.res = static_cast<unsigned>(L.res);
      fc.yrow = static_cast<unsigned>(L.yrow);
      fc.sb = static_cast<unsigned>(L.sb);
      fc.tws = static_cast<unsigned>(L.tws);
      fc.txor = static_cast<unsigned>(L.txor);
      fc.clist = static_cast<unsigned>(L.clist);
      fc.fws = static_cast<unsigned>(L.fws);
      fc.fbuf = static_cast<unsigned>(L.fbuf);
      fc.zseg = static_cast<unsigned>(L.zseg);
      fc.rowB = static_cast<unsigned>(rowB);
      fc.rows_g = rows_g;
      fc.nres = nres;
      fc.Q = p.Q;
      fc.G = G;
      fc.sw = p.sw;
      fc.rstride = p.rstride;
      fc.n = p.n;
      fc.g = g;
      fc.rows_base = p.rows_base;
      fc.rows_rem = p.rows_rem;
      int nls = 0;
      for (int j = 0; j < 4; ++j)
        if (g + j * G < p.Q) nls = j + 1;
      fc.nls = nls;
      // tall bands (many flip words per pass): one row list built by all owner warps
      // together (col_reduce) beats every warp scanning all the words
      fc.shared_list = G * p.sw > 256 ? 1 : 0;
      // Warp 0 polls every c partial at once (one butterfly at a time was 7% slower on 4096^2 and
      // 10-13% on 1024^2, 512^2 and 1024 x 4096: the decision is the late part of the pass).  On
      // bands of more than 16 rows it starts once the owner warps hold every flip word (cpar);
      // on short bands that wait cost 2-4%, so there it polls from the start.
      fc.cpar = p.rows_max > 16 ? 1 : 0;
      // every owner warp's share of the flip words fits its 32 lanes: direct form
      fc.direct = (!fc.shared_list && ((G + (NW - 1) - 1) / (NW - 1) + 1) * p.sw <= 32) ? 1 : 0;
    }
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
  // resident rows: loaded once for the whole decomposition
  for (int l = 0; l < nres; ++l) {
    const VT* src = reinterpret_cast<const VT*>(R + static_cast<size_t>(r0 + l) * pitch);
    VT* dst = reinterpret_cast<VT*>(res_base + static_cast<size_t>(l) * rowB);
    for (int v = tid; v < NV; v += blockDim.x) dst[v] = __ldcg(src + v);
  }
  __syncthreads();

  // ======================= TMA producer (one thread) =======================
  // Keep this loop lean: the producer warp shares SMSP 0 with two consumer
  // warps, and every instruction it issues is taken from them (runtime integer
  // divisions here cost ~10% of the pass; one lane per stage was slower still).
  if (warp == CW) {
    if (lane != 0 || nstream == 0) return;
    unsigned q = 0;
    int ps = 0, pph = 0;  // stage slot of piece q and its ring phase (q / D) & 1
    int prev_kind = 0;
    long long pwait = 0;
    for (int P = 0;; ++P) {
      while (ctl->decided <= P) {
        if (ctl->abort) goto drain;
#ifdef SCB_PROD_SLEEP
        __nanosleep(SCB_PROD_SLEEP);
#else
        __nanosleep(32);
#endif
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
        // the two-phase dot pass reads the streamed rows twice (y, then z); wide
        // rows go as column chunks, chunk-major in dot passes, row-major otherwise
        // (the first dot pass of a term carries the fused rank-1 update: always two-phase)
        const bool dotp = (kind & F_DOT) && (p.two_phase || (kind & F_UPD));
        const int reps = (kind & F_DELTA) ? 0 : (dotp ? 2 : 1);  // delta passes stream nothing
        for (int rep = 0; rep < reps; ++rep) {
          if (rep == 1 && (kind & F_UPD)) {  // phase C re-reads rows that phase A rewrote
            while (ctl->upd_done <= P) {
              if (ctl->abort) goto drain;
              __nanosleep(32);
            }
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
          int row = 0, chunk = 0;  // piece cursor: chunk-major in dot passes, row-major otherwise
          for (int idx = 0; idx < npieces; ++idx, ++q) {
            const int s = ps;
            if (q >= static_cast<unsigned>(D)) {
              const uint32_t ph = static_cast<uint32_t>(pph) ^ 1u;
              const long long tw0 = p.prof ? clock64() : 0;
              while (!mbar_try_wait(&ctl->empty[s], ph)) {
                if (ctl->abort) goto drain;
#ifdef SCB_PRODUCER_SLEEP
                __nanosleep(SCB_PRODUCER_SLEEP);  // yield issue slots to the consumer warps on this SMSP
#endif
              }
              if (p.prof) pwait += clock64() - tw0;
            }
            const long long c0 = static_cast<long long>(chunk) * p.chunk_cols;
            const uint32_t bytes = p.cpr == 1 ? static_cast<uint32_t>(rowB)
                                              : static_cast<uint32_t>(min(static_cast<long long>(p.chunk_cols), pitch - c0) * sizeof(E));
            mbar_expect_tx(&ctl->full[s], bytes);
            bulk_g2s(stage_base + static_cast<size_t>(s) * stageB, R + static_cast<size_t>(r0 + nres + row) * pitch + c0,
                     bytes, &ctl->full[s]);
            if (++ps == D) {  // incremental stage / phase (no division on the refill path)
              ps = 0;
              pph ^= 1;
            }
            if (dotp) {
              if (++row == nstream) { row = 0; ++chunk; }
            } else {
              if (++chunk == p.cpr) { chunk = 0; ++row; }
            }
          }
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
#ifdef SCB_PROFILE
  unsigned long long* prof = p.prof;  // clock64 breakdown (build with SCB_PROFILE=1, run with SCB_PROF=1)
#else
  constexpr unsigned long long* prof = nullptr;
#endif
  long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long pten[6] = {0, 0, 0, 0, 0, 0};  // order-k: Z reduction (+ barrier), axial step, Z barrier, axis 1, axis 2, kron
  const unsigned* errp = p.err_pass;
  int qs = 0, qph = 0;     // stage / phase of this pass's first streamed row
  unsigned gcount = 0;     // dot-partial groups published in earlier passes
  unsigned epoch = 0;      // grid barriers passed (thread 0)
  unsigned lepoch = 0;     // rank-local barriers passed (thread 0, world > 1)
  unsigned long long dot_passes[2] = {0, 0};  // CTA 0: dense, delta dot passes (-> stats[2], [3])
  unsigned long long nflip_sum = 0;  // CTA 0, thread 32: t flips over the delta passes (-> stats[7])
  int vidx[VPT];           // owned vectors (clamped to a valid address when out of range)
  bool vok[VPT];
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int v = (k * NW + warp) * 32 + lane;
    vok[k] = v < NV;
    vidx[k] = vok[k] ? v : 0;
  }

  // Owner CTAs sum the G column partials of their 32-column words in a fixed
  // order.  mode 0 (one GPU, matrix): publish sgn(z) as tagged t words; mode 1
  // (order-k): store z itself; mode 2 (row-sharded, world > 1): store the RANK
  // partial zr of the column (this rank's G partials), which the global owners
  // combine after the cross-rank barrier (col_reduce_global).  Mode 1 ends with
  // a grid barrier.
  // tbuf: the tb64 buffer the next pass reads ((pp + 1) & 1); the decision may
  // still stop the restart -- then these words are simply never read (the kept
  // triple's t lives in the other buffer).
  // Warps w0..CW-1 take part (w0 = 1: warp 0 runs the controller decision meanwhile
  // and the participants synchronise on named barrier 2).
  // Matrix delta passes: the owner's dz for column `col` from the flipped rows of the
  // rank's CTAs [gs, ge) (their flip words staged in fws after the barrier), read
  // straight from R (row-major, current in global memory for every row):
  // sum over flipped rows i, ascending, of 2 s'_i R[i, col].  A per-warp shared
  // buffer lists up to kFBuf rows at a time so that 8 row loads are in flight.
  auto flip_rows_sum = [&](int col, int gs, int ge, int lw) -> double {
    uint32_t* buf = fbuf + lw * kFBuf;
    const E* Rc = R + col;
    double acc = 0.0;
    auto drain = [&](int cnt) {
      __syncwarp();
      for (int k = 0; k < cnt; k += 8) {
        E v[8];
        uint32_t e[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          e[u] = (k + u < cnt) ? buf[k + u] : 0u;
          v[u] = (k + u < cnt) ? __ldcg(Rc + static_cast<size_t>(e[u] & 0x7fffffffu) * pitch) : E(0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (k + u < cnt) acc = fma(static_cast<double>(v[u]), (e[u] >> 31) ? -2.0 : 2.0, acc);
      }
      __syncwarp();
    };
    int nb = 0;
    for (int gp = gs; gp < ge; ++gp) {
      const int r0p = gp * p.rows_base + min(gp, p.rows_rem);
      for (int w = 0; w < p.sw; ++w) {
        const unsigned long long fw = fws[gp * p.sw + w];
        const uint32_t f = static_cast<uint32_t>(fw), sn = static_cast<uint32_t>(fw >> 32);
        if (!f) continue;
        const int cnt = __popc(f);
        if (nb + cnt > kFBuf) {
          drain(nb);
          nb = 0;
        }
        if ((f >> lane) & 1u)
          buf[nb + __popc(f & ((1u << lane) - 1u))] =
              static_cast<uint32_t>(r0p + w * 32 + lane) | (((sn >> lane) & 1u) << 31);
        nb += cnt;
      }
    }
    drain(nb);
    return acc;
  };
  auto col_reduce = [&](int mode, int P, bool delta, int tbuf, int w0) {
    const int NP = CW - w0, lw = warp - w0;
    auto psync = [&]() {
      if (w0 == 0)
        consumer_sync(CT);
      else
        asm volatile("bar.sync 2, %0;" ::"r"(NP * 32) : "memory");
    };
    const bool zstate_here = p.delta && mode != 2;  // z state kept by the owners (one GPU; order-k too)
    double zsv[4];  // warp 0: z state of its word slices, parked in zst before the combine
    unsigned long long* tout = p.tb64 + static_cast<size_t>(tbuf) * p.Q * kTbStride;
    const unsigned long long tag = static_cast<unsigned long long>(P + 1) << 32;
    const int gs = (lw * G) / NP, ge = ((lw + 1) * G) / NP;
    // Matrix delta pass: one ascending list of every flipped row of the rank (built
    // once by the participating warps, prefix-scanned), split into NP contiguous
    // slices; when it would not fit in fbuf the warps walk their CTA ranges instead.
    int nlist = -1;
    if (delta && mode != 1) {
      const int items = G * p.sw, lt = lw * 32 + lane, per = (items + NP * 32 - 1) / (NP * 32);
      const int i0 = min(items, lt * per), i1 = min(items, i0 + per);
      int cnt = 0;
      for (int i = i0; i < i1; ++i) cnt += __popc(static_cast<uint32_t>(fws[i]));
      int inc = cnt;  // inclusive warp scan
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
      }
      int* wtot = reinterpret_cast<int*>(zst);  // scratch (z state is staged later)
      if (lane == 31) wtot[lw] = inc;
      psync();
      int base = 0, total = 0;
      for (int w = 0; w < NP; ++w) {
        const int t = wtot[w];
        if (w < lw) base += t;
        total += t;
      }
      if (total <= CW * kFBuf) {
        int pos = base + inc - cnt;
        for (int i = i0; i < i1; ++i) {
          uint32_t f = static_cast<uint32_t>(fws[i]);
          const uint32_t sn = static_cast<uint32_t>(fws[i] >> 32);
          const int gp = i / p.sw, w = i - gp * p.sw;
          const int rb = gp * p.rows_base + min(gp, p.rows_rem) + w * 32;
          while (f) {
            const int b = __ffs(f) - 1;
            f &= f - 1;
            fbuf[pos++] = static_cast<uint32_t>(rb + b) | (((sn >> b) & 1u) << 31);
          }
        }
        nlist = total;
      }
      psync();
    }
    auto list_sum = [&](int col) -> double {  // this warp's slice of the list, in order
      const int k0 = (nlist * lw) / NP, k1 = (nlist * (lw + 1)) / NP;
      const E* Rc = R + col;
      double acc = 0.0;
      for (int k = k0; k < k1; k += 8) {
        E v[8];
        uint32_t e[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          e[u] = (k + u < k1) ? fbuf[k + u] : 0u;
          v[u] = (k + u < k1) ? __ldcg(Rc + static_cast<size_t>(e[u] & 0x7fffffffu) * pitch) : E(0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (k + u < k1) acc = fma(static_cast<double>(v[u]), (e[u] >> 31) ? -2.0 : 2.0, acc);
      }
      return acc;
    };
    for (int q0 = g; q0 < p.Q; q0 += G * p.zl) {
      int nls = 0;
      for (int j = 0; j < p.zl && q0 + j * G < p.Q; ++j) nls = j + 1;
      for (int j = 0; j < nls; ++j) {
        const int col = (q0 + j * G) * 32 + lane;
        const size_t par = static_cast<size_t>(P & 1) * G * pitch + col;  // pass-parity buffer
        if (zstate_here && lw == 0 && col < p.n) zsv[j] = __ldcg(p.zstate + col);  // issued early
        double a = 0.0;
        const double* zb = p.zpart + par;
        if (delta && mode != 1) {  // matrix delta pass: the flipped rows themselves (no partials)
          a = nlist >= 0 ? list_sum(col) : flip_rows_sum(col, gs, ge, lw);
        } else
        for (int g0 = gs; g0 < ge; g0 += 32) {  // one round of up to 32 L2 loads in flight
          double v[32];
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int gp = g0 + u;
            const bool take = gp < ge && (!delta || ((dzmask[gp >> 5] >> (gp & 31)) & 1u));
            v[u] = take ? __ldcg(zb + static_cast<size_t>(gp) * pitch) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 32; ++u) a += v[u];
        }
        zseg[(j * CW + lw) * 32 + lane] = a;
        if (zstate_here && lw == 0) zst[j * 32 + lane] = (col < p.n) ? zsv[j] : 0.0;
      }
      psync();
      for (int j = lw; j < nls; j += NP) {
        const int qq = q0 + j * G;
        const int col = qq * 32 + lane;
        double z = 0.0;
#pragma unroll
        for (int w = 0; w < NP; ++w) z += zseg[(j * CW + w) * 32 + lane];
        const bool valid = col < p.n;
        if (mode == 2) {  // rank partial: combined and checked by the global owners
          if (valid) __stcg(p.zr_own + static_cast<size_t>(P & 1) * pitch + col, z);
          continue;
        }
        if (zstate_here && valid) {  // z state for delta passes: dense sets it, delta adds to it
          const double zs = zst[j * 32 + lane];
          if (ctl->keep && !delta)
            z = zs;  // fixed point: z as cached
          else if (delta)
            z = zs + z;
          __stcg(p.zstate + col, z);
        }
        if (valid && !isfinite(z)) {
          atomicMin(const_cast<unsigned*>(errp) + ERR_Z, static_cast<unsigned>(P));
          ctl->zerr = 1;
        }
        if (mode == 1) {  // order-k: Z = M^T s_0 for the axial step
          if (valid) __stcg(p.zfull + col, z);
        } else {
          const unsigned word = __ballot_sync(0xffffffffu, valid && z < 0.0);
          if (lane == 0) st_relaxed64(tout + static_cast<size_t>(qq) * kTbStride, tag | word);
        }
      }
      psync();
    }
    // Order-k (single GPU): every CTA reads all of Z next, so the reduction ends
    // in a grid barrier.  Matrix mode needs none: the next pass polls the
    // pass-tagged t words, and zpart / slots / tb64 are reused only two passes
    // later, i.e. after the next pass's grid barrier, which every CTA reaches
    // only after finishing this reduction.
    if (mode == 1) {
      const long long tz = prof ? clock64() : 0;
      if (tid == 0) grid_barrier(p.bar, ++epoch * static_cast<unsigned>(G));
      consumer_sync(CT);
      if (prof && tid == 0) pten[2] += clock64() - tz;
    }
  };
  // Row-sharded (world > 1), after the cross-rank barrier: the owner of a 32-column
  // word (by global CTA index over all ranks) adds the world rank partials in rank
  // order (in delta passes only the ranks that had a flipped row), keeps the z state,
  // and publishes sgn(z) to every rank.  One warp per word; no cross-warp combine.
  auto col_reduce_global = [&](int P, bool delta, int tbuf, int w0) {
    const int NP = CW - w0, lw = warp - w0;
    const int GT = p.GT, gg = p.rank * G + g;
    const unsigned long long tag = static_cast<unsigned long long>(P + 1) << 32;
    const unsigned rdz = ctl->rank_dz;
    int k = 0;
    for (int qq = gg; qq < p.Q; qq += GT, ++k) {
      if (k % NP != lw) continue;
      const int col = qq * 32 + lane;
      const bool valid = col < p.n;
      const size_t off = static_cast<size_t>(P & 1) * pitch + col;
      const double zs = (p.delta && valid) ? __ldcg(p.zstate + col) : 0.0;
      double v[kMaxVRanks];
#pragma unroll
      for (int r = 0; r < kMaxVRanks; ++r)
        v[r] = (r < p.world && valid && (!delta || ((rdz >> r) & 1u))) ? __ldcg(p.zr_pe[r] + off) : 0.0;
      double z = 0.0;
#pragma unroll
      for (int r = 0; r < kMaxVRanks; ++r) z += v[r];
      if (p.delta && valid) {
        if (ctl->keep && !delta)
          z = zs;
        else if (delta)
          z = zs + z;
        __stcg(p.zstate + col, z);
      }
      if (valid && !isfinite(z)) atomicMin(const_cast<unsigned*>(errp) + ERR_Z, static_cast<unsigned>(P));
      const unsigned word = __ballot_sync(0xffffffffu, valid && z < 0.0);
      // every rank stages t from its own copy (lane r stores rank r's; constant-index
      // selects keep the kernel-parameter tables out of local memory)
      unsigned long long* dst = nullptr;
#pragma unroll
      for (int r = 0; r < kMaxVRanks; ++r)
        if (lane == r) dst = p.tb64_pe[r];
      if (lane < p.world) st_relaxed64_sys(dst + (static_cast<size_t>(tbuf) * p.Q + qq) * kTbStride, tag | word);
    }
  };

  for (int P = 0;; ++P) {
    const int kind = ctl->kind;
    if (kind & K_TERM) break;
    const int pp = ctl->pp;
    long long t_pass0 = prof ? clock64() : 0;
    const uint32_t* s_cur = sb + ctl->cur * p.sw;
    uint32_t* s_nxt = sb + ctl->nxt * p.sw;
    const uint32_t* s_upd = sb + ctl->best * p.sw;
    const double alpha = ctl->alpha;

    // Barrier-free delta pass (one GPU, matrices, whole rows): t staging, y update,
    // signs and the record exchange in one lean function; then the owners' column
    // reduction beside the decision, as after a barrier pass.
    const bool fast = !TS && !MR && (kind & F_DELTA) && p.fast_delta;
    if (fast) {
      fast_delta<E, NW>(static_cast<unsigned>(L.ctl), P, ctl->tsel, ctl->cur | (ctl->nxt << 2));
      if (g == 0 && tid == 32) nflip_sum += static_cast<unsigned>(ctl->nflip);
      if (g == 0 && tid == 0) ++dot_passes[1];
      gcount += static_cast<unsigned>((rows_g + RG - 1) / RG);
      if (prof && tid == 0) {
        const long long t = clock64();
        pacc[1] += t - t_pass0;
        pten[5] += t - t_pass0;
        t_pass0 = t;
      }
    } else {
    // ---- stage the sign words of this pass in shared memory ----
    if (kind & F_DOT) {
      if (ctl->tsel < 0) {
        const uint32_t* tw =
            p.t0 + (static_cast<size_t>(ctl->term) * p.restarts + ctl->restart) * p.t0_stride;
        for (int i = tid; i < p.Q; i += CT) tws[i] = __ldg(tw + i);
        if (TS) {  // drawn start signs of axes 1..k-1 (search.hpp:197)
          const uint32_t* aw = p.ax0 + (static_cast<size_t>(ctl->term) * p.restarts + ctl->restart) * p.axw;
          for (int i = tid; i < p.axw; i += CT) sax[i] = __ldg(aw + i);
        }
      } else if (!TS) {  // order-k: tws was rebuilt by the previous pass's axial step
        // t words were published before the last grid barrier, tagged with this pass
        const unsigned long long* tw = p.tb64 + static_cast<size_t>(ctl->tsel) * p.Q * kTbStride;
        if (MR && p.world > 1) {  // published by owners on every rank: bounded spin
          SpinBound sb{p.abort_word, p.timeout_ns, 0ull, 0u};
          for (int i = tid; i < p.Q; i += CT) {
            unsigned long long x;
            bool ok = true;
            do {
              x = ld_relaxed64_sys(tw + i * kTbStride);
            } while (static_cast<int>(static_cast<unsigned>(x >> 32) - static_cast<unsigned>(P)) < 0 && (ok = sb.ok()));
            if (!ok) {
              ctl->aborted = 1;
              atomicMin(const_cast<unsigned*>(errp) + 3, static_cast<unsigned>(P));
              break;
            }
            tws[i] = static_cast<uint32_t>(x);
          }
        } else {
          for (int i = tid; i < p.Q; i += CT) {
            unsigned long long x;
            do {
              x = ld_relaxed64(tw + i * kTbStride);
            } while (static_cast<int>(static_cast<unsigned>(x >> 32) - static_cast<unsigned>(P)) < 0);
            tws[i] = static_cast<uint32_t>(x);
          }
        }
      }
      {  // t flips since the previous pass (delta passes), counted exactly
        int nf = 0;
        for (int i = tid; i < p.Q; i += CT) {
          const uint32_t x = tws[i] ^ tprev[i];
          txor[i] = x;
          tprev[i] = tws[i];
          nf += __popc(x);
        }
        if (nf) atomicAdd(&ctl->nflip, nf);
        if (tid < 64) dzmask[tid] = 0u;
      }
      if (tid == 0)
        for (int i = 0; i < p.sw; ++i) s_nxt[i] = 0u;
    }
    if ((kind & F_UPD) && (kind & F_DOT) && tid == 0) {  // operands of the fused update (smem)
      ctl->ua.uws = static_cast<unsigned>(L.uws);
      ctl->ua.s_upd = static_cast<unsigned>(reinterpret_cast<const unsigned char*>(s_upd) - smem);
      ctl->ua.alpha = alpha;
      ctl->ua.Rband = R + static_cast<size_t>(r0) * pitch;
      ctl->ua.pitch = pitch;
      ctl->ua.n = p.n;
    }
    if ((kind & F_UPD) && !TS) {  // order-k: uws = kron(best axes), built at term accept
      for (int i = tid; i < p.Q; i += CT)
        uws[i] = ctl->utsel == 2 ? __ldcg(p.tbest + i)
                                 : static_cast<uint32_t>(__ldcg(p.tb64 + (static_cast<size_t>(ctl->utsel) * p.Q + i) * kTbStride));
    }
    consumer_sync(CT);
    if (MR && p.world > 1 && ctl->aborted) break;  // uniform: set before the barrier
    if (g == 0 && tid == 32 && (kind & F_DELTA)) nflip_sum += static_cast<unsigned>(ctl->nflip);
    if (prof && tid == 0) pacc[5] += clock64() - t_pass0;
    // A sweep whose t equals the previous pass's t is a fixed point of the cached
    // products: y, s' and z stay exactly as cached whatever pass form runs, so a
    // dense refresh can never nudge c by rounding there (the reference's caches
    // behave the same way outside their refreshes).
    const bool keep = (kind & F_DOT) && !TS && p.delta && pp >= 1 && ctl->nflip == 0;
    if (keep && !(kind & F_DELTA))
      for (int j = tid; j < rows_g; j += CT) ybak[j] = yrow[j];

    double nacc = 0.0;
    bool bad = false;
    int sslot = qs, sph = qph;  // streamed-row cursor (identical in all consumer threads)

    if (kind & F_DOT) {
      // ======================= dot pass (the hot loop) =======================
      DotArgs da;
      da.res = static_cast<unsigned>(L.res);
      da.stage = static_cast<unsigned>(L.stage);
      da.full = static_cast<unsigned>(reinterpret_cast<unsigned char*>(ctl->full) - smem);
      da.empty = static_cast<unsigned>(reinterpret_cast<unsigned char*>(ctl->empty) - smem);
      da.ring = static_cast<unsigned>(L.ring);
      da.rred = static_cast<unsigned>(L.rred);
      da.yrow = static_cast<unsigned>(L.yrow);
      da.s_nxt = static_cast<unsigned>(reinterpret_cast<unsigned char*>(s_nxt) - smem);
      da.tws = static_cast<unsigned>(L.tws);
      da.zrow = p.zpart + (static_cast<size_t>(P & 1) * G + g) * pitch;
      da.errp = const_cast<unsigned*>(errp);
      da.rowB = static_cast<unsigned>(rowB);
      da.rows_g = rows_g;
      da.nres = nres;
      da.D = D;
      da.NV = NV;
      da.sslot = sslot;
      da.sph = sph;
      da.P = P;
      da.gcount = gcount;
      da.wmul = p.widen_mul;
      da.ypart = static_cast<unsigned>(L.ypart);
      da.prof = prof ? prof + g * 16 + 8 : nullptr;
      da.cpr = p.cpr;
      da.chunk_cols = p.chunk_cols;
      da.upd = (kind & F_UPD) ? 1 : 0;
      da.ctl = static_cast<unsigned>(L.ctl);
      if (kind & F_DELTA) {
        DeltaArgs dl;
        dl.res = static_cast<unsigned>(L.res);
        dl.yrow = static_cast<unsigned>(L.yrow);
        dl.s_cur = static_cast<unsigned>(reinterpret_cast<const unsigned char*>(s_cur) - smem);
        dl.s_nxt = da.s_nxt;
        dl.tws = static_cast<unsigned>(L.tws);
        dl.txor = static_cast<unsigned>(L.txor);
        dl.Rrows = R + static_cast<size_t>(r0) * pitch;
        dl.zrow = da.zrow;
        dl.errp = da.errp;
        dl.has_dz = &ctl->has_dz;
        dl.nfrows = &ctl->nfrows;
        dl.local_dz = TS ? 1 : 0;
        dl.flipw = p.flipw + (static_cast<size_t>(P & 1) * G + g) * p.sw;
        dl.sw_all = p.sw;
#ifdef SCB_PROFILE
        dl.prof = prof ? p.prof + static_cast<size_t>(p.G) * 16 + g * 16 : nullptr;
#endif
        dl.pitch = pitch;
        dl.rowB = static_cast<unsigned>(rowB);
        dl.rows_g = rows_g;
        dl.nres = nres;
        dl.Q = p.Q;
        dl.NV = NV;
        dl.P = P;
        dl.cpr = p.cpr;
        delta_pass<E, NW, VPT>(dl);
      } else if (p.cpr > 1) {
        da.rowB = static_cast<unsigned>(stageB);
        nacc += dot_pass_chunked<E, NW, VPT>(da);
      } else if (p.two_phase || (kind & F_UPD)) {
        nacc += dot_pass_2ph<E, NW, VPT>(da);
      } else {
        dot_pass<E, NW, VPT, RG, CPS>(da);
      }
      if (keep && !(kind & F_DELTA)) {  // fixed point reached through a dense pass: keep the cache
        consumer_sync(CT);
        for (int j = tid; j < rows_g; j += CT) yrow[j] = ybak[j];
        for (int i = tid; i < p.sw; i += CT) s_nxt[i] = s_cur[i];
      }
      if (tid == 0) ctl->keep = keep;
      const int ngroups = (rows_g + RG - 1) / RG;
      gcount += static_cast<unsigned>(ngroups);
    } else {
      // ============ maintenance pass: update / norm / check / write-back ============
      // (rank-1 deflation R -= alpha s t^T of the previous term, flush_pending with
      // one term, decompose.hpp:200-214; ||R||_F^2; final write-back of resident rows).
      // All warps walk the rows in order (each takes a column segment), so the
      // stage ring is consumed in order and its phase parity is unambiguous.
      const int chunkVv = p.cpr > 1 ? p.chunk_cols / EPV : NV;  // vectors per piece
      for (int j = 0; j < rows_g; ++j) {
        const uint32_t sneg = ((s_upd[j >> 5] >> (j & 31)) & 1u) << 31;
        for (int k = 0; k < p.cpr; ++k) {
          VT* rv;
          int slot = -1;
          if (j < nres) {
            rv = reinterpret_cast<VT*>(res_base + static_cast<size_t>(j) * rowB);
          } else {
            slot = sslot;
            mbar_wait(&ctl->full[slot], static_cast<uint32_t>(sph));
            rv = reinterpret_cast<VT*>(stage_base + static_cast<size_t>(slot) * stageB);
            if (++sslot == D) {
              sslot = 0;
              sph ^= 1;
            }
          }
          const int v0 = k * chunkVv;  // first vector of the piece within the row
          const int nvp = min(chunkVv, NV - v0);
          VT* grow = reinterpret_cast<VT*>(R + static_cast<size_t>(r0 + j) * pitch) + v0;
          for (int v = tid; v < nvp; v += CT) {
            const int gv = v0 + v;
            E x[EPV];
            Vec<E>::split(rv[v], x);
            if (kind & F_UPD) {
              const uint32_t ub = (uws[(gv * EPV) >> 5] >> ((gv * EPV) & 31)) & ((1u << EPV) - 1u);
#pragma unroll
              for (int e = 0; e < EPV; ++e)
                if (gv * EPV + e < p.n)  // flush_pending with one term: data += flip(-alpha, s_i ^ t_j)
                  x[e] = Vec<E>::narrow(static_cast<double>(x[e]) + flipd(-alpha, sneg ^ bitmask(ub, e)));
              if (j < nres) rv[v] = Vec<E>::join(x);
            }
            if (kind & (F_UPD | F_WB)) grow[v] = Vec<E>::join(x);  // every row current in global R
#pragma unroll
            for (int e = 0; e < EPV; ++e) {
              const double d = static_cast<double>(x[e]);
              nacc += d * d;
              if (kind & F_CHECK) bad |= !isfinite(d);
            }
          }
          if (slot >= 0) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&ctl->empty[slot]);
          }
        }
      }
    }
    if (D > 0) {  // advance the stage ring past this pass's streamed rows
      const int t = qs + npieces * ((kind & F_DELTA) ? 0 : (((kind & F_DOT) && (p.two_phase || (kind & F_UPD))) ? 2 : 1));
      qph ^= (t / D) & 1;
      qs = t % D;
    }

    // ------------------------------ pass end ------------------------------
    if (prof && tid == 0) {
      const long long t = clock64();
      pacc[1] += t - t_pass0;
      if (!TS && (kind & F_DOT)) pten[(kind & F_DELTA) ? 5 : 4] += t - t_pass0;  // dense / delta split
      t_pass0 = t;
    }
    if (kind & (F_UPD | F_WB)) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __threadfence();
    }
    if (kind & F_NORM) {
      const double ws = warp_sum(nacc);
      if (lane == 0) ctl->nred[warp] = ws;
      if (bad) atomicMin(const_cast<unsigned*>(errp) + ERR_INPUT, static_cast<unsigned>(P));
    }
    consumer_sync(CT);
    if (warp == 0) {
      // this CTA's c partial: sum_i s_i y_i in row order (lane-strided, fixed tree)
      double cl = 0.0;
      if ((kind & F_DOT) && pp >= 1 && !TS)
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
          for (int w = 0; w < CW; ++w) nsum += ctl->nred[w];
        Slot* my = p.slots + g;
        __stcg(&my->c[P & 1], cl);
        __stcg(&my->n[P & 1], nsum);
        __stcg(&my->dz[P & 1], ((kind & F_DELTA) && ctl->has_dz) ? 1.0 : 0.0);
      }
    }
    consumer_sync(CT);
    if (g == 0 && tid == 0 && (kind & F_DOT)) ++dot_passes[(kind & F_DELTA) ? 1 : 0];
    if (prof && tid == 0) {  // pre-barrier part of the pass end
      const long long t = clock64();
      pacc[0] += t - t_pass0;
    }
    if (tid == 0) {
      const long long tb0 = prof ? clock64() : 0;
      if (MR && p.world > 1) {  // rank-local barrier first (the rank partials need this rank's partials)
        if (!grid_barrier_bounded<false>(p.bar_local, ++lepoch * static_cast<unsigned>(G), p.abort_word,
                                         p.timeout_ns)) {
          ctl->aborted = 1;
          atomicMin(const_cast<unsigned*>(errp) + 3, static_cast<unsigned>(P));
        }
      } else {
        grid_barrier(p.bar, ++epoch * static_cast<unsigned>(G));
      }
      if (prof) pacc[6] += clock64() - tb0;  // barrier (incl. waiting for the last CTA)
    }
    consumer_sync(CT);
    if (MR && p.world > 1 && ctl->aborted) break;
    {
      // every CTA reduces the G partials of its rank in the same fixed order
      double cs = 0.0, ns = 0.0;
      for (int i = tid; i < G; i += CT) {
        const Slot* s = p.slots + i;
        cs += __ldcg(&s->c[P & 1]);
        ns += __ldcg(&s->n[P & 1]);
        if ((kind & F_DELTA) && __ldcg(&s->dz[P & 1]) != 0.0) atomicOr(&dzmask[i >> 5], 1u << (i & 31));
      }
      if (!TS && (kind & F_DELTA) && g < p.Q) {  // owners: every CTA's flip words of this pass
        const unsigned long long* src = p.flipw + static_cast<size_t>(P & 1) * G * p.sw;
        for (int i = tid; i < G * p.sw; i += CT) fws[i] = __ldcg(src + i);
      }
      cs = warp_sum(cs);
      ns = warp_sum(ns);
      if (tid == 32) {  // error flags for the decision, off thread 0's serial path
        ctl->err_pre[0] = __ldcg(errp + ERR_Y);
        ctl->err_pre[1] = __ldcg(errp + ERR_INPUT);
        ctl->err_pre[2] = __ldcg(errp + ERR_Z);
      }
      consumer_sync(CT);  // thread 0 is done reading ctl->nred of the norm step
      if (lane == 0) {
        ctl->cred[warp] = cs;
        ctl->nred[warp] = ns;
      }
    }
    consumer_sync(CT);
    }  // !fast
    if (MR && p.world > 1) {
      // Rank stage: this rank's column partials -> one rank partial zr (local
      // owners), its slots -> one rank slot; then the cross-rank barrier, after
      // which every CTA of every rank combines the world rank slots in rank order.
      if (!TS && (kind & F_DOT)) col_reduce(2, P, (kind & F_DELTA) != 0, 0, 0);
      if (tid == 0) {
        double cs = 0.0, ns = 0.0;
        for (int w = 0; w < CW; ++w) {
          cs += ctl->cred[w];
          ns += ctl->nred[w];
        }
        unsigned anydz = 0;
        if (TS)
          for (int i = 0; i < 64; ++i) anydz |= dzmask[i];
        else if (kind & F_DELTA)  // g == 0 is an owner: its fws holds the rank's flip words
          for (int i = 0; i < G * p.sw; ++i) anydz |= static_cast<unsigned>(fws[i] != 0ull);
        if (g == 0) {
          Slot* rs = p.rslot_own;
          __stcg(&rs->c[P & 1], cs);
          __stcg(&rs->n[P & 1], ns);
          __stcg(&rs->dz[P & 1], ((kind & F_DELTA) && anydz) ? 1.0 : 0.0);
        }
      }
      consumer_sync(CT);
      if (tid == 0) {
        if (!grid_barrier_bounded<true>(p.bar, ++epoch * static_cast<unsigned>(p.GT), p.abort_word,
                                        p.timeout_ns)) {
          ctl->aborted = 1;
          atomicMin(const_cast<unsigned*>(errp) + 3, static_cast<unsigned>(P));
        }
      }
      consumer_sync(CT);
      if (ctl->aborted) break;
      if (warp == 0) {
        double c = 0.0, n2 = 0.0, dz = 0.0;
        const Slot* rs = nullptr;
#pragma unroll
        for (int r = 0; r < kMaxVRanks; ++r)
          if (lane == r) rs = p.rslot_pe[r];
        if (lane < p.world) {
          c = __ldcg(&rs->c[P & 1]);
          n2 = __ldcg(&rs->n[P & 1]);
          dz = __ldcg(&rs->dz[P & 1]);
        }
        const unsigned rdz = __ballot_sync(0xffffffffu, dz != 0.0);
        double cs = 0.0, ns = 0.0;  // rank order
        for (int r = 0; r < p.world; ++r) {
          cs += __shfl_sync(0xffffffffu, c, r);
          ns += __shfl_sync(0xffffffffu, n2, r);
        }
        if (lane == 0) {
          ctl->rank_dz = rdz;
          ctl->cred[0] = cs;
          ctl->nred[0] = ns;
          for (int w = 1; w < CW; ++w) {
            ctl->cred[w] = 0.0;
            ctl->nred[w] = 0.0;
          }
          ctl->err_pre[0] = __ldcg(errp + ERR_Y);  // rank 0's words: every rank's errors so far
          ctl->err_pre[1] = __ldcg(errp + ERR_INPUT);
          ctl->err_pre[2] = __ldcg(errp + ERR_Z);
        }
      }
      consumer_sync(CT);
    }
    if (prof && tid == 0) {
      const long long t = clock64();
      pacc[2] += t - t_pass0;
      t_pass0 = t;
    }
    if (TS && (kind & F_DOT)) {  // order-k: Z = M^T s_0, then axes 1..k-1 and c
      const long long ta = prof ? clock64() : 0;
      col_reduce(1, P, (kind & F_DELTA) != 0, 0, 0);
      const long long tb = prof ? clock64() : 0;
      axial_step<CW>(p, sax, tws, tprev, ctl, P, prof ? pten + 3 : nullptr);
      if (prof && tid == 0) {
        pten[0] += tb - ta;
        pten[1] += clock64() - tb;
      }
    }

    // Matrix dot pass: owners reduce z and publish the next t right away (it does
    // not depend on the decision), taking the decision off every CTA's critical path.
    if (!TS && (kind & F_DOT) && warp >= 1 && (!fast || (ctl->fc.shared_list && ctl->fc.nls > 0))) {  // warp 0: the decision
      const long long tc0 = (prof && tid == 32) ? clock64() : 0;
      if (MR && p.world > 1)
        col_reduce_global(P, (kind & F_DELTA) != 0, (pp + 1) & 1, 1);
      else
        col_reduce(0, P, (kind & F_DELTA) != 0, (pp + 1) & 1, 1);
      if (prof && tid == 32 && (kind & F_DELTA)) ctl->fprof[6] += clock64() - tc0;
    }
    const long long td0 = (prof && tid == 0) ? clock64() : 0;

    // ------------------------------ decision ------------------------------
    if (tid == 0) {
      // restart loop done: accept or reject the best restart's term (decompose.hpp:329-343)
      auto accept_term = [&]() -> int {
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
          if (g == 0 && TS) {  // axes 1..k-1 of the accepted term
            for (int i = 0; i < p.axw; ++i) p.AX_out[static_cast<size_t>(term) * p.axw + i] = sax_best[i];
          }
          if (g == 0) {
            uint32_t* trow = p.T_out + static_cast<size_t>(term) * p.t_stride;
            const int nw = min(p.t_stride, p.Q);  // words past Q are pad (zero)
            if (TS) {
              for (int i = 0; i < nw; ++i) trow[i] = 0u;  // order-k: per-axis words are in AX_out
            } else if (ctl->best_tsel == 2) {
              for (int i = 0; i < nw; ++i) trow[i] = __ldcg(p.tbest + i);
            } else {
              const unsigned long long* src = p.tb64 + static_cast<size_t>(ctl->best_tsel) * p.Q * kTbStride;
              for (int i = 0; i < nw; ++i) trow[i] = static_cast<uint32_t>(__ldcg(src + i * kTbStride));
            }
            for (int i = nw; i < p.t_stride; ++i) trow[i] = 0u;
            p.c_out[term] = bc;
            p.sweeps_out[term] = static_cast<uint32_t>(ctl->best_sweeps);
            p.stats[0] = static_cast<unsigned long long>(term + 1);
            if (term == 0) p.stats[4] = static_cast<unsigned long long>(ctl->best_restart);
          }
          ctl->alpha = bc / p.numel_d;  // alpha = c / numel (decompose.hpp:340)
          ctl->utsel = ctl->best_tsel;
          ctl->kron_upd = TS;  // order-k: uws = kron(best axes) after the decision
          ctl->term = static_cast<int>(term + 1);
          ctl->norm_idx = static_cast<int>(term + 1);
          if (term + 1 >= p.width) {
            return F_UPD | F_NORM | F_WB;
          } else {
            ctl->pp = TS ? 1 : 0;
            ctl->restart = 0;
            ctl->tsel = -1;
            ctl->c_prev = -INFINITY;
            // the next term's first dot pass deflates R by this term as it streams it
            // (north-star kernel 3): sweeps + 1 passes per cut, no maintenance pass
#ifdef SCB_NO_FUSE
            return F_UPD | F_NORM;
#else
            return p.fuse_update ? (F_DOT | F_UPD | F_NORM) : (F_UPD | F_NORM);
#endif
          }
        } else {
          // min_value_fraction stop (decompose.hpp:337-338): nothing appended
          ctl->norm_idx = static_cast<int>(term);
          return F_NORM | F_WB;
        }
      };
      // (only the first ceil(G / 32) butterflies hold CTAs; the others added zeros)
      double cs = 0.0, ns = 0.0;
      const int nwz = min(CW, (G + 31) >> 5);
      for (int w = 0; w < nwz; ++w) cs += ctl->cred[w];
      if (kind & F_NORM)
        for (int w = 0; w < nwz; ++w) ns += ctl->nred[w];
      int next;
      int need_reduce = 0;
      const unsigned ey = ctl->err_pre[0], ei = ctl->err_pre[1], ez = ctl->err_pre[2];
      if (ey <= static_cast<unsigned>(P) || ei <= static_cast<unsigned>(P) ||
          ez < static_cast<unsigned>(P)) {
        next = K_TERM;
      } else {
        if ((kind & F_NORM) && g == 0) p.norm2_out[ctl->norm_idx] = ns;
        if (kind & F_WB) {
          next = K_TERM;  // final write-back done
        } else if (!(kind & F_DOT)) {
          next = F_DOT;   // maintenance pass (initial norm / rank-1 update) -> search
        } else if (!TS && pp == 0) {
          const int t = ctl->cur;  // s_1 (just computed) becomes current
          ctl->cur = ctl->nxt;
          ctl->nxt = t;
          ctl->pp = 1;
          ctl->tsel = 1;
          need_reduce = 1;
          next = F_DOT;
          ctl->since_dense = 0;
        } else {
          // matrix: c = <s_pp, R t_pp> from this pass's y; order-k: c of this sweep's axial step
          const double c = TS ? ctl->ax_c : cs;
          // SearchDiagnostics::sweep_values of term 0 (search.hpp:177, :207), per restart
          if (p.sweep_vals != nullptr && ctl->term == 0 && g == 0)
            p.sweep_vals[static_cast<size_t>(ctl->restart) * p.max_sweeps + (pp - 1)] = c;
          const bool stop = (c <= ctl->c_prev) || (pp >= p.max_sweeps);
          if (!stop) {
            ctl->c_prev = c;
            ctl->pp = pp + 1;
            next = F_DOT;
            if (TS) {
              next = tensor_continue(ctl, p.delta, p.delta_refresh, p.delta_div, p.n);
            } else {
              const int t = ctl->cur;
              ctl->cur = ctl->nxt;
              ctl->nxt = t;
              ctl->tsel = (pp + 1) & 1;
              need_reduce = 1;
              // delta pass next unless it is time to refresh the caches (every 64th
              // sweep; the reference refreshes every 16th) or many columns flipped last time
              if (p.delta && ctl->since_dense + 1 < p.delta_refresh &&
                  static_cast<long long>(ctl->nflip) * p.delta_div <= p.n) {
                next |= F_DELTA;
                ctl->since_dense += 1;
              } else {
                ctl->since_dense = 0;
              }
            }
          } else if (TS) {
            // axial_run returns the current sweep's (c, signs) (search.hpp:206, :210)
            const bool better = (ctl->restart == 0) || (c > ctl->best_c);
            if (better) {
              ctl->best_c = c;
              ctl->best_sweeps = pp;
              ctl->best_restart = ctl->restart;
              uint32_t* sbest = sb + ctl->best * p.sw;
              for (int i = 0; i < p.sw; ++i) sbest[i] = s_nxt[i];
              for (int i = 0; i < p.axw; ++i) sax_best[i] = sax[i];
            }
            ctl->restart += 1;
            if (ctl->restart < p.restarts) {
              ctl->pp = 1;
              ctl->tsel = -1;
              ctl->c_prev = -INFINITY;
              next = F_DOT;
            } else {
              next = accept_term();
            }
          } else {
            // restart result (c, s_pp, t_pp, pp): search.hpp:178-180 / :185
            const bool better = (ctl->restart == 0) || (c > ctl->best_c);
            if (better) {
              ctl->best_c = c;
              ctl->best_sweeps = pp;
              ctl->best_restart = ctl->restart;
              uint32_t* sbest = sb + ctl->best * p.sw;
              for (int i = 0; i < p.sw; ++i) sbest[i] = s_cur[i];
              if (ctl->restart + 1 < p.restarts) {
                if (g == 0) {
                  const unsigned long long* src = p.tb64 + static_cast<size_t>(pp & 1) * p.Q * kTbStride;
                  for (int i = 0; i < p.Q; ++i) p.tbest[i] = static_cast<uint32_t>(__ldcg(src + i * kTbStride));
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
              next = accept_term();
            }
          }
        }
      }
      ctl->kind = next;
      ctl->need_reduce = need_reduce;
      ctl->nflip = 0;  // recounted at the next staging
      ctl->kind_ring[(P + 1) & 3] = next;
      __threadfence_block();
      ctl->decided = P + 2;
      if ((next & K_TERM) && g == 0) p.stats[1] = static_cast<unsigned long long>(P + 1);
      if (prof && (kind & F_DELTA)) ctl->fprof[7] += clock64() - td0;
    }
    consumer_sync(CT);
    if (prof && tid == 0) {
      const long long t = clock64();
      pacc[3] += t - t_pass0;
      t_pass0 = t;
    }
    if (TS && ctl->kron_upd) {  // order-k: t of the rank-1 update = kron(best axes)
      for (int q = tid; q < p.Q; q += CT) uws[q] = kron_word(p, ctl, sax_best, q);
      consumer_sync(CT);
      if (tid == 0) ctl->kron_upd = 0;
    }

    // --------------------- column reduction: t' = sgn(z) ---------------------
    if (prof && tid == 0) pacc[4] += clock64() - t_pass0;
  }
  if (tid == 0) {
    ctl->abort = 1;  // release a producer still waiting on an unconsumed stage
    // traffic counters (the host turns them into bytes, sc_result::device_bytes)
    atomicAdd(p.stats + 5, static_cast<unsigned long long>(ctl->nfrows));
    atomicAdd(p.stats + 6, static_cast<unsigned long long>(ctl->ndz));
  }
  if (g == 0 && tid == 32) p.stats[7] = nflip_sum;
  if (g == 0 && tid == 0) {
    p.stats[2] = dot_passes[0];
    p.stats[3] = dot_passes[1];
  }
  if (prof && tid == 0) {
    for (int k = 0; k < 16; ++k)  // fast-delta / decision sections (shared-memory accumulators)
      if (ctl->fprof[k]) prof[static_cast<size_t>(p.G) * 16 + g * 16 + k] = static_cast<unsigned long long>(ctl->fprof[k]);
    for (int i = 0; i < 7; ++i) prof[g * 16 + i] = static_cast<unsigned long long>(pacc[i]);
    prof[g * 16 + 12] = static_cast<unsigned long long>(pten[0]);
    prof[g * 16 + 13] = static_cast<unsigned long long>(pten[1]);
    prof[g * 16 + 14] = static_cast<unsigned long long>(pten[2]);
    prof[g * 16 + 15] = static_cast<unsigned long long>(pten[3]);
    prof[g * 16 + 8] = static_cast<unsigned long long>(pten[4]);
    prof[g * 16 + 9] = static_cast<unsigned long long>(pten[5]);
  }
}

// TS: order-k (tensor) instantiation.  Matrix kernels carry no order-k code at all,
// which keeps their per-pass serial sections compact.
template <typename E, int NW, int VPT, int RG, bool TS>
__global__ void __launch_bounds__((NW + 1) * 32, 1) sweep_kernel(const KParams p) {
  sweep_body<E, NW, VPT, RG, 1, TS>(p, blockIdx.x);
}
template <typename E, int NW, int VPT, int RG>
__global__ void __maxnreg__(112) sweep_kernel2(const KParams p) {
  sweep_body<E, NW, VPT, RG, 2, false>(p, blockIdx.x);
}
// Row sharding emulated on one GPU (KParamsVR): CTA block r of the one
// cooperative launch runs rank r's band with rank r's parameters and exchange
// region; the code path is the multi-rank one (rank partials, bounded barriers).
template <typename E, int NW, int VPT, int RG>
__global__ void __launch_bounds__((NW + 1) * 32, 1) sweep_kernel_vr(const __grid_constant__ KParamsVR pv) {
  const int G = pv.r[0].G;
  const int rank = static_cast<int>(blockIdx.x) / G;
  sweep_body<E, NW, VPT, RG, 1, false, true>(pv.r[rank], static_cast<int>(blockIdx.x) - rank * G);
}
// Row-sharded rank on its own GPU (world > 1, peer-mapped exchange regions).
template <typename E, int NW, int VPT, int RG>
__global__ void __launch_bounds__((NW + 1) * 32, 1) sweep_kernel_mr(const KParams p) {
  sweep_body<E, NW, VPT, RG, 1, false, true>(p, blockIdx.x);
}


}  // namespace
}  // namespace scb
