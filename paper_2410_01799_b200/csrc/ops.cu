// ops.cu -- auxiliary sm_100a kernels around the decomposition:
//
//   expand_kernel    accumulate_terms / expand (decompose.hpp:128-197, :266-270):
//                    every output element is a dependent chain of `nterms` f64
//                    additions in term order, so this is FP64-pipe bound, not
//                    HBM bound (4096^2 x 16320 terms = 2.7e11 DFMA vs 128 MiB out).
//   kron_kernel      Kronecker column sign bits of order-k / channel layouts.
//   gram_kernel      XOR-popcount Gram block (gram_column, decompose.hpp:367-381).
//   contract_kernel  <sign outer product, A> for a batch of terms (contract_term,
//                    decompose.hpp:218-260); one streaming pass over A per batch.
//   sqnorm_kernel    ||x||^2 in a fixed order.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "ops.h"

namespace scb {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// expansion
// ---------------------------------------------------------------------------
constexpr int XK = 32;  // terms per chunk (one u32 of column bits)
// Tile shapes (template): XR rows per CTA tile (f64 accumulators per column per
// thread), XW warps per CTA (a warp owns 64 columns: lane, lane + 32), MINB CTAs/SM.

// 32x32 bit transpose across a warp: lane c returns the word whose bit L is bit c
// of lane L's input (five butterfly rounds).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int j = 16 >> r;
    const uint32_t m = masks[r];
    const uint32_t y = __shfl_xor_sync(kFull, x, j);
    x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y & m) << j));
  }
  return x;
}

// +-1.0 from bit b of `bits` (set = -1): a DFMA with it is an exact sign flip.
__device__ __forceinline__ double pm1(uint32_t bits, int b) {
  return __hiloint2double(static_cast<int>(0x3FF00000u | ((bits << (31 - b)) & 0x80000000u)), 0);
}

// flip_sign_if (kernels.hpp:18-20): XOR of the f64 sign bit.
__device__ __forceinline__ double flipd(double x, uint32_t bit) {
  return __hiloint2double(__double2hiint(x) ^ static_cast<int>(bit << 31), __double2loint(x));
}

// One thread: 2 columns (q0 = warp base + lane, q1 = q0 + 32) x XR rows, 2 XR f64
// chains.  Per chunk of XK terms the CTA stages rho[r][b] (the row factor) in
// shared memory; each thread forms kappa (the column factor) from the column bits
// of its two columns, transposed in registers from the term-major V rows.  One of
// rho / kappa is +-1, so fma(kappa, rho, acc) == acc + flip(scale * coef, parity)
// exactly: mode A (COLCH = false) rho = flip(scale coef, u), kappa = +-1 (column
// bit); mode B (COLCH, per-column channel coefficient) rho = +-1 (row bit),
// kappa = flip(scale coef[ch(q)], v).
template <bool COLCH, int XR, int XW, int MINB>
__global__ void __launch_bounds__(XW * 32, MINB) expand_kernel(ExpandParams p) {
  __shared__ __align__(16) double rho[2][XR][XK];
  __shared__ double cc[2][XK][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long qw = (static_cast<long long>(blockIdx.x) * XW + warp) * 64;
  const long long q0 = qw + lane, q1 = q0 + 32;
  const int nchunks = static_cast<int>((p.nterms + XK - 1) / XK);
  int ch0 = 0, ch1 = 0;
  if (COLCH) {
    ch0 = static_cast<int>((q0 / p.cstride) % p.nch);
    ch1 = static_cast<int>((q1 / p.cstride) % p.nch);
  }
  const long long vwi = qw >> 5;  // first u32 word of this warp's 64 columns

  for (long long p0 = static_cast<long long>(blockIdx.y) * XR; p0 < p.P; p0 += static_cast<long long>(gridDim.y) * XR) {
    auto fill = [&](int c, int buf) {
      for (int e = tid; e < XR * XK; e += XW * 32) {
        const int r = e / XK, b = e % XK;
        const long long j = static_cast<long long>(c) * XK + b;
        const long long pp = p0 + r;
        double v = 0.0;
        if (j < p.nterms && pp < p.P) {
          const uint32_t ub = p.U ? (p.U[j * p.u_stride + (pp >> 5)] >> (pp & 31)) & 1u : 0u;
          if (COLCH) {
            v = ub ? -1.0 : 1.0;
          } else {
            const double cf = p.scale * p.coef[j * p.nch + (p.chan == 1 ? pp : 0)];
            v = flipd(cf, ub);
          }
        }
        rho[buf][r][b] = v;
      }
      if (COLCH && p.nch <= 8) {  // more channels: coefficients read directly (ccoef below)
        for (int e = tid; e < XK * p.nch; e += XW * 32) {
          const int b = e / p.nch, ch = e % p.nch;
          const long long j = static_cast<long long>(c) * XK + b;
          cc[buf][b][ch] = j < p.nterms ? p.scale * p.coef[j * p.nch + ch] : 0.0;
        }
      }
    };
    // lane L fetches the two column words of term (chunk c, L)
    auto load_v = [&](int c, uint32_t& w0, uint32_t& w1) {
      const long long j = static_cast<long long>(c) * XK + lane;
      w0 = w1 = 0u;
      if (p.V != nullptr && j < p.nterms) {
        const uint32_t* row = p.V + j * p.v_stride;
        if (vwi < p.v_words) w0 = __ldg(row + vwi);
        if (vwi + 1 < p.v_words) w1 = __ldg(row + vwi + 1);
      }
    };

    // scale * coef of (term b of chunk c, channel ch): staged for <= 8 channels, else global
    auto ccoef = [&](int c, int buf, int b, int ch) -> double {
      if (p.nch <= 8) return cc[buf][b][ch];
      const long long j = static_cast<long long>(c) * XK + b;
      return j < p.nterms ? p.scale * __ldg(p.coef + j * p.nch + ch) : 0.0;
    };
    double acc[XR][2];
#pragma unroll
    for (int r = 0; r < XR; ++r) acc[r][0] = acc[r][1] = 0.0;
    uint32_t nw0, nw1;
    load_v(0, nw0, nw1);
    fill(0, 0);
    __syncthreads();
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c & 1;
      const uint32_t v0 = warp_transpose32(nw0, lane);  // bit b = column q0's sign of term c*XK + b
      const uint32_t v1 = warp_transpose32(nw1, lane);
      if (c + 1 < nchunks) {
        load_v(c + 1, nw0, nw1);
        fill(c + 1, buf ^ 1);
      }
      const long long left = p.nterms - static_cast<long long>(c) * XK;
      if (left >= XK) {
#pragma unroll
        for (int b = 0; b < XK; b += 2) {
          double k00, k01, k10, k11;
          if (COLCH) {
            k00 = flipd(ccoef(c, buf, b, ch0), (v0 >> b) & 1u);
            k01 = flipd(ccoef(c, buf, b + 1, ch0), (v0 >> (b + 1)) & 1u);
            k10 = flipd(ccoef(c, buf, b, ch1), (v1 >> b) & 1u);
            k11 = flipd(ccoef(c, buf, b + 1, ch1), (v1 >> (b + 1)) & 1u);
          } else {
            k00 = pm1(v0, b);
            k01 = pm1(v0, b + 1);
            k10 = pm1(v1, b);
            k11 = pm1(v1, b + 1);
          }
#pragma unroll
          for (int r = 0; r < XR; ++r) {
            const double2 x = *reinterpret_cast<const double2*>(&rho[buf][r][b]);
            acc[r][0] = fma(k00, x.x, acc[r][0]);
            acc[r][1] = fma(k10, x.x, acc[r][1]);
            acc[r][0] = fma(k01, x.y, acc[r][0]);
            acc[r][1] = fma(k11, x.y, acc[r][1]);
          }
        }
      } else {
        for (int b = 0; b < static_cast<int>(left); ++b) {
          double k0, k1;
          if (COLCH) {
            k0 = flipd(ccoef(c, buf, b, ch0), (v0 >> b) & 1u);
            k1 = flipd(ccoef(c, buf, b, ch1), (v1 >> b) & 1u);
          } else {
            k0 = pm1(v0, b);
            k1 = pm1(v1, b);
          }
#pragma unroll
          for (int r = 0; r < XR; ++r) {
            const double x = rho[buf][r][b];
            acc[r][0] = fma(k0, x, acc[r][0]);
            acc[r][1] = fma(k1, x, acc[r][1]);
          }
        }
      }
      __syncthreads();
    }
    // data[e] += acc (decompose.hpp:158)
#pragma unroll
    for (int r = 0; r < XR; ++r) {
      const long long pp = p0 + r;
      if (pp < p.P) {
        double* row = p.data + pp * p.Q;
        if (q0 < p.Q) row[q0] = __dadd_rn(row[q0], acc[r][0]);
        if (q1 < p.Q) row[q1] = __dadd_rn(row[q1], acc[r][1]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Kronecker column bits
// ---------------------------------------------------------------------------
__global__ void kron_kernel(KronParams p) {
  const long long vw = (p.Q + 31) / 32;
  const long long total = p.nterms * vw;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long j = i / vw, w = i % vw;
    uint32_t word = 0;
    for (int b = 0; b < 32; ++b) {
      const long long q = w * 32 + b;
      if (q >= p.Q) break;
      uint32_t par = 0;
      for (int a = 0; a < p.nax; ++a) {
        const long long idx = (q / p.ax_stride[a]) % p.ax_n[a];
        par ^= static_cast<uint32_t>((p.fac[a][j * p.fac_words[a] + (idx >> 6)] >> (idx & 63)) & 1u);
      }
      word |= par << b;
    }
    p.V[j * p.v_stride + w] = word;
  }
}

// ---------------------------------------------------------------------------
// Gram block: 32 x 32 pairs per CTA (one warp row of i per thread-row)
// ---------------------------------------------------------------------------
constexpr int GT = 32;
constexpr int GKW = 32;  // u32 words per smem chunk

__global__ void __launch_bounds__(256) gram_kernel(GramParams p) {
  __shared__ uint32_t si[GT][GKW + 1];
  __shared__ uint32_t sj[GT][GKW + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of warps, 4 i per thread
  const long long i0 = static_cast<long long>(blockIdx.y) * GT, j0 = static_cast<long long>(blockIdx.x) * GT;
  double g[4] = {1.0, 1.0, 1.0, 1.0};
  for (int a = 0; a < p.nax; ++a) {
    int pc[4] = {0, 0, 0, 0};
    for (long long k0 = 0; k0 < p.fw[a]; k0 += GKW) {
      for (int e = threadIdx.x; e < GT * GKW; e += 256) {
        const int r = e / GKW, k = e % GKW;
        const long long kk = k0 + k;
        si[r][k] = (i0 + r < p.rows && kk < p.fw[a]) ? p.Fi[a][(i0 + r) * p.fw[a] + kk] : 0u;
        sj[r][k] = (j0 + r < p.cols && kk < p.fw[a]) ? p.Fj[a][(j0 + r) * p.fw[a] + kk] : 0u;
      }
      __syncthreads();
#pragma unroll 8
      for (int k = 0; k < GKW; ++k) {
        const uint32_t wj = sj[tx][k];
#pragma unroll
        for (int u = 0; u < 4; ++u) pc[u] += __popc(si[ty * 4 + u][k] ^ wj);
      }
      __syncthreads();
    }
    // sign_dot = n - 2 popcount(a ^ b); g *= dot in axis order (gram_column :371-374)
#pragma unroll
    for (int u = 0; u < 4; ++u) g[u] *= static_cast<double>(p.n[a] - 2LL * pc[u]);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const long long i = i0 + ty * 4 + u, j = j0 + tx;
    if (i < p.rows && j < p.cols) p.G[i * p.ldg + j] = g[u];
  }
}

// ---------------------------------------------------------------------------
// signed contraction of A against up to kContractTerms sign outer products
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

template <bool F32, int T, int NC>
__global__ void __launch_bounds__(256) contract_kernel(ContractParams p) {
  __shared__ double wred[8][T * NC];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nout = static_cast<int>(p.nterms) * NC;
  double cta = 0.0;  // CTA partial of output `tid` (tid < nout)
  for (long long r = blockIdx.x; r < p.P; r += gridDim.x) {
    double acc[T * NC];
#pragma unroll
    for (int i = 0; i < T * NC; ++i) acc[i] = 0.0;
    for (long long q = tid; q < p.Q; q += 256) {
      const double a = F32 ? static_cast<double>(static_cast<const float*>(p.A)[r * p.Q + q])
                           : static_cast<const double*>(p.A)[r * p.Q + q];
      const int ch = NC == 1 ? 0 : (p.chan == 2 ? static_cast<int>((q / p.cstride) % p.nch) : static_cast<int>(r));
#pragma unroll
      for (int j = 0; j < T; ++j) {
        if (j < p.nterms) {
          const uint32_t vb = p.V ? (__ldg(p.V + j * p.v_stride + (q >> 5)) >> (q & 31)) & 1u : 0u;
          const double x = flipd(a, vb);
#pragma unroll
          for (int c = 0; c < NC; ++c)
            if (c == ch) acc[j * NC + c] += x;
        }
      }
    }
    // fixed-order reduction: warp butterfly, then the 8 warps in order
#pragma unroll
    for (int i = 0; i < T * NC; ++i) {
      const double v = warp_sum(acc[i]);
      if (lane == 0) wred[warp][i] = v;
    }
    __syncthreads();
    if (tid < nout) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += wred[w][tid];
      const int j = tid / NC;
      const uint32_t ub = p.U ? (p.U[j * p.u_stride + (r >> 5)] >> (r & 31)) & 1u : 0u;
      cta += flipd(s, ub);
    }
    __syncthreads();
  }
  if (tid < nout) p.part[static_cast<long long>(blockIdx.x) * nout + tid] = cta;
}

__global__ void contract_finish(ContractParams p, int grid) {
  const int nout = static_cast<int>(p.nterms) * (p.chan == 0 ? 1 : 8);
  const int t = threadIdx.x;
  if (t < nout) {
    double s = 0.0;
    for (int g = 0; g < grid; ++g) s += p.part[static_cast<long long>(g) * nout + t];
    p.out[t] = s;
  }
}

// ---------------------------------------------------------------------------
// sum of squares
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) sqnorm_kernel(const double* x, long long n, double* part) {
  __shared__ double wred[8];
  double acc = 0.0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += static_cast<long long>(gridDim.x) * 256)
    acc = fma(x[i], x[i], acc);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) wred[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += wred[w];
    part[blockIdx.x] = s;
  }
}

__global__ void sqnorm_finish(const double* part, int grid, double* out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int g = 0; g < grid; ++g) s += part[g];
    *out = s;
  }
}

__global__ void widen_kernel(const float* src, double* dst, long long n) {
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += static_cast<long long>(gridDim.x) * 256)
    dst[i] = static_cast<double>(src[i]);
}

}  // namespace

cudaError_t launch_widen(const float* src, double* dst, long long n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<long long>((n + 255) / 256, 148 * 8));
  widen_kernel<<<grid, 256, 0, st>>>(src, dst, n);
  return cudaGetLastError();
}

template <int XR, int XW, int MINB>
cudaError_t launch_expand_t(const ExpandParams& p, cudaStream_t st) {
  const long long gx = (p.Q + XW * 64 - 1) / (XW * 64);
  const long long gy = std::min<long long>((p.P + XR - 1) / XR, 65535);
  if (gx > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
  if (p.chan == 2)
    expand_kernel<true, XR, XW, MINB><<<grid, XW * 32, 0, st>>>(p);
  else
    expand_kernel<false, XR, XW, MINB><<<grid, XW * 32, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_expand(const ExpandParams& p, cudaStream_t st) {
  if (p.P <= 0 || p.Q <= 0 || p.nterms <= 0) return cudaSuccess;
  return launch_expand_t<16, 8, 2>(p, st);
}

cudaError_t launch_kron(const KronParams& p, cudaStream_t st) {
  const long long total = p.nterms * ((p.Q + 31) / 32);
  if (total <= 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 16));
  kron_kernel<<<grid, 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_gram(const GramParams& p, cudaStream_t st) {
  if (p.rows <= 0 || p.cols <= 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>((p.cols + GT - 1) / GT), static_cast<unsigned>((p.rows + GT - 1) / GT));
  if (grid.y > 65535) return cudaErrorInvalidConfiguration;
  gram_kernel<<<grid, 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_contract(const ContractParams& p, cudaStream_t st) {
  if (p.nterms <= 0) return cudaSuccess;
  // one coefficient per term: up to kContractTerms terms per pass over A; channel
  // slices (<= 8): one term per pass, outputs [ch] padded to 8
  if (p.chan == 0 ? p.nterms > kContractTerms : (p.nterms > 1 || p.nch > 8)) return cudaErrorInvalidValue;
  const int grid = static_cast<int>(std::min<long long>(p.P, kContractCtas));
  if (p.chan == 0) {
    if (p.a_f32)
      contract_kernel<true, kContractTerms, 1><<<grid, 256, 0, st>>>(p);
    else
      contract_kernel<false, kContractTerms, 1><<<grid, 256, 0, st>>>(p);
  } else {
    if (p.a_f32)
      contract_kernel<true, 1, 8><<<grid, 256, 0, st>>>(p);
    else
      contract_kernel<false, 1, 8><<<grid, 256, 0, st>>>(p);
  }
  contract_finish<<<1, 64, 0, st>>>(p, grid);
  return cudaGetLastError();
}

cudaError_t launch_sqnorm(const double* x, long long n, double* part, double* out, cudaStream_t st) {
  const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 592)));
  sqnorm_kernel<<<grid, 256, 0, st>>>(x, n, part);
  sqnorm_finish<<<1, 32, 0, st>>>(part, grid, out);
  return cudaGetLastError();
}

}  // namespace scb
