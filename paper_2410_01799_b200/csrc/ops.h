// ops.h -- launch parameters of the auxiliary kernels (ops.cu) behind the C ABI
// in ops.cpp: expansion / accumulation of sign terms, Kronecker column bits,
// the XOR-popcount Gram system and signed contractions.  No torch types.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace scb {

// data[p][q] += sum_{j < nterms} flip(scale * coef[j][ch], u_j(p) ^ v_j(q)), the
// terms summed one after another in f64 starting from 0.0 and the sum added to
// data last -- the arithmetic of accumulate_terms (decompose.hpp:128-180), so the
// result is bit-identical to the reference.  The tensor is viewed as P x Q
// (rows = axis 0, columns = the trailing axes; order 1: P = 1).  All term-indexed
// pointers start at the first term to add.
struct ExpandParams {
  double* data;            // P x Q row-major f64, in/out
  long long P, Q;
  const uint32_t* U;       // [nterms][u_stride] row sign bits (nullptr: no row sign axis)
  long long u_stride;
  const uint32_t* V;       // [nterms][v_stride] column sign bits (nullptr: none)
  long long v_stride;
  long long v_words;       // valid u32 words per term row of V (ceil(Q / 32))
  const double* coef;      // [nterms][nch]
  int nch;
  int chan;                // 0: one coefficient per term; 1: channel = row p; 2: channel = (q / cstride) % nch
  long long cstride;
  long long nterms;
  double scale;
};
cudaError_t launch_expand(const ExpandParams& p, cudaStream_t st);

// V[j][w] bit b = XOR over the trailing sign axes a of factor_a[j] at the
// axis-a index of column q = 32 w + b (row-major multi-index of the trailing
// axes, channel axis included in the strides but carrying no sign).
struct KronParams {
  uint32_t* V;
  long long v_stride;      // u32 words per term row
  long long Q;
  long long nterms;
  int nax;                 // sign axes among the trailing axes
  long long ax_n[7], ax_stride[7];
  const uint64_t* fac[7];  // [nterms][fac_words] per sign axis
  long long fac_words[7];
};
cudaError_t launch_kron(const KronParams& p, cudaStream_t st);

// Gram column block: G[i][j] = prod_a (n_a - 2 popcount(F_a[i] ^ F_a[j])) for
// i in [0, rows), j in [0, cols) (gram_column, decompose.hpp:367-381; sign_dot,
// sign_vector.hpp:118-127); the products are integers, exact in f64.
struct GramParams {
  double* G;               // rows x ldg
  long long ldg;
  long long rows, cols;
  int nax;
  const uint32_t* Fi[8];   // [rows][fw] u32 words per axis (term-major)
  const uint32_t* Fj[8];   // [cols][fw]
  long long fw[8];         // u32 words per term (2 * ceil(n/64))
  long long n[8];
};
cudaError_t launch_gram(const GramParams& p, cudaStream_t st);

// Signed contractions out[j] = < sign outer product of term j, A > for nterms
// terms (contract_term, decompose.hpp:218-260), A viewed as P x Q like
// ExpandParams; f64 accumulation in a fixed order (per-row partials, then rows in
// order per CTA, then CTAs in order).
struct ContractParams {
  const void* A;           // P x Q row-major, f32 or f64
  int a_f32;
  long long P, Q;
  const uint32_t* U;       // [nterms][u_stride] or nullptr
  long long u_stride;
  const uint32_t* V;       // [nterms][v_stride] or nullptr
  long long v_stride;
  long long nterms;        // <= kContractTerms per launch
  int nch;                 // channel slices (1: none)
  int chan;                // as ExpandParams
  long long cstride;
  double* part;            // [grid][nterms * nch] per-CTA partials
  double* out;             // [nterms * nch]
};
constexpr int kContractTerms = 8;
constexpr int kContractCtas = 296;
cudaError_t launch_contract(const ContractParams& p, cudaStream_t st);

// dst[i] = (double) src[i] (f32 input widened exactly, like the DTEN f32 path).
cudaError_t launch_widen(const float* src, double* dst, long long n, cudaStream_t st);

// Sequential f64 sum of squares (frobenius_norm of a residual), fixed order.
cudaError_t launch_sqnorm(const double* x, long long n, double* part, double* out, cudaStream_t st);

}  // namespace scb
