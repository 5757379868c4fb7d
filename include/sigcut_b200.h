/*
 * sigcut_b200.h -- C ABI of the B200-native greedy signed-cut engine.
 *
 * Drop-in boundary for the reference's decomposition entry points
 * (reference tree /root/reference/proj/include/sigcut/):
 *
 *   sc_greedy_decompose  replaces  sigcut::greedy_decompose(const DenseTensor&,
 *                                   const DecomposeConfig&)       decompose.hpp:314-361
 *                        and       sigcut::decompose(...)         decompose.hpp:472-476
 *                                   (method kGreedy)
 *   sc_greedy_decompose with seed_mode = SC_SEED_DIRECT and width = 1 replaces
 *                                  sigcut::greedy_signed_cut /
 *                                  sigcut::axial_greedy_cut       search.hpp:259-272
 *   sc_validate_problem  restates  detail::check_decompose_config decompose.hpp:290-298,
 *                                  DenseTensor shape checks       dense_tensor.hpp:57-79,
 *                                  best_of_restarts checks        search.hpp:217-218
 *   sc_start_vectors     restates  the per-cut start draw of greedy_matrix_run /
 *                                  axial_run (search.hpp:149-150, :197) seeded by
 *                                  term_search_config (decompose.hpp:300-304) and
 *                                  best_of_restarts (search.hpp:222)
 *   sc_width_for_compression restates width_for_compression  metrics.hpp:55-63
 *
 * Plain pointers and sizes only.  Status codes map 1:1 onto the reference's
 * exceptions: SC_INVALID_ARGUMENT <-> std::invalid_argument,
 * SC_RUNTIME_ERROR <-> std::runtime_error (include/sigcut_b200.hpp does the mapping).
 * One context per device; calls on one context are serialised by the caller;
 * distinct contexts are independent.  There is no CPU fallback: without a
 * usable sm_100 device sc_create fails with SC_CUDA_ERROR.
 */
#ifndef SIGCUT_B200_H
#define SIGCUT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SC_ABI_VERSION 1
#define SC_MAX_ORDER 8

typedef enum sc_status {
  SC_OK = 0,
  SC_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  SC_RUNTIME_ERROR = 2,    /* std::runtime_error in the reference */
  SC_CUDA_ERROR = 3,       /* device / driver failure (no reference analogue) */
  SC_NOT_SUPPORTED = 4     /* shape outside the kernels' envelope */
} sc_status;

typedef enum sc_dtype { SC_F32 = 0, SC_F64 = 1 } sc_dtype;

typedef enum sc_seed_mode {
  SC_SEED_PER_TERM = 0, /* term k searches with substream(seed, k): greedy_decompose */
  SC_SEED_DIRECT = 1    /* term 0 searches with seed itself: greedy_signed_cut      */
} sc_seed_mode;

typedef struct sc_ctx sc_ctx;

/* Input tensor + DecomposeConfig/SearchConfig mirror (decompose.hpp:273-286,
 * search.hpp:20-24).  data is row-major (last axis fastest) in `dtype`; it is a
 * device pointer when data_on_device != 0, else host memory. */
typedef struct sc_problem {
  int32_t dtype; /* sc_dtype: storage and streaming type of the remainder */
  int32_t order; /* 2 = matrix (order-k tensors: see sc_greedy_decompose) */
  const uint64_t* shape;
  const void* data;
  int32_t data_on_device;
  int32_t seed_mode;    /* sc_seed_mode */
  uint64_t width;       /* DecomposeConfig::width */
  uint64_t flush_width; /* DecomposeConfig::flush_width: curve re-anchor cadence */
  uint64_t seed;        /* SearchConfig::seed */
  uint64_t restarts;    /* SearchConfig::restarts */
  uint64_t max_sweeps;  /* SearchConfig::max_sweeps */
  double min_value_fraction;
  uint64_t max_factor_bytes;
} sc_problem;

/* Caller-owned host output buffers sized for `width` terms (NULL = not wanted,
 * except sign_words / cut_value which are required).
 *   sign_words[axis]   width x ceil(shape[axis]/64) u64, term-major, bit b of
 *                      word u = entry 64u+b, set bit = -1, pad bits 0
 *                      (SignVector layout, sign_vector.hpp:15-84)
 *   alpha              CutDecomposition::coefficients (c_k / numel)
 *   cut_value          CutStep::cut_value (c_k)
 *   resid_norm         CutStep::residual_norm (reference recurrence with exact
 *                      re-anchors every flush_width terms and at the end)
 *   resid_norm_exact   exact ||R_k||_F after each term (device-computed)
 *   sweeps             alternation sweeps of the winning restart (CutResult::iterations)
 *   remainder          R_w, row-major, in the input dtype (numel elements)
 */
typedef struct sc_result {
  uint64_t* sign_words[SC_MAX_ORDER];
  double* alpha;
  double* cut_value;
  double* resid_norm;
  double* resid_norm_exact;
  uint32_t* sweeps;
  void* remainder;
  /* filled by the call */
  uint64_t width_done;
  double input_norm;
  double final_residual_norm;
  uint64_t passes;          /* streaming passes over the remainder executed */
  double kernel_ms;         /* device time of the decomposition kernel(s) */
  double total_ms;          /* host wall time of the whole call */
  uint64_t h2d_bytes;       /* bytes copied host->device by this call */
  uint64_t d2h_bytes;       /* bytes copied device->host by this call */
  int32_t kernel_launches;  /* kernels launched by this call */
} sc_result;

const char* sc_version(void);
int sc_abi_version(void);

sc_status sc_create(sc_ctx** out, int device);
void sc_destroy(sc_ctx* ctx);
const char* sc_last_error(const sc_ctx* ctx);

/* Greedy width-w signed-cut decomposition on the device (Alg. 5/13). */
sc_status sc_greedy_decompose(sc_ctx* ctx, const sc_problem* problem, sc_result* result);

/* Host-only validation with the reference's error semantics; writes a message
 * into msg (may be NULL).  Does not touch the GPU. */
sc_status sc_validate_problem(const sc_problem* problem, char* msg, size_t msg_len);

/* The start sign vector(s) of (term, restart) exactly as the reference draws
 * them: order 2 -> the t0 words (ceil(n/64)); order k -> one vector per axis,
 * concatenated in axis order.  Returns the number of words written. */
uint64_t sc_start_vectors(const sc_problem* problem, uint64_t term, uint64_t restart,
                          uint64_t* out_words);

/* Seeded synthetic input streams (Xoshiro256pp, rng.hpp:26-71). */
void sc_fill_normal_f64(uint64_t seed, uint64_t count, double* out);
void sc_fill_normal_f32(uint64_t seed, uint64_t count, float* out);

uint64_t sc_width_for_compression(int coeff_bits, int source_bits, int order,
                                  const uint64_t* shape, double rate);

/* Longest-processing-time-first assignment of `count` independent jobs with
 * the given costs to `bins` devices; writes the bin of each job.  Used by the
 * multi-GPU batch path (one process per GPU, no data-path collective). */
void sc_lpt_schedule(const double* costs, uint64_t count, uint32_t bins, uint32_t* bin_of_job);

/* ------------------------------------------------------------------------ */
/* Row-sharded decomposition of ONE matrix over `world` GPUs (one process and
 * one context per GPU).  Rank r owns the contiguous row band
 * [row0, row0 + local rows) of the m_global x n matrix.  The persistent kernel
 * of every rank joins one grid: per pass the z partials and the c / ||R||^2
 * partials of all ranks' CTAs are reduced in the same fixed order through
 * peer-mapped buffers (CUDA IPC over NVLink), owner CTAs publish the next t to
 * every rank, and one system-scope barrier separates the passes -- the
 * allreduce of R^T s and of the objective is fused into the kernel.
 * Protocol (all ranks):
 *   1. sc_shard_open(ctx, cfg, handle)   allocate + export this rank's buffers
 *   2. all-gather the world handles      (e.g. torch.distributed)
 *   3. sc_shard_connect(ctx, handles)    map the peers (world * 64 bytes)
 *   4. per decomposition: sc_shard_reset on every rank, a host barrier, then
 *      sc_greedy_decompose_sharded on every rank concurrently.
 * Results: sign_words[0] = this rank's row signs (local rows, bit 0 = row0),
 * sign_words[1] = t, coefficients and curve identical on all ranks. */
#define SC_IPC_HANDLE_BYTES 64
typedef struct sc_shard_config {
  int32_t rank, world;
  uint64_t m_global; /* rows of the whole matrix */
  uint64_t row0;     /* first global row of this rank's band */
  uint64_t n;        /* columns */
  int32_t dtype;     /* sc_dtype */
  int32_t ctas;      /* CTAs per rank, identical on all ranks; 0 = min(SMs, m_global / world) */
} sc_shard_config;

sc_status sc_shard_open(sc_ctx* ctx, const sc_shard_config* cfg, void* handle_out);
sc_status sc_shard_connect(sc_ctx* ctx, const void* handles);
sc_status sc_shard_reset(sc_ctx* ctx);
sc_status sc_greedy_decompose_sharded(sc_ctx* ctx, const sc_problem* local, const sc_shard_config* cfg,
                                      sc_result* result);
void sc_shard_close(sc_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* SIGCUT_B200_H */
