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
 *   sc_batch_decompose   runs independent greedy_decompose calls over several
 *                                  devices (the reference's "concurrent calls on
 *                                  distinct inputs are safe", README:179-181)
 *   sc_start_vectors     restates  the per-cut start draw of greedy_matrix_run /
 *                                  axial_run (search.hpp:149-150, :197) seeded by
 *                                  term_search_config (decompose.hpp:300-304) and
 *                                  best_of_restarts (search.hpp:222)
 *   sc_width_for_compression restates width_for_compression  metrics.hpp:55-63
 *
 * Around the path, same boundary rules:
 *   sc_accumulate_expansion replaces detail::accumulate_expansion decompose.hpp:182-197
 *                        and (zero_fill)  sigcut::expand            decompose.hpp:266-270
 *   sc_gram_matrix       replaces  detail::build_gram (Gram part)   decompose.hpp:383-393
 *   sc_contract_terms    replaces  detail::contract_term            decompose.hpp:218-260
 *   sc_solve_gram        restates  sigcut::solve_gram               gram.hpp:83-107
 *   sc_solve_gram_leading  the same for every leading block (lstsq's term loop), O(k^2) each
 *   sc_correct_coefficients replaces sigcut::correct_coefficients  decompose.hpp:418-428
 *   sc_lstsq_decompose   replaces  sigcut::lstsq_decompose          decompose.hpp:434-469
 *                        and (channel_axis >= 0) rgb_scalars_decompose :485-536
 *   sc_write_scd / sc_read_scd(_header) restate write_scd / read_scd io.hpp:135-213
 *   sc_write_dten / sc_read_dten(_header) restate write_raw / read_raw io.hpp:226-292
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
  SC_NOT_SUPPORTED = 4,    /* shape outside the kernels' envelope */
  SC_IO_ERROR = 5          /* sigcut::io_error (io.hpp:22-24) in the reference */
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
  /* optional (NULL = not wanted): SearchDiagnostics::sweep_values (search.hpp:37-40)
   * of term 0's winning restart -- the cut value c after every sweep; room for
   * max_sweeps values.  n_sweep_values receives their count (= sweeps[0]). */
  double* sweep_values;
  uint64_t n_sweep_values;
  /* filled by the call: dot passes by form, and the bytes the kernel moved through
   * L2 / HBM (streamed rows of R, delta-pass gathers at sector granularity, rank-1
   * update write-backs, column-partial exchange; shared-memory-resident rows excluded) */
  uint64_t dense_passes;
  uint64_t delta_passes;
  uint64_t device_bytes;
} sc_result;

const char* sc_version(void);
int sc_abi_version(void);

sc_status sc_create(sc_ctx** out, int device);
void sc_destroy(sc_ctx* ctx);
const char* sc_last_error(const sc_ctx* ctx);

/* Engine options of this context (tuning / test knobs; the defaults are the
 * measured best).  Names: "ctas" (CTA cap, 0 auto), "delta" (sparse delta passes,
 * 1), "delta_div" (0 = auto: 4 with the barrier-free delta pass, else 32), "delta_refresh" (64), "two_phase" (dot-pass form: -1 auto,
 * 0 fused single read, 1 two-phase), "stages" (TMA ring depth, 0 auto),
 * "res_rows" (cap on SMEM-resident rows, -1 none), "fuse_update" (rank-1 update
 * fused into the next term's first dot pass, 1), "variant" (tile override
 * nw*1000000 + vpt*10000 + rg*100 + cps, 0 auto), "fast_delta" (delta
 * passes exchange self-tagged records instead of meeting at a grid barrier, 1),
 * "l2_persist" (R as a persisting-L2 window during the launch, 0), "profile" (clock64 breakdown of
 * SCB_PROFILE builds to stderr, 0), "poison" (test hook: fill the device arena with
 * NaN bytes before each call, so any read of a never-written word shows, 0).  No
 * option changes results except through the
 * documented summation orders (signs and sweep counts are option-independent). */
sc_status sc_set_option(sc_ctx* ctx, const char* name, int64_t value);
sc_status sc_get_option(const sc_ctx* ctx, const char* name, int64_t* value);
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

/* A batch of independent decompositions over several devices (
 * the reference's concurrency contract: concurrent calls on distinct inputs are
 * safe).  Jobs are assigned longest-processing-time first (cost =
 * width x numel, sc_lpt_schedule) to `devices`; one host thread and one context
 * per device run their jobs longest first, with no data-path communication.
 * Every job's result equals sc_greedy_decompose of it on any device.  Returns
 * SC_OK when every job succeeded, else the first failure's status (message in
 * msg); each job's own status and device are written back. */
typedef struct sc_batch_job {
  sc_problem problem;  /* host or device data (device data must live on the job's device) */
  sc_result* result;   /* caller-owned outputs, as for sc_greedy_decompose */
  int32_t status;      /* out: sc_status of this job */
  int32_t device;      /* out: device that ran it */
} sc_batch_job;
sc_status sc_batch_decompose(const int32_t* devices, int32_t ndevices, sc_batch_job* jobs, uint64_t njobs,
                             char* msg, size_t msg_len);
/* Longest-processing-time-first assignment of `count` independent jobs with
 * the given costs to `bins` devices; writes the bin of each job.  Used by the
 * multi-GPU batch path (one process per GPU, no data-path collective). */
void sc_lpt_schedule(const double* costs, uint64_t count, uint32_t bins, uint32_t* bin_of_job);

/* ------------------------------------------------------------------------ */
/* Sign-term factors of a CutDecomposition (decompose.hpp:30-100) in host
 * memory.  sign_words[i] belongs to the i-th SIGN axis in ascending axis order
 * (every axis except channel_axis): width x ceil(n/64) u64, term-major,
 * SignVector layout.  coefficients: width x channels, term-major (channels =
 * shape[channel_axis], or 1 when channel_axis == -1). */
typedef struct sc_factors {
  int32_t order;
  const uint64_t* shape;
  int32_t channel_axis;
  uint64_t width;
  const uint64_t* sign_words[SC_MAX_ORDER];
  const double* coefficients;
} sc_factors;

/* Per-call accounting of the auxiliary ops. */
typedef struct sc_op_stats {
  double kernel_ms;
  double total_ms;
  uint64_t h2d_bytes;
  uint64_t d2h_bytes;
  int32_t kernel_launches;
} sc_op_stats;

/* data[e] += sum over terms j in [first_term, last_term) of
 * flip(scale * coef_j(channel of e), parity_j(e)), summed in term order from 0.0
 * and added last (accumulate_terms, decompose.hpp:128-180): bit-identical to the
 * reference.  data: numel f64, row-major, host (data_on_device = 0) or device.
 * zero_fill != 0 zeroes data first (expand).  stats may be NULL. */
sc_status sc_accumulate_expansion(sc_ctx* ctx, const sc_factors* d, double scale, uint64_t first_term,
                                  uint64_t last_term, double* data, int32_t data_on_device, int32_t zero_fill,
                                  sc_op_stats* stats);

/* gram[i * width + j] = prod over sign axes of sign_dot(f_i, f_j): width x width
 * (exact integers in f64; bit-identical to gram_column). */
sc_status sc_gram_matrix(sc_ctx* ctx, const sc_factors* d, double* gram, sc_op_stats* stats);

/* rhs[(j - first_term) * channels + ch] = <sign outer product of term j, channel
 * ch of A> for j in [first_term, first_term + count).  A: numel values of
 * a_dtype (sc_dtype) in the factors' shape, host or device.  f64 sums in a fixed
 * parallel order (the reference sums sequentially: agreement to rounding). */
sc_status sc_contract_terms(sc_ctx* ctx, const sc_factors* d, int32_t a_dtype, const void* a, int32_t a_on_device,
                            uint64_t first_term, uint64_t count, double* rhs, sc_op_stats* stats);

/* Host Cholesky solve of the normal equations with the reference's ridge retry
 * (gram.hpp:48-107, same loop order).  gram: width x width; rhs / out: width x
 * channels, term-major.  SC_RUNTIME_ERROR when the factorisation fails. */
sc_status sc_solve_gram(uint64_t width, uint64_t channels, const double* gram, const double* rhs, double* out,
                        char* msg, size_t msg_len);

/* The same solve for every leading block k = 1..width of one system, as lstsq_decompose
 * (decompose.hpp:434-469) needs it term by term: the factor grows by one row per block
 * (the reference's column order leaves earlier rows unchanged), so block k costs O(k^2)
 * and every result equals sc_solve_gram of that block bit for bit.  out: the k x channels
 * solutions one after another, k = 1..width (width (width + 1) / 2 x channels doubles). */
sc_status sc_solve_gram_leading(uint64_t width, uint64_t channels, const double* gram, const double* rhs, double* out,
                                char* msg, size_t msg_len);

/* correct_coefficients (decompose.hpp:418-428): refit with the signs held fixed;
 * keeps the old coefficients when the solve is not better.  coeffs_out: width x
 * channels. */
sc_status sc_correct_coefficients(sc_ctx* ctx, const sc_factors* d, int32_t a_dtype, const void* a,
                                  int32_t a_on_device, double* coeffs_out, sc_op_stats* stats);

/* lstsq_decompose (decompose.hpp:434-469; channel_axis == -1) or
 * rgb_scalars_decompose (:485-536; channel_axis >= 0, channels <= 8): every
 * term is searched on the device on the explicit residual A - expand(d), the
 * coefficients are re-solved, and the residual is re-expanded on the device.
 * result: sign_words per SIGN axis (ascending), alpha = width x channels
 * coefficients, cut_value, resid_norm (= ||A - expand||_F after each term),
 * sweeps; resid_norm_exact and remainder as in sc_greedy_decompose. */
sc_status sc_lstsq_decompose(sc_ctx* ctx, const sc_problem* problem, int32_t channel_axis, sc_result* result);

/* SCD container (io.hpp:113-213), bytes identical to write_scd. */
uint64_t sc_scd_size(const sc_factors* d, int coeff_bits);
sc_status sc_write_scd(const sc_factors* d, int coeff_bits, uint8_t* out, uint64_t capacity, uint64_t* written,
                       char* msg, size_t msg_len);
/* shape must hold SC_MAX_ORDER entries. */
sc_status sc_read_scd_header(const uint8_t* in, uint64_t size, int32_t* order, uint64_t* shape,
                             int32_t* channel_axis, uint64_t* width, int32_t* coeff_bits, char* msg, size_t msg_len);
/* sign_words[i]: width x ceil(n/64) per sign axis; coefficients: width x channels. */
sc_status sc_read_scd(const uint8_t* in, uint64_t size, uint64_t** sign_words, double* coefficients, char* msg,
                      size_t msg_len);

/* DTEN raw tensors (io.hpp:215-292).  raw_dtype: 0 f64, 1 f32, 2 u8 (RawDType).
 * sc_write_dten encodes f64 values; sc_read_dten widens to f64 like read_raw. */
uint64_t sc_dten_size(int32_t order, const uint64_t* shape, int32_t raw_dtype);
sc_status sc_write_dten(int32_t order, const uint64_t* shape, const double* data, int32_t raw_dtype, uint8_t* out,
                        uint64_t capacity, uint64_t* written, char* msg, size_t msg_len);
sc_status sc_read_dten_header(const uint8_t* in, uint64_t size, int32_t* order, uint64_t* shape, int32_t* raw_dtype,
                              char* msg, size_t msg_len);
sc_status sc_read_dten(const uint8_t* in, uint64_t size, double* data, char* msg, size_t msg_len);

/* ------------------------------------------------------------------------ */
/* Row-sharded decomposition of ONE matrix over `world` GPUs (one process and
 * one context per GPU).  Rank r owns the contiguous row band
 * [row0, row0 + local rows) of the m_global x n matrix.  The persistent kernel
 * of every rank joins one grid.  Per pass each rank reduces its CTAs' column
 * partials of R^T s into one rank partial (n f64) and its c / ||R||^2 partials
 * into one rank slot behind a rank-local barrier; after one system-scope
 * barrier the owner CTA of every 32-column word adds the world rank partials in
 * rank order through peer-mapped buffers (CUDA IPC over NVLink) and publishes
 * the next t to every rank, and every CTA adds the world rank slots -- the
 * allreduce of R^T s and of the objective is fused into the kernel.  Every
 * cross-rank spin is bounded: after timeout_ms (or when any rank has set the
 * shared abort word) the kernel stops and the call returns SC_RUNTIME_ERROR.
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
  uint32_t timeout_ms; /* bound of every cross-rank spin in the kernel; 0 = 30000 */
} sc_shard_config;

sc_status sc_shard_open(sc_ctx* ctx, const sc_shard_config* cfg, void* handle_out);
sc_status sc_shard_connect(sc_ctx* ctx, const void* handles);
sc_status sc_shard_reset(sc_ctx* ctx);
sc_status sc_greedy_decompose_sharded(sc_ctx* ctx, const sc_problem* local, const sc_shard_config* cfg,
                                      sc_result* result);
void sc_shard_close(sc_ctx* ctx);
/* The same row-sharded protocol with `world` VIRTUAL ranks on this context's one
 * device, for machines with fewer GPUs than ranks: the ranks' kernels wait on
 * one another, so they run as ONE cooperative launch (CTA block r plays rank r
 * with rank r's band, parameters and exchange region; peer pointers are the
 * other ranks' regions on the same device).  `problem` is the WHOLE matrix; the
 * result is the gathered one (global row signs, t, c, curve), after checking
 * that every rank took the same decisions.  opts == NULL: world 1. */
typedef struct sc_shard_emulation {
  int32_t world;       /* virtual ranks, 1..8 */
  int32_t ctas;        /* CTAs per rank; 0 = SMs / world */
  uint32_t timeout_ms; /* as sc_shard_config::timeout_ms */
  int32_t dead_rank;   /* test hook: this rank's CTAs exit at once (a rank that never
                          joins; the others time out -> SC_RUNTIME_ERROR); -1 = none */
} sc_shard_emulation;
sc_status sc_greedy_decompose_sharded_emulated(sc_ctx* ctx, const sc_problem* problem,
                                               const sc_shard_emulation* opts, sc_result* result);

#ifdef __cplusplus
}
#endif

#endif /* SIGCUT_B200_H */
