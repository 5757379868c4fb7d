// sweep.h -- launch parameters and shared-memory layout shared by the host
// driver (capi.cpp) and the persistent fused-sweep kernel (sweep.cu).
// No torch types anywhere.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace scb {

// Pass kinds (bit flags) published by the consumer controller to the TMA
// producer through shared memory.
enum PassFlags : int {
  F_DOT = 1,     // y = R t, s' = sgn(y), z = R^T s', c = <s, y>
  F_UPD = 2,     // R -= alpha s t^T applied while streaming (with F_DOT: fused into the term's first dot pass)
  F_NORM = 4,    // ||R||_F^2 accumulated (f64)
  F_WB = 8,      // write SMEM-resident rows back to global (end of run)
  F_CHECK = 16,  // reject non-finite input values (first pass)
  F_DELTA = 32,  // with F_DOT: update the cached y, z from the flipped t columns / s rows only
  K_TERM = 256,  // no more passes
};

enum ErrSlot : int { ERR_Y = 0, ERR_Z = 1, ERR_INPUT = 2 };
// err_pass[3] (world > 1): first pass at which a cross-rank spin timed out or saw the abort word

// Per-CTA scalar partials of a pass, double-buffered by pass parity (a CTA can
// run at most one pass ahead of the slowest reader).
struct Slot {
  double c[2];   // sum_i s_i y_i over the CTA's rows
  double n[2];   // ||R_rows||^2
  double dz[2];  // delta passes: 1 if this CTA wrote a z partial (some row flipped sign)
};

constexpr int kMaxStages = 16;
// Tagged t words sit one per 128-byte line: all CTAs poll them while the owners
// publish, and packing 16 per line made the pass time depend on which L2 slices
// those few lines hash to ("Placement of the exchange words").
constexpr int kTbStride = 16;

// Operands of the rank-1 update fused into a term's first dot pass (written by
// thread 0 at the pass's staging; read by the dot pass from shared memory).
struct UpdArgs {
  double alpha;
  void* Rband;      // global row 0 of the CTA's band
  long long pitch;
  int n;
  unsigned uws, s_upd;  // smem offsets: t of the update (Q words), s of the update (band words)
};

// Pass-invariant operands of the barrier-free delta pass (filled once per launch).
struct FastConst {
  const void* Rrows;  // global row 0 of the CTA's band
  const void* R;
  unsigned long long* drec;
  unsigned long long* tb64;
  double* zstate;
  unsigned* errp;
  unsigned long long* prof;  // [16] cycle sums (SCB_PROFILE builds) or nullptr
  long long pitch;
  unsigned res, yrow, sb, tws, txor, clist, fws, fbuf, zseg, rowB;  // shared-memory offsets, row bytes
  int rows_g, nres, Q, G, sw, rstride, n, g, rows_base, rows_rem;
  int nls;  // 32-column words this CTA owns (words g, g + G, ...; 0: not an owner)
  int direct;       // 1: each owner warp polls the flip words of its own CTA range (no staging)
  int cpar;         // 1: warp 0 polls every c partial at once (else one butterfly's worth at a time)
  int shared_list;  // 1: the owners' flipped-row list is built by col_reduce (many flip words)
};

// Per-CTA controller block in shared memory.
struct Ctl {
  unsigned long long full[kMaxStages];   // TMA -> dot warps
  unsigned long long empty[kMaxStages];  // z warps -> TMA
  volatile int decided;  // kinds of passes [0, decided) are published
  volatile int stored;   // global-R writes of passes [0, stored) are complete
  volatile int abort;
  volatile int aborted;  // world > 1: a cross-rank spin of this CTA timed out / saw the abort word
  volatile int upd_done;  // fused-update dot pass P: phase A's write-back is complete (P + 1)
  UpdArgs ua;
  FastConst fc;
  long long fprof[16];  // SCB_PROFILE builds: cycle sums of the barrier-free delta pass sections
  volatile int kind_ring[4];
  // controller state (thread 0 writes, consumers read after a named barrier)
  int kind, pp, term, restart, tsel, utsel, best_tsel, best_sweeps, best_restart;
  int cur, nxt, best, need_reduce, norm_idx, kron_upd;
  double alpha, c_prev, best_c, first_value;
  double ax_c;  // order-k mode: c = <s_{k-1}, v_{k-1}> of the axial step
  unsigned err_pre[4];  // error flags prefetched after the pass's grid barrier
  int nflip;            // columns of t that changed at this pass's staging (all CTAs agree); order-k:
                        // recounted by the axial step for the next pass's t (read by the decision)
  int since_dense;      // delta passes since the last dense dot pass
  int has_dz;           // this CTA wrote a z partial in a delta pass
  int nfrows, ndz;      // run totals: flipped streamed rows read by delta passes, dz partials written
  int keep;             // t unchanged since the last dot pass: y, s, z stay exactly as cached
  volatile int zerr;    // an owner warp of this CTA saw a non-finite z (carried into the next record)
  unsigned rank_dz;     // world > 1: ranks whose rank partial holds a delta-pass dz
  double cred[64];  // per-warp partials (axial step: 4 outputs x up to 16 warps)
  int axn[8], axoff[8];  // order-k: n_1..n_{k-1} and their axis-word offsets (shared-memory copies)
  double nred[32];
};

struct KParams {
  void* R;             // m x pitch, row-major, pad columns zero
  long long pitch;     // elements per row (multiple of 32)
  int m, n;
  int G;               // CTAs (one per SM)
  int rows_base, rows_rem;
  int res_rows;        // rows per CTA kept resident in shared memory
  int stages;          // TMA ring depth (one row per stage)
  int Q;               // 32-column slices = pitch / 32
  int sw;              // u32 words of per-CTA sign bits
  int zl;              // local slices per reduction group (zseg capacity)
  int rows_max;        // max rows per CTA
  const uint32_t* t0;  // [width][restarts][t0_stride] start vectors (u32 view)
  int t0_stride;       // u32 words per start vector (= 2 * ceil(n/64))
  unsigned long long* tb64;  // [2][Q] t words tagged with the consuming pass: (P << 32) | word,
                             // one per kTbStride u64s (a 128-byte line each)
  uint32_t* tbest;     // [Q] t of the best restart so far (restarts > 1)
  double* zpart;       // [2][G][pitch] per-CTA column partials, by pass parity
  Slot* slots;         // [G] c / ||R||^2 partials
  unsigned* bar;       // grid barrier counter
  unsigned* err_pass;  // [3] first pass index that saw an error (UINT_MAX = none)
  uint32_t* S_out;     // [width][s_stride] u32 view of packed row signs
  int s_stride;
  uint32_t* T_out;     // [width][t_stride]
  int t_stride;
  double* c_out;       // [width]
  uint32_t* sweeps_out;  // [width]
  double* norm2_out;   // [width + 1]: [0] = ||A||^2, [k+1] = ||R after term k||^2
  unsigned long long* stats;  // [0] width_done, [1] passes, [2]/[3] dense/delta dot passes, [4] term 0's winning restart,
                              // traffic counters: [5] flipped streamed rows read by delta passes, [6] delta
                              //     dz partials written, [7] t flips summed over delta passes (CTA 0)
  double* sweep_vals;  // [restarts][max_sweeps] c of every sweep of term 0 (SearchDiagnostics) or nullptr
  long long width, restarts, max_sweeps;
  double min_frac;
  double numel_d;
  int widen_mul;       // 1 << 29, passed at run time so ptxas emits IMAD.WIDE (not 3 shifts)
  // order-k tensors (k == 1 or k >= 3; axial_run, search.hpp:191-213): the kernel
  // runs on the matrix view M = n_0 x (n_1 ... n_{k-1}); axes 1..k-1 are updated
  // from Z = M^T s_0 by every CTA after the column reduction.
  int tensor;          // 1: order-k axial mode
  int kax;             // trailing axes (k - 1)
  int ax_n[7];         // n_1 .. n_{k-1}
  int ax_off[7];       // u32 word offset of axis i+1 within an axis-word record
  int axw;             // u32 words per axis-word record (even)
  const uint32_t* ax0; // [width][restarts][axw] start words of axes 1..k-1
  uint32_t* AX_out;    // [width][axw] accepted axis words
  double* zfull;       // [pitch] reduced z (order-k mode)
  int two_phase;       // 1: dot pass as (A) y = R t, (B) z = R^T s' (rows streamed twice)
  int delta;           // 1: sparse delta passes between dense refreshes (matrix mode)
  int fuse_update;     // 1: the rank-1 update rides on the next term's first dot pass (else its own pass)
  int delta_div;       // delta pass only if the last sweep flipped <= n / delta_div columns
  int delta_refresh;   // dense refresh every delta_refresh sweeps
  double* zstate;      // [pitch] z = R^T s of the previous pass (owners' columns)
  unsigned long long* flipw;  // [2][G][sw] per-CTA (flip | s' << 32) words of a matrix delta pass, by parity
  // Barrier-free delta passes (one GPU, matrices, whole rows): every CTA publishes one
  // self-tagged record per pass -- sw pairs {P << 32 | flip word, P << 32 | s' word} and
  // one pair {tag | hi(c), tag | lo(c)} with its objective partial (tag bit 31: the CTA saw
  // a non-finite y, or a non-finite z as an owner in the previous pass) -- and polls
  // the others' records instead of meeting them at a grid barrier.
  unsigned long long* drec;   // [2][G][rstride] records by pass parity
  int rstride;                // u64 words per record (a multiple of 16: whole 128-byte lines)
  int fast_delta;             // 1: delta passes exchange records (else slots + flip words behind the barrier)
  // wide rows: every row is streamed as cpr column chunks of chunk_cols
  // elements (one stage each); cpr == 1, chunk_cols == pitch otherwise
  int cpr;
  int chunk_cols;
  // Row-sharded multi-GPU (one process per GPU): every rank runs this
  // kernel on its row band with the same G; the exchange buffers of all ranks are
  // peer-mapped (CUDA IPC over NVLink) and the CTAs of all ranks form one grid:
  // global CTA gg = rank * G + g, GT = world * G.  world == 1: the local buffers.
  // Per pass each rank first reduces its own G column partials into one rank
  // partial (zr, n f64) and its G slots into one rank slot, behind a rank-local
  // barrier; only those cross NVLink (n f64 + 3 f64 per rank and pass).
  int world, rank, GT;
  double* zr_pe[8];                  // per-rank [2][pitch] rank column partials (by pass parity)
  Slot* rslot_pe[8];                 // per-rank rank slot (c, ||R||^2, any dz), by pass parity
  double* zr_own;                    // = zr_pe[rank]
  Slot* rslot_own;                   // = rslot_pe[rank]
  unsigned long long* tb64_pe[8];    // per-rank [2][Q] tagged t words (owners write all)
  unsigned* bar_local;               // this rank's local barrier counter (world > 1)
  unsigned* abort_word;              // rank 0's: set by any CTA whose spin timed out (world > 1)
  long long timeout_ns;              // bound of every cross-rank spin (world > 1)
  int fault;                         // test hook: 1 = this rank's CTAs exit at once (a dead rank)
  unsigned long long* prof;  // [G][16] clock64 breakdown or nullptr
};

// Virtual ranks (row-sharding emulated on one GPU): ONE cooperative launch of
// world * G CTAs; CTA block r plays rank r with its own parameters.  The ranks
// wait on one another, so they must be one launch (co-resident), never separate
// kernels on one device.
constexpr int kMaxVRanks = 8;
struct KParamsVR {
  KParams r[kMaxVRanks];
  int world;
};

// Kernel variant: consumer warps and per-thread register tiles.
struct Variant {
  int dtype;  // 0 f32, 1 f64
  int nw;     // consumer warps (each owns a column segment of every row)
  int vpt;    // 16-byte vectors per thread per row
  int rg;     // rows per group (one dot-partial publication per group)
  int cps;    // CTAs per SM (2: 113-register budget, raw lag buffers)
  int tensor; // order-k instantiation (set by the host after pick_variant)
  int mr;     // multi-rank (row-sharded world > 1) instantiation (set by the host)
};

constexpr int kRing = 4;  // dot-partial ring depth (groups)

// Shared-memory carve-up (byte offsets from the dynamic smem base).
struct Layout {
  size_t stage, res, ctl, ring, rred, yrow, tws, uws, zseg, sb, ax, ypart, txor, dzmask, ybak, zst, fws, fbuf, clist, total;
};

constexpr int kCList = 256;  // flipped-column list entries per gather round (barrier-free delta pass)

constexpr int kFBuf = 64;  // per-warp flipped-row list entries (owners' delta-pass dz)

inline __host__ __device__ size_t align16(size_t x) { return (x + 15) & ~static_cast<size_t>(15); }

inline __host__ __device__ Layout make_layout(size_t rowB, int stages, int res_rows, int rg, int nw, int rows_max,
                                              int Q, int zl, int sw, int axw, int G) {
  Layout L;
  size_t o = 0;
  L.stage = o;
  o += static_cast<size_t>(stages) * rowB;
  L.res = o;
  o += static_cast<size_t>(res_rows) * rowB;
  L.ctl = o;
  o += align16(sizeof(Ctl));
  L.ring = o;
  o += align16(static_cast<size_t>(kRing) * 8);
  L.rred = o;
  o += align16(static_cast<size_t>(kRing) * rg * nw * 8);
  L.yrow = o;
  o += align16(static_cast<size_t>(rows_max) * 8);
  L.tws = o;
  o += align16(static_cast<size_t>(Q) * 4);
  L.uws = o;
  o += align16(static_cast<size_t>(Q) * 4);
  L.zseg = o;
  o += static_cast<size_t>(zl) * nw * 32 * 8;
  L.sb = o;
  o += align16(static_cast<size_t>(3) * sw * 4);
  L.ax = o;  // [2][axw]: current / best axis words (order-k mode)
  o += align16(static_cast<size_t>(2) * axw * 4);
  L.ypart = o;  // [rows_max][nw]: per-warp row partials of the two-phase dot pass
  o += align16(static_cast<size_t>(rows_max) * nw * 8);
  L.txor = o;  // [2][Q]: t XOR previous t, previous t (delta passes)
  o += align16(static_cast<size_t>(2) * Q * 4);
  L.dzmask = o;  // [64]: CTAs (global index) that wrote a z partial in a delta pass
  o += align16(64 * 4);
  L.ybak = o;  // [rows_max]: y kept across a sweep whose t did not change
  o += align16(static_cast<size_t>(rows_max) * 8);
  L.zst = o;  // [zl][32]: z state of the owner's column words (delta passes)
  o += static_cast<size_t>(zl) * 32 * 8;
  L.fws = o;  // [G][sw]: every CTA's (flip | s' << 32) words of a matrix delta pass (owners)
  o += static_cast<size_t>(G) * sw * 8;
  L.fbuf = o;  // [nw][kFBuf]: per-warp flipped-row lists (owners)
  o += static_cast<size_t>(nw) * kFBuf * 4;
  L.clist = o;  // [kCList]: flipped columns of this pass, ascending, bit 31 = the new t bit
  o += static_cast<size_t>(kCList) * 4;
  L.total = o;
  return L;
}

// Returns 0 on success.
int pick_variant(int dtype, long long pitch, Variant* v, long long override_code = 0);
cudaError_t set_smem_limit(const Variant& v, size_t bytes);
int blocks_per_sm(const Variant& v, size_t smem_bytes);  // co-resident CTAs at this smem
cudaError_t launch_sweep(const Variant& v, const KParams& p, size_t smem_bytes, cudaStream_t st);
// virtual-rank launch (world * G CTAs); false from has_vr: no such instantiation
bool has_vr(const Variant& v);
cudaError_t set_smem_limit_vr(const Variant& v, size_t bytes);
cudaError_t launch_sweep_vr(const Variant& v, const KParamsVR& p, int G, size_t smem_bytes, cudaStream_t st);

}  // namespace scb
