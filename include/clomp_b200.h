/*
 * clomp_b200.h — C-ABI of the B200-native CLOMP reconstruction loop.
 *
 * Drop-in boundary for the reference's hot path.  The reference
 * exposes a static C++ API, not an FFI; each entry point below says which
 * reference function it replaces.  Plain pointers and sizes only: no torch, no
 * C++ types.  The C++ shim (paper_2501_11592_b200/csrc/shim/cskit_clomp_shim.cpp)
 * re-exposes these under the reference's own signatures, and INTEGRATION.md
 * shows the bindings.
 *
 * Numeric contract
 *   * Operands A and y are fp32 (north star).  Every product and reduction on
 *     the learning path is carried in fp64.  At th == 1 the batched
 *     correlation runs on the tcgen05 tensor cores as a split-fp16 GEMM
 *     (s*x = hi + lo, three kind::f16 MMAs hi.lo + lo.hi + hi.hi accumulated
 *     in fp32 TMEM, ~fp32 accuracy), and every selection whose top-2 gap lies
 *     inside that GEMM's error bound (delta_for in clomp_api.cu: (1e-5 +
 *     ldm/8 * 1.2e-7) * max||a|| * ||r||) is re-decided from exact fp64
 *     scores of the atoms in the band.  th < 1, B <= 4 (GEMV) and the fused
 *     small-problem path score in fp64 directly.  Supports therefore match
 *     the fp64 reference (clomp.cpp:211-292); coefficients agree to ~1e-12
 *     relative on the golden cases.
 *   * Priors (w_tv/w_lv > 0 after resolve_weights, clomp.cpp:131-140): TV-1D
 *     on single-column solves and TV-2D + local variance on multi-column
 *     joint batches (the reference's image mode) run on the GPU once a
 *     synthesis basis is set (cl_set_basis); separable and column-sharded
 *     contexts return CL_ERR_UNSUPPORTED.  Never a CPU fallback.
 *
 *   * Support capacity per signal: th == 1 adds one atom per outer iteration
 *     (plus exact ties), so the capacity is max_outer + 16.  1D contexts keep a
 *     Gram matrix per signal and serve up to 2048 atoms (th < 1: a signal that
 *     outgrows it ends with CL_ERR_CAPACITY); separable contexts switch to
 *     direct-form learning (cl_set_direct_form) and have no limit below n.
 *
 * Threading: one context per host thread; calls on distinct contexts may run
 * concurrently.  A context owns one device, one stream and its workspace.
 */
#ifndef CLOMP_B200_H
#define CLOMP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CL_ABI_VERSION 1

/* Status codes.  2/3/4 are the reference's CLI exit codes for ConfigError,
 * DimensionError and NumericalError (errors.hpp:10-37, cskit.cpp:1074-1093). */
typedef enum cl_status {
  CL_OK = 0,
  CL_ERR_INTERNAL = 1,
  CL_ERR_CONFIG = 2,       /* cskit::ConfigError    (clomp.cpp:18-30)          */
  CL_ERR_DIMENSION = 3,    /* cskit::DimensionError (clomp.cpp:215-218)        */
  CL_ERR_NUMERICAL = 4,    /* cskit::NumericalError (clomp.cpp:255-256)        */
  CL_ERR_UNSUPPORTED = 5,  /* a combination this build does not serve (message says which) */
  CL_ERR_CUDA = 6,         /* CUDA runtime / no device / extension missing     */
  CL_ERR_CAPACITY = 7      /* support grew past the per-signal capacity        */
} cl_status;

/* Optimizers (clomp.hpp:14, gradient_step clomp.cpp:171-209). */
enum { CL_OPT_PLAIN = 0, CL_OPT_MOMENTUM = 1, CL_OPT_ADAM = 2 };

/* Solve semantics.
 *   JOINT      = clomp_solve_batch (clomp.cpp:211-292): batch-global eps test,
 *                mask_changed, stall counter and best iterate.
 *   PER_SIGNAL = clomp_solve (clomp.cpp:294-311) on every column: the CLI's
 *                per-signal loop (cskit.cpp:543-551).  Columns never interact,
 *                which is what lets batches shard across GPUs with no traffic. */
enum { CL_MODE_JOINT = 0, CL_MODE_PER_SIGNAL = 1 };

/* Layouts.  REF = the reference's la::Mat row-major (A: m x n, y: m x B,
 * linalg.hpp:12-29).  T = transposed (A atom-major n x m, y signal-major B x m). */
enum { CL_LAYOUT_REF = 0, CL_LAYOUT_T = 1 };

/* ClompConfig (clomp.hpp:16-33), same field order and meaning. */
typedef struct cl_config {
  double th;                /* injection threshold in (0, 1]               */
  uint64_t max_outer;       /* outer iterations                            */
  double eps;               /* stop when ||r|| < eps                       */
  uint64_t inner_steps;     /* optimizer steps per outer iteration         */
  double lr;                /* step size; the gradient is 2 A^T r          */
  int32_t opt;              /* CL_OPT_*                                    */
  int32_t pad0;
  double w_tv;              /* negative = auto 0.01*mean(y^2); 0 = off     */
  double w_lv;
  uint64_t lv_window;       /* LvParams (priors.hpp:22-25)                 */
  uint64_t lv_stride;
  double stall_tol;
  uint64_t stall_patience;
} cl_config;

/* The reference defaults (clomp.hpp:16-33): th 0.7, max_outer 200, eps 1e-6,
 * inner 50, lr 0.01, Adam, auto priors, LvParams{3,2}, stall 1e-4 x 2. */
void cl_config_default(cl_config* cfg);

/* Results, caller-owned host buffers.  NULL pointers are skipped.
 * `cap` is the per-signal length of support/coef.  The support of signal b is
 * support[b*cap .. b*cap+count[b]) in ascending atom order with coef aligned. */
#define CL_RESULT_PREZEROED 1  /* cl_result::flags: s and mask are already all zero */
typedef struct cl_result {
  int64_t cap;
  int32_t* support;             /* [B][cap]                                */
  double* coef;                 /* [B][cap]                                */
  int32_t* count;               /* [B]                                     */
  double* s;                    /* dense n x B, REF layout (BatchSolveResult::s)   */
  uint8_t* mask;                /* dense n x B, REF layout (BatchSolveResult::mask) */
  int64_t* iterations;          /* [B]  (JOINT: identical)                 */
  double* final_residual_norm;  /* [B]  (JOINT: the batch Frobenius norm)  */
  uint8_t* converged;           /* [B]                                     */
  int32_t* status;              /* [B]  cl_status per signal               */
  double* x_hat;                /* dense n x B, REF layout: basis * (s .* mask)
                                 * (BatchSolveResult::x_hat, clomp.cpp:289); needs
                                 * cl_set_basis + cl_set_synthesis(ctx, 1)          */
  int32_t flags;                /* CL_RESULT_* (0: the library zero-fills s / mask) */
  int32_t pad0;
} cl_result;

typedef struct cl_ctx cl_ctx;

/* Upload the dictionary once.  Replaces the per-call LossOps transpose
 * (clomp.cpp:57-66, 224): A is stored atom-major fp32 in HBM.
 * a: host pointer, m x n (CL_LAYOUT_REF) or n x m (CL_LAYOUT_T).
 * Returns NULL on failure with *status set (cl_last_error(NULL) explains). */
cl_ctx* cl_create(int device, const float* a, int64_t m, int64_t n,
                  int a_layout, int* status);
void cl_destroy(cl_ctx* ctx);

/* Separable 2D operator Y = A_r S A_c^T (north star "2D mode"):
 * the dictionary is A = A_c (x) A_r with column-major vec, i.e. atom
 * p = i + n_r*j (S[i][j]) and measurement q = qr + m_r*qc (Y[qr][qc]); y
 * passed to cl_solve_batch is vec(Y) per signal (m = m_r*m_c rows).  The
 * Kronecker matrix is never formed.  a_r: m_r x n_r, a_c: m_c x n_c
 * (CL_LAYOUT_REF) or their transposes (CL_LAYOUT_T). */
cl_ctx* cl_create_sep(int device, const float* a_r, int64_t m_r, int64_t n_r,
                      const float* a_c, int64_t m_c, int64_t n_c, int layout,
                      int* status);

/* Column-sharded dictionary over `world` GPUs (one process per GPU, SURVEY.md
 * §8e): every rank passes the whole dictionary and the same batch; rank r runs
 * the correlation GEMM on atoms [r n/world, (r+1) n/world) for all signals and
 * learns signals [r B/world, (r+1) B/world).  Per outer iteration the ranks
 * exchange the per-(signal, atom tile) correlation candidates and the new
 * residual rows with ncclAllGather and sum the active-signal count with
 * ncclAllReduce; every rank returns the results of the whole batch.
 * Per-signal mode with th = 1; n divisible by world * 256.  nccl_id: the
 * 128-byte ncclUniqueId from cl_nccl_unique_id on rank 0, shared by the caller
 * (e.g. torch.distributed.broadcast_object_list).  world == 1 needs no id. */
int cl_nccl_unique_id(void* id_out);
cl_ctx* cl_create_colshard(int device, const float* a, int64_t m, int64_t n,
                           int a_layout, int rank, int world,
                           const void* nccl_id, int* status);
/* Test hook: run the column-sharded algorithm with `shards` virtual shards on
 * this one GPU (the exchange is a local copy instead of NCCL). */
int cl_set_virtual_shards(cl_ctx* ctx, int shards);

/* Multi-GPU context group in ONE process: one context per
 * listed device, driven by one host thread per device inside each call.
 *   CL_GROUP_SIGNAL_SHARD: the batch's independent signals (CL_MODE_PER_SIGNAL,
 *     the CLI's per-signal loop cskit.cpp:543-551) are split into contiguous
 *     ranges, one per device, with no data-path communication; every device
 *     holds the whole dictionary.  A device may be listed more than once.
 *   CL_GROUP_COLUMN_SHARD: one large dictionary sharded by atoms
 *     (cl_create_colshard over NCCL, distinct devices): every device solves
 *     the whole batch together; rank 0's results are returned.
 * cl_group_solve_batch has cl_solve_batch's arguments and result layout. */
enum { CL_GROUP_SIGNAL_SHARD = 0, CL_GROUP_COLUMN_SHARD = 1 };
typedef struct cl_group cl_group;
cl_group* cl_create_group(const int* devices, int ndev, const float* a, int64_t m, int64_t n,
                          int a_layout, int mode, int* status);
void cl_destroy_group(cl_group* g);
int cl_group_size(const cl_group* g);
cl_ctx* cl_group_context(cl_group* g, int index);   /* borrowed: knobs, stats */
const char* cl_group_last_error(const cl_group* g); /* NULL: last failing cl_create_group */
int cl_group_solve_batch(cl_group* g, const float* y, int64_t batch, int y_layout,
                         const cl_config* cfg, int mode, cl_result* out);

/* Message of the last failing call on ctx (or of the last failing cl_create
 * on this thread when ctx is NULL). */
const char* cl_last_error(const cl_ctx* ctx);

/* Replaces clomp_solve_batch (clomp.cpp:211-292) and, with batch == 1,
 * clomp_solve (clomp.cpp:294-311).  Host buffers; blocking.
 * y: m x B (CL_LAYOUT_REF) or B x m (CL_LAYOUT_T).
 * Returns the call status: JOINT -> the exception the reference would throw;
 * PER_SIGNAL -> CL_OK unless the call itself is invalid (per-signal failures
 * are in out->status). */
int cl_solve_batch(cl_ctx* ctx, const float* y, int64_t batch, int y_layout,
                   const cl_config* cfg, int mode, cl_result* out);

/* Pipelined form of cl_solve_batch for streams of batches (throughput):
 * cl_submit validates, starts the host->device copy of y on a copy stream and
 * queues the whole solve and the device->host copy of its compact results
 * behind it; cl_wait blocks until the OLDEST submitted batch's results are in
 * host memory and expands them into `out` exactly as cl_solve_batch does.  Up
 * to two batches may be in flight per context, so batch i + 1's upload and
 * batch i's download overlap the other's solve (cl_solve_batch = cl_submit +
 * cl_wait).  y must stay valid until the matching cl_wait returns when it is
 * page-locked (it is read by the DMA engine); a pageable y is copied to the
 * context's pinned staging before cl_submit returns.  Errors of the call
 * itself (config, dimensions, allocation) are returned by cl_submit and leave
 * nothing in flight; solve results and JOINT-mode failures by cl_wait. */
int cl_submit(cl_ctx* ctx, const float* y, int64_t batch, int y_layout,
              const cl_config* cfg, int mode);
int cl_wait(cl_ctx* ctx, cl_result* out);

/* Device-resident variant for throughput: d_y is a device pointer, signal-major
 * B x m fp32 (leading dimension m).  Results are written to device buffers
 * (any may be NULL): support/coef [B][cap], count/iterations(int32)/
 * final_rn/converged/status [B].  Runs on the context stream; the host reads
 * the active-signal count between graph chunks, so the call returns with the
 * results written (cl_synchronize afterwards is harmless). */
typedef struct cl_device_result {
  int64_t cap;
  int32_t* support;
  double* coef;
  int32_t* count;
  int32_t* iterations;
  double* final_residual_norm;
  uint8_t* converged;
  int32_t* status;
} cl_device_result;
int cl_solve_batch_device(cl_ctx* ctx, const float* d_y, int64_t batch,
                          const cl_config* cfg, int mode,
                          const cl_device_result* out);
int cl_synchronize(cl_ctx* ctx);

/* Replaces inject_support (clomp.cpp:142-154): mask |= { j : |a_j^T r| >= th *
 * max_j |a_j^T r| } per column, skipping zero columns.
 * r: host m x B fp64 (REF layout); mask: host n x B (REF layout), in/out. */
int cl_inject_support(cl_ctx* ctx, const double* r, int64_t batch, double th,
                      uint8_t* mask);

/* Introspection for tests and the bench. */
typedef struct cl_stats {
  int64_t kernel_launches;      /* kernels launched by the last solve       */
  int64_t rescans;              /* selections re-decided in fp64            */
  int64_t outer_iterations;     /* outer iterations executed (max over B)   */
  double corr_ms;               /* device time of the correlation kernels   */
  double learn_ms;              /* device time of the learning kernels      */
  double total_ms;              /* device time of the whole solve           */
  int32_t corr_path;            /* 0 fp64 SIMT, 1 tcgen05 split-f16, 2 fused, 3 GEMV */
  int32_t pad0;
  double e2e_ms;                /* cl_solve_batch: wall clock of the whole call  */
  double select_ms;             /* device time of select + fp64 rescans     */
  int64_t h2d_bytes;            /* bytes copied host->device by that call   */
  int64_t d2h_bytes;            /* bytes copied device->host by that call   */
} cl_stats;
int cl_get_stats(const cl_ctx* ctx, cl_stats* out);

/* Tuning / test knobs: 0 = auto (GEMV for B <= 4, else tcgen05 at th == 1,
 * else fp64 SIMT), 1 = force the fp64 correlation, 2 = force the tcgen05
 * split-fp16 correlation (th == 1 only; separable contexts: stage 2 of
 * A_r^T R A_c as K1 on the rows of R A_c, needs n_r a multiple of 256),
 * 3 = force the HBM-bound GEMV (1 <= B <= 4, 1D). */
int cl_set_corr_path(cl_ctx* ctx, int path);
/* Dictionary Gram cache G = A^T A (fp64, n x n) used to extend each signal's
 * support Gram matrix by a gather instead of re-streaming atoms:
 * 1 = build, 0 = drop, -1 = auto (built by cl_create when n*n*8 <= min(8 GiB,
 * free/4)). */
int cl_set_gram_cache(cl_ctx* ctx, int mode);
/* Small problems (n*m <= 4M words, supports <= 32 atoms, per-signal
 * semantics) run the whole solve in one persistent block per signal; 0
 * forces the batched kernel pipeline instead (tests compare the two). */
int cl_set_fused(cl_ctx* ctx, int on);
/* Synthesis basis D (n x n, x = D s; MeasurementSetup::basis, sensing.hpp:37-45)
 * for the priors and the synthesis x_hat = D s.  Single-column solves
 * (CL_MODE_PER_SIGNAL — the CLI's 1D path, clomp_solve per column — or a
 * one-column batch) run the TV prior (priors.cpp:11-26, chained through D^T,
 * clomp.cpp:93-119) folded into the support Gram system; multi-column joint
 * batches (the reference's image mode, cskit.cpp:620-652) run TV-2D + local
 * variance per epoch.  layout CL_LAYOUT_REF: basis[q * n + j] = D(q, j)
 * (la::Mat row-major); CL_LAYOUT_T: the transpose.  NULL clears.  Priors
 * without a basis, or on separable / column-sharded contexts, return
 * CL_ERR_UNSUPPORTED. */
int cl_set_basis(cl_ctx* ctx, const double* basis, int64_t n, int layout);
/* Synthesis x_hat = D (s .* mask) (clomp.cpp:289) on the GPU: when on, every
 * host-buffer solve of a context with a basis also forms x_hat from the
 * compact supports (n x count multiply-adds per signal instead of the
 * reference's dense n x n x B product) and returns it in cl_result::x_hat
 * (n x B fp64 more per download).  Off by default; a non-NULL x_hat without
 * it (or without a basis) fails with CL_ERR_UNSUPPORTED. */
int cl_set_synthesis(cl_ctx* ctx, int on);
/* Separable contexts, large supports: learn in DIRECT form — the reference's
 * epoch (clomp.cpp:83-91, 120-123) applied through the factors, V = A_r C
 * (column-sorted sparse), R = V A_c^T - Y and U = R A_c as fp64 GEMMs, the
 * gradient 2 a_r,i . U_j on the support entries only — instead of the Gram
 * form, whose t x t matrix per image stops fitting (above 2048 atoms: config
 * 5's K = 13107) or costs more to stream than the operator costs to apply.
 * from_outer: -1 auto (every iteration without a Gram buffer; otherwise from
 * t^2 > m_r n_c m_c / 16 on), 0 never (supports above 2048 atoms then fail
 * with CL_ERR_UNSUPPORTED), k > 0 from outer iteration k on (tests). */
int cl_set_direct_form(cl_ctx* ctx, int from_outer);
/* Supports of 33..256 atoms learn on CTA clusters with the support Gram
 * matrix in registers (default 1); 0 keeps them on the block-per-signal
 * kernel (tests compare them). */
int cl_set_cluster_learn(cl_ctx* ctx, int on);
/* Plain gradient descent on cluster-learned supports (33..256 atoms): run the
 * E epochs as E mod 2^L plain steps, L batched squarings of T = I - 2 lr G on
 * the fp64 tensor cores and E / 2^L steps of c <- T^(2^L) c + d (the same
 * iterate in exact arithmetic).  levels: -1 auto (default, L = 3), 0 off (one
 * cluster epoch per reference epoch), 1..8 explicit. */
int cl_set_power_levels(cl_ctx* ctx, int levels);
/* Enable per-kernel CUDA-event timing in cl_get_stats (adds syncs). */
int cl_set_profiling(cl_ctx* ctx, int on);
/* Run this context's work on a caller-owned cudaStream_t (NULL restores the
 * context's own stream).  Lets a caller order the solve with its own work and
 * time it with events on that stream. */
int cl_set_stream(cl_ctx* ctx, void* stream);

/* Test hook: correlation scores A^T r for a batch of fp32 residuals
 * r (B x m, signal-major host) through the fp64 SIMT kernel (path 1, |scores|),
 * the tcgen05 split-fp16 kernel (path 2, signed scores) or the GEMV (path 3,
 * |scores|, B <= 4); scores: host B x n. */
int cl_debug_scores(cl_ctx* ctx, const float* r, int64_t batch, int path,
                    double* scores);

int cl_abi_version(void);
int cl_device_count(void);
/* sizeof cl_config, cl_result, cl_device_result, cl_stats as this library was
 * compiled: bindings in other languages check their struct mirrors against it. */
void cl_abi_struct_sizes(int64_t out[4]);

#ifdef __cplusplus
}
#endif

#endif /* CLOMP_B200_H */
