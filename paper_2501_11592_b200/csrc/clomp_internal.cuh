// clomp_internal.cuh — device-side data layout and kernel launchers shared by
// the CUDA translation units of libclomp_b200.so.  Not a public header.
//
// HBM layout:
//   at32   [n][ldm] fp32   dictionary, atom-major (K-major GEMM operand); the
//                          reference keeps A row-major m x n plus a transposed
//                          copy per call (clomp.cpp:57-66).
//   y32/y64, r32/r64 [B][ldm]   measurements and residuals, signal-major.
//   per-signal state: support list in insertion order, coefficients, Gram
//   G = A_S^T A_S (fp64, cap x cap), b = A_S^T y, optimizer moments, best
//   snapshot, loss/stall bookkeeping (clomp.cpp:226-273).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <utility>

// Debug build (python -m paper_2501_11592_b200.build --debug ->
// _build/libclomp_b200_dbg.so, -DCL_DEBUG_CHECKS): device-side assert on every
// index the kernels form from data (atoms, support slots, list slots, tiles),
// standing in for compute-sanitizer where the tool is not available.  A failed
// check traps the kernel; the call returns CL_ERR_CUDA ("device-side assert").
#ifdef CL_DEBUG_CHECKS
#include <cassert>
#define CL_CHECK(cond) assert(cond)
#else
#define CL_CHECK(cond) ((void)0)
#endif

namespace clb {

// ---- per-device host caches
// One slot per device for a host-computed value of one call site (SM count,
// co-resident clusters, the dynamic shared-memory limit already raised).
// Racing initialisers compute the same value and the slots are atomics, so
// concurrent calls on distinct contexts (clomp_b200.h threading rule) are
// data-race free, and a second device never reuses the first one's value.
constexpr int kMaxDevices = 64;
struct DevSlots {
  std::atomic<long long> v[kMaxDevices];
  long long get(int dev) const { return v[dev & (kMaxDevices - 1)].load(std::memory_order_relaxed); }
  void set(int dev, long long x) { v[dev & (kMaxDevices - 1)].store(x, std::memory_order_relaxed); }
};
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
inline int device_sms(int dev) {
  static DevSlots cache;
  long long v = cache.get(dev);
  if (v <= 0) {
    int s = 0;
    if (cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || s <= 0) {
      cudaGetLastError();
      s = 148;
    }
    cache.set(dev, s);
    v = s;
  }
  return (int)v;
}
// Raise kern's dynamic shared-memory limit on the current device to at least
// `bytes` (once per device and size).
template <class K>
inline void ensure_smem_limit(DevSlots& slot, K kern, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  const int dev = current_device();
  if ((long long)bytes <= slot.get(dev)) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  slot.set(dev, (long long)bytes);
}

constexpr int kCorrTileAtoms = 64;    // fp64 SIMT correlation tile (atoms)
constexpr int kCorrTileSignals = 64;  // fp64 SIMT correlation tile (signals)
constexpr int kWarpCap = 32;          // register-resident learning kernel limit

// Correlation summary of one (signal, atom tile): the two largest |scores|
// with their atoms (the lowest atom wins an exact tie) and the third largest
// value.  A near-tied selection is re-decided exactly from these alone unless
// a third atom of the tile also lies inside the error band.
struct __align__(16) Cand {
  double v1, v2, v3;
  int32_t i1, i2;
};

// Insert score x of atom k into a descending (v1,i1) (v2,i2) v3 summary.
__host__ __device__ __forceinline__ void cand_insert(double& v1, int& i1, double& v2, int& i2,
                                                     double& v3, double x, int k) {
  if (x > v1 || (x == v1 && k < i1)) {
    v3 = v2;
    v2 = v1;
    i2 = i1;
    v1 = x;
    i1 = k;
  } else if (x > v2 || (x == v2 && k < i2)) {
    v3 = v2;
    v2 = x;
    i2 = k;
  } else if (x > v3) {
    v3 = x;
  }
}

__host__ __device__ __forceinline__ void cand_merge(Cand& a, const Cand& b) {
  double v1 = a.v1, v2 = a.v2, v3 = a.v3;
  int i1 = a.i1, i2 = a.i2;
  cand_insert(v1, i1, v2, i2, v3, b.v1, b.i1);
  cand_insert(v1, i1, v2, i2, v3, b.v2, b.i2);
  v3 = v3 > b.v3 ? v3 : b.v3;
  a.v1 = v1; a.v2 = v2; a.v3 = v3; a.i1 = i1; a.i2 = i2;
}

__host__ __device__ __forceinline__ Cand cand_empty() {
  Cand c;
  c.v1 = c.v2 = c.v3 = -1.0;
  c.i1 = c.i2 = 0x7fffffff;
  return c;
}

// Power-of-two scale for the fp16 split of a vector of 2-norm sqrt(L): every
// entry of the scaled vector is below 2^14 (fp16 max 65504), typical entries
// ~2^14/sqrt(m) keep the lo halves well above the fp16 subnormal range.
__host__ __device__ __forceinline__ float split_scale(double L) {
  if (!(L > 0.0) || !(L < 1e300)) return 1.0f;
  int k = 0;
  (void)frexp(sqrt(L), &k);  // sqrt(L) = f 2^k, f in [0.5, 1)
  k = k < -100 ? -100 : (k > 100 ? 100 : k);
  return ldexpf(1.0f, 14 - k);
}

// s*x = hi + lo + O(2^-22 |s x|), both fp16 (s = 2^e, exact).
__device__ __forceinline__ void split_f16(double x, float s, __half& hi, __half& lo) {
  const float f = (float)x * s;
  hi = __float2half_rn(f);
  lo = __float2half_rn(f - __half2float(hi));
}

struct SolveParams {
  int64_t B, n, m, ldm, cap, ntile;
  int64_t tile_atoms;       // atoms per correlation tile (candidate granularity)
  // Column-sharded contexts (cl_create_colshard): this rank learns signals
  // [sig_lo, sig_hi) and correlates atoms [atom0, atom0 + n_corr) for every
  // signal into ntl local tiles.  Single-GPU: 0, B, 0, n, ntile.
  int64_t sig_lo, sig_hi, atom0, n_corr, ntl;
  int64_t mwords;           // 32-bit words per signal in the mask bitmap
  double th, eps, lr, stall_tol;
  int32_t stall_patience, opt, inner, max_outer, mode;
  const double* bc1;        // Adam bias corrections per global step (1-based)
  const double* bc2;
  double delta_rel;         // correlation error bound / (||a||max * ||r||)
  double colnorm_max;
  // separable 2D operator A = A_c (x) A_r (atom p = i + nr*j, row q = qr + mr*qc)
  int32_t sep;
  int64_t nr, nc, mr, mc, ldr, ldc;
  // separable contexts: this iteration learns in direct form (k_sep.cu)
  int32_t direct;
  // th == 1 selection runs inside the learning kernel (warp per signal)
  int32_t fuse_select;
  double a_inv_scale;       // 1 / (power-of-two scale of the fp16 dictionary split)
  // supports of 33..256 atoms learn on CTA clusters with register-resident
  // Gram blocks (k_learn_cluster); 0 keeps them on k_learn_block (tests)
  int32_t cluster_learn;
  // power form of plain GD for cluster-sized supports (k_pow_sq): E = 2^L q + r
  // epochs run as r plain steps, L batched squarings of T = I - 2 lr G on the
  // fp64 tensor cores, then q steps of c <- T^(2^L) c + d_(2^L); the first
  // pw_slots big-list signals use it (0 levels: per-epoch cluster learning)
  int32_t pw_levels, pw_q, pw_r, pw_slots, pw_ld;
  // TV-1D prior (single-column solves): the Gram system carries
  // G + w_b H, H = (Delta D_S)^T (Delta D_S) / n, extended by k_prior_ext; the
  // learning kernels store the residual loss and k_prior_control adds w_b c^T H c
  // and runs the stopping rules (clomp.cpp:93-119, 253-273)
  int32_t prior;
  // image mode (prior == 2): multi-column joint batch with TV-2D / local
  // variance on x = D S (clomp.cpp:93-119), batch-global weights
  double w_tv_g, w_lv_g;
  int32_t lv_on, lv_window, lv_stride, lv_nr, lv_nc;
  // warp learners (plain GD): power levels L for support buckets of 8 / 16 /
  // 24 / 32 atoms (E = 2^L q + r epochs as L squarings + q + popcount(r) steps)
  int32_t warp_L[4];
};

struct Work {
  // operands
  const float* at32 = nullptr;   // [n][ldm]
  const __half* at_hi = nullptr;  // [n][ldm] scaled fp16 split (tensor path)
  const __half* at_lo = nullptr;
  const double* gfull = nullptr; // [n][n] fp64 A^T A (optional, per context)
  float* y32 = nullptr;          // [B][ldm]
  double* y64 = nullptr;
  double* r64 = nullptr;
  __half* r_hi = nullptr;        // [B][ldm] scaled fp16 split of the residual
  __half* r_lo = nullptr;
  float* r_scale = nullptr;      // [B] 1 / (its power-of-two scale)
  // separable 2D mode
  const double* at_r64 = nullptr;  // [nr][ldr] A_r atom-major
  const double* at_c64 = nullptr;  // [nc][ldc] A_c atom-major
  const double* gr = nullptr;      // [nr][nr] A_r^T A_r
  const double* gc = nullptr;      // [nc][nc] A_c^T A_c
  double* zb = nullptr;            // [B][n] A_r^T Y A_c (b values of every atom)
  double* sep_scratch = nullptr;   // [B][nc][mr] U = R A_c  /  V = A_r C
  double* lpart = nullptr;         // [B][tiles] residual sum-of-squares partials
  // separable correlation on the tensor cores: stage 2 (A_r^T U) is the K1
  // kernel on B nc pseudo-signals (the rows U_b[j][:] of U = R A_c)
  __half* u_hi = nullptr;          // [B nc][ldr] scaled fp16 split of U
  __half* u_lo = nullptr;
  float* u_scale = nullptr;        // [B nc] 1 / scale
  int32_t* u_active = nullptr;     // [B nc] the image's active flag per row
  // direct-form learning (large supports): second scratch for U = R A_c and the
  // support sorted by coefficient column
  double* sep_scratch2 = nullptr;  // [B][nc][mr]
  double* sep_z2 = nullptr;        // [B][nc][mr] Y A_c (constant part of U = R A_c)
  int32_t* csc_ptr = nullptr;      // [B][nc + 1]
  int32_t* csc_perm = nullptr;     // [B][cap] support entries by column
  Cand* xg = nullptr;            // column sharding: per-shard candidates [W][B][ntl]
  Cand* cand = nullptr;          // correlation candidates [B][ntile]
  double* scores = nullptr;      // [B][n] |A^T r| (th < 1 path)
  // per-signal state
  int32_t* sup = nullptr;        // [B][cap] insertion order
  int32_t* cnt = nullptr;        // [B]
  int32_t* gcnt = nullptr;       // [B] atoms whose Gram row/col is built
  double* coef = nullptr;        // [B][cap]
  double* mom1 = nullptr;        // [B][cap]
  double* mom2 = nullptr;        // [B][cap]
  double* gram = nullptr;        // [B][cap][cap]
  double* bvec = nullptr;        // [B][cap]
  uint32_t* maskbits = nullptr;  // [B][mwords]
  double* best_coef = nullptr;   // [B][cap]
  int32_t* best_cnt = nullptr;
  double* best_L = nullptr;
  double* prev_L = nullptr;
  double* loss = nullptr;        // [B] current loss ||A_S c - y||^2
  int32_t* stall = nullptr;
  int32_t* iters = nullptr;
  int32_t* active = nullptr;
  uint8_t* conv = nullptr;       // eps break happened
  int32_t* status = nullptr;
  int32_t* changed = nullptr;
  int32_t* big_list = nullptr;     // [B] signals queued for the block learner
  double* pw_t = nullptr;          // [2][pw_slots][pw_ld][pw_ld] powers T^(2^l) (ping-pong)
  double* pw_d = nullptr;          // [2][pw_slots][pw_ld] offsets d_(2^l)
  double* pw_part = nullptr;       // [pw_slots][row chunks] residual sum-of-squares partials
  int32_t* pw_cnt = nullptr;       // [pw_slots] finished row chunks (reset by the last one)
  int32_t* counters = nullptr;     // see Counter
  double* joint = nullptr;         // see Joint
  // priors (SolveParams::prior)
  const double* ddt = nullptr;     // [n][ldd] Delta D atom-major (fp64)
  int64_t ldd = 0;
  double* hgram = nullptr;         // [B][cap][cap] H of the support
  double* wtv = nullptr;           // [B] resolved TV weight per signal
  double* rloss = nullptr;         // [B] residual part of the current loss
  double* best_R = nullptr;        // [B] residual part of the best snapshot's loss
  // image mode
  const double* dt = nullptr;      // [n][n] basis atom-major: dt[k][q] = D[q][k]
  double* img_x = nullptr;         // [B][n] x = D S_eff, signal-major (pixel (q, b))
  double* img_gx = nullptr;        // [B][n] prior gradient in x-space
  double* img_gd = nullptr;        // [B][cap] data gradient 2 (G c - b)
  double* lv_mean = nullptr;       // [nr * nc] window means
  double* lv_scale = nullptr;      // [nr * nc] inv_blocks / (count sd), 0 when sd == 0
  double* lv_sd = nullptr;         // [nr * nc] window standard deviations
  const int32_t* lv_rows = nullptr;   // [nr] window row origins
  const int32_t* lv_cols = nullptr;   // [nc] window column origins
  const int32_t* lv_rowcov = nullptr; // [n][8] row-window indices covering row q (-1 pad)
  const int32_t* lv_colcov = nullptr; // [B][8] column-window indices covering column b
  double* img_part = nullptr;      // [1024] loss partials
};

enum Counter {
  kCounter0 = 0,      // (unused)
  kCounter1 = 1,      // (unused)
  kMaxCount = 2,      // max support size over the batch
  kRescanTotal = 3,   // rescans over the whole solve
  kBigCount = 4,      // signals queued for the block learning kernel; slots
                      // 4 + (outer & 1), the block kernel clears the other one
  kActive0 = 6,       // signals still iterating after outer iteration o: slot
                      // 6 + (o & 1) (active_slot), incremented by the stopping
                      // rules of iteration o and cleared by the learning kernel
                      // of iteration o - 1, i.e. one whole kernel boundary
                      // before any increment (no in-grid store/atomic race)
  kNumCounters = 8
};

__host__ __device__ __forceinline__ int active_slot(int outer) { return kActive0 + (outer & 1); }

enum Joint {
  kJBest = 0, kJPrev = 1, kJTotal = 2, kJStall = 3, kJImproved = 4,
  kJStop = 5, kJConv = 6, kJStatus = 7, kJIters = 8, kJFinalRn = 9,
  kJPrior = 10,   // image mode: w_tv tv + w_lv lv of the current coefficients
  kJTotalR = 11,  // image mode: residual part of kJTotal
  kJBestR = 12,   // image mode: residual part of kJBest
  kNumJoint = 16
};

// Programmatic dependent launch (PDL): kernels of the per-iteration chain are
// launched with cudaLaunchAttributeProgrammaticStreamSerialization, let their
// successor start launching as soon as every CTA is resident (pdl_trigger),
// and wait for their predecessor's completion and memory (pdl_wait) before
// touching its outputs, so launch latency and prologues overlap the previous
// kernel's tail.  Both are no-ops without a programmatic dependency.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---- launchers (k_corr.cu) ----
// fp64 SIMT correlation with fused top-2 epilogue (th == 1) or full |scores|.
void launch_corr_f64(const SolveParams& p, const Work& w, bool full_scores,
                     cudaStream_t s);
// K1b (k_corr_gemv.cu): HBM-bound fp64-accumulating GEMV for B <= 8 residuals,
// the same candidate records (and optional |scores|) as launch_corr_f64.
bool corr_gemv_supported(int64_t ldm, int64_t B);
int64_t corr_gemv_tile_atoms();
void launch_corr_gemv(const SolveParams& p, const Work& w, bool full_scores,
                      cudaStream_t s);
// tcgen05 3xTF32 correlation with fused top-2 epilogue (th == 1).
bool corr_tc_available();
int corr_tc_trace(unsigned long long* out, int max_ctas);
int cluster_trace(unsigned long long* out);
int learn_trace(unsigned long long* out, int max_signals);
int64_t corr_tc_tile_atoms();
// false: the tensor maps could not be encoded or the launch failed (the
// caller reports CL_ERR_CUDA; stale candidate records are never consumed).
bool launch_corr_tc(const SolveParams& p, const Work& w, cudaStream_t s);
// Same kernel, additionally writing the signed fp32 scores [B][n] (tests).
bool launch_corr_tc_debug(const SolveParams& p, const Work& w, float* scores,
                          cudaStream_t s);
void launch_split_dict(const float* src, __half* hi, __half* lo, int64_t count, float scale,
                       cudaStream_t s);
// Residual fp16 split from r64 (warp per signal; init / unit paths).
void launch_split_resid(const SolveParams& p, const Work& w, cudaStream_t s);
// ---- launchers (k_sep.cu) ----
void launch_sep_corr(const SolveParams& p, const Work& w, const double* r_src,
                     double* dst, bool abs_scores, cudaStream_t s);
// Tensor-core variant (th == 1, nr a multiple of the K1 atom tile): stage 1 in
// fp64, its rows split to fp16, stage 2 = K1 with the fused candidate
// records (global atom indices); false when a launch could not be enqueued.
bool launch_sep_corr_tc(const SolveParams& p, const Work& w, cudaStream_t s);
void launch_sep_resid(const SolveParams& p, const Work& w, int outer, int tb,
                      cudaStream_t s);
// All epochs of one outer iteration in direct form (no support Gram matrix);
// bound: upper bound on the support sizes.  Returns the kernels launched.
int launch_sep_direct_learn(const SolveParams& p, const Work& w, int outer, int bound,
                            cudaStream_t s);
// Once per solve, before the first direct-form iteration: Z2 = Y A_c.
void launch_sep_direct_prepare(const SolveParams& p, const Work& w, cudaStream_t s);
int64_t sep_resid_tiles(const SolveParams& p);

// ---- launchers (k_gram.cu) ----
void launch_gram_full(const float* at, int64_t n, int64_t ldm, double* g,
                      cudaStream_t s);

// fp32 -> fp64 (exact).  The hardware F2F.F64.F32 keeps pace with DFMA on
// sm_100a (tools/micro/cvt.cu: ~61 conversions per SM-cycle); integer
// bit-assembly with special-case selects measured 10x slower.
__device__ __forceinline__ double f2d(float f) { return (double)f; }

// ---- optimizer steps (gradient_step, clomp.cpp:171-209), shared by k_solve.cu / k_sep.cu
template <int OPT>
__device__ __forceinline__ void opt_step(double& c, double g, double& m1,
                                         double& m2, double lr, double bc1,
                                         double bc2) {
  if (OPT == 0) {  // plain: s -= lr * g (clomp.cpp:178-181)
    c = __dsub_rn(c, __dmul_rn(lr, g));
  } else if (OPT == 1) {  // momentum (clomp.cpp:182-188)
    m1 = __dadd_rn(__dmul_rn(0.9, m1), g);
    c = __dsub_rn(c, __dmul_rn(lr, m1));
  } else {  // Adam (clomp.cpp:189-206)
    const double b1 = 0.9, b2 = 0.999, tiny = 1e-8;
    m1 = __dadd_rn(__dmul_rn(b1, m1), __dmul_rn(1.0 - b1, g));
    m2 = __dadd_rn(__dmul_rn(b2, m2), __dmul_rn(__dmul_rn(1.0 - b2, g), g));
    const double mhat = __ddiv_rn(m1, bc1);
    const double vhat = __ddiv_rn(m2, bc2);
    c = __dsub_rn(c, __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(sqrt(vhat), tiny)));
  }
}

// ---- launchers (k_solve.cu) ----
void launch_init(const SolveParams& p, const Work& w, const float* y_in,
                 int y_layout, bool y_on_device_signal_major, cudaStream_t s);
void launch_select(const SolveParams& p, const Work& w, bool full_scores,
                   cudaStream_t s);
int launch_learn(const SolveParams& p, const Work& w, int outer, int max_cnt,
                  cudaStream_t s);
void launch_joint_control(const SolveParams& p, const Work& w, int outer,
                          bool init, cudaStream_t s);
void launch_joint_snapshot(const SolveParams& p, const Work& w,
                           cudaStream_t s);
void launch_finalize(const SolveParams& p, const Work& w, int64_t out_cap,
                     int32_t* sup_out, double* coef_out, int32_t* cnt_out,
                     int32_t* iters_out, double* rn_out, uint8_t* conv_out,
                     int32_t* status_out, cudaStream_t s);
// ---- colshard.cu ----
bool nccl_available();
int nccl_unique_id(void* out);
void* nccl_comm_init(int world, int rank, const void* id, std::string* err);
void nccl_comm_destroy(void* comm);
bool nccl_allgather_inplace(void* comm, void* buf, size_t count_per_rank, int bytes_per_elem,
                            int rank, cudaStream_t s);
bool nccl_allreduce_sum_i32(void* comm, int32_t* buf, size_t count, cudaStream_t s);
void launch_cand_exchange(const Cand* g, Cand* cand, int64_t B, int64_t ntl, int world,
                          int64_t atoms_per_rank, cudaStream_t s);

// Priors: Gram + H extension for the atoms selected this iteration (before
// the learning kernels), and loss / stopping rules after them.
void launch_prior_ext(const SolveParams& p, const Work& w, cudaStream_t s);
void launch_prior_control(const SolveParams& p, const Work& w, int outer, cudaStream_t s);
// Image mode: the coupled epochs of one outer iteration and the residual /
// prior loss after them (joint control follows).
void launch_image_learn(const SolveParams& p, const Work& w, int outer, cudaStream_t s);
constexpr int kLvCover = 8;  // max windows covering one row / column

// ---- k_synth.cu: x_hat[b][q] = sum_k D[q][sup_k] coef_k from the compact results
void launch_synth(const double* dt, int64_t n, int64_t B, int64_t out_cap, const int32_t* sup,
                  const double* coef, const int32_t* cnt, double* xhat, cudaStream_t s);

// Whole per-signal solve in one persistent block per signal (small problems):
// init, every outer iteration and the result compaction in one kernel.
// y_in: m x B (y_ref) or signal-major B x m.
void launch_solve_fused(const SolveParams& p, const Work& w, const float* y_in, int y_ref,
                        int64_t out_cap, int32_t* sup_out, double* coef_out, int32_t* cnt_out,
                        int32_t* iters_out, double* rn_out, uint8_t* conv_out, int32_t* status_out,
                        cudaStream_t s);
// inject_support unit path: residual already in w.r64 (and split), mask in
// w.maskbits; appends nothing to the learning state.
void launch_inject_finish(const SolveParams& p, const Work& w, cudaStream_t s);

}  // namespace clb
