// clomp_api.cu — host side of the C-ABI (include/clomp_b200.h).
//
// Owns the device copy of the dictionary, the batch workspace and the outer
// loop that sequences the kernels of one CLOMP solve:
//
//   init -> [ corr (K1) -> select (K1c, exact near-tie rescoring) + learn (K2)
//             -> residual + control ]*
//        -> finalize
//
// Validation, error classes and messages follow the reference
// (clomp.cpp:18-30, 131-140, 211-218); there is no CPU compute path.
#include <cuda_runtime.h>

#include <chrono>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/clomp_b200.h"
#include "clomp_internal.cuh"

using namespace clb;

namespace {

thread_local std::string g_create_error;

constexpr int64_t kTieSlack = 16;

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Carver {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    off = align_up(off, 256);
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += count * sizeof(T);
    return p;
  }
};

#ifndef CL_CHUNK_ITERS
#define CL_CHUNK_ITERS 16
#endif
constexpr int kChunkIters = CL_CHUNK_ITERS;  // outer iterations per captured graph

// The fused small solve is one kernel (init, iterations, result compaction),
// launched as a cached one-node graph.  Keyed by everything the node reads.
struct FusedGraphKey {
  unsigned char p[sizeof(SolveParams)];
  unsigned char w[sizeof(Work)];
  const void* y = nullptr;
  int layout_ref = 0;
  const void* out[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int64_t out_cap = 0;
  cudaStream_t stream = nullptr;
  bool operator==(const FusedGraphKey& o) const { return std::memcmp(this, &o, sizeof(*this)) == 0; }
};

struct GraphKey {
  SolveParams p{};
  Work w{};  // every device pointer a captured kernel reads
  const void* wbuf = nullptr;
  bool tensor = false, full = false, gemv = false;
  cudaStream_t stream = nullptr;
  bool operator==(const GraphKey& o) const {
    return std::memcmp(&p, &o.p, sizeof(p)) == 0 && std::memcmp(&w, &o.w, sizeof(w)) == 0 &&
           wbuf == o.wbuf && tensor == o.tensor && gemv == o.gemv &&
           full == o.full && stream == o.stream;
  }
};

}  // namespace

struct cl_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;      // stream all work is issued on
  cudaStream_t own_stream = nullptr;  // created by cl_create
  int64_t m = 0, n = 0, ldm = 0;
  float* at32 = nullptr;
  __half* at_hi = nullptr;   // scaled fp16 split of at32 (tensor path)
  __half* at_lo = nullptr;
  float a_scale = 1.0f;      // its power-of-two scale
  double* gfull = nullptr;  // A^T A fp64 [n][n], built once (k_gram.cu)
  // synthesis basis for the priors (cl_set_basis): Delta D atom-major,
  // ddt[j][q] = D[q][j] - D[q+1][j] (q < n - 1), fp64, row stride ldd
  double* ddt = nullptr;
  int64_t ldd = 0;
  double* dt = nullptr;         // the basis atom-major (dt[k][q] = D[q][k]), image mode
  std::vector<double> prior_w;  // this call's per-signal TV weights (empty: off)
  // this call's image-mode priors (multi-column joint batch): batch-global
  // weights and the local-variance window layout
  bool img = false;
  double img_wtv = 0.0, img_wlv = 0.0;
  bool img_lv = false;
  int img_window = 0, img_stride = 0;
  std::vector<int32_t> lv_rows, lv_cols, lv_rowcov, lv_colcov;
  int32_t* lv_tab = nullptr;  // device copy of the four tables
  size_t lv_tab_bytes = 0;
  // separable 2D contexts (cl_create_sep)
  bool sep = false;
  int64_t mr = 0, nr = 0, mc = 0, nc = 0, ldr = 0, ldc = 0;
  float* at_r32 = nullptr;
  float* at_c32 = nullptr;
  double* at_r64 = nullptr;
  double* at_c64 = nullptr;
  double* gr = nullptr;
  double* gc = nullptr;
  double colnorm_max = 0.0;
  std::string err;
  // batch workspace
  void* wbuf = nullptr;
  size_t wbytes = 0;
  Work w;
  // Adam bias-correction tables
  double* bc = nullptr;
  size_t bc_len = 0;
  // host-call staging: two slots, so cl_submit of batch i + 1 can copy its y
  // in while batch i solves and batch i's results copy out while i + 1 solves
  struct Slot {
    char* d_stage = nullptr;   // device: y, then the compact results
    size_t d_bytes = 0;
    char* h_io = nullptr;      // pinned host: compact results (+ a pageable y staged)
    size_t h_bytes = 0;
    cudaEvent_t ev_in = nullptr, ev_solve = nullptr, ev_out = nullptr;
    bool busy = false;
    int64_t batch = 0, cap = 0;
    size_t ybytes = 0, out_bytes = 0;
    int mode = 0;
    bool fused = false;
    bool xhat = false;  // x_hat = D s was formed and downloaded with the results
    std::chrono::steady_clock::time_point t_start;
  };
  Slot slot[2];
  int slot_head = 0;     // next slot cl_submit fills
  int slot_inflight = 0; // submitted and not yet waited (0..2)
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  int32_t* h_counters = nullptr;  // pinned
  int32_t* h_chunk = nullptr;     // pinned, 2 x kNumCounters (graph chunks)
  cudaEvent_t chunk_ev[2] = {nullptr, nullptr};
  GraphKey gkey;
  std::vector<cudaGraphExec_t> graphs;
  std::vector<std::pair<FusedGraphKey, cudaGraphExec_t>> fused_graphs;  // a few (two staging slots)
  int corr_force = 0;
  bool want_xhat = false;  // cl_set_synthesis
  int direct_mode = -1;  // separable direct-form learning: -1 auto, 0 off, k > 0 from iteration k
  bool fused_ok = true;  // small problems: one persistent block per signal
  int cluster_learn = 1;  // supports of 33..256 atoms on CTA clusters (0: block kernel)
  int power_levels = -1;  // plain GD on cluster-sized supports: squaring levels (-1 auto, 0 off)
  double* pw_buf = nullptr;  // power-form buffers (Work::pw_t / pw_d)
  size_t pw_bytes = 0;
  // column sharding (cl_create_colshard); vshards emulates W shards on one GPU
  int rank = 0, world = 1, vshards = 1;
  void* comm = nullptr;
  bool profiling = false;
  cl_stats stats{};
  int sms = 148;
  bool tc_ok = false;
};

namespace {

int fail(cl_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

int cuda_fail(cl_ctx* ctx, cudaError_t e, const char* where) {
  std::string msg = std::string("CUDA error in ") + where + ": " +
                    cudaGetErrorString(e);
  cudaGetLastError();
  return fail(ctx, CL_ERR_CUDA, msg);
}

#define CL_CUDA(ctx, call)                                   \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
  } while (0)

int validate(cl_ctx* ctx, const cl_config* c) {
  if (!c) return fail(ctx, CL_ERR_CONFIG, "clomp: null config");
  if (!(c->th > 0.0) || c->th > 1.0)
    return fail(ctx, CL_ERR_CONFIG, "clomp: th must be in (0, 1]");
  if (c->max_outer == 0) return fail(ctx, CL_ERR_CONFIG, "clomp: max_outer must be >= 1");
  if (c->eps < 0.0) return fail(ctx, CL_ERR_CONFIG, "clomp: eps must be non-negative");
  if (c->inner_steps == 0)
    return fail(ctx, CL_ERR_CONFIG, "clomp: inner_steps must be >= 1");
  if (!(c->lr > 0.0)) return fail(ctx, CL_ERR_CONFIG, "clomp: lr must be positive");
  if (c->stall_tol < 0.0)
    return fail(ctx, CL_ERR_CONFIG, "clomp: stall_tol must be non-negative");
  if (c->stall_patience == 0)
    return fail(ctx, CL_ERR_CONFIG, "clomp: stall_patience must be >= 1");
  if (c->opt < 0 || c->opt > 2) return fail(ctx, CL_ERR_CONFIG, "clomp: unknown optimizer");
  if (c->max_outer > (1u << 30) || c->inner_steps > (1u << 30))
    return fail(ctx, CL_ERR_CONFIG, "clomp: iteration counts out of range");
  return CL_OK;
}

// kern::sum_sq as the reference computes it on x86 (the AVX2 dot of
// kernels_avx2.cpp:30-58: 4 x 4 accumulators over 16-wide blocks, a 4-wide
// block loop, pairwise combination, FMA tail), so automatic prior weights
// (resolve_weights, clomp.cpp:131-140) are the reference's bits.
double ref_sum_sq(const double* v, int64_t n) {
  double acc[4][4] = {};
  int64_t i = 0;
  for (; i + 16 <= n; i += 16)
    for (int k = 0; k < 4; ++k)
      for (int l = 0; l < 4; ++l) acc[k][l] = std::fma(v[i + 4 * k + l], v[i + 4 * k + l], acc[k][l]);
  for (; i + 4 <= n; i += 4)
    for (int l = 0; l < 4; ++l) acc[0][l] = std::fma(v[i + l], v[i + l], acc[0][l]);
  double q[4];
  for (int l = 0; l < 4; ++l) q[l] = (acc[0][l] + acc[1][l]) + (acc[2][l] + acc[3][l]);
  double total = (q[0] + q[2]) + (q[1] + q[3]);
  for (; i < n; ++i) total = std::fma(v[i], v[i], total);
  return total;
}

// resolve_weights (clomp.cpp:131-140) and whether loss_impl would run a prior
// (clomp.cpp:93-94: LV only when the batch fits its window).
bool priors_active(const cl_config* c, double mean_sq, int64_t batch, int64_t n) {
  const double auto_w = 0.01 * mean_sq;
  const double w_tv = c->w_tv < 0.0 ? auto_w : c->w_tv;
  const double w_lv = c->w_lv < 0.0 ? auto_w : c->w_lv;
  const bool lv_fits = (uint64_t)batch >= c->lv_window && (uint64_t)n >= c->lv_window;
  return w_tv > 0.0 || (w_lv > 0.0 && lv_fits);
}

// Per-signal support capacity.  th == 1 adds one atom per outer iteration
// except on exact ties (clomp.cpp:49-51 injects every tie), hence the slack.
constexpr int64_t kGramCapMax = 2048;  // largest support with a Gram matrix per signal

int64_t support_cap(const cl_ctx* ctx, const cl_config* c) {
  if (c->th >= 1.0) return std::min<int64_t>(ctx->n, (int64_t)c->max_outer + kTieSlack);
  // th < 1 can select any number of atoms per iteration.  Separable contexts
  // switch to direct-form learning (no Gram matrix), so every atom fits; 1D
  // contexts keep a Gram matrix per signal and stop a signal that outgrows it
  // with CL_ERR_CAPACITY.
  if (ctx->sep) return ctx->n;
  return std::min<int64_t>(ctx->n, kGramCapMax);
}

// First outer iteration that learns in direct form on a separable context
// (launch_sep_direct_learn), 0 = never.  Without a Gram buffer (capacity above
// kGramCapMax) every iteration does; otherwise the Gram form runs while
// streaming G (8 t^2 bytes per epoch) is cheaper than applying the operator
// (two mr x nc x mc fp64 GEMMs per epoch): t^2 < mr nc mc / 16 from the measured
// costs at config 4 (Gram form ~5.3e-12 t^2 s, direct form ~3.4e-13 mr nc mc s
// per image and epoch).  th < 1 has no per-iteration bound on t.
int64_t direct_from(const cl_ctx* ctx, const cl_config* c, int64_t cap) {
  if (!ctx->sep || ctx->direct_mode == 0) return 0;
  if (cap > kGramCapMax) return 1;
  if (ctx->direct_mode > 0) return ctx->direct_mode;
  if (c->th < 1.0) return 0;
  const double tstar = std::sqrt((double)ctx->mr * (double)ctx->nc * (double)ctx->mc / 16.0);
  const int64_t from = std::max<int64_t>(257, (int64_t)tstar + 1);
  return from <= (int64_t)c->max_outer ? from : 0;
}

// Carve the workspace for (B, cap); reallocate only when it grows.
int ensure_workspace(cl_ctx* ctx, int64_t B, int64_t cap, bool need_scores,
                     bool need_split, int64_t ntile, bool need_prior = false,
                     bool need_image = false, bool sep_tc = false, bool with_direct = false) {
  const int64_t ldm = ctx->ldm;
  const int64_t mwords = (ctx->n + 31) / 32;
  auto carve = [&](Carver& cv, Work& w) {
    w.y32 = cv.take<float>(B * ldm);
    w.y64 = cv.take<double>(B * ldm);
    w.r64 = cv.take<double>(B * ldm);
    w.r_hi = need_split ? cv.take<__half>(B * ldm) : nullptr;
    w.r_lo = need_split ? cv.take<__half>(B * ldm) : nullptr;
    w.r_scale = need_split ? cv.take<float>(B) : nullptr;
    w.cand = cv.take<Cand>(B * ntile);
    w.scores = need_scores ? cv.take<double>(B * ctx->n) : nullptr;
    if (ctx->sep) {
      w.zb = cv.take<double>(B * ctx->n);
      w.sep_scratch = cv.take<double>(B * ctx->nc * ctx->mr);
      w.lpart = cv.take<double>(B * (((ctx->mr + 63) / 64) * ((ctx->mc + 63) / 64)));
      if (with_direct) {
        w.sep_scratch2 = cv.take<double>(B * ctx->nc * ctx->mr);
        w.sep_z2 = cv.take<double>(B * ctx->nc * ctx->mr);
        w.csc_ptr = cv.take<int32_t>(B * (ctx->nc + 1));
        w.csc_perm = cv.take<int32_t>(B * cap);
      }
      if (sep_tc) {
        w.u_hi = cv.take<__half>(B * ctx->nc * ctx->ldr);
        w.u_lo = cv.take<__half>(B * ctx->nc * ctx->ldr);
        w.u_scale = cv.take<float>(B * ctx->nc);
        w.u_active = cv.take<int32_t>(B * ctx->nc);
      }
    }
    if (ctx->world > 1 || ctx->vshards > 1) {
      w.xg = cv.take<Cand>(B * ntile);
    }
    w.sup = cv.take<int32_t>(B * cap);
    w.cnt = cv.take<int32_t>(B);
    w.gcnt = cv.take<int32_t>(B);
    w.coef = cv.take<double>(B * cap);
    w.mom1 = cv.take<double>(B * cap);
    w.mom2 = cv.take<double>(B * cap);
    w.gram = cap <= kGramCapMax ? cv.take<double>(B * cap * cap) : nullptr;
    w.bvec = cv.take<double>(B * cap);
    w.maskbits = cv.take<uint32_t>(B * mwords);
    w.best_coef = cv.take<double>(B * cap);
    w.best_cnt = cv.take<int32_t>(B);
    w.best_L = cv.take<double>(B);
    w.prev_L = cv.take<double>(B);
    w.loss = cv.take<double>(B);
    w.stall = cv.take<int32_t>(B);
    w.iters = cv.take<int32_t>(B);
    w.active = cv.take<int32_t>(B);
    w.conv = cv.take<uint8_t>(B);
    w.status = cv.take<int32_t>(B);
    w.changed = cv.take<int32_t>(B);
    w.big_list = cv.take<int32_t>(B);
    w.counters = cv.take<int32_t>(kNumCounters);
    w.joint = cv.take<double>(kNumJoint);
    if (need_prior) {
      w.hgram = cv.take<double>(B * cap * cap);
      w.wtv = cv.take<double>(B);
      w.rloss = cv.take<double>(B);
      w.best_R = cv.take<double>(B);
    }
    if (need_image) {
      const int64_t nwin = (int64_t)ctx->lv_rows.size() * (int64_t)ctx->lv_cols.size();
      w.img_x = cv.take<double>(B * ctx->n);
      w.img_gx = cv.take<double>(B * ctx->n);
      w.img_gd = cv.take<double>(B * cap);
      w.lv_mean = cv.take<double>(std::max<int64_t>(nwin, 1));
      w.lv_scale = cv.take<double>(std::max<int64_t>(nwin, 1));
      w.lv_sd = cv.take<double>(std::max<int64_t>(nwin, 1));
      w.img_part = cv.take<double>(1024);
    }
  };
  Carver probe{nullptr};
  Work tmp;
  carve(probe, tmp);
  const size_t need = probe.off + 256;
  if (need > ctx->wbytes) {
    if (ctx->wbuf) cudaFree(ctx->wbuf);
    ctx->wbuf = nullptr;
    ctx->wbytes = 0;
    cudaError_t e = cudaMalloc(&ctx->wbuf, need);
    if (e != cudaSuccess) {
      return cuda_fail(ctx, e, "workspace allocation");
    }
    ctx->wbytes = need;
  }
  Carver real{static_cast<char*>(ctx->wbuf)};
  Work w;
  carve(real, w);
  w.at32 = ctx->at32;
  w.at_hi = ctx->at_hi;
  w.at_lo = ctx->at_lo;
  w.gfull = ctx->gfull;
  w.at_r64 = ctx->at_r64;
  w.at_c64 = ctx->at_c64;
  w.gr = ctx->gr;
  w.gc = ctx->gc;
  w.ddt = need_prior ? ctx->ddt : nullptr;
  w.ldd = ctx->ldd;
  if (need_image) {
    w.dt = ctx->dt;
    const int32_t* t = ctx->lv_tab;
    w.lv_rows = t;
    w.lv_cols = t + ctx->lv_rows.size();
    w.lv_rowcov = w.lv_cols + ctx->lv_cols.size();
    w.lv_colcov = w.lv_rowcov + ctx->lv_rowcov.size();
  }
  ctx->w = w;
  return CL_OK;
}

int ensure_adam_tables(cl_ctx* ctx, const cl_config* c) {
  if (c->opt != CL_OPT_ADAM) return CL_OK;
  const size_t len = (size_t)c->max_outer * (size_t)c->inner_steps;
  if (len > ctx->bc_len) {
    if (ctx->bc) cudaFree(ctx->bc);
    ctx->bc = nullptr;
    CL_CUDA(ctx, cudaMalloc(&ctx->bc, 2 * len * sizeof(double)));
    ctx->bc_len = len;
  }
  // bc1/bc2 exactly as gradient_step computes them (clomp.cpp:191-195).
  std::vector<double> h(2 * len);
  for (size_t s = 0; s < len; ++s) {
    h[s] = 1.0 - std::pow(0.9, (double)(s + 1));
    h[len + s] = 1.0 - std::pow(0.999, (double)(s + 1));
  }
  CL_CUDA(ctx, cudaMemcpy(ctx->bc, h.data(), 2 * len * sizeof(double),
                          cudaMemcpyHostToDevice));
  return CL_OK;
}

bool use_tensor_path(const cl_ctx* ctx, const cl_config* c) {
  if (c->th < 1.0) return false;
  if (ctx->corr_force == 1) return false;
  return ctx->tc_ok;
}

// Correlation error bound relative to max||a_j|| * ||r||.  fp64 SIMT: a few
// hundred ulps of the dot length covers summation-order differences with the
// reference's sequential FMA (kernels_avx2.cpp:164-236).  3xTF32: see
// DESIGN.md §4 (measured worst error x safety factor).
double delta_for(bool tensor, int64_t ldm) {
  if (!tensor) return 1e-12;
  // 3xTF32: per-product split error ~3*2^-20, plus fp32 accumulation in TMEM
  // (one rounding per 8-wide MMA K step).  Worst-case style bound, checked
  // against measured errors by tests/test_gpu_corr.py.
  return 1e-5 + (double)(ldm / 8) * 1.2e-7;
}

void enqueue_count(const SolveParams& p, const cl_config* c, int mode, int64_t cap,
                   int64_t* per_iter) {
  (void)c;
  if (p.sep)
    *per_iter = 3 + 2 + (cap > 8 ? 2 : 1) + 3 + (mode == CL_MODE_JOINT ? 2 : 0) +
                (p.tile_atoms == corr_tc_tile_atoms() ? 2 : 0);
  else
    *per_iter = 3 + (cap > 8 ? 3 : 2) + (mode == CL_MODE_JOINT ? 2 : 0) + (p.prior ? 3 : 0);
}

struct OutPtrs {
  int64_t cap;
  int32_t* sup;
  double* coef;
  int32_t* cnt;
  int32_t* iters;
  double* rn;
  uint8_t* conv;
  int32_t* status;
};

// The outer loop shared by the host-buffer and device-buffer entry points.
// y_dev: device pointer, layout_ref ? m x B : B x m.
// Power levels of the warp learners' affine form (k_solve.cu epochs_plain):
// E = 2^L q + r epochs cost popcount(r) + q matvec steps, L offset doublings
// and L squarings of T = I - 2 lr G; a squaring on the fp64 tensor cores costs
// about sq[b] matvec steps for a support bucket of 8 (b + 1) atoms (one 8 x 8
// output block at 8 atoms, ten at 32).  CL_SQ_COSTS="c8,c16,c24,c32" overrides.
static void warp_power_levels(int E, int32_t out[4]) {
  int sq[4] = {5, 5, 5, 5};
  if (const char* e = getenv("CL_SQ_COSTS"))
    sscanf(e, "%d,%d,%d,%d", &sq[0], &sq[1], &sq[2], &sq[3]);
  for (int b = 0; b < 4; ++b) {
    int best_l = 0, best = E;
    for (int l = 1; l <= 8; ++l) {
      const int cost = __builtin_popcount((unsigned)(E & ((1 << l) - 1))) + (1 + sq[b]) * l + (E >> l);
      if ((E >> l) >= 1 && cost < best) {
        best = cost;
        best_l = l;
      }
    }
    out[b] = best_l;
  }
}

// host_sync = false (cl_solve_batch): the fused and graph paths return with
// the work queued; the caller's one synchronise after its D2H of the results
// completes them (one host round trip per call instead of two), and it then
// reads the rescan counter (stats.rescans) from the pinned counter copy.
int solve_core(cl_ctx* ctx, const float* y_dev, int layout_ref, int64_t B,
               const cl_config* c, int mode, const OutPtrs& out, bool host_sync = true) {
  // K1b: a handful of residuals (the CLI's one-signal-at-a-time path) makes
  // the correlation an HBM-bound GEMV; auto below 9 signals, or forced (3).
  const bool gemv_fit = !ctx->sep && corr_gemv_supported(ctx->ldm, B);
  if (ctx->corr_force == 3 && !gemv_fit)
    return fail(ctx, CL_ERR_UNSUPPORTED,
                "cl_set_corr_path(3): the GEMV correlation needs 1 <= B <= 8 on a 1D dictionary");
  const bool gemv = gemv_fit && (ctx->corr_force == 0 || ctx->corr_force == 3);
  const bool tensor = !ctx->sep && !gemv && use_tensor_path(ctx, c);
  // separable contexts: stage 2 of the correlation on the tensor cores (K1 on
  // the rows of U = R A_c) with candidate records instead of B x n fp64 scores
  const bool sep_tc = ctx->sep && use_tensor_path(ctx, c);
  if (ctx->sep && ctx->corr_force == 2 && !sep_tc)
    return fail(ctx, CL_ERR_UNSUPPORTED,
                "cl_set_corr_path(2): the separable tcgen05 correlation needs th = 1 and n_r a "
                "multiple of 256");
  const bool full_scores = c->th < 1.0 || (ctx->sep && !sep_tc);
  const int64_t cap = support_cap(ctx, c);
  const int W = ctx->world > 1 ? ctx->world : ctx->vshards;
  const bool colshard = W > 1;
  if (colshard) {
    const int64_t tile = tensor ? corr_tc_tile_atoms() : gemv ? corr_gemv_tile_atoms() : kCorrTileAtoms;
    if (ctx->sep || c->th < 1.0 || mode != CL_MODE_PER_SIGNAL)
      return fail(ctx, CL_ERR_UNSUPPORTED,
                  "column sharding: per-signal mode with th = 1 on 1D dictionaries only");
    if (ctx->n % (W * tile) != 0)
      return fail(ctx, CL_ERR_DIMENSION, "column sharding: n must be a multiple of shards x " +
                                             std::to_string(tile));
    if (ctx->world > 1 && B % ctx->world != 0)
      return fail(ctx, CL_ERR_DIMENSION, "column sharding: batch must divide by the world size");
  }
  const int64_t dfrom = direct_from(ctx, c, cap);
  if (cap > kGramCapMax && dfrom != 1)
    return fail(ctx, CL_ERR_UNSUPPORTED,
                "clomp: more than 2048 atoms per signal (max_outer) needs the direct-form "
                "learner (separable contexts; cl_set_direct_form)");
  // Latency path: the whole solve in one persistent block per signal when the
  // dictionary is small (config 1) and supports stay register-resident.
  const bool image = ctx->img;
  const bool prior = !ctx->prior_w.empty() || image;
  const bool fused = ctx->fused_ok && !ctx->sep && !colshard && !prior &&
                     (mode == CL_MODE_PER_SIGNAL || B == 1) &&
                     cap <= kWarpCap && ctx->n * ctx->ldm <= (int64_t)1 << 22 &&
                     B <= 4 * (int64_t)ctx->sms;
  const int64_t tile_atoms =
      (tensor || sep_tc) ? corr_tc_tile_atoms() : gemv ? corr_gemv_tile_atoms() : kCorrTileAtoms;
  const int64_t ntile = (ctx->n + tile_atoms - 1) / tile_atoms;
  if (image) {  // local-variance window tables -> device
    // (a batch submitted earlier may still read the tables: cl_submit pipelining)
    CL_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    const size_t cnt = ctx->lv_rows.size() + ctx->lv_cols.size() + ctx->lv_rowcov.size() +
                       ctx->lv_colcov.size();
    if (cnt * 4 > ctx->lv_tab_bytes) {
      cudaFree(ctx->lv_tab);
      ctx->lv_tab = nullptr;
      CL_CUDA(ctx, cudaMalloc(&ctx->lv_tab, std::max<size_t>(cnt, 1) * 4));
      ctx->lv_tab_bytes = std::max<size_t>(cnt, 1) * 4;
    }
    std::vector<int32_t> all;
    for (auto* v : {&ctx->lv_rows, &ctx->lv_cols, &ctx->lv_rowcov, &ctx->lv_colcov})
      all.insert(all.end(), v->begin(), v->end());
    if (!all.empty())
      CL_CUDA(ctx, cudaMemcpy(ctx->lv_tab, all.data(), all.size() * 4, cudaMemcpyHostToDevice));
  }
  int st = ensure_workspace(ctx, B, cap, full_scores || fused, tensor && !fused, ntile,
                            prior && !image, image, sep_tc, dfrom > 0);
  if (st) return st;
  if (prior && !image)
    CL_CUDA(ctx, cudaMemcpyAsync(ctx->w.wtv, ctx->prior_w.data(), (size_t)B * sizeof(double),
                                 cudaMemcpyHostToDevice, ctx->stream));
  st = ensure_adam_tables(ctx, c);
  if (st) return st;

  SolveParams p{};
  p.B = B;
  p.n = ctx->n;
  p.m = ctx->m;
  p.ldm = ctx->ldm;
  p.cap = cap;
  p.ntile = ntile;
  p.tile_atoms = tile_atoms;
  p.sig_lo = 0;
  p.sig_hi = B;
  p.atom0 = 0;
  p.n_corr = ctx->n;
  p.ntl = ntile;
  if (colshard) {
    p.n_corr = ctx->n / W;
    p.ntl = p.n_corr / tile_atoms;
    if (ctx->world > 1) {
      p.sig_lo = (int64_t)ctx->rank * (B / ctx->world);
      p.sig_hi = p.sig_lo + B / ctx->world;
    }
  }
  p.mwords = (ctx->n + 31) / 32;
  p.th = c->th;
  p.eps = c->eps;
  p.lr = c->lr;
  p.stall_tol = c->stall_tol;
  p.stall_patience = (int32_t)std::min<uint64_t>(c->stall_patience, 1u << 30);
  p.opt = c->opt;
  p.inner = (int32_t)c->inner_steps;
  warp_power_levels(p.inner, p.warp_L);
  p.max_outer = (int32_t)c->max_outer;
  // A one-column joint solve is exactly clomp_solve (clomp.cpp:294-311), so
  // the fused path runs everything with per-signal state.
  p.mode = (fused || (prior && !image && B == 1)) ? CL_MODE_PER_SIGNAL : mode;
  p.prior = image ? 2 : prior ? 1 : 0;
  p.w_tv_g = ctx->img_wtv;
  p.w_lv_g = ctx->img_wlv;
  p.lv_on = image && ctx->img_lv ? 1 : 0;
  p.lv_window = ctx->img_window;
  p.lv_stride = ctx->img_stride;
  p.lv_nr = (int32_t)ctx->lv_rows.size();
  p.lv_nc = (int32_t)ctx->lv_cols.size();
  p.bc1 = ctx->bc;
  p.bc2 = ctx->bc ? ctx->bc + ctx->bc_len : nullptr;
  p.delta_rel = delta_for(tensor || sep_tc, sep_tc ? ctx->ldr : ctx->ldm);
  p.colnorm_max = ctx->colnorm_max;
  p.a_inv_scale = 1.0 / (double)ctx->a_scale;
  p.sep = ctx->sep ? 1 : 0;
  p.nr = ctx->nr;
  p.nc = ctx->nc;
  p.mr = ctx->mr;
  p.mc = ctx->mc;
  p.ldr = ctx->ldr;
  p.ldc = ctx->ldc;
  // th == 1: the selection (K1c, near-tie rescoring included) runs at the top
  // of the learning kernel, one warp per signal, instead of its own launch.
  p.fuse_select = (!full_scores && !p.sep && !prior) ? 1 : 0;
  p.cluster_learn = ctx->cluster_learn;
  // Power form for the cluster-learned supports (plain GD only: momentum and
  // Adam are not affine in c).  Auto: L = 3 (E = 200 -> 25 steps of T^8).
  {
    const int64_t nsig = p.sig_hi - p.sig_lo;
    int L = ctx->power_levels < 0 ? 3 : ctx->power_levels;
    while (L > 0 && ((int64_t)1 << L) > (int64_t)c->inner_steps) --L;
    const bool use = L > 0 && c->opt == CL_OPT_PLAIN && !prior && !ctx->sep &&
                     ctx->cluster_learn == 1 && cap > kWarpCap;
    if (use) {
      const int64_t ld = std::min<int64_t>(256, (cap + 63) / 64 * 64);
      // big-list slots with power buffers (signals past them learn per epoch);
      // CL_PW_MAX_SLOTS lowers the cap (tests exercise the overflow path)
      const char* env_slots = getenv("CL_PW_MAX_SLOTS");
      const int64_t max_slots = env_slots ? std::max<int64_t>(1, atoll(env_slots)) : 1024;
      const int64_t slots = std::min<int64_t>(nsig, max_slots);
      const int64_t nchunk = (ctx->ldm + 511) / 512;  // k_pw_resid row chunks
      const size_t bytes =
          (size_t)(2 * slots * (ld * ld + ld) + slots * nchunk) * sizeof(double) +
          (size_t)slots * sizeof(int32_t);
      if (bytes > ctx->pw_bytes) {
        if (ctx->pw_buf) cudaFree(ctx->pw_buf);
        ctx->pw_buf = nullptr;
        ctx->pw_bytes = 0;
        CL_CUDA(ctx, cudaMalloc(&ctx->pw_buf, bytes));
        CL_CUDA(ctx, cudaMemset(ctx->pw_buf, 0, bytes));  // chunk counters start at 0
        ctx->pw_bytes = bytes;
      }
      ctx->w.pw_t = ctx->pw_buf;
      ctx->w.pw_d = ctx->pw_buf + 2 * slots * ld * ld;
      ctx->w.pw_part = ctx->w.pw_d + 2 * slots * ld;
      ctx->w.pw_cnt = reinterpret_cast<int32_t*>(ctx->w.pw_part + slots * nchunk);
      p.pw_levels = L;
      p.pw_q = (int32_t)(c->inner_steps >> L);
      p.pw_r = (int32_t)(c->inner_steps & ((1u << L) - 1));
      p.pw_slots = (int32_t)slots;
      p.pw_ld = (int32_t)ld;
    } else {
      ctx->w.pw_t = ctx->w.pw_d = ctx->w.pw_part = nullptr;
      ctx->w.pw_cnt = nullptr;
    }
  }
  const Work& w = ctx->w;
  cudaStream_t s = ctx->stream;
  cl_stats stats{};
  stats.corr_path = (tensor || sep_tc) ? 1 : gemv ? 3 : 0;

  // One outer iteration (clomp.cpp:235-274): counters reset, K1, K1c (with
  // exact fp64 rescoring of near-ties; fused into the learning kernel when
  // th == 1), learning + residual + stopping rules.  th == 1 adds one atom per
  // iteration, so the learning kernel's support bucket follows `outer`
  // (signals grown past it by ties are finished by the block kernel).
  // false once a launch or collective could not be enqueued (tensor-map
  // encode, cudaLaunchKernelEx, NCCL): the call fails with CL_ERR_CUDA.
  bool enq_ok = true;
  auto enqueue_iteration = [&](int outer, int64_t* launches) {
    // (the active count is cleared by the learning kernel, see k_learn_warp)
    if (p.sep) {
      if (sep_tc) {
        enq_ok &= launch_sep_corr_tc(p, w, s);
        launch_select(p, w, false, s);
        *launches += 2;  // + the row split and the record index fix-up
      } else {
        launch_sep_corr(p, w, w.r64, w.scores, true, s);
        launch_select(p, w, true, s);
      }
      const int bound = c->th >= 1.0 ? (int)std::min<int64_t>(cap, outer + kTieSlack) : (int)cap;
      if (dfrom > 0 && outer >= dfrom) {
        SolveParams pd = p;
        pd.direct = 1;
        *launches += launch_sep_direct_learn(pd, w, outer, bound, s);
        launch_sep_resid(pd, w, outer, bound, s);
        *launches += 3 + 2 + 3;
      } else {
        launch_learn(p, w, outer, c->th >= 1.0 ? outer : (int)cap, s);
        launch_sep_resid(p, w, outer, bound, s);
        *launches += 3 + 2 + (cap > 8 ? 2 : 1) + 3;
      }
      if (mode == CL_MODE_JOINT) {
        launch_joint_control(p, w, outer, false, s);
        launch_joint_snapshot(p, w, s);
        *launches += 2;
      }
      return;
    }
    if (colshard) {
      // K1 per column shard into [W][B][ntl], exchange, then global tiles.
      const int r0 = ctx->world > 1 ? ctx->rank : 0, r1 = ctx->world > 1 ? ctx->rank + 1 : W;
      for (int r = r0; r < r1; ++r) {
        SolveParams pk = p;
        pk.atom0 = (int64_t)r * p.n_corr;
        Work wk = w;
        wk.cand = w.xg + (int64_t)r * B * p.ntl;
        if (tensor)
          enq_ok &= launch_corr_tc(pk, wk, s);
        else if (gemv)
          launch_corr_gemv(pk, wk, false, s);
        else
          launch_corr_f64(pk, wk, false, s);
        ++*launches;
      }
      if (ctx->world > 1) {
        const size_t cnt = (size_t)(B * p.ntl);
        enq_ok &= nccl_allgather_inplace(ctx->comm, w.xg, cnt * sizeof(Cand), 1, ctx->rank, s);
      }
      launch_cand_exchange(w.xg, w.cand, B, p.ntl, W, p.n_corr, s);
      *launches += launch_learn(p, w, outer, outer, s);  // selection fused (p.fuse_select)
      *launches += 1 + (cap > 8 ? 3 : 2);
      if (ctx->world > 1) {
        const size_t rows = (size_t)((p.sig_hi - p.sig_lo) * p.ldm);
        if (w.r_hi) {
          enq_ok &= nccl_allgather_inplace(ctx->comm, w.r_hi, rows * sizeof(__half), 1, ctx->rank, s);
          enq_ok &= nccl_allgather_inplace(ctx->comm, w.r_lo, rows * sizeof(__half), 1, ctx->rank, s);
          enq_ok &= nccl_allgather_inplace(ctx->comm, w.r_scale, (size_t)(p.sig_hi - p.sig_lo), 4,
                                           ctx->rank, s);
        } else {
          enq_ok &= nccl_allgather_inplace(ctx->comm, w.r64, rows, 8, ctx->rank, s);
        }
        enq_ok &= nccl_allreduce_sum_i32(ctx->comm, &w.counters[active_slot(outer)], 1, s);
      }
      return;
    }
    if (tensor) {
      enq_ok &= launch_corr_tc(p, w, s);
    } else if (gemv)
      launch_corr_gemv(p, w, full_scores, s);
    else
      launch_corr_f64(p, w, full_scores, s);
    if (!p.fuse_select) launch_select(p, w, full_scores, s);
    if (p.prior) launch_prior_ext(p, w, s);
    const int bound = c->th >= 1.0 ? outer : (int)cap;
    if (p.prior == 2) {  // image mode: coupled epochs, residual, prior loss
      launch_image_learn(p, w, outer, s);
      *launches += 2 + (int64_t)p.inner * (p.lv_on ? 4 : 3) + 3 + p.lv_on;
    } else {
      *launches += launch_learn(p, w, outer, bound, s);
      if (p.prior) launch_prior_control(p, w, outer, s);
      *launches += (p.fuse_select ? 1 : 2) + (cap > 8 ? 3 : 2) + (p.prior ? 2 : 0);
    }
    if (mode == CL_MODE_JOINT) {
      launch_joint_control(p, w, outer, false, s);
      launch_joint_snapshot(p, w, s);
      *launches += 2;
    }
  };

  int64_t launches = 0;
  if (fused) {
    FusedGraphKey key;
    std::memset(&key, 0, sizeof(key));
    std::memcpy(key.p, &p, sizeof(p));
    std::memcpy(key.w, &w, sizeof(w));
    key.y = y_dev;
    key.layout_ref = layout_ref;
    const void* optr[7] = {out.sup, out.coef, out.cnt, out.iters, out.rn, out.conv, out.status};
    std::memcpy(key.out, optr, sizeof(optr));
    key.out_cap = out.cap;
    key.stream = s;
    cudaGraphExec_t ge = nullptr;
    for (auto& kv : ctx->fused_graphs)
      if (kv.first == key) ge = kv.second;
    if (!ge) {
      cudaGraph_t g = nullptr;
      CL_CUDA(ctx, cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
      launch_solve_fused(p, w, y_dev, layout_ref ? 1 : 0, out.cap, out.sup, out.coef, out.cnt,
                         out.iters, out.rn, out.conv, out.status, s);
      CL_CUDA(ctx, cudaStreamEndCapture(s, &g));
      CL_CUDA(ctx, cudaGraphInstantiate(&ge, g, 0));
      cudaGraphDestroy(g);
      if (ctx->fused_graphs.size() >= 8) {  // callers cycling through many buffers
        cudaGraphExecDestroy(ctx->fused_graphs.front().second);
        ctx->fused_graphs.erase(ctx->fused_graphs.begin());
      }
      ctx->fused_graphs.emplace_back(key, ge);
    }
    CL_CUDA(ctx, cudaGraphLaunch(ge, s));
    launches += 1;
    CL_CUDA(ctx, cudaGetLastError());
    if (host_sync) CL_CUDA(ctx, cudaStreamSynchronize(s));
    stats.kernel_launches = launches;
    stats.rescans = 0;
    stats.outer_iterations = p.max_outer;
    stats.corr_path = 2;
    ctx->stats = stats;
    return CL_OK;
  }
  CL_CUDA(ctx, cudaMemsetAsync(w.counters, 0, kNumCounters * sizeof(int32_t), s));
  std::memset(ctx->h_counters, 0, kNumCounters * sizeof(int32_t));
  launch_init(p, w, y_dev, layout_ref ? 0 : 1, false, s);
  launches += (layout_ref && p.B > 1) ? 2 : 1;  // + the tiled transpose of m x B y
  if (p.sep) {  // b values of every atom: Z = A_r^T Y A_c
    launch_sep_corr(p, w, w.y64, w.zb, false, s);
    launches += 2;
    if (dfrom > 0) {  // direct form: the constant part of U = R A_c
      launch_sep_direct_prepare(p, w, s);
      ++launches;
    }
  }
  if (p.mode == CL_MODE_JOINT) {
    launch_joint_control(p, w, 0, true, s);
    ++launches;
  }
  int outer_done = 0;
  if (ctx->profiling) {
    // Per-phase CUDA-event timing (outside the graph path).
    cudaEvent_t ev[5];
    for (auto& e : ev) cudaEventCreate(&e);
    cudaEventRecord(ev[0], s);
    for (int outer = 1; outer <= p.max_outer; ++outer) {
      if (p.sep) {
        enqueue_iteration(outer, &launches);
        CL_CUDA(ctx, cudaMemcpyAsync(ctx->h_counters, w.counters, kNumCounters * sizeof(int32_t),
                                     cudaMemcpyDeviceToHost, s));
        CL_CUDA(ctx, cudaStreamSynchronize(s));
        outer_done = outer;
        if (ctx->h_counters[active_slot(outer)] == 0) break;
        continue;
      }
      // 1D: events around every phase, the stream synchronised once per
      // chunk of kChunkIters iterations (the active count is checked there),
      // so the kernels run back to back as in the timed graph path.
      const int o1 = std::min(p.max_outer, outer + kChunkIters - 1);
      std::vector<cudaEvent_t> pe((size_t)(4 * (o1 - outer + 1)));
      for (auto& e : pe) cudaEventCreate(&e);
      for (int o = outer; o <= o1; ++o) {
        cudaEvent_t* e = &pe[(size_t)(4 * (o - outer))];
        cudaEventRecord(e[0], s);
        if (tensor)
          enq_ok &= launch_corr_tc(p, w, s);
        else if (gemv)
          launch_corr_gemv(p, w, full_scores, s);
        else
          launch_corr_f64(p, w, full_scores, s);
        cudaEventRecord(e[1], s);
        if (!p.fuse_select) launch_select(p, w, full_scores, s);
        if (p.prior) launch_prior_ext(p, w, s);
        cudaEventRecord(e[2], s);
        if (p.prior == 2) {
          launch_image_learn(p, w, o, s);
        } else {
          launches += launch_learn(p, w, o, c->th >= 1.0 ? o : (int)cap, s);
          if (p.prior) launch_prior_control(p, w, o, s);
        }
        launches += (p.fuse_select ? 1 : 2) + (cap > 8 ? 3 : 2) + (p.prior ? 2 : 0);
        if (mode == CL_MODE_JOINT) {
          launch_joint_control(p, w, o, false, s);
          launch_joint_snapshot(p, w, s);
          launches += 2;
        }
        cudaEventRecord(e[3], s);
      }
      CL_CUDA(ctx, cudaGetLastError());
      if (!enq_ok) return fail(ctx, CL_ERR_CUDA, "clomp: correlation kernel launch failed");
      CL_CUDA(ctx, cudaMemcpyAsync(ctx->h_counters, w.counters, kNumCounters * sizeof(int32_t),
                                   cudaMemcpyDeviceToHost, s));
      CL_CUDA(ctx, cudaStreamSynchronize(s));
      for (int o = outer; o <= o1; ++o) {
        cudaEvent_t* e = &pe[(size_t)(4 * (o - outer))];
        float a = 0.f, b2 = 0.f, c2 = 0.f;
        cudaEventElapsedTime(&a, e[0], e[1]);
        cudaEventElapsedTime(&c2, e[1], e[2]);
        cudaEventElapsedTime(&b2, e[2], e[3]);
        stats.corr_ms += a;
        stats.select_ms += c2;
        stats.learn_ms += b2;
      }
      for (auto& e : pe) cudaEventDestroy(e);
      outer_done = o1;
      outer = o1;
      if (ctx->h_counters[active_slot(o1)] == 0) break;
    }
    launch_finalize(p, w, out.cap, out.sup, out.coef, out.cnt, out.iters, out.rn,
                    out.conv, out.status, s);
    ++launches;
    cudaEventRecord(ev[3], s);
    CL_CUDA(ctx, cudaMemcpyAsync(ctx->h_counters, w.counters, kNumCounters * sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, s));
    CL_CUDA(ctx, cudaStreamSynchronize(s));
    float t = 0.f;
    cudaEventElapsedTime(&t, ev[0], ev[3]);
    stats.total_ms = t;
    for (auto& e : ev) cudaEventDestroy(e);
  } else {
    // Graph path: the iterations are captured in chunks of chunk_iters into
    // CUDA graphs (cached per launch configuration) and replayed back to back.
    // After each chunk the active-signal count is copied to pinned memory; the
    // host checks it one chunk behind, so the GPU never waits for the host.
    // The host sees a finished batch one chunk late, so a solve of at most two
    // chunks runs every iteration anyway: it is captured as ONE graph (no
    // mid-solve counter copy breaking the programmatic-launch chain).
    const int chunk_iters = p.max_outer <= 2 * kChunkIters ? p.max_outer : kChunkIters;
    GraphKey key{};
    key.p = p;
    key.w = w;
    key.wbuf = ctx->wbuf;
    key.tensor = tensor;
    key.gemv = gemv;
    key.full = full_scores;
    key.stream = s;
    if (!(key == ctx->gkey)) {
      for (auto& g : ctx->graphs)
        if (g) cudaGraphExecDestroy(g);
      ctx->graphs.assign(0, nullptr);
      ctx->gkey = key;
    }
    const int nchunks = (p.max_outer + chunk_iters - 1) / chunk_iters;
    if ((int)ctx->graphs.size() < nchunks) ctx->graphs.resize((size_t)nchunks, nullptr);
    // chunks whose iterations learn in direct form launch ~4 kernels per epoch:
    // they are enqueued directly (like the NCCL chunks), not captured
    auto chunk_direct = [&](int ch) {
      return dfrom > 0 && std::min(p.max_outer, (ch + 1) * chunk_iters) >= dfrom;
    };
    for (int ch = 0; ch < nchunks && !colshard; ++ch) {
      if (chunk_direct(ch)) continue;
      if (!ctx->graphs[(size_t)ch]) {
        const int o0 = ch * chunk_iters + 1;
        const int o1 = std::min(p.max_outer, o0 + chunk_iters - 1);
        int64_t dummy = 0;
        cudaGraph_t g = nullptr;
        CL_CUDA(ctx, cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        for (int o = o0; o <= o1; ++o) enqueue_iteration(o, &dummy);
        cudaMemcpyAsync(ctx->h_chunk + (ch & 1) * kNumCounters, w.counters,
                        kNumCounters * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        CL_CUDA(ctx, cudaStreamEndCapture(s, &g));
        if (!enq_ok) {
          cudaGraphDestroy(g);
          return fail(ctx, CL_ERR_CUDA, "clomp: correlation kernel launch failed (capture)");
        }
        cudaGraphExec_t ge = nullptr;
        CL_CUDA(ctx, cudaGraphInstantiate(&ge, g, 0));
        cudaGraphDestroy(g);
        ctx->graphs[(size_t)ch] = ge;
      }
    }
    int64_t per_iter = 0;
    enqueue_count(p, c, mode, cap, &per_iter);
    for (int ch = 0; ch < nchunks; ++ch) {
      if (colshard || chunk_direct(ch)) {  // NCCL / direct-form epochs inside: not captured
        const int o0 = ch * chunk_iters + 1;
        const int o1c = std::min(p.max_outer, o0 + chunk_iters - 1);
        int64_t dummy = 0;
        for (int o = o0; o <= o1c; ++o) enqueue_iteration(o, &dummy);
        if (!enq_ok) return fail(ctx, CL_ERR_CUDA, "clomp: launch or collective failed");
        if (!colshard) launches += dummy - per_iter * (o1c - o0 + 1);  // counted below at per_iter
        cudaMemcpyAsync(ctx->h_chunk + (ch & 1) * kNumCounters, w.counters,
                        kNumCounters * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
      } else {
        CL_CUDA(ctx, cudaGraphLaunch(ctx->graphs[(size_t)ch], s));
      }
      cudaEventRecord(ctx->chunk_ev[ch & 1], s);
      const int o1 = std::min(p.max_outer, (ch + 1) * chunk_iters);
      launches += per_iter * (o1 - ch * chunk_iters);
      outer_done = o1;
      if (ch >= 1) {
        CL_CUDA(ctx, cudaEventSynchronize(ctx->chunk_ev[(ch - 1) & 1]));
        const int o_prev = std::min(p.max_outer, ch * chunk_iters);  // last iteration of chunk ch - 1
        if (ctx->h_chunk[((ch - 1) & 1) * kNumCounters + active_slot(o_prev)] == 0) break;
      }
    }
    launch_finalize(p, w, out.cap, out.sup, out.coef, out.cnt, out.iters, out.rn,
                    out.conv, out.status, s);
    ++launches;
    if (colshard && ctx->world > 1) {  // every rank returns the whole batch
      const size_t ns = (size_t)(p.sig_hi - p.sig_lo);
      bool ok = true;
      if (out.sup) ok &= nccl_allgather_inplace(ctx->comm, out.sup, ns * out.cap, 4, ctx->rank, s);
      if (out.coef) ok &= nccl_allgather_inplace(ctx->comm, out.coef, ns * out.cap, 8, ctx->rank, s);
      if (out.cnt) ok &= nccl_allgather_inplace(ctx->comm, out.cnt, ns, 4, ctx->rank, s);
      if (out.iters) ok &= nccl_allgather_inplace(ctx->comm, out.iters, ns, 4, ctx->rank, s);
      if (out.rn) ok &= nccl_allgather_inplace(ctx->comm, out.rn, ns, 8, ctx->rank, s);
      if (out.conv) ok &= nccl_allgather_inplace(ctx->comm, out.conv, ns, 1, ctx->rank, s);
      if (out.status) ok &= nccl_allgather_inplace(ctx->comm, out.status, ns, 4, ctx->rank, s);
      if (!ok) return fail(ctx, CL_ERR_CUDA, "clomp: result all-gather failed");
    }
    CL_CUDA(ctx, cudaGetLastError());
    CL_CUDA(ctx, cudaMemcpyAsync(ctx->h_counters, w.counters, kNumCounters * sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, s));
    if (host_sync) CL_CUDA(ctx, cudaStreamSynchronize(s));
  }
  stats.kernel_launches = launches;
  stats.rescans = ctx->h_counters[kRescanTotal];  // refreshed by the caller if !host_sync
  stats.outer_iterations = outer_done;
  ctx->stats = stats;
  return CL_OK;
}

char* slot_device(cl_ctx* ctx, cl_ctx::Slot& sl, size_t bytes) {
  if (bytes > sl.d_bytes) {
    if (sl.d_stage) {
      cudaStreamSynchronize(ctx->stream);  // the previous solve may still read it
      cudaFree(sl.d_stage);
    }
    sl.d_stage = nullptr;
    sl.d_bytes = 0;
    if (cudaMalloc(&sl.d_stage, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    sl.d_bytes = bytes;
  }
  return sl.d_stage;
}

char* slot_host(cl_ctx::Slot& sl, size_t bytes) {
  if (bytes > sl.h_bytes) {
    if (sl.h_io) cudaFreeHost(sl.h_io);
    sl.h_io = nullptr;
    sl.h_bytes = 0;
    if (cudaMallocHost(&sl.h_io, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    sl.h_bytes = bytes;
  }
  return sl.h_io;
}

bool slot_events(cl_ctx* ctx, cl_ctx::Slot& sl) {
  if (!ctx->copy_in &&
      (cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking) != cudaSuccess ||
       cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking) != cudaSuccess))
    return false;
  if (sl.ev_in) return true;
  return cudaEventCreateWithFlags(&sl.ev_in, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&sl.ev_solve, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&sl.ev_out, cudaEventDisableTiming) == cudaSuccess;
}

}  // namespace

extern "C" {

int cl_abi_version(void) { return CL_ABI_VERSION; }

void cl_abi_struct_sizes(int64_t out[4]) {
  if (!out) return;
  out[0] = (int64_t)sizeof(cl_config);
  out[1] = (int64_t)sizeof(cl_result);
  out[2] = (int64_t)sizeof(cl_device_result);
  out[3] = (int64_t)sizeof(cl_stats);
}

int cl_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void cl_config_default(cl_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->th = 0.7;
  c->max_outer = 200;
  c->eps = 1e-6;
  c->inner_steps = 50;
  c->lr = 0.01;
  c->opt = CL_OPT_ADAM;
  c->w_tv = -1.0;
  c->w_lv = -1.0;
  c->lv_window = 3;
  c->lv_stride = 2;
  c->stall_tol = 1e-4;
  c->stall_patience = 2;
}

const char* cl_last_error(const cl_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

cl_ctx* cl_create(int device, const float* a, int64_t m, int64_t n,
                  int a_layout, int* status) {
  auto bail = [&](int code, const std::string& msg) -> cl_ctx* {
    g_create_error = msg;
    if (status) *status = code;
    return nullptr;
  };
  if (!a || m <= 0 || n <= 0)
    return bail(CL_ERR_DIMENSION, "cl_create: empty or null dictionary");
  if (n > (1LL << 30) || m > (1LL << 30))
    return bail(CL_ERR_DIMENSION, "cl_create: dictionary too large");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return bail(CL_ERR_CUDA, std::string("cl_create: no CUDA device: ") +
                                 cudaGetErrorString(e));
  }
  if (device < 0 || device >= ndev)
    return bail(CL_ERR_CUDA, "cl_create: device index out of range");
  e = cudaSetDevice(device);
  if (e != cudaSuccess)
    return bail(CL_ERR_CUDA, std::string("cl_create: ") + cudaGetErrorString(e));
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  if (prop.major != 10)
    return bail(CL_ERR_CUDA, "cl_create: this build targets sm_100a (B200) only");

  auto* ctx = new cl_ctx();
  ctx->device = device;
  ctx->m = m;
  ctx->n = n;
  ctx->ldm = (m + 127) / 128 * 128;  // float4 x 32 lanes per row chunk
  ctx->sms = prop.multiProcessorCount;
  // Atom-major fp32 copy (the reference's LossOps transpose, clomp.cpp:57-66,
  // done once per dictionary instead of once per call).
  std::vector<float> at((size_t)(n * ctx->ldm), 0.f);
  double cmax = 0.0;
  {
    // 64 x 64 tiles so both the m x n source and the n x ldm destination are
    // walked along cache lines (the plain column walk of a 4096 x 16384
    // dictionary cost ~1.3 s of the config-3 context creation)
    std::vector<double> ss((size_t)n, 0.0);
    constexpr int64_t T = 64;
    const int64_t ldm = ctx->ldm;
    for (int64_t j0 = 0; j0 < n; j0 += T)
      for (int64_t i0 = 0; i0 < m; i0 += T) {
        const int64_t j1 = std::min(n, j0 + T), i1 = std::min(m, i0 + T);
        if (a_layout == CL_LAYOUT_REF) {
          for (int64_t i = i0; i < i1; ++i)
            for (int64_t j = j0; j < j1; ++j) at[(size_t)(j * ldm + i)] = a[i * n + j];
        } else {
          for (int64_t j = j0; j < j1; ++j)
            for (int64_t i = i0; i < i1; ++i) at[(size_t)(j * ldm + i)] = a[j * m + i];
        }
      }
    for (int64_t j = 0; j < n; ++j) {  // ascending-row sums, as before
      double acc = 0.0;
      const float* row = &at[(size_t)(j * ldm)];
      for (int64_t i = 0; i < m; ++i) acc += (double)row[i] * (double)row[i];
      ss[(size_t)j] = acc;
      cmax = std::max(cmax, std::sqrt(acc));
    }
  }
  ctx->colnorm_max = cmax;
  const size_t bytes = at.size() * sizeof(float);
  ctx->tc_ok = corr_tc_available();
  ctx->stream = nullptr;
  if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) == cudaSuccess)
    ctx->stream = ctx->own_stream;
  if (!ctx->stream || cudaMalloc(&ctx->at32, bytes) != cudaSuccess ||
      cudaMemcpy(ctx->at32, at.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMallocHost(&ctx->h_counters, kNumCounters * sizeof(int32_t)) != cudaSuccess ||
      cudaMallocHost(&ctx->h_chunk, 2 * kNumCounters * sizeof(int32_t)) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->chunk_ev[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->chunk_ev[1], cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    cl_destroy(ctx);
    return bail(CL_ERR_CUDA, "cl_create: device allocation failed");
  }
  if (ctx->tc_ok) {
    if (cudaMalloc(&ctx->at_hi, at.size() * sizeof(__half)) != cudaSuccess ||
        cudaMalloc(&ctx->at_lo, at.size() * sizeof(__half)) != cudaSuccess) {
      cudaGetLastError();
      cl_destroy(ctx);
      return bail(CL_ERR_CUDA, "cl_create: device allocation failed");
    }
    // |scale * a| < 2^14 for every entry (max |a| <= ||a||_2 <= colnorm_max)
    ctx->a_scale = split_scale(ctx->colnorm_max * ctx->colnorm_max);
    launch_split_dict(ctx->at32, ctx->at_hi, ctx->at_lo, (int64_t)at.size(), ctx->a_scale,
                      ctx->stream);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
      cudaGetLastError();
      cl_destroy(ctx);
      return bail(CL_ERR_CUDA, "cl_create: tf32 split failed");
    }
  }
  cl_set_gram_cache(ctx, -1);
  if (status) *status = CL_OK;
  return ctx;
}

cl_ctx* cl_create_sep(int device, const float* a_r, int64_t m_r, int64_t n_r,
                      const float* a_c, int64_t m_c, int64_t n_c, int layout,
                      int* status) {
  auto bail = [&](int code, const std::string& msg) -> cl_ctx* {
    g_create_error = msg;
    if (status) *status = code;
    return nullptr;
  };
  if (!a_r || !a_c || m_r <= 0 || n_r <= 0 || m_c <= 0 || n_c <= 0)
    return bail(CL_ERR_DIMENSION, "cl_create_sep: empty or null operator");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return bail(CL_ERR_CUDA, std::string("cl_create_sep: no CUDA device: ") +
                                 cudaGetErrorString(e));
  }
  if (device < 0 || device >= ndev) return bail(CL_ERR_CUDA, "cl_create_sep: bad device");
  cudaSetDevice(device);
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  if (prop.major != 10)
    return bail(CL_ERR_CUDA, "cl_create_sep: this build targets sm_100a (B200) only");
  auto* ctx = new cl_ctx();
  ctx->device = device;
  ctx->sep = true;
  ctx->mr = m_r;
  ctx->nr = n_r;
  ctx->mc = m_c;
  ctx->nc = n_c;
  ctx->m = m_r * m_c;
  ctx->n = n_r * n_c;
  ctx->ldm = (ctx->m + 127) / 128 * 128;
  ctx->ldr = (m_r + 127) / 128 * 128;
  ctx->ldc = (m_c + 127) / 128 * 128;
  ctx->sms = prop.multiProcessorCount;
  // stage 2 of the correlation (A_r^T U) runs on the K1 kernel when its 256-atom
  // tiles line up with the coefficient columns
  ctx->tc_ok = corr_tc_available() && n_r % corr_tc_tile_atoms() == 0;
  auto atom_major = [&](const float* a, int64_t m, int64_t n, int64_t ld,
                        std::vector<float>& f, std::vector<double>& d, double& cmax) {
    f.assign((size_t)(n * ld), 0.f);
    d.assign((size_t)(n * ld), 0.0);
    for (int64_t j = 0; j < n; ++j) {
      double ss = 0.0;
      for (int64_t i = 0; i < m; ++i) {
        const float v = layout == CL_LAYOUT_REF ? a[i * n + j] : a[j * m + i];
        f[(size_t)(j * ld + i)] = v;
        d[(size_t)(j * ld + i)] = v;
        ss += (double)v * v;
      }
      cmax = std::max(cmax, std::sqrt(ss));
    }
  };
  std::vector<float> fr, fc;
  std::vector<double> dr, dc;
  double cr = 0.0, cc = 0.0;
  atom_major(a_r, m_r, n_r, ctx->ldr, fr, dr, cr);
  atom_major(a_c, m_c, n_c, ctx->ldc, fc, dc, cc);
  ctx->colnorm_max = cr * cc;
  bool ok = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) == cudaSuccess;
  ctx->stream = ctx->own_stream;
  ok = ok && cudaMalloc(&ctx->at_r32, fr.size() * 4) == cudaSuccess &&
       cudaMalloc(&ctx->at_c32, fc.size() * 4) == cudaSuccess &&
       cudaMalloc(&ctx->at_r64, dr.size() * 8) == cudaSuccess &&
       cudaMalloc(&ctx->at_c64, dc.size() * 8) == cudaSuccess &&
       cudaMalloc(&ctx->gr, (size_t)(n_r * n_r) * 8) == cudaSuccess &&
       cudaMalloc(&ctx->gc, (size_t)(n_c * n_c) * 8) == cudaSuccess &&
       cudaMemcpy(ctx->at_r32, fr.data(), fr.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(ctx->at_c32, fc.data(), fc.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(ctx->at_r64, dr.data(), dr.size() * 8, cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(ctx->at_c64, dc.data(), dc.size() * 8, cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMallocHost(&ctx->h_counters, kNumCounters * sizeof(int32_t)) == cudaSuccess &&
       cudaMallocHost(&ctx->h_chunk, 2 * kNumCounters * sizeof(int32_t)) == cudaSuccess &&
       cudaEventCreateWithFlags(&ctx->chunk_ev[0], cudaEventDisableTiming) == cudaSuccess &&
       cudaEventCreateWithFlags(&ctx->chunk_ev[1], cudaEventDisableTiming) == cudaSuccess;
  if (ok && ctx->tc_ok) {  // fp16 split of A_r (the K1 dictionary operand)
    ok = cudaMalloc(&ctx->at_hi, fr.size() * sizeof(__half)) == cudaSuccess &&
         cudaMalloc(&ctx->at_lo, fr.size() * sizeof(__half)) == cudaSuccess;
    if (ok) {
      ctx->a_scale = split_scale(cr * cr);
      launch_split_dict(ctx->at_r32, ctx->at_hi, ctx->at_lo, (int64_t)fr.size(), ctx->a_scale,
                        ctx->stream);
    }
  }
  if (ok) {
    // Factor Grams in fp64 on the device (k_gram.cu): Gr = A_r^T A_r, Gc = A_c^T A_c.
    launch_gram_full(ctx->at_r32, n_r, ctx->ldr, ctx->gr, ctx->stream);
    launch_gram_full(ctx->at_c32, n_c, ctx->ldc, ctx->gc, ctx->stream);
    ok = cudaStreamSynchronize(ctx->stream) == cudaSuccess;
  }
  if (!ok) {
    cudaGetLastError();
    cl_destroy(ctx);
    return bail(CL_ERR_CUDA, "cl_create_sep: device allocation failed");
  }
  if (status) *status = CL_OK;
  return ctx;
}

int cl_set_gram_cache(cl_ctx* ctx, int mode) {
  if (!ctx) return CL_ERR_INTERNAL;
  if (ctx->sep) return CL_OK;  // separable contexts use the factor Grams
  cudaSetDevice(ctx->device);
  const size_t bytes = (size_t)ctx->n * (size_t)ctx->n * sizeof(double);
  bool want = mode > 0;
  if (mode < 0) {  // auto: when it fits comfortably
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    want = bytes <= (size_t)8 << 30 && bytes <= free_b / 4;
  }
  if (!want) {
    if (ctx->gfull) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(ctx->gfull);
      ctx->gfull = nullptr;
    }
    ctx->w.gfull = nullptr;
    return CL_OK;
  }
  if (ctx->gfull) return CL_OK;
  if (cudaMalloc(&ctx->gfull, bytes) != cudaSuccess) {
    cudaGetLastError();
    ctx->gfull = nullptr;
    return mode > 0 ? fail(ctx, CL_ERR_CUDA, "cl_set_gram_cache: allocation failed") : CL_OK;
  }
  launch_gram_full(ctx->at32, ctx->n, ctx->ldm, ctx->gfull, ctx->stream);
  CL_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->w.gfull = ctx->gfull;
  return CL_OK;
}

void cl_destroy(cl_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->copy_in) cudaStreamSynchronize(ctx->copy_in);
  if (ctx->copy_out) cudaStreamSynchronize(ctx->copy_out);
  cudaFree(ctx->at32);
  cudaFree(ctx->at_hi);
  cudaFree(ctx->at_lo);
  cudaFree(ctx->gfull);
  cudaFree(ctx->ddt);
  cudaFree(ctx->dt);
  cudaFree(ctx->lv_tab);
  cudaFree(ctx->at_r32);
  cudaFree(ctx->at_c32);
  cudaFree(ctx->at_r64);
  cudaFree(ctx->at_c64);
  cudaFree(ctx->gr);
  cudaFree(ctx->gc);
  cudaFree(ctx->wbuf);
  cudaFree(ctx->pw_buf);
  cudaFree(ctx->bc);
  for (auto& sl : ctx->slot) {
    cudaFree(sl.d_stage);
    if (sl.h_io) cudaFreeHost(sl.h_io);
    for (cudaEvent_t e : {sl.ev_in, sl.ev_solve, sl.ev_out})
      if (e) cudaEventDestroy(e);
  }
  if (ctx->copy_in) cudaStreamDestroy(ctx->copy_in);
  if (ctx->copy_out) cudaStreamDestroy(ctx->copy_out);
  if (ctx->h_counters) cudaFreeHost(ctx->h_counters);
  if (ctx->h_chunk) cudaFreeHost(ctx->h_chunk);
  if (ctx->comm) nccl_comm_destroy(ctx->comm);
  for (auto& e : ctx->chunk_ev)
    if (e) cudaEventDestroy(e);
  for (auto& g : ctx->graphs)
    if (g) cudaGraphExecDestroy(g);
  for (auto& kv : ctx->fused_graphs)
    if (kv.second) cudaGraphExecDestroy(kv.second);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

int cl_set_corr_path(cl_ctx* ctx, int path) {
  if (!ctx) return CL_ERR_INTERNAL;
  if (path < 0 || path > 3) return fail(ctx, CL_ERR_CONFIG, "cl_set_corr_path: 0, 1, 2 or 3");
  if (path == 2 && !corr_tc_available())
    return fail(ctx, CL_ERR_UNSUPPORTED, "tcgen05 correlation kernel not available");
  ctx->corr_force = path;
  return CL_OK;
}

int cl_set_stream(cl_ctx* ctx, void* stream) {
  if (!ctx) return CL_ERR_INTERNAL;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  return CL_OK;
}

int cl_nccl_unique_id(void* id_out) {
  if (!id_out) return CL_ERR_INTERNAL;
  return nccl_unique_id(id_out) == 0 ? CL_OK : CL_ERR_CUDA;
}

cl_ctx* cl_create_colshard(int device, const float* a, int64_t m, int64_t n, int a_layout,
                           int rank, int world, const void* nccl_id, int* status) {
  if (world < 1 || rank < 0 || rank >= world || (world > 1 && !nccl_id)) {
    g_create_error = "cl_create_colshard: bad rank / world / id";
    if (status) *status = CL_ERR_CONFIG;
    return nullptr;
  }
  cl_ctx* ctx = cl_create(device, a, m, n, a_layout, status);
  if (!ctx || world == 1) return ctx;
  std::string err;
  cudaSetDevice(device);
  ctx->comm = nccl_comm_init(world, rank, nccl_id, &err);
  if (!ctx->comm) {
    cl_destroy(ctx);
    g_create_error = "cl_create_colshard: " + err;
    if (status) *status = CL_ERR_CUDA;
    return nullptr;
  }
  ctx->rank = rank;
  ctx->world = world;
  return ctx;
}

int cl_set_virtual_shards(cl_ctx* ctx, int shards) {
  if (!ctx || shards < 1) return CL_ERR_INTERNAL;
  if (ctx->world > 1) return fail(ctx, CL_ERR_CONFIG, "context is already column-sharded");
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->vshards = shards;
  // force a fresh workspace carve with the shard buffers (and fresh power-form
  // buffers: their slot count follows the per-rank signal range)
  cudaFree(ctx->wbuf);
  cudaFree(ctx->pw_buf);
  ctx->wbuf = nullptr;
  ctx->wbytes = 0;
  ctx->pw_buf = nullptr;
  ctx->pw_bytes = 0;
  ctx->w = Work{};
  return CL_OK;
}

int cl_set_fused(cl_ctx* ctx, int on) {
  if (!ctx) return CL_ERR_INTERNAL;
  ctx->fused_ok = on != 0;
  return CL_OK;
}

int cl_set_basis(cl_ctx* ctx, const double* basis, int64_t n, int layout) {
  if (!ctx) return CL_ERR_INTERNAL;
  cudaSetDevice(ctx->device);
  if (ctx->sep)
    return fail(ctx, CL_ERR_UNSUPPORTED, "cl_set_basis: priors on separable contexts are not implemented");
  if (layout != CL_LAYOUT_REF && layout != CL_LAYOUT_T)
    return fail(ctx, CL_ERR_CONFIG, "cl_set_basis: unknown layout");
  cudaFree(ctx->ddt);
  cudaFree(ctx->dt);
  ctx->ddt = nullptr;
  ctx->dt = nullptr;
  ctx->ldd = 0;
  if (!basis) return CL_OK;  // cleared
  if (n != ctx->n)
    return fail(ctx, CL_ERR_DIMENSION, "cl_set_basis: basis is " + std::to_string(n) + " x " +
                                           std::to_string(n) + ", the dictionary has n = " +
                                           std::to_string(ctx->n) + " atoms");
  // Delta D atom-major: row j holds D[q][j] - D[q+1][j], q < n - 1 (fp64,
  // exact differences of the caller's fp64 basis), zero padded to ldd.
  const int64_t ldd = std::max<int64_t>(32, (n - 1 + 31) / 32 * 32);
  std::vector<double> h((size_t)(n * ldd), 0.0);
  auto at = [&](int64_t q, int64_t j) {  // D[q][j]
    return layout == CL_LAYOUT_REF ? basis[q * n + j] : basis[j * n + q];
  };
  for (int64_t j = 0; j < n; ++j)
    for (int64_t q = 0; q + 1 < n; ++q) h[(size_t)(j * ldd + q)] = at(q, j) - at(q + 1, j);
  CL_CUDA(ctx, cudaMalloc(&ctx->ddt, h.size() * sizeof(double)));
  CL_CUDA(ctx, cudaMemcpy(ctx->ddt, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
  ctx->ldd = ldd;
  // the basis itself, atom-major (synthesis x = D s and the chain D^T gx of
  // the image mode)
  h.assign((size_t)(n * n), 0.0);
  for (int64_t k = 0; k < n; ++k)
    for (int64_t q = 0; q < n; ++q) h[(size_t)(k * n + q)] = at(q, k);
  CL_CUDA(ctx, cudaMalloc(&ctx->dt, h.size() * sizeof(double)));
  CL_CUDA(ctx, cudaMemcpy(ctx->dt, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
  return CL_OK;
}

int cl_set_synthesis(cl_ctx* ctx, int on) {
  if (!ctx) return CL_ERR_INTERNAL;
  if (ctx->slot_inflight != 0)
    return fail(ctx, CL_ERR_CONFIG, "cl_set_synthesis: batches are in flight");
  ctx->want_xhat = on != 0;
  return CL_OK;
}

int cl_set_direct_form(cl_ctx* ctx, int from_outer) {
  if (!ctx) return CL_ERR_INTERNAL;
  if (!ctx->sep)
    return fail(ctx, CL_ERR_UNSUPPORTED, "cl_set_direct_form: separable contexts only");
  ctx->direct_mode = from_outer < 0 ? -1 : from_outer;
  return CL_OK;
}

int cl_set_cluster_learn(cl_ctx* ctx, int on) {
  if (!ctx) return CL_ERR_INTERNAL;
  ctx->cluster_learn = on <= 0 ? 0 : 1;
  return CL_OK;
}

int cl_set_power_levels(cl_ctx* ctx, int levels) {
  if (!ctx) return CL_ERR_INTERNAL;
  ctx->power_levels = levels < 0 ? -1 : std::min(levels, 8);
  return CL_OK;
}

int cl_set_profiling(cl_ctx* ctx, int on) {
  if (!ctx) return CL_ERR_INTERNAL;
  ctx->profiling = on != 0;
  return CL_OK;
}

int cl_get_stats(const cl_ctx* ctx, cl_stats* out) {
  if (!ctx || !out) return CL_ERR_INTERNAL;
  *out = ctx->stats;
  return CL_OK;
}

int cl_synchronize(cl_ctx* ctx) {
  if (!ctx) return CL_ERR_INTERNAL;
  cudaSetDevice(ctx->device);
  CL_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return CL_OK;
}

// Priors the B200 path runs: TV-1D (priors.cpp:11-26) on single-column
// solves — clomp_solve on every column (the CLI's 1D path) or a one-column
// batch — folded into the support Gram system (k_prior_ext).  Multi-column
// joint batches (TV-2D + local variance) and separable contexts are
// rejected.  col_ms: mean(y^2) per column (automatic weights).
// block_starts (priors.cpp:63-70): window origins along one axis.
static std::vector<int32_t> block_starts(int64_t dim, int64_t window, int64_t stride) {
  std::vector<int32_t> v;
  for (int64_t s = 0; s + window <= dim; s += stride) v.push_back((int32_t)s);
  const int64_t last = dim - window;
  if (v.empty() || v.back() != last) v.push_back((int32_t)last);
  return v;
}

// Image mode: the priors of a multi-column joint batch (TV-2D + local
// variance on x = D S, batch-global weights; clomp.cpp:93-119, 131-140).
static int setup_image_mode(cl_ctx* ctx, int64_t batch, const cl_config* cfg, double mean_sq,
                            bool have_ms) {
  if (ctx->sep)
    return fail(ctx, CL_ERR_UNSUPPORTED, "clomp: priors on separable contexts are not implemented");
  if (ctx->world > 1 || ctx->vshards > 1)
    return fail(ctx, CL_ERR_UNSUPPORTED, "clomp: priors on column-sharded contexts are not implemented");
  if (!ctx->dt)
    return fail(ctx, CL_ERR_UNSUPPORTED, "clomp: the priors need the synthesis basis (cl_set_basis)");
  if ((cfg->w_tv < 0.0 || cfg->w_lv < 0.0) && !have_ms)
    return fail(ctx, CL_ERR_UNSUPPORTED,
                "cl_solve_batch_device: automatic prior weights need y on the host; pass "
                "explicit w_tv / w_lv");
  const double auto_w = 0.01 * mean_sq;
  const double w_tv = cfg->w_tv < 0.0 ? auto_w : cfg->w_tv;
  const double w_lv = cfg->w_lv < 0.0 ? auto_w : cfg->w_lv;
  const int64_t n = ctx->n, W = (int64_t)cfg->lv_window;
  const bool lv_on = w_lv > 0.0 && batch >= W && n >= W;
  ctx->lv_rows.clear();
  ctx->lv_cols.clear();
  ctx->lv_rowcov.clear();
  ctx->lv_colcov.clear();
  if (lv_on) {  // local_variance's own checks (priors.cpp:77-84)
    if (W < 2) return fail(ctx, CL_ERR_CONFIG, "local_variance: window must be >= 2");
    if (cfg->lv_stride < 1 || cfg->lv_stride >= cfg->lv_window)
      return fail(ctx, CL_ERR_CONFIG, "local_variance: stride must be in [1, window)");
    ctx->lv_rows = block_starts(n, W, (int64_t)cfg->lv_stride);
    ctx->lv_cols = block_starts(batch, W, (int64_t)cfg->lv_stride);
    auto cover = [&](const std::vector<int32_t>& starts, int64_t dim, std::vector<int32_t>& cov) {
      cov.assign((size_t)(dim * kLvCover), -1);
      for (size_t wi = 0; wi < starts.size(); ++wi)
        for (int64_t q = starts[wi]; q < starts[wi] + W; ++q) {
          int32_t* c = &cov[(size_t)(q * kLvCover)];
          int a = 0;
          while (a < kLvCover && c[a] >= 0) ++a;
          if (a == kLvCover) return false;
          c[a] = (int32_t)wi;
        }
      return true;
    };
    if (!cover(ctx->lv_rows, n, ctx->lv_rowcov) || !cover(ctx->lv_cols, batch, ctx->lv_colcov))
      return fail(ctx, CL_ERR_UNSUPPORTED,
                  "local_variance: more than 8 windows cover one pixel (window / stride)");
  }
  ctx->img = true;
  ctx->img_wtv = w_tv > 0.0 ? w_tv : 0.0;
  ctx->img_wlv = lv_on ? w_lv : 0.0;
  ctx->img_lv = lv_on;
  ctx->img_window = (int)W;
  ctx->img_stride = (int)cfg->lv_stride;
  return CL_OK;
}

static int check_call(cl_ctx* ctx, int64_t batch, const cl_config* cfg, int mode,
                      double mean_sq_all, const std::vector<double>* col_ms) {
  ctx->prior_w.clear();
  ctx->img = false;
  int st = validate(ctx, cfg);
  if (st) return st;
  if (!col_ms && (cfg->w_tv < 0.0 || cfg->w_lv < 0.0))
    return fail(ctx, CL_ERR_UNSUPPORTED,
                "cl_solve_batch_device: automatic prior weights (w < 0) need y on the host; "
                "pass explicit w_tv / w_lv");
  if (batch <= 0) return fail(ctx, CL_ERR_DIMENSION, "clomp: empty batch");
  if (mode != CL_MODE_JOINT && mode != CL_MODE_PER_SIGNAL)
    return fail(ctx, CL_ERR_CONFIG, "clomp: unknown solve mode");
  const bool single = mode == CL_MODE_PER_SIGNAL || batch == 1;
  bool pri = false;
  if (!single) {
    pri = priors_active(cfg, mean_sq_all, batch, ctx->n);
  } else if (col_ms) {
    for (double ms : *col_ms) pri = pri || priors_active(cfg, ms, 1, ctx->n);
  } else {
    pri = cfg->w_tv > 0.0 || (cfg->w_lv > 0.0 && cfg->lv_window <= 1);
  }
  if (!pri) return CL_OK;
  if (!single) return setup_image_mode(ctx, batch, cfg, mean_sq_all, col_ms != nullptr);
  if (ctx->sep)
    return fail(ctx, CL_ERR_UNSUPPORTED, "clomp: priors on separable contexts are not implemented");
  if (ctx->world > 1 || ctx->vshards > 1)
    return fail(ctx, CL_ERR_UNSUPPORTED, "clomp: priors on column-sharded contexts are not implemented");
  // local_variance runs on a single column only when its window is < 2,
  // which it rejects (priors.cpp:77-79)
  if (cfg->w_lv != 0.0 && cfg->lv_window <= 1 && (uint64_t)ctx->n >= cfg->lv_window) {
    for (int64_t b = 0; b < batch; ++b) {
      const double w_lv = cfg->w_lv < 0.0 ? 0.01 * (col_ms ? (*col_ms)[(size_t)b] : 0.0) : cfg->w_lv;
      if (w_lv > 0.0) return fail(ctx, CL_ERR_CONFIG, "local_variance: window must be >= 2");
    }
  }
  if (cfg->w_tv == 0.0) return CL_OK;  // only LV was configured: it never runs here
  if (!ctx->ddt)
    return fail(ctx, CL_ERR_UNSUPPORTED,
                "clomp: the TV prior needs the synthesis basis (cl_set_basis)");
  if (cfg->w_tv < 0.0 && !col_ms)
    return fail(ctx, CL_ERR_UNSUPPORTED,
                "cl_solve_batch_device: automatic prior weights need y on the host; pass "
                "an explicit w_tv");
  ctx->prior_w.assign((size_t)batch, cfg->w_tv);
  if (cfg->w_tv < 0.0)
    for (int64_t b = 0; b < batch; ++b) ctx->prior_w[(size_t)b] = 0.01 * (*col_ms)[(size_t)b];
  return CL_OK;
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  const bool ok = cudaPointerGetAttributes(&at, p) == cudaSuccess;
  cudaGetLastError();
  return ok && at.type == cudaMemoryTypeHost;
}

// Pipelined host-buffer solve, first half: validate, copy y to the device on
// the copy-in stream (it overlaps the previous batch still solving), enqueue
// the whole solve on the context stream behind that copy, and the copy of the
// compact results to pinned host memory on the copy-out stream behind the
// solve.  Returns with everything queued (the host only waited for graph
// chunks one behind, see solve_core).
int cl_submit(cl_ctx* ctx, const float* y, int64_t batch, int y_layout,
              const cl_config* cfg, int mode) {
  if (!ctx) return CL_ERR_INTERNAL;
  if (!y && batch > 0) return fail(ctx, CL_ERR_DIMENSION, "clomp: null y");
  if (ctx->slot_inflight >= 2)
    return fail(ctx, CL_ERR_CONFIG, "cl_submit: two batches already in flight; call cl_wait");
  cudaSetDevice(ctx->device);
  cl_ctx::Slot& sl = ctx->slot[ctx->slot_head];
  sl.t_start = std::chrono::steady_clock::now();
  const int64_t m = ctx->m;
  // mean(y^2) for resolve_weights (clomp.cpp:134-136), per batch and per
  // column; only automatic prior weights (w < 0) depend on it.
  std::vector<double> col_ms;
  double all = 0.0;
  if (batch > 0 && cfg && (cfg->w_tv < 0.0 || cfg->w_lv < 0.0)) {
    col_ms.assign((size_t)batch, 0.0);
    std::vector<double> col((size_t)m), rowmajor;
    for (int64_t b = 0; b < batch; ++b) {
      for (int64_t i = 0; i < m; ++i)
        col[(size_t)i] = y_layout == CL_LAYOUT_REF ? y[i * batch + b] : y[b * m + i];
      col_ms[(size_t)b] = ref_sum_sq(col.data(), m) / (double)m;
    }
    // the whole batch in the reference's row-major order (m x B)
    rowmajor.resize((size_t)(m * batch));
    for (int64_t i = 0; i < m; ++i)
      for (int64_t b = 0; b < batch; ++b)
        rowmajor[(size_t)(i * batch + b)] =
            y_layout == CL_LAYOUT_REF ? y[i * batch + b] : y[b * m + i];
    all = ref_sum_sq(rowmajor.data(), m * batch) / (double)(m * batch);
  }
  int st = check_call(ctx, batch, cfg, mode, all, col_ms.empty() ? nullptr : &col_ms);
  if (st) return st;

  const int64_t cap = support_cap(ctx, cfg);
  const size_t ybytes = (size_t)(m * batch) * sizeof(float);
  const bool xhat = ctx->want_xhat && ctx->dt != nullptr;
  const size_t obytes = align_up((size_t)(batch * cap) * 4, 256) +
                        align_up((size_t)(batch * cap) * 8, 256) +
                        4 * align_up((size_t)batch * 8, 256) + 256 +
                        (xhat ? align_up((size_t)(batch * ctx->n) * 8, 256) + 256 : 0);
  if (!slot_events(ctx, sl)) return fail(ctx, CL_ERR_CUDA, "clomp: stream / event creation failed");
  char* stg = slot_device(ctx, sl, align_up(ybytes, 256) + obytes);
  if (!stg) return fail(ctx, CL_ERR_CUDA, "clomp: staging allocation failed");
  float* d_y = reinterpret_cast<float*>(stg);
  Carver cv{stg + align_up(ybytes, 256)};
  OutPtrs o{};
  o.cap = cap;
  o.sup = cv.take<int32_t>(batch * cap);
  o.coef = cv.take<double>(batch * cap);
  o.cnt = cv.take<int32_t>(batch);
  o.iters = cv.take<int32_t>(batch);
  o.rn = cv.take<double>(batch);
  o.conv = cv.take<uint8_t>(batch);
  o.status = cv.take<int32_t>(batch);
  double* d_xhat = xhat ? cv.take<double>(batch * ctx->n) : nullptr;
  const size_t out_bytes = cv.off;  // the compact results (+ x_hat), one D2H copy

  // Host side: pinned caller buffers go straight to the DMA engine; pageable
  // ones are staged through the slot's pinned buffer, which also receives the
  // compact results.
  const bool y_pinned = is_pinned(y);
  char* hio = slot_host(sl, out_bytes + (y_pinned ? 0 : align_up(ybytes, 256)));
  if (!hio) return fail(ctx, CL_ERR_CUDA, "clomp: pinned host staging allocation failed");
  cudaStream_t s = ctx->stream;
  if (y_pinned) {
    CL_CUDA(ctx, cudaMemcpyAsync(d_y, y, ybytes, cudaMemcpyHostToDevice, ctx->copy_in));
  } else {
    char* hy = hio + out_bytes;
    std::memcpy(hy, y, ybytes);
    CL_CUDA(ctx, cudaMemcpyAsync(d_y, hy, ybytes, cudaMemcpyHostToDevice, ctx->copy_in));
  }
  CL_CUDA(ctx, cudaEventRecord(sl.ev_in, ctx->copy_in));
  CL_CUDA(ctx, cudaStreamWaitEvent(s, sl.ev_in, 0));
  st = solve_core(ctx, d_y, y_layout == CL_LAYOUT_REF, batch, cfg, mode, o, false);
  if (st) {
    cudaStreamSynchronize(ctx->copy_in);
    cudaStreamSynchronize(s);
    return st;
  }
  if (xhat) {  // x_hat = D (s .* mask) from the compact results (clomp.cpp:289)
    launch_synth(ctx->dt, ctx->n, batch, cap, o.sup, o.coef, o.cnt, d_xhat, s);
    ++ctx->stats.kernel_launches;
  }
  CL_CUDA(ctx, cudaEventRecord(sl.ev_solve, s));
  CL_CUDA(ctx, cudaStreamWaitEvent(ctx->copy_out, sl.ev_solve, 0));
  CL_CUDA(ctx, cudaMemcpyAsync(hio, stg + align_up(ybytes, 256), out_bytes,
                               cudaMemcpyDeviceToHost, ctx->copy_out));
  CL_CUDA(ctx, cudaEventRecord(sl.ev_out, ctx->copy_out));
  sl.busy = true;
  sl.batch = batch;
  sl.cap = cap;
  sl.ybytes = ybytes;
  sl.out_bytes = out_bytes;
  sl.mode = mode;
  sl.fused = ctx->stats.corr_path == 2;
  sl.xhat = xhat;
  ctx->slot_head ^= 1;
  ++ctx->slot_inflight;
  return CL_OK;
}

// Second half: block until the oldest submitted batch's results are in host
// memory and expand them into the caller's buffers.
int cl_wait(cl_ctx* ctx, cl_result* out) {
  if (!ctx) return CL_ERR_INTERNAL;
  if (ctx->slot_inflight <= 0) return fail(ctx, CL_ERR_CONFIG, "cl_wait: nothing in flight");
  cudaSetDevice(ctx->device);
  cl_ctx::Slot& sl = ctx->slot[(ctx->slot_head + 2 - ctx->slot_inflight) & 1];
  --ctx->slot_inflight;
  sl.busy = false;
  CL_CUDA(ctx, cudaEventSynchronize(sl.ev_out));
  const int64_t batch = sl.batch, cap = sl.cap, n = ctx->n;
  if (!sl.fused) ctx->stats.rescans = ctx->h_counters[kRescanTotal];
  // host views of the compact results (same carving as the device side)
  Carver hv{sl.h_io};
  const int32_t* h_sup = hv.take<int32_t>(batch * cap);
  const double* h_coef = hv.take<double>(batch * cap);
  const int32_t* h_cnt = hv.take<int32_t>(batch);
  const int32_t* h_it = hv.take<int32_t>(batch);
  const double* h_rn = hv.take<double>(batch);
  const uint8_t* h_cv = hv.take<uint8_t>(batch);
  const int32_t* h_st = hv.take<int32_t>(batch);
  const double* h_xh = sl.xhat ? hv.take<double>(batch * n) : nullptr;

  if (out) {
    if (out->x_hat && h_xh) {  // device result is signal-major [B][n]
      if (batch == 1) {
        std::memcpy(out->x_hat, h_xh, sizeof(double) * (size_t)n);
      } else {
        constexpr int64_t T = 32;
        for (int64_t q0 = 0; q0 < n; q0 += T)
          for (int64_t b0 = 0; b0 < batch; b0 += T)
            for (int64_t q = q0; q < std::min(n, q0 + T); ++q)
              for (int64_t b = b0; b < std::min(batch, b0 + T); ++b)
                out->x_hat[q * batch + b] = h_xh[b * n + q];
      }
    }
    const bool prezeroed = (out->flags & CL_RESULT_PREZEROED) != 0;
    if (out->s && !prezeroed) std::memset(out->s, 0, sizeof(double) * (size_t)(n * batch));
    if (out->mask && !prezeroed) std::memset(out->mask, 0, (size_t)(n * batch));
    for (int64_t b = 0; b < batch; ++b) {
      const int cnt = h_cnt[b];
      for (int k = 0; k < cnt; ++k) {
        const int32_t j = h_sup[b * cap + k];
        const double v = h_coef[b * cap + k];
        if (k < out->cap) {
          if (out->support) out->support[b * out->cap + k] = j;
          if (out->coef) out->coef[b * out->cap + k] = v;
        }
        if (out->s) out->s[(int64_t)j * batch + b] = v;
        if (out->mask) out->mask[(int64_t)j * batch + b] = 1;
      }
      // the compact rows are fully written (zeros past the count), so callers
      // may hand in uninitialised buffers
      for (int64_t k = cnt < out->cap ? cnt : out->cap; k < out->cap; ++k) {
        if (out->support) out->support[b * out->cap + k] = 0;
        if (out->coef) out->coef[b * out->cap + k] = 0.0;
      }
      if (out->count) out->count[b] = cnt;
      if (out->iterations) out->iterations[b] = h_it[b];
      if (out->final_residual_norm) out->final_residual_norm[b] = h_rn[b];
      if (out->converged) out->converged[b] = h_cv[b];
      if (out->status) out->status[b] = h_st[b];
    }
  }
  // End to end through submit + wait: host y in, host results out (wall clock;
  // with two batches in flight it includes the time queued behind the other).
  ctx->stats.e2e_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - sl.t_start)
          .count();
  ctx->stats.h2d_bytes = (int64_t)sl.ybytes;
  ctx->stats.d2h_bytes = (int64_t)sl.out_bytes;
  if (out && out->x_hat && !h_xh)
    return fail(ctx, CL_ERR_UNSUPPORTED,
                "clomp: x_hat needs a synthesis basis (cl_set_basis) and cl_set_synthesis(ctx, 1)");
  if (sl.mode == CL_MODE_JOINT && batch > 0 && h_st[0] != CL_OK) {
    return fail(ctx, h_st[0],
                h_st[0] == CL_ERR_NUMERICAL ? "clomp: loss diverged; reduce lr"
                                            : "clomp: support capacity exceeded");
  }
  return CL_OK;
}

int cl_solve_batch(cl_ctx* ctx, const float* y, int64_t batch, int y_layout,
                   const cl_config* cfg, int mode, cl_result* out) {
  if (!ctx) return CL_ERR_INTERNAL;
  if (ctx->slot_inflight != 0)
    return fail(ctx, CL_ERR_CONFIG, "cl_solve_batch: batches submitted with cl_submit are still in flight");
  const int st = cl_submit(ctx, y, batch, y_layout, cfg, mode);
  if (st) return st;
  return cl_wait(ctx, out);
}

int cl_solve_batch_device(cl_ctx* ctx, const float* d_y, int64_t batch,
                          const cl_config* cfg, int mode,
                          const cl_device_result* out) {
  if (!ctx) return CL_ERR_INTERNAL;
  cudaSetDevice(ctx->device);
  // Automatic prior weights need mean(y^2) of host data: the device path
  // takes explicit weights only (check_call).
  int st = check_call(ctx, batch, cfg, mode, 0.0, nullptr);
  if (st) return st;
  if (!out) return fail(ctx, CL_ERR_DIMENSION, "cl_solve_batch_device: null result");
  OutPtrs o{out->cap,  out->support, out->coef, out->count, out->iterations,
            out->final_residual_norm, out->converged, out->status};
  return solve_core(ctx, d_y, 0, batch, cfg, mode, o);
}

int cl_inject_support(cl_ctx* ctx, const double* r, int64_t batch, double th,
                      uint8_t* mask) {
  if (!ctx) return CL_ERR_INTERNAL;
  if (ctx->sep)
    return fail(ctx, CL_ERR_UNSUPPORTED, "inject_support: not available on separable contexts");
  if (!(th > 0.0) || th > 1.0)
    return fail(ctx, CL_ERR_CONFIG, "inject_support: th must be in (0, 1]");
  if (batch <= 0 || !r || !mask)
    return fail(ctx, CL_ERR_DIMENSION, "inject_support: mask size mismatch");
  cudaSetDevice(ctx->device);
  const int64_t m = ctx->m, n = ctx->n, ldm = ctx->ldm;
  const bool full = th < 1.0;
  const int64_t ntile = (n + kCorrTileAtoms - 1) / kCorrTileAtoms;
  int st = ensure_workspace(ctx, batch, n, full, false, ntile);
  if (st) return st;
  SolveParams p{};
  p.B = batch;
  p.n = n;
  p.m = m;
  p.ldm = ldm;
  p.cap = n;
  p.ntile = ntile;
  p.tile_atoms = kCorrTileAtoms;
  p.sig_lo = 0;
  p.sig_hi = batch;
  p.atom0 = 0;
  p.n_corr = n;
  p.ntl = ntile;
  p.mwords = (n + 31) / 32;
  p.th = th;
  p.delta_rel = delta_for(false, ldm);
  p.colnorm_max = ctx->colnorm_max;
  Work w = ctx->w;
  w.r_hi = w.r_lo = nullptr;
  std::vector<double> rt((size_t)(batch * ldm), 0.0);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t b = 0; b < batch; ++b) rt[(size_t)(b * ldm + i)] = r[i * batch + b];
  std::vector<uint32_t> bits((size_t)(batch * p.mwords), 0u);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t b = 0; b < batch; ++b)
      if (mask[j * batch + b]) bits[(size_t)(b * p.mwords + j / 32)] |= 1u << (j % 32);
  cudaStream_t s = ctx->stream;
  CL_CUDA(ctx, cudaMemcpyAsync(w.r64, rt.data(), rt.size() * 8, cudaMemcpyHostToDevice, s));
  CL_CUDA(ctx, cudaMemcpyAsync(w.maskbits, bits.data(), bits.size() * 4,
                               cudaMemcpyHostToDevice, s));
  CL_CUDA(ctx, cudaMemsetAsync(w.counters, 0, kNumCounters * sizeof(int32_t), s));
  launch_inject_finish(p, w, s);
  launch_corr_f64(p, w, full, s);
  launch_select(p, w, full, s);
  CL_CUDA(ctx, cudaGetLastError());
  CL_CUDA(ctx, cudaMemcpyAsync(bits.data(), w.maskbits, bits.size() * 4,
                               cudaMemcpyDeviceToHost, s));
  CL_CUDA(ctx, cudaStreamSynchronize(s));
  for (int64_t j = 0; j < n; ++j)
    for (int64_t b = 0; b < batch; ++b)
      mask[j * batch + b] = (bits[(size_t)(b * p.mwords + j / 32)] >> (j % 32)) & 1u;
  return CL_OK;
}

int cl_debug_cluster_trace(unsigned long long* out) { return cluster_trace(out); }

int cl_debug_learn_trace(unsigned long long* out, int max_signals) {
  return learn_trace(out, max_signals);
}

int cl_debug_k1_trace(unsigned long long* out, int max_ctas) {
  return corr_tc_trace(out, max_ctas);
}

int cl_debug_scores(cl_ctx* ctx, const float* r, int64_t batch, int path,
                    double* scores) {
  if (!ctx || !r || !scores || batch <= 0) return CL_ERR_INTERNAL;
  cudaSetDevice(ctx->device);
  if (path == 2 && !ctx->tc_ok)
    return fail(ctx, CL_ERR_UNSUPPORTED, "tcgen05 correlation kernel not available");
  if (path == 3 && !corr_gemv_supported(ctx->ldm, batch))
    return fail(ctx, CL_ERR_UNSUPPORTED, "GEMV correlation: 1 <= batch <= 4");
  const int64_t m = ctx->m, n = ctx->n, ldm = ctx->ldm;
  const bool tc = path == 2;
  const int64_t tile = tc ? corr_tc_tile_atoms() : path == 3 ? corr_gemv_tile_atoms() : kCorrTileAtoms;
  const int64_t ntile = (n + tile - 1) / tile;
  int st = ensure_workspace(ctx, batch, 1, true, true, ntile);
  if (st) return st;
  SolveParams p{};
  p.B = batch;
  p.n = n;
  p.m = m;
  p.ldm = ldm;
  p.cap = 1;
  p.ntile = ntile;
  p.sig_lo = 0;
  p.sig_hi = batch;
  p.atom0 = 0;
  p.n_corr = n;
  p.ntl = ntile;
  p.mwords = (n + 31) / 32;
  p.a_inv_scale = 1.0 / (double)ctx->a_scale;
  const Work& w = ctx->w;
  std::vector<double> r64((size_t)(batch * ldm), 0.0);
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < m; ++i) r64[(size_t)(b * ldm + i)] = r[b * m + i];
  std::vector<int32_t> ones((size_t)batch, 1);
  cudaStream_t s = ctx->stream;
  CL_CUDA(ctx, cudaMemcpyAsync(w.r64, r64.data(), r64.size() * 8, cudaMemcpyHostToDevice, s));
  CL_CUDA(ctx, cudaMemcpyAsync(w.active, ones.data(), ones.size() * 4, cudaMemcpyHostToDevice, s));
  if (tc) launch_split_resid(p, w, s);
  if (tc) {
    float* d = nullptr;
    CL_CUDA(ctx, cudaMalloc(&d, (size_t)(batch * n) * 4));
    if (!launch_corr_tc_debug(p, w, d, s)) {
      cudaFree(d);
      return fail(ctx, CL_ERR_CUDA, "cl_debug_scores: tcgen05 launch failed");
    }
    std::vector<float> h((size_t)(batch * n));
    CL_CUDA(ctx, cudaMemcpyAsync(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost, s));
    CL_CUDA(ctx, cudaStreamSynchronize(s));
    cudaFree(d);
    for (size_t e = 0; e < h.size(); ++e) scores[e] = h[e];
  } else {
    if (path == 3)
      launch_corr_gemv(p, w, true, s);
    else
      launch_corr_f64(p, w, true, s);
    CL_CUDA(ctx, cudaMemcpyAsync(scores, w.scores, (size_t)(batch * n) * 8,
                                 cudaMemcpyDeviceToHost, s));
    CL_CUDA(ctx, cudaStreamSynchronize(s));
  }
  CL_CUDA(ctx, cudaGetLastError());
  return CL_OK;
}

}  // extern "C"
