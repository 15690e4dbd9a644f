// cskit_clomp_shim.cpp — the reference's own CLOMP entry points, implemented on
// the B200 C-ABI.
//
// Drop-in for /root/reference/proj/src/clomp.cpp:211-311: a cskit build that
// compiles this file instead of clomp.cpp (and links libclomp_b200.so) runs
// cskit::clomp_solve_batch / cskit::clomp_solve on the GPU with the same
// signatures, exceptions and result types (include/cskit/clomp.hpp:82-101).
// It is compiled against the reference's headers, which are not copied here.
//
// * The dictionary setup.a is uploaded once per host thread and reused while
//   the caller keeps passing the same MeasurementSetup (the reference
//   re-transposes A on every call, clomp.cpp:224).  "The same" is decided by
//   a cheap key — the data pointer, the shape and a word-wise hash of the
//   matrix (all of it up to 1 Mi entries, 64 Ki evenly spread 16-word runs
//   beyond: ~0.2 ms at config 3's 512 MB) — instead of hashing every byte on
//   every call.  A caller that edits a large matrix in place between calls
//   without touching any sampled word must call cskit_b200_invalidate().
// * Inputs are rounded to fp32 (the GPU operand precision); results are fp64.
// * x_hat = basis * (s .* mask) (clomp.cpp:289): an identity basis returns
//   s_eff itself; any other basis is uploaded once with the dictionary and the
//   product is formed on the GPU from the compact supports (cl_set_synthesis,
//   k_synth.cu), n x |support| multiply-adds per signal instead of the
//   reference's dense n x n x B host product.
// * Priors: setup.basis is handed to cl_set_basis when a prior weight is
//   non-zero: TV-1D on single-column solves (clomp_solve, one-column batches:
//   the CLI's 1D path) and TV-2D + local variance on multi-column batches
//   (the reference's image mode, cskit.cpp:620-652) run on the GPU.
// * Device: CSKIT_B200_DEVICE (environment) or cskit_b200_set_device(); each
//   host thread owns its context, so threads never serialise on each other
//   (the reference library is re-entrant).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "clomp_b200.h"
#include "cskit/clomp.hpp"
#include "cskit/errors.hpp"

namespace {

struct MatKey {
  const double* ptr = nullptr;
  std::size_t rows = 0, cols = 0;
  uint64_t hash = 0;
  bool operator==(const MatKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && hash == o.hash;
  }
};

inline uint64_t mix(uint64_t h, uint64_t w) {
  h ^= w + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h *= 0xff51afd7ed558ccdull;
  return h ^ (h >> 32);
}

// Word-wise hash: everything up to 1 Mi doubles, evenly spread 16-word runs
// (64 Ki of them) above.
uint64_t sample_hash(const double* p, std::size_t count) {
  uint64_t h = 0x243f6a8885a308d3ull ^ count;
  const uint64_t* w = reinterpret_cast<const uint64_t*>(p);
  constexpr std::size_t kFull = std::size_t(1) << 20;
  if (count <= kFull) {
    // four independent chains (the multiply latency would serialise one)
    uint64_t l0 = h, l1 = h + 1, l2 = h + 2, l3 = h + 3;
    std::size_t i = 0;
    for (; i + 4 <= count; i += 4) {
      l0 = mix(l0, w[i]);
      l1 = mix(l1, w[i + 1]);
      l2 = mix(l2, w[i + 2]);
      l3 = mix(l3, w[i + 3]);
    }
    for (; i < count; ++i) l0 = mix(l0, w[i]);
    return mix(mix(l0, l1), mix(l2, l3));
  }
  constexpr std::size_t kRuns = std::size_t(1) << 16, kRun = 16;
  const std::size_t stride = (count - kRun) / (kRuns - 1);
  for (std::size_t r = 0; r < kRuns; ++r) {
    const uint64_t* q = w + r * stride;
    for (std::size_t i = 0; i < kRun; ++i) h = mix(h, q[i]);
  }
  return h;
}

MatKey key_of(const cskit::la::Mat& m) {
  return MatKey{m.data(), m.rows, m.cols, m.a.empty() ? 0 : sample_hash(m.data(), m.a.size())};
}

struct CachedCtx {
  cl_ctx* ctx = nullptr;
  MatKey a_key, basis_key;
  bool basis_identity = false;
  bool basis_uploaded = false;
  int device = 0;
  ~CachedCtx() {
    if (ctx) cl_destroy(ctx);
  }
};

thread_local std::unique_ptr<CachedCtx> t_cache;
int g_device = -1;  // -1: CSKIT_B200_DEVICE or 0

int chosen_device() {
  if (g_device >= 0) return g_device;
  if (const char* e = std::getenv("CSKIT_B200_DEVICE")) return std::atoi(e);
  return 0;
}

[[noreturn]] void rethrow(int code, const char* msg) {
  const std::string m = msg ? msg : "clomp (B200)";
  switch (code) {
    case CL_ERR_CONFIG: throw cskit::ConfigError(m);
    case CL_ERR_DIMENSION: throw cskit::DimensionError(m);
    case CL_ERR_NUMERICAL: throw cskit::NumericalError(m);
    case CL_ERR_UNSUPPORTED: throw cskit::ConfigError(m);
    default: throw cskit::Error(m);
  }
}

bool is_identity(const cskit::la::Mat& b) {
  if (b.rows != b.cols) return false;
  const std::size_t n = b.rows;
  for (std::size_t i = 0; i < n; ++i) {
    const double* row = b.data() + i * n;
    for (std::size_t j = 0; j < n; ++j)
      if (row[j] != (i == j ? 1.0 : 0.0)) return false;
  }
  return true;
}

// The basis goes to the device when the solve needs it there: a prior is
// configured (clomp.cpp:93-119) or x_hat needs a real product.
void sync_basis(CachedCtx& c, const cskit::MeasurementSetup& setup, bool priors) {
  const bool square = setup.basis.rows == setup.n && setup.basis.cols == setup.n;
  const MatKey bk = square ? key_of(setup.basis) : MatKey{};
  if (!(bk == c.basis_key)) {
    c.basis_key = bk;
    c.basis_identity = square && is_identity(setup.basis);
    if (c.basis_uploaded) {
      cl_set_basis(c.ctx, nullptr, 0, CL_LAYOUT_REF);
      c.basis_uploaded = false;
    }
  }
  const bool need = square && (priors || !c.basis_identity);
  if (need && !c.basis_uploaded) {
    const int st = cl_set_basis(c.ctx, setup.basis.data(), static_cast<int64_t>(setup.n),
                                CL_LAYOUT_REF);
    if (st != CL_OK) rethrow(st, cl_last_error(c.ctx));
    c.basis_uploaded = true;
  }
  cl_set_synthesis(c.ctx, c.basis_uploaded && !c.basis_identity ? 1 : 0);
}

CachedCtx& context_for(const cskit::MeasurementSetup& setup, bool priors) {
  const MatKey ak = key_of(setup.a);
  const int dev = chosen_device();
  if (!(t_cache && t_cache->a_key == ak && t_cache->device == dev)) {
    std::vector<float> a32(setup.a.a.size());
    for (std::size_t i = 0; i < a32.size(); ++i) a32[i] = static_cast<float>(setup.a.a[i]);
    t_cache.reset();  // free the previous dictionary before uploading the next
    int st = 0;
    cl_ctx* ctx = cl_create(dev, a32.data(), static_cast<int64_t>(setup.m),
                            static_cast<int64_t>(setup.n), CL_LAYOUT_REF, &st);
    if (!ctx) rethrow(st, cl_last_error(nullptr));
    t_cache = std::make_unique<CachedCtx>();
    t_cache->ctx = ctx;
    t_cache->a_key = ak;
    t_cache->device = dev;
  }
  sync_basis(*t_cache, setup, priors);
  return *t_cache;
}

// Host-side bulk work (fp64 -> fp32 of y, the dense result copies) split over
// a few threads: first-touch page faults and conversions scale with cores.
template <class F>
void par_chunks(std::size_t total, F&& fn) {
  const std::size_t min_chunk = std::size_t(1) << 18;
  std::size_t nt = std::min<std::size_t>(8, std::max<std::size_t>(1, total / min_chunk));
  nt = std::min<std::size_t>(nt, std::max(1u, std::thread::hardware_concurrency()));
  if (nt <= 1) {
    fn(0, total);
    return;
  }
  std::vector<std::thread> th;
  const std::size_t per = (total + nt - 1) / nt;
  for (std::size_t t = 1; t < nt; ++t)
    th.emplace_back([&, t] { fn(std::min(total, t * per), std::min(total, (t + 1) * per)); });
  fn(0, std::min(total, per));
  for (auto& x : th) x.join();
}

cl_config to_c(const cskit::ClompConfig& c) {
  cl_config k;
  cl_config_default(&k);
  k.th = c.th;
  k.max_outer = c.max_outer;
  k.eps = c.eps;
  k.inner_steps = c.inner_steps;
  k.lr = c.lr;
  k.opt = c.opt == cskit::Optimizer::plain ? CL_OPT_PLAIN
          : c.opt == cskit::Optimizer::momentum ? CL_OPT_MOMENTUM
                                                : CL_OPT_ADAM;
  k.w_tv = c.w_tv;
  k.w_lv = c.w_lv;
  k.lv_window = c.lv.window;
  k.lv_stride = c.lv.stride;
  k.stall_tol = c.stall_tol;
  k.stall_patience = c.stall_patience;
  return k;
}

}  // namespace

extern "C" {
// Device the shim's contexts live on (default: CSKIT_B200_DEVICE or 0).
void cskit_b200_set_device(int device) { g_device = device; }
// Drop this thread's cached dictionary (after editing setup.a in place).
void cskit_b200_invalidate(void) { t_cache.reset(); }
}

namespace cskit {

BatchSolveResult clomp_solve_batch(const MeasurementSetup& setup, const la::Mat& y_cols,
                                   const ClompConfig& cfg) {
  const auto t0 = std::chrono::steady_clock::now();
  if (y_cols.rows != setup.m)
    throw DimensionError("clomp: y rows " + std::to_string(y_cols.rows) + " vs m=" +
                         std::to_string(setup.m));
  if (y_cols.cols == 0) throw DimensionError("clomp: empty batch");
  const bool priors = cfg.w_tv != 0.0 || cfg.w_lv != 0.0;
  static const bool trace = std::getenv("CSKIT_B200_TRACE") != nullptr;
  auto lap = [&, last = t0](const char* what) mutable {
    if (!trace) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[shim] %-22s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
  };
  CachedCtx& cc = context_for(setup, priors);
  lap("context (keys)");
  cl_ctx* ctx = cc.ctx;
  const std::size_t n = setup.n, B = y_cols.cols;
  std::unique_ptr<float[]> y32(new float[y_cols.a.size()]);  // uninitialised on purpose
  par_chunks(y_cols.a.size(), [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) y32[i] = static_cast<float>(y_cols.a[i]);
  });
  BatchSolveResult out;
  out.s = la::Mat(n, B);
  out.mask.assign(n * B, 0);
  const bool gpu_xhat = cc.basis_uploaded && !cc.basis_identity;
  if (gpu_xhat) out.x_hat = la::Mat(n, B);
  std::vector<int64_t> iters(B);
  std::vector<double> rn(B);
  std::vector<uint8_t> conv(B);
  std::vector<int32_t> status(B);
  cl_result r{};
  r.cap = 0;
  r.flags = CL_RESULT_PREZEROED;  // la::Mat / assign() zero-filled s and mask
  r.s = out.s.data();
  r.mask = out.mask.data();
  r.iterations = iters.data();
  r.final_residual_norm = rn.data();
  r.converged = conv.data();
  r.status = status.data();
  r.x_hat = gpu_xhat ? out.x_hat.data() : nullptr;
  const cl_config c = to_c(cfg);
  lap("host buffers");
  const int code = cl_solve_batch(ctx, y32.get(), static_cast<int64_t>(B), CL_LAYOUT_REF, &c,
                                  CL_MODE_JOINT, &r);
  if (code != CL_OK) rethrow(code, cl_last_error(ctx));
  if (trace) {
    cl_stats stt{};
    cl_get_stats(ctx, &stt);
    std::fprintf(stderr, "[shim] cl_solve_batch e2e_ms %.3f (h2d %lld B, d2h %lld B)\n", stt.e2e_ms,
                 (long long)stt.h2d_bytes, (long long)stt.d2h_bytes);
  }
  lap("cl_solve_batch");
  out.iterations = static_cast<std::size_t>(iters[0]);
  out.final_residual_norm = rn[0];
  out.converged = conv[0] != 0;
  if (!gpu_xhat) {
    if (cc.basis_identity) {  // x_hat = I s_eff; s is already zero off the mask
      out.x_hat = out.s;
    } else {  // no usable basis: what the reference's matmul would return / throw
      out.x_hat = la::matmul(setup.basis, out.s);
    }
  }
  lap("x_hat / epilogue");
  out.wall_time_s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return out;
}

SolveResult clomp_solve(const MeasurementSetup& setup, const la::Vec& y,
                        const ClompConfig& cfg) {
  la::Mat y_cols(setup.m, 1);
  if (y.size() != setup.m)
    throw DimensionError("clomp: y has " + std::to_string(y.size()) +
                         " entries, setup expects " + std::to_string(setup.m));
  y_cols.a = y;
  const BatchSolveResult batch = clomp_solve_batch(setup, y_cols, cfg);
  SolveResult out;
  out.s.values = batch.s.a;
  out.s.mask = batch.mask;
  out.x_hat = batch.x_hat.a;
  out.iterations = batch.iterations;
  out.final_residual_norm = batch.final_residual_norm;
  out.converged = batch.converged;
  out.wall_time_s = batch.wall_time_s;
  return out;
}

}  // namespace cskit
