// ref_harness.cpp — C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled (by oracle/Makefile) together with the
// reference sources where they lie under /root/reference/proj/src into
// oracle/_ref/libcskit_ref.so.  It lets the Python tests and bench.py's
// reference arm call cskit::clomp_solve_batch / clomp_solve (clomp.cpp:211-311)
// and the unit-level entry points through ctypes.  Nothing here computes; it
// marshals plain arrays into cskit types and maps the reference exceptions
// (errors.hpp:10-37) onto the status codes of include/clomp_b200.h.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <utility>
#include <vector>

#include "cskit/clomp.hpp"
#include "cskit/errors.hpp"
#include "cskit/kernels.hpp"
#include "cskit/rng.hpp"
#include "cskit/sensing.hpp"

extern "C" {
// Same layout as cl_config (include/clomp_b200.h) and orc_config.
struct ref_config {
  double th;
  uint64_t max_outer;
  double eps;
  uint64_t inner_steps;
  double lr;
  int32_t opt;
  int32_t pad0;
  double w_tv;
  double w_lv;
  uint64_t lv_window;
  uint64_t lv_stride;
  double stall_tol;
  uint64_t stall_patience;
};
}

namespace {

cskit::ClompConfig to_cfg(const ref_config* c) {
  cskit::ClompConfig cfg;
  cfg.th = c->th;
  cfg.max_outer = c->max_outer;
  cfg.eps = c->eps;
  cfg.inner_steps = c->inner_steps;
  cfg.lr = c->lr;
  cfg.opt = c->opt == 0   ? cskit::Optimizer::plain
            : c->opt == 1 ? cskit::Optimizer::momentum
                          : cskit::Optimizer::adam;
  cfg.w_tv = c->w_tv;
  cfg.w_lv = c->w_lv;
  cfg.lv.window = c->lv_window;
  cfg.lv.stride = c->lv_stride;
  cfg.stall_tol = c->stall_tol;
  cfg.stall_patience = c->stall_patience;
  return cfg;
}

// MeasurementSetup with a 1 x n dummy basis: with priors off the
// basis is read only for x_hat = basis * s_eff (clomp.cpp:289).
cskit::MeasurementSetup to_setup(const double* a, int64_t m, int64_t n,
                                 const double* basis) {
  cskit::MeasurementSetup s;
  s.n = static_cast<std::size_t>(n);
  s.m = static_cast<std::size_t>(m);
  s.a = cskit::la::Mat(s.m, s.n);
  std::memcpy(s.a.data(), a, sizeof(double) * s.m * s.n);
  if (basis) {
    s.basis = cskit::la::Mat(s.n, s.n);
    std::memcpy(s.basis.data(), basis, sizeof(double) * s.n * s.n);
  } else {
    s.basis = cskit::la::Mat(1, s.n);
  }
  return s;
}

int code_of(const std::exception& e) {
  if (dynamic_cast<const cskit::ConfigError*>(&e)) return 2;
  if (dynamic_cast<const cskit::DimensionError*>(&e)) return 3;
  if (dynamic_cast<const cskit::NumericalError*>(&e)) return 4;
  return 1;
}

void put_err(char* err, int errlen, const char* what) {
  if (err && errlen > 0) {
    std::strncpy(err, what, static_cast<std::size_t>(errlen) - 1);
    err[errlen - 1] = 0;
  }
}

}  // namespace

extern "C" {

// isa: 0 scalar, 1 avx2 (kern::force, kernels.cpp:40-44).
int ref_force_isa(int isa) {
  try {
    cskit::kern::force(isa ? cskit::kern::Isa::avx2 : cskit::kern::Isa::scalar);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// basis: n x n row-major synthesis matrix (x = basis * s) or NULL for the
// 1 x n dummy; the priors (w_tv / w_lv) need the real one.
int ref_clomp_solve_batch_b(const double* a, int64_t m, int64_t n, const double* basis,
                            const double* y, int64_t batch, const ref_config* c,
                            double* s_out, uint8_t* mask_out, int64_t* iterations,
                            double* final_rn, uint8_t* converged, double* x_hat,
                            double* wall_s, char* err, int errlen) {
  try {
    const auto setup = to_setup(a, m, n, basis);
    cskit::la::Mat yc(static_cast<std::size_t>(m), static_cast<std::size_t>(batch));
    if (batch > 0) std::memcpy(yc.data(), y, sizeof(double) * yc.a.size());
    const auto res = cskit::clomp_solve_batch(setup, yc, to_cfg(c));
    std::memcpy(s_out, res.s.data(), sizeof(double) * res.s.a.size());
    std::memcpy(mask_out, res.mask.data(), res.mask.size());
    *iterations = static_cast<int64_t>(res.iterations);
    *final_rn = res.final_residual_norm;
    *converged = res.converged ? 1 : 0;
    if (x_hat && basis) std::memcpy(x_hat, res.x_hat.data(), sizeof(double) * res.x_hat.a.size());
    if (wall_s) *wall_s = res.wall_time_s;
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return code_of(e);
  }
}

int ref_clomp_solve_batch(const double* a, int64_t m, int64_t n,
                          const double* y, int64_t batch, const ref_config* c,
                          double* s_out, uint8_t* mask_out, int64_t* iterations,
                          double* final_rn, uint8_t* converged,
                          double* wall_s, char* err, int errlen) {
  try {
    const auto setup = to_setup(a, m, n, nullptr);
    cskit::la::Mat yc(static_cast<std::size_t>(m), static_cast<std::size_t>(batch));
    if (batch > 0) std::memcpy(yc.data(), y, sizeof(double) * yc.a.size());
    const auto res = cskit::clomp_solve_batch(setup, yc, to_cfg(c));
    std::memcpy(s_out, res.s.data(), sizeof(double) * res.s.a.size());
    std::memcpy(mask_out, res.mask.data(), res.mask.size());
    *iterations = static_cast<int64_t>(res.iterations);
    *final_rn = res.final_residual_norm;
    *converged = res.converged ? 1 : 0;
    if (wall_s) *wall_s = res.wall_time_s;
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return code_of(e);
  }
}

int ref_clomp_solve(const double* a, int64_t m, int64_t n, const double* y,
                    const ref_config* c, double* s_out, uint8_t* mask_out,
                    int64_t* iterations, double* final_rn, uint8_t* converged,
                    double* wall_s, char* err, int errlen) {
  try {
    const auto setup = to_setup(a, m, n, nullptr);
    cskit::la::Vec yv(y, y + m);
    const auto res = cskit::clomp_solve(setup, yv, to_cfg(c));
    std::memcpy(s_out, res.s.values.data(), sizeof(double) * res.s.values.size());
    std::memcpy(mask_out, res.s.mask.data(), res.s.mask.size());
    *iterations = static_cast<int64_t>(res.iterations);
    *final_rn = res.final_residual_norm;
    *converged = res.converged ? 1 : 0;
    if (wall_s) *wall_s = res.wall_time_s;
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return code_of(e);
  }
}

int ref_inject_support(const double* a, int64_t m, int64_t n, const double* r,
                       int64_t batch, double th, uint8_t* mask) {
  try {
    const auto setup = to_setup(a, m, n, nullptr);
    cskit::la::Mat rc(static_cast<std::size_t>(m), static_cast<std::size_t>(batch));
    std::memcpy(rc.data(), r, sizeof(double) * rc.a.size());
    std::vector<std::uint8_t> mk(mask, mask + n * batch);
    cskit::inject_support(setup, rc, th, mk);
    std::memcpy(mask, mk.data(), mk.size());
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_clomp_loss(const double* a, int64_t m, int64_t n, const double* y,
                   int64_t batch, const double* s, const uint8_t* mask,
                   const ref_config* c, double* loss, double* grad) {
  try {
    const auto setup = to_setup(a, m, n, nullptr);
    cskit::la::Mat yc(static_cast<std::size_t>(m), static_cast<std::size_t>(batch));
    std::memcpy(yc.data(), y, sizeof(double) * yc.a.size());
    cskit::ClompState st(static_cast<std::size_t>(n), static_cast<std::size_t>(batch));
    std::memcpy(st.s.data(), s, sizeof(double) * st.s.a.size());
    std::memcpy(st.mask.data(), mask, st.mask.size());
    cskit::la::Mat g;
    const auto lb = cskit::clomp_loss(setup, yc, st, to_cfg(c), grad ? &g : nullptr);
    *loss = lb.total;
    if (grad) std::memcpy(grad, g.data(), sizeof(double) * g.a.size());
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_gradient_step(double* s, const uint8_t* mask, double* m1, double* m2,
                      uint64_t* adam_steps, const double* grad, int64_t total,
                      const ref_config* c) {
  try {
    cskit::ClompState st(static_cast<std::size_t>(total), 1);
    std::memcpy(st.s.data(), s, sizeof(double) * total);
    std::memcpy(st.mask.data(), mask, total);
    std::memcpy(st.m1.data(), m1, sizeof(double) * total);
    std::memcpy(st.m2.data(), m2, sizeof(double) * total);
    st.adam_steps = *adam_steps;
    cskit::la::Mat g(static_cast<std::size_t>(total), 1);
    std::memcpy(g.data(), grad, sizeof(double) * total);
    cskit::gradient_step(st, g, to_cfg(c));
    std::memcpy(s, st.s.data(), sizeof(double) * total);
    std::memcpy(m1, st.m1.data(), sizeof(double) * total);
    std::memcpy(m2, st.m2.data(), sizeof(double) * total);
    *adam_steps = st.adam_steps;
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// Draws from cskit::Rng (rng.hpp:13-79): kind 0 next_u64 (as double bits via
// out_u64), 1 uniform, 2 normal, 3 uniform_below(bound).
void ref_rng_draws(uint64_t seed, int kind, uint64_t bound, int64_t count,
                   double* out, uint64_t* out_u64) {
  cskit::Rng rng(seed);
  for (int64_t i = 0; i < count; ++i) {
    switch (kind) {
      case 0: out_u64[i] = rng.next_u64(); break;
      case 1: out[i] = rng.uniform(); break;
      case 2: out[i] = rng.normal(); break;
      default: out_u64[i] = rng.uniform_below(bound); break;
    }
  }
}

// The harness's seeded 1D problem drawn from the reference's
// own cskit::Rng (rng.hpp:13-79), so bench.py's reference arm generates its
// inputs without loading the B200 library.  Same draw order as the product's
// cl_gen_problem_1d (tests/test_datagen.py pins the two bit for bit): A
// entries normal()/sqrt(m) row-major, columns normalised in fp64, rounded to
// fp32; per signal a partial Fisher-Yates support (uniform_below) then k
// values (normal(), or sign from uniform() < 0.5 times 1 + uniform());
// y = A x in fp64; per-signal noise sd = rms(A x_b) 10^(-snr/20) drawn after
// every signal; y rounded to fp32.  A m x n fp32, X n x B fp64 (may be NULL),
// Y m x B fp32, all row-major.
int ref_gen_problem_1d(uint64_t seed, int64_t m, int64_t n, int64_t k, int64_t batch,
                       int normalize, int value_law, double snr_db, float* A, double* X,
                       float* Y) {
  if (m <= 0 || n <= 0 || batch <= 0 || k < 0 || k > n) return 3;
  cskit::Rng rng(seed);
  std::vector<double> a(static_cast<size_t>(m * n));
  const double scale = 1.0 / std::sqrt(static_cast<double>(m));
  for (auto& e : a) e = scale * rng.normal();
  if (normalize) {
    for (int64_t j = 0; j < n; ++j) {
      double ss = 0.0;
      for (int64_t i = 0; i < m; ++i) ss += a[i * n + j] * a[i * n + j];
      const double nrm = std::sqrt(ss);
      if (nrm > 0.0)
        for (int64_t i = 0; i < m; ++i) a[i * n + j] /= nrm;
    }
  }
  for (int64_t e = 0; e < m * n; ++e) A[e] = static_cast<float>(a[e]);
  std::vector<int64_t> perm(static_cast<size_t>(n)), sup(static_cast<size_t>(k * batch));
  std::vector<double> vals(static_cast<size_t>(k * batch));
  for (int64_t b = 0; b < batch; ++b) {
    for (int64_t j = 0; j < n; ++j) perm[j] = j;
    for (int64_t q = 0; q < k; ++q) {
      const int64_t r = q + static_cast<int64_t>(rng.uniform_below(static_cast<uint64_t>(n - q)));
      std::swap(perm[q], perm[r]);
    }
    for (int64_t q = 0; q < k; ++q) {
      double v;
      if (value_law == 1) {
        const double sgn = rng.uniform() < 0.5 ? -1.0 : 1.0;
        v = sgn * (1.0 + rng.uniform());
      } else {
        v = rng.normal();
      }
      sup[b * k + q] = perm[q];
      vals[b * k + q] = v;
    }
  }
  if (X) std::memset(X, 0, sizeof(double) * n * batch);
  std::vector<double> yall(static_cast<size_t>(m * batch)), rms(static_cast<size_t>(batch));
  for (int64_t b = 0; b < batch; ++b) {
    if (X)
      for (int64_t q = 0; q < k; ++q) X[sup[b * k + q] * batch + b] = vals[b * k + q];
    double ss = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int64_t q = 0; q < k; ++q)
        acc += static_cast<double>(A[i * n + sup[b * k + q]]) * vals[b * k + q];
      yall[i * batch + b] = acc;
      ss += acc * acc;
    }
    rms[b] = std::sqrt(ss / static_cast<double>(m));
  }
  if (snr_db >= 0.0 && std::isfinite(snr_db)) {
    const double f = std::pow(10.0, -snr_db / 20.0);
    for (int64_t b = 0; b < batch; ++b)
      for (int64_t i = 0; i < m; ++i) yall[i * batch + b] += rms[b] * f * rng.normal();
  }
  for (int64_t e = 0; e < m * batch; ++e) Y[e] = static_cast<float>(yall[e]);
  return 0;
}

// dct_basis (sensing.cpp:13-29), n x n row-major.
void ref_dct_basis(int64_t n, double* out) {
  const auto b = cskit::dct_basis(static_cast<std::size_t>(n));
  std::memcpy(out, b.d.data(), sizeof(double) * b.d.a.size());
}

}  // extern "C"
