// shim_parity.cpp — the reference's own C++ API, served by the B200 shim.
//
// TEST INFRASTRUCTURE.  Linked (oracle/Makefile, target shim) from: this file,
// paper_2501_11592_b200/csrc/shim/cskit_clomp_shim.cpp (first, so its
// cskit::clomp_solve / clomp_solve_batch win), the unmodified reference
// objects (everything incl. clomp.o, via --allow-multiple-definition), the
// oracle restatement, and libclomp_b200.so.  Solves reference-style problems
// (make_setup: Gaussian sensing composed with the DCT basis, sensing.cpp:77-79)
// through cskit::clomp_solve and compares with the oracle: identical supports
// and iteration counts, coefficients within 1e-9, x_hat within 1e-9.
#include <cmath>
#include <cstdio>
#include <vector>

#include "cskit/clomp.hpp"
#include "cskit/errors.hpp"
#include "cskit/rng.hpp"
#include "cskit/sensing.hpp"

extern "C" {
#include "clomp_oracle.h"
}

using namespace cskit;

static la::Mat round32(const la::Mat& m) {
  la::Mat r = m;
  for (double& v : r.a) v = static_cast<double>(static_cast<float>(v));
  return r;
}

int main() {
  int failures = 0;
  for (int seed = 1; seed <= 6; ++seed) {
    MeasurementSetup setup = make_setup(64, 0.5, 100 + seed);
    setup.a = round32(setup.a);  // the GPU's fp32 operands, seen by both sides
    Rng rng(static_cast<uint64_t>(seed));
    la::Vec x(setup.n, 0.0);
    for (int k = 0; k < 4; ++k) x[rng.uniform_below(setup.n)] = rng.normal();
    la::Vec y = la::matvec(setup.a, x);
    for (double& v : y) v = static_cast<double>(static_cast<float>(v));
    ClompConfig cfg;
    cfg.th = seed % 2 ? 1.0 : 0.7;
    cfg.opt = seed % 3 == 0 ? Optimizer::adam : Optimizer::plain;
    cfg.lr = cfg.opt == Optimizer::adam ? 0.02 : 0.1;
    cfg.max_outer = 8;
    cfg.inner_steps = 60;
    cfg.w_tv = 0.0;
    cfg.w_lv = 0.0;
    const SolveResult got = clomp_solve(setup, y, cfg);  // -> shim -> GPU

    orc_config oc{cfg.th, cfg.max_outer, cfg.eps, cfg.inner_steps, cfg.lr,
                  static_cast<int32_t>(cfg.opt == Optimizer::plain ? 0 : cfg.opt == Optimizer::momentum ? 1 : 2),
                  0, 0.0, 0.0, cfg.lv.window, cfg.lv.stride, cfg.stall_tol, cfg.stall_patience};
    std::vector<double> s(setup.n);
    std::vector<uint8_t> mk(setup.n);
    int64_t it = 0;
    double rn = 0.0;
    uint8_t cv = 0;
    int32_t st = 0;
    orc_clomp_solve_batch(setup.a.data(), setup.m, setup.n, y.data(), 1, &oc, ORC_ISA_AVX2,
                          ORC_MODE_JOINT, s.data(), mk.data(), &it, &rn, &cv, &st, nullptr,
                          nullptr, 0);
    double cmax = 0.0, err = 0.0, xerr = 0.0;
    bool same_mask = true;
    for (std::size_t j = 0; j < setup.n; ++j) {
      same_mask = same_mask && (got.s.mask[j] == mk[j]);
      cmax = std::fmax(cmax, std::fabs(s[j]));
      err = std::fmax(err, std::fabs(got.s.values[j] - s[j]));
    }
    // x_hat = basis * s_eff (clomp.cpp:289) from the oracle's coefficients
    for (std::size_t i = 0; i < setup.n; ++i) {
      double acc = 0.0;
      for (std::size_t j = 0; j < setup.n; ++j) acc += setup.basis(i, j) * (mk[j] ? s[j] : 0.0);
      xerr = std::fmax(xerr, std::fabs(acc - got.x_hat[i]));
    }
    const bool ok = st == 0 && same_mask && got.iterations == static_cast<std::size_t>(it) &&
                    err <= 1e-9 * std::fmax(cmax, 1.0) && xerr <= 1e-9 &&
                    got.converged == (cv != 0);
    std::printf("seed %d th %.1f opt %d: mask %s iters %zu/%lld coef err %.2e x_hat err %.2e %s\n",
                seed, cfg.th, oc.opt, same_mask ? "same" : "DIFF", got.iterations,
                static_cast<long long>(it), err, xerr, ok ? "ok" : "FAIL");
    failures += ok ? 0 : 1;
  }
  // The reference's default configuration (Adam, th = 0.7, automatic TV / LV
  // weights): the TV prior runs on the GPU through the basis the shim hands
  // over (LV never applies to one column).
  for (int seed = 1; seed <= 3; ++seed) {
    MeasurementSetup setup = make_setup(64, 0.5, 200 + seed);
    setup.a = round32(setup.a);
    Rng rng(static_cast<uint64_t>(seed + 50));
    la::Vec x(setup.n, 0.0);
    for (int k = 0; k < 4; ++k) x[rng.uniform_below(setup.n)] = rng.normal();
    la::Vec y = la::matvec(setup.a, x);
    for (double& v : y) v = static_cast<double>(static_cast<float>(v));
    ClompConfig cfg;  // defaults: priors on
    cfg.max_outer = 12;
    const SolveResult got = clomp_solve(setup, y, cfg);
    orc_config oc{cfg.th, cfg.max_outer, cfg.eps, cfg.inner_steps, cfg.lr, 2, 0, cfg.w_tv,
                  cfg.w_lv, cfg.lv.window, cfg.lv.stride, cfg.stall_tol, cfg.stall_patience};
    std::vector<double> s(setup.n);
    std::vector<uint8_t> mk(setup.n);
    int64_t it = 0;
    double rn = 0.0;
    uint8_t cv = 0;
    int32_t st = 0;
    orc_clomp_solve_batch_basis(setup.a.data(), setup.m, setup.n, setup.basis.data(), y.data(),
                                1, &oc, ORC_ISA_AVX2, ORC_MODE_PER_SIGNAL, s.data(), mk.data(),
                                &it, &rn, &cv, &st, nullptr, nullptr, 0);
    double cmax = 0.0, err = 0.0;
    bool same_mask = true;
    for (std::size_t j = 0; j < setup.n; ++j) {
      same_mask = same_mask && (got.s.mask[j] == mk[j]);
      cmax = std::fmax(cmax, std::fabs(s[j]));
      err = std::fmax(err, std::fabs(got.s.values[j] - s[j]));
    }
    const bool ok = st == 0 && same_mask && got.iterations == static_cast<std::size_t>(it) &&
                    err <= 1e-9 * std::fmax(cmax, 1.0) &&
                    std::fabs(got.final_residual_norm - rn) <= 1e-9 * std::fmax(rn, 1e-12);
    std::printf("default config (priors) seed %d: mask %s iters %zu/%lld coef err %.2e %s\n",
                seed, same_mask ? "same" : "DIFF", got.iterations, static_cast<long long>(it),
                err, ok ? "ok" : "FAIL");
    failures += ok ? 0 : 1;
  }
  // Multi-column batches: x_hat for every column formed on the GPU
  // (cl_set_synthesis) with the DCT basis, returned as-is for an identity
  // basis; priors off, then the reference's image mode (TV-2D + local
  // variance, default Adam / th = 0.7) against the oracle's joint solve.
  for (int variant = 0; variant < 3; ++variant) {
    const std::size_t n = 48, B = 7;
    MeasurementSetup setup = variant == 1
                                 ? compose_setup(gaussian_sensing_matrix(n, 0.5, 321), identity_basis(n))
                                 : make_setup(n, 0.5, 300 + variant);
    setup.a = round32(setup.a);
    Rng rng(static_cast<uint64_t>(900 + variant));
    la::Mat y(setup.m, B);
    for (std::size_t b = 0; b < B; ++b) {
      la::Vec x(setup.n, 0.0);
      for (int k = 0; k < 3; ++k) x[rng.uniform_below(setup.n)] = rng.normal();
      const la::Vec yb = la::matvec(setup.a, x);
      for (std::size_t i = 0; i < setup.m; ++i) y(i, b) = static_cast<double>(static_cast<float>(yb[i]));
    }
    ClompConfig cfg;
    cfg.max_outer = 6;
    if (variant < 2) {
      cfg.th = 1.0;
      cfg.opt = Optimizer::plain;
      cfg.lr = 0.1;
      cfg.inner_steps = 40;
      cfg.w_tv = cfg.w_lv = 0.0;
    }
    const BatchSolveResult got = clomp_solve_batch(setup, y, cfg);
    orc_config oc{cfg.th, cfg.max_outer, cfg.eps, cfg.inner_steps, cfg.lr,
                  static_cast<int32_t>(cfg.opt == Optimizer::plain ? 0 : 2), 0, cfg.w_tv, cfg.w_lv,
                  cfg.lv.window, cfg.lv.stride, cfg.stall_tol, cfg.stall_patience};
    std::vector<double> s(n * B);
    std::vector<uint8_t> mk(n * B);
    std::vector<int64_t> it(B);
    std::vector<double> rn(B);
    std::vector<uint8_t> cv(B);
    std::vector<int32_t> st(B);
    const int code = orc_clomp_solve_batch_basis(setup.a.data(), setup.m, setup.n, setup.basis.data(),
                                                 y.data(), B, &oc, ORC_ISA_AVX2, ORC_MODE_JOINT,
                                                 s.data(), mk.data(), it.data(), rn.data(), cv.data(),
                                                 st.data(), nullptr, nullptr, 0);
    double cmax = 0.0, err = 0.0, xerr = 0.0;
    bool same_mask = true;
    for (std::size_t e = 0; e < n * B; ++e) {
      same_mask = same_mask && (got.mask[e] == mk[e]);
      cmax = std::fmax(cmax, std::fabs(s[e]));
      err = std::fmax(err, std::fabs(got.s.a[e] - s[e]));
    }
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t b = 0; b < B; ++b) {
        double acc = 0.0;
        for (std::size_t j = 0; j < n; ++j) acc += setup.basis(i, j) * (mk[j * B + b] ? s[j * B + b] : 0.0);
        xerr = std::fmax(xerr, std::fabs(acc - got.x_hat(i, b)));
      }
    const bool ok = code == 0 && same_mask && got.iterations == static_cast<std::size_t>(it[0]) &&
                    err <= 1e-9 * std::fmax(cmax, 1.0) && xerr <= 1e-9 &&
                    got.x_hat.rows == n && got.x_hat.cols == B;
    std::printf("batch of %zu (%s): mask %s iters %zu/%lld coef err %.2e x_hat err %.2e %s\n", B,
                variant == 0 ? "DCT basis, priors off" : variant == 1 ? "identity basis" : "image mode priors",
                same_mask ? "same" : "DIFF", got.iterations, static_cast<long long>(it[0]), err, xerr,
                ok ? "ok" : "FAIL");
    failures += ok ? 0 : 1;
  }
  // The dictionary cache: a different matrix at the same address is seen
  // (content hash), the same matrix is not uploaded again.
  {
    MeasurementSetup setup = make_setup(32, 0.5, 11);
    setup.a = round32(setup.a);
    la::Vec y(setup.m, 0.0);
    for (std::size_t i = 0; i < setup.m; ++i) y[i] = static_cast<double>(static_cast<float>(setup.a(i, 3)));
    ClompConfig cfg;
    cfg.th = 1.0;
    cfg.opt = Optimizer::plain;
    cfg.lr = 0.1;
    cfg.max_outer = 2;
    cfg.w_tv = cfg.w_lv = 0.0;
    const SolveResult r1 = clomp_solve(setup, y, cfg);
    for (std::size_t i = 0; i < setup.m; ++i) std::swap(setup.a(i, 3), setup.a(i, 9));  // in place
    const SolveResult r2 = clomp_solve(setup, y, cfg);
    const bool ok = r1.s.mask[3] == 1 && r2.s.mask[9] == 1 && r2.s.mask[3] == 0;
    std::printf("dictionary edited in place: %s\n", ok ? "seen ok" : "STALE CONTEXT FAIL");
    failures += ok ? 0 : 1;
  }
  // Error mapping: a diverging lr raises cskit::NumericalError through the shim.
  try {
    MeasurementSetup setup = make_setup(32, 0.5, 7);
    setup.a = round32(setup.a);
    la::Vec y(setup.m, 0.25);
    ClompConfig cfg;
    cfg.th = 1.0;
    cfg.opt = Optimizer::plain;
    cfg.lr = 1e6;
    cfg.w_tv = cfg.w_lv = 0.0;
    clomp_solve(setup, y, cfg);
    std::printf("divergence: no exception FAIL\n");
    ++failures;
  } catch (const NumericalError&) {
    std::printf("divergence: NumericalError ok\n");
  }
  std::printf("%s\n", failures ? "SHIM PARITY FAILED" : "SHIM PARITY OK");
  return failures ? 1 : 0;
}
