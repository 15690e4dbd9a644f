// shim_bench.cpp — times the drop-in boundary itself: cskit::clomp_solve_batch
// (the reference's own signature) served by the B200 shim, host fp64 buffers in
// and host fp64 results (s, mask, x_hat) out, at BASELINE config 2's shape.
//
// TEST / MEASUREMENT INFRASTRUCTURE (links the reference's objects for
// make_setup and la::Mat; built by oracle/Makefile target shim).  Prints one
// JSON line; bench.py adds it to its output as "shim".
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cskit/clomp.hpp"
#include "cskit/rng.hpp"
#include "cskit/sensing.hpp"

using namespace cskit;

int main(int argc, char** argv) {
  const std::size_t n = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 1024;
  const std::size_t B = argc > 2 ? std::strtoul(argv[2], nullptr, 10) : 4096;
  const std::size_t K = argc > 3 ? std::strtoul(argv[3], nullptr, 10) : 32;
  const int reps = argc > 4 ? std::atoi(argv[4]) : 5;
  const bool identity = argc > 5 && std::atoi(argv[5]) != 0;
  const auto tb0 = std::chrono::steady_clock::now();
  MeasurementSetup setup = identity
                               ? compose_setup(gaussian_sensing_matrix(n, 0.5, 1), identity_basis(n))
                               : make_setup(n, 0.5, 1);
  const double build_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - tb0).count();
  Rng rng(7);
  la::Mat x(n, B);
  for (std::size_t b = 0; b < B; ++b)
    for (std::size_t k = 0; k < K; ++k) x(rng.uniform_below(n), b) = rng.normal();
  la::Mat y = la::matmul(setup.a, x);
  ClompConfig cfg;
  cfg.th = 1.0;
  cfg.max_outer = K;
  cfg.inner_steps = 200;
  cfg.lr = 0.1;
  cfg.opt = Optimizer::plain;
  cfg.w_tv = cfg.w_lv = 0.0;
  double first_ms = 0.0, sum_ms = 0.0;
  std::size_t iters = 0;
  double x_err = 0.0;
  for (int r = 0; r <= reps; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    const BatchSolveResult res = clomp_solve_batch(setup, y, cfg);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (r == 0) {
      first_ms = ms;  // includes the dictionary / basis upload
      iters = res.iterations;
      // recovered signal vs the truth in the signal domain (sanity, not parity)
      const la::Mat xt = la::matmul(setup.basis, x);
      double num = 0.0, den = 0.0;
      for (std::size_t e = 0; e < xt.a.size(); ++e) {
        num += (xt.a[e] - res.x_hat.a[e]) * (xt.a[e] - res.x_hat.a[e]);
        den += xt.a[e] * xt.a[e];
      }
      x_err = std::sqrt(num / den);
    } else {
      sum_ms += ms;
    }
  }
  const double ms = sum_ms / reps;
  std::printf("{\"path\": \"cskit::clomp_solve_batch via cskit_clomp_shim (joint mode, fp64 host buffers in, "
              "dense s / mask / x_hat out)\", \"n\": %zu, \"m\": %zu, \"batch\": %zu, \"k\": %zu, "
              "\"basis\": \"%s\", \"ms_per_call\": %.3f, \"signals_per_s\": %.1f, "
              "\"first_call_ms\": %.1f, \"iterations\": %zu, \"x_hat_rel_err\": %.3e, "
              "\"setup_build_s\": %.2f}\n",
              n, setup.m, B, K, identity ? "identity" : "dct", ms, 1000.0 * B / ms, first_ms, iters,
              x_err, build_s);
  return 0;
}
