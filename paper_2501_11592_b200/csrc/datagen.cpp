// datagen.cpp — seeded synthetic inputs for the BASELINE configs (host only,
// not on the hot path).  The generator is a restatement of cskit::Rng
// (xoshiro256++ seeded through splitmix64, 53-bit uniforms, Marsaglia polar
// normals, unbiased uniform_below: /root/reference/proj/include/cskit/rng.hpp:13-79)
// so the same seed yields the same stream as the reference's own generator;
// tests/test_datagen.py pins it against oracle/_ref.
//
// Draw order, one Rng(seed) stream for the whole problem:
//   1. A[i][j] = normal()/sqrt(m), row-major (as gaussian_sensing_matrix,
//      sensing.cpp:36-58); optionally each column divided by its fp64 norm;
//      then rounded to fp32.
//   2. per signal b: support by partial Fisher-Yates on [0, n) with
//      uniform_below, then k values in support order:
//        law 0: normal()                      (configs 1, 2)
//        law 1: sign = uniform() < 0.5 ? -1 : +1, value = sign*(1 + uniform())
//                                             (config 3)
//   3. y = A x in fp64 from the fp32 A.
//   4. if snr_db >= 0: sigma_b = rms(A x_b) * 10^(-snr/20); noise normal(),
//      signal by signal, after all signals.
//   5. y rounded to fp32.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

class Rng {
 public:
  explicit Rng(uint64_t seed) {
    uint64_t x = seed;
    for (auto& w : s_) w = splitmix64(x);
  }
  uint64_t next_u64() {
    const uint64_t result = rotl(s_[0] + s_[3], 23) + s_[0];
    const uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return result;
  }
  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  uint64_t uniform_below(uint64_t bound) {
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
      const uint64_t r = next_u64();
      if (r >= threshold) return r % bound;
    }
  }
  double normal() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    double u, v, s;
    do {
      u = 2.0 * uniform() - 1.0;
      v = 2.0 * uniform() - 1.0;
      s = u * u + v * v;
    } while (s >= 1.0 || s == 0.0);
    const double f = std::sqrt(-2.0 * std::log(s) / s);
    spare_ = v * f;
    has_spare_ = true;
    return u * f;
  }

 private:
  static uint64_t splitmix64(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t s_[4] = {0, 0, 0, 0};
  double spare_ = 0.0;
  bool has_spare_ = false;
};

}  // namespace

extern "C" {

void cl_rng_draws(uint64_t seed, int kind, uint64_t bound, int64_t count,
                  double* out, uint64_t* out_u64) {
  Rng rng(seed);
  for (int64_t i = 0; i < count; ++i) {
    switch (kind) {
      case 0: out_u64[i] = rng.next_u64(); break;
      case 1: out[i] = rng.uniform(); break;
      case 2: out[i] = rng.normal(); break;
      default: out_u64[i] = rng.uniform_below(bound); break;
    }
  }
}

// A: m x n fp32 row-major; X: n x B fp64 row-major (may be NULL);
// Y: m x B fp32 row-major; supp: B x k int32 (support in draw order, may be NULL).
int cl_gen_problem_1d(uint64_t seed, int64_t m, int64_t n, int64_t k,
                      int64_t batch, int normalize, int value_law,
                      double snr_db, float* A, double* X, float* Y,
                      int32_t* supp) {
  if (m <= 0 || n <= 0 || batch <= 0 || k < 0 || k > n) return 3;
  Rng rng(seed);
  std::vector<double> a(static_cast<size_t>(m * n));
  const double scale = 1.0 / std::sqrt(static_cast<double>(m));
  for (auto& e : a) e = scale * rng.normal();
  if (normalize) {
    for (int64_t j = 0; j < n; ++j) {
      double s = 0.0;
      for (int64_t i = 0; i < m; ++i) s += a[i * n + j] * a[i * n + j];
      const double nrm = std::sqrt(s);
      if (nrm > 0.0)
        for (int64_t i = 0; i < m; ++i) a[i * n + j] /= nrm;
    }
  }
  for (int64_t e = 0; e < m * n; ++e) A[e] = static_cast<float>(a[e]);

  std::vector<int64_t> perm(static_cast<size_t>(n));
  std::vector<double> xs(static_cast<size_t>(k));
  std::vector<int64_t> sup(static_cast<size_t>(k * batch));
  std::vector<double> vals(static_cast<size_t>(k * batch));
  for (int64_t b = 0; b < batch; ++b) {
    for (int64_t j = 0; j < n; ++j) perm[j] = j;
    for (int64_t q = 0; q < k; ++q) {
      const int64_t r = q + static_cast<int64_t>(rng.uniform_below(
                                static_cast<uint64_t>(n - q)));
      const int64_t tmp = perm[q];
      perm[q] = perm[r];
      perm[r] = tmp;
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
  std::vector<double> y(static_cast<size_t>(m));
  std::vector<double> sig(static_cast<size_t>(batch), 0.0);
  std::vector<double> yall(static_cast<size_t>(m * batch));
  for (int64_t b = 0; b < batch; ++b) {
    for (int64_t q = 0; q < k; ++q) {
      if (X) X[sup[b * k + q] * batch + b] = vals[b * k + q];
      if (supp) supp[b * k + q] = static_cast<int32_t>(sup[b * k + q]);
    }
    double ss = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int64_t q = 0; q < k; ++q)
        acc += static_cast<double>(A[i * n + sup[b * k + q]]) * vals[b * k + q];
      yall[i * batch + b] = acc;
      ss += acc * acc;
    }
    sig[b] = std::sqrt(ss / static_cast<double>(m));
  }
  if (snr_db >= 0.0 && std::isfinite(snr_db)) {
    const double f = std::pow(10.0, -snr_db / 20.0);
    for (int64_t b = 0; b < batch; ++b) {
      const double sd = sig[b] * f;
      for (int64_t i = 0; i < m; ++i) yall[i * batch + b] += sd * rng.normal();
    }
  }
  for (int64_t e = 0; e < m * batch; ++e) Y[e] = static_cast<float>(yall[e]);
  return 0;
}

}  // extern "C"
