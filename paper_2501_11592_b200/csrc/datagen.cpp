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

// dct_basis (sensing.cpp:13-29): orthonormal DCT-II, d[j][k] = c_k cos(pi(2j+1)k/(2n)).
static void dct(int64_t n, std::vector<double>& d) {
  d.assign(static_cast<size_t>(n * n), 0.0);
  const double c0 = std::sqrt(1.0 / static_cast<double>(n));
  const double ck = std::sqrt(2.0 / static_cast<double>(n));
  const double base = 3.14159265358979323846 / (2.0 * static_cast<double>(n));
  for (int64_t j = 0; j < n; ++j) {
    const double phase = static_cast<double>(2 * j + 1) * base;
    for (int64_t k = 0; k < n; ++k)
      d[j * n + k] = (k == 0 ? c0 : ck) * std::cos(phase * static_cast<double>(k));
  }
}

// The synthesis basis of make_setup problems (x = D s), for cl_set_basis.
int cl_dct_basis(int64_t n, double* out) {
  if (n <= 0 || !out) return 3;
  std::vector<double> d;
  dct(n, d);
  std::memcpy(out, d.data(), sizeof(double) * d.size());
  return 0;
}

// Separable 2D problem (BASELINE configs 4-5):
//   Phi_r (m_r x n_r), Phi_c (m_c x n_c) i.i.d. normal()/sqrt(m), row-major;
//   A_r = fp32(Phi_r D_r), A_c = fp32(Phi_c D_c) with D the orthonormal DCT;
//   per image: k positions of the n_r x n_c coefficient grid by partial
//   Fisher-Yates, values normal() / (1 + i + j) at frequency (i, j);
//   Y = A_r S A_c^T in fp64, rounded to fp32.
// Column-major vec: p = i + n_r j (S), q = qr + m_r qc (Y).
// Outputs: Ar m_r x n_r, Ac m_c x n_c (fp32 row-major), S (n_r n_c) x B fp64
// (may be NULL), Y (m_r m_c) x B fp32.
int cl_gen_problem_2d(uint64_t seed, int64_t n_r, int64_t n_c, int64_t m_r, int64_t m_c,
                      int64_t k, int64_t batch, float* Ar, float* Ac, double* S, float* Y) {
  const int64_t N = n_r * n_c, M = m_r * m_c;
  if (n_r <= 0 || n_c <= 0 || m_r <= 0 || m_c <= 0 || batch <= 0 || k < 0 || k > N) return 3;
  Rng rng(seed);
  std::vector<double> phr(static_cast<size_t>(m_r * n_r)), phc(static_cast<size_t>(m_c * n_c));
  for (auto& e : phr) e = rng.normal() / std::sqrt(static_cast<double>(m_r));
  for (auto& e : phc) e = rng.normal() / std::sqrt(static_cast<double>(m_c));
  std::vector<double> dr, dc;
  dct(n_r, dr);
  dct(n_c, dc);
  std::vector<double> ar(static_cast<size_t>(m_r * n_r)), ac(static_cast<size_t>(m_c * n_c));
  for (int64_t i = 0; i < m_r; ++i)
    for (int64_t j = 0; j < n_r; ++j) {
      double acc = 0.0;
      for (int64_t t = 0; t < n_r; ++t) acc += phr[i * n_r + t] * dr[t * n_r + j];
      Ar[i * n_r + j] = static_cast<float>(acc);
      ar[i * n_r + j] = Ar[i * n_r + j];
    }
  for (int64_t i = 0; i < m_c; ++i)
    for (int64_t j = 0; j < n_c; ++j) {
      double acc = 0.0;
      for (int64_t t = 0; t < n_c; ++t) acc += phc[i * n_c + t] * dc[t * n_c + j];
      Ac[i * n_c + j] = static_cast<float>(acc);
      ac[i * n_c + j] = Ac[i * n_c + j];
    }
  if (S) std::memset(S, 0, sizeof(double) * N * batch);
  std::vector<int64_t> perm(static_cast<size_t>(N));
  std::vector<double> v(static_cast<size_t>(m_r * n_c));
  for (int64_t b = 0; b < batch; ++b) {
    for (int64_t p = 0; p < N; ++p) perm[p] = p;
    for (int64_t q = 0; q < k; ++q) {
      const int64_t r = q + static_cast<int64_t>(rng.uniform_below(static_cast<uint64_t>(N - q)));
      const int64_t tmp = perm[q];
      perm[q] = perm[r];
      perm[r] = tmp;
    }
    std::fill(v.begin(), v.end(), 0.0);  // V = A_r S  (m_r x n_c)
    for (int64_t q = 0; q < k; ++q) {
      const int64_t p = perm[q], i = p % n_r, j = p / n_r;
      const double val = rng.normal() / (1.0 + static_cast<double>(i + j));
      if (S) S[p * batch + b] = val;
      for (int64_t qr = 0; qr < m_r; ++qr) v[qr * n_c + j] += ar[qr * n_r + i] * val;
    }
    for (int64_t qc = 0; qc < m_c; ++qc)
      for (int64_t qr = 0; qr < m_r; ++qr) {
        double acc = 0.0;
        for (int64_t j = 0; j < n_c; ++j) acc += v[qr * n_c + j] * ac[qc * n_c + j];
        Y[(qr + m_r * qc) * batch + b] = static_cast<float>(acc);
      }
  }
  return 0;
}

}  // extern "C"
