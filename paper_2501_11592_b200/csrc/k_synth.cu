// k_synth.cu — synthesis x_hat = D (s .* mask) on the device (clomp.cpp:289).
//
// The reference forms x_hat with a dense n x n x B product; here s is known by
// its compact support, so each signal costs n x count multiply-adds.  The
// basis is the context's atom-major copy dt[k][q] = D[q][k] (cl_set_basis),
// so consecutive threads read consecutive q of one atom row (coalesced).  The
// support is in ascending atom order (k_finalize), the order in which the
// reference's sequential-k product meets the non-zero terms (its zero terms
// add exactly 0), and every term is one fma as in its AVX2 GEMM
// (kernels_avx2.cpp:164-236).
#include "clomp_internal.cuh"

namespace clb {
namespace {

constexpr int kSynthThreads = 256;
constexpr int kSynthChunk = 64;  // support entries staged per pass

__global__ void k_synth(const double* __restrict__ dt, int64_t n, int64_t out_cap,
                        const int32_t* __restrict__ sup, const double* __restrict__ coef,
                        const int32_t* __restrict__ cnt, double* __restrict__ xhat) {
  __shared__ int32_t s_idx[kSynthChunk];
  __shared__ double s_c[kSynthChunk];
  const int64_t b = blockIdx.y;
  const int64_t q = (int64_t)blockIdx.x * kSynthThreads + threadIdx.x;
  const int t = min((int64_t)cnt[b], out_cap);
  double acc = 0.0;
  for (int k0 = 0; k0 < t; k0 += kSynthChunk) {
    const int kn = min(kSynthChunk, t - k0);
    __syncthreads();
    if ((int)threadIdx.x < kn) {
      s_idx[threadIdx.x] = sup[b * out_cap + k0 + threadIdx.x];
      s_c[threadIdx.x] = coef[b * out_cap + k0 + threadIdx.x];
    }
    __syncthreads();
    if (q < n)
      for (int k = 0; k < kn; ++k) acc = fma(dt[(int64_t)s_idx[k] * n + q], s_c[k], acc);
  }
  if (q < n) xhat[b * n + q] = acc;
}

}  // namespace

void launch_synth(const double* dt, int64_t n, int64_t B, int64_t out_cap, const int32_t* sup,
                  const double* coef, const int32_t* cnt, double* xhat, cudaStream_t s) {
  if (B <= 0 || n <= 0) return;
  // grid.y carries the batch (<= 65535 per launch)
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    const int64_t nb = B - b0 < 65535 ? B - b0 : 65535;
    dim3 grid((unsigned)((n + kSynthThreads - 1) / kSynthThreads), (unsigned)nb);
    k_synth<<<grid, kSynthThreads, 0, s>>>(dt, n, out_cap, sup + b0 * out_cap, coef + b0 * out_cap,
                                           cnt + b0, xhat + b0 * n);
  }
}

}  // namespace clb
