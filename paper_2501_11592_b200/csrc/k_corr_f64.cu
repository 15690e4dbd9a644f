// k_corr_f64.cu — K1 (fp64 path): scores = A^T R for a batch of residuals.
//
// Replaces la::matmul(ops.at, r) + inject_from_scores' max scan
// (clomp.cpp:245, clomp.cpp:41-53).  fp64 FMA accumulation of fp32 atoms and
// fp64 residuals; the epilogue keeps, per (atom tile, signal), the largest and
// second-largest |score| and the argmax, so the full N x B score matrix never
// touches HBM on the th == 1 path.  With th < 1 the |scores| are written out
// for the threshold pass (clomp.cpp:49-51).
//
// This is the exact-scores path: it serves th < 1, the unit-level
// cl_inject_support and GPUs without the tcgen05 kernel.  The th == 1 solve
// path uses k_corr_tc.cu (3xTF32 on tcgen05) and falls back to an fp64 rescan
// only for near-tied selections.
#include "clomp_internal.cuh"

namespace clb {
namespace {

constexpr int BM = kCorrTileAtoms;
constexpr int BN = kCorrTileSignals;
constexpr int BK = 16;

__global__ void __launch_bounds__(256)
k_corr_f64(const float* __restrict__ at, const double* __restrict__ r,
           const int32_t* __restrict__ active, int64_t n, int64_t B,
           int64_t ldm, int64_t ntile, Cand* __restrict__ cand,
           double* __restrict__ scores) {
  __shared__ double As[BK][BM + 2];
  __shared__ double Rs[BK][BN + 2];
  __shared__ Cand red[8][BN];

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t j0 = (int64_t)blockIdx.x * BM;
  const int64_t b0 = (int64_t)blockIdx.y * BN;

  // Skip tiles whose signals are all finished.
  __shared__ int any_active;
  if (tid == 0) any_active = 0;
  __syncthreads();
  if (tid < BN && b0 + tid < B && active[b0 + tid]) any_active = 1;
  __syncthreads();
  if (!any_active) return;

  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) acc[i][jj] = 0.0;

  const int lrow = tid >> 2;        // 0..63
  const int lk = (tid & 3) * 4;     // 0,4,8,12
  const int64_t arow = j0 + lrow;
  const int64_t rrow = b0 + lrow;

  for (int64_t k0 = 0; k0 < ldm; k0 += BK) {
    float4 av = make_float4(0.f, 0.f, 0.f, 0.f);
    if (arow < n) av = *reinterpret_cast<const float4*>(at + arow * ldm + k0 + lk);
    double2 r01 = make_double2(0.0, 0.0), r23 = make_double2(0.0, 0.0);
    if (rrow < B) {
      const double2* rp = reinterpret_cast<const double2*>(r + rrow * ldm + k0 + lk);
      r01 = rp[0];
      r23 = rp[1];
    }
    As[lk + 0][lrow] = av.x;
    As[lk + 1][lrow] = av.y;
    As[lk + 2][lrow] = av.z;
    As[lk + 3][lrow] = av.w;
    Rs[lk + 0][lrow] = r01.x;
    Rs[lk + 1][lrow] = r01.y;
    Rs[lk + 2][lrow] = r23.x;
    Rs[lk + 3][lrow] = r23.y;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      double a[4], rv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) rv[jj] = Rs[k][tx * 4 + jj];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][jj] = fma(a[i], rv[jj], acc[i][jj]);
    }
    __syncthreads();
  }

  if (scores) {
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int64_t b = b0 + tx * 4 + jj;
      if (b >= B) continue;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t j = j0 + ty * 4 + i;
        if (j < n) scores[b * n + j] = fabs(acc[i][jj]);
      }
    }
  }

  // Per-signal candidate record over this thread's 4 atoms (ascending, so the
  // lowest atom wins an exact tie), then across the 16 ty rows (two rounds
  // through an 8-row shared buffer).
  Cand c[4];
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    c[jj] = cand_empty();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t j = j0 + ty * 4 + i;
      if (j < n) cand_insert(c[jj].v1, c[jj].i1, c[jj].v2, c[jj].i2, c[jj].v3, fabs(acc[i][jj]), (int)j);
    }
  }
  if (ty >= 8)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) red[ty - 8][tx * 4 + jj] = c[jj];
  __syncthreads();
  if (ty < 8)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      cand_merge(c[jj], red[ty][tx * 4 + jj]);
      red[ty][tx * 4 + jj] = c[jj];
    }
  __syncthreads();
  if (tid < BN) {
    const int64_t b = b0 + tid;
    if (b < B) {
      Cand m = red[0][tid];
      for (int t = 1; t < 8; ++t) cand_merge(m, red[t][tid]);
      cand[b * ntile + blockIdx.x] = m;
    }
  }
}

}  // namespace

void launch_corr_f64(const SolveParams& p, const Work& w, bool full_scores,
                     cudaStream_t s) {
  // Column shard: atoms [atom0, atom0 + n_corr) into ntl local tiles (the
  // candidate indices are shifted back to global atom numbers by the caller's
  // exchange; single-GPU: atom0 = 0, n_corr = n, ntl = ntile).
  dim3 grid((unsigned)((p.n_corr + BM - 1) / BM), (unsigned)((p.B + BN - 1) / BN));
  k_corr_f64<<<grid, 256, 0, s>>>(w.at32 + p.atom0 * p.ldm, w.r64, w.active, p.n_corr, p.B,
                                  p.ldm, p.ntl, w.cand, full_scores ? w.scores : nullptr);
}

}  // namespace clb
