// k_gram.cu — the dictionary Gram matrix G = A^T A in fp64, built once per
// context.
//
// The learning step needs, for every newly injected atom j, the Gram row
// G[S, j] (A_S^T A_S c - A_S^T y is the reference gradient A^T (A s - y)
// restricted to the mask, clomp.cpp:84-91, 120-122).  Computing those rows on
// demand re-streams t atoms of M floats per signal per outer iteration; with
// G precomputed the row is a gather of t doubles.  Products of two fp32 values
// are exact in fp64 and are summed with FMA in fp64, so G holds the same
// values the on-demand path would compute.
//
// Tiling: 64 x 64 output tiles, 16-deep K slices staged through shared memory,
// 4 x 4 register block per thread; only tiles on or above the diagonal are
// computed and mirrored.
#include "clomp_internal.cuh"

namespace clb {
namespace {

constexpr int T = 64;
constexpr int KB = 16;

__global__ void __launch_bounds__(256)
k_gram_full(const float* __restrict__ at, int64_t n, int64_t ldm, double* __restrict__ g) {
  if (blockIdx.y > blockIdx.x) return;  // lower triangle mirrored below
  __shared__ double As[KB][T + 2];
  __shared__ double Bs[KB][T + 2];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t i0 = (int64_t)blockIdx.y * T, j0 = (int64_t)blockIdx.x * T;
  const int lrow = tid >> 2, lk = (tid & 3) * 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t k0 = 0; k0 < ldm; k0 += KB) {
    float4 av = make_float4(0.f, 0.f, 0.f, 0.f), bv = av;
    if (i0 + lrow < n) av = *reinterpret_cast<const float4*>(at + (i0 + lrow) * ldm + k0 + lk);
    if (j0 + lrow < n) bv = *reinterpret_cast<const float4*>(at + (j0 + lrow) * ldm + k0 + lk);
    As[lk + 0][lrow] = av.x;
    As[lk + 1][lrow] = av.y;
    As[lk + 2][lrow] = av.z;
    As[lk + 3][lrow] = av.w;
    Bs[lk + 0][lrow] = bv.x;
    Bs[lk + 1][lrow] = bv.y;
    Bs[lk + 2][lrow] = bv.z;
    Bs[lk + 3][lrow] = bv.w;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = As[k][ty * 4 + q];
        b[q] = Bs[k][tx * 4 + q];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int64_t i = i0 + ty * 4 + x, j = j0 + tx * 4 + y;
      if (i < n && j < n) {
        g[i * n + j] = acc[x][y];
        g[j * n + i] = acc[x][y];
      }
    }
}

}  // namespace

void launch_gram_full(const float* at, int64_t n, int64_t ldm, double* g,
                      cudaStream_t s) {
  const unsigned tiles = (unsigned)((n + T - 1) / T);
  k_gram_full<<<dim3(tiles, tiles), 256, 0, s>>>(at, n, ldm, g);
}

}  // namespace clb
