// fp32 -> fp64 conversion throughput: F2F.F64.F32 vs integer bit tricks.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ double f2d_full(float f) {
  const uint32_t u = __float_as_uint(f);
  const uint32_t sign = u & 0x80000000u;
  const uint32_t e = (u >> 23) & 0xffu;
  const uint32_t man_hi = (u >> 3) & 0x000FFFFFu;
  uint32_t hi = sign | ((e + 896u) << 20) | man_hi;
  uint32_t lo = u << 29;
  hi = (e == 0u) ? sign : hi;
  lo = (e == 0u) ? 0u : lo;
  hi = (e == 0xffu) ? (sign | 0x7FF00000u | man_hi) : hi;
  return __hiloint2double((int)hi, (int)lo);
}
__device__ __forceinline__ double f2d_lite(float f) {  // finite normals and zeros
  const uint32_t u = __float_as_uint(f);
  const uint32_t mag = u & 0x7fffffffu;
  uint32_t hi = (u & 0x80000000u) | ((mag >> 3) + (mag ? 0x38000000u : 0u));
  return __hiloint2double((int)hi, (int)(u << 29));
}
template <int V>
__global__ void k(const float* a, double* out, int iters) {
  float x[4];
  for (int q = 0; q < 4; ++q) x[q] = a[threadIdx.x + q];
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double d;
      if (V == 0) d = (double)x[q];
      else if (V == 1) d = f2d_full(x[q]);
      else d = f2d_lite(x[q]);
      if (q == 0) acc0 = fma(d, 1.0000001, acc0);
      if (q == 1) acc1 = fma(d, 1.0000001, acc1);
      if (q == 2) acc2 = fma(d, 1.0000001, acc2);
      if (q == 3) acc3 = fma(d, 1.0000001, acc3);
      x[q] = __uint_as_float(__float_as_uint(x[q]) ^ 1u);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}
int main() {
  float* a; double* o;
  cudaMalloc(&a, 4096 * 4); cudaMemset(a, 0x3f, 4096 * 4);
  cudaMalloc(&o, 148 * 8 * 256 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  const char* names[3] = {"F2F (double)x", "f2d full", "f2d lite"};
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (v == 0) k<0><<<148 * 8, 256>>>(a, o, iters);
      if (v == 1) k<1><<<148 * 8, 256>>>(a, o, iters);
      if (v == 2) k<2><<<148 * 8, 256>>>(a, o, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double conv = 148.0 * 8 * 256 * iters * 4;
      if (rep) printf("%-14s %.1f Gconv/s  (%.1f per SM-cycle @1.9GHz)\n", names[v], conv / ms / 1e6,
                      conv / ms / 1e6 / 148 / 1.9);
    }
  }
  return 0;
}
