// Microbenchmark: dependent-latency of DFMA / DADD / LDS.64 and fp64 throughput
// on this GPU (B200).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dfma(double* out, long long* cyc, double a, double b, int n) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}
__global__ void lat_dadd(double* out, long long* cyc, double a, double b, int n) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + b;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}
__global__ void lat_lds(double* out, long long* cyc, int n) {
  __shared__ int idx[64];
  idx[threadIdx.x] = (threadIdx.x + 1) & 31;
  __syncwarp();
  int j = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) j = idx[j];
  long long t1 = clock64();
  out[threadIdx.x] = j;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}
// throughput: many independent DFMA chains per warp, many warps
__global__ void thr_dfma(double* out, double a, double b, int n) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = a + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], b, a);
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 26); cudaMalloc(&cyc, 64);
  long long h; const int n = 4096;
  lat_dfma<<<1, 32>>>(out, cyc, 1.0, 0.999, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  lat_dfma<<<1, 32>>>(out, cyc, 1.0, 0.999, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / n);
  lat_dadd<<<1, 32>>>(out, cyc, 1.0, 0.999, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", (double)h / n);
  lat_lds<<<1, 32>>>(out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("LDS.32 dependent latency: %.2f cycles\n", (double)h / n);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 4096;
    thr_dfma<<<sms, warps * 32>>>(out, 1.0, 0.999, iters);
    cudaEventRecord(e0);
    thr_dfma<<<sms, warps * 32>>>(out, 1.0, 0.999, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)sms * warps * 32;
    printf("DFMA throughput %2d warps/SM: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  return 0;
}
