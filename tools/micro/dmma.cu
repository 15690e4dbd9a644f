// Does fp64 mma.sync (DMMA) exist on sm_100a, and how fast is it next to DFMA?
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int n) {
  double a = threadIdx.x * 0.001, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out, int n) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], 0.999, 1e-3);
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// both at once: half the warps DMMA, half DFMA
__global__ void k_mix(double* out, int n) {
  if ((threadIdx.x >> 5) & 1) {
    double x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < n * 4; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], 0.999, 1e-3);
    double s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  } else {
    double a = threadIdx.x * 0.001, b = 1.0;
    double c[8][2];
    for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
    for (int i = 0; i < n; ++i)
#pragma unroll
      for (int t = 0; t < 8; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    double s = 0;
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  }
}

int main() {
  double* out; cudaMalloc(&out, 1 << 26);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int n = 2048, threads = 512;
  float ms;
  k_dmma<<<sms, threads>>>(out, n);
  cudaEventRecord(e0); k_dmma<<<sms, threads>>>(out, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 256 * 8 * n * (double)sms * threads / 32;
  printf("DMMA m8n8k4: %.2f TFLOP/s (%s)\n", flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  k_dfma<<<sms, threads>>>(out, n);
  cudaEventRecord(e0); k_dfma<<<sms, threads>>>(out, n * 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  flops = 2.0 * 8 * n * 4 * (double)sms * threads;
  printf("DFMA: %.2f TFLOP/s\n", flops / ms / 1e9);
  cudaEventRecord(e0); k_mix<<<sms, threads>>>(out, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  flops = 2.0 * 256 * 8 * n * (double)sms * (threads / 2) / 32 + 2.0 * 8 * n * 4 * (double)sms * threads / 2;
  printf("mixed (half DMMA warps, half DFMA warps): %.2f TFLOP/s combined in %.3f ms\n", flops / ms / 1e9, ms);
  return 0;
}
