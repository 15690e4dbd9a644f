// Broadcast-read throughput of shared memory vs SHFL (one consumer LOP3 per
// two loaded 32-bit words so the ALU is not the limiter).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned lop3x(unsigned a, unsigned b, unsigned c) {
  unsigned d;
  asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

template <int MODE>
__global__ void k(unsigned* out, int n, long long* cyc) {
  __shared__ __align__(16) unsigned buf[4][128];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 512; i += blockDim.x) (&buf[0][0])[i] = i * 2654435761u;
  __syncthreads();
  unsigned x = lane;
  const int grp = MODE == 2 ? (lane >> 4) : (MODE == 3 ? (lane >> 3) : 0);
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int j = 0; j < 64; j += 4) {
      if (MODE == 0) {  // LDS.128 bcast: 4 words
        uint4 c = *reinterpret_cast<const uint4*>(&buf[0][j + (it & 1)]);
        x = lop3x(x, c.x, c.z);
      } else if (MODE >= 1 && MODE <= 3) {  // LDS.64 with 1/2/4 addresses: 2 loads
        uint2 a = *reinterpret_cast<const uint2*>(&buf[grp][j + (it & 1) * 2]);
        uint2 b = *reinterpret_cast<const uint2*>(&buf[grp][j + 2 + (it & 1) * 2]);
        x = lop3x(x, a.x, b.x);
      } else {  // 2 SHFL of 32-bit (one double's worth)
        unsigned a = __shfl_sync(0xffffffff, x + j, j & 31);
        unsigned b = __shfl_sync(0xffffffff, x + j + 1, (j + 1) & 31);
        x = lop3x(x, a, b);
      }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  unsigned* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // per iteration: 16 "steps"; bytes broadcast per step: LDS.128 16B; LDS.64 x2 16B; SHFL x2 8B
  const char* names[] = {"LDS.128 bcast", "LDS.64 bcast", "LDS.64 2-addr", "LDS.64 4-addr", "SHFL x2"};
  const double doubles_per_step[] = {2, 2, 2, 2, 1};
  const int n = 512, warps = 16;
  for (int mode = 0; mode < 5; ++mode) {
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      switch (mode) {
        case 0: k<0><<<sms, warps * 32>>>(out, n, cyc); break;
        case 1: k<1><<<sms, warps * 32>>>(out, n, cyc); break;
        case 2: k<2><<<sms, warps * 32>>>(out, n, cyc); break;
        case 3: k<3><<<sms, warps * 32>>>(out, n, cyc); break;
        default: k<4><<<sms, warps * 32>>>(out, n, cyc); break;
      }
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    }
    const double steps = (double)n * 16 * warps;
    printf("%-14s: %.3f SM-cycles per step, %.3f SM-cycles per broadcast double per warp\n",
           names[mode], h / steps, h / steps / doubles_per_step[mode]);
  }
  return 0;
}
