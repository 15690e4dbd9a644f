// k_corr_tc.cu — K1 on the tcgen05 tensor cores (3xTF32).  Placeholder until
// the kernel lands; the fp64 SIMT path in k_corr_f64.cu serves meanwhile.
#include "clomp_internal.cuh"

namespace clb {

namespace {
__global__ void k_split_tf32(const float* __restrict__ src, float* __restrict__ hi,
                             float* __restrict__ lo, int64_t count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const float x = src[i];
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  const float hf = __uint_as_float(h);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(x - hf));
  hi[i] = hf;
  lo[i] = __uint_as_float(l);
}
}  // namespace

bool corr_tc_available() { return false; }

void launch_corr_tc(const SolveParams&, const Work&, cudaStream_t) {}

void launch_split_tf32(const float* src, float* hi, float* lo, int64_t count,
                       cudaStream_t s) {
  const int64_t blocks = (count + 255) / 256;
  k_split_tf32<<<(unsigned)blocks, 256, 0, s>>>(src, hi, lo, count);
}

}  // namespace clb
