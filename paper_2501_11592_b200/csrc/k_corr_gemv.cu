// k_corr_gemv.cu — K1b: scores = A^T r for a handful of residuals (B <= 4).
//
// Replaces la::matmul(ops.at, r) + inject_from_scores' max scan
// (clomp.cpp:245, clomp.cpp:41-53) on the per-signal path: the CLI solves one
// signal at a time (cskit.cpp:543-551 -> clomp_solve, clomp.cpp:294-311), where
// the reference's GEMM degenerates to its leftover-column loop
// (kernels_avx2.cpp:225-235).  On B200 that is an HBM-bound GEMV: every byte of
// the fp32 dictionary is read once per outer iteration and each element feeds
// NB fp64 FMAs, far below the fp64 pipe's balance point.
//
// Layout: dictionary atom-major at32[n][ldm] (fp32), residuals r64[B][ldm].
// One CTA per (64-atom candidate tile, group of NB signals).  The measurement
// axis is split over the CTA's G warps: warp w owns columns
// [w*128V, (w+1)*128V), lane l the float4s at w*128V + 4*(l + 32v), v < V, so
// every load instruction of a warp reads 512 contiguous bytes and the
// residual slice a lane needs for its columns (4V values per signal) lives in
// registers for the whole kernel.  Atoms go through in batches of 4: 4V
// independent 16-byte loads per lane in flight, fp32 -> fp64 conversion, fp64
// FMAs, then a transposed butterfly reduction across the warp (P = 4*NB
// partial dots in P-1 + 5-log2(P) shuffles instead of 5P) and one shared-memory
// slot per (dot, warp).  Warp 0 sums the G warp partials in a fixed order
// (deterministic), takes |.| and feeds the running candidate record of each
// signal (two best atoms + third value, lowest atom wins exact ties — the
// same records k_corr_f64 / k_corr_tc emit), double-buffered so the other
// warps stream the next batch meanwhile.  With `scores` the |scores| are also
// written for the th < 1 threshold pass.
#include "clomp_internal.cuh"

namespace clb {
namespace {

constexpr unsigned kFull = 0xffffffffu;

constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

// Atoms per batch: at most 16 float4 loads in flight per lane (64 registers),
// fewer partial dots when NB = 4 keeps more residual registers live.
constexpr int apb_for(int nb, int v) {
  return (16 / v < 4 ? (16 / v < 1 ? 1 : 16 / v) : 4) > (nb >= 4 ? 2 : 4)
             ? (nb >= 4 ? 2 : 4)
             : (16 / v < 4 ? (16 / v < 1 ? 1 : 16 / v) : 4);
}

// Transposed butterfly: v[0..P) partial sums per lane -> lane l ends with the
// warp total of entry idx(l) = l >> (5 - log2 P), in every lane of its group.
template <int P>
__device__ __forceinline__ double warp_reduce_transposed(double (&v)[P], int lane) {
#pragma unroll
  for (int h = P / 2, o = 16; h >= 1; h >>= 1, o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = up ? v[i] : v[i + h];
      const double keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(kFull, send, o);
    }
  }
  constexpr int kLogP = ilog2(P);
  double x = v[0];
#pragma unroll
  for (int o = 16 >> kLogP; o >= 1; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

template <int NB, int V>
__global__ void __launch_bounds__(512, 1)
k_corr_gemv(const float* __restrict__ at, const double* __restrict__ r,
            const int32_t* __restrict__ active, int64_t n, int64_t B, int64_t ldm,
            int64_t ntile, Cand* __restrict__ cand, double* __restrict__ scores) {
  constexpr int kAPB = apb_for(NB, V);
  constexpr int P = kAPB * NB;  // partial dots per batch: index a * NB + b
  constexpr int kTile = kCorrTileAtoms;
  __shared__ double part[2][P][17];
  __shared__ int any_active;

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int G = blockDim.x >> 5;
  const int64_t tile = blockIdx.x;
  const int64_t b0 = (int64_t)blockIdx.y * NB;

  if (threadIdx.x == 0) {
    int a = 0;
    for (int b = 0; b < NB; ++b)
      if (b0 + b < B && active[b0 + b]) a = 1;
    any_active = a;
  }
  __syncthreads();
  if (!any_active) return;

  // Residual slice in registers (zero for padding signals).
  const int64_t col0 = (int64_t)warp * 128 * V + 4 * lane;
  double rr[NB][V][4];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int v = 0; v < V; ++v) {
      double2 x01 = make_double2(0.0, 0.0), x23 = make_double2(0.0, 0.0);
      if (b0 + b < B) {
        const double2* rp = reinterpret_cast<const double2*>(r + (b0 + b) * ldm + col0 + 128 * v);
        x01 = rp[0];
        x23 = rp[1];
      }
      rr[b][v][0] = x01.x;
      rr[b][v][1] = x01.y;
      rr[b][v][2] = x23.x;
      rr[b][v][3] = x23.y;
    }

  const int64_t j_begin = tile * kTile;
  const int64_t j_end = min(n, j_begin + kTile);
  double c1 = -1.0, c2 = -1.0, c3 = -1.0;  // warp 0, lane b < NB: running record
  int i1 = 0x7fffffff, i2 = 0x7fffffff;

  int buf = 0;
  for (int64_t j0 = j_begin; j0 < j_end; j0 += kAPB, buf ^= 1) {
    float4 a[kAPB][V];
#pragma unroll
    for (int k = 0; k < kAPB; ++k) {
      const int64_t j = j0 + k < j_end ? j0 + k : j_end - 1;  // clamp: duplicate, ignored below
      const float4* ap = reinterpret_cast<const float4*>(at + j * ldm + col0);
#pragma unroll
      for (int v = 0; v < V; ++v) a[k][v] = __ldg(ap + 32 * v);
    }
    double acc[P];
#pragma unroll
    for (int k = 0; k < kAPB; ++k)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        double s = 0.0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          s = fma(f2d(a[k][v].x), rr[b][v][0], s);
          s = fma(f2d(a[k][v].y), rr[b][v][1], s);
          s = fma(f2d(a[k][v].z), rr[b][v][2], s);
          s = fma(f2d(a[k][v].w), rr[b][v][3], s);
        }
        acc[k * NB + b] = s;
      }
    const double tot = warp_reduce_transposed<P>(acc, lane);
    constexpr int kShift = 5 - ilog2(P);
    if ((lane & ((1 << kShift) - 1)) == 0) part[buf][lane >> kShift][warp] = tot;
    __syncthreads();
    if (warp == 0) {
      // Lane t < P: dot t summed over the warps in ascending order.
      double sc = 0.0;
      if (lane < P) {
        for (int g = 0; g < G; ++g) sc += part[buf][lane][g];
        sc = fabs(sc);
        const int k = lane / NB, b = lane % NB;
        if (scores && j0 + k < j_end && b0 + b < B) scores[(b0 + b) * n + j0 + k] = sc;
      }
      // Lane b < NB inserts its signal's APB scores in ascending atom order.
#pragma unroll
      for (int k = 0; k < kAPB; ++k) {
        const double x = __shfl_sync(kFull, sc, (k * NB + lane) & 31);
        if (lane < NB && j0 + k < j_end) cand_insert(c1, i1, c2, i2, c3, x, (int)(j0 + k));
      }
    }
  }
  if (warp == 0 && lane < NB && b0 + lane < B) {
    Cand c;
    c.v1 = c1;
    c.v2 = c2;
    c.v3 = c3;
    c.i1 = i1;
    c.i2 = i2;
    cand[(b0 + lane) * ntile + tile] = c;
  }
}

template <int NB, int V>
void launch_nb(const SolveParams& p, const Work& w, bool full_scores, cudaStream_t s) {
  const int G = (int)(p.ldm / (128 * V));
  dim3 grid((unsigned)p.ntl, (unsigned)((p.B + NB - 1) / NB));
  k_corr_gemv<NB, V><<<grid, 32 * G, 0, s>>>(w.at32 + p.atom0 * p.ldm, w.r64, w.active,
                                             p.n_corr, p.B, p.ldm, p.ntl, w.cand,
                                             full_scores ? w.scores : nullptr);
}

// Float4s per lane: the largest power of two <= pref that divides the
// measurement axis into <= 16 warp slices, else the smallest larger one that
// does; 0 when none keeps NB * V <= 8 (residual registers per lane: 8 NB V).
int pick_v(int64_t ldm, int nb, int pref) {
  for (int v = pref; v >= 1; v /= 2)
    if (ldm % (128 * v) == 0 && ldm / (128 * v) <= 16) return v;
  for (int v = pref * 2; nb * v <= 8; v *= 2)
    if (ldm % (128 * v) == 0 && ldm / (128 * v) <= 16) return v;
  return 0;
}

int nb_for(int64_t B) { return B <= 1 ? 1 : B <= 2 ? 2 : 4; }
int pref_for(int nb) { return nb == 1 ? 4 : 2; }

}  // namespace

bool corr_gemv_supported(int64_t ldm, int64_t B) {
  if (B < 1 || B > 4 || ldm % 128 != 0) return false;
  const int nb = nb_for(B);
  return pick_v(ldm, nb, pref_for(nb)) != 0;
}

void launch_corr_gemv(const SolveParams& p, const Work& w, bool full_scores, cudaStream_t s) {
  const int nb = nb_for(p.B);
  const int v = pick_v(p.ldm, nb, pref_for(nb));
#define CL_GEMV_CASE(NB_, V_) \
  if (nb == NB_ && v == V_) return launch_nb<NB_, V_>(p, w, full_scores, s);
  CL_GEMV_CASE(1, 1) CL_GEMV_CASE(1, 2) CL_GEMV_CASE(1, 4) CL_GEMV_CASE(1, 8)
  CL_GEMV_CASE(2, 1) CL_GEMV_CASE(2, 2) CL_GEMV_CASE(2, 4)
  CL_GEMV_CASE(4, 1) CL_GEMV_CASE(4, 2)
#undef CL_GEMV_CASE
}

}  // namespace clb
