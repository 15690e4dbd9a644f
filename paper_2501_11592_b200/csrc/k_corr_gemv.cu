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
// Persistent grid, one CTA per SM, each streaming a contiguous range of
// candidate tiles (kGemvTile atoms each).  A producer warp keeps a ring of
// shared-memory stages full with one TMA bulk copy per stage (SA consecutive
// atom rows are contiguous in HBM), completing on the stage's mbarrier, so
// ~190 KB per SM are always in flight independent of the consumers.  The
// measurement axis is split over the G consumer warps: warp w owns columns
// [w*128V, (w+1)*128V), lane l the float4s at w*128V + 4*(l + 32v), v < V
// (conflict-free 512-byte shared-memory reads), and the residual slice those
// columns need (4V values per signal) lives in registers for the whole
// kernel.  Atoms go through in batches of APB: fp32 -> fp64 conversion, fp64
// FMAs, a transposed butterfly reduction across the warp (P = APB*NB partial
// dots in P-1 + 5-log2(P) shuffles instead of 5P) and one shared-memory slot
// per (dot, warp).  Warp 0 sums the G warp partials in a fixed order
// (deterministic), takes |.| and feeds each signal's running candidate record
// (two best atoms + third value, lowest atom wins exact ties — the records
// k_corr_f64 / k_corr_tc emit), double-buffered so the other warps go on with
// the next batch.  With `scores` the |scores| are also written (th < 1).
#include <algorithm>

#include "clomp_internal.cuh"

namespace clb {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kGemvTile = 16;      // atoms per candidate record on this path
constexpr int kMaxStages = 8;
constexpr int kRingBytes = 192 * 1024;

constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

// Atoms per register batch: at most 8 float4s per lane in flight.
constexpr int apb_for(int nb, int v) { return (8 / v) < 1 ? 1 : (8 / v); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
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
  double x = v[0];
#pragma unroll
  for (int o = 16 >> ilog2(P); o >= 1; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

template <int NB, int V>
__global__ void __launch_bounds__(32 * 10, 1)
k_corr_gemv(const float* __restrict__ at, const double* __restrict__ r,
            const int32_t* __restrict__ active, int64_t n, int64_t B, int64_t ldm,
            int64_t ntile, int sa, int stages, Cand* __restrict__ cand,
            double* __restrict__ scores) {
  constexpr int APB = apb_for(NB, V);
  constexpr int P = APB * NB;  // partial dots per batch: index k * NB + b
  extern __shared__ __align__(128) unsigned char ring[];
  // full/empty: atom-row stages (producer -> consumers); pfull/pempty: the
  // per-stage partial-dot slots (consumers -> merger).
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages], pfull[kMaxStages],
      pempty[kMaxStages];

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int G = (blockDim.x >> 5) - 2;  // consumer warps; warp G produces, G+1 merges
  const int64_t t_lo = (int64_t)blockIdx.x * ntile / gridDim.x;
  const int64_t t_hi = (int64_t)(blockIdx.x + 1) * ntile / gridDim.x;
  const int64_t j_lo = t_lo * kGemvTile;
  const int64_t j_hi = min(n, t_hi * kGemvTile);
  if (j_lo >= j_hi) return;
  {
    int a = 0;
    for (int b = 0; b < NB; ++b)
      if (b < B && active[b]) a = 1;
    if (!a) return;  // uniform: every thread reads the same flags
  }
  const int64_t row_bytes = ldm * 4;
  // partial slots after the row stages: [stage][sa * NB][G] doubles
  double* part = reinterpret_cast<double*>(ring + (size_t)stages * sa * row_bytes);
  const int slot = sa * NB * G;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(G));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&pfull[s])), "r"(G));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&pempty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == G) {
    // ---------------- producer: one bulk copy of SA atom rows per stage
    if (lane == 0) {
      int st = 0;
      for (int64_t j = j_lo; j < j_hi; j += sa, ++st) {
        const int s = st % stages;
        mbar_wait(&empty[s], ((st / stages) & 1) ^ 1);
        const uint32_t bytes = (uint32_t)(min((int64_t)sa, j_hi - j) * row_bytes);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         smem_u32(&full[s])),
                     "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(ring + (size_t)s * sa * row_bytes)),
            "l"(at + j * ldm), "r"(bytes), "r"(smem_u32(&full[s]))
            : "memory");
      }
    }
    return;
  }

  if (warp == G + 1) {
    // ---------------- merger: warp sums in a fixed order, |.|, candidate
    // records (lane b < NB inserts its signal's scores in ascending atoms and
    // emits the record at the end of every candidate tile)
    double c1 = -1.0, c2 = -1.0, c3 = -1.0;
    int i1 = 0x7fffffff, i2 = 0x7fffffff;
    int st = 0;
    for (int64_t j = j_lo; j < j_hi; j += sa, ++st) {
      const int s = st % stages;
      mbar_wait(&pfull[s], (st / stages) & 1);
      const int na = (int)min((int64_t)sa, j_hi - j);
      const double* ps = part + (size_t)s * slot;
      for (int q0 = 0; q0 < na * NB; q0 += 32) {
        const int q = q0 + lane;  // dot q = k * NB + b
        double sc = 0.0;
        if (q < na * NB) {
          for (int g = 0; g < G; ++g) sc += ps[q * G + g];
          sc = fabs(sc);
          if (scores && q % NB < B) scores[(q % NB) * n + j + q / NB] = sc;
        }
        const int kmax = min(32 / NB, na - q0 / NB);
        for (int k = 0; k < kmax; ++k) {
          const double x = __shfl_sync(kFull, sc, (k * NB + lane) & 31);
          const int64_t jj = j + q0 / NB + k;
          if (lane < NB) {
            cand_insert(c1, i1, c2, i2, c3, x, (int)jj);
            if ((jj + 1) % kGemvTile == 0 || jj + 1 == j_hi) {
              if (lane < B) {
                Cand c;
                c.v1 = c1;
                c.v2 = c2;
                c.v3 = c3;
                c.i1 = i1;
                c.i2 = i2;
                cand[lane * ntile + jj / kGemvTile] = c;
              }
              c1 = c2 = c3 = -1.0;
              i1 = i2 = 0x7fffffff;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                         smem_u32(&pempty[s]))
                     : "memory");
    }
    return;
  }

  // ---------------- consumers
  const int col0 = warp * 128 * V + 4 * lane;
  double rr[NB][V][4];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int v = 0; v < V; ++v) {
      double2 x01 = make_double2(0.0, 0.0), x23 = make_double2(0.0, 0.0);
      if (b < B) {
        const double2* rp = reinterpret_cast<const double2*>(r + b * ldm + col0 + 128 * v);
        x01 = rp[0];
        x23 = rp[1];
      }
      rr[b][v][0] = x01.x;
      rr[b][v][1] = x01.y;
      rr[b][v][2] = x23.x;
      rr[b][v][3] = x23.y;
    }

  int st = 0;
  for (int64_t j = j_lo; j < j_hi; j += sa, ++st) {
    const int s = st % stages;
    const uint32_t ph = (st / stages) & 1;
    mbar_wait(&full[s], ph);
    mbar_wait(&pempty[s], ph ^ 1);  // the merger is done with this partial slot
    const int na = (int)min((int64_t)sa, j_hi - j);
    const float* stg = reinterpret_cast<const float*>(ring + (size_t)s * sa * row_bytes);
    double* ps = part + (size_t)s * slot;
    for (int k0 = 0; k0 < na; k0 += APB) {
      float4 a[APB][V];
#pragma unroll
      for (int k = 0; k < APB; ++k) {
        const int kk = k0 + k < na ? k0 + k : na - 1;  // clamp: duplicate, dropped below
        const float4* ap = reinterpret_cast<const float4*>(stg + (int64_t)kk * ldm + col0);
#pragma unroll
        for (int v = 0; v < V; ++v) a[k][v] = ap[32 * v];
      }
      if (k0 + APB >= na) {  // stage consumed by this warp: release the rows
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                           smem_u32(&empty[s]))
                       : "memory");
      }
      double acc[P];
#pragma unroll
      for (int k = 0; k < APB; ++k)
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          double x = 0.0;
#pragma unroll
          for (int v = 0; v < V; ++v) {
            x = fma(f2d(a[k][v].x), rr[b][v][0], x);
            x = fma(f2d(a[k][v].y), rr[b][v][1], x);
            x = fma(f2d(a[k][v].z), rr[b][v][2], x);
            x = fma(f2d(a[k][v].w), rr[b][v][3], x);
          }
          acc[k * NB + b] = x;
        }
      const double tot = warp_reduce_transposed<P>(acc, lane);
      constexpr int kShift = 5 - ilog2(P);
      const int q = lane >> kShift;  // dot k * NB + b of this batch
      if ((lane & ((1 << kShift) - 1)) == 0 && k0 + q / NB < na)
        ps[(k0 * NB + q) * G + warp] = tot;
    }
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                       smem_u32(&pfull[s]))
                   : "memory");
  }
}

int num_sms() { return device_sms(current_device()); }

template <int NB, int V>
void launch_nb(const SolveParams& p, const Work& w, bool full_scores, cudaStream_t s) {
  constexpr int APB = apb_for(NB, V);
  const int G = (int)(p.ldm / (128 * V));
  const int64_t row_bytes = p.ldm * 4;
  // Stage: ~32 KB of whole atom rows, a multiple of the batch; as many
  // stages as fit the ring.
  int sa = (int)std::max<int64_t>(1, 32768 / row_bytes);
  sa = (sa + APB - 1) / APB * APB;
  const int64_t stage_bytes = sa * (row_bytes + (int64_t)NB * G * 8);
  int stages = (int)std::min<int64_t>(kMaxStages, kRingBytes / stage_bytes);
  if (stages < 2) {
    sa = APB;
    stages = (int)std::min<int64_t>(kMaxStages,
                                    kRingBytes / (sa * (row_bytes + (int64_t)NB * G * 8)));
  }
  const size_t smem = (size_t)stages * sa * (row_bytes + (size_t)NB * G * 8);
  static DevSlots attr_set;
  ensure_smem_limit(attr_set, k_corr_gemv<NB, V>, kRingBytes);
  const int grid = (int)std::min<int64_t>(p.ntl, num_sms());
  k_corr_gemv<NB, V><<<grid, 32 * (G + 2), smem, s>>>(
      w.at32 + p.atom0 * p.ldm, w.r64, w.active, p.n_corr, p.B, p.ldm, p.ntl, sa, stages,
      w.cand, full_scores ? w.scores : nullptr);
}

// Float4s per lane: the largest power of two <= pref that splits the
// measurement axis into <= 8 warp slices, else the smallest larger one that
// does; 0 when none keeps NB * V <= 16 (residual registers per lane: 8 NB V).
int pick_v(int64_t ldm, int nb, int pref) {
  for (int v = pref; v >= 1; v /= 2)
    if (ldm % (128 * v) == 0 && ldm / (128 * v) <= 8) return v;
  for (int v = pref * 2; nb * v <= 16; v *= 2)
    if (ldm % (128 * v) == 0 && ldm / (128 * v) <= 8) return v;
  return 0;
}

int nb_for(int64_t B) { return B <= 1 ? 1 : B <= 2 ? 2 : 4; }
// Eight consumer warps where the measurement axis allows it.
int pref_for(int64_t ldm) {
  int v = (int)(ldm / (128 * 8));
  return v >= 8 ? 8 : v >= 4 ? 4 : v >= 2 ? 2 : 1;
}

}  // namespace

int64_t corr_gemv_tile_atoms() { return kGemvTile; }

bool corr_gemv_supported(int64_t ldm, int64_t B) {
  if (B < 1 || B > 4 || ldm % 128 != 0) return false;
  const int nb = nb_for(B);
  const int v = pick_v(ldm, nb, pref_for(ldm));
  // one batch of rows (+ partial slots) must fit the ring twice
  return v != 0 && 2 * apb_for(nb, v) * (ldm * 4 + nb * 8 * 8) <= kRingBytes;
}

void launch_corr_gemv(const SolveParams& p, const Work& w, bool full_scores, cudaStream_t s) {
  const int nb = nb_for(p.B);
  const int v = pick_v(p.ldm, nb, pref_for(p.ldm));
#define CL_GEMV_CASE(NB_, V_) \
  if (nb == NB_ && v == V_) return launch_nb<NB_, V_>(p, w, full_scores, s);
  CL_GEMV_CASE(1, 1) CL_GEMV_CASE(1, 2) CL_GEMV_CASE(1, 4) CL_GEMV_CASE(1, 8)
  CL_GEMV_CASE(2, 1) CL_GEMV_CASE(2, 2) CL_GEMV_CASE(2, 4) CL_GEMV_CASE(2, 8)
  CL_GEMV_CASE(4, 1) CL_GEMV_CASE(4, 2) CL_GEMV_CASE(4, 4)
#undef CL_GEMV_CASE
}

}  // namespace clb
