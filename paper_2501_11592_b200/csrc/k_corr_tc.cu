// k_corr_tc.cu — K1 on the 5th-generation tensor cores: scores = R A^T in
// 3xFP16 (split fp16 operands, fp32 accumulation) with the argmax selection
// fused into the TMEM epilogue.
//
// Replaces la::matmul(ops.at, r) (clomp.cpp:245) and the max scan of
// inject_from_scores (clomp.cpp:45-47) on the th == 1 path.
//
// Shape: one CTA per 128-signal x 256-atom tile.  UMMA M = signals (TMEM
// lanes), N = atoms (TMEM columns), K = measurements, both operands K-major in
// shared memory with the 64-byte swizzle that TMA writes.  Every operand x is
// scaled by an exact power of two (per signal for the residual, from its norm;
// once for the dictionary) so |s x| < 2^14, and split into fp16
// hi = fp16(s x), lo = fp16(s x - hi); the product is accumulated as
// hi*hi + hi*lo + lo*hi in fp32 in TMEM (~fp32 accuracy; the dropped lo*lo
// term is ~2^-22 |a||r|) at twice the tf32 tensor rate, and the epilogue
// divides the scales back out exactly.
//
// Roles (256 threads): warp 0 lane 0 issues TMA into a 4-stage ring,
// warp 1 lane 0 issues tcgen05.mma (single thread per CTA), warp 2 owns the
// TMEM allocation.  After the last commit all eight warps drain TMEM with
// tcgen05.ld: thread = signal (its TMEM lane; warps w and w + 4 share lanes
// and split the columns), so the per-signal candidate record over the tile's
// 256 atoms (top-2 atoms + third value, Cand) is a register scan with no
// shuffles and one shared-memory merge of the two halves.  Only that record per (signal, atom tile)
// reaches HBM; the selection merges tiles and re-decides near-ties (gap inside
// the split-fp16 error bound) from exact fp64 scores of the few atoms in the band.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "clomp_internal.cuh"

namespace clb {
namespace {

constexpr int TM = 128;  // signals per tile  (UMMA M, TMEM lanes)
constexpr int TN = 256;  // atoms per tile    (UMMA N, TMEM columns)
// K slice per pipeline stage: 16 fp32 = one 64-byte swizzle row, so a stage
// (R hi/lo + A hi/lo) is 48 KB and four stages fit beside the epilogue.
constexpr int BK = 32;  // fp16 elements per operand row per stage (64 bytes)
constexpr int STAGES = 4;
constexpr int ROW_BYTES = BK * 2;             // bytes per operand row in smem
constexpr uint64_t kSwizzleMode = 4;          // UMMA layout type: SWIZZLE_64B
constexpr int R_BYTES = TM * BK * 2;  // 8 KB
constexpr int A_BYTES = TN * BK * 2;  // 16 KB
constexpr int STAGE_BYTES = 2 * R_BYTES + 2 * A_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t TMEM_COLS = 256;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// Multicast variant: the box lands at the same smem offset in every CTA of
// `mask` and completes `bytes` on each destination CTA's mbarrier.
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar,
                                               int c0, int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// Shared-memory matrix descriptor: K-major, ROW_BYTES swizzle, 8-row groups
// 8 * ROW_BYTES apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;                        // LBO (unused for swizzled K-major)
  d |= (uint64_t)((8 * ROW_BYTES) >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;                        // descriptor version
  d |= kSwizzleMode << 61;                       // swizzle mode
  return d;
}

// Instruction descriptor (kind::f16): D f32, A/B f16, both K-major,
// M = 128, N = 256.
constexpr uint32_t kIdesc = (1u << 4)           // D format f32
                            | (0u << 7)         // A format f16
                            | (0u << 10)        // B format f16
                            | ((TN >> 3) << 17) // N
                            | ((TM >> 4) << 24);// M

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld_32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ---------------------------------------------------------------- the kernel
// Insert 32 consecutive scores (atoms ka, ka+1, ...) into a signal's
// candidate summary.  Branch-free because the lanes hold different signals:
// sorted insert of the values by min/max, indices by two predicates on the old
// values; ascending atoms with strict compares keep the lowest atom on ties.
template <bool CHECK>
__device__ __forceinline__ void cand_scan32(const float (&v)[32], int ka, int lim, float& v1,
                                            int& i1, float& v2, int& i2, float& v3) {
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    const float x = (!CHECK || q < lim) ? fabsf(v[q]) : -1.f;
    const int k = ka + q;
    const bool g1 = x > v1, g2 = x > v2;
    i2 = g1 ? i1 : (g2 ? k : i2);
    i1 = g1 ? k : i1;
    v3 = fmaxf(v3, fminf(x, v2));
    v2 = fmaxf(v2, fminf(x, v1));
    v1 = fmaxf(v1, x);
  }
}

#ifdef CL_K1_TRACE
__device__ unsigned long long g_k1_trace[1024][16];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define K1_MARK(i) \
  do { g_k1_trace[blockIdx.y * gridDim.x + blockIdx.x][i] = gtimer(); } while (0)
#define K1_MARK_T(i, tid) do { if (threadIdx.x == (tid)) K1_MARK(i); } while (0)
#else
#define K1_MARK(i) do { } while (0)
#define K1_MARK_T(i, tid) do { } while (0)
#endif

// TMEM -> registers without the wait (the caller batches loads, then waits once).
__device__ __forceinline__ void tmem_ld_32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}

// Epilogue: thread = signal (its TMEM lane); NW warps, warp w reads the 32
// lanes of quarter w % 4 and column part w / 4 of P = NW / 4 equal parts
// (TN / (32 P) chunks of 32 columns, loaded back to back, one wait).  Each
// part's record is merged into part 0's through the (idle) stage ring in
// ascending part order, so strict inserts keep the lowest atom on ties.
template <int NW>
__device__ __forceinline__ void tile_epilogue(uint8_t* smem, uint32_t tmem, uint64_t* accum,
                                              int64_t m0, int64_t n0, int64_t n, int64_t B,
                                              int64_t ntile, const float* __restrict__ r_scale,
                                              double a_inv_scale, Cand* __restrict__ cand,
                                              float* __restrict__ scores_dbg, int warp, int lane,
                                              int64_t tile) {
  constexpr int P = NW / 4;
  constexpr int CH = TN / (32 * P);  // chunks of 32 columns per thread
  __syncwarp();
  mbar_wait(accum, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int part = warp >> 2, wl = warp & 3;
  const int64_t b = m0 + wl * 32 + lane;
  float v1 = -1.f, v2 = -1.f, v3 = -1.f;
  int i1 = 0x7fffffff, i2 = 0x7fffffff;
  const uint32_t lane_base = (uint32_t)(wl * 32) << 16;
  uint32_t raw[CH][32];
#pragma unroll
  for (int c = 0; c < CH; ++c)
    tmem_ld_32_nowait(tmem + lane_base + (uint32_t)(part * (TN / P) + c * 32), raw[c]);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  K1_MARK_T(7, 96);
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int col = part * (TN / P) + c * 32;
    float v[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(raw[c][q]);
    const int64_t a0 = n0 + col;
    if (scores_dbg && b < B) {
      const double u = (double)r_scale[b] * a_inv_scale;
      for (int q = 0; q < 32; ++q)
        if (a0 + q < n) scores_dbg[b * n + a0 + q] = (float)((double)v[q] * u);
    }
    if (a0 + 32 <= n)
      cand_scan32<false>(v, (int)a0, 32, v1, i1, v2, i2, v3);
    else  // ragged last tile: atoms past n never enter
      cand_scan32<true>(v, (int)a0, (int)(n - a0), v1, i1, v2, i2, v3);
  }
  // the stage ring is idle now (every MMA retired): reuse it for the merge
  float* mv = reinterpret_cast<float*>(smem);       // [P][3][TM]
  int* mi = reinterpret_cast<int*>(mv + P * 3 * TM);  // [P][2][TM]
  const int row = wl * 32 + lane;
  K1_MARK_T(8, 96);
  K1_MARK_T(9, 480);
  if (part > 0) {
    mv[(part * 3 + 0) * TM + row] = v1;
    mv[(part * 3 + 1) * TM + row] = v2;
    mv[(part * 3 + 2) * TM + row] = v3;
    mi[(part * 2 + 0) * TM + row] = i1;
    mi[(part * 2 + 1) * TM + row] = i2;
  }
  __syncthreads();
  K1_MARK_T(10, 0);
  if (part == 0 && b < B) {
    auto ins = [&](float x, int k) {  // the cand_scan32 update
      const bool g1 = x > v1, g2 = x > v2;
      i2 = g1 ? i1 : (g2 ? k : i2);
      i1 = g1 ? k : i1;
      v3 = fmaxf(v3, fminf(x, v2));
      v2 = fmaxf(v2, fminf(x, v1));
      v1 = fmaxf(v1, x);
    };
#pragma unroll
    for (int q = 1; q < P; ++q) {
      ins(mv[(q * 3 + 0) * TM + row], mi[(q * 2 + 0) * TM + row]);
      ins(mv[(q * 3 + 1) * TM + row], mi[(q * 2 + 1) * TM + row]);
      v3 = fmaxf(v3, mv[(q * 3 + 2) * TM + row]);
    }
    // back to true units: both operand scales are exact powers of two
    const double u = (double)r_scale[b] * a_inv_scale;
    Cand r;
    r.v1 = v1 >= 0.f ? (double)v1 * u : -1.0;
    r.v2 = v2 >= 0.f ? (double)v2 * u : -1.0;
    r.v3 = v3 >= 0.f ? (double)v3 * u : -1.0;
    r.i1 = i1;
    r.i2 = i2;
    CL_CHECK(tile >= 0 && tile < ntile && (i1 == 0x7fffffff || (i1 >= n0 && i1 < n0 + TN && i1 < n)) &&
             (i2 == 0x7fffffff || (i2 >= n0 && i2 < n0 + TN && i2 < n)));
    cand[b * ntile + tile] = r;
    K1_MARK_T(11, 0);
  }
}

// CL: CTAs per cluster along the signal dimension.  With CL > 1 the atom tile
// (the operand every CTA of the cluster shares) is fetched once per cluster:
// CTA r loads rows [r*TN/CL, (r+1)*TN/CL) of A_hi/A_lo and multicasts them, and
// a stage is refilled only after all CL MMA issuers released it.
template <int CL>
__global__ void __launch_bounds__(256, 1)
k_corr_tc(const __grid_constant__ CUtensorMap tm_rhi, const __grid_constant__ CUtensorMap tm_rlo,
          const __grid_constant__ CUtensorMap tm_ahi, const __grid_constant__ CUtensorMap tm_alo,
          int64_t n, int64_t B, int kblocks, int64_t ntile, const int32_t* __restrict__ active,
          const float* __restrict__ r_scale, double a_inv_scale, Cand* __restrict__ cand,
          float* __restrict__ scores_dbg) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* accum = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.y * TM;  // first signal
  const int64_t n0 = (int64_t)blockIdx.x * TN;  // first atom

  pdl_wait();  // the residual split of the previous kernel
  pdl_trigger();
  // Whole tile finished?  (uniform per CTA; a cluster must stay together)
  if (CL == 1) {
    int mine = 0;
    const int64_t b = m0 + (threadIdx.x & (TM - 1));
    mine = (b < B) ? active[b] : 0;
    if (!__syncthreads_or(mine)) return;
  }
  const uint32_t crank = CL > 1 ? cluster_rank() : 0;
  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1u);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL);
    }
    mbar_init(accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_rhi)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_rlo)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_ahi)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_alo)));
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CL > 1) cluster_sync();  // peers' barriers exist before any multicast
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      uint8_t* st = smem + s * STAGE_BYTES;
      mbar_expect_tx(&full[s], STAGE_BYTES);
      const int k0 = kb * BK;
      tma_load_2d(st, &tm_rhi, &full[s], k0, (int)m0);
      tma_load_2d(st + R_BYTES, &tm_rlo, &full[s], k0, (int)m0);
      if (CL == 1) {
        tma_load_2d(st + 2 * R_BYTES, &tm_ahi, &full[s], k0, (int)n0);
        tma_load_2d(st + 2 * R_BYTES + A_BYTES, &tm_alo, &full[s], k0, (int)n0);
      } else {
        constexpr int rows = TN / CL;
        const uint32_t off = crank * rows * BK * 2;
        const int a_row = (int)n0 + (int)crank * rows;
        tma_load_2d_mc(st + 2 * R_BYTES + off, &tm_ahi, &full[s], k0, a_row, kMask);
        tma_load_2d_mc(st + 2 * R_BYTES + A_BYTES + off, &tm_alo, &full[s], k0, a_row, kMask);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (one thread for the CTA)
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(&full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint8_t* st = smem + s * STAGE_BYTES;
      const uint64_t d_rhi = sw128_desc(smem_u32(st));
      const uint64_t d_rlo = sw128_desc(smem_u32(st + R_BYTES));
      const uint64_t d_ahi = sw128_desc(smem_u32(st + 2 * R_BYTES));
      const uint64_t d_alo = sw128_desc(smem_u32(st + 2 * R_BYTES + A_BYTES));
#pragma unroll
      for (int j = 0; j < BK / 16; ++j) {  // 16 fp16 (32 bytes) per MMA K step
        const uint64_t adv = (uint64_t)(j * 32) >> 4;
        mma_f16(tmem, d_rhi + adv, d_alo + adv, (kb | j) != 0);
        mma_f16(tmem, d_rlo + adv, d_ahi + adv, 1);
        mma_f16(tmem, d_rhi + adv, d_ahi + adv, 1);
      }
      // Stage free once these MMAs retire (in every CTA of the cluster that
      // multicasts into it).  The last STAGES releases are never waited for.
      if (kb < kblocks - STAGES) {
        if (CL == 1)
          mma_commit(&empty[s]);
        else
          mma_commit_mc(&empty[s], kMask);
      }
    }
    mma_commit(accum);        // accumulator complete
  }

  tile_epilogue<8>(smem, tmem, accum, m0, n0, n, B, ntile, r_scale, a_inv_scale, cand, scores_dbg,
                   warp, lane, blockIdx.x);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CL > 1) cluster_sync();  // no CTA leaves while a peer may still write into it
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

// ------------------------------------------------ CTA-pair (cta_group::2)
// Two SMs of a TPC share one 256-signal x 256-atom tile: UMMA M = 256
// (each CTA's 128 signals in its own TMEM lanes), N = 256 atoms split over
// the pair's shared memory (each CTA holds 128 atom rows of every stage).  The
// leader (cluster rank 0) issues every tcgen05.mma.cta_group::2; both CTAs'
// TMA loads complete on the leader's stage barrier (.cta_group::2), and the
// leader's commits arrive on both CTAs' empty / accumulator barriers.  Each
// SM now ingests 32 KB per stage (its R slice + half the atom slice) instead
// of 48 KB for the same MMA work, which is what limits the one-SM kernel at
// short K (config 2: K = 512, 16 k-blocks).
constexpr int A2_BYTES = (TN / 2) * BK * 2;  // 8 KB: half the atom tile
constexpr int STAGE2_BYTES = 2 * R_BYTES + 2 * A2_BYTES;
constexpr int STAGES2 = 6;
constexpr int SMEM2_BYTES = STAGES2 * STAGE2_BYTES + 1024 + 256;
constexpr uint32_t kIdesc2 = (1u << 4) | ((TN >> 3) << 17) | ((2 * TM >> 4) << 24);
constexpr int kPairWarps = 16;  // epilogue: four column parts per TMEM lane quarter

__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map,
                                                 uint32_t leader_bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}

__device__ __forceinline__ void mma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc2), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__global__ void __launch_bounds__(32 * kPairWarps, 1)
k_corr_tc2(const __grid_constant__ CUtensorMap tm_rhi, const __grid_constant__ CUtensorMap tm_rlo,
           const __grid_constant__ CUtensorMap tm_ahi, const __grid_constant__ CUtensorMap tm_alo,
           int64_t n, int64_t B, int kblocks, int64_t ntile, const float* __restrict__ r_scale,
           double a_inv_scale, Cand* __restrict__ cand, float* __restrict__ scores_dbg,
           const int32_t* __restrict__ active) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES2 * STAGE2_BYTES);
  uint64_t* empty = full + STAGES2;
  uint64_t* accum = empty + STAGES2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();  // 0 = leader
  // the pair spans cluster x (cta_group::2 pairs along x): blockIdx.x = signal
  // tile, blockIdx.y = atom tile
  const int64_t m0 = (int64_t)blockIdx.x * TM;  // this CTA's 128 signals
  const int64_t n0 = (int64_t)blockIdx.y * TN;  // the pair's 256 atoms
  if (threadIdx.x == 0) K1_MARK(0);

  // Setup that does not read the previous kernel's output runs before the
  // dependency wait (PDL): barriers, TMEM, tensor-map prefetch.
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_rhi)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_rlo)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_ahi)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_alo)));
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();  // both CTAs' barriers and TMEM exist before any cross-CTA traffic
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the residual split of the previous kernel
  pdl_trigger();
  if (threadIdx.x == 0) K1_MARK(1);
  // A pair whose 256 signals have all stopped has no reader for its records:
  // both CTAs read the same flags and skip to the teardown together (batches
  // that finish early replay the rest of their graph chunk nearly for free).
  int live_sig = 0;
  if (threadIdx.x < 2 * TM) {
    const int64_t sb = (int64_t)(blockIdx.x & ~1u) * TM + threadIdx.x;
    live_sig = sb < B && active[sb] != 0;
  }
  if (__syncthreads_or(live_sig)) {

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs): own R slice + own half of the
    // atom slice, completing on the leader's stage barrier
    const uint32_t full0 = mapa_u32(smem_u32(&full[0]), 0);
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % STAGES2;
      const uint32_t ph = (kb / STAGES2) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      if (rank == 0) mbar_expect_tx(&full[s], 2 * STAGE2_BYTES);
      uint8_t* st = smem + s * STAGE2_BYTES;
      const uint32_t bar = full0 + (uint32_t)(s * 8);
      const int k0 = kb * BK;
      const int arow = (int)n0 + (int)rank * (TN / 2);
      tma_load_2d_pair(st, &tm_rhi, bar, k0, (int)m0);
      tma_load_2d_pair(st + R_BYTES, &tm_rlo, bar, k0, (int)m0);
      tma_load_2d_pair(st + 2 * R_BYTES, &tm_ahi, bar, k0, arow);
      tma_load_2d_pair(st + 2 * R_BYTES + A2_BYTES, &tm_alo, bar, k0, arow);
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    // ---------------- MMA issuer: the leader's single thread for the pair
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % STAGES2;
      const uint32_t ph = (kb / STAGES2) & 1;
      mbar_wait(&full[s], ph);
      if (kb == 0) K1_MARK(2);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint8_t* st = smem + s * STAGE2_BYTES;
      const uint64_t d_rhi = sw128_desc(smem_u32(st));
      const uint64_t d_rlo = sw128_desc(smem_u32(st + R_BYTES));
      const uint64_t d_ahi = sw128_desc(smem_u32(st + 2 * R_BYTES));
      const uint64_t d_alo = sw128_desc(smem_u32(st + 2 * R_BYTES + A2_BYTES));
#pragma unroll
      for (int j = 0; j < BK / 16; ++j) {
        const uint64_t adv = (uint64_t)(j * 32) >> 4;
        mma_f16_pair(tmem, d_rhi + adv, d_alo + adv, (kb | j) != 0);
        mma_f16_pair(tmem, d_rlo + adv, d_ahi + adv, 1);
        mma_f16_pair(tmem, d_rhi + adv, d_ahi + adv, 1);
      }
      if (kb < kblocks - STAGES2) mma_commit_pair(&empty[s]);  // stage free in both CTAs
    }
    K1_MARK(3);
    mma_commit_pair(accum);  // accumulators complete in both CTAs
  }

#ifdef CL_K1_TRACE
  if (threadIdx.x == 96) {
    mbar_wait(accum, 0);
    K1_MARK(4);
  }
#endif
  tile_epilogue<kPairWarps>(smem, tmem, accum, m0, n0, n, B, ntile, r_scale, a_inv_scale, cand,
                            scores_dbg, warp, lane, blockIdx.y);
  }  // live pair
  if (threadIdx.x == 0) K1_MARK(5);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();  // the pair's MMAs / commits are done before TMEM goes
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
  if (threadIdx.x == 64) K1_MARK(6);
}

// fp16 split of the dictionary: scale*x = hi + lo with scale = 2^e chosen by
// the host so that |scale*x| < 2^14; hi = fp16(scale*x), lo = fp16(rest).
__global__ void k_split_dict(const float* __restrict__ src, __half* __restrict__ hi,
                             __half* __restrict__ lo, int64_t count, float scale) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  split_f16(src[i], scale, hi[i], lo[i]);
}

// ---------------------------------------------------------------- host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
    cudaGetLastError();
  });
  return fn;
}

// 2-D fp16 row-major [rows][ld], box [box_rows][BK] (64 bytes), 64-byte swizzle.
bool make_map(CUtensorMap* map, const __half* base, int64_t rows, int64_t ld, int box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            ROW_BYTES == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct MapCache {
  const void* key[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t rows[4] = {0, 0, 0, 0};
  int box[4] = {0, 0, 0, 0};
  int64_t ld[4] = {0, 0, 0, 0};
  CUtensorMap map[4];
};
thread_local MapCache g_maps;

const CUtensorMap* cached_map(int slot, const __half* base, int64_t rows, int64_t ld,
                              int box_rows) {
  if (g_maps.key[slot] != base || g_maps.rows[slot] != rows || g_maps.box[slot] != box_rows ||
      g_maps.ld[slot] != ld) {
    if (!make_map(&g_maps.map[slot], base, rows, ld, box_rows)) return nullptr;
    g_maps.key[slot] = base;
    g_maps.rows[slot] = rows;
    g_maps.box[slot] = box_rows;
    g_maps.ld[slot] = ld;
  }
  return &g_maps.map[slot];
}

}  // namespace

bool corr_tc_available() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return prop.major == 10 && encode_fn() != nullptr;
}

int64_t corr_tc_tile_atoms() { return TN; }

constexpr int kCluster = 4;

static std::atomic<int> g_tc_mode{-1};  // -1 auto, 0 one-SM kernel, 1 CTA pair (CL_TC_PAIR)

static bool launch_tc_impl(const SolveParams& p, const Work& w, float* scores_dbg,
                           cudaStream_t s) {
  const int64_t mtiles = (p.B + TM - 1) / TM;
  if (g_tc_mode < 0) {
    const char* e = getenv("CL_TC_PAIR");
    g_tc_mode.store(e ? atoi(e) : 1);
  }
  if (g_tc_mode >= 1 && mtiles >= 2) {
    const CUtensorMap* rhi = cached_map(0, w.r_hi, p.B, p.ldm, TM);
    const CUtensorMap* rlo = cached_map(1, w.r_lo, p.B, p.ldm, TM);
    const CUtensorMap* ahi = cached_map(2, w.at_hi + p.atom0 * p.ldm, p.n_corr, p.ldm, TN / 2);
    const CUtensorMap* alo = cached_map(3, w.at_lo + p.atom0 * p.ldm, p.n_corr, p.ldm, TN / 2);
    if (!rhi || !rlo || !ahi || !alo) return false;
    cudaFuncSetAttribute(k_corr_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)((mtiles + 1) / 2 * 2), (unsigned)((p.n_corr + TN - 1) / TN));
    cfg.blockDim = dim3(32 * kPairWarps);
    cfg.dynamicSmemBytes = SMEM2_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, k_corr_tc2, *rhi, *rlo, *ahi, *alo, p.n_corr, p.B,
                              (int)(p.ldm / BK), p.ntl, (const float*)w.r_scale, p.a_inv_scale,
                              w.cand, scores_dbg, (const int32_t*)w.active) == cudaSuccess;
  }
  const bool clustered = mtiles >= kCluster;
  const int arows = clustered ? TN / kCluster : TN;
  const CUtensorMap* rhi = cached_map(0, w.r_hi, p.B, p.ldm, TM);
  const CUtensorMap* rlo = cached_map(1, w.r_lo, p.B, p.ldm, TM);
  const CUtensorMap* ahi = cached_map(2, w.at_hi + p.atom0 * p.ldm, p.n_corr, p.ldm, arows);
  const CUtensorMap* alo = cached_map(3, w.at_lo + p.atom0 * p.ldm, p.n_corr, p.ldm, arows);
  if (!rhi || !rlo || !ahi || !alo) return false;
  const int kblocks = (int)(p.ldm / BK);
  if (!clustered) {
    cudaFuncSetAttribute(k_corr_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    dim3 grid((unsigned)((p.n_corr + TN - 1) / TN), (unsigned)mtiles);
    return launch_pdl(k_corr_tc<1>, grid, dim3(256), (size_t)SMEM_BYTES, s, *rhi, *rlo, *ahi, *alo,
                      p.n_corr, p.B, kblocks, p.ntl, (const int32_t*)w.active,
                      (const float*)w.r_scale, p.a_inv_scale, w.cand, scores_dbg) == cudaSuccess;
  }
  cudaFuncSetAttribute(k_corr_tc<kCluster>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       SMEM_BYTES);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)((p.n_corr + TN - 1) / TN),
                     (unsigned)((mtiles + kCluster - 1) / kCluster * kCluster));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = kCluster;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see pdl_wait
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k_corr_tc<kCluster>, *rhi, *rlo, *ahi, *alo, p.n_corr, p.B,
                            kblocks, p.ntl, w.active, w.r_scale, p.a_inv_scale, w.cand,
                            scores_dbg) == cudaSuccess;
}

// Debug: per-CTA globaltimer marks of the last pair-kernel launch (build with
// CL_NVCC_EXTRA=-DCL_K1_TRACE): entry, after setup, first stage, last MMA,
// accumulator ready, epilogue done, exit.  Returns CTAs written (0: not built in).
int corr_tc_trace(unsigned long long* out, int max_ctas) {
#ifdef CL_K1_TRACE
  const int n = max_ctas < 1024 ? max_ctas : 1024;
  cudaMemcpyFromSymbol(out, g_k1_trace, (size_t)n * 16 * sizeof(unsigned long long));
  return n;
#else
  (void)out;
  (void)max_ctas;
  return 0;
#endif
}

bool launch_corr_tc(const SolveParams& p, const Work& w, cudaStream_t s) {
  return launch_tc_impl(p, w, nullptr, s);
}

bool launch_corr_tc_debug(const SolveParams& p, const Work& w, float* scores,
                          cudaStream_t s) {
  return launch_tc_impl(p, w, scores, s);
}

void launch_split_dict(const float* src, __half* hi, __half* lo, int64_t count, float scale,
                       cudaStream_t s) {
  const int64_t blocks = (count + 255) / 256;
  k_split_dict<<<(unsigned)blocks, 256, 0, s>>>(src, hi, lo, count, scale);
}

}  // namespace clb
