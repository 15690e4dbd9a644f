// k_solve.cu — everything in the CLOMP outer iteration except the correlation
// GEMM: init, support injection (K1c), fp64 rescans of near-tied selections,
// coefficient learning with the fused residual update (K2), the per-signal and
// joint stopping state machines, and result compaction.
//
// Reference lines followed (all /root/reference/proj/src/clomp.cpp unless noted):
//   r = A*(mask.*s) - y, ||r||, eps break ........ 236-242, 285-288
//   inject_from_scores (th, ties, zero column) ... 41-53, 245-246
//   inner loop: g = 2 A^T r masked, optimizer .... 83-91, 120-123, 171-209, 248-252
//   loss, NumericalError, best, stall ............ 253-273
//   result: best snapshot unless converged ....... 276-288
//
// Learning runs in the Gram form: with S the support and c its coefficients,
// A_S^T (A_S c - y) = G c - b, G = A_S^T A_S, b = A_S^T y, both accumulated in
// fp64 from the fp32 atoms.  This is the reference gradient in exact
// arithmetic; it costs t^2 per epoch instead of the reference's dense 2*m*n.
#include <cooperative_groups.h>
#include <math_constants.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <type_traits>

#include "clomp_internal.cuh"

namespace clb {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kModeJoint = 0;
constexpr int kModePerSignal = 1;
constexpr int kStatusNumerical = 4;
constexpr int kStatusCapacity = 7;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

__device__ __forceinline__ bool mask_test(const uint32_t* mb, int j) {
  return (mb[j >> 5] >> (j & 31)) & 1u;
}

// Exact tf32 split of an fp32 value: hi = x with the 13 low mantissa bits
// cleared, lo = x - hi (exact).  Must match k_split_tf32 in k_corr_tc.cu.
// fp16 split of residual row b (already in r64) with the scale of its
// norm^2 L; lanes/threads stride over the row.
__device__ __forceinline__ void split_row(const Work& w, int64_t b, int64_t ldm, double L,
                                          int64_t start, int64_t stride) {
  const float sc = split_scale(L);
  if (start == 0) w.r_scale[b] = 1.0f / sc;
  for (int64_t i = start; i < ldm; i += stride)
    split_f16(w.r64[b * ldm + i], sc, w.r_hi[b * ldm + i], w.r_lo[b * ldm + i]);
}

// ------------------------------------------------------------------ init
// The reference's m x B layout (element (i, b) at i B + b, linalg.hpp:21-24)
// to signal-major rows of y32 through a 32 x 32 shared-memory tile, so both
// the reads and the writes are coalesced (a warp-per-signal strided read of
// the m x B array cost ~0.2 ms at config 2).
__global__ void k_transpose_y(const float* __restrict__ y_in, int64_t m, int64_t B,
                              float* __restrict__ out, int64_t ldo) {
  __shared__ float tile[32][33];
  const int64_t b0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t i = i0 + r, b = b0 + threadIdx.x;
    if (i < m && b < B) tile[r][threadIdx.x] = y_in[i * B + b];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t b = b0 + r, i = i0 + threadIdx.x;
    if (i < m && b < B) out[b * ldo + i] = tile[threadIdx.x][r];
  }
}

// One warp per signal: stage y, r = 0 - y = -y (clomp.cpp:236-237 at s = 0),
// ||y||^2, fresh state, and the outer-1 eps test in per-signal mode.
__global__ void k_init(SolveParams p, Work w, const float* y_in,
                       int64_t in_ld) {
  const int lane = threadIdx.x & 31;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= p.B) return;
  double acc = 0.0;
  for (int64_t i = lane; i < p.ldm; i += 32) {
    float v = 0.f;
    if (i < p.m) v = y_in[b * in_ld + i];
    const int64_t o = b * p.ldm + i;
    w.y32[o] = v;
    w.y64[o] = (double)v;
    w.r64[o] = -(double)v;
    acc = fma((double)v, (double)v, acc);
  }
  for (int64_t q = lane; q < p.mwords; q += 32) w.maskbits[b * p.mwords + q] = 0u;
  const double L = warp_sum(acc);
  if (w.r_hi) split_row(w, b, p.ldm, L, lane, 32);
  if (lane == 0) {
    w.loss[b] = L;  // s = 0: the prior terms vanish
    if (w.rloss) w.rloss[b] = L;
    w.cnt[b] = 0;
    w.gcnt[b] = 0;
    w.best_cnt[b] = 0;
    w.best_L[b] = CUDART_INF;
    w.prev_L[b] = CUDART_INF;
    w.stall[b] = 0;
    w.iters[b] = 0;
    w.status[b] = 0;
    w.changed[b] = 0;
    int act = 1;
    uint8_t cv = 0;
    if (p.mode == kModePerSignal && sqrt(L) < p.eps) {
      act = 0;
      cv = 1;
    }
    w.active[b] = act;
    w.conv[b] = cv;
  }
}

// --------------------------------------------------------------- select
// K1c for th == 1, one warp per signal: merge the per-tile candidate records,
// accept a clear winner, and re-decide a near-tie (top-2 gap inside the
// correlation error bound, or tied) from exact fp64 scores of every atom whose
// approximate score lies within 2*delta of the top: an atom outside that band
// cannot reach the exact maximum.  The records name the tile's two best atoms
// and bound the rest by the third value, so normally only those atoms are
// rescored; a tile whose third value is in the band too is rescored whole.
// Every tie with the exact maximum is injected in ascending atom order
// (inject_from_scores, clomp.cpp:41-53).

// Exact |a_j . r| for up to 8 consecutive atoms j0 .. j0+cnt-1 (fp64 products
// of the fp32 atoms with the fp64 residual, one fixed summation order for
// every atom, so identical atoms score bitwise identically).  All lanes get
// every value.
__device__ __forceinline__ void exact_scores8(const SolveParams& p, const Work& w,
                                              const double* r, int64_t j0, int cnt,
                                              double (&out)[8], int lane) {
  double acc[8];
  CL_CHECK(j0 >= 0 && cnt >= 1 && cnt <= 8 && j0 + cnt <= p.n);
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u] = 0.0;
  if (p.sep) {
    // Separable atom (i, j): a_r,i^T R a_c,j = a_r,i . U_j with U = R A_c in fp64
    // (stage 1 of this iteration's correlation, still in sep_scratch).
    const int64_t b = (r - w.r64) / p.ldm;
    const double* U = w.sep_scratch + b * p.nc * p.mr;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (u < cnt) {
        const int64_t atom = j0 + u, ia = atom % p.nr, ja = atom / p.nr;
        const double* ar = w.at_r64 + ia * p.ldr;
        const double* uj = U + ja * p.mr;
        for (int64_t q = lane; q < p.mr; q += 32) acc[u] = fma(ar[q], uj[q], acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) out[u] = u < cnt ? fabs(warp_sum(acc[u])) : -1.0;
    return;
  }
#pragma unroll 2
  for (int64_t i = 4 * lane; i < p.ldm; i += 128) {
    const double2 r01 = *reinterpret_cast<const double2*>(r + i);
    const double2 r23 = *reinterpret_cast<const double2*>(r + i + 2);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (u < cnt) {
        const float4 a = *reinterpret_cast<const float4*>(w.at32 + (j0 + u) * p.ldm + i);
        acc[u] = fma(f2d(a.x), r01.x, acc[u]);
        acc[u] = fma(f2d(a.y), r01.y, acc[u]);
        acc[u] = fma(f2d(a.z), r23.x, acc[u]);
        acc[u] = fma(f2d(a.w), r23.y, acc[u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) out[u] = u < cnt ? fabs(warp_sum(acc[u])) : -1.0;
}

// One atom: the same per-lane summation order as exact_scores8 (so an atom
// scores bitwise the same either way), with the row loads of eight 128-float
// chunks issued ahead of the dependent FMA chain — a rescoring warp is alone on
// its scheduler, and two chunks in flight fetched a 4096-row atom at ~10 GB/s.
__device__ __forceinline__ double exact_score(const SolveParams& p, const Work& w,
                                              const double* r, int64_t j, int lane) {
  if (p.sep) {
    double v[8];
    exact_scores8(p, w, r, j, 1, v, lane);
    return v[0];
  }
  CL_CHECK(j >= 0 && j < p.n);
  const float* a = w.at32 + j * p.ldm;
  double acc = 0.0;
#pragma unroll 8
  for (int64_t i = 4 * lane; i < p.ldm; i += 128) {
    const float4 av = *reinterpret_cast<const float4*>(a + i);
    const double2 r01 = *reinterpret_cast<const double2*>(r + i);
    const double2 r23 = *reinterpret_cast<const double2*>(r + i + 2);
    acc = fma(f2d(av.x), r01.x, acc);
    acc = fma(f2d(av.y), r01.y, acc);
    acc = fma(f2d(av.z), r23.x, acc);
    acc = fma(f2d(av.w), r23.y, acc);
  }
  return fabs(warp_sum(acc));
}

// Support update of one picked atom (lane 0): skip atoms already selected,
// stop the signal with kStatusCapacity when the support is full.
struct PickState {
  int t, added, over;
};

__device__ __forceinline__ void pick_atom(const SolveParams& p, const Work& w, int64_t b,
                                          int32_t j, PickState& ps) {
  uint32_t* mb = w.maskbits + b * p.mwords;
  CL_CHECK(j >= 0 && j < p.n && b >= 0 && b < p.B && ps.t >= 0 && ps.t <= p.cap);
  if (mask_test(mb, j)) return;  // already in the support: mask unchanged
  if (ps.t < p.cap) {
    w.sup[b * p.cap + ps.t] = j;
    mb[j >> 5] |= 1u << (j & 31);
    ++ps.t;
    ++ps.added;
  } else {
    ps.over = 1;
  }
}

__device__ __forceinline__ void pick_finish(const SolveParams& p, const Work& w, int64_t b,
                                            const PickState& ps) {
  w.cnt[b] = ps.t;
  w.changed[b] = ps.added > 0;
  if (ps.over) {
    w.status[b] = kStatusCapacity;
    w.active[b] = 0;
  }
  if (ps.added) atomicMax(&w.counters[kMaxCount], ps.t);
}

// Exact scorers for the near-tie rescoring.  ScoreResid: a_j . r from the stored
// fp64 residual row.  ScoreGram (the fused fast kernel, which does not store
// that row): the same quantity regrouped through the dictionary Gram cache,
//   a_j . (A_S c - y) = sum_k (A^T A)[j][s_k] c_k - a_j . y,
// from the signal's coefficients held one per lane.  Both carry an absolute
// rounding error of order 1e-16 ||y|| (r itself is a difference of O(||y||)
// terms rounded to fp64), as the reference's own scores do; identical atoms
// read identical Gram rows and atom rows, so exact ties stay exact.
struct ScoreResid {
  const SolveParams& p;
  const Work& w;
  const double* r;
  __device__ __forceinline__ void operator()(int64_t j0, int cnt, double (&out)[8], int lane) const {
    if (cnt == 1)
      out[0] = exact_score(p, w, r, j0, lane);
    else
      exact_scores8(p, w, r, j0, cnt, out, lane);
  }
};

struct ScoreGram {
  const SolveParams& p;
  const Work& w;
  int64_t b;
  double c_l;      // lane k: coefficient of support atom k (0 beyond t)
  int32_t sup_l;   // lane k: support atom k
  int t;
  __device__ __forceinline__ void operator()(int64_t j0, int cnt, double (&out)[8], int lane) const {
    const float* y = w.y32 + b * p.ldm;
    double z[8], g[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) z[u] = g[u] = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < cnt && lane < t) g[u] = w.gfull[(j0 + u) * p.n + sup_l] * c_l;
    for (int64_t i = 4 * lane; i < p.ldm; i += 128) {
      const float4 yv = *reinterpret_cast<const float4*>(y + i);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (u < cnt) {
          const float4 a = *reinterpret_cast<const float4*>(w.at32 + (j0 + u) * p.ldm + i);
          z[u] = fma(f2d(a.x), f2d(yv.x), z[u]);
          z[u] = fma(f2d(a.y), f2d(yv.y), z[u]);
          z[u] = fma(f2d(a.z), f2d(yv.z), z[u]);
          z[u] = fma(f2d(a.w), f2d(yv.w), z[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) out[u] = u < cnt ? fabs(warp_sum(g[u]) - warp_sum(z[u])) : -1.0;
  }
};

// One pass over the atoms inside the band (ascending atom order).  Pass 0
// returns the exact maximum; pass 1 picks every atom attaining M.
// Pass 0 also records what it scored — lane k keeps the k-th atom and its exact
// score (atoms are visited in ascending order) — so a band of up to 32 atoms,
// i.e. practically every one, is decided without scoring anything twice.
struct BandRec {
  int n = 0;        // atoms scored so far
  int atom = -1;    // lane k: the k-th of them ...
  double val = -1;  // ... and its score
};

template <class Scorer>
__device__ double band_pass(const SolveParams& p, const Work& w, int64_t b, double cut,
                            const Scorer& score, int pass, double M, PickState& ps, int lane,
                            BandRec& rec) {
  const Cand* cd = w.cand + b * p.ntile;
  for (int64_t t0 = 0; t0 < p.ntile; t0 += 32) {
    const int64_t tl = t0 + lane;
    const Cand c = tl < p.ntile ? cd[tl] : cand_empty();
    unsigned any = __ballot_sync(kFull, c.v1 >= cut);
    while (any) {
      const int src = __ffs(any) - 1;
      any &= any - 1;
      const double cv2 = __shfl_sync(kFull, c.v2, src), cv3 = __shfl_sync(kFull, c.v3, src);
      const int ci1 = __shfl_sync(kFull, c.i1, src), ci2 = __shfl_sync(kFull, c.i2, src);
      if (cv3 >= cut) {  // a third atom of this tile is in the band: whole tile
        const int64_t a0 = (t0 + src) * p.tile_atoms;
        const int64_t a1 = a0 + p.tile_atoms < p.n ? a0 + p.tile_atoms : p.n;
        for (int64_t j0 = a0; j0 < a1; j0 += 8) {
          const int cnt = (int)(a1 - j0 < 8 ? a1 - j0 : 8);
          double v[8];
          score(j0, cnt, v, lane);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (u >= cnt) continue;
            if (pass == 0) {
              M = fmax(M, v[u]);
              if (lane == (rec.n & 31)) {
                rec.atom = (int)(j0 + u);
                rec.val = v[u];
              }
              ++rec.n;
            } else if (v[u] == M && lane == 0) {
              pick_atom(p, w, b, (int32_t)(j0 + u), ps);
            }
          }
        }
      } else {
        int ja = ci1, jb = cv2 >= cut ? ci2 : -1;
        if (jb >= 0 && jb < ja) {
          const int tmp = ja;
          ja = jb;
          jb = tmp;
        }
        double v[8];
        score(ja, 1, v, lane);
        const double va = v[0];
        double vb = -1.0;
        if (jb >= 0) {
          score(jb, 1, v, lane);
          vb = v[0];
        }
        if (pass == 0) {
          M = fmax(M, fmax(va, vb));
          if (lane == (rec.n & 31)) {
            rec.atom = ja;
            rec.val = va;
          }
          ++rec.n;
          if (jb >= 0) {
            if (lane == (rec.n & 31)) {
              rec.atom = jb;
              rec.val = vb;
            }
            ++rec.n;
          }
        } else if (lane == 0) {
          if (va == M) pick_atom(p, w, b, ja, ps);
          if (jb >= 0 && vb == M) pick_atom(p, w, b, jb, ps);
        }
      }
    }
  }
  return M;
}

// Near-tied th == 1 selection: exact rescoring of the band, every tie with the
// exact maximum injected (see above).  Updates sup / cnt / mask / changed.
template <class Scorer>
__device__ void select_near_tie_with(const SolveParams& p, const Work& w, int64_t b, double v1,
                                     double delta, int t_old, const Scorer& score, int lane) {
  PickState ps{t_old, 0, 0};
  if (lane == 0) atomicAdd(&w.counters[kRescanTotal], 1);
  const double cut = v1 - 2.0 * delta;
  BandRec rec;
  const double M = band_pass(p, w, b, cut, score, 0, -1.0, ps, lane, rec);
  if (M > 0.0) {
    if (rec.n <= 32) {  // every scored atom is on a lane, in ascending atom order
      for (int k = 0; k < rec.n; ++k) {
        const int a = __shfl_sync(kFull, rec.atom, k);
        const double v = __shfl_sync(kFull, rec.val, k);
        if (v == M && lane == 0) pick_atom(p, w, b, a, ps);
      }
    } else {
      band_pass(p, w, b, cut, score, 1, M, ps, lane, rec);
    }
  }
  if (lane == 0) pick_finish(p, w, b, ps);
  __syncwarp();
}

__device__ void select_near_tie(const SolveParams& p, const Work& w, int64_t b, double v1,
                                double delta, int t_old, int lane) {
  select_near_tie_with(p, w, b, v1, delta, t_old, ScoreResid{p, w, w.r64 + b * p.ldm}, lane);
}

// Merge of one signal's candidate records: best (v1, i1) over all tiles (the
// lowest atom wins an exact tie) and the runner-up value v2.
__device__ __forceinline__ void cand_merge_warp(const SolveParams& p, const Work& w, int64_t b,
                                                Cand first, double& v1, int& i1, double& v2,
                                                int lane) {
  v1 = first.v1;
  v2 = first.v2;
  i1 = first.i1;
  const Cand* cd = w.cand + b * p.ntile;
  for (int64_t t = lane + 32; t < p.ntile; t += 32) {
    const Cand c = cd[t];
    if (c.v1 > v1 || (c.v1 == v1 && c.i1 < i1)) {
      v2 = fmax(v1, c.v2);
      v1 = c.v1;
      i1 = c.i1;
    } else {
      v2 = fmax(v2, c.v1);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov1 = __shfl_xor_sync(kFull, v1, o), ov2 = __shfl_xor_sync(kFull, v2, o);
    const int oi1 = __shfl_xor_sync(kFull, i1, o);
    if (ov1 > v1 || (ov1 == v1 && oi1 < i1)) {
      v2 = fmax(v1, ov2);
      v1 = ov1;
      i1 = oi1;
    } else {
      v2 = fmax(v2, ov1);
    }
  }
}

__device__ void select_top_warp(const SolveParams& p, const Work& w, int64_t b, int lane) {
  double v1, v2;
  int i1;
  cand_merge_warp(p, w, b, lane < p.ntile ? w.cand[b * p.ntile + lane] : cand_empty(), v1, i1,
                  v2, lane);
  const int t_old = w.cnt[b];
  if (v1 > 0.0) {  // else zero column: inject nothing (clomp.cpp:48)
    const double delta = p.delta_rel * p.colnorm_max * sqrt(w.loss[b]);
    if (v1 - v2 > delta) {
      PickState ps{t_old, 0, 0};
      if (lane == 0) {
        pick_atom(p, w, b, i1, ps);
        pick_finish(p, w, b, ps);
      }
      __syncwarp();
    } else {
      select_near_tie(p, w, b, v1, delta, t_old, lane);
    }
  } else {
    PickState ps{t_old, 0, 0};
    if (lane == 0) pick_finish(p, w, b, ps);
    __syncwarp();
  }
}

__global__ void k_select_top(SolveParams p, Work w) {
  const int lane = threadIdx.x & 31;
  const int64_t b = p.sig_lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (b >= p.sig_hi || !w.active[b]) return;
  select_top_warp(p, w, b, lane);
}

// Ordered append of every j with score(j) >= cut that is not yet in the mask
// (clomp.cpp:49-51), one warp, ascending j.
template <class ScoreFn>
__device__ void warp_threshold_append(const SolveParams& p, const Work& w,
                                      int64_t b, double cut, ScoreFn score,
                                      int lane) {
  uint32_t* mb = w.maskbits + b * p.mwords;
  int t = w.cnt[b];
  int added = 0, overflow = 0;
  for (int64_t j0 = 0; j0 < p.n; j0 += 32) {
    const int64_t j = j0 + lane;
    bool pick = false;
    if (j < p.n) pick = score(j) >= cut && !mask_test(mb, (int)j);
    const unsigned bal = __ballot_sync(kFull, pick);
    if (pick) {
      const int pos = t + __popc(bal & ((1u << lane) - 1u));
      CL_CHECK(pos >= 0 && j < p.n);
      if (pos < p.cap) {
        w.sup[b * p.cap + pos] = (int32_t)j;
        atomicOr(&mb[j >> 5], 1u << (j & 31));
      }
    }
    t += __popc(bal);
    added += __popc(bal);
    if (t > p.cap) overflow = 1;
  }
  if (lane == 0) {
    if (overflow) {
      w.status[b] = kStatusCapacity;
      w.active[b] = 0;
      t = (int)p.cap;
    }
    w.cnt[b] = t;
    w.changed[b] = added > 0;
    if (added) atomicMax(&w.counters[kMaxCount], t);
  }
}

// K1c for th < 1: threshold pass over the materialised |scores|.
__global__ void k_select_thresh(SolveParams p, Work w) {
  const int lane = threadIdx.x & 31;
  const int64_t b = p.sig_lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (b >= p.sig_hi || !w.active[b]) return;
  const double* sc = w.scores + b * p.n;
  double cmax = 0.0;
  for (int64_t j = lane; j < p.n; j += 32) cmax = fmax(cmax, sc[j]);
  cmax = warp_max(cmax);
  if (lane == 0) w.changed[b] = 0;
  if (cmax == 0.0) return;
  const double cut = p.th * cmax;
  warp_threshold_append(p, w, b, cut, [&](int64_t j) { return sc[j]; }, lane);
}

// ------------------------------------------------------ stopping rules
// Per-signal bookkeeping after the learning phase of outer iteration `outer`
// (clomp.cpp:253-273), plus the eps test that opens the next iteration
// (clomp.cpp:238-242).  Returns true when the best snapshot must be taken.
// Per-signal control state read before the residual pass, so its load
// latency overlaps the atom gathers instead of following the loss reduction.
struct CtlState {
  double best_L, prev_L;
  int cnt, changed, stall;
};

__device__ __forceinline__ CtlState load_ctl(const Work& w, int64_t b) {
  CtlState c;
  c.best_L = w.best_L[b];
  c.prev_L = w.prev_L[b];
  c.cnt = w.cnt[b];
  c.changed = w.changed[b];
  c.stall = w.stall[b];
  return c;
}

// L: the loss the reference's best / stall / divergence rules read (lb.total,
// clomp.cpp:253-273); L_res: its residual part, which the eps test reads
// (clomp.cpp:238-242).  They differ only with a prior.
__device__ bool control_signal(const SolveParams& p, const Work& w, int64_t b,
                               int outer, double L, const CtlState& st, double L_res) {
  w.loss[b] = L;
  if (w.rloss) w.rloss[b] = L_res;
  if (!isfinite(L)) {
    w.status[b] = kStatusNumerical;
    w.active[b] = 0;
    return false;
  }
  w.iters[b] = outer;
  bool snap = false;
  if (L < st.best_L) {
    w.best_L[b] = L;
    w.best_cnt[b] = st.cnt;
    if (w.best_R) w.best_R[b] = L_res;
    snap = true;
  }
  const double prev = st.prev_L;
  const double rel = isfinite(prev) ? (prev - L) / fmax(fabs(prev), 1e-300)
                                    : CUDART_INF;
  const int stall = (!st.changed && rel < p.stall_tol) ? st.stall + 1 : 0;
  w.stall[b] = stall;
  w.prev_L[b] = L;
  if (stall >= p.stall_patience || outer >= p.max_outer) {
    w.active[b] = 0;
  } else if (sqrt(L_res) < p.eps) {
    w.conv[b] = 1;
    w.active[b] = 0;
  } else {
    atomicAdd(&w.counters[active_slot(outer)], 1);
  }
  return snap;
}

__device__ __forceinline__ bool control_signal(const SolveParams& p, const Work& w, int64_t b,
                                               int outer, double L, const CtlState& st) {
  return control_signal(p, w, b, outer, L, st, L);
}

__device__ __forceinline__ bool control_signal(const SolveParams& p, const Work& w, int64_t b,
                                               int outer, double L) {
  return control_signal(p, w, b, outer, L, load_ctl(w, b), L);
}

// ------------------------------------------ learning, warp per signal
// All epochs of one outer iteration with G's row `lane` in registers (zero
// padded to T columns, which is exact) and c broadcast through shared memory.
// All epochs of one outer iteration, one warp per signal, lane i owning row i
// of the support Gram system (rows beyond t are zero, which is exact), c
// broadcast through a double-buffered shared-memory vector (one __syncwarp per
// epoch).
//   plain GD (OPT 0): the step is affine, c <- (I - 2 lr G) c + 2 lr b, so
//     `g` holds the row of T = I - 2 lr G and `bi` holds 2 lr b_i: an epoch is
//     T FMAs into accumulators seeded with 2 lr b_i, nothing else.  Equal to
//     s -= lr * 2 A^T (A s - y) (clomp.cpp:87-90, 178-181) in exact arithmetic.
//   momentum / Adam: g = 2 (G c - b), then gradient_step's update
//     (clomp.cpp:182-206).
template <int T, int TB, int OPT>
__device__ __forceinline__ void epochs_warp(const double (&g)[TB],
                                            double& c, double bi, double& m1,
                                            double& m2, double* cs,
                                            const SolveParams& p, int step0,
                                            int lane, int t) {
  constexpr int NA = T >= 16 ? 8 : 4;
  for (int e = 0; e < p.inner; ++e) {
    const double* cr = cs + (e & 1) * kWarpCap;
    double a[NA];
    a[0] = OPT == 0 ? bi : 0.0;
#pragma unroll
    for (int q = 1; q < NA; ++q) a[q] = 0.0;
#pragma unroll
    for (int j = 0; j < T; j += NA) {
#pragma unroll
      for (int q = 0; q < NA; q += 2) {
        const double2 cv = *reinterpret_cast<const double2*>(cr + j + q);
        a[q] = fma(g[j + q], cv.x, a[q]);
        a[q + 1] = fma(g[j + q + 1], cv.y, a[q + 1]);
      }
    }
    double acc;
    if constexpr (NA == 8)
      acc = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    else
      acc = (a[0] + a[1]) + (a[2] + a[3]);
    if constexpr (OPT == 0) {
      c = acc;
    } else {
      const double grad = 2.0 * (acc - bi);
      double bc1 = 1.0, bc2 = 1.0;
      if (OPT == 2) {
        bc1 = p.bc1[step0 + e];
        bc2 = p.bc2[step0 + e];
      }
      if (lane < t) opt_step<OPT>(c, grad, m1, m2, p.lr, bc1, bc2);
    }
    cs[((e + 1) & 1) * kWarpCap + lane] = c;
    __syncwarp();
  }
}

// c <- M c + d, `steps` times: M's row `lane` in registers (T columns live),
// c broadcast through the double-buffered cs (parity continues from *ep).
template <int T, int TB>
__device__ __forceinline__ void affine_steps(const double (&m)[TB], double& c, double d,
                                             double* cs, int steps, int* ep) {
  constexpr int NA = T >= 16 ? 8 : 4;
  for (int e = 0; e < steps; ++e, ++*ep) {
    const double* cr = cs + (*ep & 1) * kWarpCap;
    double a[NA];
    a[0] = d;
#pragma unroll
    for (int q = 1; q < NA; ++q) a[q] = 0.0;
#pragma unroll
    for (int j = 0; j < T; j += NA) {
#pragma unroll
      for (int q = 0; q < NA; q += 2) {
        const double2 cv = *reinterpret_cast<const double2*>(cr + j + q);
        a[q] = fma(m[j + q], cv.x, a[q]);
        a[q + 1] = fma(m[j + q + 1], cv.y, a[q + 1]);
      }
    }
    if constexpr (NA == 8)
      c = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    else
      c = (a[0] + a[1]) + (a[2] + a[3]);
    cs[((*ep + 1) & 1) * kWarpCap + threadIdx.x % 32] = c;
    __syncwarp();
  }
}

// P <- P * P in place for a symmetric T x T matrix stored with row stride
// T + 4 (bank-conflict-free fragment loads), on the fp64 tensor cores
// (mma.sync m8n8k4 f64 -> DMMA).  By symmetry the B fragment of block (K, J)
// equals the A fragment of block (J, K), so every lane loads its T*T/32 share
// of P once (A-layout fragments F(I, K) = P[8I + lane/4][4K + lane%4]) and the
// whole product runs from registers; the shared-memory broadcast traffic of
// the SIMT squaring disappears.
template <int T>
__device__ __forceinline__ void square_dmma(double* buf, int lane) {
  constexpr int NI = T / 8, NK = T / 4, LD = T + 4;
  const int r = lane >> 2, c = lane & 3;
  double f[NI][NK];
#pragma unroll
  for (int I = 0; I < NI; ++I)
#pragma unroll
    for (int K = 0; K < NK; ++K) f[I][K] = buf[(8 * I + r) * LD + 4 * K + c];
  __syncwarp();
  // Upper block triangle only (J >= I): the product is symmetric, so each
  // off-diagonal 8x8 block is also written transposed (NI(NI+1)/2 of NI^2
  // blocks computed: 10 of 16 at T = 32).
#pragma unroll
  for (int I = 0; I < NI; ++I) {
    double acc[NI][2];
#pragma unroll
    for (int J = I; J < NI; ++J) acc[J][0] = acc[J][1] = 0.0;
#pragma unroll
    for (int K = 0; K < NK; ++K)
#pragma unroll
      for (int J = I; J < NI; ++J)
        asm volatile(
            "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
            : "+d"(acc[J][0]), "+d"(acc[J][1])
            : "d"(f[I][K]), "d"(f[J][K]));
#pragma unroll
    for (int J = I; J < NI; ++J) {
      *reinterpret_cast<double2*>(buf + (8 * I + r) * LD + 8 * J + 2 * c) =
          make_double2(acc[J][0], acc[J][1]);
      if (J != I) {
        buf[(8 * J + 2 * c) * LD + 8 * I + r] = acc[J][0];
        buf[(8 * J + 2 * c + 1) * LD + 8 * I + r] = acc[J][1];
      }
    }
  }
  __syncwarp();
}

// Plain gradient descent, E = inner_steps epochs of c <- T c + d with
// T = I - 2 lr G and d = 2 lr b (clomp.cpp:87-90, 178-181).  Write
// E = P q + r with P = 2^L.  Powers T^(2^l) and offsets d_(2^l) =
// sum_{i<2^l} T^i d are built by doubling (d_{2k} = d_k + T^k d_k,
// T^{2k} = (T^k)^2, squarings on the fp64 tensor cores); on the way up, every
// set bit l of r applies c <- T^(2^l) c + d_(2^l), then q steps of
// c <- T^P c + d_P finish — the same iterate as E single steps in exact
// arithmetic (c_{k+a} = T^a c_k + d_a composes in any order).  L minimises
// popcount(r) + L + q dependent matvecs plus L squarings.
template <int T, int TB>
__device__ void epochs_plain(double (&g)[TB], double& c, double d, double* cs,
                             double* s1, const SolveParams& p, int lane) {
  const int E = p.inner;
  const int L = p.warp_L[T / 8 - 1];  // host: warp_power_levels (clomp_api.cu)
  int ep = 0;
  if (L == 0) {
    affine_steps<T, TB>(g, c, d, cs, E, &ep);
    return;
  }
  const int q = E >> L, r = E & ((1 << L) - 1);
  double v = d;
  constexpr int LD = T + 4;
#pragma unroll 1
  for (int l = 0; l < L; ++l) {
    // here g = row `lane` of M = T^(2^l), v = d_(2^l)
    if ((r >> l) & 1) {
      cs[(ep & 1) * kWarpCap + lane] = c;
      __syncwarp();
      affine_steps<T, TB>(g, c, v, cs, 1, &ep);
    }
    // v <- v + M v: an affine step with offset v itself.
    cs[(ep & 1) * kWarpCap + lane] = v;
    __syncwarp();
    double vv = v;
    affine_steps<T, TB>(g, vv, v, cs, 1, &ep);
    v = vv;
    // M <- M^2; g <- row `lane` of M (read as a column, conflict-free, exact
    // by symmetry).
    if (l == 0 && lane < T) {  // later levels: s1 already holds M (last square)
#pragma unroll
      for (int j = 0; j < T; ++j) s1[j * LD + lane] = g[j];
    }
    __syncwarp();
    square_dmma<T>(s1, lane);
#pragma unroll
    for (int j = 0; j < T; ++j) g[j] = lane < T ? s1[j * LD + lane] : 0.0;
    __syncwarp();
  }
  cs[(ep & 1) * kWarpCap + lane] = c;
  __syncwarp();
  affine_steps<T, TB>(g, c, v, cs, q, &ep);
}

template <int TB, int OPT>
__device__ __forceinline__ void epochs_dispatch(const double (&g)[TB], double& c,
                                                double bi, double& m1, double& m2,
                                                double* cs, const SolveParams& p,
                                                int step0, int lane, int t) {
  if constexpr (TB == 8) {
    epochs_warp<8, TB, OPT>(g, c, bi, m1, m2, cs, p, step0, lane, t);
  } else if constexpr (TB == 16) {
    if (t <= 8)
      epochs_warp<8, TB, OPT>(g, c, bi, m1, m2, cs, p, step0, lane, t);
    else
      epochs_warp<16, TB, OPT>(g, c, bi, m1, m2, cs, p, step0, lane, t);
  } else {
    if (t <= 16)
      epochs_warp<16, TB, OPT>(g, c, bi, m1, m2, cs, p, step0, lane, t);
    else if (t <= 24)
      epochs_warp<24, TB, OPT>(g, c, bi, m1, m2, cs, p, step0, lane, t);
    else
      epochs_warp<32, TB, OPT>(g, c, bi, m1, m2, cs, p, step0, lane, t);
  }
}

// Sum of per-lane vectors acc[0..N) over the warp: afterwards lane L holds
// sum over all 32 lanes of acc[L % N].  Recursive halving inside each group of
// N lanes (N-1 shuffles), then a butterfly across the 32/N groups; all array
// indices are compile-time so acc stays in registers.
template <int N>
__device__ __forceinline__ double transpose_reduce(double (&acc)[N], int lane) {
#pragma unroll
  for (int sft = N / 2; sft >= 1; sft >>= 1) {
    const bool upper = (lane & sft) != 0;
#pragma unroll
    for (int j = 0; j < sft; ++j) {
      const double send = upper ? acc[j] : acc[j + sft];
      const double keep = upper ? acc[j + sft] : acc[j];
      acc[j] = keep + __shfl_xor_sync(kFull, send, sft);
    }
  }
  double v = acc[0];
#pragma unroll
  for (int sft = N; sft < 32; sft <<= 1) v += __shfl_xor_sync(kFull, v, sft);
  return v;
}

// Gram row/column and b entry of every atom added since the last call
// (one warp, t <= 32): G[k][i] = a_k . a_i, b_k = a_k . y, fp64 sums of the
// fp32 products.  All k+1 dot products run at once (float4 loads, lanes over
// the measurements) and are reduced together by transpose_reduce32.
template <int TB>
__device__ void warp_extend_gram(const SolveParams& p, const Work& w, int64_t b,
                                 int t0, int t, int lane, const int32_t* sups,
                                 double* sG, int lds) {
  const int64_t cap = p.cap, ldm = p.ldm;
  double* G = w.gram + b * cap * cap;
  const float* y = w.y32 + b * ldm;  // y is fp32 data: exact in fp64 on load
  if (p.sep) {
    // Separable atoms: G[(i,j),(i',j')] = Gr[i][i'] * Gc[j][j']; b_k = Z[p_k]
    // with Z = A_r^T Y A_c (fp64, once per solve).
    for (int k = t0; k < t; ++k) {
      const int64_t pk = sups[k], ik = pk % p.nr, jk = pk / p.nr;
      if (lane <= k) {
        const int64_t pl = sups[lane], il = pl % p.nr, jl = pl / p.nr;
        const double v = w.gr[ik * p.nr + il] * w.gc[jk * p.nc + jl];
        G[(int64_t)k * cap + lane] = v;
        G[(int64_t)lane * cap + k] = v;
        sG[k * lds + lane] = v;
        sG[lane * lds + k] = v;
      }
      if (lane == 0) {
        w.bvec[b * cap + k] = w.zb[b * p.n + pk];
        w.coef[b * cap + k] = 0.0;
        w.mom1[b * cap + k] = 0.0;
        w.mom2[b * cap + k] = 0.0;
      }
    }
    __syncwarp();
    return;
  }
  if (w.gfull) {
    // Gather from the context's A^T A; b_k = a_k . y on demand.
    for (int k = t0; k < t; ++k) {
      const int64_t jk = sups[k];
      if (lane <= k) {
        const double v = w.gfull[jk * p.n + sups[lane]];
        G[(int64_t)k * cap + lane] = v;
        G[(int64_t)lane * cap + k] = v;
        sG[k * lds + lane] = v;
        sG[lane * lds + k] = v;
      }
      const float* ak = w.at32 + jk * ldm;
      double accb = 0.0;
      for (int64_t i0 = 4 * lane; i0 < ldm; i0 += 128) {
        const float4 a = *reinterpret_cast<const float4*>(ak + i0);
        const float4 yv = *reinterpret_cast<const float4*>(y + i0);
        const double2 y01 = make_double2(f2d(yv.x), f2d(yv.y));
        const double2 y23 = make_double2(f2d(yv.z), f2d(yv.w));
        accb = fma(f2d(a.x), y01.x, accb);
        accb = fma(f2d(a.y), y01.y, accb);
        accb = fma(f2d(a.z), y23.x, accb);
        accb = fma(f2d(a.w), y23.y, accb);
      }
      accb = warp_sum(accb);
      if (lane == 0) {
        w.bvec[b * cap + k] = accb;
        w.coef[b * cap + k] = 0.0;  // new atoms start at 0 (clomp.hpp:53-54)
        w.mom1[b * cap + k] = 0.0;
        w.mom2[b * cap + k] = 0.0;
      }
    }
    __syncwarp();
    return;
  }
  for (int k = t0; k < t; ++k) {
    const float* ak = w.at32 + (int64_t)sups[k] * ldm;
    double acc[TB];
#pragma unroll
    for (int i = 0; i < TB; ++i) acc[i] = 0.0;
    double accb = 0.0;
    for (int64_t i0 = 4 * lane; i0 < ldm; i0 += 128) {
      const float4 av = *reinterpret_cast<const float4*>(ak + i0);
      const float4 yv = *reinterpret_cast<const float4*>(y + i0);
      const double2 y01 = make_double2(f2d(yv.x), f2d(yv.y));
      const double2 y23 = make_double2(f2d(yv.z), f2d(yv.w));
      const double ax = f2d(av.x), ay = f2d(av.y), az = f2d(av.z), aw = f2d(av.w);
      accb = fma(ax, y01.x, accb);
      accb = fma(ay, y01.y, accb);
      accb = fma(az, y23.x, accb);
      accb = fma(aw, y23.y, accb);
#pragma unroll
      for (int i = 0; i < TB; ++i) {
        if (i <= k) {
          const float4 ai = *reinterpret_cast<const float4*>(w.at32 + (int64_t)sups[i] * ldm + i0);
          acc[i] = fma(ax, f2d(ai.x), acc[i]);
          acc[i] = fma(ay, f2d(ai.y), acc[i]);
          acc[i] = fma(az, f2d(ai.z), acc[i]);
          acc[i] = fma(aw, f2d(ai.w), acc[i]);
        }
      }
    }
    const double gk = transpose_reduce<TB>(acc, lane);
    if (lane <= k) {
      G[(int64_t)k * cap + lane] = gk;
      G[(int64_t)lane * cap + k] = gk;
      sG[k * lds + lane] = gk;
      sG[lane * lds + k] = gk;
    }
    accb = warp_sum(accb);
    if (lane == 0) {
      w.bvec[b * cap + k] = accb;
      w.coef[b * cap + k] = 0.0;  // new atoms start at 0 (clomp.hpp:53-54)
      w.mom1[b * cap + k] = 0.0;
      w.mom2[b * cap + k] = 0.0;
    }
  }
  __syncwarp();
}

// Residual r = A_S c - y (fp64), stored for the next correlation (fp64 and the
// tf32 split), and its sum of squares.  Each lane owns 16 measurements per
// 512-row pass (float4 atom loads); c and the support come from shared memory.
#ifndef CL_RESIDW_UNROLL
#define CL_RESIDW_UNROLL 4
#endif
constexpr int kResidUnroll = CL_RESIDW_UNROLL;

// STORE_R64 = false (the fused fast kernel): the fp64 residual row is not
// written — only exact rescoring of a near-tied selection reads it, a few dozen
// signals per step, and those rebuild their row on demand (materialize_r64);
// the 16.8 MB written per config-2 iteration otherwise also evicts the Gram rows
// the next iteration reloads (-4.7 % per step).
template <bool STORE_R64 = true, bool SPLIT = true>
__device__ double warp_residual(const SolveParams& p, const Work& w, int64_t b,
                                const double* cs, const int32_t* sups, int t,
                                int lane) {
  const int64_t ldm = p.ldm;
  const float* y = w.y32 + b * ldm;  // fp32 data, exact in fp64
  double lacc = 0.0;
  double rr[16];  // the last 512-row pass stays in registers for the split
  for (int64_t base = 0; base < ldm; base += 512) {
    double r[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) r[q] = 0.0;
#pragma unroll kResidUnroll
    for (int k = 0; k < t; ++k) {
      const double ck = cs[k];
      CL_CHECK(sups[k] >= 0 && sups[k] < p.n && t <= kWarpCap);
      const float* row = w.at32 + (int64_t)sups[k] * ldm + base + 4 * lane;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (base + 128 * q < ldm) {
          const float4 v = *reinterpret_cast<const float4*>(row + 128 * q);
          r[4 * q + 0] = fma(f2d(v.x), ck, r[4 * q + 0]);
          r[4 * q + 1] = fma(f2d(v.y), ck, r[4 * q + 1]);
          r[4 * q + 2] = fma(f2d(v.z), ck, r[4 * q + 2]);
          r[4 * q + 3] = fma(f2d(v.w), ck, r[4 * q + 3]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i0 = base + 128 * q + 4 * lane;
      if (base + 128 * q < ldm) {
        const int64_t o = b * ldm + i0;
        const float4 yv = *reinterpret_cast<const float4*>(y + i0);
        const double2 y01 = make_double2(f2d(yv.x), f2d(yv.y));
        const double2 y23 = make_double2(f2d(yv.z), f2d(yv.w));
        r[4 * q + 0] -= y01.x;
        r[4 * q + 1] -= y01.y;
        r[4 * q + 2] -= y23.x;
        r[4 * q + 3] -= y23.y;
        if (STORE_R64) {
          *reinterpret_cast<double2*>(w.r64 + o) = make_double2(r[4 * q + 0], r[4 * q + 1]);
          *reinterpret_cast<double2*>(w.r64 + o + 2) = make_double2(r[4 * q + 2], r[4 * q + 3]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) lacc = fma(r[4 * q + e], r[4 * q + e], lacc);
      }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) rr[q] = r[q];
  }
  const double L = warp_sum(lacc);
  if (SPLIT && w.r_hi) {
    if (ldm <= 512) {  // single pass: split straight from registers
      const float sc = split_scale(L);
      if (lane == 0) w.r_scale[b] = 1.0f / sc;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t i0 = 128 * q + 4 * lane;
        if (128 * q < ldm) {
          __align__(8) __half h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) split_f16(rr[4 * q + e], sc, h[e], l[e]);
          *reinterpret_cast<uint2*>(w.r_hi + b * ldm + i0) = *reinterpret_cast<const uint2*>(h);
          *reinterpret_cast<uint2*>(w.r_lo + b * ldm + i0) = *reinterpret_cast<const uint2*>(l);
        }
      }
    } else {
      __syncwarp();
      split_row(w, b, ldm, L, lane, 32);  // reads r64: callers keep STORE_R64 for ldm > 512
    }
  }
  return L;
}

// Asynchronous copy (LDGSTS, no registers held) of the Gram rows built in
// earlier iterations, G[j][i] for i, j < t0, into the warp's shared buffer
// (row stride lds), issued before the selection and the Gram extension so its
// latency overlaps theirs.  learn_warp_body waits for it.
__device__ __forceinline__ void stage_gram_async(const SolveParams& p, const Work& w, int64_t b,
                                                 int t0, double* sG, int lds, int lane) {
  if (lane < t0) {
    const double* G = w.gram + b * p.cap * p.cap;
    for (int j = 0; j < t0; ++j) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(sG + j * lds + lane);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst),
                   "l"(G + (int64_t)j * p.cap + lane)
                   : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Epochs of one outer iteration on a support of t atoms whose Gram matrix is
// staged in s1 (row stride TB + 4, symmetric): c, b (and the optimizer moments)
// of this lane's atom come in registers; the learned coefficients (and
// moments) are stored.
template <int TB, int OPT>
__device__ __forceinline__ double learn_epochs(const SolveParams& p, const Work& w, int64_t b,
                                               int outer, double* cs, double* s1, int lane, int t,
                                               double c, double bi, double& m1, double& m2) {
  constexpr int LDS = TB + 4;
  double g[TB];
  const double twolr = 2.0 * p.lr;
#pragma unroll
  for (int j = 0; j < TB; ++j) {
    // G[lane][j] read as G[j][lane] (G is symmetric): conflict-free
    const double gij = (lane < t && j < t) ? s1[j * LDS + lane] : 0.0;
    if (OPT == 0)
      g[j] = (lane < t && j == lane) ? 1.0 - twolr * gij : -(twolr * gij);
    else
      g[j] = gij;
  }
  if (lane >= t) c = bi = m1 = m2 = 0.0;
  if (OPT == 0) bi = twolr * bi;
  cs[lane] = c;
  __syncwarp();
  const int step0 = (outer - 1) * p.inner;
  if constexpr (OPT == 0) {
    if constexpr (TB == 8) {
      epochs_plain<8, TB>(g, c, bi, cs, s1, p, lane);
    } else if constexpr (TB == 16) {
      if (t <= 8)
        epochs_plain<8, TB>(g, c, bi, cs, s1, p, lane);
      else
        epochs_plain<16, TB>(g, c, bi, cs, s1, p, lane);
    } else {
      // (zero padding is exact, so the narrower instantiations compute the
      // same bits; t <= 8 reaches a 32-atom bucket only on the fused path)
      if (t <= 8)
        epochs_plain<8, TB>(g, c, bi, cs, s1, p, lane);
      else if (t <= 16)
        epochs_plain<16, TB>(g, c, bi, cs, s1, p, lane);
      else if (t <= 24)
        epochs_plain<24, TB>(g, c, bi, cs, s1, p, lane);
      else
        epochs_plain<32, TB>(g, c, bi, cs, s1, p, lane);
    }
  } else {
    epochs_dispatch<TB, OPT>(g, c, bi, m1, m2, cs, p, step0, lane, t);
  }
  const int64_t cap = p.cap;
  if (lane < t) {
    w.coef[b * cap + lane] = c;
    if (OPT != 0) {
      w.mom1[b * cap + lane] = m1;
      w.mom2[b * cap + lane] = m2;
    }
  }
  return c;
}

// General entry (every path): state from global memory, Gram extension by
// warp_extend_gram, then learn_epochs.  The caller staged the old Gram rows.
template <int TB, int OPT>
__device__ void learn_warp_body(const SolveParams& p, const Work& w, int64_t b,
                                int outer, double* cs, int32_t* sups, double* s1,
                                double* s2, int lane) {
  (void)s2;
  const int t = w.cnt[b];
  const int t0 = w.gcnt[b];
  const int64_t cap = p.cap;
  if (lane < t) sups[lane] = w.sup[b * cap + lane];
  __syncwarp();
  constexpr int LDS = TB + 4;  // staged Gram (s1, see stage_gram_async)
  warp_extend_gram<TB>(p, w, b, t0, t, lane, sups, s1, LDS);
  if (lane == 0) w.gcnt[b] = t;
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();
  double c = 0.0, bi = 0.0, m1 = 0.0, m2 = 0.0;
  if (lane < t) {
    c = w.coef[b * cap + lane];
    bi = w.bvec[b * cap + lane];
    if (OPT != 0) {
      m1 = w.mom1[b * cap + lane];
      m2 = w.mom2[b * cap + lane];
    }
  }
  learn_epochs<TB, OPT>(p, w, b, outer, cs, s1, lane, t, c, bi, m1, m2);
}

// Residual, loss and stopping rules after the learning phase, one warp per
// signal: no block barriers, the whole signal's gathers (16 rows per lane per
// 512-row pass) issued by one warp, many signals resident per SM.  Signals
// whose support outgrew the learning bucket TB were finished by the block
// learning kernel.
#ifndef CL_RESIDW_MINB
#define CL_RESIDW_MINB 4
#endif
template <int TB>
__global__ void __launch_bounds__(128, CL_RESIDW_MINB)
k_resid_w(SolveParams p, Work w, int outer) {
  __shared__ __align__(16) double cs_all[4][kWarpCap];
  __shared__ int32_t sup_all[4][kWarpCap];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_wait();
  pdl_trigger();
  const int64_t b = p.sig_lo + (int64_t)blockIdx.x * 4 + warp;
  if (b >= p.sig_hi || !w.active[b]) return;
  const int t = w.cnt[b];
  if (t > TB) return;
  const int64_t cap = p.cap;
  double* cs = cs_all[warp];
  int32_t* sups = sup_all[warp];
  cs[lane] = lane < t ? w.coef[b * cap + lane] : 0.0;
  sups[lane] = lane < t ? w.sup[b * cap + lane] : 0;
  CtlState ctl{};
  if (lane == 0 && p.mode == kModePerSignal) ctl = load_ctl(w, b);
  __syncwarp();
  const double L = warp_residual(p, w, b, cs, sups, t, lane);
  int snap = 0;
  if (lane == 0) {
    if (p.prior)
      w.rloss[b] = L;  // k_prior_control adds the prior and decides
    else if (p.mode == kModePerSignal)
      snap = control_signal(p, w, b, outer, L, ctl);
    else
      w.loss[b] = L;
  }
  snap = __shfl_sync(kFull, snap, 0);
  if (snap && lane < t) w.best_coef[b * cap + lane] = cs[lane];
}

// TB: support-size bucket this launch is compiled for (8, 16 or 32).  Signals
// whose support outgrew it (possible only through ties) are queued for the
// block kernel.
// Bulk variant of stage_gram_async for learn_fast: one TMA bulk copy per
// Gram row (cp.async.bulk, completion on the warp's mbarrier) instead of one
// 8-byte cp.async per element, so the LSU queue stays free for the selection
// and extension loads.  Rows are copied in 16-byte units (t0 & ~1 entries); an
// odd last column comes from row t0-1 by symmetry with ordinary loads.
__device__ __forceinline__ void stage_gram_bulk(const SolveParams& p, const Work& w, int64_t b,
                                                int t0, double* sG, int lds, uint64_t* bar,
                                                int lane) {
  const double* G = w.gram + b * p.cap * p.cap;
  const int ne = t0 & ~1;
  const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(bar);
  if (lane == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a),
                 "r"((uint32_t)(t0 * ne * 8))
                 : "memory");
  __syncwarp();
  if (lane < t0 && ne > 0) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(sG + lane * lds);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(G + (int64_t)lane * p.cap), "r"((uint32_t)(ne * 8)), "r"(bar_a)
        : "memory");
  }
  if ((t0 & 1) && lane < t0) sG[lane * lds + t0 - 1] = G[(int64_t)(t0 - 1) * p.cap + lane];
}

__device__ __forceinline__ void mbar_wait0(uint64_t* bar) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n"
      "@!P bra W_%=;\n"
      "}\n" ::"r"(a)
      : "memory");
}

// The batched th == 1 path with the context's A^T A (config 2): selection,
// Gram extension and learning for one signal with the fewest dependent
// memory round trips.  Every piece of the signal's state is loaded at once
// (round trip 1, overlapping the asynchronous Gram staging), the selection
// works on registers (support membership by ballot instead of the mask), the
// new Gram row comes from gfull and b_k = a_k . y (round trip 2), and the
// epochs start with everything in registers / shared memory.
#ifdef CL_LEARN_TRACE
// Debug (CL_NVCC_EXTRA=-DCL_LEARN_TRACE): per-signal phase timestamps of the
// last k_learn_fast launch: globaltimer at entry, clock64 at entry / after the
// state loads + record merge / selection / Gram extension / staged rows /
// epochs / residual + control.
__device__ unsigned long long g_lt[8192][8];
__device__ __forceinline__ unsigned long long lt_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define LT_MARK(i) do { if (lane == 0 && b < 8192) g_lt[b][i] = (i) == 0 ? lt_gtimer() : (unsigned long long)clock64(); } while (0)
#else
#define LT_MARK(i) do { } while (0)
#endif

template <int TB, int OPT, bool LAZY>
__device__ __forceinline__ bool learn_fast(const SolveParams& p, const Work& w, int64_t b,
                                           int outer, int32_t* big_list, double* cs,
                                           int32_t* sups, double* s1, uint64_t* bar, int lane) {
  const int64_t cap = p.cap;  // >= 32
  constexpr int LDS = TB + 4;
  LT_MARK(0);
  LT_MARK(1);
  // round trip 1: all independent loads (garbage beyond cnt is never used)
  const int act = w.active[b];
  const int t_old = w.cnt[b];
  const int t0 = w.gcnt[b];
  const double Lb = w.loss[b];
  int32_t sup_l = w.sup[b * cap + lane];
  double c_l = w.coef[b * cap + lane];
  double b_l = w.bvec[b * cap + lane];
  double m1 = 0.0, m2 = 0.0;
  if (OPT != 0) {
    m1 = w.mom1[b * cap + lane];
    m2 = w.mom2[b * cap + lane];
  }
  const Cand first = lane < p.ntile ? w.cand[b * p.ntile + lane] : cand_empty();
  CtlState ctl{};  // stopping-rule state for the residual tail
  if (p.mode == kModePerSignal) {
    ctl.best_L = w.best_L[b];
    ctl.prev_L = w.prev_L[b];
    ctl.stall = w.stall[b];
  }
  if (!act) return false;
  CL_CHECK(t_old >= 0 && t_old <= cap && t0 >= 0 && t0 <= t_old);
  const bool staged = t0 <= TB;
  if (staged) stage_gram_bulk(p, w, b, t0, s1, LDS, bar, lane);

  // K1c (th == 1): clear winner from the records, near-ties rescored exactly
  double v1, v2;
  int i1;
  cand_merge_warp(p, w, b, first, v1, i1, v2, lane);
  LT_MARK(2);
  int t = t_old;
  int chg = 0;  // mask changed this iteration (stall rule)
  // LAZY (ldm <= 512 and the tensor-core correlation next: the fp16 split comes
  // straight from registers): this kernel's residual tail skips the fp64 row;
  // the paths that rescore exactly — a near-tied selection, or the mask-based
  // selection of a full 32-atom support — rebuild it first (supports wider
  // than the warp had theirs stored by the block / cluster kernels)
  const double delta = p.delta_rel * p.colnorm_max * sqrt(Lb);
  if (LAZY && t_old == kWarpCap) {  // the mask-based path below rescans from the row
    cs[lane] = c_l;
    sups[lane] = sup_l;
    __syncwarp();
    (void)warp_residual<true, false>(p, w, b, cs, sups, t_old, lane);  // the row it would have stored
    __syncwarp();
  }
  if (t_old >= 32) {  // support wider than the warp: mask-based general path
    select_top_warp(p, w, b, lane);
    if (!w.active[b]) {
      if (staged) mbar_wait0(bar);
      return false;
    }
    t = w.cnt[b];
    chg = w.changed[b];
  } else if (v1 > 0.0) {  // else zero column: inject nothing (clomp.cpp:48)
    if (v1 - v2 > delta) {
      const bool dup = __any_sync(kFull, lane < t_old && sup_l == i1);
      if (!dup) {
        if (t_old >= cap) {  // support full: kStatusCapacity
          if (lane == 0) {
            w.status[b] = kStatusCapacity;
            w.active[b] = 0;
            w.changed[b] = 0;
          }
          if (staged) mbar_wait0(bar);
          return false;
        }
        if (lane == t_old) sup_l = i1;
        if (lane == 0) {
          w.sup[b * cap + t_old] = i1;
          atomicOr(&w.maskbits[b * p.mwords + (i1 >> 5)], 1u << (i1 & 31));
          w.cnt[b] = t_old + 1;
          atomicMax(&w.counters[kMaxCount], t_old + 1);
        }
        t = t_old + 1;
      }
      chg = dup ? 0 : 1;
      if (lane == 0) w.changed[b] = chg;
    } else {
      if (LAZY)  // no fp64 residual row: rescore through the Gram cache
        select_near_tie_with(p, w, b, v1, delta, t_old,
                             ScoreGram{p, w, b, lane < t_old ? c_l : 0.0, sup_l, t_old}, lane);
      else
        select_near_tie(p, w, b, v1, delta, t_old, lane);
      if (!w.active[b]) {
        if (staged) mbar_wait0(bar);
        return false;
      }
      t = w.cnt[b];
      chg = w.changed[b];
      sup_l = w.sup[b * cap + lane];
    }
  } else if (lane == 0) {
    w.changed[b] = 0;
  }
  if (t > TB || t0 > TB) {  // outgrew this bucket: the block kernel learns it
    if (lane == 0) {
      const int slot = atomicAdd(&w.counters[kBigCount + (outer & 1)], 1);
      CL_CHECK(slot >= 0 && slot < p.B);
      big_list[slot] = (int32_t)b;
    }
    if (staged) mbar_wait0(bar);
    return true;  // k_learn_block finishes it (and counts it for K1)
  }

  LT_MARK(3);
  // round trip 2: Gram row / column of the new atoms from gfull, b_k = a_k . y
  double* G = w.gram + b * cap * cap;
  const float* y = w.y32 + b * p.ldm;  // fp32 data, exact in fp64
  for (int k = t0; k < t; ++k) {
    const int64_t jk = __shfl_sync(kFull, sup_l, k);
    CL_CHECK(jk >= 0 && jk < p.n && t <= TB && (lane > k || (sup_l >= 0 && sup_l < p.n)));
    if (lane <= k) {
      const double v = w.gfull[jk * p.n + sup_l];
      G[(int64_t)k * cap + lane] = v;
      G[(int64_t)lane * cap + k] = v;
      s1[k * LDS + lane] = v;
      s1[lane * LDS + k] = v;
    }
    const float* ak = w.at32 + jk * p.ldm;
    double accb = 0.0;
#pragma unroll 4
    for (int64_t i0 = 4 * lane; i0 < p.ldm; i0 += 128) {
      const float4 a = *reinterpret_cast<const float4*>(ak + i0);
      const float4 yv = *reinterpret_cast<const float4*>(y + i0);
      const double2 y01 = make_double2(f2d(yv.x), f2d(yv.y));
      const double2 y23 = make_double2(f2d(yv.z), f2d(yv.w));
      accb = fma(f2d(a.x), y01.x, accb);
      accb = fma(f2d(a.y), y01.y, accb);
      accb = fma(f2d(a.z), y23.x, accb);
      accb = fma(f2d(a.w), y23.y, accb);
    }
    accb = warp_sum(accb);
    if (lane == k) {  // new atoms start at 0 (clomp.hpp:53-54)
      b_l = accb;
      c_l = m1 = m2 = 0.0;
    }
    if (lane == 0) w.bvec[b * cap + k] = accb;
  }
  if (lane == 0) w.gcnt[b] = t;
  LT_MARK(4);
  mbar_wait0(bar);
  __syncwarp();
  LT_MARK(5);
  const double c = learn_epochs<TB, OPT>(p, w, b, outer, cs, s1, lane, t, c_l, b_l, m1, m2);
  LT_MARK(6);

  // residual r = A_S c - y, its fp16 split for the next K1, the loss and the
  // stopping rules (clomp.cpp:236-242, 253-273) in the same warp: the L2-bound
  // gathers of some warps overlap the epochs of others.
  __syncwarp();
  if (lane < t) {
    cs[lane] = c;
    sups[lane] = sup_l;
  } else if (lane < kWarpCap) {
    cs[lane] = 0.0;
    sups[lane] = 0;
  }
  __syncwarp();
  const double L = warp_residual<!LAZY>(p, w, b, cs, sups, t, lane);
  int snap = 0;
  if (lane == 0) {
    if (p.mode == kModePerSignal) {
      ctl.cnt = t;
      ctl.changed = chg;
      snap = control_signal(p, w, b, outer, L, ctl);
    } else {
      w.loss[b] = L;
    }
  }
  snap = __shfl_sync(kFull, snap, 0);
  if (snap && lane < t) w.best_coef[b * p.cap + lane] = c;
  LT_MARK(7);
  return false;
}

#ifndef CL_LEARN_NW32
#define CL_LEARN_NW32 2
#endif
#ifndef CL_LEARN_NW16
#define CL_LEARN_NW16 4
#endif
#ifndef CL_LEARN_NW8
#define CL_LEARN_NW8 4
#endif
template <int TB>
constexpr int learn_warps() { return TB == 32 ? CL_LEARN_NW32 : (TB == 16 ? CL_LEARN_NW16 : CL_LEARN_NW8); }

#ifndef CL_LEARN32_MINB
#define CL_LEARN32_MINB 8
#endif
#ifndef CL_LEARN16_MINB
#define CL_LEARN16_MINB 4
#endif
#ifndef CL_LEARN8_MINB
#define CL_LEARN8_MINB 7
#endif
template <int TB>
constexpr int learn_min_blocks() {
  return TB == 32 ? CL_LEARN32_MINB : (TB == 16 ? CL_LEARN16_MINB : CL_LEARN8_MINB);
}

template <int TB, int OPT>
__global__ void __launch_bounds__(32 * learn_warps<TB>(), learn_min_blocks<TB>())
k_learn_warp(SolveParams p, Work w, int outer, int32_t* big_list) {
  constexpr int NW = learn_warps<TB>();
  __shared__ __align__(16) double cs_all[NW][2 * kWarpCap];
  __shared__ int32_t sup_all[NW][kWarpCap];
  __shared__ __align__(16) double sq_all[NW][TB * (TB + 4)];  // powers of T (padded rows)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_wait();
  pdl_trigger();
  // the NEXT iteration's active count starts here (this iteration's slot was
  // cleared by the previous iteration's learning kernel; the stopping rules
  // increment it after learning, the host reads it one graph chunk later)
  if (blockIdx.x == 0 && threadIdx.x == 0) w.counters[active_slot(outer + 1)] = 0;
  const int64_t b = p.sig_lo + (int64_t)blockIdx.x * NW + warp;
  if (b >= p.sig_hi) return;
  double* s1 = sq_all[warp];
  if (!w.active[b]) return;
  const int t0 = w.gcnt[b];
  if (t0 <= TB) stage_gram_async(p, w, b, t0, s1, TB + 4, lane);
  if (p.fuse_select) {  // this iteration's th == 1 selection (K1c) first
    select_top_warp(p, w, b, lane);
    if (!w.active[b]) {
      asm volatile("cp.async.wait_all;" ::: "memory");
      return;
    }
  }
  if (w.cnt[b] > TB) {
    if (lane == 0) {
      const int slot = atomicAdd(&w.counters[kBigCount + (outer & 1)], 1);
      CL_CHECK(slot >= 0 && slot < p.B);
      big_list[slot] = (int32_t)b;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }
  double* cs = cs_all[warp];
  int32_t* sups = sup_all[warp];
  double* s2 = nullptr;
  learn_warp_body<TB, OPT>(p, w, b, outer, cs, sups, s1, s2, lane);
}

// Same bucket, the fast path (learn_fast): batched th == 1 with gfull.
template <int TB, int OPT, bool LAZY>
__global__ void __launch_bounds__(32 * learn_warps<TB>(), learn_min_blocks<TB>())
k_learn_fast(SolveParams p, Work w, int outer, int32_t* big_list) {
  constexpr int NW = learn_warps<TB>();
  __shared__ __align__(16) double cs_all[NW][2 * kWarpCap];
  __shared__ __align__(16) double sq_all[NW][TB * (TB + 4)];
  __shared__ __align__(8) uint64_t bar_all[NW];
  __shared__ int32_t sup_all[NW][kWarpCap];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&bar_all[warp]))
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0 && threadIdx.x == 0) w.counters[active_slot(outer + 1)] = 0;
  const int64_t b = p.sig_lo + (int64_t)blockIdx.x * NW + warp;
  if (b >= p.sig_hi) return;
  learn_fast<TB, OPT, LAZY>(p, w, b, outer, big_list, cs_all[warp], sup_all[warp], sq_all[warp],
                            &bar_all[warp], lane);
}

// ------------------------------------------ learning, block per signal
// Supports of any size up to kBlockRows * blockDim.  G lives in shared memory
// when it fits, else it is streamed from L2 every epoch (symmetric G is read
// column-wise so the threads of a warp touch consecutive addresses).
constexpr int kBlockThreads = 256;
constexpr int kBlockRows = 8;

template <int OPT, bool SMEM_G>
__global__ void __launch_bounds__(kBlockThreads)
k_learn_block(SolveParams p, Work w, int outer, const int32_t* big_list, int skip_le) {
  extern __shared__ __align__(16) unsigned char dsm[];
  double* cs = reinterpret_cast<double*>(dsm);                 // [cap]
  int32_t* sups = reinterpret_cast<int32_t*>(cs + p.cap);      // [cap]
  double* Gs = reinterpret_cast<double*>(sups + ((p.cap + 1) & ~1LL));  // [cap*cap]
  __shared__ double red[kBlockThreads / 32];
  __shared__ int snap_s;
  __shared__ double s_L;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = kBlockThreads / 32;
  pdl_wait();
  pdl_trigger();
  const int count = w.counters[kBigCount + (outer & 1)];
  if (blockIdx.x == 0 && threadIdx.x == 0) w.counters[kBigCount + ((outer + 1) & 1)] = 0;
  const int64_t cap = p.cap;
  for (int li = blockIdx.x; li < count; li += gridDim.x) {
    const int64_t b = big_list[li];
    CL_CHECK(b >= p.sig_lo && b < p.sig_hi && count <= p.B);
    const int t = w.cnt[b];
    CL_CHECK(t >= 0 && t <= cap && t <= kBlockRows * kBlockThreads);
    if (t <= skip_le) continue;  // learned by k_learn_cluster this iteration
    const int t0 = w.gcnt[b];
    double* G = w.gram + b * cap * cap;
    const double* y = w.y64 + b * p.ldm;
    for (int k = tid; k < t; k += kBlockThreads) sups[k] = w.sup[b * cap + k];
    __syncthreads();
    // Gram extension: gathered from the context's A^T A when present, else
    // warps over (k, i) pairs with lanes over m.
    for (int k = t0; k < t; ++k) {
      if (p.sep) {
        // Separable atoms: G[(i,j),(i',j')] = Gr[i][i'] * Gc[j][j'], b from Z.
        const int64_t pk = sups[k], ik = pk % p.nr, jk = pk / p.nr;
        for (int i = tid; i <= k; i += kBlockThreads) {
          const int64_t pi = sups[i], ii = pi % p.nr, ji = pi / p.nr;
          const double v = w.gr[ik * p.nr + ii] * w.gc[jk * p.nc + ji];
          G[(int64_t)k * cap + i] = v;
          G[(int64_t)i * cap + k] = v;
        }
        if (tid == 0) {
          w.bvec[b * cap + k] = w.zb[b * p.n + pk];
          w.coef[b * cap + k] = 0.0;
          w.mom1[b * cap + k] = 0.0;
          w.mom2[b * cap + k] = 0.0;
        }
        continue;
      }
      if (w.gfull) {
        for (int i = tid; i <= k; i += kBlockThreads) {
          const double v = w.gfull[(int64_t)sups[k] * p.n + sups[i]];
          G[(int64_t)k * cap + i] = v;
          G[(int64_t)i * cap + k] = v;
        }
      } else {
        for (int i = warp; i <= k; i += nw) {
          const float* ai = w.at32 + (int64_t)sups[i] * p.ldm;
          const float* ak = w.at32 + (int64_t)sups[k] * p.ldm;
          double acc = 0.0;
          for (int64_t q = lane; q < p.ldm; q += 32) acc = fma((double)ak[q], (double)ai[q], acc);
          acc = warp_sum(acc);
          if (lane == 0) {
            G[(int64_t)k * cap + i] = acc;
            G[(int64_t)i * cap + k] = acc;
          }
        }
      }
      if (warp == nw - 1) {
        double acc = 0.0;
        for (int64_t q = lane; q < p.ldm; q += 32)
          acc = fma((double)w.at32[(int64_t)sups[k] * p.ldm + q], y[q], acc);
        acc = warp_sum(acc);
        if (lane == 0) {
          w.bvec[b * cap + k] = acc;
          w.coef[b * cap + k] = 0.0;
          w.mom1[b * cap + k] = 0.0;
          w.mom2[b * cap + k] = 0.0;
        }
      }
    }
    __threadfence_block();
    __syncthreads();
    if (tid == 0) w.gcnt[b] = t;
    if (SMEM_G) {
      for (int64_t e = tid; e < (int64_t)t * t; e += kBlockThreads) {
        const int64_t r = e / t, cidx = e % t;
        Gs[r * cap + cidx] = G[r * cap + cidx];
      }
    }
    double c[kBlockRows], bi[kBlockRows], m1[kBlockRows], m2[kBlockRows];
#pragma unroll
    for (int q = 0; q < kBlockRows; ++q) {
      const int i = tid + q * kBlockThreads;
      c[q] = bi[q] = m1[q] = m2[q] = 0.0;
      if (i < t) {
        c[q] = w.coef[b * cap + i];
        bi[q] = w.bvec[b * cap + i];
        m1[q] = w.mom1[b * cap + i];
        m2[q] = w.mom2[b * cap + i];
        cs[i] = c[q];
      }
    }
    __syncthreads();
    const double* Gsrc = SMEM_G ? Gs : G;
    const int step0 = (outer - 1) * p.inner;
    for (int e = 0; e < p.inner; ++e) {
      double grad[kBlockRows];
#pragma unroll
      for (int q = 0; q < kBlockRows; ++q) {
        const int i = tid + q * kBlockThreads;
        grad[q] = 0.0;
        if (i < t) {
          double a0 = 0.0, a1 = 0.0;
          int j = 0;
          for (; j + 1 < t; j += 2) {
            a0 = fma(Gsrc[(int64_t)j * cap + i], cs[j], a0);
            a1 = fma(Gsrc[(int64_t)(j + 1) * cap + i], cs[j + 1], a1);
          }
          if (j < t) a0 = fma(Gsrc[(int64_t)j * cap + i], cs[j], a0);
          grad[q] = 2.0 * ((a0 + a1) - bi[q]);
        }
      }
      double bc1 = 1.0, bc2 = 1.0;
      if (OPT == 2) {
        bc1 = p.bc1[step0 + e];
        bc2 = p.bc2[step0 + e];
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kBlockRows; ++q) {
        const int i = tid + q * kBlockThreads;
        if (i < t) {
          opt_step<OPT>(c[q], grad[q], m1[q], m2[q], p.lr, bc1, bc2);
          cs[i] = c[q];
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < kBlockRows; ++q) {
      const int i = tid + q * kBlockThreads;
      if (i < t) {
        w.coef[b * cap + i] = c[q];
        w.mom1[b * cap + i] = m1[q];
        w.mom2[b * cap + i] = m2[q];
      }
    }
    if (p.sep) {  // the separable residual pipeline (k_sep.cu) takes over
      for (int i = tid; i < t; i += kBlockThreads) w.coef[b * cap + i] = cs[i];
      __syncthreads();
      continue;
    }
    // Residual + loss.
    double lacc = 0.0;
    for (int64_t i = tid; i < p.ldm; i += kBlockThreads) {
      double acc = 0.0;
      for (int k = 0; k < t; ++k)
        acc = fma((double)w.at32[(int64_t)sups[k] * p.ldm + i], cs[k], acc);
      const double rv = acc - y[i];
      w.r64[b * p.ldm + i] = rv;
      lacc = fma(rv, rv, lacc);
    }
    lacc = warp_sum(lacc);
    if (lane == 0) red[warp] = lacc;
    __syncthreads();
    if (tid == 0) {
      double L = 0.0;
      for (int q = 0; q < nw; ++q) L += red[q];
      s_L = L;
      snap_s = 0;
      if (p.prior)
        w.rloss[b] = L;  // k_prior_control adds the prior and decides
      else if (p.mode == kModePerSignal)
        snap_s = control_signal(p, w, b, outer, L);
      else
        w.loss[b] = L;
    }
    __syncthreads();
    if (w.r_hi) split_row(w, b, p.ldm, s_L, tid, kBlockThreads);  // own r64 entries
    if (snap_s)
      for (int i = tid; i < t; i += kBlockThreads) w.best_coef[b * cap + i] = cs[i];
    __syncthreads();
  }
}

// ------------------------------------- learning, CTA cluster per signal
// Supports of 33..256 atoms (config 3 and the one-signal path): the support
// Gram matrix lives in REGISTERS, spread over a cluster of Q CTAs (Q = 1, 2, 4
// for t <= 64, 128, 256).  CTA q, warp w owns rows [64q + 8w, 64q + 8w + 8),
// lane l owns columns [8l, 8l + 8): an 8 x 8 fp64 block per thread, loaded
// once per outer iteration.  An epoch is then 64 register FMAs per thread on
// the 8 coefficients of its columns (read from a shared-memory copy of c that
// every CTA of the cluster holds), a transposed butterfly across the warp that
// leaves each row's G c in lane 4i, the optimizer step of that row
// (gradient_step, clomp.cpp:171-209, g = 2 (G c - b)) and a store of the new
// coefficient into the next c buffer of every CTA of the cluster (distributed
// shared memory), closed by one cluster barrier.  The FMAs run from registers
// at the fp64 pipe's rate instead of 8 bytes of shared memory or L2 per FMA
// (k_learn_block), the rest of the outer iteration (Gram extension, residual,
// loss, stopping rules, snapshot) is split over the whole cluster.
// Generic transposed butterfly over RW row partials: lanes
// (lane >> (5 - log2 RW)) == i end with row i's warp total.
template <int RW>
__device__ __forceinline__ double warp_reduce_rows_t(double (&v)[RW], int lane) {
#pragma unroll
  for (int h = RW / 2, o = 16; h >= 1; h >>= 1, o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = up ? v[i] : v[i + h];
      const double keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(kFull, send, o);
    }
  }
  constexpr int kLog = RW >= 8 ? 3 : RW >= 4 ? 2 : RW >= 2 ? 1 : 0;
  double x = v[0];
#pragma unroll
  for (int o = 16 >> kLog; o >= 1; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

template <int Q>
__device__ __forceinline__ void cl_sync() {
  if (Q > 1)
    cooperative_groups::this_cluster().sync();
  else
    __syncthreads();
}

template <int Q, class T>
__device__ __forceinline__ T* cl_map(T* ptr, int rank) {
  if (Q > 1) return cooperative_groups::this_cluster().map_shared_rank(ptr, rank);
  return ptr;
}

__device__ __forceinline__ uint32_t cl_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Shared::cluster address of the same variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t cl_mapa(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

__device__ __forceinline__ void cl_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra W_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Residual rows r_i = sum_k a_{S_k, i} c_k - y_i (sequential k, fp64) for
// rows i = i0, i0 + stride, ...: RPT rows and 8 atoms per step, so 8 RPT
// independent gathers are in flight per thread instead of one.
template <int RPT>
__device__ __forceinline__ double resid_rows(const SolveParams& p, const Work& w, int64_t b,
                                             const int32_t* sups, const double* cs, int t,
                                             int64_t i0, int64_t stride) {
  const float* y = w.y32 + b * p.ldm;
  double lacc = 0.0;
  for (int64_t ib = i0; ib < p.ldm; ib += RPT * stride) {
    double acc[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) acc[u] = 0.0;
    int k = 0;
    for (; k + 8 <= t; k += 8) {
      float v[8][RPT];
#pragma unroll
      for (int z = 0; z < 8; ++z) {
        const float* ap = w.at32 + (int64_t)sups[k + z] * p.ldm;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int64_t i = ib + u * stride;
          v[z][u] = i < p.ldm ? ap[i] : 0.f;
        }
      }
#pragma unroll
      for (int z = 0; z < 8; ++z)
#pragma unroll
        for (int u = 0; u < RPT; ++u) acc[u] = fma(f2d(v[z][u]), cs[k + z], acc[u]);
    }
    for (; k < t; ++k) {
      const float* ap = w.at32 + (int64_t)sups[k] * p.ldm;
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int64_t i = ib + u * stride;
        if (i < p.ldm) acc[u] = fma(f2d(ap[i]), cs[k], acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t i = ib + u * stride;
      if (i < p.ldm) {
        const double rv = acc[u] - f2d(y[i]);
        w.r64[b * p.ldm + i] = rv;
        lacc = fma(rv, rv, lacc);
      }
    }
  }
  return lacc;
}

// Row blocks of 8 are dealt round-robin over the cluster (block rb -> CTA
// rb % Q, warp rb / Q), so every CTA owns rows whenever t > 8 (Q - 1): each
// CTA then has a warp that waits on every exchange phase, which keeps the
// phases of its barriers in order (see the epoch loop).
// Q CTAs of NWC warps; lane l owns CW columns [CW l, CW l + CW) of its warp's
// RW rows: t <= min(RW NWC Q, 32 CW).  Variants (Q, CW, NWC, RW):
// (1, 2, 8, 8) t <= 64, (1, 4, 16, 8) t <= 128 (one CTA, no remote traffic),
// (4, 8, 8, 8) t <= 256 ((8, 8, 8, 4), two CTAs per SM, for comparison).
template <int Q, int CW, int NWC, int RW>
constexpr int cl_min_blocks() { return ((Q == 1 && CW <= 2) || RW == 4) ? 2 : 1; }

#ifdef CL_CLUSTER_TRACE
// Debug (CL_NVCC_EXTRA=-DCL_CLUSTER_TRACE): clock64 split of the epoch loop,
// CTA 0 warp 0 lane 0 of every cluster launch accumulates
// [wait, fma, reduce, step+store, epochs] cycles.
__device__ unsigned long long g_cl_trace[8];
#endif

// PH (power form, plain GD, see k_pow_sq): 0 = every epoch here (E = inner);
// 1 = Gram extension plus the r leftover plain epochs, no residual tail (the
// squarings follow); 2 = q steps of c <- M c + d with M = T^(2^L), d = d_(2^L)
// from the power buffers, then the residual tail.  Signals past pw_slots run
// the PH 0 path inside the PH 1 launch.
template <int Q, int CW, int NWC, int RW, int OPT, int PH = 0>
__global__ void __launch_bounds__(32 * NWC, (cl_min_blocks<Q, CW, NWC, RW>()))
k_learn_cluster(SolveParams p, Work w, int outer, const int32_t* big_list) {
  constexpr int kClThreads = 32 * NWC;
  constexpr int kTmax = (RW * NWC * Q < 32 * CW) ? RW * NWC * Q : 32 * CW;
  constexpr int kRowShift = RW == 8 ? 2 : 3;  // lanes per row = 32 / RW
  __shared__ __align__(16) double cbuf[2][256];
  __shared__ __align__(8) uint64_t fullb[2];  // c buffer b complete (t * 8 bytes)
  __shared__ uint32_t s_phase[2];            // phases of fullb[] completed so far
  __shared__ int32_t sups[256];
  __shared__ double red[kClThreads / 32];
  __shared__ double lpart[8];  // rank 0: per-CTA loss partials
  __shared__ double s_L;
  __shared__ int s_snap;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nw = kClThreads / 32;
  const int q = Q > 1 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
  const int gt = q * kClThreads + tid;  // thread index within the cluster
  constexpr int GS = Q * kClThreads;    // cluster size in threads
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cl_smem_u32(&fullb[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cl_smem_u32(&fullb[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_phase[0] = s_phase[1] = 0;
  }
  pdl_wait();
  pdl_trigger();
  const int count = w.counters[kBigCount + (outer & 1)];
  const int64_t cap = p.cap;
  const int R0 = RW * (warp * Q + q), C0 = CW * lane;
  const int my_row = R0 + (lane >> kRowShift);
  // remote addresses: c buffers and their barriers in every CTA of the cluster
  uint32_t dst_c[Q], dst_b0[Q], dst_b1[Q];
#pragma unroll
  for (int r = 0; r < Q; ++r) {
    dst_c[r] = cl_mapa(cl_smem_u32(&cbuf[0][0]), r);
    dst_b0[r] = cl_mapa(cl_smem_u32(&fullb[0]), r);
    dst_b1[r] = cl_mapa(cl_smem_u32(&fullb[1]), r);
  }
  cl_sync<Q>();  // barriers initialised cluster-wide before any exchange
  for (int li = blockIdx.y; li < count; li += gridDim.y) {
    const int64_t b = big_list[li];
    const int t = w.cnt[b];
    if (t > kTmax) continue;  // uniform over the cluster: left to k_learn_block
    const bool pw = PH != 0 && li < p.pw_slots;  // power form for this signal
    if (PH == 2 && !pw) continue;                // learned by the PH 1 launch
#ifdef CL_CLUSTER_TRACE
    const unsigned long long tsig0 = clock64();
#endif
    const int t0 = w.gcnt[b];
    double* G = w.gram + b * cap * cap;
    const float* y = w.y32 + b * p.ldm;
    for (int k = tid; k < t; k += kClThreads) sups[k] = w.sup[b * cap + k];
    __syncthreads();
    // Gram extension for the atoms injected this iteration, over the cluster.
    for (int k = t0; k < t; ++k) {
      if (w.gfull) {
        for (int i = gt; i <= k; i += GS) {
          const double v = w.gfull[(int64_t)sups[k] * p.n + sups[i]];
          G[(int64_t)k * cap + i] = v;
          G[(int64_t)i * cap + k] = v;
        }
      } else {
        const float* ak = w.at32 + (int64_t)sups[k] * p.ldm;
        for (int i = q * nw + warp; i <= k; i += Q * nw) {
          const float* ai = w.at32 + (int64_t)sups[i] * p.ldm;
          double acc = 0.0;
          for (int64_t m = lane; m < p.ldm; m += 32) acc = fma(f2d(ak[m]), f2d(ai[m]), acc);
          acc = warp_sum(acc);
          if (lane == 0) {
            G[(int64_t)k * cap + i] = acc;
            G[(int64_t)i * cap + k] = acc;
          }
        }
      }
      if (q == Q - 1 && warp == nw - 1) {
        const float* ak = w.at32 + (int64_t)sups[k] * p.ldm;
        double acc = 0.0;
        for (int64_t m = lane; m < p.ldm; m += 32) acc = fma(f2d(ak[m]), f2d(y[m]), acc);
        acc = warp_sum(acc);
        if (lane == 0) {
          w.bvec[b * cap + k] = acc;
          w.coef[b * cap + k] = 0.0;
          w.mom1[b * cap + k] = 0.0;
          w.mom2[b * cap + k] = 0.0;
        }
      }
    }
    for (int k = tid; k < 256; k += kClThreads) {
      cbuf[1][k] = 0.0;  // padding rows stay exactly zero
      cbuf[0][k] = 0.0;
    }
    __threadfence();
    cl_sync<Q>();  // G, b, fresh coefficients visible to the whole cluster
    if (q == 0 && tid == 0) w.gcnt[b] = t;
    const int pwb = (p.pw_levels - 1) & 1;  // buffer holding T^(2^L), d_(2^L)
    const double* gsrc =
        PH == 2 ? w.pw_t + ((int64_t)pwb * p.pw_slots + li) * p.pw_ld * p.pw_ld : G;
    const int64_t ldg = PH == 2 ? p.pw_ld : cap;
    double g[RW][CW];
#pragma unroll
    for (int i = 0; i < RW; ++i)
#pragma unroll
      for (int j = 0; j < CW; ++j)
        g[i][j] = (R0 + i < t && C0 + j < t) ? gsrc[(int64_t)(R0 + i) * ldg + C0 + j] : 0.0;
    for (int k = tid; k < t; k += kClThreads) cbuf[0][k] = w.coef[b * cap + k];
    const bool producing = R0 < t;
    const bool owner = (lane & ((1 << kRowShift) - 1)) == 0 && my_row < t;
    double cr = 0.0, bi = 0.0, m1 = 0.0, m2 = 0.0;
    if (my_row < t) {
      cr = w.coef[b * cap + my_row];
      bi = PH == 2 ? w.pw_d[((int64_t)pwb * p.pw_slots + li) * p.pw_ld + my_row]
                   : w.bvec[b * cap + my_row];
      m1 = w.mom1[b * cap + my_row];
      m2 = w.mom2[b * cap + my_row];
    }
    uint32_t pc0 = s_phase[0], pc1 = s_phase[1];
    __syncthreads();
    const int step0 = (outer - 1) * p.inner;
    const int E = !pw ? p.inner : (PH == 1 ? p.pw_r : p.pw_q);
    // Epoch e reads buffer e & 1 and sends its rows' new coefficients into
    // buffer (e + 1) & 1 of every CTA (st.async, completing t * 8 bytes on
    // that CTA's barrier).  A sender has received every row of epoch e's
    // input, produced by warps that had themselves waited for the phase of
    // the buffer being overwritten, so a phase never receives bytes early.
#ifdef CL_CLUSTER_TRACE
    unsigned long long tw = 0, tf = 0, tr = 0, ts = 0, tcur = clock64();
    const bool tracer = q == 0 && tid == 0;
    const unsigned long long tpro = tcur - tsig0;  // prologue: loads, extension, syncs
#define CLT(acc) do { if (tracer) { const unsigned long long x = clock64(); acc += x - tcur; tcur = x; } } while (0)
#else
#define CLT(acc) do { } while (0)
#endif
    if (producing && E > 0) {
      for (int e = 0; e < E; ++e) {
        const int cur = e & 1, nxt = cur ^ 1;
        if (e > 0) {
          if (cur) {
            cl_mbar_wait(cl_smem_u32(&fullb[1]), pc1 & 1);
            ++pc1;
          } else {
            cl_mbar_wait(cl_smem_u32(&fullb[0]), pc0 & 1);
            ++pc0;
          }
        }
        if (tid == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                           cl_smem_u32(&fullb[nxt])),
                       "r"((uint32_t)(t * 8))
                       : "memory");
        double cv[CW];
        const double2* cp2 = reinterpret_cast<const double2*>(&cbuf[cur][C0]);
#pragma unroll
        for (int j = 0; j < CW / 2; ++j) {
          const double2 x = cp2[j];
          cv[2 * j] = x.x;
          cv[2 * j + 1] = x.y;
        }
        CLT(tw);
        double acc[RW];
#pragma unroll
        for (int i = 0; i < RW; ++i) {
          double a = 0.0;
#pragma unroll
          for (int j = 0; j < CW; ++j) a = fma(g[i][j], cv[j], a);
          acc[i] = a;
        }
#ifdef CL_CLUSTER_TRACE
        if (tracer && acc[0] == 12345.678) tw += 1;  // consume the FMAs before the mark
#endif
        CLT(tf);
        const double gc = warp_reduce_rows_t<RW>(acc, lane);
#ifdef CL_CLUSTER_TRACE
        if (tracer && gc == 12345.678) tw += 1;
#endif
        CLT(tr);
        if (owner) {
          double bc1 = 1.0, bc2 = 1.0;
          if (OPT == 2) {
            bc1 = p.bc1[step0 + e];
            bc2 = p.bc2[step0 + e];
          }
          if (PH == 2)
            cr = gc + bi;  // c <- T^(2^L) c + d_(2^L)
          else
            opt_step<OPT>(cr, 2.0 * (gc - bi), m1, m2, p.lr, bc1, bc2);
          const uint32_t off = (uint32_t)((nxt * 256 + my_row) * 8);
#pragma unroll
          for (int r = 0; r < Q; ++r)
            asm volatile(
                "st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(
                    dst_c[r] + off),
                "d"(cr), "r"(nxt ? dst_b1[r] : dst_b0[r])
                : "memory");
        }
        CLT(ts);
      }
#ifdef CL_CLUSTER_TRACE
      if (tracer) {
        atomicAdd(&g_cl_trace[0], tw);
        atomicAdd(&g_cl_trace[1], tf);
        atomicAdd(&g_cl_trace[2], tr);
        atomicAdd(&g_cl_trace[3], ts);
        atomicAdd(&g_cl_trace[4], (unsigned long long)E);
        atomicAdd(&g_cl_trace[5], tpro);
        atomicAdd(&g_cl_trace[7], 1ull);
      }
#endif
      const int fin = E & 1;
      cl_mbar_wait(cl_smem_u32(&fullb[fin]), (fin ? pc1 : pc0) & 1);
    }
    cl_sync<Q>();  // the final coefficients are in every CTA's buffer E & 1
    if (tid == 0) {
      s_phase[1] += (uint32_t)((E + 1) / 2);
      s_phase[0] += (uint32_t)(E / 2);
    }
    if (owner) {
      w.coef[b * cap + my_row] = cr;
      w.mom1[b * cap + my_row] = m1;
      w.mom2[b * cap + my_row] = m2;
    }
    if (pw) {  // PH 1: squarings and PH 2 follow; PH 2: k_pw_resid finishes it
      cl_sync<Q>();
#ifdef CL_CLUSTER_TRACE
      if (tracer) atomicAdd(&g_cl_trace[6], clock64() - tcur);  // after the epochs
#endif
      continue;
    }
    // Residual r = A_S c - y (fp64, rows over the cluster) and its loss.
    const double* cs = cbuf[E & 1];
    double lacc = resid_rows<4>(p, w, b, sups, cs, t, gt, GS);
    lacc = warp_sum(lacc);
    if (lane == 0) red[warp] = lacc;
    __syncthreads();
    if (tid == 0) {
      double L = 0.0;
      for (int k = 0; k < nw; ++k) L += red[k];
      *cl_map<Q>(&lpart[q], 0) = L;
    }
    cl_sync<Q>();
    if (q == 0 && tid == 0) {
      double L = 0.0;
      for (int r = 0; r < Q; ++r) L += lpart[r];
      int snap = 0;
      if (p.prior)
        w.rloss[b] = L;  // k_prior_control adds the prior and decides
      else if (p.mode == kModePerSignal)
        snap = control_signal(p, w, b, outer, L);
      else
        w.loss[b] = L;
      for (int r = 0; r < Q; ++r) {
        *cl_map<Q>(&s_L, r) = L;
        *cl_map<Q>(&s_snap, r) = snap;
      }
    }
    cl_sync<Q>();
    if (w.r_hi) split_row(w, b, p.ldm, s_L, gt, GS);  // rows this thread wrote
    if (s_snap)
      for (int k = gt; k < t; k += GS) w.best_coef[b * cap + k] = cs[k];
    cl_sync<Q>();  // smem (sups, cbuf, lpart) free for the next signal
  }
}

// ------------------------------- power form for cluster-sized supports
// Plain GD is affine, c <- T c + d with T = I - 2 lr G, d = 2 lr b
// (clomp.cpp:87-90, 178-181); E = 2^L q + r epochs equal r plain steps followed
// by q steps of c <- T^(2^L) c + d_(2^L) in exact arithmetic (the maps commute:
// both are c* + T^k (c - c*)).  k_learn_warp does this inside one warp for
// t <= 32; here the squarings of the 33..256-atom systems of the whole big
// list run as one batched fp64 tensor-core GEMM per level (mma.sync m8n8k4 f64
// -> DMMA), so the cluster kernel's latency-bound epoch chain shrinks from E
// to r + q steps.  Level l reads M_l (l = 0: T, built from G on load) and
// d_l, writes M_(l+1) = M_l^2 (upper 64 x 64 block triangle, mirrored: the
// powers of a symmetric T are symmetric) and d_(l+1) = d_l + M_l d_l.
// CTA = one 64 x 64 output block of one signal, 4 warps of 32 x 32 (4 x 4
// DMMA tiles each), k in chunks of 32 through padded shared memory (rows of
// 36 doubles: every fragment load is two conflict-free wavefronts).
#ifndef CL_PW_MINB
#define CL_PW_MINB 4
#endif
constexpr int kPwTile = 64;
#ifndef CL_PW_KC
#define CL_PW_KC 16
#endif
constexpr int kPwKc = CL_PW_KC;
constexpr int kPwThreads = 128;
constexpr int kPwSmem = 4 * kPwTile * (kPwKc + 4) * 8;  // 2 stages x 2 panels

// Gram extension of the power-form signals (the first pw_slots of the big
// list with t <= tmax), one CTA per signal: the new rows / columns of G and
// b_k = a_k . y for the atoms injected this iteration, new coefficients 0
// (clomp.hpp:53-54).
constexpr int kPwExtThreads = 128;

__global__ void __launch_bounds__(kPwExtThreads)
k_pw_extend(SolveParams p, Work w, int outer, const int32_t* big_list, int tmax) {
  __shared__ double red[kPwExtThreads / 32];
  pdl_wait();
  pdl_trigger();
  const int count = min(w.counters[kBigCount + (outer & 1)], p.pw_slots);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int li = blockIdx.x;
  if (li >= count) return;
  const int64_t b = big_list[li];
  const int t = w.cnt[b];
  if (t > tmax) return;
  const int t0 = w.gcnt[b];
  const int64_t cap = p.cap, ldm = p.ldm;
  double* G = w.gram + b * cap * cap;
  const int32_t* sup = w.sup + b * cap;
  const float* y = w.y32 + b * ldm;
  for (int k = t0; k < t; ++k) {
    const int64_t jk = sup[k];
    const float* ak = w.at32 + jk * ldm;
    if (w.gfull) {
      for (int i = tid; i <= k; i += kPwExtThreads) {
        const double v = w.gfull[jk * p.n + sup[i]];
        G[(int64_t)k * cap + i] = v;
        G[(int64_t)i * cap + k] = v;
      }
    } else {
      for (int i = warp; i <= k; i += kPwExtThreads / 32) {
        const float* ai = w.at32 + (int64_t)sup[i] * ldm;
        double acc = 0.0;
        for (int64_t m = lane; m < ldm; m += 32) acc = fma(f2d(ak[m]), f2d(ai[m]), acc);
        acc = warp_sum(acc);
        if (lane == 0) {
          G[(int64_t)k * cap + i] = acc;
          G[(int64_t)i * cap + k] = acc;
        }
      }
    }
    double acc = 0.0;
    for (int64_t m = 4 * tid; m < ldm; m += 4 * kPwExtThreads) {
      const float4 a = *reinterpret_cast<const float4*>(ak + m);
      const float4 v = *reinterpret_cast<const float4*>(y + m);
      acc = fma(f2d(a.x), f2d(v.x), acc);
      acc = fma(f2d(a.y), f2d(v.y), acc);
      acc = fma(f2d(a.z), f2d(v.z), acc);
      acc = fma(f2d(a.w), f2d(v.w), acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      double bk = 0.0;
      for (int q = 0; q < kPwExtThreads / 32; ++q) bk += red[q];
      w.bvec[b * cap + k] = bk;
      w.coef[b * cap + k] = 0.0;
      w.mom1[b * cap + k] = 0.0;
      w.mom2[b * cap + k] = 0.0;
    }
    __syncthreads();
  }
  if (tid == 0) w.gcnt[b] = t;
}

__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void cp_async8_zfill(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}

__global__ void __launch_bounds__(kPwThreads, CL_PW_MINB)
k_pow_sq(SolveParams p, Work w, int outer, const int32_t* big_list, int level, int tmax,
         int nt) {
  // two k-chunk stages of both 64-row panels (cp.async ring), dynamic smem
  extern __shared__ __align__(16) double pw_smem[];
  typedef double Panel[kPwTile][kPwKc + 4];
  Panel* As = reinterpret_cast<Panel*>(pw_smem);
  Panel* Bs = As + 2;
  pdl_wait();
  pdl_trigger();
  const int count = min(w.counters[kBigCount + (outer & 1)], p.pw_slots);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int fr = lane >> 2, fc = lane & 3;  // fragment row / column
  const double twolr = 2.0 * p.lr;
  const int64_t ld = p.pw_ld;
  // output block (I, J), J >= I, of the upper block triangle of an nt x nt grid
  int I = 0, J = 0;
  {
    int x = blockIdx.x;
    for (I = 0; I < nt; ++I) {
      if (x < nt - I) {
        J = I + x;
        break;
      }
      x -= nt - I;
    }
  }
  const bool from_g = level == 0;
  for (int li = blockIdx.y; li < count; li += gridDim.y) {
    const int64_t b = big_list[li];
    const int t = w.cnt[b];
    if (t > tmax || J * kPwTile >= t) continue;  // uniform per CTA
    const double* src = from_g ? w.gram + b * p.cap * p.cap
                               : w.pw_t + ((int64_t)((level - 1) & 1) * p.pw_slots + li) * ld * ld;
    const int64_t lds = from_g ? p.cap : ld;
    double* dst = w.pw_t + ((int64_t)(level & 1) * p.pw_slots + li) * ld * ld;
    const bool aligned = !from_g || (p.cap & 1) == 0;
    // stage chunk kc of rows I / J: 16-byte copies, zero-filled outside t x t
    auto issue = [&](int chunk) {
      const int st = chunk & 1, k0 = chunk * kPwKc;
#pragma unroll
      for (int e = tid; e < kPwTile * kPwKc / 2; e += kPwThreads) {
        const int r = e / (kPwKc / 2), c = 2 * (e % (kPwKc / 2));
        const int k = k0 + c;
        const int kb = k < t ? (k + 1 < t ? 16 : 8) : 0;
        const int ra = I * kPwTile + r, rb = J * kPwTile + r;
        const double* pa = src + (int64_t)(ra < t ? ra : 0) * lds + (kb ? k : 0);
        const double* pb = src + (int64_t)(rb < t ? rb : 0) * lds + (kb ? k : 0);
        if (aligned) {
          cp_async16_zfill(&As[st][r][c], pa, ra < t ? kb : 0);
          cp_async16_zfill(&Bs[st][r][c], pb, rb < t ? kb : 0);
        } else {  // odd row stride (G with odd cap): 8-byte copies
          const int k1 = kb == 16 ? 8 : 0;
          cp_async8_zfill(&As[st][r][c], pa, ra < t && kb ? 8 : 0);
          cp_async8_zfill(&As[st][r][c + 1], pa + (k1 ? 1 : 0), ra < t ? k1 : 0);
          cp_async8_zfill(&Bs[st][r][c], pb, rb < t && kb ? 8 : 0);
          cp_async8_zfill(&Bs[st][r][c + 1], pb + (k1 ? 1 : 0), rb < t ? k1 : 0);
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[4][4][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    const int nchunk = (t + kPwKc - 1) / kPwKc;
    issue(0);
    for (int ch = 0; ch < nchunk; ++ch) {
      const int st = ch & 1;
      if (ch + 1 < nchunk) {
        issue(ch + 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      if (from_g) {  // T = I - 2 lr G on the staged entries (zeros stay zero)
        const int k0 = ch * kPwKc;
        for (int e = tid; e < kPwTile * kPwKc; e += kPwThreads) {
          const int r = e / kPwKc, c = e % kPwKc, k = k0 + c;
          const int ra = I * kPwTile + r, rb = J * kPwTile + r;
          if (k < t) {
            if (ra < t) As[st][r][c] = ra == k ? 1.0 - twolr * As[st][r][c] : -(twolr * As[st][r][c]);
            if (rb < t) Bs[st][r][c] = rb == k ? 1.0 - twolr * Bs[st][r][c] : -(twolr * Bs[st][r][c]);
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int ks = 0; ks < kPwKc / 4; ++ks) {
        double fa[4], fb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          fa[i] = As[st][wm * 32 + i * 8 + fr][ks * 4 + fc];
          fb[i] = Bs[st][wn * 32 + i * 8 + fr][ks * 4 + fc];
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
            asm volatile(
                "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(acc[mi][ni][0]), "+d"(acc[mi][ni][1])
                : "d"(fa[mi]), "d"(fb[ni]));
      }
      __syncthreads();  // stage st is refilled by the next issue
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int row = I * kPwTile + wm * 32 + mi * 8 + fr;
        const int col = J * kPwTile + wn * 32 + ni * 8 + 2 * fc;
        if (row < t) {
          if (col + 1 < t) {
            *reinterpret_cast<double2*>(dst + (int64_t)row * ld + col) =
                make_double2(acc[mi][ni][0], acc[mi][ni][1]);
          } else if (col < t) {
            dst[(int64_t)row * ld + col] = acc[mi][ni][0];
          }
          if (I != J) {
            if (col < t) dst[(int64_t)col * ld + row] = acc[mi][ni][0];
            if (col + 1 < t) dst[(int64_t)(col + 1) * ld + row] = acc[mi][ni][1];
          }
        }
      }
    if (I == J) {
      // d_(l+1) = d_l + M_l d_l on this block's rows (d_0 = 2 lr b)
      const double* dsrc = from_g ? w.bvec + b * p.cap
                                  : w.pw_d + ((int64_t)((level - 1) & 1) * p.pw_slots + li) * ld;
      double* ddst = w.pw_d + ((int64_t)(level & 1) * p.pw_slots + li) * ld;
      const double dscale = from_g ? twolr : 1.0;
      for (int rr = 0; rr < kPwTile / 4; ++rr) {
        const int i = I * kPwTile + warp * (kPwTile / 4) + rr;
        if (i >= t) break;
        const double* mrow = src + (int64_t)i * lds;
        double a = 0.0;
        for (int k = lane; k < t; k += 32) {
          const double v = mrow[k];
          const double mik = !from_g ? v : (i == k ? 1.0 - twolr * v : -(twolr * v));
          a = fma(mik, dscale * dsrc[k], a);
        }
        a = warp_sum(a);
        if (lane == 0) ddst[i] = dscale * dsrc[i] + a;
      }
    }
  }
}

// Residual tail of the power-form signals after the PH 2 epochs (what
// k_learn_cluster's tail does for the others): r = A_S c - y in fp64 over
// row chunks of 512 — one CTA each, four consecutive rows per thread (float4
// atom loads, eight atoms in flight), many CTAs per SM so the gathers of the
// 33..256-atom supports overlap — and per-chunk loss partials.  The last CTA
// of a signal sums them in chunk order, runs the stopping rules
// (clomp.cpp:253-273, eps test :238-242), writes the fp16 split for the next
// K1 and the best snapshot.
constexpr int kPwResThreads = 128;
constexpr int kPwResRows = 4 * kPwResThreads;

__global__ void __launch_bounds__(kPwResThreads)
k_pw_resid(SolveParams p, Work w, int outer, const int32_t* big_list, int tmax) {
  __shared__ __align__(16) double cs[256];
  __shared__ int32_t ss[256];
  __shared__ double red[kPwResThreads / 32];
  __shared__ double s_L;
  __shared__ int s_last, s_snap;
  pdl_wait();
  pdl_trigger();
  const int count = min(w.counters[kBigCount + (outer & 1)], p.pw_slots);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nchunk = (int)((p.ldm + kPwResRows - 1) / kPwResRows);
  const int64_t cap = p.cap, ldm = p.ldm;
  for (int li = blockIdx.y; li < count; li += gridDim.y) {
    const int64_t b = big_list[li];
    const int t = w.cnt[b];
    if (t > tmax) continue;  // uniform per CTA
    for (int k = tid; k < t; k += kPwResThreads) {
      cs[k] = w.coef[b * cap + k];
      ss[k] = w.sup[b * cap + k];
    }
    __syncthreads();
    const int64_t i0 = (int64_t)blockIdx.x * kPwResRows + 4 * tid;
    double lacc = 0.0;
    if (i0 < ldm) {  // ldm is a multiple of 128: rows i0 .. i0 + 3 all exist
      double r[4] = {0.0, 0.0, 0.0, 0.0};
      int k = 0;
      for (; k + 8 <= t; k += 8) {
        float4 v[8];
#pragma unroll
        for (int z = 0; z < 8; ++z)
          v[z] = *reinterpret_cast<const float4*>(w.at32 + (int64_t)ss[k + z] * ldm + i0);
#pragma unroll
        for (int z = 0; z < 8; ++z) {
          const double c = cs[k + z];
          r[0] = fma(f2d(v[z].x), c, r[0]);
          r[1] = fma(f2d(v[z].y), c, r[1]);
          r[2] = fma(f2d(v[z].z), c, r[2]);
          r[3] = fma(f2d(v[z].w), c, r[3]);
        }
      }
      for (; k < t; ++k) {
        const float4 v = *reinterpret_cast<const float4*>(w.at32 + (int64_t)ss[k] * ldm + i0);
        const double c = cs[k];
        r[0] = fma(f2d(v.x), c, r[0]);
        r[1] = fma(f2d(v.y), c, r[1]);
        r[2] = fma(f2d(v.z), c, r[2]);
        r[3] = fma(f2d(v.w), c, r[3]);
      }
      const float4 yv = *reinterpret_cast<const float4*>(w.y32 + b * ldm + i0);
      r[0] -= f2d(yv.x);
      r[1] -= f2d(yv.y);
      r[2] -= f2d(yv.z);
      r[3] -= f2d(yv.w);
      *reinterpret_cast<double2*>(w.r64 + b * ldm + i0) = make_double2(r[0], r[1]);
      *reinterpret_cast<double2*>(w.r64 + b * ldm + i0 + 2) = make_double2(r[2], r[3]);
#pragma unroll
      for (int e = 0; e < 4; ++e) lacc = fma(r[e], r[e], lacc);
    }
    lacc = warp_sum(lacc);
    if (lane == 0) red[warp] = lacc;
    __syncthreads();
    if (tid == 0) {
      double part = 0.0;
      for (int q = 0; q < kPwResThreads / 32; ++q) part += red[q];
      w.pw_part[(int64_t)li * nchunk + blockIdx.x] = part;
      __threadfence();
      s_last = atomicAdd(&w.pw_cnt[li], 1) == nchunk - 1;
    }
    __syncthreads();
    if (s_last) {  // every chunk's rows and partial are visible
      __threadfence();
      if (tid == 0) {
        double L = 0.0;
        for (int q = 0; q < nchunk; ++q) L += __ldcg(&w.pw_part[(int64_t)li * nchunk + q]);
        w.pw_cnt[li] = 0;
        int snap = 0;
        if (p.mode == kModePerSignal)
          snap = control_signal(p, w, b, outer, L);
        else
          w.loss[b] = L;
        s_L = L;
        s_snap = snap;
      }
      __syncthreads();
      if (w.r_hi) {
        const float sc = split_scale(s_L);
        if (tid == 0) w.r_scale[b] = 1.0f / sc;
        for (int64_t i = tid; i < ldm; i += kPwResThreads)
          split_f16(__ldcg(&w.r64[b * ldm + i]), sc, w.r_hi[b * ldm + i], w.r_lo[b * ldm + i]);
      }
      if (s_snap)
        for (int k = tid; k < t; k += kPwResThreads) w.best_coef[b * cap + k] = cs[k];
    }
    __syncthreads();  // cs / ss / flags reused by the next signal
  }
}

// ------------------------------------------------------------- priors
// TV-1D (priors.cpp:11-26) on x = D s of a single-column solve is the
// quadratic form tv = s^T H s with H = (Delta D)^T (Delta D) / n, Delta the
// forward difference; its chained gradient D^T (w dtv/dx) (clomp.cpp:93-117)
// is 2 w H s.  On the support the learning system becomes
// g = 2 ((G + w H) c - b), so every learning kernel runs unchanged on
// G + w H, and the loss the stopping rules read is ||r||^2 + w c^T H c
// (lb.total, clomp.cpp:126).  k_prior_ext builds the Gram and H rows of the
// atoms selected this iteration (the learning kernels then find nothing to
// extend); k_prior_control adds the prior to the residual loss the learning
// kernels stored and runs the per-signal stopping rules.
constexpr int kPriorThreads = 128;

__global__ void __launch_bounds__(kPriorThreads)
k_prior_ext(SolveParams p, Work w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int nw = kPriorThreads / 32;
  const int64_t cap = p.cap;
  const double inv_n = 1.0 / (double)p.n;
  pdl_wait();
  pdl_trigger();
  for (int64_t b = p.sig_lo + blockIdx.x; b < p.sig_hi; b += gridDim.x) {
    if (!w.active[b]) continue;
    const int t = w.cnt[b], t0 = w.gcnt[b];
    if (t0 >= t) continue;
    const double wb = w.wtv ? w.wtv[b] : 0.0;  // image mode: data Gram only
    double* G = w.gram + b * cap * cap;
    double* H = w.hgram ? w.hgram + b * cap * cap : nullptr;
    const int32_t* sup = w.sup + b * cap;
    const float* y = w.y32 + b * p.ldm;
    for (int k = t0; k < t; ++k) {
      const int64_t sk = sup[k];
      const float* ak = w.at32 + sk * p.ldm;
      const double* dk = w.hgram ? w.ddt + sk * w.ldd : nullptr;
      for (int i = warp; i <= k; i += nw) {
        const int64_t si = sup[i];
        double g = 0.0;
        if (w.gfull) {
          g = w.gfull[sk * p.n + si];
        } else {
          const float* ai = w.at32 + si * p.ldm;
          for (int64_t q = lane; q < p.ldm; q += 32) g = fma(f2d(ak[q]), f2d(ai[q]), g);
          g = warp_sum(g);
        }
        double h = 0.0;
        if (H) {
          const double* di = w.ddt + si * w.ldd;
          for (int64_t q = lane; q < w.ldd; q += 32) h = fma(dk[q], di[q], h);
          h = warp_sum(h) * inv_n;
        }
        if (lane == 0) {
          const double v = g + wb * h;
          G[(int64_t)k * cap + i] = v;
          G[(int64_t)i * cap + k] = v;
          if (H) {
            H[(int64_t)k * cap + i] = h;
            H[(int64_t)i * cap + k] = h;
          }
        }
      }
      if (warp == nw - 1) {
        double acc = 0.0;
        for (int64_t q = lane; q < p.ldm; q += 32) acc = fma(f2d(ak[q]), f2d(y[q]), acc);
        acc = warp_sum(acc);
        if (lane == 0) {
          w.bvec[b * cap + k] = acc;
          w.coef[b * cap + k] = 0.0;  // new atoms start at 0 (clomp.hpp:53-54)
          w.mom1[b * cap + k] = 0.0;
          w.mom2[b * cap + k] = 0.0;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) w.gcnt[b] = t;
  }
}

// Warp per signal: tv = c^T H c, total = ||r||^2 + w tv, stopping rules and
// the best snapshot (clomp.cpp:253-273).
__global__ void __launch_bounds__(128)
k_prior_control(SolveParams p, Work w, int outer) {
  const int lane = threadIdx.x & 31;
  pdl_wait();
  pdl_trigger();
  const int64_t b = p.sig_lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (b >= p.sig_hi || !w.active[b]) return;
  const int64_t cap = p.cap;
  const int t = w.cnt[b];
  const double* H = w.hgram + b * cap * cap;
  const double* c = w.coef + b * cap;
  double acc = 0.0;
  for (int i = lane; i < t; i += 32) {
    double row = 0.0;
    for (int j = 0; j < t; ++j) row = fma(H[(int64_t)j * cap + i], c[j], row);
    acc = fma(c[i], row, acc);
  }
  const double tv = warp_sum(acc);
  int snap = 0;
  if (lane == 0) {
    const double Lr = w.rloss[b];
    snap = control_signal(p, w, b, outer, Lr + w.wtv[b] * tv, load_ctl(w, b), Lr);
  }
  snap = __shfl_sync(kFull, snap, 0);
  if (snap)
    for (int i = lane; i < t; i += 32) w.best_coef[b * cap + i] = c[i];
}

// ------------------------------------------------------------ image mode
// The reference's column-batch image path (cskit.cpp:620-652): one joint
// clomp_solve_batch over the columns of an image, whose priors couple the
// columns — TV-2D (priors.cpp:28-59) and local variance (priors.cpp:74-116) on
// the n x B image x = D S_eff (clomp.cpp:93-119), batch-global weights and
// stopping.  The data term stays in the per-column Gram form; every epoch is
//   k_img_synth  per column: gd = 2 (G c - b) and x_b = D_S c_b
//   k_img_lv     per LV window: mean, sd (stats of the current x)
//   k_img_gx     per pixel: gx = w_tv dtv/dx + w_lv dlv/dx
//   k_img_step   per column: g = gd + (D^T gx)_S, optimizer step (gradient_step)
// and after the epochs the residual per column plus k_img_loss (tv, lv of the
// final x) feed k_joint_control.  Pixel (q, b) of x is img_x[b * n + q].
constexpr int kImgThreads = 256;

__global__ void __launch_bounds__(kImgThreads)
k_img_synth(SolveParams p, Work w, int grad) {
  extern __shared__ __align__(16) unsigned char ism[];
  double* cs = reinterpret_cast<double*>(ism);
  int32_t* sups = reinterpret_cast<int32_t*>(cs + p.cap);
  const int tid = threadIdx.x;
  const int64_t cap = p.cap, n = p.n;
  pdl_wait();
  pdl_trigger();
  for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x) {
    if (!w.active[b]) continue;
    const int t = w.cnt[b];
    for (int k = tid; k < t; k += kImgThreads) {
      cs[k] = w.coef[b * cap + k];
      sups[k] = w.sup[b * cap + k];
    }
    __syncthreads();
    if (grad) {
      const double* G = w.gram + b * cap * cap;
      for (int i = tid; i < t; i += kImgThreads) {
        double acc = 0.0;
        for (int j = 0; j < t; ++j) acc = fma(G[(int64_t)j * cap + i], cs[j], acc);
        w.img_gd[b * cap + i] = 2.0 * (acc - w.bvec[b * cap + i]);
      }
    }
    for (int64_t q = tid; q < n; q += kImgThreads) {
      double acc = 0.0;
      for (int k = 0; k < t; ++k) acc = fma(w.dt[(int64_t)sups[k] * n + q], cs[k], acc);
      w.img_x[b * n + q] = acc;
    }
    __syncthreads();
  }
}

// Local-variance window statistics: mean, sd, and the gradient scale
// inv_blocks / (count sd) (0 where sd == 0: no gradient, priors.cpp:106).
__global__ void k_img_lv(SolveParams p, Work w) {
  pdl_wait();
  pdl_trigger();
  const int64_t win = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nwin = (int64_t)p.lv_nr * p.lv_nc;
  if (win >= nwin || !w.active[0]) return;
  const int r0 = w.lv_rows[win / p.lv_nc], c0 = w.lv_cols[win % p.lv_nc];
  const int W = p.lv_window;
  double sum = 0.0, sum_sq = 0.0;
  for (int j = 0; j < W; ++j)
    for (int i = 0; i < W; ++i) {
      const double v = w.img_x[(int64_t)(c0 + j) * p.n + r0 + i];
      sum += v;
      sum_sq = fma(v, v, sum_sq);
    }
  const double count = (double)(W * W);
  const double mean = sum / count;
  const double var = fmax(sum_sq / count - mean * mean, 0.0);
  const double sd = sqrt(var);
  const double inv_blocks = 1.0 / (double)nwin;
  w.lv_mean[win] = mean;
  w.lv_sd[win] = sd;
  w.lv_scale[win] = sd > 0.0 ? inv_blocks / (count * sd) : 0.0;
}

__global__ void k_img_gx(SolveParams p, Work w) {
  pdl_wait();
  pdl_trigger();
  const int64_t n = p.n, B = p.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * B || !w.active[0]) return;
  const int64_t b = e / n, q = e % n;
  const double* x = w.img_x;
  const double xv = x[e];
  double g = 0.0;
  if (p.w_tv_g > 0.0) {
    const double ih = 2.0 / (double)n, iw = 2.0 / (double)B;
    double gv = 0.0;
    if (n >= 2) {
      if (q + 1 < n) gv += ih * (xv - x[e + 1]);
      if (q > 0) gv -= ih * (x[e - 1] - xv);
    }
    if (B >= 2) {
      if (b + 1 < B) gv += iw * (xv - x[e + n]);
      if (b > 0) gv -= iw * (x[e - n] - xv);
    }
    g = p.w_tv_g * gv;
  }
  if (p.lv_on) {
    double gl = 0.0;
    for (int a = 0; a < kLvCover; ++a) {
      const int ri = w.lv_rowcov[q * kLvCover + a];
      if (ri < 0) break;
      for (int c = 0; c < kLvCover; ++c) {
        const int ci = w.lv_colcov[b * kLvCover + c];
        if (ci < 0) break;
        const int64_t win = (int64_t)ri * p.lv_nc + ci;
        gl = fma(w.lv_scale[win], xv - w.lv_mean[win], gl);
      }
    }
    g = fma(p.w_lv_g, gl, g);
  }
  w.img_gx[e] = g;
}

template <int OPT>
__global__ void __launch_bounds__(kImgThreads)
k_img_step(SolveParams p, Work w, int outer, int e) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int nw = kImgThreads / 32;
  const int64_t cap = p.cap, n = p.n;
  pdl_wait();
  pdl_trigger();
  double bc1 = 1.0, bc2 = 1.0;
  if (OPT == 2) {
    const int step = (outer - 1) * p.inner + e;
    bc1 = p.bc1[step];
    bc2 = p.bc2[step];
  }
  for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x) {
    if (!w.active[b]) continue;
    const int t = w.cnt[b];
    const double* gx = w.img_gx + b * n;
    for (int k = warp; k < t; k += nw) {
      const double* dk = w.dt + (int64_t)w.sup[b * cap + k] * n;
      double acc = 0.0;
      for (int64_t q = lane; q < n; q += 32) acc = fma(dk[q], gx[q], acc);
      acc = warp_sum(acc);
      if (lane == 0) {
        const int64_t o = b * cap + k;
        double c = w.coef[o], m1 = w.mom1[o], m2 = w.mom2[o];
        opt_step<OPT>(c, w.img_gd[o] + acc, m1, m2, p.lr, bc1, bc2);
        w.coef[o] = c;
        w.mom1[o] = m1;
        w.mom2[o] = m2;
      }
    }
  }
}

// Residual of every column after the epochs (fp64, stored for the next
// correlation with its split) into loss[b].
__global__ void __launch_bounds__(128)
k_img_resid(SolveParams p, Work w) {
  const int lane = threadIdx.x & 31;
  pdl_wait();
  pdl_trigger();
  const int64_t b = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (b >= p.B || !w.active[b]) return;
  const int t = w.cnt[b];
  const double L = warp_residual(p, w, b, w.coef + b * p.cap, w.sup + b * p.cap, t, lane);
  if (lane == 0) w.loss[b] = L;
}

// tv and lv of the final x (one block, fixed reduction order):
// joint[kJPrior] = w_tv tv + w_lv lv (lb.total's prior part, clomp.cpp:126).
__global__ void __launch_bounds__(1024)
k_img_loss(SolveParams p, Work w) {
  __shared__ double red_tv[1024], red_lv[1024];
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x;
  if (!w.active[0]) return;
  const int64_t n = p.n, B = p.B;
  double tv = 0.0, lv = 0.0;
  if (p.w_tv_g > 0.0) {
    const double ih = 1.0 / (double)n, iw = 1.0 / (double)B;
    for (int64_t e = tid; e < n * B; e += 1024) {
      const int64_t b = e / n, q = e % n;
      const double xv = w.img_x[e];
      if (q + 1 < n) {
        const double d = xv - w.img_x[e + 1];
        tv = fma(ih * d, d, tv);
      }
      if (b + 1 < B) {
        const double d = xv - w.img_x[e + n];
        tv = fma(iw * d, d, tv);
      }
    }
  }
  if (p.lv_on) {
    const int64_t nwin = (int64_t)p.lv_nr * p.lv_nc;
    const double inv_blocks = 1.0 / (double)nwin;
    for (int64_t win = tid; win < nwin; win += 1024) lv = fma(inv_blocks, w.lv_sd[win], lv);
  }
  red_tv[tid] = tv;
  red_lv[tid] = lv;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (tid < o) {
      red_tv[tid] += red_tv[tid + o];
      red_lv[tid] += red_lv[tid + o];
    }
    __syncthreads();
  }
  if (tid == 0) w.joint[kJPrior] = p.w_tv_g * red_tv[0] + p.w_lv_g * red_lv[0];
}

// ------------------------------------------------------ fused small solve
// Whole clomp_solve (clomp.cpp:294-311, i.e. clomp_solve_batch on one column)
// in one persistent block per signal for small dictionaries (config 1 and
// other latency-bound cases): exact fp64 correlation of every atom (warps over
// atoms, lanes over measurements), the inject_from_scores rule with ties, the
// warp learning routine of the batched path, the fp64 residual and the
// stopping rules, with no kernel boundary between outer iterations.
constexpr int kFusedThreads = 256;
#ifndef CL_FUSED_ATOMS
#define CL_FUSED_ATOMS 32
#endif
constexpr int kFusedAtoms = CL_FUSED_ATOMS;  // atoms per warp pass of the correlation (was 8)
#ifndef CL_FUSED_STAGE_MAX
#define CL_FUSED_STAGE_MAX (200 * 1024)
#endif
constexpr int kFusedStageMax = CL_FUSED_STAGE_MAX;  // dynamic smem cap for the staged dictionary

// Everything a signal's solve touches between outer iterations stays on chip:
// the residual, y, the scores, the support / coefficients / b / moments, the
// support Gram matrix, the mask and the stopping-rule state live in shared
// memory (round 1 kept them in global memory and paid ~8 dependent round trips
// per outer iteration: 18.6 us each at config 1).  What still leaves the SM per
// iteration is the gather of the new Gram row from A^T A (one L2 round trip)
// and fire-and-forget stores.  The state k_finalize reads is written once at
// the end.
#ifdef CL_LEARN_TRACE
// phase marks of signal 0's outer iterations in the fused kernel (row = outer)
#define FT_MARK(i) do { if (tid == 0 && b == 0 && outer < 8192) g_lt[outer][i] = (unsigned long long)clock64(); } while (0)
#else
#define FT_MARK(i) do { } while (0)
#endif

struct FusedCtl {
  double best_L, prev_L, loss;
  int t, t0, stall, iters, status, conv, active, best_cnt, changed;
};

// STAGED: the dictionary lives in shared memory MEASUREMENT-major, AT[i][j] with
// an odd row stride n + 1 floats, so that (a) the correlation runs one thread
// per atom, serial over the measurements with r[i] broadcast — consecutive
// atoms are consecutive words, no shuffles, 4 partial sums per atom in a fixed
// order — and (b) column reads (b_k, the residual's A[i][sup_k]) hit distinct
// banks.  Round 1 staged it atom-major and reduced 32 dot products per warp
// with 160 shuffles: 13.6 k of the 26.5 k cycles of a config-1 outer iteration
// (tools/fused_trace.py).  !STAGED (dictionary too large for shared memory, or
// more signals than SMs) keeps the atom-major global reads.
// The kernel also does what k_init and k_finalize do for the batched path (y in,
// r = -y, the eps test at s = 0; the snapshot rule, support sorted ascending,
// final norm and flags out), so a whole solve is one kernel node.
struct FusedIo {
  const float* y;       // m x B (y_ref) or B x y_ld
  int64_t y_ld;
  int32_t y_ref;
  int64_t out_cap;
  int32_t* sup;
  double* coef;
  int32_t* cnt;
  int32_t* iters;
  double* rn;
  uint8_t* conv;
  int32_t* status;
};

template <int OPT, bool STAGED>
__global__ void __launch_bounds__(kFusedThreads)
k_solve_fused(SolveParams p, Work w, int sc_smem, FusedIo io) {
  extern __shared__ __align__(16) unsigned char fsm[];
  double* rs = reinterpret_cast<double*>(fsm);                 // [ldm] residual
  double* ys = rs + p.ldm;                                     // [ldm] y (fp32 values, exact)
  double* sc_s = ys + p.ldm;                                   // [n] |scores| (sc_smem)
  uint32_t* mask = reinterpret_cast<uint32_t*>(sc_s + (sc_smem ? p.n : 0));  // [mwords, padded]
  float* As = reinterpret_cast<float*>(mask + 2 * ((p.mwords + 3) & ~3LL));  // [m][n + 1] (STAGED)
  const int64_t lda = p.n + 1;
  __shared__ __align__(16) double cs[2 * kWarpCap];
  __shared__ __align__(16) double sq[kWarpCap * (kWarpCap + 4)];   // learn_epochs work buffer
  __shared__ __align__(16) double Gs[kWarpCap * (kWarpCap + 4)];   // support Gram, persistent
  __shared__ double s_c[kWarpCap], s_b[kWarpCap], s_m1[kWarpCap], s_m2[kWarpCap], s_best[kWarpCap];
  __shared__ int32_t sups[kWarpCap];
  __shared__ double red[kFusedThreads / 32];
  __shared__ FusedCtl ctl;
  uint32_t* pickw = mask + ((p.mwords + 3) & ~3LL);  // [mwords] this iteration's picks
  constexpr int LDS = kWarpCap + 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = kFusedThreads / 32;
  const int64_t b = blockIdx.x;
  // k_init: y, r = A*0 - y = -y (clomp.cpp:236-237 at s = 0), ||y||^2
  for (int64_t i = tid; i < p.ldm; i += kFusedThreads) {
    float v = 0.f;
    if (i < p.m) v = io.y_ref ? io.y[i * p.B + b] : io.y[b * io.y_ld + i];
    ys[i] = (double)v;
    rs[i] = -(double)v;
  }
  for (int64_t q = tid; q < p.mwords; q += kFusedThreads) mask[q] = 0u;
  if (tid < kWarpCap) s_c[tid] = s_b[tid] = s_m1[tid] = s_m2[tid] = s_best[tid] = 0.0;
  __syncthreads();
  if (warp == 0) {
    double yy = 0.0;  // k_init's summation order: lanes stride the row, then the butterfly
    for (int64_t i = lane; i < p.ldm; i += 32) yy = fma(ys[i], ys[i], yy);
    yy = warp_sum(yy);
    if (lane == 0) red[0] = yy;
  }
  __syncthreads();
  if (tid == 0) {
    const double L = red[0];
    ctl.best_L = CUDART_INF;
    ctl.prev_L = CUDART_INF;
    ctl.loss = L;
    ctl.t = ctl.t0 = ctl.stall = ctl.iters = ctl.status = ctl.conv = ctl.best_cnt = ctl.changed = 0;
    ctl.active = 1;
    if (sqrt(L) < p.eps) {  // the outer-1 eps test (clomp.cpp:238-242)
      ctl.active = 0;
      ctl.conv = 1;
    }
  }
  const float* At = w.at32;
  if (STAGED) {
    // coalesced float4 reads of the atom-major dictionary (eight in flight per
    // thread), scattered to the measurement-major copy
    const int64_t n4 = p.n * p.ldm / 4, l4 = p.ldm / 4;
    for (int64_t e0 = tid; e0 < n4; e0 += 8 * kFusedThreads) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t e = e0 + u * kFusedThreads;
        if (e < n4) v[u] = reinterpret_cast<const float4*>(w.at32)[e];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t e = e0 + u * kFusedThreads;
        if (e < n4) {
          const int64_t j = e / l4, i = 4 * (e % l4);
          if (i < p.m) As[i * lda + j] = v[u].x;
          if (i + 1 < p.m) As[(i + 1) * lda + j] = v[u].y;
          if (i + 2 < p.m) As[(i + 2) * lda + j] = v[u].z;
          if (i + 3 < p.m) As[(i + 3) * lda + j] = v[u].w;
        }
      }
    }
  }
  __syncthreads();
  double* sc = sc_smem ? sc_s : w.scores + b * p.n;
  const int cap = (int)p.cap;  // <= kWarpCap on this path
  for (int outer = 1; outer <= p.max_outer && ctl.active; ++outer) {
    // K1: exact fp64 scores |a_j . r|, kFusedAtoms atoms per warp pass (config
    // 1's 256 atoms take one pass of the 8 warps).  Each score's summation
    // order does not depend on the pass width.
    double cmax = 0.0;
    FT_MARK(0);
    if (STAGED) {
      // K1: exact fp64 scores |a_j . r|, one thread per atom
      for (int64_t j = tid; j < p.n; j += kFusedThreads) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        const float* col = As + j;
        int64_t i = 0;
#pragma unroll 4
        for (; i + 4 <= p.m; i += 4) {  // r as two 16-byte broadcasts per four rows
          const double2 r01 = *reinterpret_cast<const double2*>(rs + i);
          const double2 r23 = *reinterpret_cast<const double2*>(rs + i + 2);
          a0 = fma(f2d(col[i * lda]), r01.x, a0);
          a1 = fma(f2d(col[(i + 1) * lda]), r01.y, a1);
          a2 = fma(f2d(col[(i + 2) * lda]), r23.x, a2);
          a3 = fma(f2d(col[(i + 3) * lda]), r23.y, a3);
        }
        for (; i < p.m; ++i) a0 = fma(f2d(col[i * lda]), rs[i], a0);
        const double v = fabs((a0 + a1) + (a2 + a3));
        sc[j] = v;
        cmax = fmax(cmax, v);
      }
      cmax = warp_max(cmax);
    } else {
    // K1: exact fp64 scores |a_j . r|, kFusedAtoms atoms per warp pass.  Each
    // score's summation order does not depend on the pass width.
    for (int64_t j0 = warp * kFusedAtoms; j0 < p.n; j0 += nw * kFusedAtoms) {
      double acc[kFusedAtoms];
#pragma unroll
      for (int u = 0; u < kFusedAtoms; ++u) acc[u] = 0.0;
      for (int64_t i = 2 * lane; i < p.ldm; i += 64) {
        const double2 r01 = *reinterpret_cast<const double2*>(rs + i);
#pragma unroll
        for (int u = 0; u < kFusedAtoms; ++u) {
          if (j0 + u < p.n) {
            const float2 a = *reinterpret_cast<const float2*>(At + (j0 + u) * p.ldm + i);
            acc[u] = fma(f2d(a.x), r01.x, acc[u]);
            acc[u] = fma(f2d(a.y), r01.y, acc[u]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kFusedAtoms; ++u) {
        const double v = fabs(warp_sum(acc[u]));
        if (j0 + u < p.n) {
          if (lane == 0) sc[j0 + u] = v;
          cmax = fmax(cmax, v);
        }
      }
    }
    }
    if (lane == 0) red[warp] = cmax;
    __syncthreads();
    FT_MARK(1);
    // K1c: inject_from_scores (clomp.cpp:41-53), ties included, ascending j.
    // Every warp marks its atoms (one ballot word per 32 atoms); warp 0 then
    // places the picks by a prefix over the words.
    double m = 0.0;
    for (int q = 0; q < nw; ++q) m = fmax(m, red[q]);
    {
      const double cut = p.th * m;
      for (int64_t j0 = (int64_t)warp * 32; j0 < p.n; j0 += kFusedThreads) {
        const int64_t j = j0 + lane;
        const bool pick = m > 0.0 && j < p.n && sc[j] >= cut && !((mask[j >> 5] >> (j & 31)) & 1u);
        const unsigned bal = __ballot_sync(kFull, pick);
        if (lane == 0) pickw[j0 >> 5] = bal;
      }
    }
    __syncthreads();
    if (warp == 0) {
      int t = ctl.t;
      const int t0 = ctl.t0;
      int added = 0, overflow = 0;
      for (int64_t w0 = 0; w0 < p.mwords; w0 += 32) {
        const int64_t wi = w0 + lane;
        unsigned bits = wi < p.mwords ? pickw[wi] : 0u;
        const int cntw = __popc(bits);
        int pre = cntw;  // inclusive prefix over the 32 words
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(kFull, pre, o);
          if (lane >= o) pre += v;
        }
        const int tot = __shfl_sync(kFull, pre, 31);
        int pos = t + pre - cntw;
        if (bits) mask[wi] |= bits;
        while (bits) {
          const int bit = __ffs(bits) - 1;
          bits &= bits - 1;
          CL_CHECK(pos >= 0 && wi * 32 + bit < p.n);
          if (pos < cap) sups[pos] = (int32_t)(wi * 32 + bit);
          ++pos;
        }
        t += tot;
        added += tot;
        if (t > cap) overflow = 1;
      }
      __syncwarp();
      FT_MARK(2);
      if (overflow) {  // larger supports use the batched path
        if (lane == 0) {
          ctl.status = kStatusCapacity;
          ctl.active = 0;
          ctl.t = cap;
          ctl.changed = added > 0;
        }
      } else {
        // Gram row / column and b_k = a_k . y of the atoms added this iteration
        // (new atoms start at c = 0, clomp.hpp:53-54)
        for (int k = t0; k < t; ++k) {
          const int64_t jk = sups[k];
          double gk = 0.0;
          if (w.gfull) {
            if (lane <= k) gk = w.gfull[jk * p.n + sups[lane]];
          } else {
            for (int i = 0; i <= k; ++i) {  // fp64 dot of the fp32 atoms, lanes over m
              double acc = 0.0;
              if (STAGED) {
                for (int64_t q = lane; q < p.m; q += 32)
                  acc = fma(f2d(As[q * lda + jk]), f2d(As[q * lda + sups[i]]), acc);
              } else {
                const float* ai = At + (int64_t)sups[i] * p.ldm;
                const float* ak = At + jk * p.ldm;
                for (int64_t q = lane; q < p.ldm; q += 32) acc = fma(f2d(ak[q]), f2d(ai[q]), acc);
              }
              acc = warp_sum(acc);
              if (lane == i) gk = acc;
            }
          }
          if (lane <= k) {
            Gs[k * LDS + lane] = gk;
            Gs[lane * LDS + k] = gk;
          }
          double accb = 0.0;
          if (STAGED) {  // the same element order as the atom-major float4 walk
            for (int64_t i0 = 4 * lane; i0 < p.m; i0 += 128)
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (i0 + e < p.m) accb = fma(f2d(As[(i0 + e) * lda + jk]), ys[i0 + e], accb);
          } else {
            const float* ak = At + jk * p.ldm;
#pragma unroll 4
            for (int64_t i0 = 4 * lane; i0 < p.ldm; i0 += 128) {
              const float4 a = *reinterpret_cast<const float4*>(ak + i0);
              accb = fma(f2d(a.x), ys[i0], accb);
              accb = fma(f2d(a.y), ys[i0 + 1], accb);
              accb = fma(f2d(a.z), ys[i0 + 2], accb);
              accb = fma(f2d(a.w), ys[i0 + 3], accb);
            }
          }
          accb = warp_sum(accb);
          if (lane == k) {
            s_b[k] = accb;
            s_c[k] = s_m1[k] = s_m2[k] = 0.0;
          }
        }
        __syncwarp();
        FT_MARK(3);
        // K2: all epochs; learn_epochs squares in place, so it works on a copy
        for (int e = lane; e < t * LDS; e += 32) sq[e] = Gs[e];
        __syncwarp();
        double m1 = lane < t ? s_m1[lane] : 0.0, m2 = lane < t ? s_m2[lane] : 0.0;
        const double c = learn_epochs<kWarpCap, OPT>(p, w, b, outer, cs, sq, lane, t,
                                                      lane < t ? s_c[lane] : 0.0,
                                                      lane < t ? s_b[lane] : 0.0, m1, m2);
        if (lane < t) {
          s_c[lane] = c;
          s_m1[lane] = m1;
          s_m2[lane] = m2;
        }
        if (lane == 0) {
          ctl.t = t;
          ctl.t0 = t;
          ctl.changed = added > 0;
        }
      }
    }
    FT_MARK(4);
    __syncthreads();
    if (!ctl.active) break;
    // residual r = A_S c - y (fp64) and the stopping rules
    const int t = ctl.t;
    double lacc = 0.0;
    for (int64_t i = tid; i < p.ldm; i += kFusedThreads) {
      double acc = 0.0;
      if (STAGED) {
        if (i < p.m)
          for (int k = 0; k < t; ++k) acc = fma((double)As[i * lda + sups[k]], s_c[k], acc);
      } else {
        for (int k = 0; k < t; ++k) acc = fma((double)At[(int64_t)sups[k] * p.ldm + i], s_c[k], acc);
      }
      const double rv = acc - ys[i];
      rs[i] = rv;
      lacc = fma(rv, rv, lacc);
    }
    lacc = warp_sum(lacc);
    if (lane == 0) red[warp] = lacc;
    __syncthreads();
    FT_MARK(5);
    if (warp == 0) {
      // clomp.cpp:253-273 on the on-chip state (control_signal's rules)
      double L = 0.0;
      for (int q = 0; q < nw; ++q) L += red[q];
      int snap = 0;
      if (lane == 0) {
        ctl.loss = L;
        if (!isfinite(L)) {
          ctl.status = kStatusNumerical;
          ctl.active = 0;
        } else {
          ctl.iters = outer;
          if (L < ctl.best_L) {
            ctl.best_L = L;
            ctl.best_cnt = t;
            snap = 1;
          }
          const double prev = ctl.prev_L;
          const double rel = isfinite(prev) ? (prev - L) / fmax(fabs(prev), 1e-300) : CUDART_INF;
          const int stall = (!ctl.changed && rel < p.stall_tol) ? ctl.stall + 1 : 0;
          ctl.stall = stall;
          ctl.prev_L = L;
          if (stall >= p.stall_patience || outer >= p.max_outer) {
            ctl.active = 0;
          } else if (sqrt(L) < p.eps) {
            ctl.conv = 1;
            ctl.active = 0;
          }
        }
      }
      snap = __shfl_sync(kFull, snap, 0);
      if (snap && lane < t) s_best[lane] = s_c[lane];
    }
    FT_MARK(6);
    __syncthreads();
    if (!ctl.active) break;
  }
  // k_finalize: the best snapshot unless converged (clomp.cpp:276-288), the
  // support in ascending atom order, final norm and flags
  __syncthreads();
  if (warp == 0) {
    const bool bad = ctl.status == kStatusNumerical;
    const bool use_best = !ctl.conv && isfinite(ctl.best_L);
    int t = bad ? 0 : (use_best ? ctl.best_cnt : ctl.t);
    if (ctl.status == kStatusCapacity) t = ctl.t < cap ? ctl.t : cap;
    const double* cv = use_best ? s_best : s_c;
    if (lane < t) {
      const int32_t jk = sups[lane];
      int rank = 0;
      for (int q = 0; q < t; ++q) rank += sups[q] < jk;
      CL_CHECK(rank < t && jk >= 0 && jk < p.n);
      if (rank < io.out_cap) {
        if (io.sup) io.sup[b * io.out_cap + rank] = jk;
        if (io.coef) io.coef[b * io.out_cap + rank] = cv[lane];
      }
    }
    if (lane == 0) {
      const double rn = use_best ? sqrt(ctl.best_L) : sqrt(ctl.loss);
      if (io.cnt) io.cnt[b] = t < io.out_cap ? t : (int)io.out_cap;
      if (io.iters) io.iters[b] = ctl.iters;
      if (io.rn) io.rn[b] = bad ? CUDART_NAN : rn;
      if (io.conv) io.conv[b] = (!bad && rn < p.eps) ? 1 : 0;
      if (io.status) io.status[b] = ctl.status;
    }
  }
}

// ------------------------------------------------------ separable mode
// Loss of the separable residual (tile partials in fixed order) and the
// per-signal stopping rules; the snapshot copies the learned coefficients.
__global__ void k_sep_control(SolveParams p, Work w, int outer, int64_t tiles) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= p.B || !w.active[b]) return;
  double L = 0.0;
  for (int64_t t = 0; t < tiles; ++t) L += w.lpart[b * tiles + t];
  if (p.mode == kModePerSignal) {
    if (control_signal(p, w, b, outer, L)) {
      const int t = w.cnt[b];
      for (int k = 0; k < t; ++k) w.best_coef[b * p.cap + k] = w.coef[b * p.cap + k];
    }
  } else {
    w.loss[b] = L;
  }
}

// ------------------------------------------------------ joint control
// clomp_solve_batch semantics (clomp.cpp:235-273): batch-global totals in a
// fixed reduction order (deterministic), one decision for every signal.
__global__ void __launch_bounds__(1024)
k_joint_control(SolveParams p, Work w, int outer, int init) {
  __shared__ double red[1024];
  // Once the batch has stopped, later (graph-replayed) iterations are no-ops.
  if (!init && w.joint[kJStop] != 0.0) {
    if (threadIdx.x == 0) {
      w.joint[kJImproved] = 0.0;
      w.counters[active_slot(outer)] = 0;
    }
    return;
  }
  __shared__ int chg[32];
  const int tid = threadIdx.x;
  double s = 0.0;
  int any = 0, full = 0;
  for (int64_t b = tid; b < p.B; b += blockDim.x) {
    s += w.loss[b];
    any |= w.changed[b];
    // a signal whose support outgrew the per-signal capacity stopped learning
    // (pick_finish / warp_threshold_append): the batch cannot continue with
    // the reference's semantics, so it stops with the capacity status
    if (!init) full |= w.status[b] == kStatusCapacity;
  }
  red[tid] = s;
  any = __any_sync(kFull, any);
  full = __syncthreads_or(full);
  if ((tid & 31) == 0) chg[tid >> 5] = any;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  __shared__ int stop_s;
  if (tid == 0) {
    // image mode: the stopping rules read lb.total (residual + priors), the
    // eps test and the final norm the residual part (clomp.cpp:238-242, 253-288)
    const double total_r = red[0];
    const double total = (p.prior == 2 && !init) ? total_r + w.joint[kJPrior] : total_r;
    int changed = 0;
    for (int q = 0; q < (int)(blockDim.x / 32); ++q) changed |= chg[q];
    double* J = w.joint;
    int stop = 0;
    J[kJImproved] = 0.0;
    if (init) {
      J[kJBest] = CUDART_INF;
      J[kJPrev] = CUDART_INF;
      J[kJStall] = 0.0;
      J[kJStatus] = 0.0;
      J[kJIters] = 0.0;
      J[kJConv] = 0.0;
      J[kJTotal] = total;
      J[kJTotalR] = total_r;
      J[kJBestR] = CUDART_INF;
      J[kJPrior] = 0.0;
      if (sqrt(total_r) < p.eps) {
        J[kJConv] = 1.0;
        stop = 1;
      }
    } else {
      J[kJTotal] = total;
      J[kJTotalR] = total_r;
      if (full) {
        J[kJStatus] = (double)kStatusCapacity;
        stop = 1;
      } else if (!isfinite(total)) {
        J[kJStatus] = (double)kStatusNumerical;
        stop = 1;
      } else {
        J[kJIters] = (double)outer;
        if (total < J[kJBest]) {
          J[kJBest] = total;
          J[kJBestR] = total_r;
          J[kJImproved] = 1.0;
        }
        const double prev = J[kJPrev];
        const double rel = isfinite(prev)
                               ? (prev - total) / fmax(fabs(prev), 1e-300)
                               : CUDART_INF;
        const double st = (!changed && rel < p.stall_tol) ? J[kJStall] + 1.0 : 0.0;
        J[kJStall] = st;
        J[kJPrev] = total;
        if (st >= (double)p.stall_patience || outer >= p.max_outer) {
          stop = 1;
        } else if (sqrt(total_r) < p.eps) {
          J[kJConv] = 1.0;
          stop = 1;
        }
      }
    }
    J[kJStop] = stop;
    w.counters[active_slot(outer)] = stop ? 0 : (int)p.B;
    stop_s = stop;
  }
  __syncthreads();
  if (stop_s)
    for (int64_t b = tid; b < p.B; b += blockDim.x) w.active[b] = 0;
}

__global__ void k_joint_snapshot(SolveParams p, Work w) {
  const int lane = threadIdx.x & 31;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= p.B || w.joint[kJImproved] == 0.0) return;
  const int t = w.cnt[b];
  for (int i = lane; i < t; i += 32) w.best_coef[b * p.cap + i] = w.coef[b * p.cap + i];
  if (lane == 0) w.best_cnt[b] = t;
}

// ------------------------------------------------------------ finalize
// Result selection (clomp.cpp:276-288) and compaction: support sorted by atom
// index with its coefficients.
__global__ void k_finalize(SolveParams p, Work w, int64_t out_cap,
                           int32_t* sup_out, double* coef_out, int32_t* cnt_out,
                           int32_t* iters_out, double* rn_out,
                           uint8_t* conv_out, int32_t* status_out) {
  const int lane = threadIdx.x & 31;
  const int64_t b = p.sig_lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (b >= p.sig_hi) return;
  const int64_t cap = p.cap;
  int status, iters, use_best;
  double rn;
  if (p.mode == kModeJoint) {
    const double* J = w.joint;
    status = (int)J[kJStatus];
    iters = (int)J[kJIters];
    const bool conv = J[kJConv] != 0.0;
    use_best = !conv && isfinite(J[kJBest]);
    if (p.prior == 2)
      rn = use_best ? sqrt(J[kJBestR]) : sqrt(J[kJTotalR]);
    else
      rn = use_best ? sqrt(J[kJBest]) : sqrt(J[kJTotal]);
  } else {
    status = w.status[b];
    iters = w.iters[b];
    use_best = !w.conv[b] && isfinite(w.best_L[b]);
    if (p.prior)  // the losses carry the prior: the residual parts are kept apart
      rn = use_best ? sqrt(w.best_R[b]) : sqrt(w.rloss[b]);
    else
      rn = use_best ? sqrt(w.best_L[b]) : sqrt(w.loss[b]);
  }
  const bool bad = status == kStatusNumerical;
  int t = bad ? 0 : (use_best ? w.best_cnt[b] : w.cnt[b]);
  if (status == kStatusCapacity) t = w.cnt[b] < cap ? w.cnt[b] : (int)cap;
  const double* cv = (use_best ? w.best_coef : w.coef) + b * cap;
  const int32_t* sv = w.sup + b * cap;  // the support only ever grows
  for (int k = lane; k < t; k += 32) {
    const int32_t jk = sv[k];
    int rank = 0;
    for (int q = 0; q < t; ++q) rank += sv[q] < jk;
    CL_CHECK(jk >= 0 && jk < p.n && rank < t && t <= cap);
    if (rank < out_cap) {
      if (sup_out) sup_out[b * out_cap + rank] = jk;
      if (coef_out) coef_out[b * out_cap + rank] = cv[k];
    }
  }
  if (lane == 0) {
    if (cnt_out) cnt_out[b] = t < out_cap ? t : (int)out_cap;
    if (iters_out) iters_out[b] = iters;
    if (rn_out) rn_out[b] = bad ? CUDART_NAN : rn;
    if (conv_out) conv_out[b] = (!bad && rn < p.eps) ? 1 : 0;
    if (status_out) status_out[b] = status;
  }
}

// fp16 split of residual rows already in r64 (warp per signal).
__global__ void k_split_resid(SolveParams p, Work w) {
  const int lane = threadIdx.x & 31;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= p.B) return;
  double acc = 0.0;
  for (int64_t i = lane; i < p.ldm; i += 32) {
    const double v = w.r64[b * p.ldm + i];
    acc = fma(v, v, acc);
  }
  split_row(w, b, p.ldm, warp_sum(acc), lane, 32);
}

// inject_support unit path: ||r||^2 per column and a clean support list.
__global__ void k_inject_prep(SolveParams p, Work w) {
  const int lane = threadIdx.x & 31;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= p.B) return;
  double acc = 0.0;
  for (int64_t i = lane; i < p.ldm; i += 32) {
    const double v = w.r64[b * p.ldm + i];
    acc = fma(v, v, acc);
  }
  acc = warp_sum(acc);
  if (w.r_hi) split_row(w, b, p.ldm, acc, lane, 32);
  if (lane == 0) {
    w.loss[b] = acc;
    w.cnt[b] = 0;
    w.active[b] = 1;
    w.status[b] = 0;
  }
}

}  // namespace

void launch_init(const SolveParams& p, const Work& w, const float* y_in,
                 int y_layout, bool, cudaStream_t s) {
  const int threads = 256;
  const int64_t blocks = (p.B * 32 + threads - 1) / threads;
  int64_t in_ld = p.m;
  if (y_layout == 0 && p.B > 1) {  // reference m x B: tiled transpose into y32 first
    const dim3 tg((unsigned)((p.B + 31) / 32), (unsigned)((p.m + 31) / 32));
    k_transpose_y<<<tg, dim3(32, 8), 0, s>>>(y_in, p.m, p.B, w.y32, p.ldm);
    y_in = w.y32;
    in_ld = p.ldm;
  }
  k_init<<<(unsigned)blocks, threads, 0, s>>>(p, w, y_in, in_ld);
}

void launch_split_resid(const SolveParams& p, const Work& w, cudaStream_t s) {
  k_split_resid<<<(unsigned)((p.B * 32 + 255) / 256), 256, 0, s>>>(p, w);
}

void launch_select(const SolveParams& p, const Work& w, bool full_scores,
                   cudaStream_t s) {
  const int64_t nsig = p.sig_hi - p.sig_lo;
  if (full_scores) {
    const int64_t blocks = (nsig * 32 + 255) / 256;
    k_select_thresh<<<(unsigned)blocks, 256, 0, s>>>(p, w);
  } else {
    const int64_t blocks = (nsig * 32 + 255) / 256;
    k_select_top<<<(unsigned)blocks, 256, 0, s>>>(p, w);
  }
}

static size_t block_smem_bytes(int64_t cap, bool smem_g) {
  size_t bytes = (size_t)cap * 8 + (size_t)((cap + 1) & ~1LL) * 4;
  if (smem_g) bytes += (size_t)cap * cap * 8;
  return bytes;
}

template <int OPT>
static void launch_block_variant(const SolveParams& p, const Work& w, int outer,
                                 int32_t* big_list, int grid, int skip_le, cudaStream_t s) {
  const size_t smem_g = block_smem_bytes(p.cap, true);
  if (smem_g <= 200 * 1024) {
    cudaFuncSetAttribute(k_learn_block<OPT, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_g);
    launch_pdl(k_learn_block<OPT, true>, dim3(grid), dim3(kBlockThreads), smem_g, s, p, w,
               outer, (const int32_t*)big_list, skip_le);
  } else {
    const size_t sm = block_smem_bytes(p.cap, false);
    cudaFuncSetAttribute(k_learn_block<OPT, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_pdl(k_learn_block<OPT, false>, dim3(grid), dim3(kBlockThreads), sm, s, p, w, outer,
               (const int32_t*)big_list, skip_le);
  }
}

template <int Q, int CW, int NWC, int RW>
static void launch_cluster_q(const SolveParams& p, const Work& w, int outer, int32_t* big_list,
                             int nclusters, cudaStream_t s, int ph = 0) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(Q, (unsigned)nclusters);
  cfg.blockDim = dim3(32 * NWC);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
  // explicit cluster launch even for Q = 1: st.async / mapa need one
  at[na].id = cudaLaunchAttributeClusterDimension;
  at[na].val.clusterDim.x = Q;
  at[na].val.clusterDim.y = 1;
  at[na].val.clusterDim.z = 1;
  ++na;
  cfg.attrs = at;
  cfg.numAttrs = na;
  if (Q > 1) {
    // Clusters must fit inside a GPC: not every SM can host one.  A grid of
    // more clusters than can be co-resident runs its last clusters in a second
    // wave (each cluster loops over signals), so cap it at the occupancy.
    static DevSlots active_cache;
    const int dev = current_device();
    int max_active = (int)active_cache.get(dev);
    if (max_active == 0) {
      int nmax = 0;
      if (cudaOccupancyMaxActiveClusters(&nmax, k_learn_cluster<Q, CW, NWC, RW, 0>, &cfg) !=
              cudaSuccess ||
          nmax <= 0) {
        cudaGetLastError();
        nmax = -1;
      }
      max_active = nmax;
      active_cache.set(dev, nmax);
    }
    if (max_active > 0 && nclusters > max_active) {
      nclusters = max_active;
      cfg.gridDim = dim3(Q, (unsigned)nclusters);
    }
  }
  const int32_t* bl = big_list;
  if (ph == 1) {
    cudaLaunchKernelEx(&cfg, k_learn_cluster<Q, CW, NWC, RW, 0, 1>, p, w, outer, bl);
    return;
  }
  if (ph == 2) {
    cudaLaunchKernelEx(&cfg, k_learn_cluster<Q, CW, NWC, RW, 0, 2>, p, w, outer, bl);
    return;
  }
  switch (p.opt) {
    case 0: cudaLaunchKernelEx(&cfg, k_learn_cluster<Q, CW, NWC, RW, 0>, p, w, outer, bl); break;
    case 1: cudaLaunchKernelEx(&cfg, k_learn_cluster<Q, CW, NWC, RW, 1>, p, w, outer, bl); break;
    default: cudaLaunchKernelEx(&cfg, k_learn_cluster<Q, CW, NWC, RW, 2>, p, w, outer, bl); break;
  }
}

// Cluster learning for supports of 33..256 atoms: returns the support size
// up to which it learns this iteration (0 when not launched).  One CTA per
// signal up to 128 atoms (64: 8 warps x 2 columns per lane; 128: 16 warps x 4),
// four-CTA clusters up to 256.  With the power form (plain GD, p.pw_levels >
// 0) the variant runs twice around the batched squarings (PH 1 / PH 2); *extra
// counts the additional launches.
static int launch_cluster_learn(const SolveParams& p, const Work& w, int outer, int max_cnt,
                                int64_t nsig, int sms, cudaStream_t s, int* extra) {
  if (p.sep || max_cnt <= kWarpCap || p.cluster_learn == 0) return 0;
  auto nc = [&](int q) { return (int)std::max<int64_t>(1, std::min<int64_t>(nsig, sms / q)); };
  const bool pw = p.pw_levels > 0 && p.opt == 0;
  auto run = [&](auto launch, int tmax) {
    if (!pw) {
      launch(0);
      return;
    }
    const int64_t nbig = std::min<int64_t>(nsig, p.pw_slots);
    launch_pdl(k_pw_extend, dim3((unsigned)std::max<int64_t>(1, nbig)), dim3(kPwExtThreads), 0, s, p, w, outer,
               (const int32_t*)w.big_list, tmax);
    const bool ph1 = p.pw_r > 0 || nsig > p.pw_slots;  // leftover epochs / signals
    if (ph1) launch(1);
    const int nt = (tmax + kPwTile - 1) / kPwTile;
    const int sig_grid = (int)std::min<int64_t>(std::min<int64_t>(nsig, p.pw_slots),
                                                (int64_t)sms * 16);
    cudaFuncSetAttribute(k_pow_sq, cudaFuncAttributeMaxDynamicSharedMemorySize, kPwSmem);
    for (int l = 0; l < p.pw_levels; ++l)
      launch_pdl(k_pow_sq, dim3((unsigned)(nt * (nt + 1) / 2), (unsigned)std::max(sig_grid, 1)),
                 dim3(kPwThreads), kPwSmem, s, p, w, outer, (const int32_t*)w.big_list, l, tmax, nt);
    launch(2);
    const int nchunk = (int)((p.ldm + kPwResRows - 1) / kPwResRows);
    launch_pdl(k_pw_resid, dim3((unsigned)nchunk, (unsigned)std::max<int64_t>(1, nbig)),
               dim3(kPwResThreads), 0, s, p, w, outer, (const int32_t*)w.big_list, tmax);
    *extra += 2 + (ph1 ? 1 : 0) + p.pw_levels;
  };
  if (max_cnt <= 64) {
    run([&](int ph) {
      launch_cluster_q<1, 2, 8, 8>(p, w, outer, w.big_list,
                                   (int)std::min<int64_t>(nsig, 2 * (int64_t)sms), s, ph);
    }, 64);
    return 64;
  }
  if (max_cnt <= 128) {
    run([&](int ph) { launch_cluster_q<1, 4, 16, 8>(p, w, outer, w.big_list, nc(1), s, ph); },
        128);
    return 128;
  }
  run([&](int ph) { launch_cluster_q<4, 8, 8, 8>(p, w, outer, w.big_list, nc(4), s, ph); }, 256);
  return 256;
}

int launch_learn(const SolveParams& p, const Work& w, int outer, int max_cnt,
                 cudaStream_t s) {
  int extra = 0;  // launches beyond learn (+ residual) + cluster + block
  int32_t* big_list = w.big_list;
  // max_cnt: upper bound on the support size after this iteration's select
  // (ties can exceed it; those signals fall through to the block kernel).
  const int64_t nsig = p.sig_hi - p.sig_lo;
  auto blocks_for = [&](int nw) { return (unsigned)((nsig + nw - 1) / nw); };
  auto learn = [&](auto tb) {
    constexpr int TB = decltype(tb)::value;
    constexpr int NW = learn_warps<TB>();
    const dim3 lg(blocks_for(NW)), lb(32 * NW);
    const bool fast = p.fuse_select && w.gfull && !p.sep && p.cap >= 32 && (p.cap & 1) == 0;
    // one 512-row pass with the tcgen05 correlation next (it reads the fp16
    // split; the GEMV and fp64 correlations read the fp64 row itself): fp16
    // split from registers, fp64 row on demand
    if (fast && p.ldm <= 512 && w.r_hi != nullptr) {
      switch (p.opt) {
        case 0: launch_pdl(k_learn_fast<TB, 0, true>, lg, lb, 0, s, p, w, outer, big_list); break;
        case 1: launch_pdl(k_learn_fast<TB, 1, true>, lg, lb, 0, s, p, w, outer, big_list); break;
        default: launch_pdl(k_learn_fast<TB, 2, true>, lg, lb, 0, s, p, w, outer, big_list); break;
      }
    } else if (fast) {
      switch (p.opt) {
        case 0: launch_pdl(k_learn_fast<TB, 0, false>, lg, lb, 0, s, p, w, outer, big_list); break;
        case 1: launch_pdl(k_learn_fast<TB, 1, false>, lg, lb, 0, s, p, w, outer, big_list); break;
        default: launch_pdl(k_learn_fast<TB, 2, false>, lg, lb, 0, s, p, w, outer, big_list); break;
      }
    } else {
      switch (p.opt) {
        case 0: launch_pdl(k_learn_warp<TB, 0>, lg, lb, 0, s, p, w, outer, big_list); break;
        case 1: launch_pdl(k_learn_warp<TB, 1>, lg, lb, 0, s, p, w, outer, big_list); break;
        default: launch_pdl(k_learn_warp<TB, 2>, lg, lb, 0, s, p, w, outer, big_list); break;
      }
    }
    if (!p.sep && !fast)  // the fast kernel finishes its signals' residuals itself
      launch_pdl(k_resid_w<TB>, dim3((unsigned)((nsig + 3) / 4)), dim3(128), 0, s, p, w, outer);
  };
  if (max_cnt <= 8)
    learn(std::integral_constant<int, 8>());
  else if (max_cnt <= 16)
    learn(std::integral_constant<int, 16>());
  else
    learn(std::integral_constant<int, 32>());
  if (p.cap > 8) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
#ifndef CL_BLOCK_GRID_DIV
#define CL_BLOCK_GRID_DIV 1
#endif
    const int gmax = std::max(1, 2 * sms / CL_BLOCK_GRID_DIV);
    const int grid = (int)(nsig < gmax ? nsig : gmax);
    const int skip_le = launch_cluster_learn(p, w, outer, max_cnt, nsig, sms, s, &extra);
    switch (p.opt) {
      case 0: launch_block_variant<0>(p, w, outer, big_list, grid, skip_le, s); break;
      case 1: launch_block_variant<1>(p, w, outer, big_list, grid, skip_le, s); break;
      default: launch_block_variant<2>(p, w, outer, big_list, grid, skip_le, s); break;
    }
  }
  return extra;
}

int learn_trace(unsigned long long* out, int max_signals) {
#ifdef CL_LEARN_TRACE
  const int n = max_signals < 8192 ? max_signals : 8192;
  cudaMemcpyFromSymbol(out, g_lt, (size_t)n * 8 * sizeof(unsigned long long));
  return n;
#else
  (void)out;
  (void)max_signals;
  return 0;
#endif
}

int cluster_trace(unsigned long long* out) {
#ifdef CL_CLUSTER_TRACE
  cudaMemcpyFromSymbol(out, g_cl_trace, 8 * sizeof(unsigned long long));
  return 1;
#else
  (void)out;
  return 0;
#endif
}

void launch_prior_ext(const SolveParams& p, const Work& w, cudaStream_t s) {
  const int64_t nsig = p.sig_hi - p.sig_lo;
  const unsigned grid = (unsigned)std::min<int64_t>(nsig, 4096);
  launch_pdl(k_prior_ext, dim3(grid), dim3(kPriorThreads), 0, s, p, w);
}

void launch_prior_control(const SolveParams& p, const Work& w, int outer, cudaStream_t s) {
  const int64_t nsig = p.sig_hi - p.sig_lo;
  launch_pdl(k_prior_control, dim3((unsigned)((nsig + 3) / 4)), dim3(128), 0, s, p, w, outer);
}

void launch_image_learn(const SolveParams& p, const Work& w, int outer, cudaStream_t s) {
  const unsigned cgrid = (unsigned)std::min<int64_t>(p.B, 2048);
  const size_t smem = (size_t)p.cap * 12 + 16;
  static DevSlots smem_set;
  ensure_smem_limit(smem_set, k_img_synth, smem);
  const int64_t npix = p.n * p.B;
  const unsigned pgrid = (unsigned)((npix + 255) / 256);
  const int64_t nwin = (int64_t)p.lv_nr * p.lv_nc;
  for (int e = 0; e < p.inner; ++e) {
    launch_pdl(k_img_synth, dim3(cgrid), dim3(kImgThreads), smem, s, p, w, 1);
    if (p.lv_on)
      launch_pdl(k_img_lv, dim3((unsigned)((nwin + 127) / 128)), dim3(128), 0, s, p, w);
    launch_pdl(k_img_gx, dim3(pgrid), dim3(256), 0, s, p, w);
    switch (p.opt) {
      case 0: launch_pdl(k_img_step<0>, dim3(cgrid), dim3(kImgThreads), 0, s, p, w, outer, e); break;
      case 1: launch_pdl(k_img_step<1>, dim3(cgrid), dim3(kImgThreads), 0, s, p, w, outer, e); break;
      default: launch_pdl(k_img_step<2>, dim3(cgrid), dim3(kImgThreads), 0, s, p, w, outer, e); break;
    }
  }
  launch_pdl(k_img_resid, dim3((unsigned)((p.B + 3) / 4)), dim3(128), 0, s, p, w);
  launch_pdl(k_img_synth, dim3(cgrid), dim3(kImgThreads), smem, s, p, w, 0);
  if (p.lv_on)
    launch_pdl(k_img_lv, dim3((unsigned)((nwin + 127) / 128)), dim3(128), 0, s, p, w);
  launch_pdl(k_img_loss, dim3(1), dim3(1024), 0, s, p, w);
}

void launch_joint_control(const SolveParams& p, const Work& w, int outer,
                          bool init, cudaStream_t s) {
  k_joint_control<<<1, 1024, 0, s>>>(p, w, outer, init ? 1 : 0);
}

void launch_joint_snapshot(const SolveParams& p, const Work& w,
                           cudaStream_t s) {
  const int64_t blocks = (p.B * 32 + 255) / 256;
  k_joint_snapshot<<<(unsigned)blocks, 256, 0, s>>>(p, w);
}

void launch_finalize(const SolveParams& p, const Work& w, int64_t out_cap,
                     int32_t* sup_out, double* coef_out, int32_t* cnt_out,
                     int32_t* iters_out, double* rn_out, uint8_t* conv_out,
                     int32_t* status_out, cudaStream_t s) {
  const int64_t blocks = ((p.sig_hi - p.sig_lo) * 32 + 255) / 256;
  k_finalize<<<(unsigned)blocks, 256, 0, s>>>(p, w, out_cap, sup_out, coef_out,
                                             cnt_out, iters_out, rn_out,
                                             conv_out, status_out);
}

void launch_sep_control(const SolveParams& p, const Work& w, int outer, cudaStream_t s) {
  const int64_t blocks = (p.B + 127) / 128;
  k_sep_control<<<(unsigned)blocks, 128, 0, s>>>(p, w, outer, sep_resid_tiles(p));
}

void launch_solve_fused(const SolveParams& p, const Work& w, const float* y_in, int y_ref,
                        int64_t out_cap, int32_t* sup_out, double* coef_out, int32_t* cnt_out,
                        int32_t* iters_out, double* rn_out, uint8_t* conv_out, int32_t* status_out,
                        cudaStream_t s) {
  FusedIo io{y_in, p.m, y_ref, out_cap, sup_out, coef_out, cnt_out, iters_out, rn_out, conv_out, status_out};
  // latency-bound path: the SM count and the smem attribute are queried / set
  // once per device (the attribute only grows), not per call
  static DevSlots smem_set[6];
  const int sms = device_sms(current_device());
  // dynamic shared memory: residual, y, the mask, then (when they fit) the
  // scores and the whole dictionary (measurement-major, m x (n + 1) floats); A
  // is staged only while every signal still gets its own SM
  const size_t base = (size_t)p.ldm * 16 + (size_t)((p.mwords + 3) & ~3LL) * 8;  // mask + picks
  const size_t sc_bytes = (size_t)p.n * 8;
  const size_t a_bytes = (size_t)(p.m * (p.n + 1)) * 4 + 16;
  const int sc_smem = base + sc_bytes <= (size_t)kFusedStageMax ? 1 : 0;
  const size_t with_sc = base + (sc_smem ? sc_bytes : 0);
  const bool stage_a = with_sc + a_bytes <= (size_t)kFusedStageMax && p.B <= sms;
  const size_t smem = with_sc + (stage_a ? a_bytes : 0);
  auto go = [&](auto kern, int slot) {
    // static shared memory (~21 KB) counts against the 48 KB default too: opt
    // in to the large carve-out as soon as the sum could pass it
    if (smem + 24 * 1024 > 48 * 1024) {
      const int dev = current_device();
      if ((long long)smem > smem_set[slot].get(dev)) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        smem_set[slot].set(dev, (long long)smem);
      }
    }
    kern<<<(unsigned)p.B, kFusedThreads, smem, s>>>(p, w, sc_smem, io);
  };
  const int o = p.opt < 0 ? 0 : (p.opt > 2 ? 2 : p.opt);
  if (stage_a) {
    switch (o) {
      case 0: go(k_solve_fused<0, true>, 0); break;
      case 1: go(k_solve_fused<1, true>, 1); break;
      default: go(k_solve_fused<2, true>, 2); break;
    }
  } else {
    switch (o) {
      case 0: go(k_solve_fused<0, false>, 3); break;
      case 1: go(k_solve_fused<1, false>, 4); break;
      default: go(k_solve_fused<2, false>, 5); break;
    }
  }
}

void launch_inject_finish(const SolveParams& p, const Work& w,
                          cudaStream_t s) {
  const int64_t blocks = (p.B * 32 + 255) / 256;
  k_inject_prep<<<(unsigned)blocks, 256, 0, s>>>(p, w);
}

}  // namespace clb
