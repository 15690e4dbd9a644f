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
#include <math_constants.h>

#include <cfloat>
#include <cmath>

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
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = x - hi;
}

__device__ __forceinline__ void store_residual(const Work& w, int64_t o,
                                               double rv) {
  w.r64[o] = rv;
  if (w.r_hi) {
    float hi, lo;
    split_tf32((float)rv, hi, lo);
    w.r_hi[o] = hi;
    w.r_lo[o] = lo;
  }
}

// ------------------------------------------------------------------ init
// One warp per signal: stage y, r = 0 - y = -y (clomp.cpp:236-237 at s = 0),
// ||y||^2, fresh state, and the outer-1 eps test in per-signal mode.
__global__ void k_init(SolveParams p, Work w, const float* __restrict__ y_in,
                       int layout_ref) {
  const int lane = threadIdx.x & 31;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= p.B) return;
  double acc = 0.0;
  for (int64_t i = lane; i < p.ldm; i += 32) {
    float v = 0.f;
    if (i < p.m) v = layout_ref ? y_in[i * p.B + b] : y_in[b * p.m + i];
    const int64_t o = b * p.ldm + i;
    w.y32[o] = v;
    w.y64[o] = (double)v;
    store_residual(w, o, -(double)v);
    acc = fma((double)v, (double)v, acc);
  }
  for (int64_t q = lane; q < p.mwords; q += 32) w.maskbits[b * p.mwords + q] = 0u;
  const double L = warp_sum(acc);
  if (lane == 0) {
    w.loss[b] = L;
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
// K1c for th == 1: merge the per-tile top-2 candidates, accept a clear winner,
// queue the signal for an fp64 rescan when the top-2 gap is inside the
// correlation error bound (or tied: all ties must be injected).
__global__ void k_select_top(SolveParams p, Work w) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= p.B || !w.active[b]) return;
  double v1 = -1.0, v2 = -1.0;
  int i1 = 0x7fffffff;
  const int64_t base = b * p.ntile;
  for (int64_t t = 0; t < p.ntile; ++t) {
    const double c1 = w.cand_v1[base + t], c2 = w.cand_v2[base + t];
    const int k1 = w.cand_i1[base + t];
    if (c1 > v1 || (c1 == v1 && k1 < i1)) {
      v2 = fmax(v1, c2);
      v1 = c1;
      i1 = k1;
    } else {
      v2 = fmax(v2, c1);
    }
  }
  w.changed[b] = 0;
  if (!(v1 > 0.0)) return;  // zero column: inject nothing (clomp.cpp:48)
  const double delta = p.delta_rel * p.colnorm_max * sqrt(w.loss[b]);
  if (v1 - v2 <= delta) {
    const int slot = atomicAdd(&w.counters[kRescanCount], 1);
    w.rescan_list[slot] = (int32_t)b;
    return;
  }
  uint32_t* mb = w.maskbits + b * p.mwords;
  if (mask_test(mb, i1)) return;  // argmax already selected: mask unchanged
  const int t = w.cnt[b];
  if (t >= p.cap) {
    w.status[b] = kStatusCapacity;
    w.active[b] = 0;
    return;
  }
  mb[i1 >> 5] |= 1u << (i1 & 31);
  w.sup[b * p.cap + t] = i1;
  w.cnt[b] = t + 1;
  w.changed[b] = 1;
  atomicMax(&w.counters[kMaxCount], t + 1);
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
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= p.B || !w.active[b]) return;
  const double* sc = w.scores + b * p.n;
  double cmax = 0.0;
  for (int64_t j = lane; j < p.n; j += 32) cmax = fmax(cmax, sc[j]);
  cmax = warp_max(cmax);
  if (lane == 0) w.changed[b] = 0;
  if (cmax == 0.0) return;
  const double cut = p.th * cmax;
  warp_threshold_append(p, w, b, cut, [&](int64_t j) { return sc[j]; }, lane);
}

// fp64 score of atom j against the fp64 residual of signal b (one warp).
__device__ __forceinline__ double warp_score64(const SolveParams& p,
                                               const Work& w, int64_t b,
                                               int64_t j, int lane) {
  const float* a = w.at32 + j * p.ldm;
  const double* r = w.r64 + b * p.ldm;
  double acc = 0.0;
  for (int64_t i = lane; i < p.ldm; i += 32) acc = fma((double)a[i], r[i], acc);
  return fabs(warp_sum(acc));
}

// Re-decide a near-tied selection from fp64 scores over all atoms: the exact
// inject_from_scores rule, including every tie.  One block per queued signal.
__global__ void __launch_bounds__(256) k_rescan(SolveParams p, Work w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  __shared__ double red[32];
  __shared__ double sc[32];
  __shared__ int s_t, s_added, s_over;
  const int count = w.counters[kRescanCount];
  for (int li = blockIdx.x; li < count; li += gridDim.x) {
    const int64_t b = w.rescan_list[li];
    double cmax = 0.0;
    for (int64_t j = warp; j < p.n; j += nw) {
      const double v = warp_score64(p, w, b, j, lane);
      cmax = fmax(cmax, v);
    }
    if (lane == 0) red[warp] = cmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = 0.0;
      for (int q = 0; q < nw; ++q) m = fmax(m, red[q]);
      red[0] = m;
      s_t = w.cnt[b];
      s_added = 0;
      s_over = 0;
    }
    __syncthreads();
    cmax = red[0];
    if (cmax > 0.0) {
      const double cut = p.th * cmax;
      uint32_t* mb = w.maskbits + b * p.mwords;
      for (int64_t j0 = 0; j0 < p.n; j0 += nw) {
        const int64_t j = j0 + warp;
        double v = -1.0;
        if (j < p.n) v = warp_score64(p, w, b, j, lane);
        if (lane == 0) sc[warp] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
          for (int q = 0; q < nw && j0 + q < p.n; ++q) {
            const int jj = (int)(j0 + q);
            if (sc[q] >= cut && !mask_test(mb, jj)) {
              if (s_t < p.cap) {
                w.sup[b * p.cap + s_t] = jj;
                mb[jj >> 5] |= 1u << (jj & 31);
                ++s_t;
                ++s_added;
              } else {
                s_over = 1;
              }
            }
          }
        }
        __syncthreads();
      }
    }
    if (threadIdx.x == 0) {
      w.cnt[b] = s_t;
      w.changed[b] = s_added > 0;
      if (s_over) {
        w.status[b] = kStatusCapacity;
        w.active[b] = 0;
      }
      if (s_added) atomicMax(&w.counters[kMaxCount], s_t);
      atomicAdd(&w.counters[kRescanTotal], 1);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------ stopping rules
// Per-signal bookkeeping after the learning phase of outer iteration `outer`
// (clomp.cpp:253-273), plus the eps test that opens the next iteration
// (clomp.cpp:238-242).  Returns true when the best snapshot must be taken.
__device__ bool control_signal(const SolveParams& p, const Work& w, int64_t b,
                               int outer, double L) {
  w.loss[b] = L;
  if (!isfinite(L)) {
    w.status[b] = kStatusNumerical;
    w.active[b] = 0;
    return false;
  }
  w.iters[b] = outer;
  bool snap = false;
  if (L < w.best_L[b]) {
    w.best_L[b] = L;
    w.best_cnt[b] = w.cnt[b];
    snap = true;
  }
  const double prev = w.prev_L[b];
  const double rel = isfinite(prev) ? (prev - L) / fmax(fabs(prev), 1e-300)
                                    : CUDART_INF;
  int stall = (!w.changed[b] && rel < p.stall_tol) ? w.stall[b] + 1 : 0;
  w.stall[b] = stall;
  w.prev_L[b] = L;
  if (stall >= p.stall_patience || outer >= p.max_outer) {
    w.active[b] = 0;
  } else if (sqrt(L) < p.eps) {
    w.conv[b] = 1;
    w.active[b] = 0;
  } else {
    atomicAdd(&w.counters[kActiveCount], 1);
  }
  return snap;
}

// ----------------------------------------------------- optimizer steps
template <int OPT>
__device__ __forceinline__ void opt_step(double& c, double g, double& m1,
                                         double& m2, double lr, double bc1,
                                         double bc2) {
  if (OPT == 0) {  // plain: s -= lr * g (clomp.cpp:178-181)
    c = __dsub_rn(c, __dmul_rn(lr, g));
  } else if (OPT == 1) {  // momentum (clomp.cpp:182-188)
    m1 = __dadd_rn(__dmul_rn(0.9, m1), g);
    c = __dsub_rn(c, __dmul_rn(lr, m1));
  } else {  // Adam (clomp.cpp:189-206)
    const double b1 = 0.9, b2 = 0.999, tiny = 1e-8;
    m1 = __dadd_rn(__dmul_rn(b1, m1), __dmul_rn(1.0 - b1, g));
    m2 = __dadd_rn(__dmul_rn(b2, m2), __dmul_rn(__dmul_rn(1.0 - b2, g), g));
    const double mhat = __ddiv_rn(m1, bc1);
    const double vhat = __ddiv_rn(m2, bc2);
    c = __dsub_rn(c, __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(sqrt(vhat), tiny)));
  }
}

// ------------------------------------------ learning, warp per signal
// All epochs of one outer iteration with G's row `lane` in registers (zero
// padded to T columns, which is exact) and c broadcast through shared memory.
template <int T, int OPT>
__device__ __forceinline__ void epochs_warp(const double (&g)[kWarpCap],
                                            double& c, double bi, double& m1,
                                            double& m2, double* cs,
                                            const SolveParams& p, int step0,
                                            int lane, int t) {
  for (int e = 0; e < p.inner; ++e) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int j = 0; j < T; j += 4) {
      const double2 c01 = *reinterpret_cast<const double2*>(cs + j);
      const double2 c23 = *reinterpret_cast<const double2*>(cs + j + 2);
      a0 = fma(g[j + 0], c01.x, a0);
      a1 = fma(g[j + 1], c01.y, a1);
      a2 = fma(g[j + 2], c23.x, a2);
      a3 = fma(g[j + 3], c23.y, a3);
    }
    const double grad = 2.0 * (((a0 + a1) + (a2 + a3)) - bi);
    double bc1 = 1.0, bc2 = 1.0;
    if (OPT == 2) {
      bc1 = p.bc1[step0 + e];
      bc2 = p.bc2[step0 + e];
    }
    if (lane < t) opt_step<OPT>(c, grad, m1, m2, p.lr, bc1, bc2);
    __syncwarp();
    cs[lane] = c;
    __syncwarp();
  }
}

template <int OPT>
__device__ __forceinline__ void epochs_dispatch(const double (&g)[kWarpCap],
                                                double& c, double bi,
                                                double& m1, double& m2,
                                                double* cs,
                                                const SolveParams& p,
                                                int step0, int lane, int t) {
  if (t <= 8)
    epochs_warp<8, OPT>(g, c, bi, m1, m2, cs, p, step0, lane, t);
  else if (t <= 16)
    epochs_warp<16, OPT>(g, c, bi, m1, m2, cs, p, step0, lane, t);
  else if (t <= 24)
    epochs_warp<24, OPT>(g, c, bi, m1, m2, cs, p, step0, lane, t);
  else
    epochs_warp<32, OPT>(g, c, bi, m1, m2, cs, p, step0, lane, t);
}

// Gram row/column and b entry for every atom added since the last call
// (one warp).  G[k][i] = a_k . a_i and b_k = a_k . y in fp64.
__device__ void warp_extend_gram(const SolveParams& p, const Work& w,
                                 int64_t b, int t0, int t, int lane) {
  const int64_t cap = p.cap;
  double* G = w.gram + b * cap * cap;
  const int32_t* sup = w.sup + b * cap;
  const double* y = w.y64 + b * p.ldm;
  for (int k = t0; k < t; ++k) {
    const float* ak = w.at32 + (int64_t)sup[k] * p.ldm;
    for (int i = 0; i <= k; ++i) {
      const float* ai = w.at32 + (int64_t)sup[i] * p.ldm;
      double acc = 0.0;
      for (int64_t q = lane; q < p.ldm; q += 32)
        acc = fma((double)ak[q], (double)ai[q], acc);
      acc = warp_sum(acc);
      if (lane == 0) {
        G[(int64_t)k * cap + i] = acc;
        G[(int64_t)i * cap + k] = acc;
      }
    }
    double acc = 0.0;
    for (int64_t q = lane; q < p.ldm; q += 32) acc = fma((double)ak[q], y[q], acc);
    acc = warp_sum(acc);
    if (lane == 0) {
      w.bvec[b * cap + k] = acc;
      w.coef[b * cap + k] = 0.0;  // new atoms start at 0 (clomp.hpp:53-54)
      w.mom1[b * cap + k] = 0.0;
      w.mom2[b * cap + k] = 0.0;
    }
  }
  __syncwarp();
}

// Residual r = A_S c - y (fp64), stored for the next correlation, and its
// sum of squares.  c is read from shared memory (cs[k] for support slot k).
__device__ double warp_residual(const SolveParams& p, const Work& w, int64_t b,
                                const double* cs, const int32_t* sups, int t,
                                int lane) {
  double lacc = 0.0;
  const double* y = w.y64 + b * p.ldm;
  for (int64_t i = lane; i < p.ldm; i += 32) {
    double acc = 0.0;
    for (int k = 0; k < t; ++k)
      acc = fma((double)w.at32[(int64_t)sups[k] * p.ldm + i], cs[k], acc);
    const double rv = acc - y[i];
    store_residual(w, b * p.ldm + i, rv);
    lacc = fma(rv, rv, lacc);
  }
  return warp_sum(lacc);
}

template <int OPT>
__device__ void learn_warp_body(const SolveParams& p, const Work& w, int64_t b,
                                int outer, double* cs, int32_t* sups,
                                int lane) {
  const int t = w.cnt[b];
  const int t0 = w.gcnt[b];
  const int64_t cap = p.cap;
  warp_extend_gram(p, w, b, t0, t, lane);
  if (lane == 0) w.gcnt[b] = t;

  double g[kWarpCap];
  const double* G = w.gram + b * cap * cap;
#pragma unroll
  for (int j = 0; j < kWarpCap; ++j)
    g[j] = (lane < t && j < t) ? G[(int64_t)lane * cap + j] : 0.0;
  double c = 0.0, bi = 0.0, m1 = 0.0, m2 = 0.0;
  if (lane < t) {
    c = w.coef[b * cap + lane];
    bi = w.bvec[b * cap + lane];
    m1 = w.mom1[b * cap + lane];
    m2 = w.mom2[b * cap + lane];
    sups[lane] = w.sup[b * cap + lane];
  }
  cs[lane] = c;
  __syncwarp();
  const int step0 = (outer - 1) * p.inner;
  epochs_dispatch<OPT>(g, c, bi, m1, m2, cs, p, step0, lane, t);
  if (lane < t) {
    w.coef[b * cap + lane] = c;
    w.mom1[b * cap + lane] = m1;
    w.mom2[b * cap + lane] = m2;
  }
  const double L = warp_residual(p, w, b, cs, sups, t, lane);
  if (p.mode == kModePerSignal) {
    bool snap = false;
    if (lane == 0) snap = control_signal(p, w, b, outer, L);
    snap = __shfl_sync(kFull, snap, 0);
    if (snap && lane < t) w.best_coef[b * cap + lane] = c;
  } else if (lane == 0) {
    w.loss[b] = L;
  }
}

__global__ void __launch_bounds__(128)
k_learn_warp(SolveParams p, Work w, int outer, int32_t* big_list) {
  __shared__ __align__(16) double cs_all[4][kWarpCap];
  __shared__ int32_t sup_all[4][kWarpCap];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * 4 + warp;
  if (b >= p.B || !w.active[b]) return;
  if (w.cnt[b] > kWarpCap) {  // handled by the block kernel
    if (lane == 0) {
      const int slot = atomicAdd(&w.counters[kRescanCount + 4], 1);
      big_list[slot] = (int32_t)b;
    }
    return;
  }
  double* cs = cs_all[warp];
  int32_t* sups = sup_all[warp];
  switch (p.opt) {
    case 0: learn_warp_body<0>(p, w, b, outer, cs, sups, lane); break;
    case 1: learn_warp_body<1>(p, w, b, outer, cs, sups, lane); break;
    default: learn_warp_body<2>(p, w, b, outer, cs, sups, lane); break;
  }
}

// ------------------------------------------ learning, block per signal
// Supports of any size up to kBlockRows * blockDim.  G lives in shared memory
// when it fits, else it is streamed from L2 every epoch (symmetric G is read
// column-wise so the threads of a warp touch consecutive addresses).
constexpr int kBlockThreads = 256;
constexpr int kBlockRows = 4;

template <int OPT, bool SMEM_G>
__global__ void __launch_bounds__(kBlockThreads)
k_learn_block(SolveParams p, Work w, int outer, const int32_t* big_list) {
  extern __shared__ __align__(16) unsigned char dsm[];
  double* cs = reinterpret_cast<double*>(dsm);                 // [cap]
  int32_t* sups = reinterpret_cast<int32_t*>(cs + p.cap);      // [cap]
  double* Gs = reinterpret_cast<double*>(sups + ((p.cap + 1) & ~1LL));  // [cap*cap]
  __shared__ double red[kBlockThreads / 32];
  __shared__ int snap_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = kBlockThreads / 32;
  const int count = w.counters[kRescanCount + 4];
  const int64_t cap = p.cap;
  for (int li = blockIdx.x; li < count; li += gridDim.x) {
    const int64_t b = big_list[li];
    const int t = w.cnt[b];
    const int t0 = w.gcnt[b];
    double* G = w.gram + b * cap * cap;
    const double* y = w.y64 + b * p.ldm;
    for (int k = tid; k < t; k += kBlockThreads) sups[k] = w.sup[b * cap + k];
    __syncthreads();
    // Gram extension: warps over (k, i) pairs, lanes over m.
    for (int k = t0; k < t; ++k) {
      const float* ak = w.at32 + (int64_t)sups[k] * p.ldm;
      for (int i = warp; i <= k; i += nw) {
        const float* ai = w.at32 + (int64_t)sups[i] * p.ldm;
        double acc = 0.0;
        for (int64_t q = lane; q < p.ldm; q += 32)
          acc = fma((double)ak[q], (double)ai[q], acc);
        acc = warp_sum(acc);
        if (lane == 0) {
          G[(int64_t)k * cap + i] = acc;
          G[(int64_t)i * cap + k] = acc;
        }
      }
      if (warp == 0) {
        double acc = 0.0;
        for (int64_t q = lane; q < p.ldm; q += 32) acc = fma((double)ak[q], y[q], acc);
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
    // Residual + loss.
    double lacc = 0.0;
    for (int64_t i = tid; i < p.ldm; i += kBlockThreads) {
      double acc = 0.0;
      for (int k = 0; k < t; ++k)
        acc = fma((double)w.at32[(int64_t)sups[k] * p.ldm + i], cs[k], acc);
      const double rv = acc - y[i];
      store_residual(w, b * p.ldm + i, rv);
      lacc = fma(rv, rv, lacc);
    }
    lacc = warp_sum(lacc);
    if (lane == 0) red[warp] = lacc;
    __syncthreads();
    if (tid == 0) {
      double L = 0.0;
      for (int q = 0; q < nw; ++q) L += red[q];
      snap_s = 0;
      if (p.mode == kModePerSignal)
        snap_s = control_signal(p, w, b, outer, L);
      else
        w.loss[b] = L;
    }
    __syncthreads();
    if (snap_s)
      for (int i = tid; i < t; i += kBlockThreads) w.best_coef[b * cap + i] = cs[i];
    __syncthreads();
  }
}

// ------------------------------------------------------ joint control
// clomp_solve_batch semantics (clomp.cpp:235-273): batch-global totals in a
// fixed reduction order (deterministic), one decision for every signal.
__global__ void __launch_bounds__(1024)
k_joint_control(SolveParams p, Work w, int outer, int init) {
  __shared__ double red[1024];
  __shared__ int chg[32];
  const int tid = threadIdx.x;
  double s = 0.0;
  int any = 0;
  for (int64_t b = tid; b < p.B; b += blockDim.x) {
    s += w.loss[b];
    any |= w.changed[b];
  }
  red[tid] = s;
  any = __any_sync(kFull, any);
  if ((tid & 31) == 0) chg[tid >> 5] = any;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  __shared__ int stop_s;
  if (tid == 0) {
    const double total = red[0];
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
      if (sqrt(total) < p.eps) {
        J[kJConv] = 1.0;
        stop = 1;
      }
    } else {
      J[kJTotal] = total;
      if (!isfinite(total)) {
        J[kJStatus] = (double)kStatusNumerical;
        stop = 1;
      } else {
        J[kJIters] = (double)outer;
        if (total < J[kJBest]) {
          J[kJBest] = total;
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
        } else if (sqrt(total) < p.eps) {
          J[kJConv] = 1.0;
          stop = 1;
        }
      }
    }
    J[kJStop] = stop;
    w.counters[kActiveCount] = stop ? 0 : (int)p.B;
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
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= p.B) return;
  const int64_t cap = p.cap;
  int status, iters, use_best;
  double rn;
  if (p.mode == kModeJoint) {
    const double* J = w.joint;
    status = (int)J[kJStatus];
    iters = (int)J[kJIters];
    const bool conv = J[kJConv] != 0.0;
    use_best = !conv && isfinite(J[kJBest]);
    rn = use_best ? sqrt(J[kJBest]) : sqrt(J[kJTotal]);
  } else {
    status = w.status[b];
    iters = w.iters[b];
    use_best = !w.conv[b] && isfinite(w.best_L[b]);
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

// inject_support unit path: ||r||^2 per column and a clean support list.
__global__ void k_inject_prep(SolveParams p, Work w) {
  const int lane = threadIdx.x & 31;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= p.B) return;
  double acc = 0.0;
  for (int64_t i = lane; i < p.ldm; i += 32) {
    const double v = w.r64[b * p.ldm + i];
    acc = fma(v, v, acc);
    if (w.r_hi) store_residual(w, b * p.ldm + i, v);
  }
  acc = warp_sum(acc);
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
  k_init<<<(unsigned)blocks, threads, 0, s>>>(p, w, y_in, y_layout == 0);
}

void launch_select(const SolveParams& p, const Work& w, bool full_scores,
                   cudaStream_t s) {
  if (full_scores) {
    const int64_t blocks = (p.B * 32 + 255) / 256;
    k_select_thresh<<<(unsigned)blocks, 256, 0, s>>>(p, w);
  } else {
    const int64_t blocks = (p.B + 255) / 256;
    k_select_top<<<(unsigned)blocks, 256, 0, s>>>(p, w);
  }
}

void launch_rescan(const SolveParams& p, const Work& w, int grid,
                   cudaStream_t s) {
  k_rescan<<<grid, 256, 0, s>>>(p, w);
}

static size_t block_smem_bytes(int64_t cap, bool smem_g) {
  size_t bytes = (size_t)cap * 8 + (size_t)((cap + 1) & ~1LL) * 4;
  if (smem_g) bytes += (size_t)cap * cap * 8;
  return bytes;
}

template <int OPT>
static void launch_block_variant(const SolveParams& p, const Work& w, int outer,
                                 int32_t* big_list, int grid, cudaStream_t s) {
  const size_t smem_g = block_smem_bytes(p.cap, true);
  if (smem_g <= 200 * 1024) {
    cudaFuncSetAttribute(k_learn_block<OPT, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_g);
    k_learn_block<OPT, true><<<grid, kBlockThreads, smem_g, s>>>(p, w, outer, big_list);
  } else {
    const size_t sm = block_smem_bytes(p.cap, false);
    cudaFuncSetAttribute(k_learn_block<OPT, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_learn_block<OPT, false><<<grid, kBlockThreads, sm, s>>>(p, w, outer, big_list);
  }
}

void launch_learn(const SolveParams& p, const Work& w, int outer, int max_cnt,
                  cudaStream_t s) {
  int32_t* big_list = w.rescan_list + p.B;  // second half of the list buffer
  cudaMemsetAsync(&w.counters[kRescanCount + 4], 0, sizeof(int32_t), s);
  const int64_t blocks = (p.B + 3) / 4;
  k_learn_warp<<<(unsigned)blocks, 128, 0, s>>>(p, w, outer, big_list);
  (void)max_cnt;
  if (p.cap > kWarpCap) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)(p.B < 2 * sms ? p.B : 2 * sms);
    switch (p.opt) {
      case 0: launch_block_variant<0>(p, w, outer, big_list, grid, s); break;
      case 1: launch_block_variant<1>(p, w, outer, big_list, grid, s); break;
      default: launch_block_variant<2>(p, w, outer, big_list, grid, s); break;
    }
  }
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
  const int64_t blocks = (p.B * 32 + 255) / 256;
  k_finalize<<<(unsigned)blocks, 256, 0, s>>>(p, w, out_cap, sup_out, coef_out,
                                             cnt_out, iters_out, rn_out,
                                             conv_out, status_out);
}

void launch_inject_finish(const SolveParams& p, const Work& w,
                          cudaStream_t s) {
  const int64_t blocks = (p.B * 32 + 255) / 256;
  k_inject_prep<<<(unsigned)blocks, 256, 0, s>>>(p, w);
}

}  // namespace clb
