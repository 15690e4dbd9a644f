// k_sep.cu — separable 2D mode: the operator A = A_c (x) A_r applied through
// its factors (the reference has no separable mode, so
// its semantics are clomp_solve on the explicit Kronecker matrix).
//
// With column-major vec (atom p = i + nr*j, measurement q = qr + mr*qc):
//   correlation  A^T r      = vec(A_r^T R A_c)            two batched GEMMs
//   residual     A_S c - y  = vec(A_r C A_c^T) - y        scatter + one GEMM
//   support Gram G[(i,j),(i',j')] = Gr[i][i'] * Gc[j][j']  (k_solve.cu)
// so no M x N Kronecker matrix is ever formed (config 4 would need 8.6 GB fp64,
// config 5 137 GB).  All arithmetic here is fp64 (SIMT); the 2D path selects
// from exact fp64 scores and needs no rescans.
#include "clomp_internal.cuh"

namespace clb {
namespace {

constexpr int GT = 64;  // output tile (X and Y)
constexpr int GK = 16;  // K slice

// C_b[x, y] = sum_k P_b[x, k] * Q_b[y, k] with arbitrary strides.
struct Gemm {
  const double* P;
  int64_t psx, psk, psb;
  const double* Q;
  int64_t qsy, qsk, qsb;
  double* C;
  int64_t csx, csy, csb;
  int64_t X, Y, K;
  int mode;  // 0 store, 1 |.|, 2 residual (acc - yref) + sum of squares, 3 acc - yref
  const double* yref;
  double* lpart;
  int64_t tiles;  // tiles per batch entry (lpart stride)
  const int32_t* active;
};

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 64 x 64 output tile per CTA on the fp64 tensor cores (mma.sync m8n8k4 f64 ->
// DMMA): four warps, each a 32 x 32 quadrant as 4 x 4 accumulator blocks of
// 8 x 8.  K runs in 16-wide chunks through two shared-memory buffers; the next
// chunk's global loads are issued into registers before the current chunk's
// MMAs and stored after them, so the ~1 us load latency hides under ~64 DMMAs
// per warp (the SIMT 4 x 4 register tile this replaces waited for every chunk
// and ran at a fifth of the pipe with the 1-2 CTAs per SM these shapes give).
// Operands with arbitrary strides; tiles are staged as Ps[k][x] with row stride
// 68 doubles, for which the A / B fragment reads (lane -> k = lane % 4,
// x = lane / 4) hit 16 distinct 8-byte slots per half warp: conflict-free.
constexpr int kGemmThreads = 256;

// TX x 64 output tile (TX = 64 or 128 rows of X): eight warps as TX/32 x 256/TX,
// each a 32 x (64 TX / 256 ... ) sub-tile of 8 x 8 accumulator blocks.  At these
// shapes (K = 128..512, operands L2-resident) the kernel is bound by the bytes
// a CTA pulls from L2 per FLOP, so the 128-row tile (10.7 FLOP/B instead of 8)
// is used wherever the output has 128 rows to give.
template <int TX>
__global__ void __launch_bounds__(kGemmThreads) k_gemm_sep(Gemm g) {
  const int64_t b = blockIdx.y;
  if (g.active && !g.active[b]) return;
  constexpr int PLD = TX + 4, QLD = GT + 4;
  extern __shared__ __align__(16) double gsm[];
  double* Ps = gsm;                      // [2][GK][PLD]
  double* Qs = gsm + 2 * GK * PLD;       // [2][GK][QLD]
  __shared__ double red[kGemmThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int WX = TX / 32;            // warps along x
  constexpr int NJ = GT / (8 / WX) / 8;  // 8-wide accumulator blocks along y per warp
  const int wx = (warp % WX) * 32, wy = (warp / WX) * (8 * NJ);
  const int64_t tiles_x = (g.X + TX - 1) / TX;
  const int64_t x0 = (blockIdx.x % tiles_x) * TX, y0 = (blockIdx.x / tiles_x) * GT;
  const double* P = g.P + b * g.psb;
  const double* Q = g.Q + b * g.qsb;
  const bool p_kfast = g.psk == 1, q_kfast = g.qsk == 1;
  constexpr int PPER = TX * GK / kGemmThreads, QPER = GT * GK / kGemmThreads;
  double pv[PPER], qv[QPER];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int u = 0; u < PPER; ++u) {
      const int e = tid + kGemmThreads * u;
      const int xx = p_kfast ? e / GK : e % TX, kk = p_kfast ? e % GK : e / TX;
      const int64_t x = x0 + xx, k = k0 + kk;
      pv[u] = (x < g.X && k < g.K) ? P[x * g.psx + k * g.psk] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < QPER; ++u) {
      const int e = tid + kGemmThreads * u;
      const int yy = q_kfast ? e / GK : e % GT, kq = q_kfast ? e % GK : e / GT;
      const int64_t y = y0 + yy, k2 = k0 + kq;
      qv[u] = (y < g.Y && k2 < g.K) ? Q[y * g.qsy + k2 * g.qsk] : 0.0;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int u = 0; u < PPER; ++u) {
      const int e = tid + kGemmThreads * u;
      const int xx = p_kfast ? e / GK : e % TX, kk = p_kfast ? e % GK : e / TX;
      Ps[(buf * GK + kk) * PLD + xx] = pv[u];
    }
#pragma unroll
    for (int u = 0; u < QPER; ++u) {
      const int e = tid + kGemmThreads * u;
      const int yy = q_kfast ? e / GK : e % GT, kq = q_kfast ? e % GK : e / GT;
      Qs[(buf * GK + kq) * QLD + yy] = qv[u];
    }
  };
  double acc[4][NJ][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int fk = lane & 3, fr = lane >> 2;
  fetch(0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = 0; k0 < g.K; k0 += GK, buf ^= 1) {
    const bool more = k0 + GK < g.K;
    if (more) fetch(k0 + GK);
#pragma unroll
    for (int ks = 0; ks < GK; ks += 4) {
      double af[4], bf[NJ];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = Ps[(buf * GK + ks + fk) * PLD + wx + 8 * i + fr];
#pragma unroll
      for (int j = 0; j < NJ; ++j) bf[j] = Qs[(buf * GK + ks + fk) * QLD + wy + 8 * j + fr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
              : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
              : "d"(af[i]), "d"(bf[j]));
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
  }
  // accumulator block (i, j): element (row = fr, cols 2 fk, 2 fk + 1)
  double* C = g.C + b * g.csb;
  double ss = 0.0;
  // Outputs contiguous along y (the MMA's column pair c0, c1 of a lane is two
  // adjacent doubles): one 16-byte access per pair, so four lanes cover 64
  // contiguous bytes instead of half of each 32-byte sector (the scalar
  // epilogue's yref reads were 37 % of this kernel's stall samples).
  const bool pair_ok = g.csy == 1 && (g.csx & 1) == 0 && (g.csb & 1) == 0 && (g.Y & 1) == 0 &&
                       (reinterpret_cast<uintptr_t>(g.C) & 15) == 0 && g.mode != 1 &&
                       (g.mode == 0 || (reinterpret_cast<uintptr_t>(g.yref) & 15) == 0);
  if (pair_ok) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int64_t x = x0 + wx + 8 * i + fr, y = y0 + wy + 8 * j + 2 * fk;
        if (x >= g.X || y >= g.Y) continue;
        const int64_t o = x * g.csx + y;
        double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
        if (g.mode >= 2) {
          const double2 r = *reinterpret_cast<const double2*>(g.yref + b * g.csb + o);
          v.x -= r.x;
          v.y -= r.y;
          if (g.mode == 2) ss = fma(v.y, v.y, fma(v.x, v.x, ss));
        }
        *reinterpret_cast<double2*>(C + o) = v;
      }
  } else
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t x = x0 + wx + 8 * i + fr, y = y0 + wy + 8 * j + 2 * fk + h;
        if (x >= g.X || y >= g.Y) continue;
        const int64_t o = x * g.csx + y * g.csy;
        double v = acc[i][j][h];
        if (g.mode == 1) {
          v = fabs(v);
        } else if (g.mode == 2) {
          v -= g.yref[b * g.csb + o];
          ss = fma(v, v, ss);
        } else if (g.mode == 3) {
          v -= g.yref[b * g.csb + o];
        }
        C[o] = v;
      }
  if (g.mode == 2) {
    ss = warp_sum_d(ss);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int q = 0; q < kGemmThreads / 32; ++q) t += red[q];
      g.lpart[b * g.tiles + blockIdx.x] = t;
    }
  }
}

// V_b = A_r C_b as its transpose VT[j][qr] = sum_{k: j_k = j} c_k A_r[qr][i_k];
// one block per image, each thread owns rows qr (no write conflicts).
__global__ void __launch_bounds__(256) k_sep_scatter(SolveParams p, Work w) {
  const int64_t b = blockIdx.x;
  if (!w.active[b]) return;
  const int t = w.cnt[b];
  double* vt = w.sep_scratch + b * p.nc * p.mr;
  for (int64_t e = threadIdx.x; e < p.nc * p.mr; e += blockDim.x) vt[e] = 0.0;
  __syncthreads();
  for (int64_t qr = threadIdx.x; qr < p.mr; qr += blockDim.x) {
    for (int k = 0; k < t; ++k) {
      const int64_t pk = w.sup[b * p.cap + k];
      const int64_t ik = pk % p.nr, jk = pk / p.nr;
      vt[jk * p.mr + qr] = fma(w.coef[b * p.cap + k], w.at_r64[ik * p.ldr + qr], vt[jk * p.mr + qr]);
    }
  }
}

// Rows of U (one per image b and coefficient column j, mr doubles) to the K1
// residual operand: per-row power-of-two scale from the row norm, fp16 hi / lo
// halves (zero padded to ldr), and the image's active flag per row.  One warp
// per row.
__global__ void __launch_bounds__(256) k_sep_split_u(SolveParams p, Work w) {
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= p.B * p.nc) return;
  const int64_t b = row / p.nc;
  const int act = w.active[b];
  if (lane == 0) w.u_active[row] = act;
  if (!act) return;
  const double* u = w.sep_scratch + row * p.mr;
  double ss = 0.0;
  for (int64_t q = lane; q < p.mr; q += 32) ss = fma(u[q], u[q], ss);
  ss = warp_sum_d(ss);
  const float sc = split_scale(ss);
  if (lane == 0) w.u_scale[row] = 1.0f / sc;
  for (int64_t q = lane; q < p.ldr; q += 32) {
    __half h = __float2half_rn(0.f), l = h;
    if (q < p.mr) split_f16(u[q], sc, h, l);
    w.u_hi[row * p.ldr + q] = h;
    w.u_lo[row * p.ldr + q] = l;
  }
}

// K1 wrote atom indices local to its pseudo-signal (i in [0, nr)); record
// (b, tile) belongs to coefficient column j = tile / (nr / tile_atoms), so the
// global atom is i + nr j.
__global__ void k_sep_fix_cand(SolveParams p, Work w) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p.B * p.ntile) return;
  const int64_t tile = e % p.ntile;
  const int32_t base = (int32_t)((tile / (p.nr / p.tile_atoms)) * p.nr);
  Cand c = w.cand[e];
  CL_CHECK((c.i1 == 0x7fffffff || (c.i1 >= 0 && c.i1 < p.nr)) &&
           (c.i2 == 0x7fffffff || (c.i2 >= 0 && c.i2 < p.nr)));
  if (c.i1 != 0x7fffffff) c.i1 += base;
  if (c.i2 != 0x7fffffff) c.i2 += base;
  w.cand[e] = c;
}

// ------------------------------------------------ direct-form learning
// Supports too large for the Gram form (G is t x t fp64 per image: 1.4 GB at
// config 5's K = 13107) or past the point where streaming G costs more than
// applying the operator (t^2 > ~ mr nc mc / 8) learn with the reference's own
// epoch (clomp.cpp:83-91, 120-123, 171-209) applied through the factors:
//   V = A_r C        sparse: per coefficient column j, sum_k c_k a_r,i_k
//   R = V A_c^T - Y  dense fp64 GEMM (mr x nc x mc)
//   U = R A_c        dense fp64 GEMM (mr x mc x nc)
//   g_k = 2 a_r,i_k . U_j_k   for the t support entries only, optimizer step
// The support is kept column-sorted (CSC) so V needs no atomics and its
// summation order is fixed.

// One block per image: zero the coefficients of the atoms selected since the
// last call (clomp.hpp:53-54), then sort the support by coefficient column
// (stable: insertion order inside a column).
__global__ void __launch_bounds__(256) k_dir_csc(SolveParams p, Work w) {
  extern __shared__ int32_t s_cnt[];  // [nc + 1]
  const int64_t b = blockIdx.x;
  if (!w.active[b]) return;
  const int t = w.cnt[b], t0 = w.gcnt[b];
  const int tid = threadIdx.x;
  for (int k = t0 + tid; k < t; k += blockDim.x) {
    w.coef[b * p.cap + k] = 0.0;
    w.mom1[b * p.cap + k] = 0.0;
    w.mom2[b * p.cap + k] = 0.0;
  }
  for (int64_t j = tid; j <= p.nc; j += blockDim.x) s_cnt[j] = 0;
  __syncthreads();
  const int32_t* sup = w.sup + b * p.cap;
  for (int k = tid; k < t; k += blockDim.x) atomicAdd(&s_cnt[sup[k] / p.nr + 1], 1);
  __syncthreads();
  if (tid == 0) {
    int run = 0;
    for (int64_t j = 0; j <= p.nc; ++j) {
      run += s_cnt[j];
      s_cnt[j] = run;
    }
  }
  __syncthreads();
  int32_t* ptr = w.csc_ptr + b * (p.nc + 1);
  for (int64_t j = tid; j <= p.nc; j += blockDim.x) ptr[j] = s_cnt[j];
  // column j's entries in insertion order: one thread per column scans the
  // support (t <= a few thousand per image; once per outer iteration)
  int32_t* perm = w.csc_perm + b * p.cap;
  CL_CHECK(t >= 0 && t <= p.cap && t0 >= 0 && t0 <= t);
  for (int64_t j = tid; j < p.nc; j += blockDim.x) {
    int pos = s_cnt[j];
    const int end = s_cnt[j + 1];
    for (int k = 0; k < t && pos < end; ++k)
      if (sup[k] / p.nr == j) perm[pos++] = k;
  }
  if (tid == 0) w.gcnt[b] = t;
}

// One epoch's sparse half, one WARP per coefficient column j of image b (the
// entries of a column share U_j and V_j and nothing else): with STEP, every
// entry's gradient g_k = 2 a_r,i_k . U_j and gradient_step on c_k (the lanes
// update the column's entries in parallel); then V_b^T[j][:] = sum over the
// column's entries of c_k a_r,i_k with the new coefficients, which the next
// epoch's residual GEMM (or the iteration's final residual) reads.  Entries in
// chunks of 32 (one per lane), rows in chunks of 32 kDirRows per lane.
constexpr int kDirWarps = 8;
constexpr int kDirRows = 8;  // rows per lane per pass (256-row passes)

template <int OPT, bool STEP>
__global__ void __launch_bounds__(32 * kDirWarps) k_dir_colstep(SolveParams p, Work w,
                                                               const double* __restrict__ u,
                                                               double* __restrict__ vt, int step) {
  const int64_t b = blockIdx.y;
  if (!w.active[b]) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * kDirWarps + warp;
  if (j >= p.nc) return;
  const int32_t* ptr = w.csc_ptr + b * (p.nc + 1);
  const int e0 = ptr[j], e1 = ptr[j + 1];
  const int32_t* perm = w.csc_perm + b * p.cap;
  const int32_t* sup = w.sup + b * p.cap;
  double* coef = w.coef + b * p.cap;
  const double* uj = u + (b * p.nc + j) * p.mr;
  double* out = vt + (b * p.nc + j) * p.mr;
  for (int64_t q0 = 0; q0 < p.mr; q0 += 32 * kDirRows) {
    double vacc[kDirRows];
#pragma unroll
    for (int r = 0; r < kDirRows; ++r) vacc[r] = 0.0;
    for (int ec = e0; ec < e1; ec += 32) {
      const int ne = min(32, e1 - ec);
      int k_l = 0;
      int64_t row_l = 0;
      double c_l = 0.0;
      if (lane < ne) {
        k_l = perm[ec + lane];
        CL_CHECK(k_l >= 0 && k_l < w.cnt[b] && sup[k_l] >= 0 && sup[k_l] < p.n &&
                 sup[k_l] / p.nr == j);
        row_l = (int64_t)(sup[k_l] % p.nr) * p.ldr;
        c_l = coef[k_l];
      }
      if (STEP && q0 == 0) {  // gradients of this chunk's entries (full-length dots)
        double g_l = 0.0;
        for (int idx = 0; idx < ne; ++idx) {
          const double* ar = w.at_r64 + __shfl_sync(0xffffffffu, row_l, idx);
          double acc = 0.0;
          for (int64_t q = lane; q < p.mr; q += 32) acc = fma(ar[q], uj[q], acc);
          acc = warp_sum_d(acc);
          if (lane == idx) g_l = acc;
        }
        if (lane < ne) {
          const int64_t o = b * p.cap + k_l;
          double m1 = 0.0, m2 = 0.0, bc1 = 1.0, bc2 = 1.0;
          if (OPT != 0) {
            m1 = w.mom1[o];
            m2 = w.mom2[o];
          }
          if (OPT == 2) {
            bc1 = p.bc1[step];
            bc2 = p.bc2[step];
          }
          opt_step<OPT>(c_l, 2.0 * g_l, m1, m2, p.lr, bc1, bc2);
          coef[k_l] = c_l;
          if (OPT != 0) {
            w.mom1[o] = m1;
            w.mom2[o] = m2;
          }
        }
      }
      for (int idx = 0; idx < ne; ++idx) {
        const double* ar = w.at_r64 + __shfl_sync(0xffffffffu, row_l, idx);
        const double c = __shfl_sync(0xffffffffu, c_l, idx);
#pragma unroll
        for (int r = 0; r < kDirRows; ++r) {
          const int64_t q = q0 + lane + 32 * r;
          if (q < p.mr) vacc[r] = fma(c, ar[q], vacc[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kDirRows; ++r) {
      const int64_t q = q0 + lane + 32 * r;
      if (q < p.mr) out[q] = vacc[r];
    }
  }
}

unsigned tiles2(int64_t X, int64_t Y) {
  return (unsigned)(((X + GT - 1) / GT) * ((Y + GT - 1) / GT));
}

// 128-row tiles wherever the output has them to give; the residual GEMM (mode
// 2) keeps 64 x 64 so its loss partials stay tiles2(m_r, m_c) per image.
void launch_gemm(const Gemm& g, int64_t B, cudaStream_t s) {
  static DevSlots attr_set[2];
  const int dev = current_device();
  if (g.mode != 2 && g.X >= 128) {
    constexpr size_t smem = (size_t)2 * GK * (128 + 4 + GT + 4) * sizeof(double);
    if (attr_set[1].get(dev) == 0) {
      cudaFuncSetAttribute(k_gemm_sep<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr_set[1].set(dev, 1);
    }
    const unsigned tiles = (unsigned)(((g.X + 127) / 128) * ((g.Y + GT - 1) / GT));
    k_gemm_sep<128><<<dim3(tiles, (unsigned)B), kGemmThreads, smem, s>>>(g);
  } else {
    constexpr size_t smem = (size_t)2 * GK * (64 + 4 + GT + 4) * sizeof(double);
    k_gemm_sep<64><<<dim3(tiles2(g.X, g.Y), (unsigned)B), kGemmThreads, smem, s>>>(g);
  }
}

}  // namespace

void launch_sep_control(const SolveParams& p, const Work& w, int outer, cudaStream_t s);

// dst_b = A_r^T Src_b A_c (vec'd), Src_b = vec(r_src_b) with leading dim ldm.
// abs_scores: |.| into the full-score buffer; else signed (Z = A_r^T Y A_c).
void launch_sep_corr(const SolveParams& p, const Work& w, const double* r_src,
                     double* dst, bool abs_scores, cudaStream_t s) {
  // stage 1: U_b[j][qr] = sum_qc A_c[qc][j] R_b[qr][qc]
  Gemm g1{};
  g1.P = w.at_c64;
  g1.psx = p.ldc;
  g1.psk = 1;
  g1.psb = 0;
  g1.Q = r_src;
  g1.qsy = 1;
  g1.qsk = p.mr;
  g1.qsb = p.ldm;
  g1.C = w.sep_scratch;
  g1.csx = p.mr;
  g1.csy = 1;
  g1.csb = p.nc * p.mr;
  g1.X = p.nc;
  g1.Y = p.mr;
  g1.K = p.mc;
  g1.mode = 0;
  g1.active = w.active;
  launch_gemm(g1, p.B, s);
  // stage 2: S_b[i][j] = sum_qr A_r[qr][i] U_b[j][qr], stored at p = i + nr*j
  Gemm g2{};
  g2.P = w.at_r64;
  g2.psx = p.ldr;
  g2.psk = 1;
  g2.psb = 0;
  g2.Q = w.sep_scratch;
  g2.qsy = p.mr;
  g2.qsk = 1;
  g2.qsb = p.nc * p.mr;
  g2.C = dst;
  g2.csx = 1;
  g2.csy = p.nr;
  g2.csb = p.n;
  g2.X = p.nr;
  g2.Y = p.nc;
  g2.K = p.mr;
  g2.mode = abs_scores ? 1 : 0;
  g2.active = w.active;
  launch_gemm(g2, p.B, s);
}

bool launch_sep_corr_tc(const SolveParams& p, const Work& w, cudaStream_t s) {
  // stage 1 (fp64): U_b[j][qr] = sum_qc A_c[qc][j] R_b[qr][qc]
  Gemm g1{};
  g1.P = w.at_c64;
  g1.psx = p.ldc;
  g1.psk = 1;
  g1.psb = 0;
  g1.Q = w.r64;
  g1.qsy = 1;
  g1.qsk = p.mr;
  g1.qsb = p.ldm;
  g1.C = w.sep_scratch;
  g1.csx = p.mr;
  g1.csy = 1;
  g1.csb = p.nc * p.mr;
  g1.X = p.nc;
  g1.Y = p.mr;
  g1.K = p.mc;
  g1.mode = 0;
  g1.active = w.active;
  launch_gemm(g1, p.B, s);
  const int64_t rows = p.B * p.nc;
  k_sep_split_u<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, s>>>(p, w);
  // stage 2 on tcgen05: scores(i, j) = a_r,i . U_j for every row as its own
  // "signal" against the dictionary A_r; the epilogue keeps the candidate
  // records per (row, 256-atom tile), which is the image's (b, tile) layout.
  SolveParams q = p;
  q.B = rows;
  q.ldm = p.ldr;
  q.m = p.mr;
  q.n = p.nr;
  q.n_corr = p.nr;
  q.atom0 = 0;
  q.ntile = p.nr / p.tile_atoms;
  q.ntl = q.ntile;
  Work v = w;
  v.r_hi = w.u_hi;
  v.r_lo = w.u_lo;
  v.r_scale = w.u_scale;
  v.active = w.u_active;
  if (!launch_corr_tc(q, v, s)) return false;
  const int64_t recs = p.B * p.ntile;
  k_sep_fix_cand<<<(unsigned)((recs + 255) / 256), 256, 0, s>>>(p, w);
  return true;
}

// R = V A_c^T - Y from V^T in `vt` (mode 2: also the loss partials).
static void launch_dir_resid_gemm(const SolveParams& p, const Work& w, const double* vt,
                                  cudaStream_t s) {
  Gemm g{};
  g.P = vt;  // VT[j][qr]
  g.psx = 1;
  g.psk = p.mr;
  g.psb = p.nc * p.mr;
  g.Q = w.at_c64;  // A_c[qc][j] = at_c64[j][qc]
  g.qsy = 1;
  g.qsk = p.ldc;
  g.qsb = 0;
  g.C = w.r64;
  g.csx = 1;
  g.csy = p.mr;
  g.csb = p.ldm;
  g.X = p.mr;
  g.Y = p.mc;
  g.K = p.nc;
  g.mode = 2;
  g.yref = w.y64;
  g.lpart = w.lpart;
  g.tiles = tiles2(p.mr, p.mc);
  g.active = w.active;
  launch_gemm(g, p.B, s);
}

// Z2_b = Y_b A_c (once per solve): the constant part of U = R A_c.
void launch_sep_direct_prepare(const SolveParams& p, const Work& w, cudaStream_t s) {
  Gemm g1{};
  g1.P = w.at_c64;
  g1.psx = p.ldc;
  g1.psk = 1;
  g1.psb = 0;
  g1.Q = w.y64;
  g1.qsy = 1;
  g1.qsk = p.mr;
  g1.qsb = p.ldm;
  g1.C = w.sep_z2;
  g1.csx = p.mr;
  g1.csy = 1;
  g1.csb = p.nc * p.mr;
  g1.X = p.nc;
  g1.Y = p.mr;
  g1.K = p.mc;
  g1.mode = 0;
  g1.active = nullptr;
  launch_gemm(g1, p.B, s);
}

// One epoch = the product(s) forming U = R A_c and one column kernel.  With
// R = V A_c^T - Y,
//   U = R A_c = V (A_c^T A_c) - Y A_c = V Gc - Z2,
// so when n_c <= 2 m_c the two m_r x n_c x m_c products collapse into one
// m_r x n_c x n_c product with the factor Gram Gc the context already holds (the
// same regrouping as the 1D Gram form's G c - b; the residual itself is then
// only formed at the end of the iteration, launch_sep_resid).
int launch_sep_direct_learn(const SolveParams& p, const Work& w, int outer, int bound,
                            cudaStream_t s) {
  (void)bound;
  k_dir_csc<<<(unsigned)p.B, 256, (size_t)(p.nc + 1) * sizeof(int32_t), s>>>(p, w);
  const dim3 cgrid((unsigned)((p.nc + kDirWarps - 1) / kDirWarps), (unsigned)p.B);
  double* vt = w.sep_scratch;
  double* u = w.sep_scratch2;
  k_dir_colstep<0, false><<<cgrid, 32 * kDirWarps, 0, s>>>(p, w, u, vt, 0);  // V of the current c
  // n_c <= 2 m_c: the regrouped product is no more work than the two it
  // replaces (m_r n_c^2 against 2 m_r m_c n_c) and saves a launch per epoch
  const bool regroup = p.nc <= 2 * p.mc;
  for (int e = 0; e < p.inner; ++e) {
    if (regroup) {
      // U_b[j][qr] = sum_j' Gc[j][j'] V_b[j'][qr] - Z2_b[j][qr]
      Gemm g{};
      g.P = w.gc;
      g.psx = p.nc;
      g.psk = 1;
      g.psb = 0;
      g.Q = vt;
      g.qsy = 1;
      g.qsk = p.mr;
      g.qsb = p.nc * p.mr;
      g.C = u;
      g.csx = p.mr;
      g.csy = 1;
      g.csb = p.nc * p.mr;
      g.X = p.nc;
      g.Y = p.mr;
      g.K = p.nc;
      g.mode = 3;
      g.yref = w.sep_z2;
      g.active = w.active;
      launch_gemm(g, p.B, s);
    } else {
      launch_dir_resid_gemm(p, w, vt, s);  // R = V A_c^T - Y
      Gemm g1{};                           // U_b[j][qr] = sum_qc A_c[qc][j] R_b[qr][qc]
      g1.P = w.at_c64;
      g1.psx = p.ldc;
      g1.psk = 1;
      g1.psb = 0;
      g1.Q = w.r64;
      g1.qsy = 1;
      g1.qsk = p.mr;
      g1.qsb = p.ldm;
      g1.C = u;
      g1.csx = p.mr;
      g1.csy = 1;
      g1.csb = p.nc * p.mr;
      g1.X = p.nc;
      g1.Y = p.mr;
      g1.K = p.mc;
      g1.mode = 0;
      g1.active = w.active;
      launch_gemm(g1, p.B, s);
    }
    const int step = (outer - 1) * p.inner + e;
    switch (p.opt) {  // the step and the next V in one pass over the columns
      case 0: k_dir_colstep<0, true><<<cgrid, 32 * kDirWarps, 0, s>>>(p, w, u, vt, step); break;
      case 1: k_dir_colstep<1, true><<<cgrid, 32 * kDirWarps, 0, s>>>(p, w, u, vt, step); break;
      default: k_dir_colstep<2, true><<<cgrid, 32 * kDirWarps, 0, s>>>(p, w, u, vt, step); break;
    }
  }
  return 2 + (regroup ? 2 : 3) * p.inner;
}

int64_t sep_resid_tiles(const SolveParams& p) { return tiles2(p.mr, p.mc); }

// r_b = vec(A_r C_b A_c^T) - y_b, its tf32 split, ||r_b||^2, stopping rules.
void launch_sep_resid(const SolveParams& p, const Work& w, int outer, int tb,
                      cudaStream_t s) {
  (void)tb;
  if (p.direct && w.csc_ptr) {  // V of the learned coefficients is in sep_scratch already
    launch_dir_resid_gemm(p, w, w.sep_scratch, s);
    launch_sep_control(p, w, outer, s);
    return;
  }
  k_sep_scatter<<<(unsigned)p.B, 256, 0, s>>>(p, w);
  Gemm g{};
  g.P = w.sep_scratch;  // VT[j][qr]
  g.psx = 1;
  g.psk = p.mr;
  g.psb = p.nc * p.mr;
  g.Q = w.at_c64;  // A_c[qc][j] = at_c64[j][qc]
  g.qsy = 1;
  g.qsk = p.ldc;
  g.qsb = 0;
  g.C = w.r64;
  g.csx = 1;
  g.csy = p.mr;
  g.csb = p.ldm;
  g.X = p.mr;
  g.Y = p.mc;
  g.K = p.nc;
  g.mode = 2;
  g.yref = w.y64;
  g.lpart = w.lpart;
  g.tiles = sep_resid_tiles(p);
  g.active = w.active;
  launch_gemm(g, p.B, s);
  launch_sep_control(p, w, outer, s);
}

}  // namespace clb
