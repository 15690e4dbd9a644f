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
  int mode;  // 0 store, 1 |.|, 2 residual (acc - yref), split + sum of squares
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

__global__ void __launch_bounds__(256) k_gemm_sep(Gemm g) {
  const int64_t b = blockIdx.y;
  if (g.active && !g.active[b]) return;
  __shared__ double Ps[GK][GT + 2];
  __shared__ double Qs[GK][GT + 2];
  __shared__ double red[8];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t tiles_x = (g.X + GT - 1) / GT;
  const int64_t x0 = (blockIdx.x % tiles_x) * GT, y0 = (blockIdx.x / tiles_x) * GT;
  const double* P = g.P + b * g.psb;
  const double* Q = g.Q + b * g.qsb;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
  const bool p_kfast = g.psk == 1, q_kfast = g.qsk == 1;
  for (int64_t k0 = 0; k0 < g.K; k0 += GK) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + 256 * u;
      const int xx = p_kfast ? e / GK : e % GT, kk = p_kfast ? e % GK : e / GT;
      const int64_t x = x0 + xx, k = k0 + kk;
      Ps[kk][xx] = (x < g.X && k < g.K) ? P[x * g.psx + k * g.psk] : 0.0;
      const int yy = q_kfast ? e / GK : e % GT, kq = q_kfast ? e % GK : e / GT;
      const int64_t y = y0 + yy, kq2 = k0 + kq;
      Qs[kq][yy] = (y < g.Y && kq2 < g.K) ? Q[y * g.qsy + kq2 * g.qsk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < GK; ++k) {
      double a[4], c[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = Ps[k][ty * 4 + q];
        c[q] = Qs[k][tx * 4 + q];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], c[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* C = g.C + b * g.csb;
  double ss = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t x = x0 + ty * 4 + i, y = y0 + tx * 4 + j;
      if (x >= g.X || y >= g.Y) continue;
      const int64_t o = x * g.csx + y * g.csy;
      double v = acc[i][j];
      if (g.mode == 1) {
        v = fabs(v);
      } else if (g.mode == 2) {
        v -= g.yref[b * g.csb + o];
        ss = fma(v, v, ss);
      }
      C[o] = v;
    }
  if (g.mode == 2) {
    ss = warp_sum_d(ss);
    if ((tid & 31) == 0) red[tid >> 5] = ss;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int q = 0; q < 8; ++q) t += red[q];
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

unsigned tiles2(int64_t X, int64_t Y) {
  return (unsigned)(((X + GT - 1) / GT) * ((Y + GT - 1) / GT));
}

}  // namespace

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
  k_gemm_sep<<<dim3(tiles2(g1.X, g1.Y), (unsigned)p.B), 256, 0, s>>>(g1);
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
  k_gemm_sep<<<dim3(tiles2(g2.X, g2.Y), (unsigned)p.B), 256, 0, s>>>(g2);
}

int64_t sep_resid_tiles(const SolveParams& p) { return tiles2(p.mr, p.mc); }

void launch_sep_control(const SolveParams& p, const Work& w, int outer, cudaStream_t s);

// r_b = vec(A_r C_b A_c^T) - y_b, its tf32 split, ||r_b||^2, stopping rules.
void launch_sep_resid(const SolveParams& p, const Work& w, int outer, int tb,
                      cudaStream_t s) {
  (void)tb;
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
  k_gemm_sep<<<dim3(tiles2(g.X, g.Y), (unsigned)p.B), 256, 0, s>>>(g);
  launch_sep_control(p, w, outer, s);
}

}  // namespace clb
