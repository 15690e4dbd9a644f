/*
 * clomp_oracle.c — fp64 CPU restatement of the reference CLOMP loop.
 *
 * TEST INFRASTRUCTURE ONLY (see clomp_oracle.h).  Never linked into, loaded by
 * or called from the product library.
 *
 * What it restates, with the reference lines it follows:
 *   validate                 clomp.cpp:18-30
 *   inject_from_scores       clomp.cpp:41-53   (select_support twin, solvers.cpp:68-80)
 *   loss_impl                clomp.cpp:74-127 (with the priors)
 *   tv_1d / tv_2d            priors.cpp:11-26 / 28-59
 *   local_variance           priors.cpp:61-116
 *   resolve_weights          clomp.cpp:131-140
 *   gradient_step            clomp.cpp:171-209
 *   clomp_solve_batch        clomp.cpp:211-292
 *   clomp_solve              clomp.cpp:294-311
 * and the arithmetic of the kernels those call:
 *   kern::gemm  avx2  kernels_avx2.cpp:164-236  (per output: sequential FMA over k)
 *               scalar kernels_scalar.cpp:62-70 (per output: sequential mul+add over k)
 *   kern::sum_sq avx2 kernels_avx2.cpp:30-58    (4x4 accumulators, hsum, FMA tail)
 *               scalar kernels_scalar.cpp:16-20
 *
 * Why it is bit-identical although it is support-restricted: the reference
 * residual A*(mask.*s) sums over all n atoms, but a term with s_j == 0 adds an
 * exact zero to a sequential accumulation, so summing only the support in
 * ascending index order gives the same bits.  Gradients are
 * only needed on the mask (loss_impl zeroes the rest, clomp.cpp:120-122).
 *
 * Build flags matter: compiled with -mfma -ffp-contract=off so that every
 * fused multiply-add below is an explicit fma() and nothing else is fused.
 */
#include "clomp_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- kernels */

/* kern::dot / sum_sq, avx2 variant (kernels_avx2.cpp:30-58). */
static double dot_avx2(const double* a, const double* b, int64_t n) {
  double acc[4][4];
  memset(acc, 0, sizeof(acc));
  int64_t i = 0;
  for (; i + 16 <= n; i += 16)
    for (int k = 0; k < 4; ++k)
      for (int l = 0; l < 4; ++l)
        acc[k][l] = fma(a[i + 4 * k + l], b[i + 4 * k + l], acc[k][l]);
  for (; i + 4 <= n; i += 4)
    for (int l = 0; l < 4; ++l) acc[0][l] = fma(a[i + l], b[i + l], acc[0][l]);
  double v[4];
  for (int l = 0; l < 4; ++l) v[l] = (acc[0][l] + acc[1][l]) + (acc[2][l] + acc[3][l]);
  /* hsum: lo = (v0+v2, v1+v3), then lo[0] + lo[1] (kernels_avx2.cpp:20-26). */
  double total = (v[0] + v[2]) + (v[1] + v[3]);
  for (; i < n; ++i) total = fma(a[i], b[i], total); /* contracted under -mfma */
  return total;
}

/* kern::sum_sq, scalar variant (kernels_scalar.cpp:16-20). */
static double dot_scalar(const double* a, const double* b, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

static double sum_sq(const double* a, int64_t n, int isa) {
  return isa == ORC_ISA_AVX2 ? dot_avx2(a, a, n) : dot_scalar(a, a, n);
}

/* One gemm accumulation step c += a*b in the reference's per-ISA arithmetic. */
static inline double mac(double acc, double a, double b, int isa) {
  return isa == ORC_ISA_AVX2 ? fma(a, b, acc) : acc + a * b;
}

/* --------------------------------------------------------------- helpers */

static void set_err(char* err, int errlen, const char* fmt, ...) {
  if (!err || errlen <= 0) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, (size_t)errlen, fmt, ap);
  va_end(ap);
}

static int validate(const orc_config* c, char* err, int errlen) {
  if (!(c->th > 0.0) || c->th > 1.0) {
    set_err(err, errlen, "clomp: th must be in (0, 1]");
    return ORC_ERR_CONFIG;
  }
  if (c->max_outer == 0) {
    set_err(err, errlen, "clomp: max_outer must be >= 1");
    return ORC_ERR_CONFIG;
  }
  if (c->eps < 0.0) {
    set_err(err, errlen, "clomp: eps must be non-negative");
    return ORC_ERR_CONFIG;
  }
  if (c->inner_steps == 0) {
    set_err(err, errlen, "clomp: inner_steps must be >= 1");
    return ORC_ERR_CONFIG;
  }
  if (!(c->lr > 0.0)) {
    set_err(err, errlen, "clomp: lr must be positive");
    return ORC_ERR_CONFIG;
  }
  if (c->stall_tol < 0.0) {
    set_err(err, errlen, "clomp: stall_tol must be non-negative");
    return ORC_ERR_CONFIG;
  }
  if (c->stall_patience == 0) {
    set_err(err, errlen, "clomp: stall_patience must be >= 1");
    return ORC_ERR_CONFIG;
  }
  if (c->opt < 0 || c->opt > 2) {
    set_err(err, errlen, "clomp: unknown optimizer");
    return ORC_ERR_CONFIG;
  }
  return ORC_OK;
}

/* resolve_weights (clomp.cpp:131-140). */
static void resolve_weights(const orc_config* c, const double* y, int64_t count,
                            int isa, double* w_tv, double* w_lv) {
  const double mean_sq = sum_sq(y, count, isa) / (double)count;
  const double auto_w = 0.01 * mean_sq;
  *w_tv = c->w_tv < 0.0 ? auto_w : c->w_tv;
  *w_lv = c->w_lv < 0.0 ? auto_w : c->w_lv;
}

/* Per-column ascending support list (the order the dense sum visits atoms). */
typedef struct {
  int64_t* idx;
  int64_t count;
} support_t;

static void support_insert(support_t* s, int64_t j) {
  int64_t pos = s->count;
  while (pos > 0 && s->idx[pos - 1] > j) {
    s->idx[pos] = s->idx[pos - 1];
    --pos;
  }
  s->idx[pos] = j;
  ++s->count;
}

typedef struct {
  const double* a;   /* m x n (NULL for the separable operator) */
  const double* at;  /* n x m (LossOps::at, clomp.cpp:57-66) */
  int64_t m, n, batch;
  int isa;
  /* Separable operator A = A_c (x) A_r, column-major vec: atom p = i + n_r j,
   * measurement q = qr + m_r qc, A[q][p] = A_c[qc][j] * A_r[qr][i] (the entry
   * an explicit np.kron / dense Kronecker matrix would hold). */
  const double* ar;  /* m_r x n_r */
  const double* ac;  /* m_c x n_c */
  int64_t mr, nr, mc, nc;
  /* Priors (single-column solves): synthesis basis D (n x n row-major,
   * x = D s), its transpose (LossOps::dt, clomp.cpp:63-65) and the resolved
   * TV weight (0 = prior branch skipped, clomp.cpp:94). */
  const double* basis;
  const double* dt;
  double w_tv;
  /* local variance (priors.cpp:74-116), evaluated when w_lv > 0 and the batch
   * fits the window (clomp.cpp:93) */
  double w_lv;
  int lv_on;
  int64_t lv_window, lv_stride;
} problem_t;

static inline double entry(const problem_t* p, int64_t q, int64_t j) {
  if (p->a) return p->a[q * p->n + j];
  const int64_t qr = q % p->mr, qc = q / p->mr, i = j % p->nr, jc = j / p->nr;
  return p->ac[qc * p->nc + jc] * p->ar[qr * p->nr + i];
}

/* r = A*(mask.*s) - y  (clomp.cpp:83-84, 236-237, 285-286), support-restricted. */
static void residual(const problem_t* p, const double* s, const support_t* sup,
                     const double* y, double* r) {
  const int64_t B = p->batch;
  if (p->at) {
    /* Same per-element sums (support order, the same mac sequence from 0.0),
     * accumulated atom by atom over contiguous rows of the transposed copy
     * instead of gathering A's strided columns (cache-friendly at config 3's
     * 512 MB dictionary; bit-identical results). */
    const int64_t m = p->m;
    for (int64_t b = 0; b < B; ++b) {
      for (int64_t i = 0; i < m; ++i) r[i * B + b] = 0.0;
      const support_t* sb = &sup[b];
      for (int64_t q = 0; q < sb->count; ++q) {
        const int64_t j = sb->idx[q];
        const double* atrow = p->at + j * m;
        const double sj = s[j * B + b];
        for (int64_t i = 0; i < m; ++i) r[i * B + b] = mac(r[i * B + b], atrow[i], sj, p->isa);
      }
      for (int64_t i = 0; i < m; ++i) r[i * B + b] = r[i * B + b] - y[i * B + b];
    }
    return;
  }
  for (int64_t i = 0; i < p->m; ++i) {
    for (int64_t b = 0; b < B; ++b) {
      double acc = 0.0;
      const support_t* sb = &sup[b];
      for (int64_t q = 0; q < sb->count; ++q) {
        const int64_t j = sb->idx[q];
        acc = mac(acc, entry(p, i, j), s[j * B + b], p->isa);
      }
      r[i * B + b] = acc - y[i * B + b];
    }
  }
}

/* x = basis * s_eff (clomp.cpp:95), n x B row-major, support-restricted like
 * residual() (exact zeros add nothing to the sequential sums). */
static void synth(const problem_t* p, const double* s, const support_t* sup, double* x) {
  const int64_t n = p->n, B = p->batch;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t b = 0; b < B; ++b) {
      double acc = 0.0;
      for (int64_t q = 0; q < sup[b].count; ++q) {
        const int64_t j = sup[b].idx[q];
        acc = mac(acc, p->basis[i * n + j], s[j * B + b], p->isa);
      }
      x[i * B + b] = acc;
    }
}

/* tv_1d (priors.cpp:11-26): mean squared forward difference and its gradient. */
static double tv_1d(const double* x, int64_t n, double* grad) {
  if (grad)
    for (int64_t i = 0; i < n; ++i) grad[i] = 0.0;
  if (n < 2) return 0.0;
  const double inv_n = 1.0 / (double)n;
  double acc = 0.0;
  for (int64_t j = 0; j + 1 < n; ++j) {
    const double d = x[j] - x[j + 1];
    acc += d * d;
    if (grad) {
      grad[j] += 2.0 * inv_n * d;
      grad[j + 1] -= 2.0 * inv_n * d;
    }
  }
  return acc * inv_n;
}

/* tv_2d (priors.cpp:28-59) of an h x w image (row-major): vertical and
 * horizontal squared differences, each averaged over its own extent. */
static double tv_2d(const double* x, int64_t h, int64_t w, double* grad) {
  if (grad)
    for (int64_t e = 0; e < h * w; ++e) grad[e] = 0.0;
  double acc = 0.0;
  if (h >= 2) {
    const double inv_h = 1.0 / (double)h;
    for (int64_t i = 0; i + 1 < h; ++i)
      for (int64_t j = 0; j < w; ++j) {
        const double d = x[i * w + j] - x[(i + 1) * w + j];
        acc += inv_h * d * d;
        if (grad) {
          grad[i * w + j] += 2.0 * inv_h * d;
          grad[(i + 1) * w + j] -= 2.0 * inv_h * d;
        }
      }
  }
  if (w >= 2) {
    const double inv_w = 1.0 / (double)w;
    for (int64_t i = 0; i < h; ++i)
      for (int64_t j = 0; j + 1 < w; ++j) {
        const double d = x[i * w + j] - x[i * w + j + 1];
        acc += inv_w * d * d;
        if (grad) {
          grad[i * w + j] += 2.0 * inv_w * d;
          grad[i * w + j + 1] -= 2.0 * inv_w * d;
        }
      }
  }
  return acc;
}

/* Window origins along one axis (priors.cpp:63-70): every stride, plus the
 * last full window if the stride missed it. */
static int64_t block_starts(int64_t dim, int64_t window, int64_t stride, int64_t* out) {
  int64_t cnt = 0;
  for (int64_t s0 = 0; s0 + window <= dim; s0 += stride) out[cnt++] = s0;
  const int64_t last = dim - window;
  if (cnt == 0 || out[cnt - 1] != last) out[cnt++] = last;
  return cnt;
}

/* local_variance (priors.cpp:74-116): mean over windows of the standard
 * deviation, with its gradient.  Parameters are validated by the caller. */
static double local_variance(const double* x, int64_t h, int64_t w, int64_t window,
                             int64_t stride, double* grad) {
  if (grad)
    for (int64_t e = 0; e < h * w; ++e) grad[e] = 0.0;
  int64_t* rows = malloc((size_t)(h + 2) * sizeof(int64_t));
  int64_t* cols = malloc((size_t)(w + 2) * sizeof(int64_t));
  const int64_t nr = block_starts(h, window, stride, rows);
  const int64_t nc = block_starts(w, window, stride, cols);
  const double count = (double)(window * window);
  const double inv_blocks = 1.0 / (double)(nr * nc);
  double acc = 0.0;
  for (int64_t a = 0; a < nr; ++a)
    for (int64_t bb = 0; bb < nc; ++bb) {
      const int64_t r0 = rows[a], c0 = cols[bb];
      double sum = 0.0, sum_sq = 0.0;
      for (int64_t i = 0; i < window; ++i)
        for (int64_t j = 0; j < window; ++j) {
          const double v = x[(r0 + i) * w + c0 + j];
          sum += v;
          sum_sq += v * v;
        }
      const double mean = sum / count;
      double var = sum_sq / count - mean * mean;
      if (var < 0.0) var = 0.0; /* std::max(var, 0.0) */
      const double sd = sqrt(var);
      acc += inv_blocks * sd;
      if (grad && sd > 0.0) {
        const double scale = inv_blocks / (count * sd);
        for (int64_t i = 0; i < window; ++i)
          for (int64_t j = 0; j < window; ++j)
            grad[(r0 + i) * w + c0 + j] += scale * (x[(r0 + i) * w + c0 + j] - mean);
      }
    }
  free(rows);
  free(cols);
  return acc;
}

/* The prior part of loss_impl (clomp.cpp:93-119): returns w_tv tv + w_lv lv
 * as the reference adds it to lb.total (tv, lv returned through *tv, *lv);
 * with g != NULL adds the chained gradient D^T gx to g on the supports.
 * x, gv, gx: n x B scratch each. */
static void prior_eval(const problem_t* p, const double* s, const support_t* sup, double* g,
                       double* x, double* gv, double* gx, double* tv, double* lv) {
  const int64_t n = p->n, B = p->batch, nb = n * B;
  synth(p, s, sup, x);
  if (g)
    for (int64_t e = 0; e < nb; ++e) gx[e] = 0.0;
  *tv = 0.0;
  *lv = 0.0;
  if (p->w_tv > 0.0) {
    if (B == 1) {
      *tv = tv_1d(x, n, g ? gv : NULL);
      if (g)
        for (int64_t i = 0; i < n; ++i) gx[i] += p->w_tv * gv[i]; /* clomp.cpp:101 */
    } else {
      *tv = tv_2d(x, n, B, g ? gv : NULL);
      if (g) /* kern::axpy (kernels_avx2.cpp:80-92: FMA; scalar: mul + add) */
        for (int64_t e = 0; e < nb; ++e) gx[e] = mac(gx[e], p->w_tv, gv[e], p->isa);
    }
  }
  if (p->lv_on) {
    *lv = local_variance(x, n, B, p->lv_window, p->lv_stride, g ? gv : NULL);
    if (g)
      for (int64_t e = 0; e < nb; ++e) gx[e] = mac(gx[e], p->w_lv, gv[e], p->isa);
  }
  if (g) /* chain = matmul(dt, gx) (clomp.cpp:114-117) on the supports */
    for (int64_t b = 0; b < B; ++b)
      for (int64_t q = 0; q < sup[b].count; ++q) {
        const int64_t j = sup[b].idx[q];
        double acc = 0.0;
        for (int64_t i = 0; i < n; ++i) acc = mac(acc, p->dt[j * n + i], gx[i * B + b], p->isa);
        g[j * B + b] += acc;
      }
}

/* (A^T r)[j, b] for one atom j: la::matmul(ops.at, r) element (clomp.cpp:89, 245). */
static inline double corr(const problem_t* p, const double* r, int64_t j,
                          int64_t b) {
  const int64_t B = p->batch;
  double acc = 0.0;
  if (p->at) {
    const double* atrow = p->at + j * p->m;
    for (int64_t q = 0; q < p->m; ++q) acc = mac(acc, atrow[q], r[q * B + b], p->isa);
  } else {
    for (int64_t q = 0; q < p->m; ++q) acc = mac(acc, entry(p, q, j), r[q * B + b], p->isa);
  }
  return acc;
}

/* (A^T r)[j, b] for up to 8 atoms at once: the same per-element sequential
 * sums as corr() (each output's mac chain in k order), interleaved so the
 * independent chains overlap instead of waiting on one FMA latency each
 * (bit-identical; the oracle's cost at config 3 is these chains). */
static void corr8(const problem_t* p, const double* r, const int64_t* js, int cnt, int64_t b,
                  double* out) {
  if (!p->at || cnt < 8) {
    for (int u = 0; u < cnt; ++u) out[u] = corr(p, r, js[u], b);
    return;
  }
  const int64_t B = p->batch, m = p->m;
  const double* a[8];
  double acc[8];
  for (int u = 0; u < 8; ++u) {
    a[u] = p->at + js[u] * m;
    acc[u] = 0.0;
  }
  if (p->isa == ORC_ISA_AVX2) {
    for (int64_t q = 0; q < m; ++q) {
      const double rq = r[q * B + b];
      for (int u = 0; u < 8; ++u) acc[u] = fma(a[u][q], rq, acc[u]);
    }
  } else {
    for (int64_t q = 0; q < m; ++q) {
      const double rq = r[q * B + b];
      for (int u = 0; u < 8; ++u) acc[u] = acc[u] + a[u][q] * rq;
    }
  }
  for (int u = 0; u < 8; ++u) out[u] = acc[u];
}

/* inject_from_scores (clomp.cpp:41-53) on freshly computed scores.
 * Returns 1 if any mask bit flipped; records the fp64 top-2 for tracing. */
static int inject(const problem_t* p, const double* r, double th,
                  uint8_t* mask, support_t* sup, double* scores,
                  double* trace_row /* per column stride handled by caller */,
                  int64_t trace_stride) {
  const int64_t B = p->batch, n = p->n;
  int changed = 0;
  for (int64_t b = 0; b < B; ++b) {
    double cmax = 0.0, second = 0.0;
    int64_t arg = -1;
    for (int64_t j0 = 0; j0 < n; j0 += 8) {
      int64_t js[8];
      const int cnt = (int)(n - j0 < 8 ? n - j0 : 8);
      for (int u = 0; u < cnt; ++u) js[u] = j0 + u;
      corr8(p, r, js, cnt, b, scores + j0);
    }
    for (int64_t j = 0; j < n; ++j) {
      const double v = fabs(scores[j]);
      scores[j] = v;
      if (v > cmax) {
        second = cmax;
        cmax = v;
        arg = j;
      } else if (v > second) {
        second = v;
      }
    }
    /* std::max semantics: cmax = max(cmax, |s|) keeps the first maximum. */
    int64_t added = 0;
    if (cmax != 0.0) {
      const double cut = th * cmax;
      for (int64_t j = 0; j < n; ++j)
        if (scores[j] >= cut && !mask[j * B + b]) {
          mask[j * B + b] = 1;
          support_insert(&sup[b], j);
          ++added;
        }
    }
    if (added) changed = 1;
    if (trace_row) {
      double* t = trace_row + b * trace_stride;
      t[0] = (double)arg;
      t[1] = cmax;
      t[2] = second;
      t[3] = (double)added;
    }
  }
  return changed;
}

/* gradient_step (clomp.cpp:171-209) restricted to the entries whose mask bit
 * is set: unmasked entries have g == 0 and zero moments forever, so every
 * update on them is an exact no-op. */
static void step_support(double* s, double* m1, double* m2, const double* g,
                         const support_t* sup, int64_t B,
                         const orc_config* c, uint64_t* adam_steps) {
  switch (c->opt) {
    case 0:
      for (int64_t b = 0; b < B; ++b)
        for (int64_t q = 0; q < sup[b].count; ++q) {
          const int64_t e = sup[b].idx[q] * B + b;
          s[e] -= c->lr * g[e];
        }
      break;
    case 1:
      for (int64_t b = 0; b < B; ++b)
        for (int64_t q = 0; q < sup[b].count; ++q) {
          const int64_t e = sup[b].idx[q] * B + b;
          m1[e] = 0.9 * m1[e] + g[e];
          s[e] -= c->lr * m1[e];
        }
      break;
    case 2: {
      const double b1 = 0.9, b2 = 0.999, tiny = 1e-8;
      ++*adam_steps;
      const double bc1 = 1.0 - pow(b1, (double)*adam_steps);
      const double bc2 = 1.0 - pow(b2, (double)*adam_steps);
      for (int64_t b = 0; b < B; ++b)
        for (int64_t q = 0; q < sup[b].count; ++q) {
          const int64_t e = sup[b].idx[q] * B + b;
          const double gg = g[e];
          m1[e] = b1 * m1[e] + (1.0 - b1) * gg;
          m2[e] = b2 * m2[e] + (1.0 - b2) * gg * gg;
          const double mhat = m1[e] / bc1;
          const double vhat = m2[e] / bc2;
          s[e] -= c->lr * mhat / (sqrt(vhat) + tiny);
        }
      break;
    }
  }
}

/* ----------------------------------------------------------- batch solve */

static int solve_joint(const problem_t* p, const double* y, const orc_config* c,
                       double* s_out, uint8_t* mask_out, int64_t* iters_out,
                       double* rn_out, uint8_t* conv_out, double* trace,
                       int64_t trace_col_stride, char* err, int errlen) {
  const int64_t m = p->m, n = p->n, B = p->batch;
  const int64_t nb = n * B, mb = m * B;
  double* s = calloc((size_t)nb, sizeof(double));
  double* m1 = calloc((size_t)nb, sizeof(double));
  double* m2 = calloc((size_t)nb, sizeof(double));
  double* g = calloc((size_t)nb, sizeof(double));
  uint8_t* mask = calloc((size_t)nb, 1);
  double* best_s = calloc((size_t)nb, sizeof(double));
  uint8_t* best_mask = calloc((size_t)nb, 1);
  double* r = calloc((size_t)mb, sizeof(double));
  double* scores = calloc((size_t)n, sizeof(double));
  support_t* sup = calloc((size_t)B, sizeof(support_t));
  support_t* best_sup = calloc((size_t)B, sizeof(support_t));
  int64_t* sup_mem = calloc((size_t)(2 * nb), sizeof(int64_t));
  for (int64_t b = 0; b < B; ++b) {
    sup[b].idx = sup_mem + b * n;
    best_sup[b].idx = sup_mem + nb + b * n;
  }
  const int prior = p->w_tv > 0.0 || p->lv_on;
  double* px = prior ? calloc((size_t)(3 * nb), sizeof(double)) : NULL;
  double tvv = 0.0, lvv = 0.0;
  uint64_t adam_steps = 0;
  double best_loss = INFINITY, prev_loss = INFINITY;
  uint64_t stall = 0;
  int converged = 0, status = ORC_OK, have_best = 0;
  int64_t iterations = 0;

  for (uint64_t outer = 1; outer <= c->max_outer; ++outer) {
    residual(p, s, sup, y, r);
    const double rn = sqrt(sum_sq(r, mb, p->isa));
    if (rn < c->eps) {
      converged = 1;
      break;
    }
    double* trow = trace ? trace + (int64_t)(outer - 1) * 4 : NULL;
    const int mask_changed = inject(p, r, c->th, mask, sup, scores, trow,
                                    trace_col_stride);
    for (uint64_t step = 0; step < c->inner_steps; ++step) {
      /* loss_impl with grad (clomp.cpp:83-91, 120-123): the residual sum of
       * squares is computed and discarded there; it does not feed the step. */
      residual(p, s, sup, y, r);
      for (int64_t b = 0; b < B; ++b)
        for (int64_t q0 = 0; q0 < sup[b].count; q0 += 8) {
          const int cnt = (int)(sup[b].count - q0 < 8 ? sup[b].count - q0 : 8);
          double v[8];
          corr8(p, r, sup[b].idx + q0, cnt, b, v);
          for (int u = 0; u < cnt; ++u) g[sup[b].idx[q0 + u] * B + b] = v[u] * 2.0;
        }
      if (prior) prior_eval(p, s, sup, g, px, px + nb, px + 2 * nb, &tvv, &lvv);
      step_support(s, m1, m2, g, sup, B, c, &adam_steps);
    }
    residual(p, s, sup, y, r);
    double loss = sum_sq(r, mb, p->isa);
    if (prior) { /* lb.total = residual + w_tv tv + w_lv lv (clomp.cpp:126) */
      prior_eval(p, s, sup, NULL, px, NULL, NULL, &tvv, &lvv);
      loss = loss + p->w_tv * tvv + p->w_lv * lvv;
    }
    if (!isfinite(loss)) {
      set_err(err, errlen, "clomp: loss diverged; reduce lr");
      status = ORC_ERR_NUMERICAL;
      goto done;
    }
    iterations = (int64_t)outer;
    if (loss < best_loss) {
      best_loss = loss;
      memcpy(best_s, s, (size_t)nb * sizeof(double));
      memcpy(best_mask, mask, (size_t)nb);
      for (int64_t b = 0; b < B; ++b) {
        best_sup[b].count = sup[b].count;
        memcpy(best_sup[b].idx, sup[b].idx, (size_t)sup[b].count * sizeof(int64_t));
      }
      have_best = 1;
    }
    const double rel = isfinite(prev_loss)
                           ? (prev_loss - loss) / fmax(fabs(prev_loss), 1e-300)
                           : INFINITY;
    if (!mask_changed && rel < c->stall_tol)
      ++stall;
    else
      stall = 0;
    prev_loss = loss;
    if (stall >= c->stall_patience) break;
  }

  {
    const double* so = s;
    const uint8_t* mo = mask;
    const support_t* su = sup;
    if (!converged && isfinite(best_loss) && have_best) {
      so = best_s;
      mo = best_mask;
      su = best_sup;
    }
    /* Final residual (clomp.cpp:285-288). */
    residual(p, so, su, y, r);
    const double frn = sqrt(sum_sq(r, mb, p->isa));
    /* Unmasked entries of s are never written (gradient_step guards every
     * update with the mask), so they are exactly 0 here as in the reference. */
    memcpy(s_out, so, (size_t)nb * sizeof(double));
    memcpy(mask_out, mo, (size_t)nb);
    for (int64_t b = 0; b < B; ++b) {
      iters_out[b] = iterations;
      rn_out[b] = frn;
      conv_out[b] = frn < c->eps;
    }
  }
done:
  free(s); free(m1); free(m2); free(g); free(mask); free(best_s);
  free(best_mask); free(r); free(scores); free(sup); free(best_sup);
  free(sup_mem); free(px);
  return status;
}

static double* transpose(const double* a, int64_t m, int64_t n) {
  double* t = malloc((size_t)(m * n) * sizeof(double));
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) t[j * m + i] = a[i * n + j];
  return t;
}

/* Which priors loss_impl evaluates for this solve (clomp.cpp:93-119): TV-1D
 * on one column, TV-2D on a multi-column batch, local variance when the batch
 * and n fit its window, with local_variance's parameter checks
 * (priors.cpp:77-84), which the reference raises at its first loss
 * evaluation (reported here before the solve). */
static int prior_setup(problem_t* p, const orc_config* c, double w_tv, double w_lv,
                       int64_t batch, char* err, int errlen) {
  p->w_tv = 0.0;
  p->w_lv = 0.0;
  p->lv_on = 0;
  const int lv_fits = batch >= (int64_t)c->lv_window && p->n >= (int64_t)c->lv_window;
  if (!(w_tv > 0.0) && !(w_lv > 0.0 && lv_fits)) return ORC_OK;
  if (!p->basis) {
    set_err(err, errlen, "clomp oracle: priors need the synthesis basis");
    return ORC_ERR_UNSUPPORTED;
  }
  if (w_lv > 0.0 && lv_fits) {
    if (c->lv_window < 2) {
      set_err(err, errlen, "local_variance: window must be >= 2");
      return ORC_ERR_CONFIG;
    }
    if (c->lv_stride < 1 || c->lv_stride >= c->lv_window) {
      set_err(err, errlen, "local_variance: stride must be in [1, window)");
      return ORC_ERR_CONFIG;
    }
    p->lv_on = 1;
    p->w_lv = w_lv;
    p->lv_window = (int64_t)c->lv_window;
    p->lv_stride = (int64_t)c->lv_stride;
  }
  p->w_tv = w_tv > 0.0 ? w_tv : 0.0;
  return ORC_OK;
}

/* Shared driver: `proto` carries the operator (dense or separable). */
static int solve_driver(problem_t proto, const double* y, int64_t batch,
                        const orc_config* cfg, int mode, double* s_out,
                        uint8_t* mask_out, int64_t* iterations, double* final_rn,
                        uint8_t* converged, int32_t* status, double* trace,
                        char* err, int errlen) {
  const int64_t m = proto.m, n = proto.n;
  const int isa = proto.isa;
  int st = validate(cfg, err, errlen);
  if (st) return st;
  if (m <= 0 || n <= 0) {
    set_err(err, errlen, "clomp: empty operator");
    return ORC_ERR_DIMENSION;
  }
  if (batch <= 0) {
    set_err(err, errlen, "clomp: empty batch");
    return ORC_ERR_DIMENSION;
  }
  if (trace)
    for (int64_t e = 0; e < batch * (int64_t)cfg->max_outer * 4; ++e) trace[e] = -1.0;

  if (mode == ORC_MODE_JOINT) {
    double w_tv, w_lv;
    resolve_weights(cfg, y, m * batch, isa, &w_tv, &w_lv);
    problem_t p = proto;
    p.batch = batch;
    st = prior_setup(&p, cfg, w_tv, w_lv, batch, err, errlen);
    if (st == ORC_OK)
      st = solve_joint(&p, y, cfg, s_out, mask_out, iterations, final_rn,
                       converged, trace, (int64_t)cfg->max_outer * 4, err, errlen);
    for (int64_t b = 0; b < batch; ++b) status[b] = st;
    return st;
  }

  /* PER_SIGNAL: clomp_solve on every column (clomp.cpp:294-311). */
  double* yc = malloc((size_t)m * sizeof(double));
  double* sc = malloc((size_t)n * sizeof(double));
  uint8_t* mc = malloc((size_t)n);
  for (int64_t b = 0; b < batch; ++b) {
    for (int64_t i = 0; i < m; ++i) yc[i] = y[i * batch + b];
    double w_tv, w_lv;
    resolve_weights(cfg, yc, m, isa, &w_tv, &w_lv);
    int sb;
    int64_t it = 0;
    double rn = 0.0;
    uint8_t cv = 0;
    problem_t p = proto;
    p.batch = 1;
    sb = prior_setup(&p, cfg, w_tv, w_lv, 1, NULL, 0);
    if (sb == ORC_OK)
      sb = solve_joint(&p, yc, cfg, sc, mc, &it, &rn, &cv,
                       trace ? trace + b * (int64_t)cfg->max_outer * 4 : NULL,
                       4, NULL, 0);
    status[b] = sb;
    if (sb != ORC_OK) {
      for (int64_t j = 0; j < n; ++j) {
        s_out[j * batch + b] = 0.0;
        mask_out[j * batch + b] = 0;
      }
      iterations[b] = 0;
      final_rn[b] = NAN;
      converged[b] = 0;
      continue;
    }
    for (int64_t j = 0; j < n; ++j) {
      s_out[j * batch + b] = sc[j];
      mask_out[j * batch + b] = mc[j];
    }
    iterations[b] = it;
    final_rn[b] = rn;
    converged[b] = cv;
  }
  free(yc); free(sc); free(mc);
  return ORC_OK;
}

int orc_clomp_solve_batch_basis(const double* a, int64_t m, int64_t n,
                                const double* basis, const double* y, int64_t batch,
                                const orc_config* cfg, int isa, int mode,
                                double* s_out, uint8_t* mask_out,
                                int64_t* iterations, double* final_rn,
                                uint8_t* converged, int32_t* status, double* trace,
                                char* err, int errlen) {
  if (m <= 0 || n <= 0) {
    set_err(err, errlen, "clomp: empty operator");
    return ORC_ERR_DIMENSION;
  }
  double* at = transpose(a, m, n);
  double* dt = basis ? transpose(basis, n, n) : NULL;
  problem_t p = {a, at, m, n, batch, isa, NULL, NULL, 0, 0, 0, 0, basis, dt, 0.0, 0.0, 0, 0, 0};
  const int st = solve_driver(p, y, batch, cfg, mode, s_out, mask_out, iterations,
                              final_rn, converged, status, trace, err, errlen);
  free(at);
  free(dt);
  return st;
}

int orc_clomp_solve_batch(const double* a, int64_t m, int64_t n,
                          const double* y, int64_t batch,
                          const orc_config* cfg, int isa, int mode,
                          double* s_out, uint8_t* mask_out,
                          int64_t* iterations, double* final_rn,
                          uint8_t* converged, int32_t* status, double* trace,
                          char* err, int errlen) {
  return orc_clomp_solve_batch_basis(a, m, n, NULL, y, batch, cfg, isa, mode, s_out,
                                     mask_out, iterations, final_rn, converged, status,
                                     trace, err, errlen);
}

int orc_clomp_solve_sep(const double* ar, int64_t mr, int64_t nr,
                        const double* ac, int64_t mc, int64_t nc,
                        const double* y, int64_t batch, const orc_config* cfg,
                        int isa, int mode, double* s_out, uint8_t* mask_out,
                        int64_t* iterations, double* final_rn, uint8_t* converged,
                        int32_t* status, double* trace, char* err, int errlen) {
  problem_t p = {NULL, NULL, mr * mc, nr * nc, batch, isa, ar, ac, mr, nr, mc, nc,
                 NULL, NULL, 0.0, 0.0, 0, 0, 0};
  return solve_driver(p, y, batch, cfg, mode, s_out, mask_out, iterations, final_rn,
                      converged, status, trace, err, errlen);
}

/* ------------------------------------------------------ unit entry points */

int orc_inject_support(const double* a, int64_t m, int64_t n, const double* r,
                       int64_t batch, double th, int isa, uint8_t* mask) {
  if (!(th > 0.0) || th > 1.0) return ORC_ERR_CONFIG;
  double* at = transpose(a, m, n);
  problem_t p = {a, at, m, n, batch, isa, NULL, NULL, 0, 0, 0, 0, NULL, NULL, 0.0, 0.0, 0, 0, 0};
  support_t* sup = calloc((size_t)batch, sizeof(support_t));
  int64_t* mem = calloc((size_t)(n * batch), sizeof(int64_t));
  for (int64_t b = 0; b < batch; ++b) {
    sup[b].idx = mem + b * n;
    for (int64_t j = 0; j < n; ++j)
      if (mask[j * batch + b]) sup[b].idx[sup[b].count++] = j;
  }
  double* scores = malloc((size_t)n * sizeof(double));
  inject(&p, r, th, mask, sup, scores, NULL, 0);
  free(scores); free(mem); free(sup); free(at);
  return ORC_OK;
}

int orc_clomp_loss(const double* a, int64_t m, int64_t n, const double* y,
                   int64_t batch, const double* s, const uint8_t* mask,
                   const orc_config* cfg, int isa, double* loss,
                   double* grad) {
  int st = validate(cfg, NULL, 0);
  if (st) return st;
  double w_tv, w_lv;
  resolve_weights(cfg, y, m * batch, isa, &w_tv, &w_lv);
  if (w_tv > 0.0 || w_lv > 0.0) return ORC_ERR_UNSUPPORTED;
  double* at = transpose(a, m, n);
  problem_t p = {a, at, m, n, batch, isa, NULL, NULL, 0, 0, 0, 0, NULL, NULL, 0.0, 0.0, 0, 0, 0};
  support_t* sup = calloc((size_t)batch, sizeof(support_t));
  int64_t* mem = calloc((size_t)(n * batch), sizeof(int64_t));
  for (int64_t b = 0; b < batch; ++b) {
    sup[b].idx = mem + b * n;
    for (int64_t j = 0; j < n; ++j)
      if (mask[j * batch + b]) sup[b].idx[sup[b].count++] = j;
  }
  double* r = malloc((size_t)(m * batch) * sizeof(double));
  residual(&p, s, sup, y, r);
  *loss = sum_sq(r, m * batch, isa);
  if (grad) {
    for (int64_t j = 0; j < n; ++j)
      for (int64_t b = 0; b < batch; ++b)
        grad[j * batch + b] = mask[j * batch + b] ? corr(&p, r, j, b) * 2.0 : 0.0;
  }
  free(r); free(mem); free(sup); free(at);
  return ORC_OK;
}

int orc_gradient_step(double* s, const uint8_t* mask, double* m1, double* m2,
                      uint64_t* adam_steps, const double* grad, int64_t total,
                      const orc_config* cfg) {
  if (!(cfg->lr > 0.0)) return ORC_ERR_CONFIG;
  switch (cfg->opt) {
    case 0:
      for (int64_t i = 0; i < total; ++i)
        if (mask[i]) s[i] -= cfg->lr * grad[i];
      break;
    case 1:
      for (int64_t i = 0; i < total; ++i) {
        m1[i] = 0.9 * m1[i] + grad[i];
        if (mask[i]) s[i] -= cfg->lr * m1[i];
      }
      break;
    case 2: {
      const double b1 = 0.9, b2 = 0.999, tiny = 1e-8;
      ++*adam_steps;
      const double bc1 = 1.0 - pow(b1, (double)*adam_steps);
      const double bc2 = 1.0 - pow(b2, (double)*adam_steps);
      for (int64_t i = 0; i < total; ++i) {
        const double g = grad[i];
        m1[i] = b1 * m1[i] + (1.0 - b1) * g;
        m2[i] = b2 * m2[i] + (1.0 - b2) * g * g;
        if (mask[i]) {
          const double mhat = m1[i] / bc1;
          const double vhat = m2[i] / bc2;
          s[i] -= cfg->lr * mhat / (sqrt(vhat) + tiny);
        }
      }
      break;
    }
    default:
      return ORC_ERR_CONFIG;
  }
  return ORC_OK;
}

/* ------------------------------------------- separable, Gram form (fast)
 * The same per-signal loop (clomp.cpp:235-291, B = 1 semantics) with the
 * separable operator, for full-size 2D parity where the matrix-free exact
 * restatement above is infeasible (config 4: K = 1500, 16384 x 65536).
 * Products are regrouped, so results are the fp64 loop's up to summation
 * order (not bit-exact with the reference; pinned against orc_clomp_solve_sep
 * on prefixes by tests/test_oracle.py):
 *   residual  R = A_r C A_c^T - Y through V = A_r C (C sparse, m_r x n_c);
 *   scores    S = A_r^T R A_c (n_r x n_c), atom p = i + n_r j;
 *   epochs    g_S = 2 (G_S c - b_S) with G_S[k][l] = Gr[i_k][i_l] Gc[j_k][j_l]
 *             (Gr = A_r^T A_r, Gc = A_c^T A_c) and b = A_r^T Y A_c, which
 *             equals 2 A_S^T (A_S c - y) (clomp.cpp:87-91) in exact arithmetic. */
static void sep_residual(const double* ar, int64_t mr, int64_t nr, const double* ac, int64_t mc,
                         int64_t nc, const support_t* sup, const double* s, const double* y,
                         double* v, double* r) {
  for (int64_t e = 0; e < mr * nc; ++e) v[e] = 0.0;
  for (int64_t q = 0; q < sup->count; ++q) {
    const int64_t pidx = sup->idx[q], i = pidx % nr, j = pidx / nr;
    const double c = s[pidx];
    for (int64_t qr = 0; qr < mr; ++qr) v[qr * nc + j] += ar[qr * nr + i] * c;
  }
  for (int64_t qc = 0; qc < mc; ++qc)
    for (int64_t qr = 0; qr < mr; ++qr) {
      const double* vr = v + qr * nc;
      const double* acr = ac + qc * nc;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int64_t j = 0;
      for (; j + 4 <= nc; j += 4) {
        a0 += vr[j] * acr[j];
        a1 += vr[j + 1] * acr[j + 1];
        a2 += vr[j + 2] * acr[j + 2];
        a3 += vr[j + 3] * acr[j + 3];
      }
      for (; j < nc; ++j) a0 += vr[j] * acr[j];
      r[qr + mr * qc] = ((a0 + a1) + (a2 + a3)) - y[qr + mr * qc];
    }
}

/* out (n_r x n_c, p = i + n_r j) = A_r^T Rm A_c with Rm[qr][qc] = r[qr + m_r qc].
 * u: scratch of n_r m_c + m_r m_c + n_r n_c doubles. */
static void sep_corr(const double* ar, int64_t mr, int64_t nr, const double* ac, int64_t mc,
                     int64_t nc, const double* r, double* u, double* out) {
  double* rm = u + nr * mc;       /* Rm row-major (m_r x m_c) */
  double* o2 = rm + mr * mc;      /* A_r^T Rm A_c row-major (n_r x n_c) */
  for (int64_t qc = 0; qc < mc; ++qc)
    for (int64_t qr = 0; qr < mr; ++qr) rm[qr * mc + qc] = r[qr + mr * qc];
  for (int64_t e = 0; e < nr * mc; ++e) u[e] = 0.0;  /* U = A_r^T Rm  (n_r x m_c) */
  for (int64_t qr = 0; qr < mr; ++qr)
    for (int64_t i = 0; i < nr; ++i) {
      const double a = ar[qr * nr + i];
      double* ur = u + i * mc;
      const double* rr = rm + qr * mc;
      for (int64_t qc = 0; qc < mc; ++qc) ur[qc] += a * rr[qc];
    }
  for (int64_t e = 0; e < nr * nc; ++e) o2[e] = 0.0;
  for (int64_t i = 0; i < nr; ++i)
    for (int64_t qc = 0; qc < mc; ++qc) {
      const double uq = u[i * mc + qc];
      const double* acr = ac + qc * nc;
      double* orow = o2 + i * nc;
      for (int64_t j = 0; j < nc; ++j) orow[j] += uq * acr[j];
    }
  for (int64_t i = 0; i < nr; ++i)
    for (int64_t j = 0; j < nc; ++j) out[i + nr * j] = o2[i * nc + j];
}

static double dot4(const double* a, const double* b, int64_t n) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int64_t k = 0;
  for (; k + 4 <= n; k += 4) {
    a0 += a[k] * b[k];
    a1 += a[k + 1] * b[k + 1];
    a2 += a[k + 2] * b[k + 2];
    a3 += a[k + 3] * b[k + 3];
  }
  for (; k < n; ++k) a0 += a[k] * b[k];
  return (a0 + a1) + (a2 + a3);
}

static int sep_gram_one(const double* ar, int64_t mr, int64_t nr, const double* ac, int64_t mc,
                        int64_t nc, const double* gr, const double* gc, const double* y,
                        const orc_config* c, double* s_out, uint8_t* mask_out, int64_t* it_out,
                        double* rn_out, uint8_t* cv_out) {
  const int64_t n = nr * nc, m = mr * mc;
  int64_t cap = (int64_t)c->max_outer + 64;
  if (c->th < 1.0 || cap > n) cap = n;
  double* s = calloc((size_t)n, sizeof(double));
  double* m1 = calloc((size_t)n, sizeof(double));
  double* m2 = calloc((size_t)n, sizeof(double));
  double* g = calloc((size_t)n, sizeof(double));
  double* best_s = calloc((size_t)n, sizeof(double));
  uint8_t* mask = calloc((size_t)n, 1);
  uint8_t* best_mask = calloc((size_t)n, 1);
  double* zb = malloc((size_t)n * sizeof(double));
  double* sc = malloc((size_t)n * sizeof(double));
  double* v = malloc((size_t)(mr * nc) * sizeof(double));
  double* u = malloc((size_t)(nr * mc + mr * mc + nr * nc) * sizeof(double));
  double* r = malloc((size_t)m * sizeof(double));
  int64_t* idx = malloc((size_t)n * sizeof(int64_t));
  int64_t* bidx = malloc((size_t)n * sizeof(int64_t));
  double* G = NULL;
  double* cs = malloc((size_t)cap * sizeof(double));
  double* bs = malloc((size_t)cap * sizeof(double));
  support_t sup = {idx, 0}, best_sup = {bidx, 0};
  int status = ORC_OK, converged = 0, have_best = 0;
  int64_t iterations = 0, gdim = -1;
  uint64_t adam_steps = 0, stall = 0;
  double best_loss = INFINITY, prev_loss = INFINITY;
  sep_corr(ar, mr, nr, ac, mc, nc, y, u, zb);  /* b = A^T y of every atom */
  for (uint64_t outer = 1; outer <= c->max_outer; ++outer) {
    sep_residual(ar, mr, nr, ac, mc, nc, &sup, s, y, v, r);
    if (sqrt(dot4(r, r, m)) < c->eps) {
      converged = 1;
      break;
    }
    sep_corr(ar, mr, nr, ac, mc, nc, r, u, sc);
    double cmax = 0.0;
    for (int64_t p = 0; p < n; ++p) {
      sc[p] = fabs(sc[p]);
      if (sc[p] > cmax) cmax = sc[p];
    }
    int changed = 0;
    if (cmax != 0.0) {
      const double cut = c->th * cmax;
      for (int64_t p = 0; p < n; ++p)
        if (sc[p] >= cut && !mask[p]) {
          if (sup.count >= cap) { status = ORC_ERR_DIMENSION; goto done; }
          mask[p] = 1;
          support_insert(&sup, p);
          changed = 1;
        }
    }
    const int64_t t = sup.count;
    if (t != gdim) {  /* support (sorted) changed: rebuild G_S and b_S */
      free(G);
      G = malloc((size_t)(t * t) * sizeof(double));
      for (int64_t k = 0; k < t; ++k) {
        const int64_t ik = idx[k] % nr, jk = idx[k] / nr;
        for (int64_t l = 0; l < t; ++l) {
          const int64_t il = idx[l] % nr, jl = idx[l] / nr;
          G[k * t + l] = gr[ik * nr + il] * gc[jk * nc + jl];
        }
        bs[k] = zb[idx[k]];
      }
      gdim = t;
    }
    for (int64_t k = 0; k < t; ++k) cs[k] = s[idx[k]];
    for (uint64_t step = 0; step < c->inner_steps; ++step) {
      for (int64_t k = 0; k < t; ++k) g[idx[k]] = 2.0 * (dot4(G + k * t, cs, t) - bs[k]);
      step_support(s, m1, m2, g, &sup, 1, c, &adam_steps);
      for (int64_t k = 0; k < t; ++k) cs[k] = s[idx[k]];
    }
    sep_residual(ar, mr, nr, ac, mc, nc, &sup, s, y, v, r);
    const double loss = dot4(r, r, m);
    if (!isfinite(loss)) { status = ORC_ERR_NUMERICAL; goto done; }
    iterations = (int64_t)outer;
    if (loss < best_loss) {
      best_loss = loss;
      memcpy(best_s, s, (size_t)n * sizeof(double));
      memcpy(best_mask, mask, (size_t)n);
      best_sup.count = sup.count;
      memcpy(bidx, idx, (size_t)sup.count * sizeof(int64_t));
      have_best = 1;
    }
    const double rel = isfinite(prev_loss) ? (prev_loss - loss) / fmax(fabs(prev_loss), 1e-300)
                                           : INFINITY;
    stall = (!changed && rel < c->stall_tol) ? stall + 1 : 0;
    prev_loss = loss;
    if (stall >= c->stall_patience) break;
  }
  {
    const double* so = s;
    const uint8_t* mo = mask;
    const support_t* su = &sup;
    if (!converged && isfinite(best_loss) && have_best) {
      so = best_s;
      mo = best_mask;
      su = &best_sup;
    }
    sep_residual(ar, mr, nr, ac, mc, nc, su, so, y, v, r);
    *rn_out = sqrt(dot4(r, r, m));
    *cv_out = *rn_out < c->eps;
    *it_out = iterations;
    memcpy(s_out, so, (size_t)n * sizeof(double));
    memcpy(mask_out, mo, (size_t)n);
  }
done:
  free(s); free(m1); free(m2); free(g); free(best_s); free(mask); free(best_mask);
  free(zb); free(sc); free(v); free(u); free(r); free(idx); free(bidx); free(G);
  free(cs); free(bs);
  return status;
}

int orc_clomp_solve_sep_gram(const double* ar, int64_t mr, int64_t nr, const double* ac,
                             int64_t mc, int64_t nc, const double* y, int64_t batch,
                             const orc_config* cfg, double* s_out, uint8_t* mask_out,
                             int64_t* iterations, double* final_rn, uint8_t* converged,
                             int32_t* status, char* err, int errlen) {
  int st = validate(cfg, err, errlen);
  if (st) return st;
  if (mr <= 0 || nr <= 0 || mc <= 0 || nc <= 0 || batch <= 0) {
    set_err(err, errlen, "clomp: empty operator or batch");
    return ORC_ERR_DIMENSION;
  }
  const int64_t n = nr * nc, m = mr * mc;
  double* gr = malloc((size_t)(nr * nr) * sizeof(double));
  double* gc = malloc((size_t)(nc * nc) * sizeof(double));
  for (int64_t i = 0; i < nr; ++i)
    for (int64_t k = 0; k < nr; ++k) {
      double acc = 0.0;
      for (int64_t q = 0; q < mr; ++q) acc += ar[q * nr + i] * ar[q * nr + k];
      gr[i * nr + k] = acc;
    }
  for (int64_t j = 0; j < nc; ++j)
    for (int64_t k = 0; k < nc; ++k) {
      double acc = 0.0;
      for (int64_t q = 0; q < mc; ++q) acc += ac[q * nc + j] * ac[q * nc + k];
      gc[j * nc + k] = acc;
    }
  double* yc = malloc((size_t)m * sizeof(double));
  double* sc = malloc((size_t)n * sizeof(double));
  uint8_t* mk = malloc((size_t)n);
  for (int64_t b = 0; b < batch; ++b) {
    for (int64_t q = 0; q < m; ++q) yc[q] = y[q * batch + b];
    int64_t it = 0;
    double rn = 0.0;
    uint8_t cv = 0;
    status[b] = sep_gram_one(ar, mr, nr, ac, mc, nc, gr, gc, yc, cfg, sc, mk, &it, &rn, &cv);
    for (int64_t p = 0; p < n; ++p) {
      s_out[p * batch + b] = status[b] ? 0.0 : sc[p];
      mask_out[p * batch + b] = status[b] ? 0 : mk[p];
    }
    iterations[b] = status[b] ? 0 : it;
    final_rn[b] = status[b] ? NAN : rn;
    converged[b] = status[b] ? 0 : cv;
  }
  free(gr); free(gc); free(yc); free(sc); free(mk);
  return ORC_OK;
}
