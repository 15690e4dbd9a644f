/*
 * clomp_oracle.h — CPU restatement of the reference CLOMP reconstruction loop.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or the timed CPU baseline.  The product path
 * (libclomp_b200.so) never links, loads or calls it.
 *
 * Parity: pinned bit-for-bit against the unmodified reference library
 * (oracle/_ref/libcskit_ref.so, compiled from /root/reference/proj/src) by the
 * fixtures in tests/golden/ (see tests/golden/make_golden.py).
 *
 * The config struct has exactly the layout of cl_config in
 * include/clomp_b200.h so one ctypes Structure serves both.
 */
#ifndef CLOMP_ORACLE_H
#define CLOMP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_config {
  double th;                /* clomp.hpp:17 */
  uint64_t max_outer;       /* clomp.hpp:18 */
  double eps;               /* clomp.hpp:19 */
  uint64_t inner_steps;     /* clomp.hpp:20 */
  double lr;                /* clomp.hpp:21 */
  int32_t opt;              /* clomp.hpp:22 — 0 plain, 1 momentum, 2 adam */
  int32_t pad0;
  double w_tv;              /* clomp.hpp:25 */
  double w_lv;              /* clomp.hpp:26 */
  uint64_t lv_window;       /* priors.hpp:23 */
  uint64_t lv_stride;       /* priors.hpp:24 */
  double stall_tol;         /* clomp.hpp:31 */
  uint64_t stall_patience;  /* clomp.hpp:32 */
} orc_config;

enum {
  ORC_OK = 0,
  ORC_ERR_CONFIG = 2,      /* cskit::ConfigError    (errors.hpp:22) */
  ORC_ERR_DIMENSION = 3,   /* cskit::DimensionError (errors.hpp:16) */
  ORC_ERR_NUMERICAL = 4,   /* cskit::NumericalError (errors.hpp:28) */
  ORC_ERR_UNSUPPORTED = 5  /* priors without a synthesis basis */
};

/* Kernel semantics to reproduce: 1 = kernels_avx2.cpp (FMA), 0 = kernels_scalar.cpp. */
enum { ORC_ISA_SCALAR = 0, ORC_ISA_AVX2 = 1 };

/* Solve semantics: JOINT = clomp_solve_batch (clomp.cpp:211-292) with batch-global
 * eps / stall / best-iterate; PER_SIGNAL = clomp_solve (clomp.cpp:294-311) applied
 * to every column independently. */
enum { ORC_MODE_JOINT = 0, ORC_MODE_PER_SIGNAL = 1 };

/*
 * a: m x n row-major (reference la::Mat layout); y: m x B row-major.
 * Outputs (caller-owned):
 *   s_out     n x B row-major coefficients (the returned snapshot, masked)
 *   mask_out  n x B
 *   iterations[B], final_rn[B], converged[B], status[B]   (JOINT: all equal)
 *   trace (optional, may be NULL): B x max_outer x 4 doubles
 *         {argmax index, top1 |score|, top2 |score|, atoms added}, -1 if not run
 * Returns the call status (JOINT: the exception the reference would throw;
 * PER_SIGNAL: ORC_OK unless the config/dimensions are invalid).
 */
int orc_clomp_solve_batch(const double* a, int64_t m, int64_t n,
                          const double* y, int64_t batch,
                          const orc_config* cfg, int isa, int mode,
                          double* s_out, uint8_t* mask_out,
                          int64_t* iterations, double* final_rn,
                          uint8_t* converged, int32_t* status, double* trace,
                          char* err, int errlen);

/* Same with the synthesis basis D (n x n row-major, x = D s; NULL = none), which
 * the priors need (clomp.cpp:93-119): TV-1D (priors.cpp:11-26) on one column,
 * TV-2D (priors.cpp:28-59) and local variance (priors.cpp:74-116) on a
 * multi-column batch, chained through D^T. */
int orc_clomp_solve_batch_basis(const double* a, int64_t m, int64_t n,
                                const double* basis, const double* y, int64_t batch,
                                const orc_config* cfg, int isa, int mode,
                                double* s_out, uint8_t* mask_out,
                                int64_t* iterations, double* final_rn,
                                uint8_t* converged, int32_t* status, double* trace,
                                char* err, int errlen);

/* Separable 2D operator A = A_c (x) A_r with column-major vec (atom
 * p = i + n_r j, measurement q = qr + m_r qc): exactly clomp_solve(_batch) run
 * on the explicit Kronecker matrix with entries A_c[qc][j] * A_r[qr][i]
 * (the reference has no separable mode).  ar: m_r x n_r,
 * ac: m_c x n_c row-major; y: (m_r m_c) x B. */
int orc_clomp_solve_sep(const double* ar, int64_t mr, int64_t nr,
                        const double* ac, int64_t mc, int64_t nc,
                        const double* y, int64_t batch, const orc_config* cfg,
                        int isa, int mode, double* s_out, uint8_t* mask_out,
                        int64_t* iterations, double* final_rn, uint8_t* converged,
                        int32_t* status, double* trace, char* err, int errlen);

/* The separable per-signal loop in Gram form (products regrouped, fp64):
 * full-size 2D parity where the exact matrix-free restatement is too slow.
 * Per-signal semantics only; status[b] per signal. */
int orc_clomp_solve_sep_gram(const double* ar, int64_t mr, int64_t nr, const double* ac,
                             int64_t mc, int64_t nc, const double* y, int64_t batch,
                             const orc_config* cfg, double* s_out, uint8_t* mask_out,
                             int64_t* iterations, double* final_rn, uint8_t* converged,
                             int32_t* status, char* err, int errlen);

/* inject_support (clomp.cpp:142-154): mask |= thresholded |A^T r| per column. */
int orc_inject_support(const double* a, int64_t m, int64_t n, const double* r,
                       int64_t batch, double th, int isa, uint8_t* mask);

/* clomp_loss (clomp.cpp:156-169) restricted to w_tv = w_lv = 0:
 * returns the residual sum of squares in *loss, the masked gradient in grad
 * (n x B, may be NULL). */
int orc_clomp_loss(const double* a, int64_t m, int64_t n, const double* y,
                   int64_t batch, const double* s, const uint8_t* mask,
                   const orc_config* cfg, int isa, double* loss,
                   double* grad);

/* gradient_step (clomp.cpp:171-209) on a dense state of `total` entries. */
int orc_gradient_step(double* s, const uint8_t* mask, double* m1, double* m2,
                      uint64_t* adam_steps, const double* grad, int64_t total,
                      const orc_config* cfg);

#ifdef __cplusplus
}
#endif

#endif
