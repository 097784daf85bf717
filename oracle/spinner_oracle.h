/* CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, fp64 restatement of the reference's structured-spinner hot path
 * (arxiv 1610.06209 reference code, /root/reference/proj).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this; the
 * product (paper_1610_06209_b200/) never links or calls it.
 *
 * Parity of this restatement is pinned two ways (tests/test_oracle.py):
 *   1. the reference's own known-answer tests, restated
 *      (proj/tests/test_transforms.cpp:11-21,109-114, test_lsh.cpp:26-35, ...);
 *   2. bit-exact comparison against the reference sources themselves compiled
 *      into oracle/_ref (tests/golden/*.npz made by tests/golden/make_golden.py).
 * Builder-defined semantics that the reference lacks (SURVEY.md §8(a) row a14:
 * random-P sampler, all-Gaussian diagonals, ReLU, multi-table seeding, int32 ids)
 * are pinned only by this file + the shared host generator ("parity unpinned").
 */
#ifndef SPINNER_ORACLE_H
#define SPINNER_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* variants: 0 = HD3HD2HD1 (Rademacher), 1 = HDgHD2HD1 (Gaussian last diagonal),
 * 100 = builder-defined all-Gaussian D1..D3 (config 5). */
enum { ORC_HD3 = 0, ORC_HDG = 1, ORC_GAUSS3 = 100 };

uint64_t orc_mix_seed(uint64_t base, uint64_t stream);          /* common.hpp:51-56 */

typedef struct {
  uint64_t mt[312];
  int mti;
  int have_spare;
  double spare;
} orc_rng;
void orc_rng_init(orc_rng* r, uint64_t seed);                     /* common.hpp:64 */
uint64_t orc_rng_next(orc_rng* r);                                /* std::mt19937_64 */
double orc_rng_uniform01(orc_rng* r);                             /* common.hpp:68-70 */
double orc_rng_gaussian(orc_rng* r);                              /* common.hpp:72-84 */
double orc_rng_rademacher(orc_rng* r);                            /* common.hpp:86 */
void orc_rng_fill(uint64_t seed, int kind, int64_t count, double* out);

/* One block's realised diagonals (spinner.cpp:137-151, draw_tail :92-106). */
void orc_realize_block(int variant, int64_t n, uint64_t spec_seed, double* d1, double* d2,
                       double* d3);
/* StackedSpinner(v,n,m,k,seed): ceil(k/m) blocks, block b seed mix_seed(seed,b)
 * (spinner.cpp:248-256).  Arrays are [blocks][n]. Returns block count. */
int64_t orc_realize_stacked(int variant, int64_t n, int64_t m, int64_t k, uint64_t seed,
                            double* d1, double* d2, double* d3);
double orc_default_scale(int variant, int64_t n);                 /* spinner.cpp:41-45 */

void orc_fwht_normalized(double* x, int64_t n);                   /* transforms.cpp:52-71 */

/* y[0..m) = scale * first_m(H D3 H D2 H D1 x)   (spinner.cpp:186-231). */
void orc_block_apply(int64_t n, int64_t m, double scale, const double* d1, const double* d2,
                     const double* d3, const double* x, double* y);
/* StackedSpinner::apply (spinner.cpp:272-283): y[0..k). */
void orc_stacked_apply(int64_t n, int64_t m, int64_t k, double scale, const double* d1,
                       const double* d2, const double* d3, const double* x, double* y);

/* signed_argmax (lsh.cpp:9-21): strict '>' scan, sign = y<0 ? -1 : +1. */
void orc_signed_argmax(const double* y, int64_t len, int64_t* index, int* sign);
/* second-largest |y| relative gap, for near-tie accounting. */
double orc_top2_gap(const double* y, int64_t len);

/* ---- batch entry points over fp32 row-major inputs (promoted exactly to fp64) ---- */
/* rows are x[b*ld + i], i < n_in, zero padded to n (dataset.cpp:162-168). */
void orc_batch_apply(int64_t n, int64_t m, int64_t k, double scale, const double* d1,
                     const double* d2, const double* d3, const float* x, int64_t batch, int64_t ld,
                     int64_t n_in, int relu, double* y /* [batch][k] */);
/* CrossPolytopeHasher::hash for `tables` tables of k rows each; diagonals are
 * [tables][blocks][n].  ids = index + (sign<0 ? k : 0); gaps = top-2 relative gap. */
void orc_batch_hash(int64_t n, int64_t m, int64_t k, int64_t tables, double scale,
                    const double* d1, const double* d2, const double* d3, const float* x,
                    int64_t batch, int64_t ld, int64_t n_in, int32_t* ids /* [batch][tables] */,
                    double* gaps /* [batch][tables] or NULL */);
/* embed (kernels.cpp:17-36).  kind 0 = gaussian -> [batch][2k]; 1 = angular -> [batch][k]. */
void orc_batch_embed(int64_t n, int64_t m, int64_t k, double scale, const double* d1,
                     const double* d2, const double* d3, int kind, double sigma, const float* x,
                     int64_t batch, int64_t ld, int64_t n_in, double* out);
/* SketchOperator::apply (newton_sketch.cpp:74-101) generalised with an explicit
 * row map: A is [N_in][d] row-major fp32 (ld_a), transform along the N axis
 * (zero padded to n), out[r][c] = norm * y[rows[r]] for r < m_out.
 * rows == NULL => first m_out rows (the reference's P).  norm = 1/sqrt(m) and
 * `scale` is the spinner scale (sqrt(n) by default). */
void orc_sketch(int64_t n, double scale, double norm, const double* d1, const double* d2,
                const double* d3, const float* a, int64_t n_in, int64_t d, int64_t ld_a,
                const int64_t* rows, int64_t m_out, double* out /* [m_out][d] */);

/* Builder-defined P: m of N indices without replacement via a
 * partial Fisher-Yates driven by Rng(mix_seed(seed, 0x5a3b)).next_u64() with
 * rejection sampling; returned sorted ascending. */
void orc_sample_rows(int64_t N, int64_t m, uint64_t seed, int64_t* out);

/* ---- sketched Newton for logistic regression (newton_sketch.cpp) ----------
 * Features row-major fp64 [n][d], labels +-1.  Sketch = first-m rows of one
 * spinner block over N = next_pow2(n) (d1..d3, scale) times norm, or exact when
 * d1 == NULL.  Status: 0 ok, 1 dimension, 7 singular (SingularSystemError). */
void orc_ar1_problem(int64_t n, int64_t d, uint64_t seed, double* a, double* labels); /* :185-204 */
double orc_logistic_loss(const double* a, const double* y, int64_t n, int64_t d, const double* x); /* :45-52 */
void orc_logistic_gradient(const double* a, const double* y, int64_t n, int64_t d, const double* x,
                           double* g);                                                     /* :54-61 */
void orc_hessian_sqrt(const double* a, int64_t n, int64_t d, const double* x, double* out); /* :63-72 */
int orc_llt_solve(double* normal, int64_t d, const double* rhs, double* x);               /* :112-121 */
int orc_sketched_step(const double* a, const double* y, int64_t n, int64_t d, const double* x, int64_t N,
                      int64_t m, double scale, double norm, const double* d1, const double* d2,
                      const double* d3, double* step);                                      /* :103-122 */

#ifdef __cplusplus
}
#endif
#endif
