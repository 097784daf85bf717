/* CPU ORACLE — TEST INFRASTRUCTURE ONLY (see spinner_oracle.h).
 * fp64 restatement of /root/reference/proj; every function cites the
 * reference lines it follows. */
#include "spinner_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* common.hpp:51-56 — splitmix64 finaliser. */
uint64_t orc_mix_seed(uint64_t base, uint64_t stream) {
  uint64_t z = base + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* std::mt19937_64 (the engine of common.hpp:61-92): w=64 n=312 m=156 r=31,
 * a=0xB5026F5AA96619E9, tempering (u,d)=(29,0x5555555555555555) (s,b)=(17,
 * 0x71D67FFFEDA60000) (t,c)=(37,0xFFF7EEE000000000) l=43, f=6364136223846793005. */
void orc_rng_init(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = 312;
  r->have_spare = 0;
  r->spare = 0.0;
}

uint64_t orc_rng_next(orc_rng* r) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  if (r->mti >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
      r->mt[i] = r->mt[(i + 156) % 312] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* common.hpp:68-70 — uniform in (0,1]. */
double orc_rng_uniform01(orc_rng* r) { return ((double)(orc_rng_next(r) >> 11) + 1.0) * 0x1p-53; }

/* common.hpp:72-84 — Box-Muller, cosine first, sine cached. */
double orc_rng_gaussian(orc_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u = orc_rng_uniform01(r);
  double v = orc_rng_uniform01(r);
  double rad = sqrt(-2.0 * log(u));
  double ang = 2.0 * M_PI * v;
  r->spare = rad * sin(ang);
  r->have_spare = 1;
  return rad * cos(ang);
}

/* common.hpp:86 */
double orc_rng_rademacher(orc_rng* r) { return (orc_rng_next(r) & 1ULL) ? 1.0 : -1.0; }

/* spinner.cpp:41-45 */
double orc_default_scale(int variant, int64_t n) {
  (void)variant; /* every variant here is Hadamard-only */
  return sqrt((double)n);
}

/* spinner.cpp:137-151 (front Rng(mix_seed(seed,1)) -> D1 then D2) and
 * draw_tail :92-106 (tail Rng(mix_seed(seed,2)) -> D3 or g).  The all-Gaussian
 * variant (builder-defined) mirrors the same streams with gaussian(). */
void orc_realize_block(int variant, int64_t n, uint64_t spec_seed, double* d1, double* d2,
                       double* d3) {
  orc_rng front, tail;
  orc_rng_init(&front, orc_mix_seed(spec_seed, 1));
  orc_rng_init(&tail, orc_mix_seed(spec_seed, 2));
  if (variant == ORC_GAUSS3) {
    for (int64_t i = 0; i < n; ++i) d1[i] = orc_rng_gaussian(&front);
    for (int64_t i = 0; i < n; ++i) d2[i] = orc_rng_gaussian(&front);
    for (int64_t i = 0; i < n; ++i) d3[i] = orc_rng_gaussian(&tail);
    return;
  }
  for (int64_t i = 0; i < n; ++i) d1[i] = orc_rng_rademacher(&front);
  for (int64_t i = 0; i < n; ++i) d2[i] = orc_rng_rademacher(&front);
  if (variant == ORC_HDG)
    for (int64_t i = 0; i < n; ++i) d3[i] = orc_rng_gaussian(&tail);
  else
    for (int64_t i = 0; i < n; ++i) d3[i] = orc_rng_rademacher(&tail);
}

/* spinner.cpp:248-256 */
int64_t orc_realize_stacked(int variant, int64_t n, int64_t m, int64_t k, uint64_t seed,
                            double* d1, double* d2, double* d3) {
  int64_t blocks = (k + m - 1) / m;
  for (int64_t b = 0; b < blocks; ++b)
    orc_realize_block(variant, n, orc_mix_seed(seed, (uint64_t)b), d1 + b * n, d2 + b * n,
                      d3 + b * n);
  return blocks;
}

/* transforms.cpp:52-71 — radix-2 butterflies h = 1, 2, ..., n/2 then x 1/sqrt(n). */
void orc_fwht_normalized(double* x, int64_t n) {
  for (int64_t h = 1; h < n; h <<= 1)
    for (int64_t i = 0; i < n; i += h << 1)
      for (int64_t j = i; j < i + h; ++j) {
        double u = x[j], v = x[j + h];
        x[j] = u + v;
        x[j + h] = u - v;
      }
  const double s = 1.0 / sqrt((double)n);
  for (int64_t i = 0; i < n; ++i) x[i] *= s;
}

/* spinner.cpp:186-231 with diag_matvec transforms.cpp:228-235. */
static void chain(int64_t n, const double* d1, const double* d2, const double* d3,
                  double* v /* in: x, out: H D3 H D2 H D1 x */) {
  for (int64_t i = 0; i < n; ++i) v[i] *= d1[i];
  orc_fwht_normalized(v, n);
  for (int64_t i = 0; i < n; ++i) v[i] *= d2[i];
  orc_fwht_normalized(v, n);
  for (int64_t i = 0; i < n; ++i) v[i] *= d3[i];
  orc_fwht_normalized(v, n);
}

void orc_block_apply(int64_t n, int64_t m, double scale, const double* d1, const double* d2,
                     const double* d3, const double* x, double* y) {
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(v, x, sizeof(double) * (size_t)n);
  chain(n, d1, d2, d3, v);
  for (int64_t i = 0; i < m; ++i) y[i] = v[i] * scale; /* resize(m) then *= scale, :228-229 */
  free(v);
}

/* spinner.cpp:272-283 */
void orc_stacked_apply(int64_t n, int64_t m, int64_t k, double scale, const double* d1,
                       const double* d2, const double* d3, const double* x, double* y) {
  double* tmp = (double*)malloc(sizeof(double) * (size_t)m);
  int64_t out = 0;
  for (int64_t b = 0; out < k; ++b) {
    orc_block_apply(n, m, scale, d1 + b * n, d2 + b * n, d3 + b * n, x, tmp);
    for (int64_t i = 0; i < m && out < k; ++i) y[out++] = tmp[i];
  }
  free(tmp);
}

/* lsh.cpp:9-21 */
void orc_signed_argmax(const double* y, int64_t len, int64_t* index, int* sign) {
  int64_t best = 0;
  double best_abs = fabs(y[0]);
  for (int64_t i = 1; i < len; ++i) {
    double a = fabs(y[i]);
    if (a > best_abs) {
      best_abs = a;
      best = i;
    }
  }
  *index = best;
  *sign = y[best] < 0.0 ? -1 : 1;
}

double orc_top2_gap(const double* y, int64_t len) {
  double a = -1.0, b = -1.0;
  for (int64_t i = 0; i < len; ++i) {
    double v = fabs(y[i]);
    if (v > a) {
      b = a;
      a = v;
    } else if (v > b) {
      b = v;
    }
  }
  if (len < 2 || a <= 0.0) return 0.0;
  return (a - b) / a;
}

static void load_row(const float* x, int64_t ld, int64_t row, int64_t n_in, int64_t n, double* v) {
  for (int64_t i = 0; i < n; ++i) v[i] = i < n_in ? (double)x[row * ld + i] : 0.0;
}

void orc_batch_apply(int64_t n, int64_t m, int64_t k, double scale, const double* d1,
                     const double* d2, const double* d3, const float* x, int64_t batch, int64_t ld,
                     int64_t n_in, int relu, double* y) {
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t b = 0; b < batch; ++b) {
    load_row(x, ld, b, n_in, n, v);
    orc_stacked_apply(n, m, k, scale, d1, d2, d3, v, y + b * k);
    if (relu)
      for (int64_t i = 0; i < k; ++i)
        if (y[b * k + i] < 0.0) y[b * k + i] = 0.0;
  }
  free(v);
}

/* CrossPolytopeHasher::hash (lsh.cpp:23-30) per table; make_hasher_factory
 * (lsh.cpp:32-36) gives each table StackedSpinner(v, n, min(m,n), m, seed_t). */
void orc_batch_hash(int64_t n, int64_t m, int64_t k, int64_t tables, double scale,
                    const double* d1, const double* d2, const double* d3, const float* x,
                    int64_t batch, int64_t ld, int64_t n_in, int32_t* ids, double* gaps) {
  const int64_t blocks = (k + m - 1) / m;
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  double* y = (double*)malloc(sizeof(double) * (size_t)k);
  for (int64_t b = 0; b < batch; ++b) {
    load_row(x, ld, b, n_in, n, v);
    for (int64_t t = 0; t < tables; ++t) {
      const int64_t off = t * blocks * n;
      orc_stacked_apply(n, m, k, scale, d1 + off, d2 + off, d3 + off, v, y);
      int64_t idx;
      int sg;
      orc_signed_argmax(y, k, &idx, &sg);
      ids[b * tables + t] = (int32_t)(idx + (sg < 0 ? k : 0));
      if (gaps) gaps[b * tables + t] = orc_top2_gap(y, k);
    }
  }
  free(v);
  free(y);
}

/* kernels.cpp:17-36 */
void orc_batch_embed(int64_t n, int64_t m, int64_t k, double scale, const double* d1,
                     const double* d2, const double* d3, int kind, double sigma, const float* x,
                     int64_t batch, int64_t ld, int64_t n_in, double* out) {
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  double* z = (double*)malloc(sizeof(double) * (size_t)k);
  const double inv_sigma = 1.0 / sigma;
  const double norm = 1.0 / sqrt((double)k);
  for (int64_t b = 0; b < batch; ++b) {
    load_row(x, ld, b, n_in, n, v);
    orc_stacked_apply(n, m, k, scale, d1, d2, d3, v, z);
    if (kind == 1) {
      for (int64_t i = 0; i < k; ++i) out[b * k + i] = z[i] < 0.0 ? -1.0 : 1.0;
    } else {
      double* o = out + b * 2 * k;
      for (int64_t i = 0; i < k; ++i) {
        const double t = z[i] * inv_sigma;
        o[i] = norm * cos(t);
        o[k + i] = norm * sin(t);
      }
    }
  }
  free(v);
  free(z);
}

/* newton_sketch.cpp:87-101: per column, zero pad to n, StackedSpinner::apply,
 * scale by norm_.  Generalised here with an explicit row list (NULL = first m). */
void orc_sketch(int64_t n, double scale, double norm, const double* d1, const double* d2,
                const double* d3, const float* a, int64_t n_in, int64_t d, int64_t ld_a,
                const int64_t* rows, int64_t m_out, double* out) {
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t c = 0; c < d; ++c) {
    for (int64_t i = 0; i < n; ++i) v[i] = i < n_in ? (double)a[i * ld_a + c] : 0.0;
    chain(n, d1, d2, d3, v);
    for (int64_t r = 0; r < m_out; ++r) {
      const int64_t i = rows ? rows[r] : r;
      out[r * d + c] = norm * (scale * v[i]);
    }
  }
  free(v);
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

void orc_sample_rows(int64_t N, int64_t m, uint64_t seed, int64_t* out) {
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
  for (int64_t i = 0; i < N; ++i) idx[i] = i;
  orc_rng r;
  orc_rng_init(&r, orc_mix_seed(seed, 0x5a3b));
  for (int64_t i = 0; i < m; ++i) {
    const uint64_t range = (uint64_t)(N - i);
    const uint64_t threshold = (0 - range) % range; /* 2^64 mod range */
    uint64_t u;
    do {
      u = orc_rng_next(&r);
    } while (u < threshold);
    const int64_t j = i + (int64_t)(u % range);
    int64_t t = idx[i];
    idx[i] = idx[j];
    idx[j] = t;
  }
  memcpy(out, idx, sizeof(int64_t) * (size_t)m);
  qsort(out, (size_t)m, sizeof(int64_t), cmp_i64);
  free(idx);
}

/* Test-input helper: `count` draws of one kind from Rng(seed) (kind 1 uniform01,
 * 2 gaussian, 3 rademacher; common.hpp:68-86). */
void orc_rng_fill(uint64_t seed, int kind, int64_t count, double* out) {
  orc_rng r;
  orc_rng_init(&r, seed);
  for (int64_t i = 0; i < count; ++i)
    out[i] = kind == 1 ? orc_rng_uniform01(&r) : kind == 2 ? orc_rng_gaussian(&r) : orc_rng_rademacher(&r);
}

/* ------------------------------------------------------------ sketched Newton */

/* newton_sketch.cpp:10-15 */
static double log1p_exp(double t) {
  if (t > 35.0) return t;
  if (t < -35.0) return exp(t);
  return log1p(exp(t));
}

/* newton_sketch.cpp:17-24 */
static double sigmoid(double t) {
  if (t >= 0.0) {
    const double e = exp(-t);
    return 1.0 / (1.0 + e);
  }
  const double e = exp(t);
  return e / (1.0 + e);
}

/* newton_sketch.cpp:185-204: AR(1) rows (rho = 0.99) from Rng(mix_seed(seed, 7)),
 * then the labels from the same stream. */
void orc_ar1_problem(int64_t n, int64_t d, uint64_t seed, double* a, double* labels) {
  const double rho = 0.99, noise = sqrt(1.0 - rho * rho);
  orc_rng r;
  orc_rng_init(&r, orc_mix_seed(seed, 7));
  for (int64_t i = 0; i < n; ++i) {
    double prev = orc_rng_gaussian(&r);
    a[i * d] = prev;
    for (int64_t j = 1; j < d; ++j) {
      prev = rho * prev + noise * orc_rng_gaussian(&r);
      a[i * d + j] = prev;
    }
  }
  for (int64_t i = 0; i < n; ++i) labels[i] = orc_rng_rademacher(&r);
}

static double margin(const double* a, int64_t d, int64_t i, const double* x) {
  double m = 0.0;
  for (int64_t k = 0; k < d; ++k) m += a[i * d + k] * x[k];
  return m;
}

/* newton_sketch.cpp:45-52 */
double orc_logistic_loss(const double* a, const double* y, int64_t n, int64_t d, const double* x) {
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) total += log1p_exp(-y[i] * margin(a, d, i, x));
  return total;
}

/* newton_sketch.cpp:54-61: A^T w, w_i = (sigmoid(y_i m_i) - 1) y_i */
void orc_logistic_gradient(const double* a, const double* y, int64_t n, int64_t d, const double* x,
                           double* g) {
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) w[i] = (sigmoid(y[i] * margin(a, d, i, x)) - 1.0) * y[i];
  for (int64_t j = 0; j < d; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i * d + j] * w[i];
    g[j] = s;
  }
  free(w);
}

/* newton_sketch.cpp:63-72: rows scaled by sqrt(s (1 - s)), s = sigmoid(a_i . x) */
void orc_hessian_sqrt(const double* a, int64_t n, int64_t d, const double* x, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    const double s = sigmoid(margin(a, d, i, x));
    const double h = sqrt(s * (1.0 - s));
    for (int64_t j = 0; j < d; ++j) out[i * d + j] = a[i * d + j] * h;
  }
}

/* Lower Cholesky (a non-positive pivot fails, as Eigen's LLT) + two triangular solves. */
static int llt(const double* A, int64_t d, double* L) {
  memset(L, 0, sizeof(double) * (size_t)(d * d));
  for (int64_t j = 0; j < d; ++j) {
    double p = A[j * d + j];
    for (int64_t k = 0; k < j; ++k) p -= L[j * d + k] * L[j * d + k];
    if (!(p > 0.0)) return 7;
    const double ljj = sqrt(p);
    L[j * d + j] = ljj;
    for (int64_t i = j + 1; i < d; ++i) {
      double s = A[i * d + j];
      for (int64_t k = 0; k < j; ++k) s -= L[i * d + k] * L[j * d + k];
      L[i * d + j] = s / ljj;
    }
  }
  return 0;
}

/* newton_sketch.cpp:112-121: LLT; on failure add 1e-10 * trace to the diagonal and
 * retry once; a second failure is SingularSystemError. */
int orc_llt_solve(double* normal, int64_t d, const double* rhs, double* x) {
  double* L = (double*)malloc(sizeof(double) * (size_t)(d * d));
  int rc = llt(normal, d, L);
  if (rc) {
    double tr = 0.0;
    for (int64_t j = 0; j < d; ++j) tr += normal[j * d + j];
    for (int64_t j = 0; j < d; ++j) normal[j * d + j] += 1e-10 * tr;
    rc = llt(normal, d, L);
  }
  if (!rc) {
    double* t = (double*)malloc(sizeof(double) * (size_t)d);
    for (int64_t i = 0; i < d; ++i) {
      double s = rhs[i];
      for (int64_t k = 0; k < i; ++k) s -= L[i * d + k] * t[k];
      t[i] = s / L[i * d + i];
    }
    for (int64_t i = d - 1; i >= 0; --i) {
      double s = t[i];
      for (int64_t k = i + 1; k < d; ++k) s -= L[k * d + i] * x[k];
      x[i] = s / L[i * d + i];
    }
    free(t);
  }
  free(L);
  return rc;
}

/* newton_sketch.cpp:103-122: S B with B = hessian_sqrt, normal = (SB)^T SB,
 * solve normal * step = -gradient. */
int orc_sketched_step(const double* a, const double* y, int64_t n, int64_t d, const double* x, int64_t N,
                      int64_t m, double scale, double norm, const double* d1, const double* d2,
                      const double* d3, double* step) {
  double* B = (double*)malloc(sizeof(double) * (size_t)(n * d));
  orc_hessian_sqrt(a, n, d, x, B);
  const int64_t rows = d1 ? m : n;
  double* SB = B;
  if (d1) {
    SB = (double*)malloc(sizeof(double) * (size_t)(m * d));
    double* v = (double*)malloc(sizeof(double) * (size_t)N);
    for (int64_t c = 0; c < d; ++c) {
      for (int64_t i = 0; i < N; ++i) v[i] = i < n ? B[i * d + c] : 0.0;
      chain(N, d1, d2, d3, v);
      for (int64_t r = 0; r < m; ++r) SB[r * d + c] = norm * (scale * v[r]);
    }
    free(v);
  }
  int rc = 0;
  if (rows < d) rc = 1;
  if (!rc) {
    double* normal = (double*)malloc(sizeof(double) * (size_t)(d * d));
    for (int64_t j = 0; j < d; ++j)
      for (int64_t k = 0; k < d; ++k) {
        double s = 0.0;
        for (int64_t r = 0; r < rows; ++r) s += SB[r * d + j] * SB[r * d + k];
        normal[j * d + k] = s;
      }
    double* rhs = (double*)malloc(sizeof(double) * (size_t)d);
    orc_logistic_gradient(a, y, n, d, x, rhs);
    for (int64_t j = 0; j < d; ++j) rhs[j] = -rhs[j];
    rc = orc_llt_solve(normal, d, rhs, step);
    free(rhs);
    free(normal);
  }
  if (SB != B) free(SB);
  free(B);
  return rc;
}
