/* spinners_b200 — C ABI of the B200-native structured-spinner hot path.
 *
 * The reference (arxiv 1610.06209 code, proj/) has no FFI: its boundary is the
 * C++ headers in proj/include/spinners/.  Each entry point below is what a
 * binding of those headers' hot-path entry points needs:
 *
 *   spn_plan_create          <- StructuredSpinner::build / StackedSpinner(v,n,m,k,seed)
 *                               (proj/include/spinners/spinner.hpp:58,110;
 *                                proj/src/spinner.cpp:137-151,248-256) and, with
 *                               tables>1, make_hasher_factory(v,n,m)(seed_t)
 *                               (proj/include/spinners/lsh.hpp:66, proj/src/lsh.cpp:32-36)
 *   spn_apply_f32            <- StackedSpinner::apply / StructuredSpinner::apply
 *                               (spinner.hpp:62,114; spinner.cpp:200-231,272-283)
 *   spn_hash_f32             <- CrossPolytopeHasher::hash + signed_argmax
 *                               (lsh.hpp:21,30; lsh.cpp:9-30)
 *   spn_embed_f32            <- embed(FeatureMap, x) (kernels.hpp:33; kernels.cpp:17-36)
 *   spn_sketch_f32           <- SketchOperator::apply (newton_sketch.hpp:64;
 *                               newton_sketch.cpp:74-101)
 *   spn_*_host               <- the same calls on host buffers (the reference's
 *                               value-semantics API), with the H2D/D2H copies inside.
 *   spn_collision_hits_f32   <- collision_curve / compare_families (lsh.hpp:38-75; lsh.cpp:38-96)
 *   spn_gram_*               <- gram_exact / gram_approx / gram_error (kernels.hpp:35-41; kernels.cpp:38-114)
 *   spn_newton_*, spn_logistic_*, spn_sketched_step_f32, spn_ar1_problem
 *                            <- the sketched Newton method that calls SketchOperator
 *                               (newton_sketch.hpp:63-86; newton_sketch.cpp:45-72,103-204)
 *
 * Conventions: plain pointers and sizes; all sizes/strides in elements;
 * device entry points are stream-ordered and asynchronous (stream = a
 * cudaStream_t, NULL = legacy default stream); `_host` entry points are
 * synchronous.  Errors are status codes; spn_last_error() holds the message
 * of the calling thread's last failure.  Reference exceptions map as
 * DimensionError -> SPN_EDIM, DomainError -> SPN_EDOMAIN (common.hpp:15-27).
 *
 * Numerics: fp32 arithmetic on the device with the reference's fp64 diagonals
 * rounded to fp32 (±1 diagonals are exact).  Per-element finiteness checks of
 * the reference (check_finite, common.hpp:37-41) are NOT done on the device
 * path; spn_check_finite_f32 exists for callers that need them.
 */
#ifndef SPINNERS_B200_H
#define SPINNERS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPN_API __attribute__((visibility("default")))

typedef enum spn_status {
  SPN_OK = 0,
  SPN_EDIM = 1,         /* DimensionError: non-pow2 n, bad m/k, length mismatch */
  SPN_EDOMAIN = 2,      /* DomainError: non-finite / zero input, bad variant or sigma */
  SPN_ECUDA = 3,        /* CUDA runtime failure */
  SPN_ENOMEM = 4,       /* device / pinned allocation failed */
  SPN_EUNSUPPORTED = 5, /* valid request this build does not implement */
  SPN_EINVAL = 6,       /* null pointer / bad argument */
  SPN_ESINGULAR = 7     /* SingularSystemError (common.hpp:25): sketched Hessian indefinite */
} spn_status;

typedef enum spn_variant {
  SPN_HD3_HD2_HD1 = 0,       /* SpinnerVariant::hd3_hd2_hd1 (spinner.hpp:19) */
  SPN_HDG_HD2_HD1 = 1,       /* SpinnerVariant::hdg_hd2_hd1 (spinner.hpp:20) */
  SPN_GCIRC_D2_HD1 = 2,      /* gcirc_d2_hd1: Gaussian circulant * D2 H D1 (spinner.hpp:21); n <= 2^13 */
  SPN_GTOEPLITZ_D2_HD1 = 3,  /* gtoeplitz_d2_hd1 (spinner.hpp:22); n <= 2^12 */
  SPN_GSKEW_CIRC_D2_HD1 = 4, /* gskew_circ_d2_hd1 (spinner.hpp:23); n <= 2^13 */
  SPN_GAUSSIAN_DENSE = 5,    /* gaussian_dense: the unstructured baseline (spinner.hpp:24) */
  SPN_GAUSS3 = 100     /* builder-defined: D1..D3 all N(0,1) (BASELINE config 5) */
} spn_variant;

typedef enum spn_embed_kind { SPN_EMBED_GAUSSIAN = 0, SPN_EMBED_ANGULAR = 1 } spn_embed_kind;

typedef struct spn_plan spn_plan;

typedef struct spn_plan_desc {
  int32_t variant;             /* spn_variant */
  int64_t n;                   /* input dimension, power of two, 2 <= n <= 2^20 */
  int64_t m;                   /* rows per block, 1 <= m <= n */
  int64_t k;                   /* rows per table (stacked blocks: ceil(k/m)), k >= 1 */
  int64_t tables;              /* independent stacked spinners (LSH tables), >= 1 */
  const uint64_t* table_seeds; /* [tables] StackedSpinner seeds; NULL => {seed} */
  uint64_t seed;               /* used when table_seeds == NULL (tables must be 1) */
  double scale;                /* 0 => default_scale(variant, n) = sqrt(n) (spinner.cpp:41-45) */
  int32_t device;              /* CUDA device ordinal */
} spn_plan_desc;

SPN_API const char* spn_status_string(spn_status s);
SPN_API const char* spn_last_error(void);
SPN_API const char* spn_version(void);

/* Realise the diagonals with the reference's seeded generator on the host
 * (mix_seed + mt19937_64 + Box-Muller, common.hpp:51-92) and upload them. */
SPN_API spn_status spn_plan_create(spn_plan** out, const spn_plan_desc* desc);
/* One m x n block realised from its spec seed directly (StructuredSpinner::build(spec),
 * spinner.cpp:137-151): any variant, k = m, one table; scale 0 => default_scale. */
SPN_API spn_status spn_plan_create_block(spn_plan** out, int32_t variant, int64_t n, int64_t m,
                                         uint64_t spec_seed, double scale, int32_t device);
/* Same, with caller-provided diagonals [tables][blocks][n] (e.g. a fitted tail
 * vector, StructuredSpinner::with_tail_vector, spinner.hpp:80). */

SPN_API spn_status spn_plan_create_explicit(spn_plan** out, int64_t n, int64_t m, int64_t k,
                                            int64_t tables, const double* d1, const double* d2,
                                            const double* d3, double scale, int32_t device);
/* StructuredSpinner::resample_last_block (mode 0) / resample_tail (mode 1)
 * (proj/include/spinners/spinner.hpp:67-74; proj/src/spinner.cpp:153-166): a new one-block plan
 * equal to `src` with the last block's randomness (D3, g, the circulant generator or the dense
 * matrix; draw_tail, spinner.cpp:92-135) redrawn from Rng(mix_seed(tail_seed, 2)) — or, mode 1,
 * D2 and then that randomness redrawn from Rng(mix_seed(tail_seed, 3)).  src: one table, one block. */
SPN_API spn_status spn_plan_resample(spn_plan** out, const spn_plan* src, int32_t mode, uint64_t tail_seed);
/* StructuredSpinner::with_tail_vector (spinner.hpp:75-77; spinner.cpp:168-184): D3 (HD3) or g (HDg)
 * replaced by r[n]; Hadamard-only variants; SPN_EDOMAIN for a non-finite entry. */
SPN_API spn_status spn_plan_with_tail(spn_plan** out, const spn_plan* src, const double* r);
SPN_API spn_status spn_plan_destroy(spn_plan* plan);
SPN_API spn_status spn_plan_query(const spn_plan* plan, int64_t* n, int64_t* m, int64_t* k,
                                  int64_t* tables, int64_t* blocks, double* scale);
/* The realised fp64 diagonals, [tables][blocks][n] each (for parity checks). */
SPN_API spn_status spn_plan_diagonals(const spn_plan* plan, double* d1, double* d2, double* d3);

/* y[b*ld_y + r] = relu?( scale * (stacked spinner x_b)[r] ), r < k.  x rows are
 * zero padded from n_in to n (dataset.cpp:162-168).  Requires tables == 1. */
SPN_API spn_status spn_apply_f32(const spn_plan* plan, const float* x, int64_t batch,
                                 int64_t ld_x, int64_t n_in, float* y, int64_t ld_y, int32_t relu,
                                 void* stream);

/* ids[b*tables + t] = index + (sign < 0 ? k : 0) of signed_argmax over table t's
 * k rows (ties -> smallest index, sign(0) = +1).  If y != NULL (tables == 1)
 * the projection is stored as by spn_apply_f32.  Any n <= 2^20: n <= 2^14 runs the fused
 * kernel, larger n the multi-pass projection followed by a row argmax. */
SPN_API spn_status spn_hash_f32(const spn_plan* plan, const float* x, int64_t batch,
                                int64_t ld_x, int64_t n_in, int32_t* ids, float* y,
                                int64_t ld_y, void* stream);

/* Gaussian: out[b*ld + i] = cos(z_i/sigma)/sqrt(k), out[b*ld + k + i] = sin(z_i/sigma)/sqrt(k);
 * angular: out[b*ld + i] = z_i < 0 ? -1 : +1.   z = scale * stacked(x).  Any n <= 2^20 (n > 2^14:
 * the multi-pass projection into out, then the feature epilogue in place). */
SPN_API spn_status spn_embed_f32(const spn_plan* plan, int32_t kind, double sigma, const float* x,
                                 int64_t batch, int64_t ld_x, int64_t n_in, float* out,
                                 int64_t ld_out, void* stream);

/* Sketch along the long (strided) axis of a row-major A[n_in][d] (ld_a):
 * out[r*ld_out + c] = norm * scale * (H D3 H D2 H D1 a_c)[rows[r]] for r < m_out,
 * a_c = column c zero padded to n.  rows == NULL => rows 0..m_out-1 of the stacked
 * output (the reference's first-m P; m_out <= k, any number of blocks: the multi-block
 * SketchOperator of newton_sketch.cpp:77-79 when rows > padded); rows is a HOST array of
 * distinct indices < n (builder-defined P; single-block plans).  Requires tables == 1. */
SPN_API spn_status spn_sketch_f32(const spn_plan* plan, const float* a, int64_t n_in, int64_t d,
                                  int64_t ld_a, const int64_t* rows, int64_t m_out, double norm,
                                  float* out, int64_t ld_out, void* stream);

/* Host-buffer variants: pinned or pageable host memory in and out; the copies
 * are pipelined with the kernels in chunks.  Synchronous. */
SPN_API spn_status spn_apply_f32_host(const spn_plan* plan, const float* x, int64_t batch,
                                      int64_t ld_x, int64_t n_in, float* y, int64_t ld_y,
                                      int32_t relu);
SPN_API spn_status spn_hash_f32_host(const spn_plan* plan, const float* x, int64_t batch,
                                     int64_t ld_x, int64_t n_in, int32_t* ids);
/* hash + projection in one call on host buffers (BASELINE config 1: CrossPolytopeHasher::hash,
 * lsh.cpp:23-30, and StructuredSpinner::apply, spinner.cpp:200-231, on the same rows):
 * ids[b] as spn_hash_f32, y[b*ld_y + r] as spn_apply_f32.  Requires tables == 1. */
SPN_API spn_status spn_hash_project_f32_host(const spn_plan* plan, const float* x, int64_t batch,
                                             int64_t ld_x, int64_t n_in, int32_t* ids, float* y,
                                             int64_t ld_y);
/* SketchOperator::apply with value semantics (newton_sketch.hpp:64; newton_sketch.cpp:87-101):
 * A and out are HOST buffers (pinned for full PCIe rate); arguments as spn_sketch_f32. */
SPN_API spn_status spn_sketch_f32_host(const spn_plan* plan, const float* a, int64_t n_in, int64_t d,
                                       int64_t ld_a, const int64_t* rows, int64_t m_out, double norm,
                                       float* out, int64_t ld_out);
SPN_API spn_status spn_embed_f32_host(const spn_plan* plan, int32_t kind, double sigma,
                                      const float* x, int64_t batch, int64_t ld_x, int64_t n_in,
                                      float* out, int64_t ld_out);

/* fwht_normalized (transforms.hpp:13; transforms.cpp:52-71) of every row: y_b = H_n x_b with the
 * orthonormal Walsh-Hadamard H_n; n a power of two <= 2^20 (n = 1: a copy).  Runs the spinner
 * kernels with unit diagonals (H H H = H) on a plan cached per (device, n); x may equal y. */
SPN_API spn_status spn_fwht_f32(int64_t n, const float* x, int64_t batch, int64_t ld_x, float* y,
                                int64_t ld_y, int32_t device, void* stream);
SPN_API spn_status spn_fwht_f32_host(int64_t n, const float* x, int64_t batch, int64_t ld_x, float* y,
                                     int64_t ld_y, int32_t device);

/* diag_matvec (transforms.hpp:59; transforms.cpp:228-235) of every row: y_b = d (.) x_b.  The
 * reference's finiteness checks stay in the C++ drop-in; the device does not scan. */
SPN_API spn_status spn_diag_f32(int64_t n, const float* d, const float* x, int64_t batch, int64_t ld_x,
                                float* y, int64_t ld_y, void* stream);
SPN_API spn_status spn_diag_f32_host(int64_t n, const float* d, const float* x, int64_t batch, int64_t ld_x,
                                     float* y, int64_t ld_y, int32_t device);

/* CirculantOperator (transforms.hpp:37-51; transforms.cpp:112-208): kind 0 circulant
 * (C[i][j] = r[(j-i) mod n]), 1 Toeplitz (T[i][j] = t[i-j]: first_col for i >= j, first_row
 * for i < j; first_col[0] == first_row[0]), 2 skew-circulant (negacyclic).  Any n >= 1 whose
 * FFT length (n, 2 next_pow2(n) for Toeplitz, next_pow2(2n) otherwise) is <= 2^13; the spectrum is
 * built on the host as the reference builds it, the correlation runs on the device in fp64.
 * apply: y_b = M x_b for every row (x may equal y). */
typedef struct spn_circulant spn_circulant;
SPN_API spn_status spn_circulant_create(spn_circulant** out, int32_t kind, int64_t n, const double* first_row,
                                        const double* first_col, int32_t device);
SPN_API spn_status spn_circulant_destroy(spn_circulant* op);
SPN_API spn_status spn_circulant_apply_f32(const spn_circulant* op, const float* x, int64_t batch, int64_t ld_x,
                                           float* y, int64_t ld_y, void* stream);
SPN_API spn_status spn_circulant_apply_f32_host(const spn_circulant* op, const float* x, int64_t batch,
                                                int64_t ld_x, float* y, int64_t ld_y);

/* Builder-defined coordinate sampler P (BASELINE config 4): m distinct indices of
 * [0, N) via a partial Fisher-Yates driven by Rng(mix_seed(seed, 0x5a3b)), sorted. */
SPN_API spn_status spn_sample_rows(int64_t N, int64_t m, uint64_t seed, int64_t* out);
/* One block's diagonals realised from its spec seed exactly as
 * StructuredSpinner::build does (spinner.cpp:137-151): d1,d2 <- Rng(mix_seed(seed,1)),
 * d3 (or g) <- Rng(mix_seed(seed,2)).  Each output has n doubles. */
SPN_API spn_status spn_realize_block(int32_t variant, int64_t n, uint64_t spec_seed, double* d1,
                                     double* d2, double* d3);
/* The reference's splitmix64 seed mixer (common.hpp:51-56). */
SPN_API uint64_t spn_mix_seed(uint64_t base, uint64_t stream);
/* Device-side finiteness / all-zero check of a batch of rows: flags[b] bit0 =
 * non-finite entry, bit1 = all zero (what hash/embed reject, lsh.cpp:24-28). */
SPN_API spn_status spn_check_rows_f32(const float* x, int64_t batch, int64_t ld_x, int64_t n_in,
                                      int32_t* flags, void* stream);

/* Multi-GPU hashing with the all-gather fused into the kernel: each id of this rank's rows
 * is stored at row row0 + v of EVERY rank's gathered [total][tables] int32 table, through
 * the device pointers in `peers` (a device array of npeers pointers mapped with CUDA IPC
 * over NVLink / NVSwitch; the local table is one of them).  After a barrier on all
 * ranks, every table holds all codes — the NCCL all-gather of config 3 without a
 * separate collective.  total = rows of every gathered table; row0 + batch <= total. */
SPN_API spn_status spn_hash_f32_peers(const spn_plan* plan, const float* x, int64_t batch, int64_t ld_x,
                                      int64_t n_in, int32_t* const* peers, int32_t npeers, int64_t row0,
                                      int64_t total, void* stream);
/* Let kernels launched on `device` load/store memory that lives on `peer_device` (the peer
 * tables of spn_hash_f32_peers on a multi-GPU node: cudaDeviceEnablePeerAccess from device's
 * context; already enabled, or device == peer_device, is SPN_OK).  SPN_EUNSUPPORTED when the
 * pair has no peer path (the caller then gathers with a collective instead). */
SPN_API spn_status spn_enable_peer_access(int32_t device, int32_t peer_device);

/* collision_curve / compare_families (lsh.cpp:38-96; lsh.hpp:38-75), the counting core.
 * plan: `trials` tables of make_hasher_factory(v, n, m) with table seeds mix_seed(seed, t)
 * (lsh.cpp:56).  xy: 2*pairs device rows, row 2p = x_p, row 2p+1 = y_p.  bucket_of: device
 * int32 [pairs] (< buckets).  hits: device int64 [buckets], accumulated with the number of
 * (pair, trial) events where hash_t(x_p) == hash_t(y_p) (same index and sign). */
SPN_API spn_status spn_collision_hits_f32(const spn_plan* plan, const float* xy, int64_t pairs, int64_t ld,
                                          int64_t n_in, const int32_t* bucket_of, int64_t buckets, int64_t* hits,
                                          void* stream);

/* Gram matrices of the feature maps (kernels.hpp:35-41; kernels.cpp:38-114), fp64 outputs,
 * device buffers.  kind: SPN_EMBED_GAUSSIAN / SPN_EMBED_ANGULAR.
 *   gram_exact:  points [count][ld] fp32 -> exact kernel matrix (diag 1);
 *   gram_approx: features = embed(fm, points) [count][ld] fp32 (width 2d' gaussian, d' angular)
 *                -> F F^T (gaussian) or 1/2 + F F^T / (2 d') (angular), diag 1;
 *   gram_error:  ||exact - approx||_F / ||exact||_F into *err (host; synchronises the stream). */
SPN_API spn_status spn_gram_exact_f32(const float* points, int64_t count, int64_t dim, int64_t ld, int32_t kind,
                                      double sigma, double* gram, int64_t ld_gram, void* stream);
SPN_API spn_status spn_gram_approx_f32(const float* features, int64_t count, int64_t width, int64_t ld,
                                       int32_t kind, int64_t dprime, double* gram, int64_t ld_gram, void* stream);
SPN_API spn_status spn_gram_error(const double* exact, const double* approx, int64_t count, int64_t ld, double* err,
                                  void* stream);
/* Host-buffer forms (synchronous): points [count][dim] fp32, gram [count][count] fp64.
 * spn_gram_approx_host embeds with `plan` (a FeatureMap's projector; kind/sigma as in
 * spn_embed_f32) and forms the approximate Gram matrix on the device. */
SPN_API spn_status spn_gram_exact_host(const float* points, int64_t count, int64_t dim, int32_t kind, double sigma,
                                       double* gram);
SPN_API spn_status spn_gram_approx_host(const spn_plan* plan, int32_t kind, double sigma, const float* points,
                                        int64_t count, int64_t dim, double* gram);
SPN_API spn_status spn_gram_error_host(const double* exact, const double* approx, int64_t count, double* err);

/* ------------------------------------------------------------------ sketched Newton
 * Logistic regression with spinner-sketched Hessians (newton_sketch.hpp:13-86).
 * Problem data on the device: A row-major fp32 [n][ld_a], labels fp32 (+-1) [n];
 * iterates, steps and gradients fp64 [d] device vectors; losses fp64 device scalars.
 * A workspace holds the per-problem scratch (margins, Hessian row scales, the
 * sketched matrix S*B, the d x d normal matrix and its Cholesky factor).  d <= 1024.
 * Calls on one workspace must be serialised by the caller. */
typedef struct spn_newton spn_newton;
SPN_API spn_status spn_newton_create(spn_newton** out, int64_t n, int64_t d, int64_t max_sketch_rows,
                                     int device);
SPN_API spn_status spn_newton_destroy(spn_newton* w);
/* loss(p, x) (newton_sketch.cpp:45-52) and gradient(p, x) (:54-61) in one pass over A;
 * either output may be NULL. */
SPN_API spn_status spn_logistic_eval_f32(spn_newton* w, const float* a, int64_t ld_a, const float* labels,
                                         const double* x, double* loss, double* grad, void* stream);
/* hessian_sqrt(p, x) (:63-72): out[i][:] = sqrt(s_i (1 - s_i)) a_i, s_i = sigmoid(a_i . x). */
SPN_API spn_status spn_hessian_sqrt_f32(spn_newton* w, const float* a, int64_t ld_a, const double* x,
                                        float* out, int64_t ld_out, void* stream);
/* sketched_step(p, x, sketch) (:103-122).  sketch = a plan made like
 * SketchOperator(variant, n, rows, seed) (:74-81: n' = next_pow2(n), m = min(rows, n'),
 * k = rows), applied with norm 1/sqrt(rows) to B = hessian_sqrt(p, x) (first `rows`
 * rows, :87-101); sketch = NULL is the exact (identity) operator.  Solves
 * ((S B)^T (S B)) step = -gradient by Cholesky with the reference's ridge retry
 * (1e-10 * trace); SPN_ESINGULAR if that fails too; SPN_EDIM if rows < d.
 * grad / loss (optional) receive gradient(p, x) / loss(p, x).  Synchronises `stream`
 * (the status depends on the factorisation). */
SPN_API spn_status spn_sketched_step_f32(spn_newton* w, const spn_plan* sketch, int64_t rows, const float* a,
                                         int64_t ld_a, const float* labels, const double* x, double* step,
                                         double* grad, double* loss, void* stream);
/* The backtracking candidates of solve() (:140-143, :160-165):
 * losses[k] = loss(p, x + (s0 * 2^-k) * step) for k < count (count <= 64). */
SPN_API spn_status spn_logistic_line_f32(spn_newton* w, const float* a, int64_t ld_a, const float* labels,
                                         const double* x, const double* step, double s0, int64_t count,
                                         double* losses, void* stream);
/* Host-buffer forms (the reference's value semantics; synchronous).  The problem is
 * uploaded once into the workspace (fp32 features [n][ld], +-1 labels); the calls then
 * move only d-vectors and scalars. */
SPN_API spn_status spn_newton_set_problem(spn_newton* w, const float* features, int64_t ld, const float* labels);
SPN_API spn_status spn_logistic_eval_host(spn_newton* w, const double* x, double* loss, double* grad);
SPN_API spn_status spn_hessian_sqrt_host(spn_newton* w, const double* x, float* out, int64_t ld_out);
SPN_API spn_status spn_sketched_step_host(spn_newton* w, const spn_plan* sketch, int64_t rows, const double* x,
                                          double* step, double* grad, double* loss);
SPN_API spn_status spn_logistic_line_host(spn_newton* w, const double* x, const double* step, double s0,
                                          int64_t count, double* losses);
/* generate_ar1_problem(n, d, seed) (:185-204) on the host (reference generator, bit-exact
 * in fp64), rounded to fp32: features [n][d], labels [n]. */
SPN_API spn_status spn_ar1_problem(int64_t n, int64_t d, uint64_t seed, float* features, float* labels);

#ifdef __cplusplus
}
#endif
#endif /* SPINNERS_B200_H */
