// TEST INFRASTRUCTURE ONLY — a C binding over the REFERENCE's own code.
//
// oracle/Makefile compiles /root/reference/proj/src/{transforms,spinner,lsh,
// kernels}.cpp unmodified (against oracle/eigen_shim for the absent Eigen3)
// together with this file into oracle/_ref/libspinners_ref.so.  Tests use it to
// pin the C restatement (spinner_oracle.c) and to make golden vectors; bench.py
// uses it as the CPU baseline ("kind": "reference") and as the --impl reference arm.
// Nothing in the product links it.
//
// newton_sketch.cpp compiles against the shim's LLT, so the sketched-Newton
// entry points below (loss, gradient, hessian_sqrt, sketched_step, solve,
// generate_ar1_problem) call the reference itself.  ref_sketch keeps its
// restatement of SketchOperator::apply because it also serves the builder-defined
// random-P mode.
#include <spinners/common.hpp>
#include <spinners/kernels.hpp>
#include <spinners/lsh.hpp>
#include <spinners/newton_sketch.hpp>
#include <spinners/spinner.hpp>
#include <spinners/transforms.hpp>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

using namespace spinners;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const DimensionError*>(&e)) return 1;
  if (dynamic_cast<const DomainError*>(&e)) return 2;
  if (dynamic_cast<const SingularSystemError*>(&e)) return 7;
  return 3;
}

SpinnerVariant variant_of(int v) {  // spinner.hpp:18-25 order
  switch (v) {
    case 1: return SpinnerVariant::hdg_hd2_hd1;
    case 2: return SpinnerVariant::gcirc_d2_hd1;
    case 3: return SpinnerVariant::gtoeplitz_d2_hd1;
    case 4: return SpinnerVariant::gskew_circ_d2_hd1;
    case 5: return SpinnerVariant::gaussian_dense;
    default: return SpinnerVariant::hd3_hd2_hd1;
  }
}

Vec64 row_of(const float* x, std::int64_t ld, std::int64_t r, std::int64_t n_in, std::int64_t n) {
  Vec64 v(static_cast<std::size_t>(n), 0.0);
  for (std::int64_t i = 0; i < n_in; ++i) v[static_cast<std::size_t>(i)] = x[r * ld + i];
  return v;
}

// Run f(row) for row in [0,batch) on `threads` std::threads (the reference's
// apply/hash/embed are const and reentrant: SPEC.md:214).
template <class F>
int parallel_rows(std::int64_t batch, int threads, F f) {
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  std::vector<int> rc(static_cast<std::size_t>(threads), 0);
  std::vector<std::string> msg(static_cast<std::size_t>(threads));
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      try {
        for (std::int64_t r = t; r < batch; r += threads) f(r);
      } catch (const std::exception& e) {
        rc[static_cast<std::size_t>(t)] = fail(e);
        msg[static_cast<std::size_t>(t)] = g_err;
      }
    });
  }
  for (auto& th : pool) th.join();
  for (int t = 0; t < threads; ++t)
    if (rc[static_cast<std::size_t>(t)]) {
      g_err = msg[static_cast<std::size_t>(t)];
      return rc[static_cast<std::size_t>(t)];
    }
  return 0;
}

std::vector<StructuredSpinner> blocks_with_scale(SpinnerVariant v, std::int64_t n, std::int64_t m,
                                                 std::int64_t k, std::uint64_t seed, double scale) {
  StackedSpinner base(v, static_cast<std::size_t>(n), static_cast<std::size_t>(m),
                      static_cast<std::size_t>(k), seed);
  std::vector<StructuredSpinner> out;
  for (const auto& b : base.blocks()) {
    SpinnerSpec s = b.spec();
    s.scale = scale;  // 0 keeps default_scale (spinner.cpp:69-71)
    out.push_back(StructuredSpinner::build(s));
  }
  return out;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_mix_seed(std::uint64_t base, std::uint64_t stream) { return mix_seed(base, stream); }

// kind 0: next_u64, 1: uniform01, 2: gaussian, 3: rademacher
void ref_rng_stream(std::uint64_t seed, std::int64_t count, int kind, double* out_f, std::uint64_t* out_u) {
  Rng r(seed);
  for (std::int64_t i = 0; i < count; ++i) {
    switch (kind) {
      case 0: out_u[i] = r.next_u64(); break;
      case 1: out_f[i] = r.uniform01(); break;
      case 2: out_f[i] = r.gaussian(); break;
      default: out_f[i] = r.rademacher(); break;
    }
  }
}

int ref_fwht(double* x, std::int64_t n) {
  try {
    Vec64 v(x, x + n);
    v = fwht_normalized(std::move(v));
    std::memcpy(x, v.data(), sizeof(double) * static_cast<std::size_t>(n));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_signed_argmax(const double* y, std::int64_t len, std::int64_t* index, int* sign) {
  try {
    SignedIndex s = signed_argmax(Vec64(y, y + len));
    *index = static_cast<std::int64_t>(s.index);
    *sign = s.sign;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// StackedSpinner(v,n,m,k,seed) realised diagonals, [blocks][n] each (spinner.cpp:248-256).
std::int64_t ref_realize_stacked(int variant, std::int64_t n, std::int64_t m, std::int64_t k,
                                 std::uint64_t seed, double* d1, double* d2, double* d3) {
  try {
    StackedSpinner s(variant_of(variant), static_cast<std::size_t>(n), static_cast<std::size_t>(m),
                     static_cast<std::size_t>(k), seed);
    std::int64_t b = 0;
    for (const auto& blk : s.blocks()) {
      const Vec64& t = blk.spec().variant == SpinnerVariant::hdg_hd2_hd1 ? blk.g_diag() : blk.d3();
      std::copy(blk.d1().begin(), blk.d1().end(), d1 + b * n);
      std::copy(blk.d2().begin(), blk.d2().end(), d2 + b * n);
      std::copy(t.begin(), t.end(), d3 + b * n);
      ++b;
    }
    return b;
  } catch (const std::exception& e) {
    return -fail(e);
  }
}

// StackedSpinner::apply on fp32 rows (zero padded from n_in to n); scale 0 = default.
int ref_batch_apply(int variant, std::int64_t n, std::int64_t m, std::int64_t k, std::uint64_t seed,
                    double scale, const float* x, std::int64_t batch, std::int64_t ld,
                    std::int64_t n_in, int relu, double* y, int threads) {
  try {
    StackedSpinner st(blocks_with_scale(variant_of(variant), n, m, k, seed, scale),
                      static_cast<std::size_t>(k));
    return parallel_rows(batch, threads, [&](std::int64_t r) {
      Vec64 out = st.apply(row_of(x, ld, r, n_in, n));
      for (std::int64_t i = 0; i < k; ++i) {
        double v = out[static_cast<std::size_t>(i)];
        y[r * k + i] = (relu && v < 0.0) ? 0.0 : v;
      }
    });
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// CrossPolytopeHasher::hash via make_hasher_factory(v,n,m)(seed_t) per table
// (lsh.cpp:23-36).  ids = index + (sign<0 ? m : 0).
int ref_batch_hash(int variant, std::int64_t n, std::int64_t m, std::int64_t tables,
                   const std::uint64_t* table_seeds, const float* x, std::int64_t batch,
                   std::int64_t ld, std::int64_t n_in, std::int32_t* ids, int threads) {
  try {
    HasherFactory f = make_hasher_factory(variant_of(variant), static_cast<std::size_t>(n),
                                          static_cast<std::size_t>(m));
    std::vector<CrossPolytopeHasher> hs;
    for (std::int64_t t = 0; t < tables; ++t) hs.push_back(f(table_seeds[t]));
    return parallel_rows(batch, threads, [&](std::int64_t r) {
      Vec64 v = row_of(x, ld, r, n_in, n);
      for (std::int64_t t = 0; t < tables; ++t) {
        SignedIndex s = hs[static_cast<std::size_t>(t)].hash(v);
        ids[r * tables + t] = static_cast<std::int32_t>(s.index) + (s.sign < 0 ? static_cast<std::int32_t>(m) : 0);
      }
    });
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// embed(FeatureMap{StackedSpinner(v, n, min(n,d'), d', seed), kind}, x) (kernels.cpp:17-36);
// kind 0 gaussian (out [batch][2d']), 1 angular (out [batch][d']).
int ref_batch_embed(int variant, std::int64_t n, std::int64_t dprime, std::uint64_t seed, int kind,
                    double sigma, const float* x, std::int64_t batch, std::int64_t ld,
                    std::int64_t n_in, double* out, int threads) {
  try {
    FeatureMap fm{StackedSpinner(variant_of(variant), static_cast<std::size_t>(n),
                                 std::min(static_cast<std::size_t>(n), static_cast<std::size_t>(dprime)),
                                 static_cast<std::size_t>(dprime), seed),
                  kind == 1 ? KernelKind::angular() : KernelKind::gaussian(sigma)};
    const std::int64_t w = kind == 1 ? dprime : 2 * dprime;
    return parallel_rows(batch, threads, [&](std::int64_t r) {
      Vec64 e = embed(fm, row_of(x, ld, r, n_in, n));
      std::copy(e.begin(), e.end(), out + r * w);
    });
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// StructuredSpinner::build(SpinnerSpec::make(v, n, m, spec_seed)) then (mode 0)
// resample_last_block(tail_seed), (1) resample_tail(tail_seed) or (2) with_tail_vector(tail)
// (spinner.cpp:153-184), applied to fp32 rows: y [batch][m].  d1/d2/d3 (optional, [n]) receive the
// resulting spinner's d1, d2 and d3 (or g_diag).
int ref_block_resampled(int variant, std::int64_t n, std::int64_t m, std::uint64_t spec_seed, int mode,
                        std::uint64_t tail_seed, const double* tail, const float* x, std::int64_t batch,
                        double* y, double* d1, double* d2, double* d3) {
  try {
    StructuredSpinner b = StructuredSpinner::build(
        SpinnerSpec::make(variant_of(variant), static_cast<std::size_t>(n), static_cast<std::size_t>(m), spec_seed));
    StructuredSpinner r = mode == 0   ? b.resample_last_block(tail_seed)
                          : mode == 1 ? b.resample_tail(tail_seed)
                                      : b.with_tail_vector(Vec64(tail, tail + n));
    for (std::int64_t row = 0; row < batch; ++row) {
      Vec64 out = r.apply(row_of(x, n, row, n, n));
      std::copy(out.begin(), out.end(), y + row * m);
    }
    if (d1 && !r.d1().empty()) std::copy(r.d1().begin(), r.d1().end(), d1);
    if (d2 && !r.d2().empty()) std::copy(r.d2().begin(), r.d2().end(), d2);
    const Vec64& t = r.spec().variant == SpinnerVariant::hdg_hd2_hd1 ? r.g_diag() : r.d3();
    if (d3 && !t.empty()) std::copy(t.begin(), t.end(), d3);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// SketchOperator(v, input_dim, rows, seed).apply(A) restated over the real
// StackedSpinner (newton_sketch.cpp:74-101).  A is [input_dim][d] row-major
// fp32.  If row_list != NULL the builder-defined random-P mode is used instead:
// one full block (m = padded) and out[r] = norm * y[row_list[r]].
int ref_sketch(int variant, std::int64_t input_dim, std::int64_t rows, std::uint64_t seed,
               const float* a, std::int64_t d, std::int64_t ld_a, const std::int64_t* row_list,
               double* out, int threads) {
  try {
    const std::size_t padded = next_power_of_two(static_cast<std::size_t>(input_dim));
    const std::size_t block = row_list ? padded : std::min(static_cast<std::size_t>(rows), padded);
    const std::size_t k = row_list ? padded : static_cast<std::size_t>(rows);
    StackedSpinner proj(variant_of(variant), padded, block, k, seed);
    const double norm = 1.0 / std::sqrt(static_cast<double>(rows));
    return parallel_rows(d, threads, [&](std::int64_t c) {
      Vec64 col(padded, 0.0);
      for (std::int64_t i = 0; i < input_dim; ++i) col[static_cast<std::size_t>(i)] = a[i * ld_a + c];
      Vec64 y = proj.apply(col);
      for (std::int64_t r = 0; r < rows; ++r) {
        const std::size_t src = row_list ? static_cast<std::size_t>(row_list[r]) : static_cast<std::size_t>(r);
        out[r * d + c] = norm * y[src];
      }
    });
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Explicit-diagonal chain with the reference's own primitives
// (fwht_normalized / diag_matvec, transforms.cpp:52-71,228-235):
// y = relu?( scale * H D3 H D2 H D1 x ).  Used for configs whose diagonals the
// reference cannot realise itself (all-Gaussian, config 5).
int ref_batch_chain(std::int64_t n, const double* d1, const double* d2, const double* d3,
                    double scale, const float* x, std::int64_t batch, std::int64_t ld, int relu,
                    double* y, int threads) {
  try {
    Vec64 D1(d1, d1 + n), D2(d2, d2 + n), D3(d3, d3 + n);
    return parallel_rows(batch, threads, [&](std::int64_t r) {
      Vec64 v = fwht_normalized(diag_matvec(D1, row_of(x, ld, r, n, n)));
      v = fwht_normalized(diag_matvec(D2, v));
      v = fwht_normalized(diag_matvec(D3, v));
      for (std::int64_t i = 0; i < n; ++i) {
        double t = scale * v[static_cast<std::size_t>(i)];
        y[r * n + i] = (relu && t < 0.0) ? 0.0 : t;
      }
    });
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// gram_exact / gram_approx / gram_error (kernels.cpp:38-114), the reference's own code.
// points [count][dim] fp32 rows; kind 0 = gaussian(sigma), 1 = angular; out [count][count].
int ref_gram_exact(const float* points, std::int64_t count, std::int64_t dim, int kind, double sigma, double* out) {
  try {
    std::vector<Vec64> pts;
    for (std::int64_t i = 0; i < count; ++i) pts.push_back(row_of(points, dim, i, dim, dim));
    Eigen::MatrixXd g = gram_exact(pts, kind == 1 ? KernelKind::angular() : KernelKind::gaussian(sigma));
    for (std::int64_t i = 0; i < count; ++i)
      for (std::int64_t j = 0; j < count; ++j) out[i * count + j] = g(i, j);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_gram_approx(int variant, std::int64_t n, std::int64_t dprime, std::uint64_t seed, int kind, double sigma,
                    const float* points, std::int64_t count, double* out) {
  try {
    std::vector<Vec64> pts;
    for (std::int64_t i = 0; i < count; ++i) pts.push_back(row_of(points, n, i, n, n));
    FeatureMap fm{StackedSpinner(variant_of(variant), static_cast<std::size_t>(n),
                                 std::min(static_cast<std::size_t>(n), static_cast<std::size_t>(dprime)),
                                 static_cast<std::size_t>(dprime), seed),
                  kind == 1 ? KernelKind::angular() : KernelKind::gaussian(sigma)};
    Eigen::MatrixXd g = gram_approx(fm, pts);
    for (std::int64_t i = 0; i < count; ++i)
      for (std::int64_t j = 0; j < count; ++j) out[i * count + j] = g(i, j);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_gram_error(const double* exact, const double* approx, std::int64_t count, double* err) {
  try {
    Eigen::MatrixXd a(count, count), b(count, count);
    for (std::int64_t i = 0; i < count; ++i)
      for (std::int64_t j = 0; j < count; ++j) {
        a(i, j) = exact[i * count + j];
        b(i, j) = approx[i * count + j];
      }
    *err = gram_error(a, b);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// collision_curve(pairs, make_hasher_factory(v, n, m), trials, seed, buckets, max_distance)
// (lsh.cpp:38-74), the reference's own driver.  xs / ys: [pairs][n] fp32 rows.
int ref_collision_curve(int variant, std::int64_t n, std::int64_t m, const float* xs, const float* ys,
                        const double* dist, std::int64_t pairs, std::int64_t trials, std::uint64_t seed,
                        std::int64_t buckets, double max_distance, double* edges, double* probs,
                        std::uint64_t* counts) {
  try {
    std::vector<HashedPair> hp(static_cast<std::size_t>(pairs));
    for (std::int64_t p = 0; p < pairs; ++p) {
      hp[p].x = row_of(xs, n, p, n, n);
      hp[p].y = row_of(ys, n, p, n, n);
      hp[p].distance = dist[p];
    }
    CollisionCurve c = collision_curve(hp, make_hasher_factory(variant_of(variant), static_cast<std::size_t>(n),
                                                               static_cast<std::size_t>(m)),
                                       static_cast<std::size_t>(trials), seed, static_cast<std::size_t>(buckets),
                                       max_distance);
    for (std::int64_t b = 0; b <= buckets; ++b) edges[b] = c.bucket_edges[b];
    for (std::int64_t b = 0; b < buckets; ++b) {
      probs[b] = c.probabilities[b];
      counts[b] = c.counts[b];
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ------------------------------------------------------------ sketched Newton
// (newton_sketch.cpp, the reference's own functions).  Features are row-major
// fp64 [n][d]; variant < 0 selects the exact (identity) sketch.

namespace {
LogisticProblem problem_of(const double* a, const double* labels, std::int64_t n, std::int64_t d) {
  LogisticProblem p;
  p.features.resize(n, d);
  for (std::int64_t i = 0; i < n; ++i)
    for (std::int64_t j = 0; j < d; ++j) p.features(i, j) = a[i * d + j];
  p.labels.resize(n);
  for (std::int64_t i = 0; i < n; ++i) p.labels(i) = labels[i];
  return p;
}
Eigen::VectorXd vec_of(const double* x, std::int64_t d) {
  Eigen::VectorXd v(d);
  for (std::int64_t j = 0; j < d; ++j) v(j) = x[j];
  return v;
}
SketchOperator sketch_of(int variant, std::int64_t n, std::int64_t rows, std::uint64_t seed) {
  if (variant < 0) return SketchOperator();
  return SketchOperator(variant_of(variant), static_cast<std::size_t>(n), static_cast<std::size_t>(rows), seed);
}
}  // namespace

int ref_ar1_problem(std::int64_t n, std::int64_t d, std::uint64_t seed, double* features, double* labels) {
  try {
    LogisticProblem p = generate_ar1_problem(static_cast<std::size_t>(n), static_cast<std::size_t>(d), seed);
    for (std::int64_t i = 0; i < n; ++i) {
      for (std::int64_t j = 0; j < d; ++j) features[i * d + j] = p.features(i, j);
      labels[i] = p.labels(i);
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_logistic(const double* a, const double* labels, std::int64_t n, std::int64_t d, const double* x,
                 double* loss_out, double* grad_out, double* hsqrt_out) {
  try {
    LogisticProblem p = problem_of(a, labels, n, d);
    Eigen::VectorXd xv = vec_of(x, d);
    if (loss_out) *loss_out = loss(p, xv);
    if (grad_out) {
      Eigen::VectorXd g = gradient(p, xv);
      for (std::int64_t j = 0; j < d; ++j) grad_out[j] = g(j);
    }
    if (hsqrt_out) {
      Eigen::MatrixXd h = hessian_sqrt(p, xv);
      for (std::int64_t i = 0; i < n; ++i)
        for (std::int64_t j = 0; j < d; ++j) hsqrt_out[i * d + j] = h(i, j);
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_sketched_step(const double* a, const double* labels, std::int64_t n, std::int64_t d, const double* x,
                      int variant, std::int64_t rows, std::uint64_t seed, double* step_out) {
  try {
    LogisticProblem p = problem_of(a, labels, n, d);
    Eigen::VectorXd s = sketched_step(p, vec_of(x, d), sketch_of(variant, n, rows, seed));
    for (std::int64_t j = 0; j < d; ++j) step_out[j] = s(j);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// solve(): iterations run, per-iteration losses / gaps, final iterate, f_star, converged.
int ref_solve(const double* a, const double* labels, std::int64_t n, std::int64_t d, int variant,
              std::int64_t rows, std::int64_t max_iters, double gap_tol, int line_search, std::uint64_t seed,
              std::int64_t* iters, double* losses, double* gaps, double* x_final, double* f_star,
              int* converged) {
  try {
    LogisticProblem p = problem_of(a, labels, n, d);
    SketchConfig cfg;
    if (variant >= 0) cfg.sketch_variant = variant_of(variant);
    cfg.sketch_rows = static_cast<std::size_t>(rows);
    cfg.max_iters = static_cast<std::size_t>(max_iters);
    cfg.gap_tolerance = gap_tol;
    cfg.line_search = line_search != 0;
    cfg.seed = seed;
    NewtonTrace t = solve(p, cfg);
    *iters = static_cast<std::int64_t>(t.losses.size());
    for (std::size_t i = 0; i < t.losses.size(); ++i) {
      losses[i] = t.losses[i];
      gaps[i] = t.gaps[i];
    }
    const Eigen::VectorXd& xf = t.iterates.back();
    for (std::int64_t j = 0; j < d; ++j) x_final[j] = xf(j);
    *f_star = t.f_star;
    *converged = t.converged ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
