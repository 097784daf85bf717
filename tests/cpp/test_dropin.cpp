// C++ drop-in tests (GPU): the reference's own test cases, restated against
// include/spinners_b200.hpp, with the C oracle (oracle/spinner_oracle.c) as the
// independent checker.  Built and run by tests/test_cpp_dropin.py.
//   proj/tests/test_lsh.cpp:26-55, test_spinner.cpp:11-59,122-153, test_kernels.cpp:28-34
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/spinners_b200.hpp"
#include "../../oracle/spinner_oracle.h"

using namespace spinners_b200;

static int g_fail = 0;
#define CHECK(c)                                                            \
  do {                                                                      \
    if (!(c)) {                                                             \
      std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #c);          \
      ++g_fail;                                                             \
    }                                                                       \
  } while (0)

template <class F>
static void test_case(const char* name, F f) {
  const int before = g_fail;
  try {
    f();
  } catch (const std::exception& e) {
    std::printf("  EXCEPTION %s\n", e.what());
    ++g_fail;
  }
  std::printf("[case] %s: %s\n", name, g_fail == before ? "PASS" : "FAIL");
}

template <class E, class F>
static bool throws(F f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static Vec64 random_vec(std::size_t n, std::uint64_t seed) {  // oracles.hpp:106-112 (same generator)
  Vec64 x(n);
  orc_rng_fill(seed, 2, static_cast<int64_t>(n), x.data());
  return x;
}

static double max_abs_diff(const Vec64& a, const Vec64& b) {
  double m = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
  return m;
}

int main() {
  test_case("fwht_normalized KATs, involution and norm; diag_matvec (test_transforms.cpp:11-42,109-114)", [] {
    Vec64 h2 = fwht_normalized({1.0, 0.0});
    CHECK(std::abs(h2[0] - 1.0 / std::sqrt(2.0)) < 1e-6 && std::abs(h2[1] - 1.0 / std::sqrt(2.0)) < 1e-6);
    Vec64 h4 = fwht_normalized({1.0, 2.0, 3.0, 4.0});  // Sylvester H_4 / 2
    const Vec64 w4 = {5.0, -1.0, -2.0, 0.0};
    CHECK(max_abs_diff(h4, w4) < 1e-6);
    for (std::size_t n : {1u, 2u, 8u, 64u, 1024u, 16384u, 65536u}) {
      Vec64 x = random_vec(n, 900 + n), want = x;
      orc_fwht_normalized(want.data(), static_cast<int64_t>(n));
      Vec64 y = fwht_normalized(x);
      double nx = 0, ny = 0, err = 0;
      for (std::size_t i = 0; i < n; ++i) {
        nx += x[i] * x[i];
        ny += y[i] * y[i];
        err += (y[i] - want[i]) * (y[i] - want[i]);
      }
      CHECK(std::sqrt(err / nx) < 1e-5);         // against the fp64 restatement
      CHECK(std::abs(std::sqrt(ny / nx) - 1.0) < 1e-5);  // orthonormal
      Vec64 back = fwht_normalized(y);            // involution
      CHECK(max_abs_diff(back, x) < 1e-5 * std::sqrt(nx));
    }
    CHECK(throws<DimensionError>([] { fwht_normalized(Vec64(3, 1.0)); }));
    CHECK(throws<DimensionError>([] { fwht_normalized(Vec64()); }));
    CHECK(throws<DomainError>([] { fwht_normalized({1.0, NAN}); }));
    Vec64 dm = diag_matvec({2.0, -1.0, 0.5}, {1.0, 3.0, -4.0});
    CHECK((dm == Vec64{2.0, -3.0, -2.0}));
    CHECK(throws<DimensionError>([] { diag_matvec({1.0, 2.0}, {1.0}); }));
    CHECK(throws<DomainError>([] { diag_matvec({1.0, INFINITY}, {1.0, 2.0}); }));
  });

  test_case("circulant / Toeplitz / skew-circulant operators vs explicit matrices (oracles.hpp:35-58)", [] {
    for (std::size_t n : {1u, 3u, 8u, 100u, 256u}) {
      Vec64 r = random_vec(n, 70 + n), c = random_vec(n, 90 + n), x = random_vec(n, 110 + n);
      c[0] = r[0];
      Vec64 yc(n, 0.0), yt(n, 0.0), ys(n, 0.0);
      for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j) {
          yc[i] += r[(j + n - i) % n] * x[j];
          yt[i] += (i >= j ? c[i - j] : r[j - i]) * x[j];
          ys[i] += (j >= i ? r[j - i] : -r[n + j - i]) * x[j];
        }
      double sx = 0;
      for (double v : x) sx += v * v;
      const double tol = 1e-5 * std::sqrt(sx) * std::sqrt(static_cast<double>(n));
      CHECK(max_abs_diff(circulant_matvec(CirculantSpec::circulant(r), x), yc) < tol);
      CHECK(max_abs_diff(toeplitz_matvec(CirculantSpec::toeplitz(c, r), x), yt) < tol);
      CHECK(max_abs_diff(skew_circulant_matvec(CirculantSpec::skew_circulant(r), x), ys) < tol);
    }
    CHECK(throws<DomainError>([] { CirculantSpec::toeplitz({1.0, 2.0}, {2.0, 2.0}); }));
    CHECK(throws<DimensionError>([] { CirculantSpec::circulant({}); }));
    CHECK(throws<DomainError>([] { toeplitz_matvec(CirculantSpec::circulant({1.0, 2.0}), {1.0, 2.0}); }));
  });

  test_case("signed_argmax: direct example, ties, sign at zero", [] {
    SignedIndex h = signed_argmax({0.1, -0.9, 0.3});
    CHECK(h.index == 1 && h.sign == -1);
    CHECK((signed_argmax({-2.0, 2.0}) == SignedIndex{0, -1}));
    CHECK((signed_argmax({0.0, 0.0}) == SignedIndex{0, 1}));
  });

  test_case("hash: positive scale invariance, antisymmetry, determinism, zero input", [] {
    const std::size_t n = 16, m = 8;
    CrossPolytopeHasher h = make_hasher_factory(SpinnerVariant::hd3_hd2_hd1, n, m)(7);
    Vec64 x = random_vec(n, 1), x3(n), neg(n);
    for (std::size_t i = 0; i < n; ++i) {
      x3[i] = 3.0 * x[i];
      neg[i] = -x[i];
    }
    SignedIndex hx = h.hash(x);
    CHECK(h.hash(x3) == hx);
    CHECK(h.hash(x) == hx);
    SignedIndex hn = h.hash(neg);
    CHECK(hn.index == hx.index && hn.sign == -hx.sign);
    CHECK(throws<DomainError>([&] { h.hash(Vec64(n, 0.0)); }));
  });

  test_case("hash matches the oracle (n=1024, 64 unit vectors, seed 42)", [] {
    const std::size_t n = 1024;
    CrossPolytopeHasher h = make_hasher_factory(SpinnerVariant::hd3_hd2_hd1, n, n)(42);
    std::vector<double> d1(n), d2(n), d3(n);
    orc_realize_stacked(0, n, n, n, 42, d1.data(), d2.data(), d3.data());
    int bad = 0;
    for (int t = 0; t < 64; ++t) {
      Vec64 x = random_vec(n, 500 + t), y(n);
      orc_block_apply(n, n, 32.0, d1.data(), d2.data(), d3.data(), x.data(), y.data());
      int64_t idx;
      int sg;
      orc_signed_argmax(y.data(), n, &idx, &sg);
      const bool tie = orc_top2_gap(y.data(), n) < 1e-5;
      SignedIndex got = h.hash(x);
      if (!tie && !(got.index == static_cast<std::size_t>(idx) && got.sign == sg)) ++bad;
    }
    CHECK(bad == 0);
  });

  test_case("build is deterministic: same spec, bit-identical operator", [] {
    auto spec = SpinnerSpec::make(SpinnerVariant::hd3_hd2_hd1, 16, 8, 42);
    auto a = StructuredSpinner::build(spec);
    auto b = StructuredSpinner::build(spec);
    Vec64 x = random_vec(16, 7);
    CHECK(a.apply(x) == b.apply(x));
    CHECK(a.d1() == b.d1() && a.d3() == b.d3());
  });

  test_case("build(spec) for every variant equals the stacked plan's block 0; apply_front_blocks", [] {
    for (SpinnerVariant v : {SpinnerVariant::hd3_hd2_hd1, SpinnerVariant::hdg_hd2_hd1, SpinnerVariant::gcirc_d2_hd1,
                             SpinnerVariant::gtoeplitz_d2_hd1, SpinnerVariant::gskew_circ_d2_hd1,
                             SpinnerVariant::gaussian_dense}) {
      auto sp = StructuredSpinner::build(SpinnerSpec::make(v, 32, 24, mix_seed(99, 0)));
      StackedSpinner st(v, 32, 24, 24, 99);
      Vec64 x = random_vec(32, 5);
      CHECK(sp.apply(x) == st.apply(x));
      if (v == SpinnerVariant::gaussian_dense) {
        CHECK(throws<DomainError>([&] { sp.apply_front_blocks(x); }));
        continue;
      }
      Vec64 f(32);
      for (std::size_t i = 0; i < 32; ++i) f[i] = static_cast<double>(static_cast<float>(sp.d1()[i])) * x[i];
      orc_fwht_normalized(f.data(), 32);
      for (std::size_t i = 0; i < 32; ++i) f[i] *= static_cast<double>(static_cast<float>(sp.d2()[i]));
      if (v == SpinnerVariant::hd3_hd2_hd1 || v == SpinnerVariant::hdg_hd2_hd1) orc_fwht_normalized(f.data(), 32);
      CHECK(max_abs_diff(sp.apply_front_blocks(x), f) < 1e-5);
    }
  });

  test_case("HD3HD2HD1 with scale 1 is an isometry at m=n", [] {
    auto spec = SpinnerSpec::make(SpinnerVariant::hd3_hd2_hd1, 64, 64, 3);
    spec.scale = 1.0;
    auto sp = StructuredSpinner::build(spec);
    for (std::uint64_t t = 0; t < 20; ++t) {
      Vec64 x = random_vec(64, 100 + t);
      double nx = 0;
      for (double v : x) nx += v * v;
      for (double& v : x) v /= std::sqrt(nx);
      Vec64 y = sp.apply(x);
      double ny = 0;
      for (double v : y) ny += v * v;
      CHECK(std::abs(std::sqrt(ny) - 1.0) < 1e-5);
    }
  });

  test_case("apply matches the dense composition oracle (n=m=16, seed 21)", [] {
    auto hd = StructuredSpinner::build(SpinnerSpec::make(SpinnerVariant::hd3_hd2_hd1, 16, 16, 21));
    for (std::uint64_t t = 0; t < 10; ++t) {
      Vec64 x = random_vec(16, 300 + t), want(16);
      orc_block_apply(16, 16, 4.0, hd.d1().data(), hd.d2().data(), hd.d3().data(), x.data(), want.data());
      CHECK(max_abs_diff(hd.apply(x), want) < 1e-5 * 16);
    }
  });

  test_case("apply: zero maps to zero, dimension mismatch rejected", [] {
    auto sp = StructuredSpinner::build(SpinnerSpec::make(SpinnerVariant::hdg_hd2_hd1, 8, 4, 1));
    for (double v : sp.apply(Vec64(8, 0.0))) CHECK(v == 0.0);
    CHECK(throws<DimensionError>([&] { sp.apply(Vec64(4, 1.0)); }));
    CHECK(throws<DimensionError>([&] { SpinnerSpec::make(SpinnerVariant::hd3_hd2_hd1, 12, 4, 0); }));
  });

  test_case("stacked spinner: blocks are the independently seeded StructuredSpinners", [] {
    const std::size_t n = 16, m = 8;
    StackedSpinner two(SpinnerVariant::hd3_hd2_hd1, n, m, 2 * m, 33);
    Vec64 x = random_vec(n, 1);
    Vec64 y = two.apply(x);
    auto b0 = StructuredSpinner::build(SpinnerSpec::make(SpinnerVariant::hd3_hd2_hd1, n, m, mix_seed(33, 0)));
    auto b1 = StructuredSpinner::build(SpinnerSpec::make(SpinnerVariant::hd3_hd2_hd1, n, m, mix_seed(33, 1)));
    Vec64 y0 = b0.apply(x), y1 = b1.apply(x);
    for (std::size_t i = 0; i < m; ++i) {
      CHECK(std::abs(y[i] - y0[i]) < 1e-5);
      CHECK(std::abs(y[m + i] - y1[i]) < 1e-5);
    }
    CHECK(max_abs_diff(y0, y1) > 1e-6);
  });

  test_case("gaussian embedding has unit self-similarity", [] {
    FeatureMap fm{StackedSpinner(SpinnerVariant::hd3_hd2_hd1, 8, 8, 16, 3), KernelKind::gaussian(2.0)};
    Vec64 e = embed(fm, random_vec(8, 4));
    double dot = 0.0;
    for (double v : e) dot += v * v;
    CHECK(std::abs(dot - 1.0) < 1e-5);
    CHECK(throws<DomainError>([] { KernelKind::gaussian(0.0); }));
  });

  test_case("SketchOperator::apply(MatrixXd) value semantics, single and multi-block (newton_sketch.cpp:74-101)", [] {
    // {input_dim, rows}: rows <= padded (one block) and rows > padded (ceil(rows / padded) blocks)
    const std::size_t shapes[3][2] = {{200, 64}, {100, 300}, {1000, 2500}};
    for (const auto& sh : shapes) {
      const std::size_t in = sh[0], rows = sh[1], d = 7;
      std::size_t N = 1;
      while (N < in) N <<= 1;
      const std::size_t blocks = (rows + N - 1) / N, m = std::min(rows, N);
      MatrixXd A(static_cast<std::ptrdiff_t>(in), static_cast<std::ptrdiff_t>(d));
      Vec64 cols = random_vec(in * d, 41 + in);
      std::vector<float> af(in * d);
      for (std::size_t i = 0; i < in; ++i)
        for (std::size_t c = 0; c < d; ++c) {
          A(i, c) = static_cast<double>(static_cast<float>(cols[i * d + c]));
          af[i * d + c] = static_cast<float>(A(i, c));
        }
      SketchOperator sk(SpinnerVariant::hd3_hd2_hd1, in, rows, 55);
      MatrixXd S = sk.apply(A);
      CHECK(S.rows() == static_cast<std::ptrdiff_t>(rows) && S.cols() == static_cast<std::ptrdiff_t>(d));
      std::vector<double> d1(blocks * N), d2(blocks * N), d3(blocks * N);
      orc_realize_stacked(0, N, m, rows, 55, d1.data(), d2.data(), d3.data());
      double err = 0, nrm = 0;
      for (std::size_t b = 0; b < blocks; ++b) {
        const std::size_t mb = std::min(m, rows - b * m);
        std::vector<double> want(mb * d);
        orc_sketch(N, std::sqrt(double(N)), 1.0 / std::sqrt(double(rows)), d1.data() + b * N, d2.data() + b * N,
                   d3.data() + b * N, af.data(), in, d, d, nullptr, mb, want.data());
        for (std::size_t r = 0; r < mb; ++r)
          for (std::size_t c = 0; c < d; ++c) {
            const double e = S(b * m + r, c) - want[r * d + c];
            err += e * e;
            nrm += want[r * d + c] * want[r * d + c];
          }
      }
      CHECK(std::sqrt(err / nrm) < 1e-5);
      CHECK(throws<DimensionError>([&] { sk.apply(MatrixXd(static_cast<std::ptrdiff_t>(in + 1), 2)); }));
    }
    MatrixXd A(5, 2);
    CHECK(SketchOperator().apply(A).rows() == 5);  // exact operator: identity
  });

  test_case("hash_project_batch: ids and y of the same rows (BASELINE config 1)", [] {
    const std::size_t n = 1024, batch = 300;
    auto sp = StackedSpinner(SpinnerVariant::hd3_hd2_hd1, n, n, n, 42, 1.0);
    CrossPolytopeHasher h(sp);
    Vec64 xv = random_vec(n * batch, 7);
    std::vector<float> x(xv.begin(), xv.end()), y(n * batch);
    std::vector<int32_t> ids(batch), ids2(batch);
    h.hash_project_batch(x.data(), batch, n, n, ids.data(), y.data(), n);
    h.hash_batch(x.data(), batch, n, n, ids2.data());
    CHECK(ids == ids2);
    std::vector<double> d1(n), d2(n), d3(n), want(n * batch);
    orc_realize_stacked(0, n, n, n, 42, d1.data(), d2.data(), d3.data());
    orc_batch_apply(n, n, n, 1.0, d1.data(), d2.data(), d3.data(), x.data(), batch, n, n, 0, want.data());
    double worst = 0;
    for (std::size_t b = 0; b < batch; ++b) {
      double e = 0, w = 0;
      for (std::size_t i = 0; i < n; ++i) {
        e += (y[b * n + i] - want[b * n + i]) * (y[b * n + i] - want[b * n + i]);
        w += want[b * n + i] * want[b * n + i];
      }
      worst = std::max(worst, std::sqrt(e / w));
    }
    CHECK(worst < 1e-5);
  });

  test_case("resample_last_block / resample_tail / with_tail_vector (spinner.cpp:153-184)", [] {
    const std::size_t n = 32, m = 32;
    auto sp = StructuredSpinner::build(SpinnerSpec::make(SpinnerVariant::hd3_hd2_hd1, n, m, 19));
    auto r0 = sp.resample_last_block(5);
    CHECK(r0.d1() == sp.d1() && r0.d2() == sp.d2());
    Vec64 t(n);
    orc_rng_fill(orc_mix_seed(5, 2), 3, static_cast<int64_t>(n), t.data());  // Rng(mix_seed(s, 2)).rademacher()
    CHECK(r0.d3() == t);
    auto r1 = sp.resample_tail(6);
    Vec64 u(2 * n);
    orc_rng_fill(orc_mix_seed(6, 3), 3, static_cast<int64_t>(2 * n), u.data());  // D2 then D3 from one stream
    CHECK(r1.d1() == sp.d1() && r1.d2() == Vec64(u.begin(), u.begin() + n) && r1.d3() == Vec64(u.begin() + n, u.end()));
    Vec64 g = random_vec(n, 3);
    auto r2 = sp.with_tail_vector(g);
    CHECK(r2.d3() == g && r2.d1() == sp.d1());
    Vec64 x = random_vec(n, 4), want(n);
    orc_block_apply(n, m, std::sqrt(double(n)), r2.d1().data(), r2.d2().data(), g.data(), x.data(), want.data());
    double e = 0, w = 0;
    Vec64 got = r2.apply(x);
    for (std::size_t i = 0; i < n; ++i) {
      e += (got[i] - want[i]) * (got[i] - want[i]);
      w += want[i] * want[i];
    }
    CHECK(std::sqrt(e / w) < 1e-5);
    CHECK(throws<DimensionError>([&] { sp.with_tail_vector(Vec64(n - 1, 1.0)); }));
    auto dense = StructuredSpinner::build(SpinnerSpec::make(SpinnerVariant::gaussian_dense, 8, 4, 1));
    CHECK(throws<DomainError>([&] { dense.with_tail_vector(Vec64(8, 1.0)); }));
  });

  test_case("sampler: distinct sorted indices", [] {
    auto r = sample_rows(1000, 100, 5);
    bool ok = r.size() == 100;
    for (std::size_t i = 1; i < r.size(); ++i) ok = ok && r[i] > r[i - 1];
    CHECK(ok && r.front() >= 0 && r.back() < 1000);
  });

  // newton_sketch.cpp via the drop-in: loss / gradient / steps against the C oracle,
  // solve() convergence (proj/tests/test_newton.cpp-style properties)
  test_case("sketched Newton: loss, gradient, exact and sketched steps match the oracle", [] {
    const std::size_t n = 300, d = 12;
    LogisticProblem p = generate_ar1_problem(n, d, 5);
    std::vector<double> a(n * d), y(n);
    orc_ar1_problem(n, d, 5, a.data(), y.data());
    for (std::size_t i = 0; i < n * d; ++i) a[i] = static_cast<double>(static_cast<float>(a[i]));
    CHECK(p.labels == y);
    Vec64 x(d);
    for (std::size_t j = 0; j < d; ++j) x[j] = -0.1 + 0.2 * j / (d - 1);
    const double f = orc_logistic_loss(a.data(), y.data(), n, d, x.data());
    CHECK(std::abs(loss(p, x) - f) <= 1e-9 * std::abs(f));
    Vec64 g(d);
    orc_logistic_gradient(a.data(), y.data(), n, d, x.data(), g.data());
    CHECK(max_abs_diff(gradient(p, x), g) <= 1e-9);
    Vec64 s(d);
    CHECK(orc_sketched_step(a.data(), y.data(), n, d, x.data(), 0, 0, 0, 0, nullptr, nullptr, nullptr, s.data()) == 0);
    CHECK(max_abs_diff(sketched_step(p, x, SketchOperator()), s) <= 1e-8);
    const std::size_t N = 512, m = 64;
    std::vector<double> d1(N), d2(N), d3(N);
    orc_realize_stacked(0, N, m, m, 99, d1.data(), d2.data(), d3.data());
    CHECK(orc_sketched_step(a.data(), y.data(), n, d, x.data(), N, m, std::sqrt(double(N)), 1 / std::sqrt(double(m)),
                            d1.data(), d2.data(), d3.data(), s.data()) == 0);
    SketchOperator sk(SpinnerVariant::hd3_hd2_hd1, n, m, 99);
    CHECK(max_abs_diff(sketched_step(p, x, sk), s) <= 1e-5);
    CHECK(throws<DimensionError>([&] { sketched_step(p, x, SketchOperator(SpinnerVariant::hd3_hd2_hd1, n, 8, 1)); }));
  });

  test_case("sketched Newton: solve converges (exact and HD3 sketch) to the same optimum", [] {
    LogisticProblem p = generate_ar1_problem(300, 12, 5);
    SketchConfig ex;
    ex.max_iters = 30;
    NewtonTrace te = solve(p, ex);
    CHECK(te.converged && te.gaps.back() <= 1e-10);
    SketchConfig sk;
    sk.sketched = true;
    sk.sketch_rows = 64;
    sk.max_iters = 30;
    sk.seed = 7;
    NewtonTrace ts = solve(p, sk);
    CHECK(ts.converged && ts.gaps.back() <= 1e-10);
    CHECK(std::abs(ts.f_star - te.f_star) <= 1e-12 * std::abs(te.f_star));
    LogisticProblem z = generate_ar1_problem(300, 12, 5);
    for (double& v : z.features) v = 0.0;
    CHECK(throws<SingularSystemError>([&] { sketched_step(z, Vec64(12, 0.0), SketchOperator()); }));
  });

  test_case("collision_curve: identical / antipodal pairs, compare_families with equal seeds", [] {
    const std::size_t n = 16, m = 8;  // test_lsh.cpp:57-78,140-146
    auto factory = make_hasher_factory(SpinnerVariant::hd3_hd2_hd1, n, m);
    std::vector<HashedPair> same, anti;
    for (std::uint64_t p = 0; p < 20; ++p) {
      Vec64 x = random_vec(n, 100 + p), neg(n);
      for (std::size_t i = 0; i < n; ++i) neg[i] = -x[i];
      same.push_back(HashedPair{x, x, 0.0});
      anti.push_back(HashedPair{x, neg, 2.0});
    }
    CollisionCurve cs = collision_curve(same, factory, 5, 11);
    CHECK(cs.counts[0] == 100 && cs.probabilities[0] == 1.0 && std::isnan(cs.probabilities[1]) && cs.counts[1] == 0);
    CollisionCurve ca = collision_curve(anti, factory, 5, 11);
    CHECK(ca.probabilities[24] == 0.0);
    CHECK(compare_families(same, factory, factory, 5, 9, 9).sup_difference == 0.0);
    CHECK(throws<DimensionError>([&] { collision_curve(same, factory, 0, 1); }));
  });

  test_case("gram_exact / gram_approx / gram_error (test_kernels.cpp:55-133)", [] {
    Vec64 a = {1.0, 0.0}, b = {0.0, 1.0};
    GramMatrix ka = gram_exact({a, a, b}, KernelKind::angular());
    CHECK(std::abs(ka(0, 1) - 1.0) < 1e-15 && std::abs(ka(0, 2) - 0.5) < 1e-15);
    CHECK(throws<DomainError>([] { gram_exact({Vec64{0.0, 0.0}}, KernelKind::angular()); }));
    FeatureMap fm{StackedSpinner(SpinnerVariant::hd3_hd2_hd1, 8, 8, 8, 8), KernelKind::angular()};
    Vec64 x = random_vec(8, 9), neg(8);
    for (std::size_t i = 0; i < 8; ++i) neg[i] = -x[i];
    GramMatrix k = gram_approx(fm, {x, neg});
    CHECK(k(0, 0) == 1.0 && k(1, 1) == 1.0 && std::abs(k(0, 1)) < 1e-15);
    GramMatrix id{2, {1.0, 0.0, 0.0, 1.0}}, kt{2, {1.0, 0.1, 0.1, 1.0}};
    CHECK(gram_error(id, id) == 0.0);
    CHECK(std::abs(gram_error(id, kt) - 0.1) < 1e-13);
  });

  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ALL PASSED", g_fail);
  return g_fail ? 1 : 0;
}
