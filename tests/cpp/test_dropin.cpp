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

  test_case("sampler: distinct sorted indices", [] {
    auto r = sample_rows(1000, 100, 5);
    bool ok = r.size() == 100;
    for (std::size_t i = 1; i < r.size(); ++i) ok = ok && r[i] > r[i - 1];
    CHECK(ok && r.front() >= 0 && r.back() < 1000);
  });

  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ALL PASSED", g_fail);
  return g_fail ? 1 : 0;
}
