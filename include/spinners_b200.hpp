// spinners_b200.hpp — C++ drop-in for the reference's hot-path entry points.
//
// Same names, argument meaning and error behaviour as the reference headers
// (proj/include/spinners/{common,spinner,lsh,kernels,newton_sketch}.hpp), in
// namespace spinners_b200, implemented over the C ABI of spinners_b200.h (link
// with -lspinners_b200).  Differences a caller should know:
//   * arithmetic is fp32 on the GPU (inputs rounded to fp32, outputs widened back
//     to double); results match the reference within 1e-5 relative L2 per vector,
//     bucket ids exactly except near-ties (top-two |y| within 1e-5 relative);
//   * every class additionally offers batch entry points on contiguous float rows
//     (host pointers: *_batch; device pointers: *_device with a cudaStream_t);
//   * Eigen is not required: SketchOperator::apply takes a row-major n x d buffer.
#pragma once

#include <chrono>
#include <cmath>
#include <cstdint>
#include <tuple>
#include <utility>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "spinners_b200.h"

namespace spinners_b200 {

using Vec64 = std::vector<double>;  // common.hpp:13

struct DimensionError : std::invalid_argument {  // common.hpp:15-17
  using std::invalid_argument::invalid_argument;
};
struct DomainError : std::domain_error {  // common.hpp:19-21
  using std::domain_error::domain_error;
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SingularSystemError : std::runtime_error {  // common.hpp:25-27
  using std::runtime_error::runtime_error;
};

inline void check(spn_status s) {
  if (s == SPN_OK) return;
  std::string msg = std::string(spn_status_string(s)) + ": " + spn_last_error();
  if (s == SPN_EDIM) throw DimensionError(msg);
  if (s == SPN_EDOMAIN) throw DomainError(msg);
  if (s == SPN_ESINGULAR) throw SingularSystemError(msg);
  throw DeviceError(msg);
}

inline std::uint64_t mix_seed(std::uint64_t base, std::uint64_t stream) { return spn_mix_seed(base, stream); }

inline void check_finite(const Vec64& x, const char* what) {  // common.hpp:37-41
  for (double v : x)
    if (!std::isfinite(v)) throw DomainError(std::string(what) + ": non-finite entry");
}

// transforms.hpp:13 / transforms.cpp:52-71 — the orthonormal Walsh-Hadamard transform, on the device
inline Vec64 fwht_normalized(Vec64 x) {
  const std::size_t n = x.size();
  if (n == 0 || (n & (n - 1)) != 0)
    throw DimensionError("fwht_normalized: length must be a power of two, got " + std::to_string(n));
  check_finite(x, "fwht_normalized");
  std::vector<float> xf(x.begin(), x.end()), yf(n);
  check(spn_fwht_f32_host(static_cast<int64_t>(n), xf.data(), 1, static_cast<int64_t>(n), yf.data(),
                          static_cast<int64_t>(n), 0));
  return Vec64(yf.begin(), yf.end());
}

// transforms.hpp:59 / transforms.cpp:228-235 — y = d (.) x, on the device
inline Vec64 diag_matvec(const Vec64& d, const Vec64& x) {
  if (d.size() != x.size())
    throw DimensionError("diag_matvec: length mismatch (" + std::to_string(d.size()) + " vs " +
                         std::to_string(x.size()) + ")");
  check_finite(d, "diag_matvec.d");
  check_finite(x, "diag_matvec.x");
  if (x.empty()) return Vec64();
  std::vector<float> df(d.begin(), d.end()), xf(x.begin(), x.end()), yf(x.size());
  const auto n = static_cast<int64_t>(x.size());
  check(spn_diag_f32_host(n, df.data(), xf.data(), 1, n, yf.data(), n, 0));
  return Vec64(yf.begin(), yf.end());
}

// transforms.hpp:15-56 — circulant-family operators; spectrum on the host (as the reference builds
// it), the fp64 correlation on the device
enum class CirculantKind { circulant = 0, toeplitz = 1, skew_circulant = 2 };

struct CirculantSpec {  // transforms.hpp:22-35
  CirculantKind kind = CirculantKind::circulant;
  Vec64 first_row;
  Vec64 first_col;  // toeplitz only; first_col[0] must equal first_row[0]

  static CirculantSpec circulant(Vec64 r) {
    CirculantSpec s;
    s.first_row = std::move(r);
    s.validate();
    return s;
  }
  static CirculantSpec toeplitz(Vec64 col, Vec64 row) {
    CirculantSpec s;
    s.kind = CirculantKind::toeplitz;
    s.first_col = std::move(col);
    s.first_row = std::move(row);
    s.validate();
    return s;
  }
  static CirculantSpec skew_circulant(Vec64 r) {
    CirculantSpec s;
    s.kind = CirculantKind::skew_circulant;
    s.first_row = std::move(r);
    s.validate();
    return s;
  }
  std::size_t dim() const { return first_row.size(); }
  void validate() const {  // transforms.cpp:98-110
    if (first_row.empty()) throw DimensionError("CirculantSpec: n must be >= 1");
    check_finite(first_row, "CirculantSpec.first_row");
    if (kind == CirculantKind::toeplitz) {
      if (first_col.size() != first_row.size())
        throw DimensionError("CirculantSpec: toeplitz first_col/first_row length mismatch");
      check_finite(first_col, "CirculantSpec.first_col");
      if (first_col[0] != first_row[0]) throw DomainError("CirculantSpec: toeplitz corner entry mismatch");
    } else if (!first_col.empty()) {
      throw DimensionError("CirculantSpec: first_col only valid for toeplitz");
    }
  }
};

class CirculantOperator {  // transforms.hpp:37-51
 public:
  explicit CirculantOperator(CirculantSpec spec, int device = 0) : spec_(std::move(spec)) {
    spec_.validate();
    spn_circulant* h = nullptr;
    check(spn_circulant_create(&h, static_cast<int32_t>(spec_.kind), static_cast<int64_t>(spec_.dim()),
                               spec_.first_row.data(),
                               spec_.kind == CirculantKind::toeplitz ? spec_.first_col.data() : nullptr, device));
    op_.reset(h, [](spn_circulant* q) { spn_circulant_destroy(q); });
  }
  Vec64 apply(const Vec64& x) const {
    const std::size_t n = spec_.dim();
    if (x.size() != n)
      throw DimensionError("CirculantOperator::apply: expected length " + std::to_string(n) + ", got " +
                           std::to_string(x.size()));
    check_finite(x, "CirculantOperator::apply");
    std::vector<float> xf(x.begin(), x.end()), yf(n);
    check(spn_circulant_apply_f32_host(op_.get(), xf.data(), 1, static_cast<int64_t>(n), yf.data(),
                                       static_cast<int64_t>(n)));
    return Vec64(yf.begin(), yf.end());
  }
  // new: device buffers, [batch][ld] rows, stream-ordered
  void apply_device(const float* x, std::size_t batch, std::size_t ld_x, float* y, std::size_t ld_y,
                    void* stream = nullptr) const {
    check(spn_circulant_apply_f32(op_.get(), x, static_cast<int64_t>(batch), static_cast<int64_t>(ld_x), y,
                                  static_cast<int64_t>(ld_y), stream));
  }
  const CirculantSpec& spec() const { return spec_; }

 private:
  CirculantSpec spec_;
  std::shared_ptr<spn_circulant> op_;
};

inline Vec64 circulant_matvec(const CirculantSpec& spec, const Vec64& x) {  // transforms.cpp:210-214
  if (spec.kind != CirculantKind::circulant) throw DomainError("circulant_matvec: spec is not circulant");
  return CirculantOperator(spec).apply(x);
}
inline Vec64 toeplitz_matvec(const CirculantSpec& spec, const Vec64& x) {  // transforms.cpp:216-220
  if (spec.kind != CirculantKind::toeplitz) throw DomainError("toeplitz_matvec: spec is not toeplitz");
  return CirculantOperator(spec).apply(x);
}
inline Vec64 skew_circulant_matvec(const CirculantSpec& spec, const Vec64& x) {  // transforms.cpp:222-226
  if (spec.kind != CirculantKind::skew_circulant)
    throw DomainError("skew_circulant_matvec: spec is not skew-circulant");
  return CirculantOperator(spec).apply(x);
}

enum class SpinnerVariant {  // spinner.hpp:18-25
  hd3_hd2_hd1 = SPN_HD3_HD2_HD1,
  hdg_hd2_hd1 = SPN_HDG_HD2_HD1,
  gcirc_d2_hd1 = SPN_GCIRC_D2_HD1,
  gtoeplitz_d2_hd1 = SPN_GTOEPLITZ_D2_HD1,
  gskew_circ_d2_hd1 = SPN_GSKEW_CIRC_D2_HD1,
  gaussian_dense = SPN_GAUSSIAN_DENSE,
  gauss3 = SPN_GAUSS3
};

inline bool has_hadamard(SpinnerVariant v) { return v != SpinnerVariant::gaussian_dense; }  // spinner.cpp:38

inline const char* to_string(SpinnerVariant v) {  // spinner.cpp:9-19
  switch (v) {
    case SpinnerVariant::hd3_hd2_hd1: return "HD3HD2HD1";
    case SpinnerVariant::hdg_hd2_hd1: return "HDgHD2HD1";
    case SpinnerVariant::gcirc_d2_hd1: return "GcircD2HD1";
    case SpinnerVariant::gtoeplitz_d2_hd1: return "GToeplitzD2HD1";
    case SpinnerVariant::gskew_circ_d2_hd1: return "GSkewCircD2HD1";
    case SpinnerVariant::gaussian_dense: return "GaussianDense";
    case SpinnerVariant::gauss3: return "Gauss3";
  }
  throw DomainError("to_string: unknown variant");
}

inline std::vector<SpinnerVariant> all_variants() {  // spinner.cpp:27-31
  return {SpinnerVariant::hd3_hd2_hd1,       SpinnerVariant::hdg_hd2_hd1,       SpinnerVariant::gcirc_d2_hd1,
          SpinnerVariant::gtoeplitz_d2_hd1, SpinnerVariant::gskew_circ_d2_hd1, SpinnerVariant::gaussian_dense};
}

inline std::vector<SpinnerVariant> structured_variants() {  // spinner.cpp:33-37
  std::vector<SpinnerVariant> v = all_variants();
  v.pop_back();
  return v;
}

inline SpinnerVariant variant_from_string(const std::string& s) {  // spinner.cpp:21-25
  for (SpinnerVariant v : all_variants())
    if (s == to_string(v)) return v;
  throw DomainError("unknown spinner variant: " + s);
}

inline double default_scale(SpinnerVariant v, std::size_t n) {  // spinner.cpp:40-45
  if (v == SpinnerVariant::hd3_hd2_hd1 || v == SpinnerVariant::hdg_hd2_hd1 || v == SpinnerVariant::gauss3)
    return std::sqrt(static_cast<double>(n));
  return 1.0;
}

struct SpinnerSpec {  // spinner.hpp:40-53
  SpinnerVariant variant = SpinnerVariant::hd3_hd2_hd1;
  std::size_t n = 0, m = 0;
  std::uint64_t seed = 0;
  double scale = 0.0;  // 0 => default_scale

  static SpinnerSpec make(SpinnerVariant v, std::size_t n, std::size_t m, std::uint64_t seed) {
    SpinnerSpec s{v, n, m, seed, 0.0};
    s.validate();
    return s;
  }
  void validate() const {  // spinner.cpp:59-67
    if (n < 1) throw DimensionError("SpinnerSpec: n must be >= 1");
    if (m < 1 || m > n) throw DimensionError("SpinnerSpec: need 1 <= m <= n");
    if (has_hadamard(variant) && (n & (n - 1)) != 0)
      throw DimensionError("SpinnerSpec: Hadamard-bearing variant requires power-of-two n, got " +
                           std::to_string(n));
    if (scale != 0.0 && !std::isfinite(scale)) throw DomainError("SpinnerSpec: non-finite scale");
  }
  double effective_scale() const { return scale == 0.0 ? default_scale(variant, n) : scale; }
};

namespace detail {
struct PlanDeleter {
  void operator()(spn_plan* p) const { spn_plan_destroy(p); }
};
using Plan = std::shared_ptr<spn_plan>;

inline std::vector<float> to_f32(const Vec64& x) { return std::vector<float>(x.begin(), x.end()); }
}  // namespace detail

// k x n stack of ceil(k/m) blocks, block b seeded mix_seed(seed, b) (spinner.cpp:248-283).
class StackedSpinner {
 public:
  StackedSpinner(SpinnerVariant v, std::size_t n, std::size_t m, std::size_t k, std::uint64_t seed,
                 double scale = 0.0, int device = 0)
      : n_(n), k_(k), device_(device) {
    if (k < 1) throw DimensionError("StackedSpinner: k must be >= 1");
    spn_plan_desc d{static_cast<int32_t>(v), static_cast<int64_t>(n), static_cast<int64_t>(m),
                    static_cast<int64_t>(k), 1, nullptr, seed, scale, device};
    spn_plan* p = nullptr;
    check(spn_plan_create(&p, &d));
    plan_ = detail::Plan(p, detail::PlanDeleter{});
  }

  std::size_t rows() const { return k_; }
  std::size_t input_dim() const { return n_; }
  int device() const { return device_; }
  const spn_plan* plan() const { return plan_.get(); }

  // Single vector, like StackedSpinner::apply (spinner.cpp:272-283).
  Vec64 apply(const Vec64& x) const {
    if (x.size() != n_)
      throw DimensionError("StructuredSpinner::apply: expected length " + std::to_string(n_) + ", got " +
                           std::to_string(x.size()));
    check_finite(x, "StructuredSpinner::apply");
    std::vector<float> xf = detail::to_f32(x), y(k_);
    check(spn_apply_f32_host(plan_.get(), xf.data(), 1, static_cast<int64_t>(n_), static_cast<int64_t>(n_),
                             y.data(), static_cast<int64_t>(k_), 0));
    return Vec64(y.begin(), y.end());
  }
  // Batch on host rows (x: batch x ld_x floats, first n_in used, zero padded to n).
  void apply_batch(const float* x, std::size_t batch, std::size_t ld_x, std::size_t n_in, float* y,
                   std::size_t ld_y, bool relu = false) const {
    check(spn_apply_f32_host(plan_.get(), x, static_cast<int64_t>(batch), static_cast<int64_t>(ld_x),
                             static_cast<int64_t>(n_in), y, static_cast<int64_t>(ld_y), relu ? 1 : 0));
  }
  // Batch on device rows, stream-ordered.
  void apply_device(const float* x, std::size_t batch, std::size_t ld_x, std::size_t n_in, float* y,
                    std::size_t ld_y, bool relu, void* stream) const {
    check(spn_apply_f32(plan_.get(), x, static_cast<int64_t>(batch), static_cast<int64_t>(ld_x),
                        static_cast<int64_t>(n_in), y, static_cast<int64_t>(ld_y), relu ? 1 : 0, stream));
  }

 protected:
  StackedSpinner() = default;
  detail::Plan plan_;
  std::size_t n_ = 0, k_ = 0;
  int device_ = 0;
};

// One realised m x n block (spinner.hpp:56-104), diagonals drawn from spec.seed.
class StructuredSpinner : public StackedSpinner {
 public:
  static StructuredSpinner build(const SpinnerSpec& spec, int device = 0) {
    spec.validate();
    spn_plan* p = nullptr;  // every variant, drawn from spec.seed itself (spinner.cpp:137-151)
    check(spn_plan_create_block(&p, static_cast<int32_t>(spec.variant), static_cast<int64_t>(spec.n),
                                static_cast<int64_t>(spec.m), spec.seed, spec.scale, device));
    return wrap(p, spec, device);
  }
  // spinner.hpp:67-69 / spinner.cpp:153-158: M1, M2 kept, the last block redrawn from mix_seed(tail_seed, 2)
  StructuredSpinner resample_last_block(std::uint64_t tail_seed) const {
    spn_plan* p = nullptr;
    check(spn_plan_resample(&p, plan_.get(), 0, tail_seed));
    return wrap(p, spec_, device_);
  }
  // spinner.hpp:71-73 / spinner.cpp:160-166: D2 and the last block redrawn from mix_seed(tail_seed, 3)
  StructuredSpinner resample_tail(std::uint64_t tail_seed) const {
    spn_plan* p = nullptr;
    check(spn_plan_resample(&p, plan_.get(), 1, tail_seed));
    return wrap(p, spec_, device_);
  }
  // spinner.hpp:75-77 / spinner.cpp:168-184: D3 (HD3) or g (HDg) replaced by r
  StructuredSpinner with_tail_vector(Vec64 r) const {
    if (r.size() != spec_.n) throw DimensionError("with_tail_vector: length mismatch");
    check_finite(r, "with_tail_vector");
    spn_plan* p = nullptr;
    check(spn_plan_with_tail(&p, plan_.get(), r.data()));
    return wrap(p, spec_, device_);
  }
  // M2 M1 x (spinner.cpp:186-198): H D2 H D1 x for the Hadamard-only variants, D2 H D1 x for the
  // circulant family — on the spinner's device (the D2 H D1 chain, plus one normalised FWHT)
  Vec64 apply_front_blocks(const Vec64& x) const {
    if (!has_hadamard(spec_.variant)) throw DomainError("apply_front_blocks: dense baseline has no block structure");
    if (x.size() != spec_.n) throw DimensionError("apply_front_blocks: length mismatch");
    check_finite(x, "apply_front_blocks");
    const auto n = static_cast<int64_t>(spec_.n);
    if (!front_) {  // H (1) H D2 H D1 = D2 H D1 (H H = I), scale 1; made once per spinner
      Vec64 ones(spec_.n, 1.0);
      spn_plan* p = nullptr;
      check(spn_plan_create_explicit(&p, n, n, n, 1, d1_.data(), d2_.data(), ones.data(), 1.0, device_));
      front_ = detail::Plan(p, detail::PlanDeleter{});
    }
    std::vector<float> xf = detail::to_f32(x), y(spec_.n);
    check(spn_apply_f32_host(front_.get(), xf.data(), 1, n, n, y.data(), n, 0));
    const bool hadamard_only = spec_.variant == SpinnerVariant::hd3_hd2_hd1 ||
                               spec_.variant == SpinnerVariant::hdg_hd2_hd1 || spec_.variant == SpinnerVariant::gauss3;
    if (hadamard_only) check(spn_fwht_f32_host(n, y.data(), 1, n, y.data(), n, device_));
    return Vec64(y.begin(), y.end());
  }
  const SpinnerSpec& spec() const { return spec_; }
  const Vec64& d1() const { return d1_; }
  const Vec64& d2() const { return d2_; }
  const Vec64& d3() const { return d3_; }      // HD3HD2HD1
  const Vec64& g_diag() const { return d3_; }  // HDgHD2HD1

 private:
  static StructuredSpinner wrap(spn_plan* p, const SpinnerSpec& spec, int device) {
    StructuredSpinner s;
    s.plan_ = detail::Plan(p, detail::PlanDeleter{});
    s.spec_ = spec;
    s.n_ = spec.n;
    s.k_ = spec.m;
    s.device_ = device;
    s.d1_.resize(spec.n);
    s.d2_.resize(spec.n);
    s.d3_.resize(spec.n);
    check(spn_plan_diagonals(p, s.d1_.data(), s.d2_.data(), s.d3_.data()));
    return s;
  }
  SpinnerSpec spec_;
  Vec64 d1_, d2_, d3_;
  mutable detail::Plan front_;
};

struct SignedIndex {  // lsh.hpp:13-17
  std::size_t index = 0;
  int sign = 1;
  bool operator==(const SignedIndex&) const = default;
};

inline SignedIndex signed_argmax(const Vec64& y) {  // lsh.cpp:9-21
  if (y.empty()) throw DimensionError("signed_argmax: empty vector");
  std::size_t best = 0;
  double best_abs = std::abs(y[0]);
  for (std::size_t i = 1; i < y.size(); ++i)
    if (std::abs(y[i]) > best_abs) {
      best_abs = std::abs(y[i]);
      best = i;
    }
  return SignedIndex{best, y[best] < 0.0 ? -1 : 1};
}

inline SignedIndex decode_bucket(int32_t id, std::size_t k) {
  return static_cast<std::size_t>(id) >= k ? SignedIndex{static_cast<std::size_t>(id) - k, -1}
                                           : SignedIndex{static_cast<std::size_t>(id), 1};
}

class CrossPolytopeHasher {  // lsh.hpp:26-36
 public:
  explicit CrossPolytopeHasher(StackedSpinner projector) : projector_(std::move(projector)) {}

  SignedIndex hash(const Vec64& x) const {  // lsh.cpp:23-30
    check_finite(x, "CrossPolytopeHasher::hash");
    bool zero = true;
    for (double v : x)
      if (v != 0.0) {
        zero = false;
        break;
      }
    if (zero) throw DomainError("CrossPolytopeHasher::hash: zero vector");
    if (x.size() != projector_.input_dim()) throw DimensionError("CrossPolytopeHasher::hash: length mismatch");
    std::vector<float> xf = detail::to_f32(x);
    int32_t id = 0;
    check(spn_hash_f32_host(projector_.plan(), xf.data(), 1, static_cast<int64_t>(xf.size()),
                            static_cast<int64_t>(xf.size()), &id));
    return decode_bucket(id, projector_.rows());
  }
  // int32 bucket ids (index + k if negative) for a batch of host rows.
  void hash_batch(const float* x, std::size_t batch, std::size_t ld_x, std::size_t n_in, int32_t* ids) const {
    check(spn_hash_f32_host(projector_.plan(), x, static_cast<int64_t>(batch), static_cast<int64_t>(ld_x),
                            static_cast<int64_t>(n_in), ids));
  }
  // ids and the projection y = scale * stacked(x) of the same host rows in one call (BASELINE config 1)
  void hash_project_batch(const float* x, std::size_t batch, std::size_t ld_x, std::size_t n_in, int32_t* ids,
                          float* y, std::size_t ld_y) const {
    check(spn_hash_project_f32_host(projector_.plan(), x, static_cast<int64_t>(batch), static_cast<int64_t>(ld_x),
                                    static_cast<int64_t>(n_in), ids, y, static_cast<int64_t>(ld_y)));
  }
  void hash_device(const float* x, std::size_t batch, std::size_t ld_x, std::size_t n_in, int32_t* ids,
                   void* stream) const {
    check(spn_hash_f32(projector_.plan(), x, static_cast<int64_t>(batch), static_cast<int64_t>(ld_x),
                       static_cast<int64_t>(n_in), ids, nullptr, 0, stream));
  }
  const StackedSpinner& projector() const { return projector_; }

 private:
  StackedSpinner projector_;
};

using HasherFactory = std::function<CrossPolytopeHasher(std::uint64_t seed)>;

inline HasherFactory make_hasher_factory(SpinnerVariant v, std::size_t n, std::size_t m) {  // lsh.cpp:32-36
  return [v, n, m](std::uint64_t seed) {
    return CrossPolytopeHasher(StackedSpinner(v, n, std::min(m, n), m, seed));
  };
}

// ------------------------------------------------------------------ collision curves
struct HashedPair {  // lsh.hpp:38-44
  Vec64 x;
  Vec64 y;
  double distance = 0.0;
};

struct CollisionCurve {  // lsh.hpp:46-50
  std::vector<double> bucket_edges;
  std::vector<double> probabilities;  // NaN where a bucket saw no pairs
  std::vector<std::size_t> counts;
};

// lsh.cpp:38-74.  Every trial's hasher hashes all 2 * pairs vectors in one device batch.
inline CollisionCurve collision_curve(const std::vector<HashedPair>& pairs, const HasherFactory& factory,
                                      std::size_t trials, std::uint64_t seed, std::size_t buckets = 25,
                                      double max_distance = 2.0) {
  if (trials < 1) throw DimensionError("collision_curve: trials must be >= 1");
  if (buckets < 1) throw DimensionError("collision_curve: need at least one bucket");
  const std::size_t P = pairs.size();
  std::vector<std::size_t> bucket_of(P);
  const double width = max_distance / static_cast<double>(buckets);
  for (std::size_t p = 0; p < P; ++p) {
    const double d = pairs[p].distance;
    if (d < 0.0 || !std::isfinite(d)) throw DomainError("collision_curve: distances must be finite and nonnegative");
    bucket_of[p] = std::min(static_cast<std::size_t>(d / width), buckets - 1);
  }
  std::vector<std::size_t> counts(buckets, 0), hits(buckets, 0);
  if (P > 0) {
    const std::size_t n = pairs[0].x.size();
    std::vector<float> xy(2 * P * n);
    for (std::size_t p = 0; p < P; ++p) {
      if (pairs[p].x.size() != n || pairs[p].y.size() != n)
        throw DimensionError("CrossPolytopeHasher::hash: length mismatch");
      for (const Vec64* v : {&pairs[p].x, &pairs[p].y}) {
        check_finite(*v, "CrossPolytopeHasher::hash");
        bool zero = true;
        for (double e : *v) zero = zero && e == 0.0;
        if (zero) throw DomainError("CrossPolytopeHasher::hash: zero vector");
      }
      for (std::size_t i = 0; i < n; ++i) {
        xy[(2 * p) * n + i] = static_cast<float>(pairs[p].x[i]);
        xy[(2 * p + 1) * n + i] = static_cast<float>(pairs[p].y[i]);
      }
    }
    std::vector<int32_t> ids(2 * P);
    for (std::size_t t = 0; t < trials; ++t) {
      const CrossPolytopeHasher hasher = factory(mix_seed(seed, t));
      hasher.hash_batch(xy.data(), 2 * P, n, n, ids.data());
      for (std::size_t p = 0; p < P; ++p) {
        counts[bucket_of[p]]++;
        if (ids[2 * p] == ids[2 * p + 1]) hits[bucket_of[p]]++;
      }
    }
  }
  CollisionCurve curve;
  curve.bucket_edges.resize(buckets + 1);
  for (std::size_t b = 0; b <= buckets; ++b) curve.bucket_edges[b] = width * static_cast<double>(b);
  curve.counts = counts;
  curve.probabilities.resize(buckets);
  for (std::size_t b = 0; b < buckets; ++b)
    curve.probabilities[b] = counts[b] == 0 ? std::nan("")
                                            : static_cast<double>(hits[b]) / static_cast<double>(counts[b]);
  return curve;
}

struct FamilyComparison {  // lsh.hpp:68-73
  CollisionCurve curve_a, curve_b;
  std::vector<double> bucket_differences;
  double sup_difference = 0.0;
};

inline FamilyComparison compare_families(const std::vector<HashedPair>& pairs, const HasherFactory& family_a,
                                         const HasherFactory& family_b, std::size_t trials, std::uint64_t seed_a,
                                         std::uint64_t seed_b, std::size_t buckets = 25,
                                         double max_distance = 2.0) {  // lsh.cpp:76-96
  FamilyComparison cmp;
  cmp.curve_a = collision_curve(pairs, family_a, trials, seed_a, buckets, max_distance);
  cmp.curve_b = collision_curve(pairs, family_b, trials, seed_b, buckets, max_distance);
  cmp.bucket_differences.resize(buckets);
  for (std::size_t b = 0; b < buckets; ++b) {
    const double pa = cmp.curve_a.probabilities[b], pb = cmp.curve_b.probabilities[b];
    if (std::isnan(pa) || std::isnan(pb)) {
      cmp.bucket_differences[b] = std::nan("");
    } else {
      cmp.bucket_differences[b] = std::abs(pa - pb);
      cmp.sup_difference = std::max(cmp.sup_difference, cmp.bucket_differences[b]);
    }
  }
  return cmp;
}

struct KernelKind {  // kernels.hpp:11-24
  enum class Tag { gaussian, angular };
  Tag tag = Tag::gaussian;
  double sigma = 1.0;
  static KernelKind gaussian(double sigma) {
    if (!(sigma > 0.0)) throw DomainError("KernelKind: sigma must be positive");
    return KernelKind{Tag::gaussian, sigma};
  }
  static KernelKind angular() { return KernelKind{Tag::angular, 0.0}; }
};

struct FeatureMap {  // kernels.hpp:26-30
  StackedSpinner projector;
  KernelKind kind;
};

inline Vec64 embed(const FeatureMap& fm, const Vec64& x) {  // kernels.cpp:17-36
  check_finite(x, "embed");
  const int32_t kind = fm.kind.tag == KernelKind::Tag::gaussian ? SPN_EMBED_GAUSSIAN : SPN_EMBED_ANGULAR;
  if (kind == SPN_EMBED_ANGULAR) {
    bool zero = true;
    for (double v : x)
      if (v != 0.0) zero = false;
    if (zero) throw DomainError("embed: angular kernel undefined at the zero vector");
  }
  const std::size_t w = kind == SPN_EMBED_GAUSSIAN ? 2 * fm.projector.rows() : fm.projector.rows();
  std::vector<float> xf = detail::to_f32(x), out(w);
  check(spn_embed_f32_host(fm.projector.plan(), kind, fm.kind.sigma, xf.data(), 1,
                           static_cast<int64_t>(xf.size()), static_cast<int64_t>(xf.size()), out.data(),
                           static_cast<int64_t>(w)));
  return Vec64(out.begin(), out.end());
}

inline void embed_batch(const FeatureMap& fm, const float* x, std::size_t batch, std::size_t ld_x, std::size_t n_in,
                        float* out, std::size_t ld_out) {
  const int32_t kind = fm.kind.tag == KernelKind::Tag::gaussian ? SPN_EMBED_GAUSSIAN : SPN_EMBED_ANGULAR;
  check(spn_embed_f32_host(fm.projector.plan(), kind, fm.kind.sigma, x, static_cast<int64_t>(batch),
                           static_cast<int64_t>(ld_x), static_cast<int64_t>(n_in), out,
                           static_cast<int64_t>(ld_out)));
}

// Minimal column-major dense matrix with the slice of Eigen::MatrixXd's interface the reference's
// SketchOperator uses (rows(), cols(), operator()(i, j), (rows, cols) constructor).  Callers that
// have Eigen pass Eigen::MatrixXd to SketchOperator::apply unchanged (it is a template).
class MatrixXd {
 public:
  MatrixXd() = default;
  MatrixXd(std::ptrdiff_t rows, std::ptrdiff_t cols)
      : r_(rows), c_(cols), v_(static_cast<std::size_t>(rows * cols), 0.0) {}
  std::ptrdiff_t rows() const { return r_; }
  std::ptrdiff_t cols() const { return c_; }
  double& operator()(std::ptrdiff_t i, std::ptrdiff_t j) { return v_[static_cast<std::size_t>(j * r_ + i)]; }
  double operator()(std::ptrdiff_t i, std::ptrdiff_t j) const { return v_[static_cast<std::size_t>(j * r_ + i)]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }

 private:
  std::ptrdiff_t r_ = 0, c_ = 0;
  std::vector<double> v_;
};

// Spinner sketch on n-row matrices (newton_sketch.hpp:50-71, newton_sketch.cpp:74-101).
class SketchOperator {
 public:
  SketchOperator() = default;  // the exact (identity) operator, newton_sketch.hpp:55-56
  bool is_exact() const { return !projector_; }
  const spn_plan* plan() const { return projector_ ? projector_->plan() : nullptr; }
  // newton_sketch.cpp:74-81: padded = next_pow2(input_dim), StackedSpinner(v, padded, min(rows, padded),
  // rows, seed) — rows > padded stacks ceil(rows / padded) blocks — and norm 1/sqrt(rows)
  SketchOperator(SpinnerVariant v, std::size_t input_dim, std::size_t rows, std::uint64_t seed, int device = 0)
      : input_dim_(input_dim), rows_(rows) {
    padded_ = 1;
    while (padded_ < input_dim) padded_ <<= 1;
    projector_ = std::make_shared<StackedSpinner>(v, padded_, std::min(rows, padded_), rows, seed, 0.0, device);
    norm_ = 1.0 / std::sqrt(static_cast<double>(rows));
  }
  std::size_t rows(std::size_t input_dim) const { return is_exact() ? input_dim : rows_; }
  std::size_t input_dim() const { return input_dim_; }

  // newton_sketch.hpp:64 / newton_sketch.cpp:87-101 with value semantics: any Eigen-like column
  // matrix (Eigen::MatrixXd or spinners_b200::MatrixXd) of input_dim rows -> rows x cols sketch.
  template <class Mat>
  Mat apply(const Mat& columns) const {
    if (is_exact()) return columns;
    if (static_cast<std::size_t>(columns.rows()) != input_dim_)
      throw DimensionError("SketchOperator::apply: row count mismatch");
    const std::size_t d = static_cast<std::size_t>(columns.cols());
    std::vector<float> a(input_dim_ * d), o(rows_ * d);
    for (std::size_t i = 0; i < input_dim_; ++i)
      for (std::size_t c = 0; c < d; ++c) {
        const double v = columns(static_cast<std::ptrdiff_t>(i), static_cast<std::ptrdiff_t>(c));
        if (!std::isfinite(v)) throw DomainError("SketchOperator::apply: non-finite entry");
        a[i * d + c] = static_cast<float>(v);
      }
    if (d > 0) apply_host(a.data(), d, d, o.data(), d);
    Mat out(static_cast<std::ptrdiff_t>(rows_), static_cast<std::ptrdiff_t>(d));
    for (std::size_t r = 0; r < rows_; ++r)
      for (std::size_t c = 0; c < d; ++c)
        out(static_cast<std::ptrdiff_t>(r), static_cast<std::ptrdiff_t>(c)) = static_cast<double>(o[r * d + c]);
    return out;
  }
  // Row-major host buffers: a [input_dim][ld_a] -> out [rows][ld_out] (spn_sketch_f32_host).
  void apply_host(const float* a, std::size_t d, std::size_t ld_a, float* out, std::size_t ld_out,
                  const std::vector<int64_t>* row_list = nullptr) const {
    check(spn_sketch_f32_host(projector_->plan(), a, static_cast<int64_t>(input_dim_), static_cast<int64_t>(d),
                              static_cast<int64_t>(ld_a), row_list ? row_list->data() : nullptr,
                              static_cast<int64_t>(rows_), norm_, out, static_cast<int64_t>(ld_out)));
  }
  // columns: row-major [input_dim][d] on the DEVICE; out: [rows][d] on the device.
  void apply_device(const float* columns, std::size_t d, float* out, void* stream,
                    const std::vector<int64_t>* row_list = nullptr) const {
    check(spn_sketch_f32(projector_->plan(), columns, static_cast<int64_t>(input_dim_), static_cast<int64_t>(d),
                         static_cast<int64_t>(d), row_list ? row_list->data() : nullptr,
                         static_cast<int64_t>(rows_), norm_, out, static_cast<int64_t>(d), stream));
  }

 private:
  std::size_t input_dim_ = 0, rows_ = 0, padded_ = 1;
  double norm_ = 1.0;
  std::shared_ptr<StackedSpinner> projector_;
};

inline std::vector<int64_t> sample_rows(std::int64_t N, std::int64_t m, std::uint64_t seed) {
  std::vector<int64_t> out(static_cast<std::size_t>(m));
  check(spn_sample_rows(N, m, seed, out.data()));
  return out;
}

// ------------------------------------------------------------------ Gram matrices
// kernels.hpp:35-41 without Eigen: a dense row-major count x count matrix.
struct GramMatrix {
  std::size_t n = 0;
  std::vector<double> v;
  double operator()(std::size_t i, std::size_t j) const { return v[i * n + j]; }
  std::size_t rows() const { return n; }
  std::size_t cols() const { return n; }
};

namespace detail {
inline std::vector<float> pack_points(const std::vector<Vec64>& points, const char* what) {
  if (points.empty()) throw DimensionError(std::string(what) + ": empty dataset");
  const std::size_t dim = points.front().size();
  std::vector<float> f(points.size() * dim);
  for (std::size_t i = 0; i < points.size(); ++i) {
    if (points[i].size() != dim) throw DimensionError(std::string(what) + ": ragged dataset");
    check_finite(points[i], what);
    for (std::size_t t = 0; t < dim; ++t) f[i * dim + t] = static_cast<float>(points[i][t]);
  }
  return f;
}
}  // namespace detail

inline GramMatrix gram_exact(const std::vector<Vec64>& points, const KernelKind& kind) {  // kernels.cpp:38-76
  std::vector<float> f = detail::pack_points(points, "gram_exact");
  if (kind.tag == KernelKind::Tag::angular)
    for (const auto& p : points) {
      bool zero = true;
      for (double e : p) zero = zero && e == 0.0;
      if (zero) throw DomainError("gram_exact: angular kernel undefined at the zero vector");
    }
  GramMatrix g{points.size(), std::vector<double>(points.size() * points.size())};
  check(spn_gram_exact_host(f.data(), static_cast<int64_t>(points.size()), static_cast<int64_t>(points[0].size()),
                            kind.tag == KernelKind::Tag::angular ? SPN_EMBED_ANGULAR : SPN_EMBED_GAUSSIAN,
                            kind.sigma, g.v.data()));
  return g;
}

inline GramMatrix gram_approx(const FeatureMap& fm, const std::vector<Vec64>& points) {  // kernels.cpp:78-103
  std::vector<float> f = detail::pack_points(points, "gram_approx");
  GramMatrix g{points.size(), std::vector<double>(points.size() * points.size())};
  check(spn_gram_approx_host(fm.projector.plan(),
                             fm.kind.tag == KernelKind::Tag::angular ? SPN_EMBED_ANGULAR : SPN_EMBED_GAUSSIAN,
                             fm.kind.sigma, f.data(), static_cast<int64_t>(points.size()),
                             static_cast<int64_t>(points[0].size()), g.v.data()));
  return g;
}

inline double gram_error(const GramMatrix& exact, const GramMatrix& approx) {  // kernels.cpp:105-112
  if (exact.n != approx.n) throw DimensionError("gram_error: shape mismatch");
  double err = 0.0;
  check(spn_gram_error_host(exact.v.data(), approx.v.data(), static_cast<int64_t>(exact.n), &err));
  return err;
}

// ------------------------------------------------------------------ sketched Newton
// newton_sketch.hpp:13-86 / newton_sketch.cpp:28-204.  Features are a row-major
// n x d host matrix (no Eigen); the problem is uploaded once (fp32) to a device
// workspace, every numeric step runs on the GPU, vectors come back as fp64.
struct LogisticProblem {
  std::size_t n = 0, d = 0;
  std::vector<double> features;  // row-major n x d
  Vec64 labels;                  // +-1
  int device = 0;

  void validate() const {  // newton_sketch.cpp:28-37
    if (n < 1 || d < 1) throw DimensionError("LogisticProblem: empty data");
    if (labels.size() != n) throw DimensionError("LogisticProblem: label count mismatch");
    for (double v : features)
      if (!std::isfinite(v)) throw DomainError("LogisticProblem: non-finite features");
    for (double y : labels)
      if (y != 1.0 && y != -1.0) throw DomainError("LogisticProblem: labels must be +-1");
  }
  std::size_t observations() const { return n; }
  std::size_t dim() const { return d; }

  // device workspace with the problem resident (created on first use, grown for larger sketches)
  spn_newton* workspace(std::size_t rows = 0) const {
    if (!ws_ || ws_rows_ < rows) {
      spn_newton* w = nullptr;
      check(spn_newton_create(&w, static_cast<int64_t>(n), static_cast<int64_t>(d), static_cast<int64_t>(rows),
                              device));
      ws_.reset(w, [](spn_newton* q) { spn_newton_destroy(q); });
      ws_rows_ = rows;
      std::vector<float> f(features.begin(), features.end()), y(labels.begin(), labels.end());
      check(spn_newton_set_problem(w, f.data(), static_cast<int64_t>(d), y.data()));
    }
    return ws_.get();
  }

 private:
  mutable std::shared_ptr<spn_newton> ws_;
  mutable std::size_t ws_rows_ = 0;
};

struct SketchConfig {  // newton_sketch.hpp:23-33
  bool sketched = false;  // std::optional<SpinnerVariant> in the reference
  SpinnerVariant sketch_variant = SpinnerVariant::hd3_hd2_hd1;
  std::size_t sketch_rows = 0;
  std::size_t max_iters = 50;
  double gap_tolerance = 1e-10;
  bool line_search = true;
  std::uint64_t seed = 0;

  void validate(const LogisticProblem& p) const {  // newton_sketch.cpp:39-43
    if (sketched && sketch_rows < p.dim()) throw DimensionError("SketchConfig: sketch_rows must be >= d");
    if (max_iters < 1) throw DimensionError("SketchConfig: max_iters must be >= 1");
  }
};

struct NewtonTrace {  // newton_sketch.hpp:35-42
  std::vector<Vec64> iterates;
  std::vector<double> losses, gaps, seconds;
  double f_star = 0.0;
  bool converged = false;
};

inline double loss(const LogisticProblem& p, const Vec64& x) {  // newton_sketch.cpp:45-52
  if (x.size() != p.d) throw DimensionError("loss: dimension mismatch");
  double f = 0.0;
  check(spn_logistic_eval_host(p.workspace(), x.data(), &f, nullptr));
  return f;
}

inline Vec64 gradient(const LogisticProblem& p, const Vec64& x) {  // newton_sketch.cpp:54-61
  if (x.size() != p.d) throw DimensionError("gradient: dimension mismatch");
  Vec64 g(p.d);
  check(spn_logistic_eval_host(p.workspace(), x.data(), nullptr, g.data()));
  return g;
}

// newton_sketch.cpp:63-72, row-major n x d
inline std::vector<double> hessian_sqrt(const LogisticProblem& p, const Vec64& x) {
  if (x.size() != p.d) throw DimensionError("hessian_sqrt: dimension mismatch");
  std::vector<float> h(p.n * p.d);
  check(spn_hessian_sqrt_host(p.workspace(), x.data(), h.data(), static_cast<int64_t>(p.d)));
  return std::vector<double>(h.begin(), h.end());
}

namespace detail {
inline Vec64 step_at(const LogisticProblem& p, const Vec64& x, const SketchOperator& sketch, Vec64* grad,
                     double* f) {
  if (x.size() != p.d) throw DimensionError("sketched_step: dimension mismatch");
  const std::size_t rows = sketch.rows(p.n);
  Vec64 step(p.d);
  check(spn_sketched_step_host(p.workspace(sketch.is_exact() ? 0 : rows), sketch.plan(), static_cast<int64_t>(rows),
                               x.data(), step.data(), grad ? grad->data() : nullptr, f));
  return step;
}

// Backtracking Armijo, alpha 0.1, beta 0.5 (newton_sketch.cpp:140-142,163-164): returns
// (s, loss(x + s step)); the 2^-k candidates come from one pass over A on the device.
inline std::pair<double, double> backtrack(const LogisticProblem& p, const Vec64& x, const Vec64& step, double f0,
                                           double slope) {
  constexpr int kMax = 41;
  double losses[kMax];
  spn_newton* w = p.workspace();
  check(spn_logistic_line_host(w, x.data(), step.data(), 1.0, 4, losses));
  bool found = false;
  for (int k = 0; k < 4 && !found; ++k) found = !(losses[k] > f0 + 0.1 * std::ldexp(1.0, -k) * slope);
  if (!found) check(spn_logistic_line_host(w, x.data(), step.data(), 1.0, kMax, losses));
  double s = 1.0;
  for (int k = 0; k < kMax; ++k) {
    if (!(s > 1e-12) || !(losses[k] > f0 + 0.1 * s * slope)) return {s, losses[k]};
    s *= 0.5;
  }
  return {s, loss(p, x)};
}
}  // namespace detail

// newton_sketch.cpp:103-122
inline Vec64 sketched_step(const LogisticProblem& p, const Vec64& x, const SketchOperator& sketch) {
  return detail::step_at(p, x, sketch, nullptr, nullptr);
}

// newton_sketch.cpp:124-183
inline NewtonTrace solve(const LogisticProblem& p, const SketchConfig& cfg) {
  p.validate();
  cfg.validate(p);
  const std::size_t d = p.dim(), n = p.observations();
  double f_star;
  {
    Vec64 x(d, 0.0), g(d);
    const SketchOperator exact;
    for (int it = 0; it < 200; ++it) {
      double f0 = 0.0;
      const Vec64 step = detail::step_at(p, x, exact, &g, &f0);
      double decrement = 0.0;
      for (std::size_t j = 0; j < d; ++j) decrement -= g[j] * step[j];
      const double s = detail::backtrack(p, x, step, f0, -decrement).first;
      for (std::size_t j = 0; j < d; ++j) x[j] += s * step[j];
      if (decrement / 2.0 < 1e-13) break;
    }
    f_star = loss(p, x);
  }
  NewtonTrace trace;
  trace.f_star = f_star;
  Vec64 x(d, 0.0), g(d);
  for (std::size_t t = 0; t < cfg.max_iters; ++t) {
    const auto tic = std::chrono::steady_clock::now();
    SketchOperator sketch;  // fresh sketch every iteration
    if (cfg.sketched) sketch = SketchOperator(cfg.sketch_variant, n, cfg.sketch_rows, mix_seed(cfg.seed, t), p.device);
    double f0 = 0.0;
    const Vec64 step = detail::step_at(p, x, sketch, &g, &f0);
    double s = 1.0, f_next;
    if (cfg.line_search) {
      double slope = 0.0;
      for (std::size_t j = 0; j < d; ++j) slope += g[j] * step[j];
      std::tie(s, f_next) = detail::backtrack(p, x, step, f0, slope);
    } else {
      double l1 = 0.0;
      check(spn_logistic_line_host(p.workspace(), x.data(), step.data(), 1.0, 1, &l1));
      f_next = l1;
    }
    if (!cfg.line_search && f_next > f0)
      throw SingularSystemError("solve: loss increased under a full step (divergence)");
    for (std::size_t j = 0; j < d; ++j) x[j] += s * step[j];
    const auto toc = std::chrono::steady_clock::now();
    trace.iterates.push_back(x);
    trace.losses.push_back(f_next);
    trace.gaps.push_back(f_next - f_star);
    trace.seconds.push_back(std::chrono::duration<double>(toc - tic).count());
    if (f_next - f_star <= cfg.gap_tolerance) {
      trace.converged = true;
      break;
    }
  }
  return trace;
}

// newton_sketch.cpp:185-204 (the reference generator; features rounded to fp32 like the device copy)
inline LogisticProblem generate_ar1_problem(std::size_t n, std::size_t d, std::uint64_t seed, int device = 0) {
  std::vector<float> f(n * d), y(n);
  check(spn_ar1_problem(static_cast<int64_t>(n), static_cast<int64_t>(d), seed, f.data(), y.data()));
  LogisticProblem p;
  p.n = n;
  p.d = d;
  p.features.assign(f.begin(), f.end());
  p.labels.assign(y.begin(), y.end());
  p.device = device;
  return p;
}

}  // namespace spinners_b200
