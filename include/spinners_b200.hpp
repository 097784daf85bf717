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

#include <cmath>
#include <cstdint>
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

inline void check(spn_status s) {
  if (s == SPN_OK) return;
  std::string msg = std::string(spn_status_string(s)) + ": " + spn_last_error();
  if (s == SPN_EDIM) throw DimensionError(msg);
  if (s == SPN_EDOMAIN) throw DomainError(msg);
  throw DeviceError(msg);
}

inline std::uint64_t mix_seed(std::uint64_t base, std::uint64_t stream) { return spn_mix_seed(base, stream); }

inline void check_finite(const Vec64& x, const char* what) {  // common.hpp:37-41
  for (double v : x)
    if (!std::isfinite(v)) throw DomainError(std::string(what) + ": non-finite entry");
}

enum class SpinnerVariant { hd3_hd2_hd1 = SPN_HD3_HD2_HD1, hdg_hd2_hd1 = SPN_HDG_HD2_HD1, gauss3 = SPN_GAUSS3 };

inline double default_scale(SpinnerVariant, std::size_t n) { return std::sqrt(static_cast<double>(n)); }

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
    if ((n & (n - 1)) != 0)
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
      : n_(n), k_(k) {
    if (k < 1) throw DimensionError("StackedSpinner: k must be >= 1");
    spn_plan_desc d{static_cast<int32_t>(v), static_cast<int64_t>(n), static_cast<int64_t>(m),
                    static_cast<int64_t>(k), 1, nullptr, seed, scale, device};
    spn_plan* p = nullptr;
    check(spn_plan_create(&p, &d));
    plan_ = detail::Plan(p, detail::PlanDeleter{});
  }

  std::size_t rows() const { return k_; }
  std::size_t input_dim() const { return n_; }
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
};

// One realised m x n block (spinner.hpp:56-104), diagonals drawn from spec.seed.
class StructuredSpinner : public StackedSpinner {
 public:
  static StructuredSpinner build(const SpinnerSpec& spec, int device = 0) {
    spec.validate();
    StructuredSpinner s;
    s.spec_ = spec;
    s.n_ = spec.n;
    s.k_ = spec.m;
    s.d1_.resize(spec.n);
    s.d2_.resize(spec.n);
    s.d3_.resize(spec.n);
    check(spn_realize_block(static_cast<int32_t>(spec.variant), static_cast<int64_t>(spec.n), spec.seed,
                            s.d1_.data(), s.d2_.data(), s.d3_.data()));
    spn_plan* p = nullptr;
    check(spn_plan_create_explicit(&p, static_cast<int64_t>(spec.n), static_cast<int64_t>(spec.m),
                                   static_cast<int64_t>(spec.m), 1, s.d1_.data(), s.d2_.data(), s.d3_.data(),
                                   spec.scale, device));
    s.plan_ = detail::Plan(p, detail::PlanDeleter{});
    return s;
  }
  const SpinnerSpec& spec() const { return spec_; }
  const Vec64& d1() const { return d1_; }
  const Vec64& d2() const { return d2_; }
  const Vec64& d3() const { return d3_; }      // HD3HD2HD1
  const Vec64& g_diag() const { return d3_; }  // HDgHD2HD1

 private:
  SpinnerSpec spec_;
  Vec64 d1_, d2_, d3_;
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

// Spinner sketch on n-row matrices (newton_sketch.hpp:50-71, newton_sketch.cpp:74-101).
class SketchOperator {
 public:
  SketchOperator(SpinnerVariant v, std::size_t input_dim, std::size_t rows, std::uint64_t seed, int device = 0)
      : input_dim_(input_dim), rows_(rows) {
    padded_ = 1;
    while (padded_ < input_dim) padded_ <<= 1;
    if (rows > padded_) throw DeviceError("SketchOperator: rows > padded dimension not supported");
    projector_ = std::make_unique<StackedSpinner>(v, padded_, std::min(rows, padded_), rows, seed, 0.0, device);
    norm_ = 1.0 / std::sqrt(static_cast<double>(rows));
  }
  std::size_t rows(std::size_t) const { return rows_; }
  // columns: row-major [input_dim][d] on the DEVICE; out: [rows][d] on the device.
  void apply_device(const float* columns, std::size_t d, float* out, void* stream,
                    const std::vector<int64_t>* row_list = nullptr) const {
    check(spn_sketch_f32(projector_->plan(), columns, static_cast<int64_t>(input_dim_), static_cast<int64_t>(d),
                         static_cast<int64_t>(d), row_list ? row_list->data() : nullptr,
                         static_cast<int64_t>(rows_), norm_, out, static_cast<int64_t>(d), stream));
  }

 private:
  std::size_t input_dim_, rows_, padded_ = 1;
  double norm_ = 1.0;
  std::unique_ptr<StackedSpinner> projector_;
};

inline std::vector<int64_t> sample_rows(std::int64_t N, std::int64_t m, std::uint64_t seed) {
  std::vector<int64_t> out(static_cast<std::size_t>(m));
  check(spn_sample_rows(N, m, seed, out.data()));
  return out;
}

}  // namespace spinners_b200
