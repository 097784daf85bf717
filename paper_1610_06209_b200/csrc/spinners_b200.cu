// spinners_b200: plan management + C ABI (include/spinners_b200.h) over the
// sm_100a spinner kernels.  No CPU fallback: every compute entry point launches
// a CUDA kernel or fails with a status code.
#include "../../include/spinners_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "errors.hpp"
#include "family.hpp"
#include "host_params.hpp"
#include "internal.hpp"
#include "spinner_big.cuh"
#include "spinner_vec.cuh"
#include "vec_launch.cuh"

namespace {

spn_status fail(spn_status s, const std::string& msg) { return spn::set_error(s, msg); }
spn_status cuda_fail(cudaError_t e, const char* where) { return spn::cuda_error(e, where); }

#define SPN_CUDA(call)                                         \
  do {                                                         \
    cudaError_t e_ = (call);                                   \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);        \
  } while (0)

bool is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }
int ilog2(int64_t n) {
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  return l;
}

struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// What kind of memory a caller's pointer is (pageable host memory reports cudaMemoryTypeUnregistered).
cudaMemoryType host_ptr_kind(const void* ptr) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return cudaMemoryTypeUnregistered;
  }
  return at.type;
}

using spn::kMaxLogNVec;
constexpr int kMaxLogN = 20;     // multi-pass path up to 2^20

}  // namespace

// ----------------------------------------------------------------------------- plan

struct spn_plan {
  int variant = 0;
  int64_t n = 0, m = 0, k = 0, tables = 0, blocks = 0;
  int log_n = 0;
  double scale = 0.0;
  int device = 0;
  int sms = 0;
  std::vector<double> d[3];  // realised fp64 diagonals [tables][blocks][n]
  int dsign[3] = {0, 0, 0};
  // Single-block Rademacher plans with n > 2^14 (a sketch: SketchOperator, one per Newton
  // iteration) defer the host draws: the sketch realises its diagonals on the device from
  // the same generator; d is drawn on the host only if something asks for it.
  bool lazy_d = false;
  uint64_t spec_seed = 0;
  std::once_flag d_once;
  void ensure_host_d() {
    if (!lazy_d) return;
    std::call_once(d_once, [this] {
      for (auto& v : d) v.resize(static_cast<size_t>(n));
      spn::realize_block(spn::V_HD3, n, spec_seed, d[0].data(), d[1].data(), d[2].data());
    });
  }
  // circulant family / dense baseline (family.cu): Toeplitz first rows, dense matrices
  std::vector<double> trow, dense;
  spn::FamilyPlan* fam = nullptr;

  // vector-kernel layouts (n <= 2^14): [diag][layout]
  uint32_t* vsgn[3][2] = {};
  float* vflt[3][2] = {};
  uint32_t* vsgnL[3] = {};     // n = 2^11 all-sign plans: layout-B masks in pb() order (looped hash kernel)
  uint32_t* vsgnP[3][2] = {};  // n = 1024 sign masks in permuted coordinates (OP_EMBED_GAUSS_P)
  // multi-pass layouts (n > 2^14)
  spn::BigPlan big;

  // multi-block sketch: one single-block plan per block (sketch_subplans)
  std::mutex sub_mu;
  std::vector<spn_plan*> sub;

  // host-API staging (lazily grown; guarded by mu)
  std::mutex mu;
  static constexpr int kHostStreams = 4;  // host-buffer pipeline streams (host_streams() in use)
  cudaStream_t hs[kHostStreams] = {};
  void* hbuf[kHostStreams][3] = {};  // [stream][x | out0 | out1]
  size_t hbuf_bytes[kHostStreams][3] = {};
  void* hstage[kHostStreams][2] = {};  // pinned staging of pageable outputs [stream][out0 | out1]
  size_t hstage_bytes[kHostStreams][2] = {};

  ~spn_plan();
};

namespace {
spn_status plan_destroy_impl(spn_plan* p);
}  // namespace

spn_plan::~spn_plan() {
  {
    for (spn_plan* q : sub) plan_destroy_impl(q);
    DeviceGuard g(device);
    if (fam) spn::family_destroy(fam);
    for (auto& a : vsgn)
      for (auto* p : a)
        if (p) cudaFree(p);
    for (auto& a : vflt)
      for (auto* p : a)
        if (p) cudaFree(p);
    for (auto& a : vsgnP)
      for (auto* p : a)
        if (p) cudaFree(p);
    for (auto* p : vsgnL)
      if (p) cudaFree(p);
    big.release();
    for (auto& a : hbuf)
      for (auto* p : a)
        if (p) cudaFree(p);
    for (auto& a : hstage)
      for (auto* p : a)
        if (p) cudaFreeHost(p);
    for (auto s : hs)
      if (s) cudaStreamDestroy(s);
  }
}

namespace {
spn_status plan_destroy_impl(spn_plan* p) {
  delete p;
  return SPN_OK;
}
}  // namespace

namespace {

// Element held by thread t in register j of a (LOG_R, LOG_T) group, per layout.
inline int64_t elem(int layout, int LOG_R, int LOG_T, int64_t t, int64_t j) {
  return layout == spn::LAY_A ? (t << LOG_R) + j : (j << LOG_T) + t;
}

spn_status upload(const void* src, size_t bytes, void** dst) {
  SPN_CUDA(cudaMalloc(dst, bytes));
  SPN_CUDA(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
  return SPN_OK;
}

// Inverse of the n = 1024 coordinate permutation of OP_EMBED_GAUSS_P (spinner_vec.cuh):
// e' = ((e >> 2) & 31) | ((e & 3) << 5) | (e & 0x380).
inline int64_t perm1024_inv(int64_t ep) { return ((ep >> 5) & 3) | ((ep & 31) << 2) | (ep & 0x380); }

// Bit-packed sign masks of one diagonal in one layout (optionally in permuted coordinates).
std::vector<uint32_t> pack_signs(const double* D, int64_t TB, int64_t N, int LOG_R, int LOG_T, int lay,
                                 bool perm, bool pib = false) {
  const int64_t R = int64_t(1) << LOG_R, T = int64_t(1) << LOG_T;
  const int64_t WORDS = R >= 32 ? R / 32 : 1, BITS = R >= 32 ? 32 : R;
  std::vector<uint32_t> w(static_cast<size_t>(TB * WORDS * T), 0u);
  for (int64_t tb = 0; tb < TB; ++tb)
    for (int64_t q = 0; q < WORDS; ++q)
      for (int64_t t = 0; t < T; ++t) {
        uint32_t word = 0;
        for (int64_t jj = 0; jj < BITS; ++jj) {
          int64_t j = q * 32 + jj;
          // looped R == 2T chain (VCfg::LOOPED_ODD): layout-B register pb(j) holds standard register j
          if (pib) j = ((j & (R / 2 - 1)) << 1) | (j >> (LOG_R - 1));
          int64_t e = elem(lay, LOG_R, LOG_T, t, j);
          if (perm) e = perm1024_inv(e);
          if (D[tb * N + e] < 0.0) word |= 1u << jj;
        }
        w[static_cast<size_t>(tb * WORDS * T + q * T + t)] = word;
      }
  return w;
}

// Pack the diagonals in the exact register order each kernel layout consumes.
spn_status build_vec_layouts(spn_plan* p) {
  const int LOG_R = (p->log_n + 1) / 2, LOG_T = p->log_n / 2;
  const int64_t R = int64_t(1) << LOG_R, T = int64_t(1) << LOG_T, N = p->n;
  const int64_t TB = p->tables * p->blocks;
  const bool all_sign = p->dsign[0] && p->dsign[1] && p->dsign[2];
  for (int di = 0; di < 3; ++di) {
    const double* D = p->d[di].data();
    for (int lay = 0; lay < 2; ++lay) {
      if (p->dsign[di]) {
        // all-sign plans run the SIGNS kernels, whose R == 2T chains number layout B's registers pb(j)
        const bool pib = all_sign && lay == spn::LAY_B && LOG_R == LOG_T + 1 && R >= SPN_LOOP_ODD_MIN_R;
        std::vector<uint32_t> w = pack_signs(D, TB, N, LOG_R, LOG_T, lay, false, pib);
        spn_status s = upload(w.data(), w.size() * 4, reinterpret_cast<void**>(&p->vsgn[di][lay]));
        if (s) return s;
        // n = 2^11: only the hash kernels run the looped chain (VCfg::looped_odd): a second copy in pb() order
        if (all_sign && lay == spn::LAY_B && LOG_R == LOG_T + 1 && !pib && R >= SPN_LOOP_ODD_HASH_MIN_R) {
          w = pack_signs(D, TB, N, LOG_R, LOG_T, lay, false, true);
          s = upload(w.data(), w.size() * 4, reinterpret_cast<void**>(&p->vsgnL[di]));
          if (s) return s;
        }
        if (N == 1024 && all_sign) {  // permuted-coordinate embed kernel
          w = pack_signs(D, TB, N, LOG_R, LOG_T, lay, true);
          s = upload(w.data(), w.size() * 4, reinterpret_cast<void**>(&p->vsgnP[di][lay]));
          if (s) return s;
        }
      } else {
        std::vector<float> f(static_cast<size_t>(TB * N));
        for (int64_t tb = 0; tb < TB; ++tb)
          for (int64_t t = 0; t < T; ++t)
            for (int64_t j = 0; j < R; ++j) {
              const int64_t pos = R >= 4 ? ((j / 4) * T + t) * 4 + (j % 4) : j * T + t;
              f[static_cast<size_t>(tb * N + pos)] =
                  static_cast<float>(D[tb * N + elem(lay, LOG_R, LOG_T, t, j)]);
            }
        spn_status s = upload(f.data(), f.size() * 4, reinterpret_cast<void**>(&p->vflt[di][lay]));
        if (s) return s;
      }
    }
  }
  return SPN_OK;
}

spn_status finish_plan(spn_plan* p) {
  p->log_n = ilog2(p->n);
  for (int di = 0; di < 3 && !p->lazy_d; ++di) {
    bool all = true;
    for (double v : p->d[di])
      if (v != 1.0 && v != -1.0) {
        all = false;
        break;
      }
    p->dsign[di] = all ? 1 : 0;
  }
  DeviceGuard g(p->device);
  if (!g.ok) return fail(SPN_ECUDA, "cudaSetDevice failed");
  SPN_CUDA(cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, p->device));
  if (spn::family_variant(p->variant))
    return spn::family_build(&p->fam, p->variant, p->n, p->m, p->k, p->tables, p->blocks, p->d, p->trow, p->dense,
                             p->scale, p->device);
  if (p->log_n <= kMaxLogNVec) return build_vec_layouts(p);
  return p->big.build(p->n, p->tables * p->blocks, p->d, p->dsign);
}

spn_status validate_shape(int64_t n, int64_t m, int64_t k, int64_t tables) {
  if (!is_pow2(n) || n < 2)
    return fail(SPN_EDIM, "n must be a power of two >= 2, got " + std::to_string(n));
  if (ilog2(n) > kMaxLogN) return fail(SPN_EUNSUPPORTED, "n > 2^20 not supported");
  if (m < 1 || m > n) return fail(SPN_EDIM, "need 1 <= m <= n");
  if (k < 1) return fail(SPN_EDIM, "k must be >= 1");
  if (tables < 1) return fail(SPN_EDIM, "tables must be >= 1");
  if (k > (int64_t(1) << 30)) return fail(SPN_EDIM, "k too large");
  return SPN_OK;
}

// ------------------------------------------------------------ vector-kernel dispatch

spn::LaunchFn vec_launcher(int log_n, int op, int signs) {
  switch (op) {
    case spn::OP_HASH: return spn::vec_launcher_hash(log_n, signs);
    case spn::OP_APPLY: return spn::vec_launcher_apply(log_n, signs);
    case spn::OP_EMBED_GAUSS: return spn::vec_launcher_gauss(log_n, signs);
    default: return spn::vec_launcher_ang(log_n, signs);
  }
}

spn::VecParams base_params(const spn_plan* p) {
  spn::VecParams v{};
  v.m = p->m;
  v.k = p->k;
  v.blocks = static_cast<int>(p->blocks);
  v.tables = static_cast<int>(p->tables);
  for (int di = 0; di < 3; ++di) {
    v.dsign[di] = p->dsign[di];
    for (int lay = 0; lay < 2; ++lay) v.d[di][lay] = {p->vsgn[di][lay], p->vflt[di][lay]};
  }
  v.c = static_cast<float>(p->scale * std::pow(static_cast<double>(p->n), -1.5));
  return v;
}

spn_status check_io(const spn_plan* p, const void* x, int64_t batch, int64_t ld_x, int64_t n_in) {
  if (!p) return fail(SPN_EINVAL, "null plan");
  if (batch < 0) return fail(SPN_EINVAL, "batch < 0");
  if (batch > 0 && !x) return fail(SPN_EINVAL, "null input");
  if (n_in < 1 || n_in > p->n)
    return fail(SPN_EDIM, "input length " + std::to_string(n_in) + " not in [1, n=" + std::to_string(p->n) + "]");
  if (ld_x < n_in) return fail(SPN_EINVAL, "ld_x < n_in");
  return SPN_OK;
}

spn_status run_vec(const spn_plan* p, int op, spn::VecParams& v, cudaStream_t s) {
  const int64_t items = v.batch * (op == spn::OP_HASH ? p->tables : 1);
  if (items == 0) return SPN_OK;
  DeviceGuard g(p->device);
  const int signs = p->dsign[0] && p->dsign[1] && p->dsign[2];
  if (op == spn::OP_HASH && signs && p->vsgnL[0])  // n = 2^11: the looped hash kernel's layout-B mask order
    for (int di = 0; di < 3; ++di) v.d[di][spn::LAY_B].sgn = p->vsgnL[di];
  const spn::LaunchFn fn = (op == spn::OP_APPLY && v.perm) ? spn::vec_launcher_apply_perm()
                                                           : vec_launcher(p->log_n, op, signs);
  cudaError_t e = fn(v, s, p->sms, items);
  if (e != cudaSuccess) return cuda_fail(e, "spinner_vec_kernel launch");
  return SPN_OK;
}

// n > 2^14: the multi-pass apply per table into y (or a chunked workspace), then the signed
// argmax per row (lsh.cpp:23-30 over the stacked rows; SURVEY a14.6 multi-table encoding).
spn_status big_hash(spn_plan* p, const float* x, int64_t batch, int64_t ld_x, int64_t n_in, int32_t* ids,
                    float* y, int64_t ld_y, cudaStream_t s) {
  if (batch == 0) return SPN_OK;
  DeviceGuard g(p->device);
  p->ensure_host_d();
  const double c = p->scale * std::pow(static_cast<double>(p->n), -1.5);
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(batch, int64_t(p->sms) * 8));
  if (y) {  // single table: y is the caller's buffer
    if (spn_status st = p->big.apply(x, batch, ld_x, n_in, y, ld_y, 0, p->k, p->m, p->blocks, c, p->sms, s)) return st;
    spn::rows_signed_argmax_kernel<<<grid, 256, 0, s>>>(y, ld_y, p->k, batch, ids, p->tables, 0);
    SPN_CUDA(cudaGetLastError());
    return SPN_OK;
  }
  const int64_t ld = (p->k + 3) / 4 * 4;
  const int64_t rows = std::max<int64_t>(1, std::min<int64_t>(batch, (int64_t(256) << 20) / (ld * 4)));
  spn::Scratch ws;
  SPN_CUDA(ws.alloc(sizeof(float) * static_cast<size_t>(rows * ld), s));
  float* w = static_cast<float*>(ws.p);
  for (int64_t r0 = 0; r0 < batch; r0 += rows) {
    const int64_t nr = std::min(rows, batch - r0);
    for (int64_t t = 0; t < p->tables; ++t) {
      if (spn_status st = p->big.apply(x + r0 * ld_x, nr, ld_x, n_in, w, ld, 0, p->k, p->m, p->blocks, c, p->sms, s,
                                        t * p->blocks))
        return st;
      spn::rows_signed_argmax_kernel<<<static_cast<unsigned>(std::min<int64_t>(nr, int64_t(p->sms) * 8)), 256, 0, s>>>(
          w, ld, p->k, nr, ids + r0 * p->tables, p->tables, t);
      SPN_CUDA(cudaGetLastError());
    }
  }
  return SPN_OK;
}

// n > 2^14: z = the multi-pass apply straight into the feature rows, then the cos/sin (or sign)
// epilogue in place (kernels.cpp:17-36).
spn_status big_embed(spn_plan* p, int32_t kind, double sigma, const float* x, int64_t batch, int64_t ld_x,
                     int64_t n_in, float* out, int64_t ld_out, cudaStream_t s) {
  if (batch == 0) return SPN_OK;
  DeviceGuard g(p->device);
  p->ensure_host_d();
  const double c = p->scale * std::pow(static_cast<double>(p->n), -1.5);
  if (spn_status st = p->big.apply(x, batch, ld_x, n_in, out, ld_out, 0, p->k, p->m, p->blocks, c, p->sms, s))
    return st;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(batch, int64_t(p->sms) * 8));
  spn::rows_embed_kernel<<<grid, 256, 0, s>>>(out, ld_out, p->k, batch, kind == SPN_EMBED_GAUSSIAN ? 1 : 0,
                                               static_cast<float>(1.0 / sigma),
                                               static_cast<float>(1.0 / std::sqrt(static_cast<double>(p->k))));
  SPN_CUDA(cudaGetLastError());
  return SPN_OK;
}

}  // namespace

// ------------------------------------------------------------------------ sketches
namespace {

// SketchOperator::apply argument checks (newton_sketch.cpp:87-90).  rows == NULL is the reference's
// P = first m_out rows of the stacked output; a row list (builder-defined P) indexes the n outputs
// of a single-block plan.
spn_status sketch_check(const spn_plan* p, const float* a, int64_t n_in, int64_t d, int64_t ld_a,
                        const int64_t* rows, int64_t m_out, const float* out, int64_t ld_out) {
  if (!p) return fail(SPN_EINVAL, "null plan");
  if (p->fam) return fail(SPN_EUNSUPPORTED, "sketch: Hadamard-only variants (HD3/HDg) on the device");
  if (p->tables != 1) return fail(SPN_EUNSUPPORTED, "sketch needs a single-table plan");
  if (n_in < 1 || n_in > p->n) return fail(SPN_EDIM, "SketchOperator::apply: row count mismatch");
  if (d < 0 || m_out < 0) return fail(SPN_EDIM, "bad sketch shape");
  if (ld_a < d || ld_out < d) return fail(SPN_EINVAL, "bad leading dimension");
  if (d > 0 && m_out > 0 && (!a || !out)) return fail(SPN_EINVAL, "null pointer");
  if (!rows && m_out > p->k) return fail(SPN_EDIM, "first-m sketch: m_out > k");
  if (rows) {
    if (p->blocks != 1) return fail(SPN_EUNSUPPORTED, "row-sampled sketch needs a single-block plan");
    if (m_out > p->n) return fail(SPN_EDIM, "bad sketch shape");
    for (int64_t r = 0; r < m_out; ++r)
      if (rows[r] < 0 || rows[r] >= p->n) return fail(SPN_EDIM, "row index out of range");
  }
  return SPN_OK;
}

// Multi-block sketches (rows > next_pow2(input_dim): StackedSpinner(v, padded, padded, rows, seed),
// newton_sketch.cpp:77-79): block b produces output rows [b*m, b*m + m) from its own single-block
// plan, made once from the realised diagonals of (table 0, block b).
spn_status sketch_subplans(spn_plan* p) {
  std::lock_guard<std::mutex> lock(p->sub_mu);
  if (!p->sub.empty()) return SPN_OK;
  std::vector<spn_plan*> sub;
  for (int64_t b = 0; b < p->blocks; ++b) {
    spn_plan* q = nullptr;
    const int64_t off = b * p->n;
    spn_status st = spn_plan_create_explicit(&q, p->n, p->n, p->n, 1, p->d[0].data() + off, p->d[1].data() + off,
                                             p->d[2].data() + off, p->scale, p->device);
    if (st) {
      for (spn_plan* r : sub) spn_plan_destroy(r);
      return st;
    }
    sub.push_back(q);
  }
  p->sub = std::move(sub);
  return SPN_OK;
}

spn_status sketch_dispatch(const spn_plan* cp, const float* a, int64_t n_in, int64_t d, int64_t ld_a,
                           const int64_t* rows, int64_t m_out, double norm, float* out, int64_t ld_out,
                           cudaStream_t s, const float* row_scale) {
  if (spn_status st = sketch_check(cp, a, n_in, d, ld_a, rows, m_out, out, ld_out)) return st;
  if (d == 0 || m_out == 0) return SPN_OK;
  auto* p = const_cast<spn_plan*>(cp);
  DeviceGuard g(p->device);
  if (p->blocks == 1)
    return spn::sketch_run(p->n, p->d, p->dsign, a, n_in, d, ld_a, rows, m_out,
                           p->scale * std::pow(static_cast<double>(p->n), -1.5) * norm, out, ld_out, p->sms, s,
                           &p->big, row_scale);
  if (spn_status st = sketch_subplans(p)) return st;
  for (int64_t b = 0; b < p->blocks && b * p->m < m_out; ++b) {
    const int64_t mb = std::min(p->m, m_out - b * p->m);
    const spn_plan* q = p->sub[static_cast<size_t>(b)];
    if (spn_status st = spn::sketch_run(q->n, q->d, q->dsign, a, n_in, d, ld_a, nullptr, mb,
                                        q->scale * std::pow(static_cast<double>(q->n), -1.5) * norm,
                                        out + b * p->m * ld_out, ld_out, q->sms, s,
                                        const_cast<spn::BigPlan*>(&q->big), row_scale))
      return st;
  }
  return SPN_OK;
}

}  // namespace

// =============================================================================== C ABI

extern "C" {

const char* spn_status_string(spn_status s) {
  switch (s) {
    case SPN_OK: return "ok";
    case SPN_EDIM: return "dimension error";
    case SPN_EDOMAIN: return "domain error";
    case SPN_ECUDA: return "cuda error";
    case SPN_ENOMEM: return "out of memory";
    case SPN_EUNSUPPORTED: return "unsupported";
    case SPN_EINVAL: return "invalid argument";
    case SPN_ESINGULAR: return "singular system";
  }
  return "unknown status";
}

const char* spn_last_error(void) { return spn::last_error().c_str(); }
const char* spn_version(void) { return "spinners_b200 0.1 (sm_100a)"; }
uint64_t spn_mix_seed(uint64_t base, uint64_t stream) { return spn::mix_seed(base, stream); }

spn_status spn_sample_rows(int64_t N, int64_t m, uint64_t seed, int64_t* out) { SPN_TRY
  if (!out) return fail(SPN_EINVAL, "null out");
  if (N < 1 || m < 0 || m > N) return fail(SPN_EDIM, "need 0 <= m <= N, N >= 1");
  std::vector<int64_t> r = spn::sample_rows(N, m, seed);
  std::copy(r.begin(), r.end(), out);
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_realize_block(int32_t variant, int64_t n, uint64_t spec_seed, double* d1, double* d2,
                             double* d3) { SPN_TRY
  if (!d1 || !d2 || !d3) return fail(SPN_EINVAL, "null argument");
  if (variant != SPN_HD3_HD2_HD1 && variant != SPN_HDG_HD2_HD1 && variant != SPN_GAUSS3)
    return fail(SPN_EDOMAIN, "unknown spinner variant " + std::to_string(variant));
  if (n < 1) return fail(SPN_EDIM, "n must be >= 1");
  spn::realize_block(variant, n, spec_seed, d1, d2, d3);
  return SPN_OK;
  SPN_CATCH
}

}  // extern "C"

namespace {
// raw_spec_seed: d->seed is the single block's spec seed itself (StructuredSpinner::build,
// spinner.cpp:137-151) instead of the stacked seed whose block b draws from mix_seed(seed, b)
spn_status plan_create_impl(spn_plan** out, const spn_plan_desc* d, bool raw_spec_seed);
}  // namespace

extern "C" {

spn_status spn_plan_create(spn_plan** out, const spn_plan_desc* d) { SPN_TRY return plan_create_impl(out, d, false);   SPN_CATCH
}

spn_status spn_plan_create_block(spn_plan** out, int32_t variant, int64_t n, int64_t m, uint64_t spec_seed,
                                 double scale, int32_t device) { SPN_TRY
  const spn_plan_desc d{variant, n, m, m, 1, nullptr, spec_seed, scale, device};
  return plan_create_impl(out, &d, true);
  SPN_CATCH
}

}  // extern "C"

namespace {
spn_status plan_create_impl(spn_plan** out, const spn_plan_desc* d, bool raw_spec_seed) {
  if (!out || !d) return fail(SPN_EINVAL, "null argument");
  *out = nullptr;
  const bool fam = spn::family_variant(d->variant);
  if (d->variant != SPN_HD3_HD2_HD1 && d->variant != SPN_HDG_HD2_HD1 && d->variant != SPN_GAUSS3 && !fam)
    return fail(SPN_EDOMAIN, "unknown spinner variant " + std::to_string(d->variant));
  if (d->variant == SPN_GAUSSIAN_DENSE) {  // no Hadamard stage: any n >= 1 (spinner.cpp:59-67)
    if (d->n < 1 || d->m < 1 || d->m > d->n) return fail(SPN_EDIM, "SpinnerSpec: need 1 <= m <= n");
    if (d->k < 1 || d->tables < 1) return fail(SPN_EDIM, "k and tables must be >= 1");
  } else if (spn_status s = validate_shape(d->n, d->m, d->k, d->tables)) {
    return s;
  }
  if (fam && d->variant != SPN_GAUSSIAN_DENSE && d->n > (d->variant == SPN_GTOEPLITZ_D2_HD1 ? 4096 : 8192))
    return fail(SPN_EUNSUPPORTED, "circulant family: n > 2^13 (Toeplitz 2^12) not supported (fp64 FFT in smem)");
  if (!d->table_seeds && d->tables != 1) return fail(SPN_EINVAL, "tables > 1 needs table_seeds");
  if (d->scale != 0.0 && !std::isfinite(d->scale)) return fail(SPN_EDOMAIN, "non-finite scale");
  // owned until the end: a host allocation that throws (std::bad_alloc -> SPN_ENOMEM at the ABI
  // barrier) must not leak the half-built plan
  std::unique_ptr<spn_plan> owner(new spn_plan());
  auto* p = owner.get();
  p->variant = d->variant;
  p->n = d->n;
  p->m = d->m;
  p->k = d->k;
  p->tables = d->tables;
  p->blocks = (d->k + d->m - 1) / d->m;
  p->device = d->device;
  // default_scale: sqrt(n) for the Hadamard-only variants, 1 for the circulant family and
  // the dense baseline (spinner.cpp:41-45,69-71)
  p->scale = d->scale != 0.0 ? d->scale : (fam ? 1.0 : std::sqrt(static_cast<double>(d->n)));
  const int64_t per = p->blocks * p->n;
  if (d->variant == SPN_HD3_HD2_HD1 && p->tables == 1 && p->blocks == 1 && ilog2(p->n) > kMaxLogNVec) {
    p->lazy_d = true;
    p->spec_seed = raw_spec_seed ? d->seed : spn::mix_seed(d->table_seeds ? d->table_seeds[0] : d->seed, 0);
    for (int di = 0; di < 3; ++di) p->dsign[di] = 1;
    if (spn_status s = finish_plan(p)) return s;
    p->big.dev_rad = true;
    p->big.dev_seed = p->spec_seed;
    {
      DeviceGuard g(p->device);
      if (spn_status s = p->big.prefetch_sketch(p->n)) return s;
    }
    *out = owner.release();
    return SPN_OK;
  }
  for (auto& v : p->d) v.resize(static_cast<size_t>(p->tables * per));
  if (d->variant == SPN_GTOEPLITZ_D2_HD1) p->trow.resize(static_cast<size_t>(p->tables * per));
  if (d->variant == SPN_GAUSSIAN_DENSE) p->dense.resize(static_cast<size_t>(p->tables * p->blocks * p->m * p->n));
  // every (table, block) has its own generators: realise them in parallel when there is work
  auto realize = [&](int64_t tb) {
    const int64_t t = tb / p->blocks, b = tb - t * p->blocks;
    const uint64_t seed = d->table_seeds ? d->table_seeds[t] : d->seed;
    const int64_t off = t * per + b * p->n;
    const uint64_t spec_seed = raw_spec_seed ? seed : spn::mix_seed(seed, static_cast<uint64_t>(b));
    if (fam)
      spn::family_realize(d->variant, p->n, p->m, spec_seed, p->d[0].data() + off, p->d[1].data() + off,
                          p->d[2].data() + off, p->trow.empty() ? nullptr : p->trow.data() + off,
                          p->dense.empty() ? nullptr : p->dense.data() + (t * p->blocks + b) * p->m * p->n);
    else
      spn::realize_block(d->variant, p->n, spec_seed, p->d[0].data() + off, p->d[1].data() + off,
                         p->d[2].data() + off);
  };
  const int64_t nblk = p->tables * p->blocks;
  if (nblk > 1 && nblk * p->n >= (int64_t(1) << 16))
    spn::parallel_for(nblk, realize);
  else
    for (int64_t i = 0; i < nblk; ++i) realize(i);
  if (spn_status s = finish_plan(p)) return s;
  *out = owner.release();
  return SPN_OK;
}
}  // namespace

extern "C" {

spn_status spn_plan_create_explicit(spn_plan** out, int64_t n, int64_t m, int64_t k,
                                    int64_t tables, const double* d1, const double* d2,
                                    const double* d3, double scale, int32_t device) { SPN_TRY
  if (!out || !d1 || !d2 || !d3) return fail(SPN_EINVAL, "null argument");
  *out = nullptr;
  if (spn_status s = validate_shape(n, m, k, tables)) return s;
  if (scale != 0.0 && !std::isfinite(scale)) return fail(SPN_EDOMAIN, "non-finite scale");
  auto* p = new spn_plan();
  p->variant = -1;
  p->n = n;
  p->m = m;
  p->k = k;
  p->tables = tables;
  p->blocks = (k + m - 1) / m;
  p->device = device;
  p->scale = scale != 0.0 ? scale : std::sqrt(static_cast<double>(n));
  const size_t total = static_cast<size_t>(tables * p->blocks * n);
  const double* src[3] = {d1, d2, d3};
  for (int di = 0; di < 3; ++di) {
    p->d[di].assign(src[di], src[di] + total);
    for (double v : p->d[di])
      if (!std::isfinite(v)) {
        delete p;
        return fail(SPN_EDOMAIN, "non-finite diagonal entry");  // diag_matvec check, transforms.cpp:230
      }
  }
  if (spn_status s = finish_plan(p)) {
    delete p;
    return s;
  }
  *out = p;
  return SPN_OK;
  SPN_CATCH
}

// StructuredSpinner::resample_last_block / resample_tail / with_tail_vector (spinner.hpp:67-77,
// spinner.cpp:153-184): a new one-block plan with the source's realised parameters and the tail
// (and for resample_tail also D2) redrawn or replaced.
namespace {
spn_plan* clone_block(const spn_plan* src) {
  auto* p = new spn_plan();
  p->variant = src->variant;
  p->n = src->n;
  p->m = src->m;
  p->k = src->k;
  p->tables = 1;
  p->blocks = 1;
  p->device = src->device;
  p->scale = src->scale;
  for (int di = 0; di < 3; ++di) p->d[di] = src->d[di];
  p->trow = src->trow;
  p->dense = src->dense;
  return p;
}
spn_status one_block(const spn_plan* src, const char* what) {
  if (!src) return fail(SPN_EINVAL, "null plan");
  if (src->tables != 1 || src->blocks != 1)
    return fail(SPN_EUNSUPPORTED, std::string(what) + ": needs a one-block plan (StructuredSpinner)");
  return SPN_OK;
}
}  // namespace

spn_status spn_plan_resample(spn_plan** out, const spn_plan* src, int32_t mode, uint64_t tail_seed) { SPN_TRY
  if (!out) return fail(SPN_EINVAL, "null argument");
  *out = nullptr;
  if (spn_status st = one_block(src, "resample")) return st;
  if (mode != 0 && mode != 1) return fail(SPN_EINVAL, "resample: mode must be 0 (last block) or 1 (tail)");
  if (src->variant < 0) return fail(SPN_EUNSUPPORTED, "resample: plan was made from explicit diagonals");
  const_cast<spn_plan*>(src)->ensure_host_d();
  spn_plan* p = clone_block(src);
  const int64_t n = p->n;
  spn::HostRng rng(spn::mix_seed(tail_seed, mode == 0 ? 2 : 3));  // spinner.cpp:154 / :161
  if (mode == 1 && p->variant != SPN_GAUSSIAN_DENSE) {
    // resample_tail redraws D2 first (Rademacher; the builder-defined Gauss3 keeps its N(0,1) D2)
    for (int64_t i = 0; i < n; ++i) p->d[1][static_cast<size_t>(i)] = p->variant == SPN_GAUSS3 ? rng.gaussian() : rng.rademacher();
  }
  spn::draw_tail(p->variant, n, p->m, rng, p->d[2].data(), p->trow.empty() ? nullptr : p->trow.data(),
                 p->dense.empty() ? nullptr : p->dense.data());
  if (spn_status st = finish_plan(p)) {
    delete p;
    return st;
  }
  *out = p;
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_plan_with_tail(spn_plan** out, const spn_plan* src, const double* r) { SPN_TRY
  if (!out || !r) return fail(SPN_EINVAL, "null argument");
  *out = nullptr;
  if (spn_status st = one_block(src, "with_tail_vector")) return st;
  if (src->variant != SPN_HD3_HD2_HD1 && src->variant != SPN_HDG_HD2_HD1 && src->variant != SPN_GAUSS3 &&
      src->variant != -1)
    return fail(SPN_EDOMAIN, "with_tail_vector: only valid for Hadamard-only variants");
  for (int64_t i = 0; i < src->n; ++i)
    if (!std::isfinite(r[i])) return fail(SPN_EDOMAIN, "with_tail_vector: non-finite entry");
  const_cast<spn_plan*>(src)->ensure_host_d();
  spn_plan* p = clone_block(src);
  p->d[2].assign(r, r + p->n);
  if (spn_status st = finish_plan(p)) {
    delete p;
    return st;
  }
  *out = p;
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_plan_destroy(spn_plan* p) { SPN_TRY
  delete p;
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_plan_query(const spn_plan* p, int64_t* n, int64_t* m, int64_t* k, int64_t* tables,
                          int64_t* blocks, double* scale) { SPN_TRY
  if (!p) return fail(SPN_EINVAL, "null plan");
  if (n) *n = p->n;
  if (m) *m = p->m;
  if (k) *k = p->k;
  if (tables) *tables = p->tables;
  if (blocks) *blocks = p->blocks;
  if (scale) *scale = p->scale;
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_plan_diagonals(const spn_plan* p, double* d1, double* d2, double* d3) { SPN_TRY
  if (!p) return fail(SPN_EINVAL, "null plan");
  double* dst[3] = {d1, d2, d3};
  const_cast<spn_plan*>(p)->ensure_host_d();
  for (int di = 0; di < 3; ++di)
    if (dst[di]) std::copy(p->d[di].begin(), p->d[di].end(), dst[di]);
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_apply_f32(const spn_plan* p, const float* x, int64_t batch, int64_t ld_x,
                         int64_t n_in, float* y, int64_t ld_y, int32_t relu, void* stream) { SPN_TRY
  if (spn_status s = check_io(p, x, batch, ld_x, n_in)) return s;
  if (p->tables != 1) return fail(SPN_EINVAL, "apply needs a single-table plan");
  if (batch > 0 && !y) return fail(SPN_EINVAL, "null output");
  if (ld_y < p->k) return fail(SPN_EINVAL, "ld_y < k");
  if (p->fam) {
    DeviceGuard g(p->device);
    return spn::family_run(p->fam, 0, x, batch, ld_x, n_in, y, ld_y, relu, 0.0, static_cast<cudaStream_t>(stream));
  }
  if (p->log_n > kMaxLogNVec) {
    DeviceGuard g(p->device);
    const_cast<spn_plan*>(p)->ensure_host_d();
    return const_cast<spn_plan*>(p)->big.apply(x, batch, ld_x, n_in, y, ld_y, relu, p->k, p->m, p->blocks,
                        p->scale * std::pow(static_cast<double>(p->n), -1.5), p->sms,
                        static_cast<cudaStream_t>(stream));
  }
  spn::VecParams v = base_params(p);
  v.x = x;
  v.ld_x = ld_x;
  v.n_in = n_in;
  v.batch = batch;
  v.y = y;
  v.ld_y = ld_y;
  v.relu = relu;
  // 16-B aligned rows: the apply kernel may bulk-prefetch its next row into L2
  v.x_vec_ok = reinterpret_cast<uintptr_t>(x) % 16 == 0 && ld_x % 4 == 0;
  return run_vec(p, spn::OP_APPLY, v, static_cast<cudaStream_t>(stream));
  SPN_CATCH
}

spn_status spn_hash_f32(const spn_plan* p, const float* x, int64_t batch, int64_t ld_x,
                        int64_t n_in, int32_t* ids, float* y, int64_t ld_y, void* stream) { SPN_TRY
  if (spn_status s = check_io(p, x, batch, ld_x, n_in)) return s;
  if (batch > 0 && !ids) return fail(SPN_EINVAL, "null ids");
  if (p->fam) {
    if (y) return fail(SPN_EUNSUPPORTED, "hash with y output: circulant family / dense baseline");
    if (p->k >= (int64_t(1) << 30)) return fail(SPN_EDIM, "2k must fit int32 ids");
    DeviceGuard g(p->device);
    return spn::family_run(p->fam, 1, x, batch, ld_x, n_in, ids, p->tables, 0, 0.0, static_cast<cudaStream_t>(stream));
  }
  if (y && p->tables != 1) return fail(SPN_EINVAL, "y output needs a single-table plan");
  if (y && ld_y < p->k) return fail(SPN_EINVAL, "ld_y < k");
  if (p->k >= (int64_t(1) << 30)) return fail(SPN_EDIM, "2k must fit int32 ids");
  if (p->log_n > kMaxLogNVec)
    return big_hash(const_cast<spn_plan*>(p), x, batch, ld_x, n_in, ids, y, ld_y, static_cast<cudaStream_t>(stream));
  spn::VecParams v = base_params(p);
  v.x = x;
  v.ld_x = ld_x;
  v.n_in = n_in;
  v.batch = batch;
  v.ids = ids;
  v.y = y;
  v.ld_y = ld_y;
  // hash + y at n = 1024 in permuted coordinates (16-B x loads and y stores): full single-block rows,
  // sign diagonals, 16-B aligned rows (SPN_APPLY_PERM=0 turns it off)
  static const bool perm_on = [] {
    const char* e = std::getenv("SPN_APPLY_PERM");
    return !(e && e[0] == '0');
  }();
  auto al16 = [](const void* q, int64_t ld) { return reinterpret_cast<uintptr_t>(q) % 16 == 0 && ld % 4 == 0; };
  v.x_vec_ok = al16(x, ld_x);  // 16-B aligned rows: the apply kernel may bulk-prefetch its next row
  if (perm_on && y && ids && p->n == 1024 && p->vsgnP[0][0] && p->blocks == 1 && p->tables == 1 && p->m == 1024 &&
      p->k == 1024 && n_in == 1024 && al16(x, ld_x) && al16(y, ld_y)) {
    v.perm = 1;
    for (int di = 0; di < 3; ++di)
      for (int lay = 0; lay < 2; ++lay) v.d[di][lay].sgn = p->vsgnP[di][lay];
  }
  return run_vec(p, y ? spn::OP_APPLY : spn::OP_HASH, v, static_cast<cudaStream_t>(stream));
  SPN_CATCH
}

// collision_curve's counting core (lsh.cpp:54-61): per pair, how many tables give
// hash(x) == hash(y); one thread per pair, one atomic per pair.
__global__ void collision_count_kernel(const int32_t* __restrict__ ids, int64_t pairs, int tables,
                                       const int32_t* __restrict__ bucket_of,
                                       unsigned long long* __restrict__ hits) {
  for (int64_t pr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pr < pairs; pr += (int64_t)gridDim.x * blockDim.x) {
    const int32_t* a = ids + (2 * pr) * tables;
    const int32_t* b = a + tables;
    unsigned h = 0;
    for (int t = 0; t < tables; ++t) h += a[t] == b[t];
    if (h) atomicAdd(hits + bucket_of[pr], (unsigned long long)h);
  }
}

spn_status spn_collision_hits_f32(const spn_plan* p, const float* xy, int64_t pairs, int64_t ld, int64_t n_in,
                                  const int32_t* bucket_of, int64_t buckets, int64_t* hits, void* stream) { SPN_TRY
  if (spn_status s = check_io(p, xy, 2 * pairs, ld, n_in)) return s;
  if (pairs > 0 && (!bucket_of || !hits)) return fail(SPN_EINVAL, "null pointer");
  if (buckets < 1) return fail(SPN_EDIM, "collision_curve: need at least one bucket");
  if (pairs == 0) return SPN_OK;
  DeviceGuard g(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // ids for a chunk of pairs: [2 * chunk][tables] int32, <= 64 MB of stream-ordered scratch
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(pairs, (int64_t(8) << 20) / p->tables));
  spn::Scratch scratch;
  SPN_CUDA(scratch.alloc(sizeof(int32_t) * static_cast<size_t>(2 * chunk * p->tables), s));
  int32_t* ids = static_cast<int32_t*>(scratch.p);
  for (int64_t p0 = 0; p0 < pairs; p0 += chunk) {
    const int64_t pc = std::min(chunk, pairs - p0);
    if (spn_status st = spn_hash_f32(p, xy + 2 * p0 * ld, 2 * pc, ld, n_in, ids, nullptr, 0, stream)) return st;
    const int64_t blocks = std::min<int64_t>((pc + 255) / 256, int64_t(p->sms) * 8);
    collision_count_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
        ids, pc, static_cast<int>(p->tables), bucket_of + p0, reinterpret_cast<unsigned long long*>(hits));
    SPN_CUDA(cudaGetLastError());
  }
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_enable_peer_access(int32_t device, int32_t peer_device) { SPN_TRY
  int count = 0;
  SPN_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count || peer_device < 0 || peer_device >= count)
    return fail(SPN_EINVAL, "peer access: device index out of range");
  if (device == peer_device) return SPN_OK;
  int can = 0;
  SPN_CUDA(cudaDeviceCanAccessPeer(&can, device, peer_device));
  if (!can)
    return fail(SPN_EUNSUPPORTED, "no peer access from cuda:" + std::to_string(device) + " to cuda:" +
                                      std::to_string(peer_device));
  DeviceGuard g(device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    (void)cudaGetLastError();  // clear the (non-sticky) error state
    return SPN_OK;
  }
  SPN_CUDA(e);
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_hash_f32_peers(const spn_plan* p, const float* x, int64_t batch, int64_t ld_x, int64_t n_in,
                              int32_t* const* peers, int32_t npeers, int64_t row0, int64_t total,
                              void* stream) { SPN_TRY
  if (spn_status s = check_io(p, x, batch, ld_x, n_in)) return s;
  if (npeers < 1 || !peers) return fail(SPN_EINVAL, "need >= 1 peer table");
  if (row0 < 0 || row0 + batch > total)
    return fail(SPN_EINVAL, "peer hash: rows [row0, row0 + batch) outside the gathered table");
  if (p->fam) return fail(SPN_EUNSUPPORTED, "peer hash: Hadamard-only variants");
  if (p->k >= (int64_t(1) << 30)) return fail(SPN_EDIM, "2k must fit int32 ids");
  if (p->log_n > kMaxLogNVec) return fail(SPN_EUNSUPPORTED, "hash with n > 2^14 not implemented");
  spn::VecParams v = base_params(p);
  v.x = x;
  v.ld_x = ld_x;
  v.n_in = n_in;
  v.batch = batch;
  v.peers = peers;
  v.npeers = npeers;
  v.peer_row0 = row0;
  return run_vec(p, spn::OP_HASH, v, static_cast<cudaStream_t>(stream));
  SPN_CATCH
}

spn_status spn_embed_f32(const spn_plan* p, int32_t kind, double sigma, const float* x,
                         int64_t batch, int64_t ld_x, int64_t n_in, float* out, int64_t ld_out,
                         void* stream) { SPN_TRY
  if (spn_status s = check_io(p, x, batch, ld_x, n_in)) return s;
  if (p->tables != 1) return fail(SPN_EINVAL, "embed needs a single-table plan");
  if (kind != SPN_EMBED_GAUSSIAN && kind != SPN_EMBED_ANGULAR) return fail(SPN_EDOMAIN, "unknown kernel kind");
  if (kind == SPN_EMBED_GAUSSIAN && !(sigma > 0.0))
    return fail(SPN_EDOMAIN, "KernelKind: sigma must be positive");  // kernels.hpp:17
  if (batch > 0 && !out) return fail(SPN_EINVAL, "null output");
  if (ld_out < (kind == SPN_EMBED_GAUSSIAN ? 2 * p->k : p->k)) return fail(SPN_EINVAL, "ld_out too small");
  if (p->fam) {
    DeviceGuard g(p->device);
    return spn::family_run(p->fam, kind == SPN_EMBED_GAUSSIAN ? 2 : 3, x, batch, ld_x, n_in, out, ld_out, 0, sigma,
                           static_cast<cudaStream_t>(stream));
  }
  if (p->log_n > kMaxLogNVec)
    return big_embed(const_cast<spn_plan*>(p), kind, sigma, x, batch, ld_x, n_in, out, ld_out,
                     static_cast<cudaStream_t>(stream));
  spn::VecParams v = base_params(p);
  v.x = x;
  v.ld_x = ld_x;
  v.n_in = n_in;
  v.batch = batch;
  v.y = out;
  v.ld_y = ld_out;
  v.c2 = static_cast<float>(p->scale * std::pow(static_cast<double>(p->n), -1.5) / sigma);
  v.norm = static_cast<float>(1.0 / std::sqrt(static_cast<double>(p->k)));
  v.x_vec_ok = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && (ld_x % 4 == 0);
  // n = 1024, sign diagonals, full 1024-row blocks, 16-B aligned rows: permuted-coordinate
  // kernel with 16-B feature stores (config 2's shape)
  if (kind == SPN_EMBED_GAUSSIAN && p->n == 1024 && p->vsgnP[0][0] && v.x_vec_ok && p->m == 1024 &&
      p->k % 1024 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0 && ld_out % 4 == 0) {
    if (batch == 0) return SPN_OK;
    for (int di = 0; di < 3; ++di)
      for (int lay = 0; lay < 2; ++lay) v.d[di][lay].sgn = p->vsgnP[di][lay];
    DeviceGuard g(p->device);
    cudaError_t e = spn::vec_launcher_gauss_perm()(v, static_cast<cudaStream_t>(stream), p->sms, batch);
    return e == cudaSuccess ? SPN_OK : cuda_fail(e, "spinner_vec_kernel (permuted embed) launch");
  }
  return run_vec(p, kind == SPN_EMBED_GAUSSIAN ? spn::OP_EMBED_GAUSS : spn::OP_EMBED_ANG, v,
                 static_cast<cudaStream_t>(stream));
  SPN_CATCH
}

spn_status spn_sketch_f32(const spn_plan* p, const float* a, int64_t n_in, int64_t d, int64_t ld_a,
                          const int64_t* rows, int64_t m_out, double norm, float* out,
                          int64_t ld_out, void* stream) { SPN_TRY
  return sketch_dispatch(p, a, n_in, d, ld_a, rows, m_out, norm, out, ld_out, static_cast<cudaStream_t>(stream),
                         nullptr);
  SPN_CATCH
}

// SketchOperator::apply with the reference's value semantics (newton_sketch.cpp:87-101): host A in,
// host sketch out.  A goes to the device in one pass (linear copies when the rows are packed at a
// 16-B multiple), the sketch runs there, the m_out x d result comes back.
spn_status spn_sketch_f32_host(const spn_plan* cp, const float* a, int64_t n_in, int64_t d, int64_t ld_a,
                               const int64_t* rows, int64_t m_out, double norm, float* out,
                               int64_t ld_out) { SPN_TRY
  if (spn_status st = sketch_check(cp, a, n_in, d, ld_a, rows, m_out, out, ld_out)) return st;
  if (d == 0 || m_out == 0) return SPN_OK;
  if (host_ptr_kind(a) == cudaMemoryTypeDevice || host_ptr_kind(out) == cudaMemoryTypeDevice)
    return fail(SPN_EINVAL, "host entry point given a device pointer");
  auto* p = const_cast<spn_plan*>(cp);
  std::lock_guard<std::mutex> lock(p->mu);
  DeviceGuard g(p->device);
  if (!p->hs[0]) SPN_CUDA(cudaStreamCreateWithFlags(&p->hs[0], cudaStreamNonBlocking));
  cudaStream_t s = p->hs[0];
  const int64_t ldd = (d + 3) / 4 * 4;  // 16-B aligned device rows (the TMA column passes need them)
  spn::Scratch da, dout;
  SPN_CUDA(da.alloc(sizeof(float) * static_cast<size_t>(n_in * ldd), s));
  SPN_CUDA(dout.alloc(sizeof(float) * static_cast<size_t>(m_out * ldd), s));
  struct Drain {  // the copies reference the caller's buffers: complete them on every exit
    cudaStream_t s;
    ~Drain() { cudaStreamSynchronize(s); }
  } drain{s};
  float* A = static_cast<float*>(da.p);
  if (ld_a == ldd) {  // packed rows: linear copies of <= 32 MB
    const int64_t total = n_in * ldd, piece = int64_t(8) << 20;
    for (int64_t o = 0; o < total; o += piece)
      SPN_CUDA(cudaMemcpyAsync(A + o, a + o, sizeof(float) * static_cast<size_t>(std::min(piece, total - o)),
                               cudaMemcpyHostToDevice, s));
  } else {
    SPN_CUDA(cudaMemcpy2DAsync(A, ldd * 4, a, ld_a * 4, d * 4, n_in, cudaMemcpyHostToDevice, s));
  }
  float* O = static_cast<float*>(dout.p);
  if (spn_status st = sketch_dispatch(p, A, n_in, d, ldd, rows, m_out, norm, O, ldd, s, nullptr)) return st;
  SPN_CUDA(cudaMemcpy2DAsync(out, ld_out * 4, O, ldd * 4, d * 4, m_out, cudaMemcpyDeviceToHost, s));
  SPN_CUDA(cudaStreamSynchronize(s));
  return SPN_OK;
  SPN_CATCH
}

// --------------------------------------------------------------------- host-buffer API

}  // extern "C"

namespace spn {

int plan_device(const spn_plan* p) { return p->device; }

// First-m sketch of diag(row_scale) A (the Newton step's S * hessian_sqrt, newton_sketch.cpp:87-106).
spn_status plan_sketch_scaled(const spn_plan* p, const float* a, int64_t n_in, int64_t d, int64_t ld_a,
                              int64_t m_out, double norm, const float* row_scale, float* out, int64_t ld_out,
                              cudaStream_t s) {
  return sketch_dispatch(p, a, n_in, d, ld_a, nullptr, m_out, norm, out, ld_out, s, row_scale);
}

}  // namespace spn

namespace {

#ifndef SPN_HOST_CHUNK_DIV
#define SPN_HOST_CHUNK_DIV 32  // chunk ~ 1/DIV of the traffic: fill + drain ~ 2/DIV (c5 e2e 10.5k -> 10.8k vs 8)
#endif

// One host output of host_pipeline: rows of row_bytes at a host stride of ld_bytes.
struct HostOut {
  void* ptr;
  int64_t row_bytes, ld_bytes;
};

// Pipelined host->device->host execution over row chunks on two streams (up to two outputs per
// row, e.g. ids and y).  launch(dx, rows, n_in, dout0, dout1, stream) runs the device op on a chunk.
template <class Launch>
spn_status host_pipeline(spn_plan* p, const float* x, int64_t batch, int64_t ld_x, int64_t n_in, HostOut o0,
                         HostOut o1, Launch launch) {
  if (batch == 0) return SPN_OK;
  std::lock_guard<std::mutex> lock(p->mu);
  DeviceGuard g(p->device);
  const int64_t in_row = n_in * 4;
  // Chunks of ~1/8 of the traffic, 4..128 MB (the larger of input / output row bytes): small
  // calls still overlap H2D, kernel and D2H on the two copy engines; large ones keep the
  // per-chunk launch/copy overhead small.
  const int64_t row_bytes = std::max<int64_t>(std::max<int64_t>(o0.row_bytes + o1.row_bytes, in_row), 1);
  static const int64_t cap_mb = [] {
    const char* e = std::getenv("SPN_HOST_CHUNK_MB");
    const int64_t v = e ? std::atoll(e) : 128;  // config 3 (64 GiB in): 44.2 GB/s H2D vs 42.8 at 48 MB
    return v > 0 ? v : int64_t(128);
  }();
  static const int64_t min_kb = [] {
    const char* e = std::getenv("SPN_HOST_MIN_CHUNK_KB");
    const int64_t v = e ? std::atoll(e) : 4096;
    return v > 0 ? v : int64_t(4096);
  }();
  const int64_t target = std::min<int64_t>(cap_mb << 20,
                                           std::max<int64_t>(min_kb << 10, batch * row_bytes / SPN_HOST_CHUNK_DIV));
  int64_t chunk = std::max<int64_t>(1, target / row_bytes);
  chunk = std::min(chunk, batch);
  static const int nst = [] {
    const char* e = std::getenv("SPN_HOST_STREAMS");
    const int v = e ? std::atoi(e) : 2;
    return v < 1 ? 1 : (v > spn_plan::kHostStreams ? spn_plan::kHostStreams : v);
  }();
  for (int s = 0; s < nst; ++s) {
    if (!p->hs[s]) SPN_CUDA(cudaStreamCreateWithFlags(&p->hs[s], cudaStreamNonBlocking));
    const size_t need[3] = {static_cast<size_t>(chunk * in_row), static_cast<size_t>(chunk * o0.row_bytes),
                            static_cast<size_t>(chunk * o1.row_bytes)};
    for (int b = 0; b < 3; ++b)
      if (p->hbuf_bytes[s][b] < need[b]) {
        if (p->hbuf[s][b]) cudaFree(p->hbuf[s][b]);
        p->hbuf[s][b] = nullptr;
        p->hbuf_bytes[s][b] = 0;
        SPN_CUDA(cudaMalloc(&p->hbuf[s][b], need[b]));
        p->hbuf_bytes[s][b] = need[b];
      }
  }
  // on every exit the enqueued copies are complete (they reference the caller's host buffers)
  struct Drain {
    spn_plan* p;
    ~Drain() {
      for (cudaStream_t q : p->hs)
        if (q) cudaStreamSynchronize(q);
    }
  } drain{p};
  // A D2H copy into PAGEABLE memory does not return until it has completed, so the next chunk's H2D would
  // wait for this chunk's kernel: the copy engine idles (config 3 with numpy ids: 43 vs 55 GB/s).  Pageable
  // outputs therefore land in a pinned staging buffer per stream and are copied out on the host one round
  // later, after that stream has been synchronised (the other streams' copies keep the engine busy).
  const HostOut* outs[2] = {&o0, &o1};
  bool staged[2] = {false, false};
  if (host_ptr_kind(x) == cudaMemoryTypeDevice) return fail(SPN_EINVAL, "host entry point given a device input");
  for (int b = 0; b < 2; ++b) {
    if (!outs[b]->ptr) continue;
    const cudaMemoryType kind = host_ptr_kind(outs[b]->ptr);
    if (kind == cudaMemoryTypeDevice) return fail(SPN_EINVAL, "host entry point given a device output");
    staged[b] = kind != cudaMemoryTypeHost && kind != cudaMemoryTypeManaged;
    if (!staged[b]) continue;
    const size_t need = static_cast<size_t>(chunk * outs[b]->row_bytes);
    for (int s = 0; s < nst; ++s)
      if (p->hstage_bytes[s][b] < need) {
        if (p->hstage[s][b]) cudaFreeHost(p->hstage[s][b]);
        p->hstage[s][b] = nullptr;
        p->hstage_bytes[s][b] = 0;
        SPN_CUDA(cudaMallocHost(&p->hstage[s][b], need));
        p->hstage_bytes[s][b] = need;
      }
  }
  int64_t pend_r0[spn_plan::kHostStreams], pend_rows[spn_plan::kHostStreams];
  for (int s = 0; s < spn_plan::kHostStreams; ++s) pend_rows[s] = 0;
  auto flush = [&](int s) -> cudaError_t {  // stream s's staged outputs -> the caller's buffers
    if (pend_rows[s] == 0) return cudaSuccess;
    if (cudaError_t e = cudaStreamSynchronize(p->hs[s])) return e;
    for (int b = 0; b < 2; ++b) {
      if (!staged[b]) continue;
      const HostOut& o = *outs[b];
      const char* src = static_cast<const char*>(p->hstage[s][b]);
      char* dst = static_cast<char*>(o.ptr) + pend_r0[s] * o.ld_bytes;
      if (o.ld_bytes == o.row_bytes)
        std::memcpy(dst, src, static_cast<size_t>(o.row_bytes * pend_rows[s]));
      else
        for (int64_t r = 0; r < pend_rows[s]; ++r)
          std::memcpy(dst + r * o.ld_bytes, src + r * o.row_bytes, static_cast<size_t>(o.row_bytes));
    }
    pend_rows[s] = 0;
    return cudaSuccess;
  };
  auto d2h = [&](int b, int64_t r0, int64_t rows, const void* dsrc, int s) -> cudaError_t {
    const HostOut& o = *outs[b];
    if (!o.ptr) return cudaSuccess;
    cudaStream_t st = p->hs[s];
    if (staged[b]) return cudaMemcpyAsync(p->hstage[s][b], dsrc, o.row_bytes * rows, cudaMemcpyDeviceToHost, st);
    char* dst = static_cast<char*>(o.ptr) + r0 * o.ld_bytes;
    if (o.ld_bytes == o.row_bytes) return cudaMemcpyAsync(dst, dsrc, o.row_bytes * rows, cudaMemcpyDeviceToHost, st);
    return cudaMemcpy2DAsync(dst, o.ld_bytes, dsrc, o.row_bytes, o.row_bytes, rows, cudaMemcpyDeviceToHost, st);
  };
  int c = 0;
  for (int64_t r0 = 0; r0 < batch; r0 += chunk, ++c) {
    const int s = c % nst;
    const int64_t rows = std::min(chunk, batch - r0);
    SPN_CUDA(flush(s));  // stream s's previous chunk (nst chunks ago)
    float* dx = static_cast<float*>(p->hbuf[s][0]);
    char* dout0 = static_cast<char*>(p->hbuf[s][1]);
    char* dout1 = static_cast<char*>(p->hbuf[s][2]);
    if (ld_x * 4 == in_row)  // contiguous rows: one linear copy
      SPN_CUDA(cudaMemcpyAsync(dx, x + r0 * ld_x, in_row * rows, cudaMemcpyHostToDevice, p->hs[s]));
    else
      SPN_CUDA(cudaMemcpy2DAsync(dx, in_row, x + r0 * ld_x, ld_x * 4, in_row, rows, cudaMemcpyHostToDevice,
                                 p->hs[s]));
    if (spn_status st = launch(dx, rows, n_in, dout0, dout1, p->hs[s])) return st;
    SPN_CUDA(d2h(0, r0, rows, dout0, s));
    SPN_CUDA(d2h(1, r0, rows, dout1, s));
    if (staged[0] || staged[1]) {
      pend_r0[s] = r0;
      pend_rows[s] = rows;
    }
  }
  for (int s = 0; s < nst; ++s) {
    SPN_CUDA(cudaStreamSynchronize(p->hs[s]));
    SPN_CUDA(flush(s));
  }
  return SPN_OK;
}

}  // namespace

extern "C" {

spn_status spn_apply_f32_host(const spn_plan* cp, const float* x, int64_t batch, int64_t ld_x,
                              int64_t n_in, float* y, int64_t ld_y, int32_t relu) { SPN_TRY
  if (spn_status s = check_io(cp, x, batch, ld_x, n_in)) return s;
  if (batch > 0 && !y) return fail(SPN_EINVAL, "null output");
  if (ld_y < cp->k) return fail(SPN_EINVAL, "ld_y < k");
  auto* p = const_cast<spn_plan*>(cp);
  return host_pipeline(p, x, batch, ld_x, n_in, HostOut{y, p->k * 4, ld_y * 4}, HostOut{nullptr, 0, 0},
                       [&](const float* dx, int64_t rows, int64_t nin, char* dout, char*, cudaStream_t s) {
                         return spn_apply_f32(p, dx, rows, nin, nin, reinterpret_cast<float*>(dout), p->k, relu, s);
                       });
  SPN_CATCH
}

spn_status spn_hash_f32_host(const spn_plan* cp, const float* x, int64_t batch, int64_t ld_x,
                             int64_t n_in, int32_t* ids) { SPN_TRY
  if (spn_status s = check_io(cp, x, batch, ld_x, n_in)) return s;
  if (batch > 0 && !ids) return fail(SPN_EINVAL, "null ids");
  auto* p = const_cast<spn_plan*>(cp);
  return host_pipeline(p, x, batch, ld_x, n_in, HostOut{ids, p->tables * 4, p->tables * 4}, HostOut{nullptr, 0, 0},
                       [&](const float* dx, int64_t rows, int64_t nin, char* dout, char*, cudaStream_t s) {
                         return spn_hash_f32(p, dx, rows, nin, nin, reinterpret_cast<int32_t*>(dout), nullptr, 0, s);
                       });
  SPN_CATCH
}

spn_status spn_hash_project_f32_host(const spn_plan* cp, const float* x, int64_t batch, int64_t ld_x, int64_t n_in,
                                     int32_t* ids, float* y, int64_t ld_y) { SPN_TRY
  if (spn_status s = check_io(cp, x, batch, ld_x, n_in)) return s;
  if (batch > 0 && (!ids || !y)) return fail(SPN_EINVAL, "null output");
  if (cp->tables != 1) return fail(SPN_EINVAL, "y output needs a single-table plan");
  if (ld_y < cp->k) return fail(SPN_EINVAL, "ld_y < k");
  auto* p = const_cast<spn_plan*>(cp);
  return host_pipeline(p, x, batch, ld_x, n_in, HostOut{ids, 4, 4}, HostOut{y, p->k * 4, ld_y * 4},
                       [&](const float* dx, int64_t rows, int64_t nin, char* dids, char* dy, cudaStream_t s) {
                         return spn_hash_f32(p, dx, rows, nin, nin, reinterpret_cast<int32_t*>(dids),
                                             reinterpret_cast<float*>(dy), p->k, s);
                       });
  SPN_CATCH
}

spn_status spn_embed_f32_host(const spn_plan* cp, int32_t kind, double sigma, const float* x,
                              int64_t batch, int64_t ld_x, int64_t n_in, float* out, int64_t ld_out) { SPN_TRY
  if (spn_status s = check_io(cp, x, batch, ld_x, n_in)) return s;
  const int64_t w = kind == SPN_EMBED_GAUSSIAN ? 2 * cp->k : cp->k;
  if (batch > 0 && !out) return fail(SPN_EINVAL, "null output");
  if (ld_out < w) return fail(SPN_EINVAL, "ld_out too small");
  auto* p = const_cast<spn_plan*>(cp);
  return host_pipeline(p, x, batch, ld_x, n_in, HostOut{out, w * 4, ld_out * 4}, HostOut{nullptr, 0, 0},
                       [&](const float* dx, int64_t rows, int64_t nin, char* dout, char*, cudaStream_t s) {
                         return spn_embed_f32(p, kind, sigma, dx, rows, nin, nin, reinterpret_cast<float*>(dout), w, s);
                       });
  SPN_CATCH
}

// ------------------------------------------------ standalone transforms (transforms.hpp:13,59)

}  // extern "C"

namespace {

// unit-diagonal plans for spn_fwht_f32, one per (device, n), alive for the process
spn_plan* fwht_plan(int64_t n, int32_t device, spn_status* st) {
  static std::mutex mu;
  static std::map<std::pair<int32_t, int64_t>, spn_plan*> plans;
  std::lock_guard<std::mutex> lock(mu);
  auto it = plans.find({device, n});
  if (it != plans.end()) return it->second;
  std::vector<double> ones(static_cast<size_t>(n), 1.0);
  spn_plan* p = nullptr;
  *st = spn_plan_create_explicit(&p, n, n, n, 1, ones.data(), ones.data(), ones.data(), 1.0, device);
  if (*st != SPN_OK) return nullptr;
  plans[{device, n}] = p;
  return p;
}

spn_status fwht_args(int64_t n, const void* x, int64_t batch, int64_t ld_x, const void* y, int64_t ld_y) {
  if (n < 1 || (n & (n - 1)) != 0)
    return fail(SPN_EDIM, "fwht_normalized: length must be a power of two, got " + std::to_string(n));
  if (n > (int64_t(1) << kMaxLogN)) return fail(SPN_EUNSUPPORTED, "n > 2^20 not supported");
  if (batch < 0 || ld_x < n || ld_y < n) return fail(SPN_EINVAL, "bad batch or leading dimension");
  if (batch > 0 && (!x || !y)) return fail(SPN_EINVAL, "null pointer");
  return SPN_OK;
}

__global__ void diag_rows_kernel(int64_t n, const float* __restrict__ d, const float* x, int64_t batch, int64_t ld_x,
                                 float* y, int64_t ld_y) {
  const int64_t total = n * batch;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / n, i = e - b * n;
    y[b * ld_y + i] = d[i] * x[b * ld_x + i];
  }
}

}  // namespace

extern "C" {

spn_status spn_fwht_f32(int64_t n, const float* x, int64_t batch, int64_t ld_x, float* y, int64_t ld_y,
                        int32_t device, void* stream) { SPN_TRY
  if (spn_status s = fwht_args(n, x, batch, ld_x, y, ld_y)) return s;
  if (batch == 0) return SPN_OK;
  DeviceGuard g(device);
  if (n == 1) {  // H_1 = [1]
    if (x != y)
      SPN_CUDA(cudaMemcpy2DAsync(y, ld_y * 4, x, ld_x * 4, 4, batch, cudaMemcpyDeviceToDevice,
                                 static_cast<cudaStream_t>(stream)));
    return SPN_OK;
  }
  spn_status st = SPN_OK;
  spn_plan* p = fwht_plan(n, device, &st);
  if (!p) return st;
  return spn_apply_f32(p, x, batch, ld_x, n, y, ld_y, 0, stream);
  SPN_CATCH
}

spn_status spn_fwht_f32_host(int64_t n, const float* x, int64_t batch, int64_t ld_x, float* y, int64_t ld_y,
                             int32_t device) { SPN_TRY
  if (spn_status s = fwht_args(n, x, batch, ld_x, y, ld_y)) return s;
  if (batch == 0) return SPN_OK;
  if (n == 1) {
    for (int64_t b = 0; b < batch; ++b) y[b * ld_y] = x[b * ld_x];
    return SPN_OK;
  }
  spn_status st = SPN_OK;
  spn_plan* p = fwht_plan(n, device, &st);
  if (!p) return st;
  return spn_apply_f32_host(p, x, batch, ld_x, n, y, ld_y, 0);
  SPN_CATCH
}

spn_status spn_diag_f32(int64_t n, const float* d, const float* x, int64_t batch, int64_t ld_x, float* y,
                        int64_t ld_y, void* stream) { SPN_TRY
  if (n < 1 || batch < 0 || ld_x < n || ld_y < n) return fail(SPN_EDIM, "diag_matvec: length mismatch");
  if (batch == 0) return SPN_OK;
  if (!d || !x || !y) return fail(SPN_EINVAL, "null pointer");
  int dev = 0;
  SPN_CUDA(cudaGetDevice(&dev));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n * batch + 255) / 256, int64_t(sms) * 8));
  diag_rows_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, d, x, batch, ld_x,
                                                                                                  y, ld_y);
  SPN_CUDA(cudaGetLastError());
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_diag_f32_host(int64_t n, const float* d, const float* x, int64_t batch, int64_t ld_x, float* y,
                             int64_t ld_y, int32_t device) { SPN_TRY
  if (n < 1 || batch < 0 || ld_x < n || ld_y < n) return fail(SPN_EDIM, "diag_matvec: length mismatch");
  if (batch == 0) return SPN_OK;
  if (!d || !x || !y) return fail(SPN_EINVAL, "null pointer");
  DeviceGuard g(device);
  float *dd = nullptr, *dx = nullptr;
  const size_t row = static_cast<size_t>(n) * 4;
  cudaError_t e = cudaMalloc(&dd, row);
  if (e == cudaSuccess) e = cudaMalloc(&dx, row * static_cast<size_t>(batch));
  if (e == cudaSuccess) e = cudaMemcpy(dd, d, row, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy2D(dx, row, x, ld_x * 4, row, batch, cudaMemcpyHostToDevice);
  spn_status st = e == cudaSuccess ? spn_diag_f32(n, dd, dx, batch, n, dx, n, nullptr) : cuda_fail(e, "diag_matvec");
  if (st == SPN_OK) {
    e = cudaMemcpy2D(y, ld_y * 4, dx, row, row, batch, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = cuda_fail(e, "diag_matvec");
  }
  cudaFree(dd);
  cudaFree(dx);
  return st;
  SPN_CATCH
}

}  // extern "C"

// ------------------------------------------------------------------ row checks

namespace {
__global__ void check_rows_kernel(const float* __restrict__ x, int64_t batch, int64_t ld, int64_t n_in,
                                  int32_t* flags) {
  for (int64_t r = blockIdx.x; r < batch; r += gridDim.x) {
    int bad = 0, nz = 0;
    for (int64_t i = threadIdx.x; i < n_in; i += blockDim.x) {
      const float v = x[r * ld + i];
      bad |= !isfinite(v);
      nz |= (v != 0.0f);
    }
    bad = __syncthreads_or(bad);
    nz = __syncthreads_or(nz);
    if (threadIdx.x == 0) flags[r] = (bad ? 1 : 0) | (nz ? 0 : 2);
  }
}
}  // namespace

extern "C" spn_status spn_check_rows_f32(const float* x, int64_t batch, int64_t ld_x, int64_t n_in,
                                         int32_t* flags, void* stream) { SPN_TRY
  if (batch < 0 || n_in < 1 || ld_x < n_in) return fail(SPN_EINVAL, "bad shape");
  if (batch == 0) return SPN_OK;
  if (!x || !flags) return fail(SPN_EINVAL, "null pointer");
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(batch, 65535));
  check_rows_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(x, batch, ld_x, n_in, flags);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "check_rows_kernel");
  return SPN_OK;
  SPN_CATCH
}
