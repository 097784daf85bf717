// Gram-matrix consumers of the feature maps:
// gram_exact / gram_approx / gram_error of proj/src/kernels.cpp:38-114.
//
// gram_approx is F F^T over the device features of embed() (fp32 in, fp64 sums, 64 x 64
// output tiles, lower tiles computed and mirrored); gram_exact evaluates the exact kernel
// pairwise in fp64 from fp32 points; gram_error reduces both Frobenius norms with
// per-CTA partials summed in a fixed order.  Every sum runs over its index in increasing
// order, as the reference's loops do.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "../../include/spinners_b200.h"
#include "errors.hpp"

namespace {

constexpr int kGT = 64;  // output tile
constexpr int kGK = 32;  // k chunk staged in smem

// out[i][j] = sum_k F[i][k] F[j][k]; epilogue: gaussian -> diag 1; angular -> 0.5 + dot/(2 d'), diag 1.
__global__ void __launch_bounds__(256) gram_dots_kernel(const float* __restrict__ F, int64_t ld, int64_t count,
                                                        int64_t width, int kind, double inv2dp,
                                                        double* __restrict__ out, int64_t ldo) {
  __shared__ double Fi[kGK][kGT + 1];
  __shared__ double Fj[kGK][kGT + 1];
  const int t = blockIdx.x;
  int bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
  while (bi * (bi + 1) / 2 > t) --bi;
  const int bj = t - bi * (bi + 1) / 2;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t k0 = 0; k0 < width; k0 += kGK) {
    for (int e = threadIdx.x; e < kGK * kGT; e += 256) {
      const int rr = e / kGK, kk = e - rr * kGK;  // consecutive threads walk k (coalesced rows)
      const int64_t i = (int64_t)bi * kGT + rr, j = (int64_t)bj * kGT + rr, k = k0 + kk;
      Fi[kk][rr] = (i < count && k < width) ? (double)F[i * ld + k] : 0.0;
      Fj[kk][rr] = (j < count && k < width) ? (double)F[j * ld + k] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kGK; ++kk) {
      double u[4], v[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) u[a] = Fi[kk][ty * 4 + a];
#pragma unroll
      for (int b = 0; b < 4; ++b) v[b] = Fj[kk][tx * 4 + b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(u[a], v[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t i = (int64_t)bi * kGT + ty * 4 + a, j = (int64_t)bj * kGT + tx * 4 + b;
      if (i >= count || j >= count || j > i) continue;
      double v = acc[a][b];
      if (kind == SPN_EMBED_ANGULAR) v = 0.5 + inv2dp * v;
      if (i == j) v = 1.0;
      out[i * ldo + j] = v;
      out[j * ldo + i] = v;
    }
}

__global__ void row_norms_kernel(const float* __restrict__ P, int64_t ld, int64_t count, int64_t dim,
                                 double* __restrict__ norms) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t t = 0; t < dim; ++t) {
      const double v = (double)P[i * ld + t];
      s += v * v;
    }
    norms[i] = sqrt(s);
  }
}

// kernels.cpp:55-76: thread per (i, j > i); gaussian exp(-|pi - pj|^2 / (2 sigma^2)),
// angular 1 - acos(clamp(<pi, pj> / (|pi| |pj|))) / pi; diagonal 1.
__global__ void gram_exact_kernel(const float* __restrict__ P, int64_t ld, int64_t count, int64_t dim, int kind,
                                  double sigma, const double* __restrict__ norms, double* __restrict__ out,
                                  int64_t ldo) {
  const int64_t total = count * count;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / count, j = e - i * count;
    if (j < i) continue;
    if (j == i) {
      out[i * ldo + i] = 1.0;
      continue;
    }
    const float* pi = P + i * ld;
    const float* pj = P + j * ld;
    double value;
    if (kind == SPN_EMBED_GAUSSIAN) {
      double d2 = 0.0;
      for (int64_t t = 0; t < dim; ++t) {
        const double diff = (double)pi[t] - (double)pj[t];
        d2 += diff * diff;
      }
      value = exp(-d2 / (2.0 * sigma * sigma));
    } else {
      double dot = 0.0;
      for (int64_t t = 0; t < dim; ++t) dot += (double)pi[t] * (double)pj[t];
      double c = dot / (norms[i] * norms[j]);
      c = fmin(fmax(c, -1.0), 1.0);
      value = 1.0 - acos(c) / 3.14159265358979323846;
    }
    out[i * ldo + j] = value;
    out[j * ldo + i] = value;
  }
}

// per-CTA partial sums of (exact - approx)^2 and exact^2
__global__ void __launch_bounds__(256) gram_err_partial_kernel(const double* __restrict__ E,
                                                               const double* __restrict__ A, int64_t count,
                                                               int64_t ld, double* __restrict__ part) {
  __shared__ double s0[256], s1[256];
  double a = 0.0, b = 0.0;
  const int64_t total = count * count;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / count, j = e - i * count;
    const double x = E[i * ld + j], y = A[i * ld + j];
    a += (x - y) * (x - y);
    b += x * x;
  }
  s0[threadIdx.x] = a;
  s1[threadIdx.x] = b;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s0[threadIdx.x] += s0[threadIdx.x + o];
      s1[threadIdx.x] += s1[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s0[0];
    part[2 * blockIdx.x + 1] = s1[0];
  }
}

__global__ void gram_err_final_kernel(const double* __restrict__ part, int nparts, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double a = 0.0, b = 0.0;
  for (int k = 0; k < nparts; ++k) {
    a += part[2 * k];
    b += part[2 * k + 1];
  }
  out[0] = a;
  out[1] = b;
}

spn_status fail(spn_status s, const char* msg) { return spn::set_error(s, msg); }

int sms_of_current() {
  int dev = 0, s = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
  return s > 0 ? s : 148;
}

#define GRAM_CUDA(call)                                          \
  do {                                                           \
    cudaError_t e_ = (call);                                     \
    if (e_ != cudaSuccess) return spn::cuda_error(e_, #call);    \
  } while (0)

}  // namespace

extern "C" {

spn_status spn_gram_approx_f32(const float* features, int64_t count, int64_t width, int64_t ld, int32_t kind,
                               int64_t dprime, double* gram, int64_t ld_gram, void* stream) { SPN_TRY
  if (count < 1) return fail(SPN_EDIM, "gram_approx: empty dataset");
  if (!features || !gram) return fail(SPN_EINVAL, "null pointer");
  if (ld < width || ld_gram < count || width < 1) return fail(SPN_EINVAL, "bad leading dimension");
  if (kind != SPN_EMBED_GAUSSIAN && kind != SPN_EMBED_ANGULAR) return fail(SPN_EDOMAIN, "unknown kernel kind");
  if (dprime < 1) return fail(SPN_EDIM, "gram_approx: d' must be >= 1");
  const int64_t T = (count + kGT - 1) / kGT;
  if (T * (T + 1) / 2 > (int64_t(1) << 31) - 1) return fail(SPN_EUNSUPPORTED, "gram_approx: count too large");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  gram_dots_kernel<<<static_cast<unsigned>(T * (T + 1) / 2), 256, 0, s>>>(
      features, ld, count, width, kind, 1.0 / (2.0 * static_cast<double>(dprime)), gram, ld_gram);
  GRAM_CUDA(cudaGetLastError());
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_gram_exact_f32(const float* points, int64_t count, int64_t dim, int64_t ld, int32_t kind, double sigma,
                              double* gram, int64_t ld_gram, void* stream) { SPN_TRY
  if (count < 1) return fail(SPN_EDIM, "gram_exact: empty dataset");
  if (!points || !gram) return fail(SPN_EINVAL, "null pointer");
  if (ld < dim || ld_gram < count || dim < 1) return fail(SPN_EINVAL, "bad leading dimension");
  if (kind != SPN_EMBED_GAUSSIAN && kind != SPN_EMBED_ANGULAR) return fail(SPN_EDOMAIN, "unknown kernel kind");
  if (kind == SPN_EMBED_GAUSSIAN && !(sigma > 0.0)) return fail(SPN_EDOMAIN, "KernelKind: sigma must be positive");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int sms = sms_of_current();
  double* norms = nullptr;
  if (kind == SPN_EMBED_ANGULAR) {
    GRAM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&norms), sizeof(double) * static_cast<size_t>(count), s));
    row_norms_kernel<<<static_cast<unsigned>(std::min<int64_t>((count + 255) / 256, sms * 8)), 256, 0, s>>>(
        points, ld, count, dim, norms);
  }
  const int64_t total = count * count;
  gram_exact_kernel<<<static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, int64_t(sms) * 32)), 256, 0, s>>>(
      points, ld, count, dim, kind, sigma, norms, gram, ld_gram);
  cudaError_t e = cudaGetLastError();
  if (norms) cudaFreeAsync(norms, s);
  if (e != cudaSuccess) return spn::cuda_error(e, "gram_exact");
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_gram_error(const double* exact, const double* approx, int64_t count, int64_t ld, double* err,
                          void* stream) { SPN_TRY
  if (!exact || !approx || !err) return fail(SPN_EINVAL, "null pointer");
  if (count < 1 || ld < count) return fail(SPN_EDIM, "gram_error: shape mismatch");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int parts = std::min<int64_t>((count * count + 255) / 256, int64_t(sms_of_current()) * 2);
  double* part = nullptr;
  GRAM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(double) * static_cast<size_t>(2 * parts + 2), s));
  gram_err_partial_kernel<<<parts, 256, 0, s>>>(exact, approx, count, ld, part);
  gram_err_final_kernel<<<1, 32, 0, s>>>(part, parts, part + 2 * parts);
  double h[2] = {0.0, 0.0};
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, part + 2 * parts, sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(part, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return spn::cuda_error(e, "gram_error");
  if (h[1] == 0.0) return fail(SPN_EDOMAIN, "gram_error: exact Gram matrix is zero");
  *err = std::sqrt(h[0]) / std::sqrt(h[1]);  // (exact - approx).norm() / exact.norm()
  return SPN_OK;
  SPN_CATCH
}

// ------------------------------------------------------------- host-buffer forms
namespace {
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};
}  // namespace

spn_status spn_gram_exact_host(const float* points, int64_t count, int64_t dim, int32_t kind, double sigma,
                               double* gram) { SPN_TRY
  if (!points || !gram) return fail(SPN_EINVAL, "null pointer");
  if (count < 1) return fail(SPN_EDIM, "gram_exact: empty dataset");
  DevBuf dp, dg;
  GRAM_CUDA(cudaMalloc(&dp.p, sizeof(float) * static_cast<size_t>(count * dim)));
  GRAM_CUDA(cudaMalloc(&dg.p, sizeof(double) * static_cast<size_t>(count * count)));
  GRAM_CUDA(cudaMemcpy(dp.p, points, sizeof(float) * static_cast<size_t>(count * dim), cudaMemcpyHostToDevice));
  if (spn_status st = spn_gram_exact_f32(static_cast<float*>(dp.p), count, dim, dim, kind, sigma,
                                         static_cast<double*>(dg.p), count, nullptr))
    return st;
  GRAM_CUDA(cudaMemcpy(gram, dg.p, sizeof(double) * static_cast<size_t>(count * count), cudaMemcpyDeviceToHost));
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_gram_approx_host(const spn_plan* plan, int32_t kind, double sigma, const float* points, int64_t count,
                                int64_t dim, double* gram) { SPN_TRY
  if (!plan || !points || !gram) return fail(SPN_EINVAL, "null pointer");
  if (count < 1) return fail(SPN_EDIM, "gram_approx: empty dataset");
  int64_t n = 0, m = 0, k = 0, tables = 0, blocks = 0;
  double scale = 0.0;
  if (spn_status st = spn_plan_query(plan, &n, &m, &k, &tables, &blocks, &scale)) return st;
  const int64_t width = kind == SPN_EMBED_GAUSSIAN ? 2 * k : k;
  DevBuf dp, df, dg;
  GRAM_CUDA(cudaMalloc(&dp.p, sizeof(float) * static_cast<size_t>(count * dim)));
  GRAM_CUDA(cudaMalloc(&df.p, sizeof(float) * static_cast<size_t>(count * width)));
  GRAM_CUDA(cudaMalloc(&dg.p, sizeof(double) * static_cast<size_t>(count * count)));
  GRAM_CUDA(cudaMemcpy(dp.p, points, sizeof(float) * static_cast<size_t>(count * dim), cudaMemcpyHostToDevice));
  if (spn_status st = spn_embed_f32(plan, kind, sigma, static_cast<float*>(dp.p), count, dim, dim,
                                    static_cast<float*>(df.p), width, nullptr))
    return st;
  if (spn_status st = spn_gram_approx_f32(static_cast<float*>(df.p), count, width, width, kind, k,
                                          static_cast<double*>(dg.p), count, nullptr))
    return st;
  GRAM_CUDA(cudaMemcpy(gram, dg.p, sizeof(double) * static_cast<size_t>(count * count), cudaMemcpyDeviceToHost));
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_gram_error_host(const double* exact, const double* approx, int64_t count, double* err) { SPN_TRY
  if (!exact || !approx || !err) return fail(SPN_EINVAL, "null pointer");
  if (count < 1) return fail(SPN_EDIM, "gram_error: shape mismatch");
  DevBuf da, db;
  const size_t bytes = sizeof(double) * static_cast<size_t>(count * count);
  GRAM_CUDA(cudaMalloc(&da.p, bytes));
  GRAM_CUDA(cudaMalloc(&db.p, bytes));
  GRAM_CUDA(cudaMemcpy(da.p, exact, bytes, cudaMemcpyHostToDevice));
  GRAM_CUDA(cudaMemcpy(db.p, approx, bytes, cudaMemcpyHostToDevice));
  return spn_gram_error(static_cast<double*>(da.p), static_cast<double*>(db.p), count, count, err, nullptr);
  SPN_CATCH
}

}  // extern "C"
