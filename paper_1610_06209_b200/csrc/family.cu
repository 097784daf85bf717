// The rest of the spinner family: the circulant-family
// variants G D2 H D1 with G a Gaussian circulant / Toeplitz / skew-circulant matrix
// (proj/src/spinner.cpp:108-126, transforms.cpp:112-208) and the unstructured
// Gaussian dense baseline (spinner.cpp:127-132,208-214).
//
// Circulant family: one CTA per (vector, table); the vector lives in shared memory as
// complex fp64 (N <= 2^13: 128 KB) — an fp32 FFT missed the 1e-5 feature bar (1.3-1.8e-5
// at n = 2048: the cos/sin arguments |y|/sigma reach ~100, amplifying the FFT rounding).
// Per block: D1 -> normalised FWHT -> D2 -> the correlation with the generator's first
// row / column through an in-house radix-2 FFT of length N (n, or 2n
// for the Toeplitz embedding): forward DIF (natural -> bit-reversed), multiply by the
// precomputed conj(spectrum) stored in bit-reversed order, inverse DIT (bit-reversed ->
// natural), 1/N.  Twiddles come from an fp64-computed table (transforms.cpp:24-25 uses
// the recurrence w *= wlen; the table is the exact e^{-2 pi i t / N} rounded once).
// Dense baseline: a tiled fp32 GEMM Y = scale * X G^T per block, then the epilogue.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include "../../include/spinners_b200.h"
#include "errors.hpp"
#include "family.hpp"

namespace spn {

namespace {

constexpr int kFT = 256;  // threads per family CTA

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

struct FamParams {
  const float* x;
  int64_t ld_x, n_in, batch;
  int n, N, logN, m, k, blocks, tables, kind;  // kind: 2 circ, 3 toeplitz, 4 skew
  const float* d1;     // [tables][blocks][n]
  const float* d2;
  const double2* spec;  // [tables][blocks][N], bit-reversed order, conj applied
  const double2* tw;    // [N/2]  e^{-2 pi i t / N}
  const double2* skw;   // [n]    e^{+i pi t / n} (skew twiddle)
  float scale;
  int op;              // 0 apply, 1 hash, 2 embed gaussian, 3 embed angular
  float inv_sigma, norm;
  int relu;
  void* out;
  int64_t ld_out;
};

__global__ void __launch_bounds__(kFT) family_kernel(const FamParams p) {
  extern __shared__ double2 c[];  // [N]
  __shared__ float red_v[kFT];
  __shared__ int red_i[kFT];
  __shared__ float red_y[kFT];
  const int tid = threadIdx.x;
  const int64_t items = p.batch * (p.op == 1 ? p.tables : 1);
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int64_t v = p.op == 1 ? item / p.tables : item;
    const int tab = p.op == 1 ? (int)(item - v * p.tables) : 0;
    const float* xrow = p.x + v * p.ld_x;
    float best = -1.0f, bestv = 0.0f;
    int besti = 0x7fffffff;
    for (int b = 0; b < p.blocks; ++b) {
      const int64_t tb = (int64_t)tab * p.blocks + b;
      const float* D1 = p.d1 + tb * p.n;
      const float* D2 = p.d2 + tb * p.n;
      // D1, normalised FWHT (transforms.cpp:52-71), D2 (in the real parts)
      for (int i = tid; i < p.N; i += kFT)
        c[i] = make_double2(i < p.n && i < p.n_in ? (double)xrow[i] * (double)D1[i] : 0.0, 0.0);
      __syncthreads();
      for (int h = 1; h < p.n; h <<= 1) {
        for (int q = tid; q < p.n / 2; q += kFT) {
          const int i = (q / h) * 2 * h + (q % h);
          const double u = c[i].x, w = c[i + h].x;
          c[i].x = u + w;
          c[i + h].x = u - w;
        }
        __syncthreads();
      }
      const double rn = 1.0 / sqrt((double)p.n);
      for (int i = tid; i < p.n; i += kFT) {
        const double val = c[i].x * rn * (double)D2[i];
        c[i] = p.kind == 4 ? make_double2(val * p.skw[i].x, val * p.skw[i].y) : make_double2(val, 0.0);
      }
      __syncthreads();
      // forward DIF: natural -> bit-reversed
      for (int len = p.N; len >= 2; len >>= 1) {
        const int half = len >> 1, stride = p.N / len;
        for (int q = tid; q < p.N / 2; q += kFT) {
          const int blk = q / half, kk = q - blk * half, i = blk * len + kk;
          const double2 u = c[i], w = c[i + half];
          c[i] = make_double2(u.x + w.x, u.y + w.y);
          c[i + half] = cmul(make_double2(u.x - w.x, u.y - w.y), p.tw[kk * stride]);
        }
        __syncthreads();
      }
      const double2* S = p.spec + tb * p.N;
      for (int i = tid; i < p.N; i += kFT) c[i] = cmul(c[i], S[i]);
      __syncthreads();
      // inverse DIT: bit-reversed -> natural
      for (int len = 2; len <= p.N; len <<= 1) {
        const int half = len >> 1, stride = p.N / len;
        for (int q = tid; q < p.N / 2; q += kFT) {
          const int blk = q / half, kk = q - blk * half, i = blk * len + kk;
          const double2 u = c[i], w = cmulc(c[i + half], p.tw[kk * stride]);
          c[i] = make_double2(u.x + w.x, u.y + w.y);
          c[i + half] = make_double2(u.x - w.x, u.y - w.y);
        }
        __syncthreads();
      }
      const double invN = 1.0 / (double)p.N;
      const int rows = min(p.m, p.k - b * p.m);
      for (int i = tid; i < rows; i += kFT) {
        const double2 z = c[i];
        const double yd = p.kind == 4 ? (z.x * p.skw[i].x + z.y * p.skw[i].y) : z.x;  // real(z * conj(skw))
        float y = (float)(yd * invN * (double)p.scale);
        const int64_t col = (int64_t)b * p.m + i;
        if (p.op == 0) {
          if (p.relu) y = fmaxf(y, 0.0f);
          static_cast<float*>(p.out)[v * p.ld_out + col] = y;
        } else if (p.op == 1) {
          const float a = fabsf(y);
          if (a > best || (a == best && (int)col < besti)) {
            best = a;
            besti = (int)col;
            bestv = y;
          }
        } else if (p.op == 2) {
          float sn, cs;
          sincosf(y * p.inv_sigma, &sn, &cs);
          float* o = static_cast<float*>(p.out) + v * p.ld_out;
          o[col] = p.norm * cs;
          o[p.k + col] = p.norm * sn;
        } else {
          static_cast<float*>(p.out)[v * p.ld_out + col] = y < 0.0f ? -1.0f : 1.0f;
        }
      }
      __syncthreads();
    }
    if (p.op == 1) {  // signed argmax over the k rows (lsh.cpp:9-21): strict >, smallest index wins
      red_v[tid] = best;
      red_i[tid] = besti;
      red_y[tid] = bestv;
      __syncthreads();
      for (int o = kFT / 2; o > 0; o >>= 1) {
        if (tid < o) {
          const float a = red_v[tid + o];
          const int ai = red_i[tid + o];
          if (a > red_v[tid] || (a == red_v[tid] && ai < red_i[tid])) {
            red_v[tid] = a;
            red_i[tid] = ai;
            red_y[tid] = red_y[tid + o];
          }
        }
        __syncthreads();
      }
      if (tid == 0) {
        const int id = red_i[0] + (red_y[0] < 0.0f ? p.k : 0);
        static_cast<int32_t*>(p.out)[v * p.tables + tab] = id;
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------ dense baseline
// epilogues on Y rows: relu copy / signed argmax / gaussian or angular features
__global__ void __launch_bounds__(256) dense_epilogue_kernel(const float* __restrict__ Y, int64_t ld_y, int64_t batch,
                                                             int64_t k, int op, int relu, float inv_sigma, float norm,
                                                             void* out, int64_t ld_out, int tables, int tab) {
  __shared__ float rv[256], ry[256];
  __shared__ int ri[256];
  for (int64_t v = blockIdx.x; v < batch; v += gridDim.x) {
    const float* y = Y + v * ld_y;
    float best = -1.0f, bv = 0.0f;
    int bi = 0x7fffffff;
    for (int64_t c = threadIdx.x; c < k; c += 256) {
      const float t = y[c];
      if (op == 0) {
        static_cast<float*>(out)[v * ld_out + c] = relu ? fmaxf(t, 0.0f) : t;
      } else if (op == 1) {
        if (fabsf(t) > best) {
          best = fabsf(t);
          bi = (int)c;
          bv = t;
        }
      } else if (op == 2) {
        float sn, cs;
        sincosf(t * inv_sigma, &sn, &cs);
        static_cast<float*>(out)[v * ld_out + c] = norm * cs;
        static_cast<float*>(out)[v * ld_out + k + c] = norm * sn;
      } else {
        static_cast<float*>(out)[v * ld_out + c] = t < 0.0f ? -1.0f : 1.0f;
      }
    }
    if (op == 1) {
      rv[threadIdx.x] = best;
      ri[threadIdx.x] = bi;
      ry[threadIdx.x] = bv;
      __syncthreads();
      for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
          const float a = rv[threadIdx.x + o];
          const int ai = ri[threadIdx.x + o];
          if (a > rv[threadIdx.x] || (a == rv[threadIdx.x] && ai < ri[threadIdx.x])) {
            rv[threadIdx.x] = a;
            ri[threadIdx.x] = ai;
            ry[threadIdx.x] = ry[threadIdx.x + o];
          }
        }
        __syncthreads();
      }
      if (threadIdx.x == 0)
        static_cast<int32_t*>(out)[v * tables + tab] = ri[0] + (ry[0] < 0.0f ? (int)k : 0);
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------ host FFT (fp64)
using cd = std::complex<double>;

void fft_fp64(std::vector<cd>& a) {  // transforms.cpp:15-41 (forward), same bit reversal + butterflies
  const size_t n = a.size();
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    const double ang = -2.0 * M_PI / static_cast<double>(len);
    const cd wlen(std::cos(ang), std::sin(ang));
    for (size_t i = 0; i < n; i += len) {
      cd w(1.0, 0.0);
      for (size_t kk = 0; kk < len / 2; ++kk) {
        const cd u = a[i + kk], v = a[i + kk + len / 2] * w;
        a[i + kk] = u + v;
        a[i + kk + len / 2] = u - v;
        w *= wlen;
      }
    }
  }
}

size_t bitrev(size_t i, int bits) {
  size_t r = 0;
  for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
  return r;
}

template <class T>
cudaError_t upload(const std::vector<T>& h, T** d) {
  cudaError_t e = cudaMalloc(d, h.size() * sizeof(T));
  if (e == cudaSuccess) e = cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

}  // namespace

struct FamilyPlan {
  int variant = 0, device = 0, sms = 148;
  int64_t n = 0, m = 0, k = 0, tables = 0, blocks = 0;
  int N = 0, logN = 0;
  double scale = 1.0;
  float *d1 = nullptr, *d2 = nullptr, *dense = nullptr, *dense_lo = nullptr;  // dense: G = hi + lo (TF32 split)
  float* dense32 = nullptr;                                                      // dense: G in fp32
  double2 *spec = nullptr, *tw = nullptr, *skw = nullptr;
  ~FamilyPlan() {
    for (void* q : {(void*)d1, (void*)d2, (void*)dense, (void*)dense_lo, (void*)dense32, (void*)spec, (void*)tw,
                    (void*)skw})
      if (q) cudaFree(q);
  }
};

// round an fp32 value to the nearest TF32 value (10 explicit mantissa bits), as an fp32
__host__ __device__ inline float tf32_round(float v) {
#ifdef __CUDA_ARCH__
  uint32_t u = __float_as_uint(v);
#else
  uint32_t u;
  std::memcpy(&u, &v, 4);
#endif
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x0fffu + ((u >> 13) & 1u)) & 0xffffe000u;
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float r;
  std::memcpy(&r, &u, 4);
  return r;
#endif
}

bool family_variant(int v) { return v >= SPN_GCIRC_D2_HD1 && v <= SPN_GAUSSIAN_DENSE; }

// draw_tail + StructuredSpinner::build (spinner.cpp:92-151) for the family variants.
void family_realize(int variant, int64_t n, int64_t m, uint64_t spec_seed, double* d1, double* d2, double* tail,
                    double* trow, double* dense) {
  if (variant != SPN_GAUSSIAN_DENSE) {
    HostRng front(mix_seed(spec_seed, 1));
    for (int64_t i = 0; i < n; ++i) d1[i] = front.rademacher();
    for (int64_t i = 0; i < n; ++i) d2[i] = front.rademacher();
  }
  HostRng rng(mix_seed(spec_seed, 2));
  switch (variant) {
    case SPN_GCIRC_D2_HD1:
    case SPN_GSKEW_CIRC_D2_HD1:
      for (int64_t i = 0; i < n; ++i) tail[i] = rng.gaussian();
      break;
    case SPN_GTOEPLITZ_D2_HD1:
      for (int64_t i = 0; i < n; ++i) tail[i] = rng.gaussian();
      trow[0] = tail[0];
      for (int64_t i = 1; i < n; ++i) trow[i] = rng.gaussian();
      break;
    case SPN_GAUSSIAN_DENSE:
      for (int64_t i = 0; i < m * n; ++i) dense[i] = rng.gaussian();
      break;
  }
}

spn_status family_build(FamilyPlan** out, int variant, int64_t n, int64_t m, int64_t k, int64_t tables,
                        int64_t blocks, const std::vector<double>* d, const std::vector<double>& trow,
                        const std::vector<double>& dense, double scale, int device) {
  auto* f = new FamilyPlan();
  f->variant = variant;
  f->n = n;
  f->m = m;
  f->k = k;
  f->tables = tables;
  f->blocks = blocks;
  f->scale = scale;
  f->device = device;
  cudaDeviceGetAttribute(&f->sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaSuccess;
  const int64_t tb = tables * blocks;
  if (variant == SPN_GAUSSIAN_DENSE) {
    // G (fp32) = hi + lo with hi exactly representable in TF32 (3xTF32 GEMM, dense_gemm)
    std::vector<float> hi(dense.size()), lo(dense.size());
    for (size_t i = 0; i < dense.size(); ++i) {
      const float g = static_cast<float>(dense[i]);
      hi[i] = tf32_round(g);
      lo[i] = tf32_round(g - hi[i]);
    }
    e = upload(hi, &f->dense);
    if (e == cudaSuccess) e = upload(lo, &f->dense_lo);
    if (e == cudaSuccess) {
      for (size_t i = 0; i < dense.size(); ++i) hi[i] = static_cast<float>(dense[i]);
      e = upload(hi, &f->dense32);
    }
  } else {
    int lg = 0;
    while ((int64_t(1) << lg) < n) ++lg;
    const int N = variant == SPN_GTOEPLITZ_D2_HD1 ? int(2 * n) : int(n);
    f->N = N;
    f->logN = variant == SPN_GTOEPLITZ_D2_HD1 ? lg + 1 : lg;
    std::vector<float> a(d[0].begin(), d[0].end()), b(d[1].begin(), d[1].end());
    e = upload(a, &f->d1);
    if (e == cudaSuccess) e = upload(b, &f->d2);
    // spectra: conj(FFT(first row / embedded row / twiddled row)) (transforms.cpp:116-157), bit-reversed
    std::vector<double2> spec(static_cast<size_t>(tb * N));
    std::vector<cd> z(static_cast<size_t>(N));
    for (int64_t q = 0; q < tb && e == cudaSuccess; ++q) {
      const double* r = d[2].data() + q * n;
      std::fill(z.begin(), z.end(), cd(0.0, 0.0));
      if (variant == SPN_GCIRC_D2_HD1) {
        for (int64_t i = 0; i < n; ++i) z[i] = cd(r[i], 0.0);
      } else if (variant == SPN_GTOEPLITZ_D2_HD1) {
        // first_col = tail, first_row = trow: r_emb[k] = row[k], r_emb[N-k] = col[k]
        const double* row = trow.data() + q * n;
        for (int64_t i = 0; i < n; ++i) z[i] = cd(row[i], 0.0);
        for (int64_t i = 1; i < n; ++i) z[N - i] = cd(r[i], 0.0);
      } else {
        for (int64_t i = 0; i < n; ++i) {
          const double ang = M_PI * static_cast<double>(i) / static_cast<double>(n);
          z[i] = r[i] * cd(std::cos(ang), std::sin(ang));
        }
      }
      fft_fp64(z);
      for (int j = 0; j < N; ++j) {
        const cd s = std::conj(z[bitrev(static_cast<size_t>(j), f->logN)]);
        spec[static_cast<size_t>(q * N + j)] = make_double2(s.real(), s.imag());
      }
    }
    std::vector<double2> tw(static_cast<size_t>(N / 2 > 0 ? N / 2 : 1));
    for (int t = 0; t < N / 2; ++t) {
      const double ang = -2.0 * M_PI * t / N;
      tw[t] = make_double2(std::cos(ang), std::sin(ang));
    }
    std::vector<double2> skw(static_cast<size_t>(n));
    for (int64_t t = 0; t < n; ++t) {
      const double ang = M_PI * static_cast<double>(t) / static_cast<double>(n);
      skw[t] = make_double2(std::cos(ang), std::sin(ang));
    }
    if (e == cudaSuccess) e = upload(spec, &f->spec);
    if (e == cudaSuccess) e = upload(tw, &f->tw);
    if (e == cudaSuccess) e = upload(skw, &f->skw);
  }
  if (e != cudaSuccess) {
    delete f;
    return cuda_error(e, "family plan upload");
  }
  *out = f;
  return SPN_OK;
}

void family_destroy(FamilyPlan* f) { delete f; }

// One cuBLAS handle per (thread, device): handles are not safe to share across threads that set
// different streams; created on first use and kept for the thread's lifetime.
cublasHandle_t dense_handle(int device) {
  struct Handles {
    cublasHandle_t h[64] = {};
    ~Handles() {
      for (auto q : h)
        if (q) cublasDestroy(q);
    }
  };
  static thread_local Handles hs;
  if (device < 0 || device >= 64) return nullptr;
  if (!hs.h[device] && cublasCreate(&hs.h[device]) != CUBLAS_STATUS_SUCCESS) hs.h[device] = nullptr;
  return hs.h[device];
}

// x = hi + lo per element, hi exactly representable in TF32 (round to nearest on the 13 dropped bits)
__global__ void tf32_split_kernel(const float* __restrict__ x, int64_t ld_x, int64_t n_in, int64_t batch,
                                  float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t total = n_in * batch;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / n_in, j = i - b * n_in;
    const float v = x[b * ld_x + j];
    const float h = tf32_round(v);
    hi[i] = h;
    lo[i] = tf32_round(v - h);
  }
}

// Y = scale * X G^T as a 3xTF32 product on the tensor cores: X G^T ~ Xhi Ghi^T + Xlo Ghi^T + Xhi Glo^T
// (the dropped Xlo Glo^T term is ~2^-22 relative), each a cuBLAS TF32 GEMM accumulating in fp32 —
// fp32-class accuracy (the 1e-5 bar) at tensor-core rate.  Column-major view: Y^T (k x batch, ld) =
// G (n x k, lda = n)^T * X^T (n_in x batch); G's columns >= n_in meet x's zero padding.
//
// The Gaussian random-feature epilogue multiplies the projection's error by |z| / sigma (the angle), so
// for that op the GEMM runs as a plain fp32 cuBLAS SGEMM instead (fuzz case n = 636, d' = 1272: 3xTF32
// features 2.1e-5 relative L2 vs the 1e-5 bar; the split's ~2^-22 relative residual is 4x fp32's).
spn_status dense_gemm(const FamilyPlan* f, const float* x, int64_t ld_x, int64_t n_in, int64_t batch, int64_t goff,
                      float* Y, int64_t ld_y, cudaStream_t s, bool fp32_exact) {
  cublasHandle_t h = dense_handle(f->device);
  if (!h) return set_error(SPN_ECUDA, "dense baseline: cublasCreate failed");
  if (cublasSetStream(h, s) != CUBLAS_STATUS_SUCCESS) return set_error(SPN_ECUDA, "dense baseline: cublasSetStream");
  if (fp32_exact) {
    const float alpha = static_cast<float>(f->scale), beta = 0.0f;
    const cublasStatus_t st = cublasGemmEx(
        h, CUBLAS_OP_T, CUBLAS_OP_N, static_cast<int>(f->k), static_cast<int>(batch), static_cast<int>(n_in), &alpha,
        f->dense32 + goff, CUDA_R_32F, static_cast<int>(f->n), x, CUDA_R_32F, static_cast<int>(ld_x), &beta, Y,
        CUDA_R_32F, static_cast<int>(ld_y), CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    if (st != CUBLAS_STATUS_SUCCESS)
      return set_error(SPN_ECUDA, std::string("dense baseline: cublasGemmEx status ") + std::to_string(static_cast<int>(st)));
    return SPN_OK;
  }
  float* xs = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&xs), sizeof(float) * static_cast<size_t>(2 * n_in * batch), s);
  if (e != cudaSuccess) return cuda_error(e, "dense scratch");
  float* xhi = xs;
  float* xlo = xs + n_in * batch;
  const int64_t blocks = std::min<int64_t>((n_in * batch + 255) / 256, int64_t(f->sms) * 8);
  tf32_split_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(x, ld_x, n_in, batch, xhi, xlo);
  const float alpha = static_cast<float>(f->scale), zero = 0.0f, one = 1.0f;
  const float* ghi = f->dense + goff;
  const float* glo = f->dense_lo + goff;
  auto gemm = [&](const float* g, const float* xx, const float* beta) {
    return cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, static_cast<int>(f->k), static_cast<int>(batch),
                        static_cast<int>(n_in), &alpha, g, CUDA_R_32F, static_cast<int>(f->n), xx, CUDA_R_32F,
                        static_cast<int>(n_in), beta, Y, CUDA_R_32F, static_cast<int>(ld_y),
                        CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT);
  };
  cublasStatus_t st = gemm(ghi, xlo, &zero);  // small terms first
  if (st == CUBLAS_STATUS_SUCCESS) st = gemm(glo, xhi, &one);
  if (st == CUBLAS_STATUS_SUCCESS) st = gemm(ghi, xhi, &one);
  cudaFreeAsync(xs, s);
  if (st != CUBLAS_STATUS_SUCCESS)
    return set_error(SPN_ECUDA, std::string("dense baseline: cublasGemmEx status ") + std::to_string(static_cast<int>(st)));
  e = cudaGetLastError();
  return e == cudaSuccess ? SPN_OK : cuda_error(e, "dense baseline split");
}

spn_status family_run(const FamilyPlan* f, int op, const float* x, int64_t batch, int64_t ld_x, int64_t n_in,
                      void* out, int64_t ld_out, int relu, double sigma, cudaStream_t s) {
  if (batch == 0) return SPN_OK;
  const float inv_sigma = op == 2 ? static_cast<float>(1.0 / sigma) : 0.0f;
  const float norm = static_cast<float>(1.0 / std::sqrt(static_cast<double>(f->k)));
  if (f->variant == SPN_GAUSSIAN_DENSE) {
    float* Y = nullptr;
    const bool direct = op == 0 && !relu;
    if (!direct) {
      cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&Y), sizeof(float) * static_cast<size_t>(batch * f->k), s);
      if (e != cudaSuccess) return cuda_error(e, "dense scratch");
    }
    const int passes = op == 1 ? static_cast<int>(f->tables) : 1;
    for (int t = 0; t < passes; ++t) {
      float* dst = direct ? static_cast<float*>(out) : Y;
      const int64_t ld = direct ? ld_out : f->k;
      // Y = scale * X G^T: 3xTF32 GEMMs on the tensor cores (dense_gemm)
      if (spn_status st = dense_gemm(f, x, ld_x, n_in, batch, t * f->blocks * f->m * f->n, dst, ld, s, op == 2))
        return st;
      if (!direct) {
        const int64_t g = std::min<int64_t>(batch, int64_t(f->sms) * 8);
        dense_epilogue_kernel<<<static_cast<unsigned>(g), 256, 0, s>>>(Y, f->k, batch, f->k, op, relu, inv_sigma,
                                                                       norm, out, ld_out, static_cast<int>(f->tables),
                                                                       t);
      }
    }
    cudaError_t e = cudaGetLastError();
    if (Y) cudaFreeAsync(Y, s);
    return e == cudaSuccess ? SPN_OK : cuda_error(e, "dense baseline");
  }
  FamParams p{};
  p.x = x;
  p.ld_x = ld_x;
  p.n_in = n_in;
  p.batch = batch;
  p.n = static_cast<int>(f->n);
  p.N = f->N;
  p.logN = f->logN;
  p.m = static_cast<int>(f->m);
  p.k = static_cast<int>(f->k);
  p.blocks = static_cast<int>(f->blocks);
  p.tables = static_cast<int>(f->tables);
  p.kind = f->variant;
  p.d1 = f->d1;
  p.d2 = f->d2;
  p.spec = f->spec;
  p.tw = f->tw;
  p.skw = f->skw;
  p.scale = static_cast<float>(f->scale);
  p.op = op;
  p.inv_sigma = inv_sigma;
  p.norm = norm;
  p.relu = relu;
  p.out = out;
  p.ld_out = ld_out;
  const size_t smem = sizeof(double2) * static_cast<size_t>(f->N);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(family_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 136 * 1024);
    attr = true;
  }
  const int64_t items = batch * (op == 1 ? f->tables : 1);
  const int64_t grid = std::min<int64_t>(items, int64_t(f->sms) * 4);
  family_kernel<<<static_cast<unsigned>(grid), kFT, smem, s>>>(p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPN_OK : cuda_error(e, "circulant family");
}

}  // namespace spn

// ------------------------------------------------------- standalone circulant operators
// CirculantOperator / circulant_matvec / toeplitz_matvec / skew_circulant_matvec
// (transforms.hpp:15-56, transforms.cpp:64-220) on the device: the spectrum is built on the host
// exactly as the reference does (same FFT length choice, Toeplitz embedding and skew half-root
// weights, fp64), then one CTA per vector runs the correlation with the family kernel's FFT
// (complex fp64 in shared memory: FFT length <= 2^13).

namespace spn {

namespace {

struct CircParams {
  const float* x;
  int64_t ld_x, batch;
  float* y;
  int64_t ld_y;
  int n, N, kind, direct;  // kind: 0 circulant, 1 toeplitz, 2 skew-circulant
  const double2* spec;     // [N] conj(FFT(.)), bit-reversed
  const double2* tw;       // [N/2] e^{-2 pi i t / N}
  const double2* skw;      // [n] e^{i pi t / n} (skew, direct)
};

__global__ void __launch_bounds__(kFT) circulant_kernel(const CircParams p) {
  extern __shared__ double2 c[];  // [N]
  const int tid = threadIdx.x;
  const bool skew_direct = p.kind == 2 && p.direct;
  const bool wrap = (p.kind == 0 || p.kind == 2) && !p.direct;  // periodic / negacyclic extension
  for (int64_t v = blockIdx.x; v < p.batch; v += gridDim.x) {
    const float* xr = p.x + v * p.ld_x;
    // input layouts of CirculantOperator::apply (transforms.cpp:178-199)
    for (int i = tid; i < p.N; i += kFT) {
      double val = 0.0;
      if (i < p.n) {
        val = (double)xr[i];
      } else if (wrap && i - p.n < p.n - 1) {
        val = (p.kind == 2 ? -1.0 : 1.0) * (double)xr[i - p.n];
      }
      c[i] = skew_direct ? make_double2(val * p.skw[i].x, val * p.skw[i].y) : make_double2(val, 0.0);
    }
    __syncthreads();
    for (int len = p.N; len >= 2; len >>= 1) {  // forward DIF: natural -> bit-reversed
      const int half = len >> 1, stride = p.N / len;
      for (int q = tid; q < p.N / 2; q += kFT) {
        const int blk = q / half, kk = q - blk * half, i = blk * len + kk;
        const double2 u = c[i], w = c[i + half];
        c[i] = make_double2(u.x + w.x, u.y + w.y);
        c[i + half] = cmul(make_double2(u.x - w.x, u.y - w.y), p.tw[kk * stride]);
      }
      __syncthreads();
    }
    for (int i = tid; i < p.N; i += kFT) c[i] = cmul(c[i], p.spec[i]);
    __syncthreads();
    for (int len = 2; len <= p.N; len <<= 1) {  // inverse DIT: bit-reversed -> natural
      const int half = len >> 1, stride = p.N / len;
      for (int q = tid; q < p.N / 2; q += kFT) {
        const int blk = q / half, kk = q - blk * half, i = blk * len + kk;
        const double2 u = c[i], w = cmulc(c[i + half], p.tw[kk * stride]);
        c[i] = make_double2(u.x + w.x, u.y + w.y);
        c[i + half] = make_double2(u.x - w.x, u.y - w.y);
      }
      __syncthreads();
    }
    const double invN = 1.0 / (double)p.N;
    float* yr = p.y + v * p.ld_y;
    for (int i = tid; i < p.n; i += kFT) {
      const double2 z = c[i];
      const double yd = skew_direct ? (z.x * p.skw[i].x + z.y * p.skw[i].y) : z.x;  // real(z * conj(w^i))
      yr[i] = (float)(yd * invN);
    }
    __syncthreads();
  }
}

int64_t next_pow2(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

}  // namespace

struct CirculantPlan {
  int kind = 0, direct = 0, n = 0, N = 0, logN = 0, device = 0, sms = 148;
  double2 *spec = nullptr, *tw = nullptr, *skw = nullptr;
  ~CirculantPlan() {
    for (void* q : {(void*)spec, (void*)tw, (void*)skw})
      if (q) cudaFree(q);
  }
};

}  // namespace spn

struct spn_circulant {
  spn::CirculantPlan plan;
};

extern "C" {

spn_status spn_circulant_create(spn_circulant** out, int32_t kind, int64_t n, const double* first_row,
                                const double* first_col, int32_t device) { SPN_TRY
  using spn::set_error;
  if (!out) return set_error(SPN_EINVAL, "null output");
  *out = nullptr;
  if (kind < 0 || kind > 2) return set_error(SPN_EDOMAIN, "CirculantSpec: unknown kind");
  if (n < 1) return set_error(SPN_EDIM, "CirculantSpec: n must be >= 1");
  if (!first_row) return set_error(SPN_EINVAL, "null first_row");
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(first_row[i])) return set_error(SPN_EDOMAIN, "CirculantSpec.first_row: non-finite entry");
  if (kind == 1) {  // CirculantSpec::validate (transforms.cpp:98-110)
    if (!first_col) return set_error(SPN_EDIM, "CirculantSpec: toeplitz first_col/first_row length mismatch");
    for (int64_t i = 0; i < n; ++i)
      if (!std::isfinite(first_col[i])) return set_error(SPN_EDOMAIN, "CirculantSpec.first_col: non-finite entry");
    if (first_col[0] != first_row[0]) return set_error(SPN_EDOMAIN, "CirculantSpec: toeplitz corner entry mismatch");
  } else if (first_col) {
    return set_error(SPN_EDIM, "CirculantSpec: first_col only valid for toeplitz");
  }
  // CirculantOperator::CirculantOperator (transforms.cpp:112-170)
  const bool pow2 = (n & (n - 1)) == 0;
  int direct = 0;
  int64_t N = 0;
  if (kind == 1) {
    direct = 1;
    N = 2 * spn::next_pow2(n);
  } else {
    direct = pow2 ? 1 : 0;
    N = pow2 ? n : spn::next_pow2(2 * n);
  }
  if (N > 8192) return set_error(SPN_EUNSUPPORTED, "circulant operator: FFT length > 2^13 (fp64 FFT in smem)");
  using cd = std::complex<double>;
  std::vector<cd> z(static_cast<size_t>(N), cd(0.0, 0.0));
  std::vector<double2> skw(static_cast<size_t>(n));
  for (int64_t t = 0; t < n; ++t) {
    const double ang = M_PI * static_cast<double>(t) / static_cast<double>(n);
    skw[t] = make_double2(std::cos(ang), std::sin(ang));
  }
  if (kind == 1) {
    for (int64_t k = 0; k < n; ++k) z[k] = cd(first_row[k], 0.0);
    for (int64_t k = 1; k < n; ++k) z[N - k] = cd(first_col[k], 0.0);
  } else if (kind == 2 && direct) {
    for (int64_t k = 0; k < n; ++k) z[k] = first_row[k] * cd(skw[k].x, skw[k].y);
  } else {
    for (int64_t k = 0; k < n; ++k) z[k] = cd(first_row[k], 0.0);
  }
  spn::fft_fp64(z);
  int logN = 0;
  while ((int64_t(1) << logN) < N) ++logN;
  std::vector<double2> spec(static_cast<size_t>(N));
  for (int64_t j = 0; j < N; ++j) {
    const cd s = std::conj(z[spn::bitrev(static_cast<size_t>(j), logN)]);
    spec[static_cast<size_t>(j)] = make_double2(s.real(), s.imag());
  }
  std::vector<double2> tw(static_cast<size_t>(N / 2 > 0 ? N / 2 : 1));
  for (int64_t t = 0; t < N / 2; ++t) {
    const double ang = -2.0 * M_PI * static_cast<double>(t) / static_cast<double>(N);
    tw[t] = make_double2(std::cos(ang), std::sin(ang));
  }
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return spn::cuda_error(cudaGetLastError(), "cudaSetDevice");
  auto* op = new spn_circulant();
  spn::CirculantPlan& p = op->plan;
  p.kind = kind;
  p.direct = direct;
  p.n = static_cast<int>(n);
  p.N = static_cast<int>(N);
  p.logN = logN;
  p.device = device;
  cudaDeviceGetAttribute(&p.sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = spn::upload(spec, &p.spec);
  if (e == cudaSuccess) e = spn::upload(tw, &p.tw);
  if (e == cudaSuccess) e = spn::upload(skw, &p.skw);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    delete op;
    return spn::cuda_error(e, "circulant operator upload");
  }
  *out = op;
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_circulant_destroy(spn_circulant* op) { SPN_TRY
  delete op;
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_circulant_apply_f32(const spn_circulant* op, const float* x, int64_t batch, int64_t ld_x, float* y,
                                   int64_t ld_y, void* stream) { SPN_TRY
  using spn::set_error;
  if (!op) return set_error(SPN_EINVAL, "null operator");
  const spn::CirculantPlan& p = op->plan;
  if (batch < 0 || ld_x < p.n || ld_y < p.n)
    return set_error(SPN_EDIM, "CirculantOperator::apply: expected length " + std::to_string(p.n));
  if (batch == 0) return SPN_OK;
  if (!x || !y) return set_error(SPN_EINVAL, "null pointer");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(spn::circulant_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 136 * 1024);
    attr = true;
  }
  spn::CircParams cp{x, ld_x, batch, y, ld_y, p.n, p.N, p.kind, p.direct, p.spec, p.tw, p.skw};
  const int64_t grid = std::min<int64_t>(batch, int64_t(p.sms) * 4);
  spn::circulant_kernel<<<static_cast<unsigned>(grid), spn::kFT, sizeof(double2) * static_cast<size_t>(p.N),
                          static_cast<cudaStream_t>(stream)>>>(cp);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPN_OK : spn::cuda_error(e, "circulant operator");
  SPN_CATCH
}

spn_status spn_circulant_apply_f32_host(const spn_circulant* op, const float* x, int64_t batch, int64_t ld_x,
                                        float* y, int64_t ld_y) { SPN_TRY
  using spn::set_error;
  if (!op) return set_error(SPN_EINVAL, "null operator");
  const spn::CirculantPlan& p = op->plan;
  if (batch < 0 || ld_x < p.n || ld_y < p.n)
    return set_error(SPN_EDIM, "CirculantOperator::apply: expected length " + std::to_string(p.n));
  if (batch == 0) return SPN_OK;
  if (!x || !y) return set_error(SPN_EINVAL, "null pointer");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p.device);
  const size_t row = static_cast<size_t>(p.n) * 4;
  float* d = nullptr;
  cudaError_t e = cudaMalloc(&d, row * static_cast<size_t>(batch));
  if (e == cudaSuccess) e = cudaMemcpy2D(d, row, x, ld_x * 4, row, batch, cudaMemcpyHostToDevice);
  spn_status st = e == cudaSuccess ? spn_circulant_apply_f32(op, d, batch, p.n, d, p.n, nullptr)
                                   : spn::cuda_error(e, "circulant operator");
  if (st == SPN_OK) {
    e = cudaMemcpy2D(y, ld_y * 4, d, row, row, batch, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = spn::cuda_error(e, "circulant operator");
  }
  cudaFree(d);
  cudaSetDevice(prev);
  return st;
  SPN_CATCH
}

}  // extern "C"
