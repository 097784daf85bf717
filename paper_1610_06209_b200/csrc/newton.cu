// Sketched Newton for logistic regression on the device — the caller of
// SketchOperator in the reference (proj/src/newton_sketch.cpp:45-122,
// proj/include/spinners/newton_sketch.hpp:63-86).
//
// One Newton step = one pass over A (margins, loss, gradient, Hessian row scales
// sqrt(s(1-s)) — loss/gradient/hessian_sqrt of the reference fused), the spinner
// sketch of B = diag(h) A with h folded into D1 of the sketch's first pass (B is never
// materialised), the d x d normal matrix (S B)^T (S B) in fp64, a blocked fp64
// Cholesky with the reference's ridge retry, and two triangular solves.  All sums that
// the reference does in fp64 are fp64 here; every reduction has a fixed order
// (per-CTA partials + an ordered final sum), so results are run-to-run deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/spinners_b200.h"
#include "errors.hpp"
#include "host_params.hpp"
#include "internal.hpp"

namespace {

constexpr int kMaxD = 1024;
constexpr int kPassThreads = 256;  // 8 warps, one row per warp at a time
constexpr int kNB = 32;            // Cholesky panel width
constexpr int kST = 64;            // SYRK output tile (4 x 4 per thread)

__device__ __forceinline__ double log1p_exp(double t) {  // newton_sketch.cpp:10-15
  if (t > 35.0) return t;
  if (t < -35.0) return exp(t);
  return log1p(exp(t));
}

__device__ __forceinline__ double sigmoid(double t) {  // newton_sketch.cpp:17-24
  if (t >= 0.0) {
    const double e = exp(-t);
    return 1.0 / (1.0 + e);
  }
  const double e = exp(t);
  return e / (1.0 + e);
}

// Streaming loads that stay batched: ptxas otherwise places each F2F.F64.F32 right after
// its load, and the warp then waits out every load's latency in turn.  The loads are
// volatile asm (kept in order), and a second volatile "touch" of every loaded register
// pins all conversions after the last load has been issued.
__device__ __forceinline__ float ldg_stream(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void pin(float& v) { asm volatile("" : "+f"(v)); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------- pass over A
// A warp takes RPI = 8 rows per iteration (all loads issued before any math, 8 KB in
// flight per warp at d = 256); lane l holds columns l, l+32, ... (DCH chunks).  The
// per-row scalars run one row per lane (lane q < 8): with e = exp(-|m|) shared by
// sigmoid(m) and sigmoid(y m) (bit-identical to evaluating both, y = +-1),
//   loss += log1p_exp(-y m), w = (sigmoid(y m) - 1) y, h = sqrt(s (1 - s)), s = sigmoid(m),
// then g += w a (lane-parallel over columns).  Per-CTA partials [grid][d+1] (loss last).
#ifndef SPN_PASS_RPI
#define SPN_PASS_RPI 8
#endif
#ifndef SPN_PASS_MINB  // resident CTAs per SM the pass kernels are compiled for
#define SPN_PASS_MINB 2  // <= 128 registers: the 2 x SMs grid resident at once (at 177 registers one CTA/SM
                         // fit, so it ran as two rounds of 8 warps/SM): pass over A 67 -> 51 us at the c6 shape
#endif
constexpr int kRPI = SPN_PASS_RPI;

__device__ __forceinline__ double sigmoid_e(double t, double e) {  // e = exp(-|t|)
  return t >= 0.0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
}

template <int DCH>
struct PassCfg {  // rows per warp iteration: 8 KB of loads in flight, <= 64 data registers
  static constexpr int RPI = DCH <= 8 ? kRPI : 64 / DCH;
};

template <int DCH>
__global__ void __launch_bounds__(kPassThreads, SPN_PASS_MINB) logistic_pass_kernel(const float* __restrict__ a, int64_t ld,
                                                                     const float* __restrict__ labels,
                                                                     const double* __restrict__ x, int64_t n, int d,
                                                                     double* __restrict__ part,
                                                                     double* __restrict__ margins,
                                                                     float* __restrict__ h32,
                                                                     double* __restrict__ h64) {
  extern __shared__ double red[];  // d + 1
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t nw = (int64_t)gridDim.x * (kPassThreads / 32);
  double xr[DCH], g[DCH];
#pragma unroll
  for (int c = 0; c < DCH; ++c) {
    const int col = c * 32 + lane;
    xr[c] = col < d ? x[col] : 0.0;
    g[c] = 0.0;
  }
  constexpr int RPI = PassCfg<DCH>::RPI;
  double lsum = 0.0;
  for (int64_t r0 = ((int64_t)blockIdx.x * (kPassThreads / 32) + wid) * RPI; r0 < n; r0 += nw * RPI) {
    float av[RPI][DCH];
#pragma unroll
    for (int q = 0; q < RPI; ++q) {
      const float* row = a + (r0 + q) * ld;
#pragma unroll
      for (int c = 0; c < DCH; ++c) {
        const int col = c * 32 + lane;
        av[q][c] = (r0 + q < n && col < d) ? ldg_stream(row + col) : 0.0f;
      }
    }
#pragma unroll
    for (int q = 0; q < RPI; ++q)
#pragma unroll
      for (int c = 0; c < DCH; ++c) pin(av[q][c]);
    double mine = 0.0;  // lane q < RPI: margin of row r0 + q
#pragma unroll
    for (int q = 0; q < RPI; ++q) {
      double dot = 0.0;
#pragma unroll
      for (int c = 0; c < DCH; ++c) dot = fma((double)av[q][c], xr[c], dot);
      const double m = warp_sum(dot);
      if (lane == q) mine = m;
    }
    const int64_t r = r0 + lane;
    double w = 0.0;
    if (lane < RPI && r < n) {
      const double m = mine;
      const double e = exp(-fabs(m));
      if (labels) {
        const double y = (double)__ldg(labels + r);
        const double t = -y * m;
        lsum += log1p_exp(t);
        w = (sigmoid_e(y * m, e) - 1.0) * y;
      }
      const double sg = sigmoid_e(m, e);
      const double h = sqrt(sg * (1.0 - sg));
      if (margins) margins[r] = m;
      if (h32) h32[r] = (float)h;
      if (h64) h64[r] = h;
    }
    if (labels) {
#pragma unroll
      for (int q = 0; q < RPI; ++q) {
        const double wq = __shfl_sync(0xffffffffu, w, q);
#pragma unroll
        for (int c = 0; c < DCH; ++c) g[c] = fma(wq, (double)av[q][c], g[c]);
      }
    }
  }
  if (!part) return;
  lsum = warp_sum(lsum);
  // ordered block reduction: warp 0, then 1, ... into smem
  for (int i = threadIdx.x; i <= d; i += kPassThreads) red[i] = 0.0;
  __syncthreads();
  for (int w = 0; w < kPassThreads / 32; ++w) {
    if (wid == w) {
#pragma unroll
      for (int c = 0; c < DCH; ++c) {
        const int col = c * 32 + lane;
        if (col < d) red[col] += g[c];
      }
      if (lane == 0) red[d] += lsum;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i <= d; i += kPassThreads) part[(int64_t)blockIdx.x * (d + 1) + i] = red[i];
}

// out[j] = sum_b part[b][j]: one CTA per column, strided partial sums + a fixed tree.
__global__ void __launch_bounds__(256) reduce_parts_kernel(const double* __restrict__ part, int nparts, int width,
                                                           double* __restrict__ grad, double* __restrict__ loss,
                                                           int d) {
  __shared__ double sh[256];
  const int j = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nparts; b += 256) s += part[(int64_t)b * width + j];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (j < d) {
      if (grad) grad[j] = sh[0];
    } else if (loss) {
      *loss = sh[0];
    }
  }
}

__global__ void scale_rows_f32_kernel(const float* __restrict__ a, int64_t ld, const double* __restrict__ h,
                                      int64_t n, int d, float* __restrict__ out, int64_t ld_out) {
  const int64_t total = n * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / d;
    const int j = (int)(e - i * d);
    out[i * ld_out + j] = (float)((double)a[i * ld + j] * h[i]);
  }
}

// ------------------------------------------------------------- normal matrix
// part[s][i][j] = sum over rows r of slice s of (w_r x_ri)(w_r x_rj) for the lower
// 64 x 64 tiles (bi >= bj); 256 threads, 4 x 4 outputs each, rows staged as fp64.
__global__ void __launch_bounds__(256) syrk_partial_kernel(const float* __restrict__ X, int64_t ldx,
                                                           const double* __restrict__ w, int64_t rows, int d,
                                                           int64_t rows_per_split, double* __restrict__ part) {
  __shared__ double Xi[32][kST + 1];
  __shared__ double Xj[32][kST + 1];
  const int t = blockIdx.x;
  int bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
  while (bi * (bi + 1) / 2 > t) --bi;
  const int bj = t - bi * (bi + 1) / 2;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t r1 = min(rows, r0 + rows_per_split);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t rc = r0; rc < r1; rc += 32) {
    for (int e = threadIdx.x; e < 32 * kST; e += 256) {
      const int rr = e / kST, cc = e - rr * kST;
      const int64_t r = rc + rr;
      const int ci = bi * kST + cc, cj = bj * kST + cc;
      double wi = 0.0, wj = 0.0;
      if (r < r1) {
        const double ww = w ? w[r] : 1.0;
        if (ci < d) wi = (double)X[r * ldx + ci] * ww;
        if (cj < d) wj = (double)X[r * ldx + cj] * ww;
      }
      Xi[rr][cc] = wi;
      Xj[rr][cc] = wj;
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < 32; ++rr) {
      double u[4], v[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) u[a] = Xi[rr][ty * 4 + a];
#pragma unroll
      for (int b = 0; b < 4; ++b) v[b] = Xj[rr][tx * 4 + b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(u[a], v[b], acc[a][b]);
    }
    __syncthreads();
  }
  double* out = part + (int64_t)blockIdx.y * d * d;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = bi * kST + ty * 4 + a, j = bj * kST + tx * 4 + b;
      if (i < d && j < d) out[(int64_t)i * d + j] = acc[a][b];
    }
}

// normal[i][j] = normal[j][i] = sum_s part[s][i][j] for i >= j (fixed order).
__global__ void syrk_reduce_kernel(const double* __restrict__ part, int nsplit, int d, double* __restrict__ normal) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)d * d) return;
  const int i = (int)(e / d), j = (int)(e - (int64_t)i * d);
  if (j > i) return;
  double s = 0.0;
  for (int k = 0; k < nsplit; ++k) s += part[(int64_t)k * d * d + e];
  normal[e] = s;
  normal[(int64_t)j * d + i] = s;
}

// ------------------------------------------------------------- Cholesky (lower, in place)
// Panel j0: warp 0 factors the nb x nb diagonal block in registers (lane r = row r,
// right-looking with shuffles, so every element sees its subtractions in column order,
// like the unblocked LLT); every other thread meanwhile holds one sub-diagonal row and
// then solves L21 = A21 L11^{-T} against L11 in smem.  A non-positive pivot sets *flag
// (Eigen's LLT NumericalIssue).
constexpr int kPanelThreads = 256;

// Compact code on purpose: the factorisation is a chain of nb dependent pivots, and an
// unrolled version (shuffles, 32 x 32 registers) measured 80 us per panel in instruction
// fetch (one warp streams ~48 KB of SASS once per panel).  Here every step is one
// barrier-separated parallel update over the (r, j) pairs of the 32 x 32 block (four
// pairs per thread); the sub-diagonal rows (one per thread per round) are solved after.
__global__ void __launch_bounds__(kPanelThreads) chol_panel_kernel(double* __restrict__ A, int d, int j0,
                                                                   int* __restrict__ flag) {
  __shared__ double L11[kNB][kNB + 1];  // working block: columns > k still being updated
  __shared__ double Ls[kNB][kNB + 1];   // finished, scaled columns: Ls[c][r] = L[r][c]
  __shared__ double inv_s[kNB];         // 1 / L_kk
  __shared__ int bad;
  if (*flag) return;
  const int nb = min(kNB, d - j0);
  const int tid = threadIdx.x;
  const int rq = tid >> 5, j = tid & 31;  // (row rq + 8 q, column j) pairs of the diagonal block
  if (tid == 0) bad = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = rq + 8 * q;
    if (r < nb && j <= r) L11[r][j] = A[(int64_t)(j0 + r) * d + j0 + j];
  }
  __syncthreads();
  // Two barriers per pivot (the pivot chain is the panel's critical path: tools/microbench/
  // f64lat.cu): thread 0 publishes 1/sqrt(p) (rsqrt, 66 cycles dependent latency, instead of
  // sqrt + divide, 160); then in one step the j == k threads store the scaled column k into Ls
  // (not in place, so nobody overwrites what the others read) and the j > k threads apply the
  // rank-1 update with the same rounded scaled values.
  for (int k = 0; k < nb; ++k) {
    if (tid == 0) {
      const double p = L11[k][k];
      if (!(p > 0.0)) {
        bad = 1;
      } else {
        const double ik = rsqrt(p);
        inv_s[k] = ik;
        Ls[k][k] = p * ik;  // sqrt(p) to an ulp
      }
    }
    __syncthreads();
    if (bad) break;
    const double ik = inv_s[k];
    if (j == k) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = rq + 8 * q;
        if (r > k && r < nb) Ls[k][r] = L11[r][k] * ik;
      }
    } else if (j > k && j < nb) {
      const double ljk = L11[j][k] * ik;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = rq + 8 * q;
        if (r >= j && r < nb) L11[r][j] -= (L11[r][k] * ik) * ljk;
      }
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) *flag = 1;
    return;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = rq + 8 * q;
    if (r < nb && j <= r) A[(int64_t)(j0 + r) * d + j0 + j] = Ls[j][r];
  }
  // (the block is read through a volatile view: ptxas otherwise hoists all 528 entries into
  // registers and spills — 255 registers + 112 B of stack)
  for (int i = j0 + nb + tid; i < d; i += kPanelThreads) {
    double l[kNB];
#pragma unroll
    for (int k = 0; k < kNB; ++k) l[k] = k < nb ? A[(int64_t)i * d + j0 + k] : 0.0;
#pragma unroll
    for (int k = 0; k < kNB; ++k) {
      if (k < nb) {
        double sum = l[k];
#pragma unroll
        for (int m = 0; m < k; ++m) sum -= l[m] * reinterpret_cast<volatile double(*)[kNB + 1]>(Ls)[m][k];
        l[k] = sum * inv_s[k];
      }
    }
#pragma unroll
    for (int k = 0; k < kNB; ++k)
      if (k < nb) A[(int64_t)i * d + j0 + k] = l[k];
  }
}

// Trailing update A22 -= L21 L21^T on the lower 32 x 32 tiles below/right of panel j0.
__global__ void __launch_bounds__(256) chol_update_kernel(double* __restrict__ A, int d, int j0,
                                                          const int* __restrict__ flag) {
  __shared__ double Li[kNB][kNB + 1];
  __shared__ double Lj[kNB][kNB + 1];
  if (*flag) return;
  const int t = blockIdx.x;
  int bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
  while (bi * (bi + 1) / 2 > t) --bi;
  const int bj = t - bi * (bi + 1) / 2;
  const int base = j0 + kNB;
  const int i0 = base + bi * kNB, jj0 = base + bj * kNB;
  for (int e = threadIdx.x; e < kNB * kNB; e += 256) {
    const int r = e / kNB, k = e - r * kNB;
    Li[r][k] = (i0 + r < d) ? A[(int64_t)(i0 + r) * d + j0 + k] : 0.0;
    Lj[r][k] = (jj0 + r < d) ? A[(int64_t)(jj0 + r) * d + j0 + k] : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kNB * kNB; e += 256) {
    const int r = e / kNB, c = e - r * kNB;
    const int i = i0 + r, j = jj0 + c;
    if (i < d && j < d && j <= i) {
      double s = A[(int64_t)i * d + j];
#pragma unroll 8
      for (int k = 0; k < kNB; ++k) s -= Li[r][k] * Lj[c][k];
      A[(int64_t)i * d + j] = s;
    }
  }
}

// step = -(L L^T)^{-1} grad, blocked by 32: each 32 x 32 diagonal block is staged in smem
// and solved by warp 0 (a shuffle per row, compact loop), then all threads apply the block
// to the remaining entries (one barrier pair per block instead of per row).
__global__ void __launch_bounds__(256) chol_solve_kernel(const double* __restrict__ L, int d,
                                                         const double* __restrict__ grad, double* __restrict__ step,
                                                         const int* __restrict__ flag) {
  extern __shared__ double b[];  // [d] right-hand side, then [d] reciprocals of the diagonal
  double* inv = b + d;
  __shared__ double T[32][33];
  if (*flag) return;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < d; i += blockDim.x) {
    b[i] = -grad[i];
    inv[i] = 1.0 / L[(int64_t)i * d + i];  // off the sequential chains below
  }
  __syncthreads();
  // forward: L y = b
  for (int kb = 0; kb < d; kb += 32) {
    const int nb = min(32, d - kb);
    for (int e = tid; e < 32 * 32; e += blockDim.x) {
      const int rr = e >> 5, cc = e & 31;
      T[rr][cc] = (rr < nb && cc <= rr) ? L[(int64_t)(kb + rr) * d + kb + cc] : 0.0;
    }
    __syncthreads();
    if (tid < 32) {
      double y = lane < nb ? b[kb + lane] : 0.0;
      for (int k = 0; k < nb; ++k) {
        if (lane == k) y *= inv[kb + k];
        const double yk = __shfl_sync(0xffffffffu, y, k);
        if (lane > k) y -= T[lane][k] * yk;
      }
      if (lane < nb) b[kb + lane] = y;
    }
    __syncthreads();
    for (int i = kb + nb + tid; i < d; i += blockDim.x) {
      const double* li = L + (int64_t)i * d + kb;
      double lv[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) lv[c] = c < nb ? li[c] : 0.0;  // all 32 loads in flight
      double sum = b[i];
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c < nb) sum -= lv[c] * b[kb + c];
      b[i] = sum;
    }
    __syncthreads();
  }
  // backward: L^T x = y
  for (int ke = d; ke > 0; ke -= 32) {
    const int kb = max(0, ke - 32), nb = ke - kb;
    for (int e = tid; e < 32 * 32; e += blockDim.x) {
      const int rr = e >> 5, cc = e & 31;
      T[rr][cc] = (rr < nb && cc <= rr) ? L[(int64_t)(kb + rr) * d + kb + cc] : 0.0;
    }
    __syncthreads();
    if (tid < 32) {
      double xv = lane < nb ? b[kb + lane] : 0.0;
      for (int k = nb - 1; k >= 0; --k) {
        if (lane == k) xv *= inv[kb + k];
        const double xk = __shfl_sync(0xffffffffu, xv, k);
        if (lane < k) xv -= T[k][lane] * xk;
      }
      if (lane < nb) b[kb + lane] = xv;
    }
    __syncthreads();
    for (int i = tid; i < kb; i += blockDim.x) {
      double lv[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) lv[c] = c < nb ? L[(int64_t)(kb + c) * d + i] : 0.0;
      double sum = b[i];
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c < nb) sum -= lv[c] * b[kb + c];
      b[i] = sum;
    }
    __syncthreads();
  }
  for (int i = tid; i < d; i += blockDim.x) step[i] = b[i];
}

// normal_jj += 1e-10 * trace(normal)   (newton_sketch.cpp:114-115)
__global__ void ridge_kernel(double* __restrict__ normal, int d) {
  __shared__ double tr;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int j = 0; j < d; ++j) t += normal[(int64_t)j * d + j];
    tr = t;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < d; j += blockDim.x) normal[(int64_t)j * d + j] += 1e-10 * tr;
}

// ------------------------------------------------------------- line search
// losses[k] = sum_r log1p_exp(-y_r (a_r.x + s_k a_r.step)), s_k = s0 * 2^-k.  Rows are read
// 8 per warp iteration; lane (q, k) = row q, candidate k when count <= 4 (one transcendental
// per lane per 8 rows), otherwise lane k (and k + 32) for every row.
template <int DCH>
__global__ void __launch_bounds__(kPassThreads, SPN_PASS_MINB) line_kernel(const float* __restrict__ a, int64_t ld,
                                                            const float* __restrict__ labels,
                                                            const double* __restrict__ x,
                                                            const double* __restrict__ step, int64_t n, int d,
                                                            double s0, int count, double* __restrict__ part) {
  __shared__ double red[kPassThreads / 32][64];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t nw = (int64_t)gridDim.x * (kPassThreads / 32);
  double xr[DCH], pr[DCH];
#pragma unroll
  for (int c = 0; c < DCH; ++c) {
    const int col = c * 32 + lane;
    xr[c] = col < d ? x[col] : 0.0;
    pr[c] = col < d ? step[col] : 0.0;
  }
  const bool pairs = count <= 4;
  const int kA = pairs ? (lane & 3) : lane;
  const double sA = s0 * exp2(-(double)kA), sB = s0 * exp2(-(double)(lane + 32));
  double accA = 0.0, accB = 0.0;
  for (int64_t r0 = ((int64_t)blockIdx.x * (kPassThreads / 32) + wid) * kRPI; r0 < n; r0 += nw * kRPI) {
    double mq = 0.0, qq = 0.0;  // pairs mode: this lane's row (lane >> 2)
    double mm[kRPI], qv[kRPI];
    float av[kRPI][DCH];
#pragma unroll
    for (int q = 0; q < kRPI; ++q) {
      const float* row = a + (r0 + q) * ld;
#pragma unroll
      for (int c = 0; c < DCH; ++c) {
        const int col = c * 32 + lane;
        av[q][c] = (r0 + q < n && col < d) ? ldg_stream(row + col) : 0.0f;
      }
    }
#pragma unroll
    for (int q = 0; q < kRPI; ++q)
#pragma unroll
      for (int c = 0; c < DCH; ++c) pin(av[q][c]);
#pragma unroll
    for (int q = 0; q < kRPI; ++q) {
      double dm = 0.0, dq = 0.0;
#pragma unroll
      for (int c = 0; c < DCH; ++c) {
        const double v = (double)av[q][c];
        dm = fma(v, xr[c], dm);
        dq = fma(v, pr[c], dq);
      }
      mm[q] = warp_sum(dm);
      qv[q] = warp_sum(dq);
      if ((lane >> 2) == q) {
        mq = mm[q];
        qq = qv[q];
      }
    }
    if (pairs) {
      const int64_t r = r0 + (lane >> 2);
      if (kA < count && r < n) {
        const double y = (double)__ldg(labels + r);
        accA += log1p_exp(-y * (mq + sA * qq));
      }
    } else {
#pragma unroll
      for (int q = 0; q < kRPI; ++q) {
        if (r0 + q >= n) break;
        const double y = (double)__ldg(labels + r0 + q);
        if (lane < count) accA += log1p_exp(-y * (mm[q] + sA * qv[q]));
        if (lane + 32 < count) accB += log1p_exp(-y * (mm[q] + sB * qv[q]));
      }
    }
  }
  red[wid][lane] = accA;
  red[wid][lane + 32] = accB;
  __syncthreads();
  if (threadIdx.x < count) {
    const int k = threadIdx.x;
    double s = 0.0;
    for (int w = 0; w < kPassThreads / 32; ++w) {
      if (pairs) {
        for (int q = 0; q < kRPI; ++q) s += red[w][q * 4 + k];
      } else {
        s += red[w][k];
      }
    }
    part[(int64_t)blockIdx.x * count + k] = s;
  }
}

int sm_count(int dev) {
  int s = 0;
  if (cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || s < 1) s = 148;
  return s;
}

spn_status fail(spn_status s, const char* msg) { return spn::set_error(s, msg); }

#define NWT_CUDA(call)                                                 \
  do {                                                                 \
    cudaError_t e_ = (call);                                           \
    if (e_ != cudaSuccess) return spn::cuda_error(e_, #call);          \
  } while (0)

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

struct spn_newton {
  int64_t n = 0, d = 0, max_rows = 0;
  int device = 0, sms = 148, grid = 296, nsplit_max = 1;
  double* part = nullptr;     // [grid][d+1] pass partials (also line-search partials)
  double* margins = nullptr;  // [n]
  float* h32 = nullptr;       // [n] Hessian row scales (sketch D1 scaling)
  double* h64 = nullptr;      // [n] the same in fp64 (exact normal matrix, hessian_sqrt)
  float* sb = nullptr;        // [max_rows][d] sketched S B
  double* spart = nullptr;    // [nsplit_max][d][d]
  double* normal = nullptr;   // [d][d]
  double* fact = nullptr;     // [d][d] Cholesky factor (lower)
  double* grad = nullptr;     // [d]
  double* loss = nullptr;     // [1]
  int* flag = nullptr;        // device pivot-failure flag
  int* flag_h = nullptr;      // pinned
  // resident problem for the host-buffer entry points
  float* a = nullptr;         // [n][d]
  float* labels = nullptr;    // [n]
  double* hx = nullptr;       // [3][d] x, step, scratch (+ scalars)
  cudaStream_t s = nullptr;
};

namespace {

void newton_free(spn_newton* w) {
  for (void* p : {(void*)w->part, (void*)w->margins, (void*)w->h32, (void*)w->h64, (void*)w->sb, (void*)w->spart,
                  (void*)w->normal, (void*)w->fact, (void*)w->grad, (void*)w->loss, (void*)w->flag, (void*)w->a,
                  (void*)w->labels, (void*)w->hx})
    if (p) cudaFree(p);
  if (w->flag_h) cudaFreeHost(w->flag_h);
  if (w->s) cudaStreamDestroy(w->s);
}

template <int DCH>
cudaError_t launch_pass_t(const spn_newton* w, const float* a, int64_t ld, const float* labels, const double* x,
                          bool want_part, cudaStream_t s) {
  const size_t smem = sizeof(double) * (size_t)(w->d + 1);
  logistic_pass_kernel<DCH><<<w->grid, kPassThreads, smem, s>>>(a, ld, labels, x, w->n, (int)w->d,
                                                                 want_part ? w->part : nullptr, w->margins, w->h32,
                                                                 w->h64);
  return cudaGetLastError();
}

cudaError_t launch_pass(const spn_newton* w, const float* a, int64_t ld, const float* labels, const double* x,
                        bool want_part, cudaStream_t s) {
  const int dch = (int)((w->d + 31) / 32);
  if (dch <= 2) return launch_pass_t<2>(w, a, ld, labels, x, want_part, s);
  if (dch <= 4) return launch_pass_t<4>(w, a, ld, labels, x, want_part, s);
  if (dch <= 8) return launch_pass_t<8>(w, a, ld, labels, x, want_part, s);
  if (dch <= 16) return launch_pass_t<16>(w, a, ld, labels, x, want_part, s);
  return launch_pass_t<32>(w, a, ld, labels, x, want_part, s);
}

template <int DCH>
cudaError_t launch_line_t(const spn_newton* w, const float* a, int64_t ld, const float* labels, const double* x,
                          const double* step, double s0, int count, cudaStream_t s) {
  line_kernel<DCH><<<w->grid, kPassThreads, 0, s>>>(a, ld, labels, x, step, w->n, (int)w->d, s0, count, w->part);
  return cudaGetLastError();
}

cudaError_t launch_line(const spn_newton* w, const float* a, int64_t ld, const float* labels, const double* x,
                        const double* step, double s0, int count, cudaStream_t s) {
  const int dch = (int)((w->d + 31) / 32);
  if (dch <= 2) return launch_line_t<2>(w, a, ld, labels, x, step, s0, count, s);
  if (dch <= 4) return launch_line_t<4>(w, a, ld, labels, x, step, s0, count, s);
  if (dch <= 8) return launch_line_t<8>(w, a, ld, labels, x, step, s0, count, s);
  if (dch <= 16) return launch_line_t<16>(w, a, ld, labels, x, step, s0, count, s);
  return launch_line_t<32>(w, a, ld, labels, x, step, s0, count, s);
}

// normal = X^T diag(w)^2 X over `rows` rows (w may be NULL).
spn_status normal_matrix(spn_newton* w, const float* X, int64_t ldx, const double* wt, int64_t rows, cudaStream_t s) {
  const int d = (int)w->d;
  const int T = (d + kST - 1) / kST, tiles = T * (T + 1) / 2;
  int nsplit = std::max(1, std::min<int>(w->nsplit_max, (2 * w->sms + tiles - 1) / tiles));
  nsplit = (int)std::min<int64_t>(nsplit, std::max<int64_t>(1, (rows + 255) / 256));
  const int64_t per = ((rows + nsplit - 1) / nsplit + 31) / 32 * 32;
  nsplit = (int)std::max<int64_t>(1, (rows + per - 1) / per);
  syrk_partial_kernel<<<dim3(tiles, nsplit), 256, 0, s>>>(X, ldx, wt, rows, d, per, w->spart);
  NWT_CUDA(cudaGetLastError());
  const int64_t e = (int64_t)d * d;
  syrk_reduce_kernel<<<(unsigned)((e + 255) / 256), 256, 0, s>>>(w->spart, nsplit, d, w->normal);
  NWT_CUDA(cudaGetLastError());
  return SPN_OK;
}

// fact = chol(normal); step = -(fact fact^T)^{-1} grad; returns the pivot flag (syncs s).
spn_status factor_solve(spn_newton* w, const double* grad, double* step, cudaStream_t s, int* failed) {
  const int d = (int)w->d;
  NWT_CUDA(cudaMemcpyAsync(w->fact, w->normal, sizeof(double) * (size_t)d * d, cudaMemcpyDeviceToDevice, s));
  NWT_CUDA(cudaMemsetAsync(w->flag, 0, sizeof(int), s));
  for (int j0 = 0; j0 < d; j0 += kNB) {
    chol_panel_kernel<<<1, kPanelThreads, 0, s>>>(w->fact, d, j0, w->flag);
    NWT_CUDA(cudaGetLastError());
    const int rest = d - j0 - kNB;
    if (rest > 0) {
      const int T = (rest + kNB - 1) / kNB;
      chol_update_kernel<<<T * (T + 1) / 2, 256, 0, s>>>(w->fact, d, j0, w->flag);
      NWT_CUDA(cudaGetLastError());
    }
  }
  chol_solve_kernel<<<1, 256, 2 * sizeof(double) * (size_t)d, s>>>(w->fact, d, grad, step, w->flag);
  NWT_CUDA(cudaGetLastError());
  NWT_CUDA(cudaMemcpyAsync(w->flag_h, w->flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  NWT_CUDA(cudaStreamSynchronize(s));
  *failed = *w->flag_h;
  return SPN_OK;
}

}  // namespace

extern "C" {

spn_status spn_newton_create(spn_newton** out, int64_t n, int64_t d, int64_t max_sketch_rows, int device) { SPN_TRY
  if (!out) return fail(SPN_EINVAL, "null output");
  *out = nullptr;
  if (n < 1 || d < 1) return fail(SPN_EDIM, "LogisticProblem: empty data");
  if (d > kMaxD) return fail(SPN_EUNSUPPORTED, "sketched Newton: d > 1024");
  if (max_sketch_rows < 0) return fail(SPN_EDIM, "bad sketch row count");
  DevGuard g(device);
  auto* w = new spn_newton();
  w->n = n;
  w->d = d;
  w->max_rows = max_sketch_rows;
  w->device = device;
  w->sms = sm_count(device);
  w->grid = 2 * w->sms;
  const int T = (int)((d + kST - 1) / kST), tiles = T * (T + 1) / 2;
  w->nsplit_max = std::max(1, std::min<int>((2 * w->sms + tiles - 1) / tiles,
                                            (int)((int64_t(256) << 20) / (8 * d * d))));
  cudaError_t e = cudaSuccess;
  auto al = [&](void** p, size_t bytes) {
    if (e == cudaSuccess && bytes) e = cudaMalloc(p, bytes);
  };
  al((void**)&w->part, sizeof(double) * (size_t)w->grid * (size_t)std::max<int64_t>(d + 1, 64));
  al((void**)&w->margins, sizeof(double) * (size_t)n);
  al((void**)&w->h32, sizeof(float) * (size_t)n);
  al((void**)&w->h64, sizeof(double) * (size_t)n);
  al((void**)&w->sb, sizeof(float) * (size_t)(max_sketch_rows * d));
  al((void**)&w->spart, sizeof(double) * (size_t)w->nsplit_max * (size_t)(d * d));
  al((void**)&w->normal, sizeof(double) * (size_t)(d * d));
  al((void**)&w->fact, sizeof(double) * (size_t)(d * d));
  al((void**)&w->grad, sizeof(double) * (size_t)d);
  al((void**)&w->loss, sizeof(double));
  al((void**)&w->flag, sizeof(int));
  if (e == cudaSuccess) e = cudaMallocHost((void**)&w->flag_h, sizeof(int));
  if (e != cudaSuccess) {
    newton_free(w);
    delete w;
    return spn::cuda_error(e, "spn_newton_create");
  }
  *out = w;
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_newton_destroy(spn_newton* w) { SPN_TRY
  if (!w) return SPN_OK;
  DevGuard g(w->device);
  newton_free(w);
  delete w;
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_logistic_eval_f32(spn_newton* w, const float* a, int64_t ld_a, const float* labels,
                                 const double* x, double* loss, double* grad, void* stream) { SPN_TRY
  if (!w || !a || !labels || !x) return fail(SPN_EINVAL, "null pointer");
  if (ld_a < w->d) return fail(SPN_EINVAL, "bad leading dimension");
  DevGuard g(w->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  NWT_CUDA(launch_pass(w, a, ld_a, labels, x, true, s));
  const int width = (int)w->d + 1;
  reduce_parts_kernel<<<width, 256, 0, s>>>(w->part, w->grid, width, grad, loss, (int)w->d);
  NWT_CUDA(cudaGetLastError());
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_hessian_sqrt_f32(spn_newton* w, const float* a, int64_t ld_a, const double* x, float* out,
                                int64_t ld_out, void* stream) { SPN_TRY
  if (!w || !a || !x || !out) return fail(SPN_EINVAL, "null pointer");
  if (ld_a < w->d || ld_out < w->d) return fail(SPN_EINVAL, "bad leading dimension");
  DevGuard g(w->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  NWT_CUDA(launch_pass(w, a, ld_a, nullptr, x, false, s));
  const int64_t total = w->n * w->d;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, int64_t(w->sms) * 16);
  scale_rows_f32_kernel<<<(unsigned)blocks, 256, 0, s>>>(a, ld_a, w->h64, w->n, (int)w->d, out, ld_out);
  NWT_CUDA(cudaGetLastError());
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_sketched_step_f32(spn_newton* w, const spn_plan* sketch, int64_t rows, const float* a, int64_t ld_a,
                                 const float* labels, const double* x, double* step, double* grad, double* loss,
                                 void* stream) { SPN_TRY
  if (!w || !a || !labels || !x || !step) return fail(SPN_EINVAL, "null pointer");
  if (ld_a < w->d) return fail(SPN_EINVAL, "bad leading dimension");
  const int64_t m = sketch ? rows : w->n;
  if (m < w->d) return fail(SPN_EDIM, "sketched_step: sketch dimension below d");
  if (sketch && rows > w->max_rows) return fail(SPN_EDIM, "sketch rows exceed the workspace");
  DevGuard g(w->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // gradient, loss, Hessian row scales at x (newton_sketch.cpp:105,110)
  NWT_CUDA(launch_pass(w, a, ld_a, labels, x, true, s));
  const int width = (int)w->d + 1;
  reduce_parts_kernel<<<width, 256, 0, s>>>(w->part, w->grid, width, w->grad, w->loss, (int)w->d);
  NWT_CUDA(cudaGetLastError());
  if (grad) NWT_CUDA(cudaMemcpyAsync(grad, w->grad, sizeof(double) * (size_t)w->d, cudaMemcpyDeviceToDevice, s));
  if (loss) NWT_CUDA(cudaMemcpyAsync(loss, w->loss, sizeof(double), cudaMemcpyDeviceToDevice, s));
  // normal matrix (S B)^T (S B)   (:106,109)
  if (sketch) {
    if (spn::plan_device(sketch) != w->device) return fail(SPN_EINVAL, "sketch plan on another device");
    spn_status st = spn::plan_sketch_scaled(sketch, a, w->n, w->d, ld_a, rows, 1.0 / std::sqrt((double)rows),
                                            w->h32, w->sb, w->d, s);
    if (st) return st;
    if (spn_status st2 = normal_matrix(w, w->sb, w->d, nullptr, rows, s)) return st2;
  } else {
    if (spn_status st2 = normal_matrix(w, a, ld_a, w->h64, w->n, s)) return st2;
  }
  // LLT, ridge retry, solve   (:112-121)
  int failed = 0;
  if (spn_status st = factor_solve(w, w->grad, step, s, &failed)) return st;
  if (failed) {
    ridge_kernel<<<1, 256, 0, s>>>(w->normal, (int)w->d);
    NWT_CUDA(cudaGetLastError());
    if (spn_status st = factor_solve(w, w->grad, step, s, &failed)) return st;
    if (failed) return fail(SPN_ESINGULAR, "sketched_step: sketched Hessian is indefinite; sketch dimension too small");
  }
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_logistic_line_f32(spn_newton* w, const float* a, int64_t ld_a, const float* labels, const double* x,
                                 const double* step, double s0, int64_t count, double* losses, void* stream) { SPN_TRY
  if (!w || !a || !labels || !x || !step || !losses) return fail(SPN_EINVAL, "null pointer");
  if (count < 1 || count > 64) return fail(SPN_EINVAL, "line search: 1 <= count <= 64");
  if (ld_a < w->d) return fail(SPN_EINVAL, "bad leading dimension");
  DevGuard g(w->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  NWT_CUDA(launch_line(w, a, ld_a, labels, x, step, s0, (int)count, s));
  reduce_parts_kernel<<<(unsigned)count, 256, 0, s>>>(w->part, w->grid, (int)count, losses, nullptr, (int)count);
  NWT_CUDA(cudaGetLastError());
  return SPN_OK;
  SPN_CATCH
}

// ------------------------------------------------------------- host-buffer forms
spn_status spn_newton_set_problem(spn_newton* w, const float* features, int64_t ld, const float* labels) { SPN_TRY
  if (!w || !features || !labels) return fail(SPN_EINVAL, "null pointer");
  if (ld < w->d) return fail(SPN_EINVAL, "bad leading dimension");
  DevGuard g(w->device);
  if (!w->a) NWT_CUDA(cudaMalloc(&w->a, sizeof(float) * (size_t)(w->n * w->d)));
  if (!w->labels) NWT_CUDA(cudaMalloc(&w->labels, sizeof(float) * (size_t)w->n));
  if (!w->hx) NWT_CUDA(cudaMalloc(&w->hx, sizeof(double) * (size_t)(4 * w->d + 128)));
  if (!w->s) NWT_CUDA(cudaStreamCreateWithFlags(&w->s, cudaStreamNonBlocking));
  NWT_CUDA(cudaMemcpy2D(w->a, sizeof(float) * (size_t)w->d, features, sizeof(float) * (size_t)ld,
                        sizeof(float) * (size_t)w->d, (size_t)w->n, cudaMemcpyHostToDevice));
  NWT_CUDA(cudaMemcpy(w->labels, labels, sizeof(float) * (size_t)w->n, cudaMemcpyHostToDevice));
  return SPN_OK;
  SPN_CATCH
}

namespace {
spn_status need_problem(const spn_newton* w) {
  if (!w) return fail(SPN_EINVAL, "null workspace");
  if (!w->a) return fail(SPN_EINVAL, "spn_newton_set_problem was not called");
  return SPN_OK;
}
}  // namespace

spn_status spn_logistic_eval_host(spn_newton* w, const double* x, double* loss, double* grad) { SPN_TRY
  if (spn_status st = need_problem(w)) return st;
  if (!x) return fail(SPN_EINVAL, "null pointer");
  DevGuard g(w->device);
  const size_t db = sizeof(double) * (size_t)w->d;
  double* dx = w->hx;
  double* dg = w->hx + w->d;
  double* df = w->hx + 4 * w->d;
  NWT_CUDA(cudaMemcpyAsync(dx, x, db, cudaMemcpyHostToDevice, w->s));
  if (spn_status st = spn_logistic_eval_f32(w, w->a, w->d, w->labels, dx, df, dg, w->s)) return st;
  if (grad) NWT_CUDA(cudaMemcpyAsync(grad, dg, db, cudaMemcpyDeviceToHost, w->s));
  if (loss) NWT_CUDA(cudaMemcpyAsync(loss, df, sizeof(double), cudaMemcpyDeviceToHost, w->s));
  NWT_CUDA(cudaStreamSynchronize(w->s));
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_hessian_sqrt_host(spn_newton* w, const double* x, float* out, int64_t ld_out) { SPN_TRY
  if (spn_status st = need_problem(w)) return st;
  if (!x || !out) return fail(SPN_EINVAL, "null pointer");
  if (ld_out < w->d) return fail(SPN_EINVAL, "bad leading dimension");
  DevGuard g(w->device);
  float* dout = nullptr;
  NWT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dout), sizeof(float) * (size_t)(w->n * w->d), w->s));
  NWT_CUDA(cudaMemcpyAsync(w->hx, x, sizeof(double) * (size_t)w->d, cudaMemcpyHostToDevice, w->s));
  spn_status st = spn_hessian_sqrt_f32(w, w->a, w->d, w->hx, dout, w->d, w->s);
  cudaError_t e = cudaSuccess;
  if (!st)
    e = cudaMemcpy2DAsync(out, sizeof(float) * (size_t)ld_out, dout, sizeof(float) * (size_t)w->d,
                          sizeof(float) * (size_t)w->d, (size_t)w->n, cudaMemcpyDeviceToHost, w->s);
  cudaFreeAsync(dout, w->s);
  if (st) return st;
  if (e != cudaSuccess) return spn::cuda_error(e, "hessian_sqrt copy");
  NWT_CUDA(cudaStreamSynchronize(w->s));
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_sketched_step_host(spn_newton* w, const spn_plan* sketch, int64_t rows, const double* x, double* step,
                                  double* grad, double* loss) { SPN_TRY
  if (spn_status st = need_problem(w)) return st;
  if (!x || !step) return fail(SPN_EINVAL, "null pointer");
  DevGuard g(w->device);
  const size_t db = sizeof(double) * (size_t)w->d;
  double* dx = w->hx;
  double* ds = w->hx + w->d;
  double* dg = w->hx + 2 * w->d;
  double* df = w->hx + 4 * w->d;
  NWT_CUDA(cudaMemcpyAsync(dx, x, db, cudaMemcpyHostToDevice, w->s));
  if (spn_status st = spn_sketched_step_f32(w, sketch, rows, w->a, w->d, w->labels, dx, ds, dg, df, w->s)) return st;
  NWT_CUDA(cudaMemcpyAsync(step, ds, db, cudaMemcpyDeviceToHost, w->s));
  if (grad) NWT_CUDA(cudaMemcpyAsync(grad, dg, db, cudaMemcpyDeviceToHost, w->s));
  if (loss) NWT_CUDA(cudaMemcpyAsync(loss, df, sizeof(double), cudaMemcpyDeviceToHost, w->s));
  NWT_CUDA(cudaStreamSynchronize(w->s));
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_logistic_line_host(spn_newton* w, const double* x, const double* step, double s0, int64_t count,
                                  double* losses) { SPN_TRY
  if (spn_status st = need_problem(w)) return st;
  if (!x || !step || !losses) return fail(SPN_EINVAL, "null pointer");
  if (count < 1 || count > 64) return fail(SPN_EINVAL, "line search: 1 <= count <= 64");
  DevGuard g(w->device);
  const size_t db = sizeof(double) * (size_t)w->d;
  double* dx = w->hx;
  double* ds = w->hx + w->d;
  double* dl = w->hx + 4 * w->d + 1;
  NWT_CUDA(cudaMemcpyAsync(dx, x, db, cudaMemcpyHostToDevice, w->s));
  NWT_CUDA(cudaMemcpyAsync(ds, step, db, cudaMemcpyHostToDevice, w->s));
  if (spn_status st = spn_logistic_line_f32(w, w->a, w->d, w->labels, dx, ds, s0, count, dl, w->s)) return st;
  NWT_CUDA(cudaMemcpyAsync(losses, dl, sizeof(double) * (size_t)count, cudaMemcpyDeviceToHost, w->s));
  NWT_CUDA(cudaStreamSynchronize(w->s));
  return SPN_OK;
  SPN_CATCH
}

spn_status spn_ar1_problem(int64_t n, int64_t d, uint64_t seed, float* features, float* labels) { SPN_TRY
  if (n < 1 || d < 1) return fail(SPN_EDIM, "generate_ar1_problem: n, d must be >= 1");
  if (!features || !labels) return fail(SPN_EINVAL, "null pointer");
  // newton_sketch.cpp:185-204 with the reference generator (host_params.hpp HostRng)
  const double rho = 0.99, noise = std::sqrt(1.0 - rho * rho);
  spn::HostRng rng(spn::mix_seed(seed, 7));
  for (int64_t i = 0; i < n; ++i) {
    double prev = rng.gaussian();
    features[i * d] = (float)prev;
    for (int64_t j = 1; j < d; ++j) {
      prev = rho * prev + noise * rng.gaussian();
      features[i * d + j] = (float)prev;
    }
  }
  for (int64_t i = 0; i < n; ++i) labels[i] = (float)rng.rademacher();
  return SPN_OK;
  SPN_CATCH
}

}  // extern "C"
