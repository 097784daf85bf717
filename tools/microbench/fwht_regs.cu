// Register-butterfly throughput of the spinner kernel's inner code (reg_fwht from
// spinner_vec.cuh, packed FADD2 + scalar in-pair stage), per register count R and
// resident warps per SM — the pure-FP32 ceiling of the n = 16384 hash kernel (c3).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1610_06209_b200/csrc -o fwht_regs fwht_regs.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "spinner_vec.cuh"

template <int LOG_R, int MINB, int SIGNS>
__global__ void __launch_bounds__(128, MINB) k_fwht(float* out, const unsigned* masks, int iters) {
  constexpr int R = 1 << LOG_R;
  float r[R];
#pragma unroll
  for (int j = 0; j < R; ++j) r[j] = threadIdx.x * 0.001f + j;
  unsigned w[R / 32 > 0 ? R / 32 : 1];  // R >= 64 here
#pragma unroll
  for (int q = 0; q < (R / 32 > 0 ? R / 32 : 1); ++q) w[q] = masks[q * 128 + threadIdx.x];
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    if constexpr (SIGNS == 1) {  // SHF + LOP3 per element
#pragma unroll
      for (int j = 0; j < R; ++j)
        r[j] = __uint_as_float(__float_as_uint(r[j]) ^ (__funnelshift_l(w[j / 32], w[j / 32], 31 - j % 32) & 0x80000000u));
    } else if constexpr (SIGNS == 2) {  // LOP3 only (timing probe, not a sign diagonal)
#pragma unroll
      for (int j = 0; j < R; ++j) r[j] = __uint_as_float(__float_as_uint(r[j]) ^ (w[j / 32] & 0x80000000u));
      w[0] = (w[0] << 1) | (w[0] >> 31);
    } else if constexpr (SIGNS == 4) {  // predicated negation (ptxas: R2P + FSEL per element)
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (w[j / 32] & (1u << (j % 32))) r[j] = -r[j];
    } else if constexpr (SIGNS == 5) {  // predicated XOR (ptxas: R2P + @P LOP3 per element; the kernel's form)
#pragma unroll
      for (int j = 0; j < R; ++j) spn::flip_if(r[j], w[j / 32], j % 32);
    } else if constexpr (SIGNS == 3) {  // SHF only into a sink (timing probe)
#pragma unroll
      for (int j = 0; j < R; ++j) w[0] ^= __funnelshift_l(w[j / 32 ^ 1 & (R / 32 - 1)], w[j / 32], j % 32);
    }
    spn::reg_fwht<R, 0, LOG_R>(r);
#pragma unroll
    for (int j = 0; j < R; ++j) r[j] *= 0.0883883f;  // keep values bounded (one FMUL per element)
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < R; ++j) s += r[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + __uint_as_float(w[0] & 1);
}

template <int LOG_R, int MINB, int SIGNS>
void run(float* out, const unsigned* m, int sms) {
  constexpr int R = 1 << LOG_R;
  const int iters = 2000;
  const int grid = sms * MINB;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_fwht<LOG_R, MINB, SIGNS><<<grid, 128>>>(out, m, 10);
  cudaEventRecord(a);
  k_fwht<LOG_R, MINB, SIGNS><<<grid, 128>>>(out, m, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double adds = (double)grid * 128 * iters * R * LOG_R;
  const double per_clk_sm = adds / (ms * 1e-3) / (clk * 1e3) / sms;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_fwht<LOG_R, MINB, SIGNS>);
  printf("R=%3d ctas/SM=%d (%2d warps) signs=%d regs=%3d: %.1f adds/clk/SM (at max clock %d MHz) + %d FMUL/elt\n", R, MINB,
         MINB * 4, SIGNS, fa.numRegs, per_clk_sm, clk / 1000, 1);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  unsigned* m;
  cudaMalloc(&out, sizeof(float) * sms * 16 * 128);
  cudaMalloc(&m, 4096 * 4);
  cudaMemset(m, 0x5a, 4096 * 4);
  run<7, 3, 0>(out, m, sms);
  run<7, 3, 1>(out, m, sms);
  run<7, 3, 2>(out, m, sms);
  run<7, 3, 3>(out, m, sms);
  run<7, 3, 4>(out, m, sms);
  run<7, 3, 5>(out, m, sms);
  run<6, 4, 0>(out, m, sms);
  run<6, 4, 1>(out, m, sms);
  run<6, 4, 4>(out, m, sms);
  run<6, 4, 5>(out, m, sms);
  run<5, 8, 1>(out, m, sms);
  run<5, 8, 4>(out, m, sms);
  run<5, 8, 5>(out, m, sms);
  return 0;
}
