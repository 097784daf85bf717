#include <cstdio>
#include <cuda_runtime.h>
__global__ void thr(double* out, int iters) {  // 8 independent chains per thread
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 0.999999, c = 1e-7;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void lat(double* out, int iters) {  // one dependent chain
  double a = threadIdx.x * 1e-3; const double b = 0.999999, c = 1e-7;
  for (int it = 0; it < iters; ++it) a = fma(a, b, c);
  out[threadIdx.x] = a;
}
int main() {
  double* o; cudaMalloc(&o, 1 << 24);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 1 << 14;
  thr<<<148 * 4, 512>>>(o, 16); cudaDeviceSynchronize();
  cudaEventRecord(e0); thr<<<148 * 4, 512>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double dfma = 148.0 * 4 * 512 * 8 * iters;
  printf("DFMA throughput: %.1f TFLOP/s  (%.1f DFMA/clk/SM at 1.9 GHz)\n", 2 * dfma / ms / 1e9, dfma / (ms * 1e-3) / 148 / 1.9e9);
  lat<<<1, 32>>>(o, 16); cudaDeviceSynchronize();
  cudaEventRecord(e0); lat<<<1, 32>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("DFMA dependent latency: %.1f ns = %.1f cycles at 1.9 GHz\n", ms * 1e6 / iters, ms * 1e6 / iters * 1.9);
  // single CTA 512 threads throughput
  cudaEventRecord(e0); thr<<<1, 512>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("1 CTA x 512: %.1f DFMA/clk\n", 512.0 * 8 * iters / (ms * 1e-3) / 1.9e9);
}
