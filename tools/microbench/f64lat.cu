// Latency of the fp64 pivot operations on the Cholesky chain: sqrt, 1/x, 1/sqrt via the
// rsqrt() library call and via an fp32 MUFU seed + two fp64 Newton steps.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsqrt_fast(double p) {
  double y = (double)__frsqrt_rn((float)p);
  const double h = 0.5 * p;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}
template <int K>
__global__ void chain(double* out, int iters, double x0) {
  double x = x0 + threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
    if (K == 0) x = sqrt(x) + 1.0;
    if (K == 1) x = 1.0 / x + 1.0;
    if (K == 2) x = rsqrt(x) + 1.0;
    if (K == 3) x = rsqrt_fast(x) + 1.0;
    if (K == 4) x = fma(x, 0.5, 1.0);
  }
  out[threadIdx.x] = x;
}
int main() {
  double* o; cudaMalloc(&o, 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"sqrt(x)+1", "1/x+1", "rsqrt(x)+1", "rsqrt_fast(x)+1", "fma (reference)"};
  void (*k[])(double*, int, double) = {chain<0>, chain<1>, chain<2>, chain<3>, chain<4>};
  const int iters = 1 << 14;
  for (int i = 0; i < 5; ++i) {
    k[i]<<<1, 32>>>(o, 16, 2.0); cudaDeviceSynchronize();
    cudaEventRecord(a); k[i]<<<1, 32>>>(o, iters, 2.0); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-18s %.1f ns = %.0f cycles at 1.965 GHz per dependent step\n", names[i], ms * 1e6 / iters,
           ms * 1e6 / iters * 1.965);
  }
}
