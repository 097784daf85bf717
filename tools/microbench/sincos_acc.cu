// Accuracy of the SFU sin/cos (MUFU via __sinf/__cosf) on UNREDUCED arguments vs fp64,
// to decide whether the RFF epilogue needs an explicit range reduction.
#include <cstdio>
#include <cmath>
__global__ void k(const float* t, float* s, float* c, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { s[i] = __sinf(t[i]); c[i] = __cosf(t[i]); }
}
int main() {
  const int n = 1 << 24;
  float *t, *s, *c;
  cudaMallocManaged(&t, n * 4); cudaMallocManaged(&s, n * 4); cudaMallocManaged(&c, n * 4);
  for (double lim : {3.1415926, 10.0, 20.0, 30.0, 50.0, 100.0}) {
    for (int i = 0; i < n; ++i) t[i] = (float)(-lim + 2 * lim * (i + 0.5) / n);
    k<<<(n + 255) / 256, 256>>>(t, s, c, n);
    cudaDeviceSynchronize();
    double es = 0, ec = 0;
    for (int i = 0; i < n; ++i) {
      es = fmax(es, fabs(s[i] - sin((double)t[i])));
      ec = fmax(ec, fabs(c[i] - cos((double)t[i])));
    }
    printf("|t| <= %6.1f : max abs err sin %.3e cos %.3e\n", lim, es, ec);
  }
  return 0;
}
