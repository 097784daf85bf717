// HBM write-only bandwidth (the C2 epilogue is 91% writes): plain vs streaming (.cs) stores,
// 4-B per thread (like the kernel's coalesced STG.32) and 16-B per thread.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void w32(float* o, size_t n, int cs) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    if (cs) __stcs(o + i, 1.0f); else o[i] = 1.0f;
}
__global__ void w128(float4* o, size_t n4, int cs) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    if (cs) __stcs(o + i, make_float4(1, 1, 1, 1)); else o[i] = make_float4(1, 1, 1, 1);
}
int main() {
  size_t bytes = 2ull << 30, n = bytes / 4;
  float* o; cudaMalloc(&o, bytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cs = 0; cs < 2; ++cs) for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (v) w128<<<sms * 8, 256>>>((float4*)o, n / 4, cs); else w32<<<sms * 8, 256>>>(o, n, cs);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("write %s %s: %.1f GB/s\n", v ? "16B" : "4B", cs ? "st.cs" : "st", bytes / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
