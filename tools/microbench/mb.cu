// Microbenchmarks that decide the spinner kernel design on sm_100a:
//   FADD vs packed FADD2 butterfly throughput, smem transpose throughput,
//   shuffle throughput, L2-resident read / read-modify-write bandwidth, HBM copy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb mb.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ unsigned long long pack2(float a, float b) {
  return (unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(b) << 32);
}
__device__ __forceinline__ void unpack2(unsigned long long v, float& a, float& b) {
  a = __uint_as_float((unsigned)v); b = __uint_as_float((unsigned)(v >> 32));
}

// 32-register butterfly network (5 stages) repeated `iters` times. 32*5 = 160 adds per pass.
__global__ void k_fadd(float* out, int iters) {
  float r[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = threadIdx.x * 0.001f + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int b = 0; b < 5; ++b) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j & (1 << b)) continue;
        float u = r[j], v = r[j | (1 << b)];
        r[j] = u + v; r[j | (1 << b)] = u - v;
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) s += r[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Same network with registers packed as 16 f32x2 pairs (pair = bits {0} of j); stages b>=1 use FADD2.
__global__ void k_fadd2(float* out, int iters) {
  unsigned long long p[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) p[q] = pack2(threadIdx.x * 0.001f + 2 * q, threadIdx.x * 0.001f + 2 * q + 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int b = 1; b < 5; ++b) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        if (q & (1 << (b - 1))) continue;
        unsigned long long u = p[q], v = p[q | (1 << (b - 1))], s, d;
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s) : "l"(u), "l"(v));
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(u), "l"(v));
        p[q] = s; p[q | (1 << (b - 1))] = d;
      }
    }
    // stage b=0 (within pair) scalar
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      float a, c; unpack2(p[q], a, c);
      p[q] = pack2(a + c, a - c);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 16; ++q) { float a, c; unpack2(p[q], a, c); s += a + c; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Warp-private 32x32 transpose through smem (XOR swizzle), repeated. 2048 accesses per pass per warp.
__global__ void k_smem(float* out, int iters) {
  extern __shared__ float sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* t = sm + w * 1024;
  float r[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = lane + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 32; ++j) t[lane * 32 + (j ^ lane)] = r[j];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = t[j * 32 + (lane ^ j)] + 1.0f;
    __syncwarp();
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) s += r[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Same transpose with 128-bit accesses (swizzle on 16B chunks).
__global__ void k_smem128(float* out, int iters) {
  extern __shared__ float sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4* t = reinterpret_cast<float4*>(sm + w * 1024);
  float4 r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = make_float4(lane, j, 1, 2);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) t[lane * 8 + (j ^ (lane & 7))] = r[j];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j) { float4 v = t[((j * 4 + (lane >> 3)) ) * 8 + ((lane & 7) ^ ((j * 4 + (lane >> 3)) & 7))]; r[j].x = v.x + 1.f; r[j].y = v.y; r[j].z = v.z; r[j].w = v.w; }
    __syncwarp();
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += r[j].x + r[j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_shfl(float* out, int iters) {
  float r[32];
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = lane + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = __shfl_xor_sync(0xffffffffu, r[j], (j & 31) | 1);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) s += r[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_read(const float4* __restrict__ a, size_t n4, int reps, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = a[i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

__global__ void k_rmw(float4* a, size_t n4, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = a[i];
      v.x += 1.f; a[i] = v;
    }
}

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("SMs %d, max clock %d kHz\n", sms, clk);
  float* out; CK(cudaMalloc(&out, 1 << 26));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const int threads = 256, blocks = sms * 8;
  auto timeit = [&](auto launch) { launch(); cudaDeviceSynchronize(); cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); return ms; };
  {
    int iters = 2000;
    float t = timeit([&] { k_fadd<<<blocks, threads>>>(out, iters); });
    double adds = (double)blocks * threads * iters * 160;
    printf("FADD butterfly: %.3f ms, %.2f Tadd/s, %.1f add/clk/SM @max\n", t, adds / t / 1e9, adds / (t * 1e-3) / sms / (clk * 1e3));
    t = timeit([&] { k_fadd2<<<blocks, threads>>>(out, iters); });
    printf("FADD2 butterfly: %.3f ms, %.2f Tadd/s, %.1f add/clk/SM @max\n", t, adds / t / 1e9, adds / (t * 1e-3) / sms / (clk * 1e3));
    for (int occ : {4, 8}) {
      CK(cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, threads / 32 * 4096));
      t = timeit([&] { k_smem<<<sms * occ, threads, threads / 32 * 4096>>>(out, iters / 4); });
      double acc = (double)sms * occ * threads * (iters / 4) * 64;
      printf("smem32 transpose occ%d: %.3f ms, %.1f B/clk/SM\n", occ, t, acc * 4 / (t * 1e-3) / sms / (clk * 1e3));
      CK(cudaFuncSetAttribute(k_smem128, cudaFuncAttributeMaxDynamicSharedMemorySize, threads / 32 * 4096));
      t = timeit([&] { k_smem128<<<sms * occ, threads, threads / 32 * 4096>>>(out, iters / 4); });
      printf("smem128 transpose occ%d: %.3f ms, %.1f B/clk/SM\n", occ, t, acc * 4 / (t * 1e-3) / sms / (clk * 1e3));
    }
    t = timeit([&] { k_shfl<<<blocks, threads>>>(out, iters / 4); });
    double sh = (double)blocks * threads * (iters / 4) * 32;
    printf("SHFL: %.3f ms, %.1f lane-shfl/clk/SM\n", t, sh / (t * 1e-3) / sms / (clk * 1e3));
  }
  for (size_t mb : {16, 32, 64, 96}) {
    size_t bytes = mb << 20, n4 = bytes / 16;
    float4* a; CK(cudaMalloc(&a, bytes)); cudaMemset(a, 0, bytes);
    int reps = 20;
    float t = timeit([&] { k_read<<<sms * 4, 512>>>(a, n4, reps, out); });
    printf("L2 read %zu MB: %.1f GB/s\n", mb, (double)bytes * reps / (t * 1e-3) / 1e9);
    t = timeit([&] { k_rmw<<<sms * 4, 512>>>(a, n4, reps); });
    printf("L2 rmw  %zu MB: %.1f GB/s (r+w)\n", mb, 2.0 * bytes * reps / (t * 1e-3) / 1e9);
    cudaFree(a);
  }
  {
    size_t bytes = 2ull << 30, n4 = bytes / 16;
    float4 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
    cudaMemset(a, 0, bytes);
    float t = timeit([&] { k_copy<<<sms * 4, 512>>>(a, b, n4); });
    printf("HBM copy 2 GiB: %.1f GB/s (r+w)\n", 2.0 * bytes / (t * 1e-3) / 1e9);
    t = timeit([&] { k_read<<<sms * 4, 512>>>(a, n4, 1, out); });
    printf("HBM read 2 GiB: %.1f GB/s\n", (double)bytes / (t * 1e-3) / 1e9);
  }
  return 0;
}
