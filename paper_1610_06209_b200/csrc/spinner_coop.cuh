// Vector-cooperative persistent kernel for 2^19..2^20-point spinners (config 5 shape).
//
// The 4-pass schedule (row-first: P1 row D1,Hc | P2 col Hr,D2,Hr | P3 row Hc,D3,Hc |
// P4 col Hr, scale/ReLU -> y) launched pass by pass is dominated by per-launch fill and
// drain: each pass has only a few tiles per SM.  Here ONE cooperative launch keeps every
// SM busy for the whole batch: CTAs form groups of GS that own one vector at a time
// (working set 4 MB per group, ~72 MB in flight in L2), run its four passes back to back
// and synchronise only with the GS-1 other CTAs of their group through a counter in
// global memory.  Different groups are at different passes, so there are no global
// bubbles.  Row segments: one warp each (layouts of spinner_vec.cuh, 2^LC floats);
// column tiles: 512 rows x 32 columns moved with one bulk copy per row (spinner_tma.cuh).
#pragma once

#include <cuda_runtime.h>

#include "spinner_tma.cuh"

namespace spn {

struct CoopParams {
  const float* x;
  int64_t ld_x, n_in, batch;
  float* y;          // also the workspace (in place): y row v holds the vector between passes
  int64_t ld_y, rows_valid;
  const float* d1row;  // D1, D3 in the row-pass layout-A format per segment
  const float* d3row;
  const float* d2tile; // D2 tile-permuted for the column pass
  float c;
  int relu;
  int gs;              // CTAs per group
  unsigned* counters;  // one per group (zeroed before launch)
};

// Group barrier: generation-counting, GS CTAs; release/acquire at gpu scope.
__device__ __forceinline__ void group_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

template <int LR, bool FIRST>
__device__ __forceinline__ void coop_row_segment(const float* src, int64_t valid, float* dst,
                                                 const float* dperm, float* sm, int t) {
  using C = VCfg<LR, 5>;
  float r[C::R];
  // coherent (L2) loads: the segment may have been written earlier in this launch
  if (valid >= C::N) {
#pragma unroll
    for (int j = 0; j < C::R; ++j) r[j] = __ldcg(src + j * 32 + t);
  } else {
#pragma unroll
    for (int j = 0; j < C::R; ++j) r[j] = (j * 32 + t < valid) ? __ldcg(src + j * 32 + t) : 0.0f;
  }
  if constexpr (FIRST) {
    xpose_B_to_A<C>(r, sm, t);
  } else {
    fwht_B_to_A<C>(r, sm, t);
  }
  const float4* f = reinterpret_cast<const float4*>(dperm);
#pragma unroll
  for (int q = 0; q < C::R / 4; ++q) {
    const float4 dv = __ldg(f + q * 32 + t);
    r[4 * q] *= dv.x;
    r[4 * q + 1] *= dv.y;
    r[4 * q + 2] *= dv.z;
    r[4 * q + 3] *= dv.w;
  }
  fwht_A_to_B<C>(r, sm, t);
#pragma unroll
  for (int j = 0; j < C::R; ++j) dst[j * 32 + t] = r[j];
}

// One pass of 2^9 x 32 column tiles over stripes cs = member, member + GS, ... of the
// [512][C] view of vector row `vec` (in place on y).  LAST: Hr then y epilogue; else
// Hr, D2, Hr.  phases: mbarrier parity bits carried across passes.
template <bool LAST>
__device__ __forceinline__ void coop_col_pass(const CoopParams& p, float* vec, int64_t C, int member,
                                              float* smem, uint64_t* bars, uint32_t& phases, int& cur) {
  using CC = SColCfg<9>;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nstripes = static_cast<int>(C / 32);
  const int s = threadIdx.x;  // my row
  // order the generic-proxy writes of the previous pass (other CTAs, acquired through the
  // group barrier) before this thread's bulk (async-proxy) reads
  asm volatile("fence.proxy.async;" ::: "memory");
  auto stage = [&](int cs, float* buf, uint64_t* bar) {
    mbar_arrive_tx(bar, 128);
    bulk_load(buf + s * 32, vec + (int64_t)s * C + (int64_t)cs * 32, 128, bar);
  };
  if (member < nstripes) stage(member, smem + cur * (CC::S * 32), &bars[cur]);
  for (int cs = member; cs < nstripes; cs += p.gs, cur ^= 1) {
    float* buf = smem + cur * (CC::S * 32);
    mbar_wait(&bars[cur], (phases >> cur) & 1u);
    phases ^= 1u << cur;
    const int nxt = cs + p.gs;
    if (nxt < nstripes) {
      bulk_wait_read();
      stage(nxt, smem + (cur ^ 1) * (CC::S * 32), &bars[cur ^ 1]);
    }
    float r[CC::R];
    constexpr bool START_B = !LAST;  // mid pass: H(B->A), D2@A, H(A->B); last: H(A->B)
#pragma unroll
    for (int j = 0; j < CC::R; ++j) r[j] = buf[scol_s<CC>(START_B, w, j) * 32 + lane];
    __syncthreads();
    constexpr int NPARTS = LAST ? 1 : 2;
#pragma unroll
    for (int part = 0; part < NPARTS; ++part) {
      const bool lay_b = START_B ^ ((part & 1) != 0);
      if (!LAST && part == 1) {
        const float4* Dp = reinterpret_cast<const float4*>(p.d2tile + (int64_t)cs * (CC::S * 32) + w * (CC::R * 32)) + lane;
#pragma unroll
        for (int q = 0; q < CC::R / 4; ++q) {
          const float4 dv = __ldg(Dp + q * 32);
          r[4 * q] *= dv.x;
          r[4 * q + 1] *= dv.y;
          r[4 * q + 2] *= dv.z;
          r[4 * q + 3] *= dv.w;
        }
      }
      reg_fwht<CC::R, 0, CC::LR>(r);
#pragma unroll
      for (int j = 0; j < CC::R; ++j) buf[scol_s<CC>(lay_b, w, j) * 32 + lane] = r[j];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < CC::R; ++j) r[j] = buf[scol_s<CC>(!lay_b, w, j) * 32 + lane];
      __syncthreads();
      if (!lay_b)
        reg_fwht<CC::R, CC::LR - CC::LW, CC::LR>(r);
      else
        reg_fwht<CC::R, 0, CC::LW>(r);
    }
    constexpr bool END_B = START_B ^ ((NPARTS & 1) != 0);
#pragma unroll
    for (int j = 0; j < CC::R; ++j) {
      float o = r[j];
      if constexpr (LAST) {
        o *= p.c;
        if (p.relu) o = fmaxf(o, 0.0f);
      }
      buf[scol_s<CC>(END_B, w, j) * 32 + lane] = o;
    }
    fence_proxy_async();
    __syncthreads();
    {
      const int64_t f = (int64_t)s * C + (int64_t)cs * 32;  // flat element of my row
      float* drow = vec + f;
      if (!LAST || f + 32 <= p.rows_valid) {
        bulk_store(drow, buf + s * 32, 128);
      } else {
        for (int q = 0; q < 32; ++q)
          if (f + q < p.rows_valid) drow[q] = buf[s * 32 + q];
      }
      bulk_commit();
    }
  }
  bulk_wait_all();  // this pass's stores are complete before the group barrier
  asm volatile("fence.proxy.async;" ::: "memory");
}

template <int LC>
__global__ void __launch_bounds__(512, 1) spinner_coop_kernel(const CoopParams p) {
  using RC = VCfg<LC - 5, 5>;
  extern __shared__ __align__(128) float smem[];  // 128 KB: 2 column-tile buffers / 16 warp buffers
  __shared__ __align__(8) uint64_t bars[2];
  const int64_t C = int64_t(1) << LC;              // row-segment length
  const int64_t n = C * 512;
  const int t = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ngroups = static_cast<int>(gridDim.x) / p.gs;
  const int group = static_cast<int>(blockIdx.x) / p.gs, member = static_cast<int>(blockIdx.x) % p.gs;
  if (group >= ngroups) return;  // leftover CTAs (grid not a multiple of gs)
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 512);
    mbar_init(&bars[1], 512);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phases = 0;
  int cur = 0;
  unsigned nbar = 0;
  unsigned* ctr = p.counters + group;
  float* wsm = smem + warp * RC::N;  // this warp's row-pass buffer
  for (int64_t v = group; v < p.batch; v += ngroups) {
    const float* xr = p.x + v * p.ld_x;
    float* yr = p.y + v * p.ld_y;
    // P1 row: x -> D1 -> Hc -> y (zero padded beyond n_in)
    for (int64_t seg = member + (int64_t)p.gs * warp; seg < n / C; seg += (int64_t)p.gs * 16) {
      const int64_t rem = p.n_in - seg * C;
      coop_row_segment<LC - 5, true>(xr + seg * C, rem < 0 ? 0 : rem, yr + seg * C, p.d1row + seg * C, wsm, t);
    }
    group_barrier(ctr, (++nbar) * p.gs);
    coop_col_pass<false>(p, yr, C, member, smem, bars, phases, cur);  // P2 col: Hr, D2, Hr
    group_barrier(ctr, (++nbar) * p.gs);
    for (int64_t seg = member + (int64_t)p.gs * warp; seg < n / C; seg += (int64_t)p.gs * 16)
      coop_row_segment<LC - 5, false>(yr + seg * C, C, yr + seg * C, p.d3row + seg * C, wsm, t);  // P3
    group_barrier(ctr, (++nbar) * p.gs);
    coop_col_pass<true>(p, yr, C, member, smem, bars, phases, cur);  // P4 col: Hr, epilogue
    // no barrier: the next vector's P1 touches a different row of y
    __syncthreads();  // smem buffers are reused by the next vector's row pass
  }
}

// Cooperative launch (all CTAs co-resident: the group barriers spin).  Returns
// cudaErrorNotSupported when the device cannot host one 512-thread CTA per SM.
template <int LC>
inline cudaError_t launch_coop(const CoopParams& p_in, int sms, cudaStream_t s) {
  auto kern = spinner_coop_kernel<LC>;
  constexpr size_t smem = size_t(128) << 10;
  static int occ = -1;
  if (occ < 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 512, smem);
    if (e != cudaSuccess) return e;
  }
  if (occ < 1) return cudaErrorNotSupported;
  CoopParams p = p_in;
  void* args[] = {&p};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(static_cast<unsigned>(sms)), dim3(512),
                                     args, smem, s);
}

}  // namespace spn
