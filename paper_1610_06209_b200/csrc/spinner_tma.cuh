// Column pass with bulk-copy (TMA, cp.async.bulk) row transfers.
//
// A tile is 2^LS rows x 32 floats; every row is one contiguous 128-B segment in
// global memory, and LS >= 5 gives exactly one row per thread.  So each thread moves
// its row with ONE bulk copy in (completing on an mbarrier) and ONE bulk copy out,
// instead of 32 element loads/stores with per-element address arithmetic — the
// dominant instruction cost of the element-wise pass kernels.  Two tile buffers
// double-buffer the loads against the FWHT work; the epilogue goes registers ->
// smem -> bulk store (gather epilogue: one rowmap lookup per row).
// Requirements (checked by the host): 16-B aligned base pointers and leading
// dimensions, full 32-column stripes, whole rows valid or invalid.
#pragma once

#include <cuda_runtime.h>

#include "spinner_pass.cuh"

namespace spn {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Thread s issues row s of tile ti into buf (or zero-fills it when the row lies past src_valid).
template <class C>
__device__ __forceinline__ void tma_stage_row(const ColParams& p, const TileIdx& ti, float* buf, uint64_t* bar) {
  const int s = threadIdx.x;
  const int64_t f = (ti.e0 + ((int64_t)s << p.s0)) * p.src_ld + (int64_t)ti.cs * 32;
  float* dst = buf + s * 32;
  if (f + 32 <= p.src_valid) {
    mbar_arrive_tx(bar, 128);
    bulk_load(dst, p.src + (int64_t)ti.v * p.src_vstride + f, 128, bar);
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) reinterpret_cast<float4*>(dst)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    mbar_arrive(bar);  // release: the zeros are visible after the wait
  }
}

// Buffer count: three tiles when they fit one SM (LS <= 9: 3 x 64 KB), so two tiles are
// in flight while one is computed (the passes are bound by bytes in flight per SM).
template <int LS>
struct TmaCfg {
  static constexpr size_t TILE = sizeof(float) * (size_t(1) << LS) * 32;
  static constexpr int NBUF = 3;
  static constexpr size_t SMEM = TILE * NBUF;
  static constexpr int BY_SMEM = (int)((227u * 1024u) / SMEM);
  static constexpr int BY_REGS = 512 / SColCfg<LS>::THREADS;
  static constexpr int M0 = BY_SMEM < BY_REGS ? BY_SMEM : BY_REGS;
  static constexpr int MIN_CTAS = M0 < 1 ? 1 : M0;
};

template <int LS, int NPARTS, int DMASK, bool START_B, int DMODE, int EPI>
__global__ void __launch_bounds__(SColCfg<LS>::THREADS, TmaCfg<LS>::MIN_CTAS) colpass_tma_kernel(const ColParams p) {
  using C = SColCfg<LS>;
  constexpr int NB = TmaCfg<LS>::NBUF;  // tiles in flight: NB-1 loads ahead of the compute
  static_assert(C::THREADS == C::S, "one row per thread");
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bars[NB];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t tiles = (uint32_t)(p.nvec * p.nhi * p.nlo * p.nstripes);
  constexpr bool END_B = C::W > 1 && (START_B ^ ((NPARTS & 1) != 0));
  if (threadIdx.x == 0) {
#pragma unroll
    for (int b = 0; b < NB; ++b) mbar_init(&bars[b], C::THREADS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phases = 0;  // bit b = parity of bars[b]
#pragma unroll
  for (int b = 0; b < NB - 1; ++b) {
    const uint32_t t0 = blockIdx.x + b * gridDim.x;
    if (t0 < tiles) tma_stage_row<C>(p, tile_decode(p, t0, LS), smem + b * (C::S * 32), &bars[b]);
  }
  int cur = 0;
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, cur = (cur + 1 == NB) ? 0 : cur + 1) {
    const TileIdx cti = tile_decode(p, tile, LS);
    float* buf = smem + cur * (C::S * 32);
    mbar_wait(&bars[cur], (phases >> cur) & 1u);
    phases ^= 1u << cur;
    const uint32_t nxt = tile + (NB - 1) * gridDim.x;
    if (nxt < tiles) {
      const int nb = (cur + NB - 1) % NB;  // the buffer of the previous tile
      bulk_wait_read();  // my bulk store out of that buffer has been read
      tma_stage_row<C>(p, tile_decode(p, nxt, LS), smem + nb * (C::S * 32), &bars[nb]);
    }

    float r[C::R];
    {
      constexpr bool LB = START_B && C::W > 1;
#pragma unroll
      for (int j = 0; j < C::R; ++j) r[j] = buf[scol_s<C>(LB, w, j) * 32 + lane];
    }
    __syncthreads();  // buf is reused by the transposes / epilogue
#pragma unroll
    for (int part = 0; part < NPARTS; ++part) {
      const bool lay_b = C::W > 1 && (START_B ^ ((part & 1) != 0));
      if ((DMASK >> part) & 1) {
        if constexpr (DMODE == SD_TILE) {
          const float4* Dp = reinterpret_cast<const float4*>(p.dd[part] + (int64_t)cti.cs * (C::S * 32) +
                                                             w * (C::R * 32)) + lane;
#pragma unroll
          for (int q = 0; q < C::R / 4; ++q) {
            const float4 dv = __ldg(Dp + q * 32);
            r[4 * q] *= dv.x;
            r[4 * q + 1] *= dv.y;
            r[4 * q + 2] *= dv.z;
            r[4 * q + 3] *= dv.w;
          }
        } else {
          const float* Dt = p.dd[part] + ((int64_t)cti.lo * p.nhi + cti.hi) * C::S;
          if (!lay_b) {
#pragma unroll
            for (int q = 0; q < C::R / 4; ++q) {
              const float4 dv = __ldg(reinterpret_cast<const float4*>(Dt + w * C::R) + q);
              r[4 * q] *= dv.x;
              r[4 * q + 1] *= dv.y;
              r[4 * q + 2] *= dv.z;
              r[4 * q + 3] *= dv.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < C::R; ++j) r[j] *= __ldg(Dt + scol_s<C>(lay_b, w, j));
          }
        }
      }
      reg_fwht<C::R, 0, C::LR>(r);
      if constexpr (C::W > 1) {
#pragma unroll
        for (int j = 0; j < C::R; ++j) buf[scol_s<C>(lay_b, w, j) * 32 + lane] = r[j];
        __syncthreads();
#pragma unroll
        for (int j = 0; j < C::R; ++j) r[j] = buf[scol_s<C>(!lay_b, w, j) * 32 + lane];
        __syncthreads();
        if (!lay_b)
          reg_fwht<C::R, C::LR - C::LW, C::LR>(r);
        else
          reg_fwht<C::R, 0, C::LW>(r);
      }
    }
    // epilogue: registers -> smem rows -> one bulk store per row
    float scale = 1.0f;
    if constexpr (EPI != EPI_STORE) scale = p.cscale;
#pragma unroll
    for (int j = 0; j < C::R; ++j) {
      float o = r[j];
      if constexpr (EPI != EPI_STORE) o *= scale;
      if constexpr (EPI == EPI_Y) {
        if (p.relu) o = fmaxf(o, 0.0f);
      }
      buf[scol_s<C>(END_B, w, j) * 32 + lane] = o;
    }
    fence_proxy_async();
    __syncthreads();
    {
      const int s = threadIdx.x;
      const int64_t e = cti.e0 + ((int64_t)s << p.s0);
      if constexpr (EPI == EPI_GATHER) {
        const int32_t orow = __ldg(p.rowmap + e);
        if (orow >= 0) bulk_store(p.dst + (int64_t)orow * p.ld_out + (int64_t)cti.cs * 32, buf + s * 32, 128);
      } else if constexpr (EPI == EPI_Y) {
        const int64_t f = e * p.dst_ld + (int64_t)cti.cs * 32;
        float* drow = p.dst + (int64_t)cti.v * p.dst_vstride + f;
        if (f + 32 <= p.rows_valid) {
          bulk_store(drow, buf + s * 32, 128);
        } else {
          for (int q = 0; q < 32; ++q)
            if (f + q < p.rows_valid) drow[q] = buf[s * 32 + q];
        }
      } else {
        bulk_store(p.dst + (int64_t)cti.v * p.dst_vstride + e * p.dst_ld + (int64_t)cti.cs * 32, buf + s * 32, 128);
      }
      bulk_commit();
    }
  }
  bulk_wait_all();
}

template <int LS, int NPARTS, int DMASK, bool START_B, int DMODE, int EPI>
inline cudaError_t launch_tcol(const ColParams& p_in, int sms, cudaStream_t s) {
  using C = SColCfg<LS>;
  ColParams p = p_in;
  set_tiling(p);
  auto kern = colpass_tma_kernel<LS, NPARTS, DMASK, START_B, DMODE, EPI>;
  static int occ = 0;
  if (occ == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(TmaCfg<LS>::SMEM));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, TmaCfg<LS>::SMEM);
    if (e != cudaSuccess) return e;
    occ = occ < 1 ? 1 : occ;
  }
  const int64_t tiles = p.nvec * p.nhi * p.nlo * p.nstripes;
  const int64_t grid = tiles < int64_t(sms) * occ ? (tiles < 1 ? 1 : tiles) : int64_t(sms) * occ;
  kern<<<static_cast<unsigned>(grid), C::THREADS, TmaCfg<LS>::SMEM, s>>>(p);
  return cudaGetLastError();
}

template <int LS>
inline cudaError_t launch_tcol_prog(int prog, const ColParams& p, int sms, cudaStream_t s) {
  switch (prog) {
    case SC_FIRST: return launch_tcol<LS, 1, 1, false, SD_ROW, EPI_STORE>(p, sms, s);
    case SC_MID: return launch_tcol<LS, 2, 2, true, SD_ROW, EPI_STORE>(p, sms, s);
    case SC_LAST: return launch_tcol<LS, 1, 0, false, SD_ROW, EPI_GATHER>(p, sms, s);
    case SC_SINGLE: return launch_tcol<LS, 3, 7, false, SD_ROW, EPI_GATHER>(p, sms, s);
    case SC_VMID: return launch_tcol<LS, 2, 2, true, SD_TILE, EPI_STORE>(p, sms, s);
    case SC_VLAST: return launch_tcol<LS, 1, 0, false, SD_ROW, EPI_Y>(p, sms, s);
  }
  return cudaErrorInvalidValue;
}

// LS in [5, 9]: one row per thread and two tile buffers per SM.
inline cudaError_t launch_tcol_ls(int ls, int prog, const ColParams& p, int sms, cudaStream_t s) {
  switch (ls) {
    case 5: return launch_tcol_prog<5>(prog, p, sms, s);
    case 6: return launch_tcol_prog<6>(prog, p, sms, s);
    case 7: return launch_tcol_prog<7>(prog, p, sms, s);
    case 8: return launch_tcol_prog<8>(prog, p, sms, s);
    case 9: return launch_tcol_prog<9>(prog, p, sms, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace spn
