// Column pass with TMA tensor copies.
//
// A tile is 2^LS rows x 32 floats (LS >= 5: one row per thread).  One elected thread
// moves the whole tile with ceil(2^LS / 256) cp.async.bulk.tensor copies that complete
// on an mbarrier, and stores it back the same way — per-thread 128-B bulk copies
// compile to a 32-iteration uniform-register loop per warp (R2UR/ELECT/BRA), which
// measured as ~60% of the pass's instructions.  Three tile buffers keep two tiles in
// flight while one is computed; the gather epilogue (sketch) and a ragged EPI_Y tail
// still use one bulk copy per row.  Requirements (checked by the host): 16-B aligned
// base pointers and leading dimensions; operands that are not tensor views fall back
// to the cp.async pass.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

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

// ---------------------------------------------------------------- tensor maps
// Every column-pass operand is a 4-D view (col, lo, hs, v) of a row-major buffer:
// element (v, e, col) with e = hs*2^s0 + lo lives at v*vstride + e*ld + col.  A tile
// (2^LS rows s, 32 columns) is the box {32, 1, 2^LS, 1} at (cs*32, lo, hi*2^LS, v),
// issued as ceil(2^LS / 256) tensor copies.  Rows / columns outside the view are
// zero-filled on load and skipped on store, which is exactly the pass semantics of
// zero-padded N and ragged d.
struct TmaMaps {
  CUtensorMap src;
  CUtensorMap dst;
  int tdst;  // 1: the epilogue stores through dst; 0: one 128-B bulk copy per row
};

inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      f = nullptr;
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

inline bool encode_view(CUtensorMap* m, const float* base, int64_t ncols, int64_t ld, int s0, int64_t nhs,
                        int64_t nvec, int64_t vstride, int box_s) {
  const auto enc = tmap_encoder();
  if (!enc || reinterpret_cast<uintptr_t>(base) % 16 != 0 || ld % 4 != 0 || ncols < 1 || nhs < 1 || nvec < 1)
    return false;
  if (nvec > 1 && (vstride % 4 != 0 || vstride <= 0)) return false;
  const int64_t vs = nvec > 1 ? vstride : (nhs << s0) * ld;
  const cuuint64_t dims[4] = {(cuuint64_t)ncols, (cuuint64_t)1 << s0, (cuuint64_t)nhs, (cuuint64_t)nvec};
  const cuuint64_t strides[3] = {(cuuint64_t)ld * 4, (cuuint64_t)(ld << s0) * 4, (cuuint64_t)vs * 4};
  const cuuint32_t box[4] = {32, 1, (cuuint32_t)box_s, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__device__ __forceinline__ void tensor_load4(float* sdst, const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(sdst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tensor_store4(const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                              const float* ssrc) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(ssrc))
               : "memory");
}

// Buffer count: two tiles (one load in flight while one is computed).  Three buffers
// measured slower (c4 0.208 vs 0.193 ms, c5 1.545 vs 1.519 ms): the smaller footprint
// lets the other stream's row-pass CTAs co-reside on the SM.
#ifndef SPN_TMA_NBUF
#define SPN_TMA_NBUF 2
#endif

// Tile config of the TMA column pass: 32 rows per thread (5 register bits).  SPN_TCOL_LR8 = 6 runs the
// 2^8-row tiles with 64 rows per thread on 4 warps instead (three CTAs of 128 threads per SM instead of
// two of 256, longer phases between the CTA barriers, three tiles loading per SM instead of two):
// measured equal (c5 1.290 vs 1.289 ms, grouped c4 passes 0.189 vs 0.187 ms), so the default stays 5.
#ifndef SPN_TCOL_LR8
#define SPN_TCOL_LR8 5
#endif
template <int LS_>
struct TColCfg {
  static constexpr int LS = LS_;
  static constexpr int LR = LS == 8 ? SPN_TCOL_LR8 : (LS < 5 ? LS : 5);
  static constexpr int LW = LS - LR;
  static constexpr int R = 1 << LR, W = 1 << LW, S = 1 << LS;
  static constexpr int THREADS = 32 * W;
  static constexpr int RPT = S / THREADS;  // tile rows per thread in the per-row epilogues
};

template <int LS>
struct TmaCfg {
  static constexpr size_t TILE = sizeof(float) * (size_t(1) << LS) * 32;
  static constexpr int NBUF = SPN_TMA_NBUF;
  static constexpr size_t SMEM = TILE * NBUF + 64;  // + the mbarriers
  static constexpr int BOX = LS > 8 ? 256 : (1 << LS);  // rows per tensor copy
  static constexpr int NBOX = (1 << LS) / BOX;
  static constexpr int BY_SMEM = (int)((227u * 1024u) / SMEM);
  static constexpr int BY_REGS = 512 / TColCfg<LS>::THREADS;
  static constexpr int M0 = BY_SMEM < BY_REGS ? BY_SMEM : BY_REGS;
  static constexpr int MIN_CTAS = M0 < 1 ? 1 : M0;
};

// Thread 0: the tensor copies of tile ti into buf, completing on bar.
template <int LS>
__device__ __forceinline__ void tma_issue_tile(const CUtensorMap* m, const TileIdx& ti, float* buf, uint64_t* bar) {
  using T = TmaCfg<LS>;
  mbar_arrive_tx(bar, (uint32_t)T::TILE);
#pragma unroll
  for (int b = 0; b < T::NBOX; ++b)
    tensor_load4(buf + b * T::BOX * 32, m, (int)ti.cs * 32, (int)ti.lo, (int)(ti.hi << LS) + b * T::BOX, (int)ti.v,
                 bar);
}

template <int LS, int NPARTS, int DMASK, bool START_B, int DMODE, int EPI>
__global__ void __launch_bounds__(TColCfg<LS>::THREADS, TmaCfg<LS>::MIN_CTAS)
    colpass_tma_kernel(const ColParams p, const __grid_constant__ TmaMaps tm) {
  pdl_enter();
  using C = TColCfg<LS>;
  using T = TmaCfg<LS>;
  constexpr int NB = T::NBUF;  // tiles in flight: NB-1 loads ahead of the compute
  // tile buffers at the dynamic-smem base (tensor copies need 128-B aligned smem), barriers after them
  extern __shared__ __align__(128) float smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NB * (C::S * 32));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool leader = threadIdx.x == 0;
  const uint32_t tiles = (uint32_t)(p.nvec * p.nhi * p.nlo * p.nstripes);
  constexpr bool END_B = C::W > 1 && (START_B ^ ((NPARTS & 1) != 0));
  const bool tstore = EPI != EPI_GATHER && tm.tdst;
  if (leader) {
#pragma unroll
    for (int b = 0; b < NB; ++b) mbar_init(&bars[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int b = 0; b < NB - 1; ++b) {
      const uint32_t t0 = blockIdx.x + b * gridDim.x;
      if (t0 < tiles) tma_issue_tile<LS>(&tm.src, tile_decode(p, t0, LS), smem + b * (C::S * 32), &bars[b]);
    }
  }
  __syncthreads();
  uint32_t phases = 0;  // bit b = parity of bars[b]
  int cur = 0;
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, cur = (cur + 1 == NB) ? 0 : cur + 1) {
    const TileIdx cti = tile_decode(p, tile, LS);
    float* buf = smem + cur * (C::S * 32);
    mbar_wait(&bars[cur], (phases >> cur) & 1u);
    phases ^= 1u << cur;

    float r[C::R];
    {
      constexpr bool LB = START_B && C::W > 1;
#pragma unroll
      for (int j = 0; j < C::R; ++j) r[j] = buf[scol_s<C>(LB, w, j) * 32 + lane];
    }
    if constexpr (EPI == EPI_GATHER) {
      if (p.discard_src) {  // these rows of the workspace are dead now: no write-back to HBM
#pragma unroll
        for (int h = 0; h < C::RPT; ++h) {
          const int64_t e = cti.e0 + ((int64_t)(threadIdx.x + h * C::THREADS) << p.s0);
          const int64_t off = e * p.src_ld + (int64_t)cti.cs * 32;
          if (off + 32 <= p.src_valid)
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(p.src + (int64_t)cti.v * p.src_vstride + off) : "memory");
        }
      }
    }
    bulk_wait_read();  // my bulk stores out of the buffer about to be refilled have read it
    __syncthreads();   // buf free for the transposes; the previous tile's buffer free for a load
    const uint32_t nxt = tile + (NB - 1) * gridDim.x;
    if (leader && nxt < tiles) {
      const int nb = (cur + NB - 1) % NB;  // the buffer of the previous tile
      tma_issue_tile<LS>(&tm.src, tile_decode(p, nxt, LS), smem + nb * (C::S * 32), &bars[nb]);
    }
#pragma unroll
    for (int part = 0; part < NPARTS; ++part) {
      const bool lay_b = C::W > 1 && (START_B ^ ((part & 1) != 0));
      if ((DMASK >> part) & 1) {
        if constexpr (DMODE == SD_TILE) {
          const float4* Dp = reinterpret_cast<const float4*>(p.dd[part] + (int64_t)cti.cs * (C::S * 32) +
                                                             w * (C::R * 32)) + lane;
#pragma unroll
          for (int q = 0; q < C::R / 4; ++q) {
#ifdef SPN_DBG_NODIAG_COL  // (bound experiments only: wrong results)
            const float4 dv = make_float4(1.f, -1.f, 1.f, -1.f);
#else
            const float4 dv = __ldg(Dp + q * 32);
#endif
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
    // epilogue: registers -> smem rows -> tensor store (or one bulk store per row)
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
    if (tstore) {
      if (leader) {
#pragma unroll
        for (int b = 0; b < T::NBOX; ++b)
          tensor_store4(&tm.dst, (int)cti.cs * 32, (int)cti.lo, (int)(cti.hi << LS) + b * T::BOX, (int)cti.v,
                        buf + b * T::BOX * 32);
        bulk_commit();
      }
    } else {
#pragma unroll
      for (int h = 0; h < C::RPT; ++h) {
        const int s = threadIdx.x + h * C::THREADS;
        const int64_t e = cti.e0 + ((int64_t)s << p.s0);
        if constexpr (EPI == EPI_GATHER) {
          const int32_t orow = __ldg(p.rowmap + e);
          if (orow >= 0) bulk_store(p.dst + (int64_t)orow * p.ld_out + (int64_t)cti.cs * 32, buf + s * 32, 128);
        } else {
          const int64_t f = e * p.dst_ld + (int64_t)cti.cs * 32;
          float* drow = p.dst + (int64_t)cti.v * p.dst_vstride + f;
          if (EPI == EPI_STORE || f + 32 <= p.rows_valid) {
            bulk_store(drow, buf + s * 32, 128);
          } else {
            for (int q = 0; q < 32; ++q)
              if (f + q < p.rows_valid) drow[q] = buf[s * 32 + q];
          }
        }
      }
      bulk_commit();
    }
  }
  bulk_wait_all();
}

// Host side of the tensor-map column pass: false when the operands cannot be
// described as tensor views (the caller then uses the cp.async pass).
template <int LS, int NPARTS, int DMASK, bool START_B, int DMODE, int EPI>
inline cudaError_t launch_tcol(const ColParams& p_in, int sms, cudaStream_t s, bool* done) {
  using C = TColCfg<LS>;
  using T = TmaCfg<LS>;
  *done = false;
  ColParams p = p_in;
  set_tiling(p);
  TmaMaps tm;
  std::memset(&tm, 0, sizeof(tm));
  // source rows e < E valid (E = src_valid / src_ld), as a bound on hs = e >> s0
  if (p.src_valid % p.src_ld != 0) return cudaSuccess;
  const int64_t E = p.src_valid / p.src_ld, nhs_all = p.nhi << LS;
  if (E <= 0) return cudaSuccess;
  if ((E & ((int64_t(1) << p.s0) - 1)) != 0 && E < (nhs_all << p.s0)) return cudaSuccess;
  const int64_t nhs_src = std::min<int64_t>(nhs_all, std::max<int64_t>(E >> p.s0, 1));
  if (!encode_view(&tm.src, p.src, p.ncols, p.src_ld, p.s0, nhs_src, p.nvec, p.src_vstride, T::BOX))
    return cudaSuccess;
  tm.tdst = 0;
  if (EPI == EPI_STORE) {
    tm.tdst = encode_view(&tm.dst, p.dst, p.ncols, p.dst_ld, p.s0, nhs_all, p.nvec, p.dst_vstride, T::BOX);
    if (!tm.tdst) return cudaSuccess;
  } else if (EPI == EPI_Y && p.rows_valid % p.dst_ld == 0 && p.s0 == 0) {
    const int64_t ey = std::min<int64_t>(nhs_all, p.rows_valid / p.dst_ld);
    tm.tdst = ey > 0 && encode_view(&tm.dst, p.dst, p.ncols, p.dst_ld, 0, ey, p.nvec, p.dst_vstride, T::BOX);
  }
  auto kern = colpass_tma_kernel<LS, NPARTS, DMASK, START_B, DMODE, EPI>;
  static int occ = 0;
  if (occ == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(T::SMEM));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, T::SMEM);
    if (e != cudaSuccess) return e;
    occ = occ < 1 ? 1 : occ;
  }
  const int64_t tiles = p.nvec * p.nhi * p.nlo * p.nstripes;
  const int64_t grid = tiles < int64_t(sms) * occ ? (tiles < 1 ? 1 : tiles) : int64_t(sms) * occ;
  *done = true;
  return launch_pdl(p.pdl != 0, kern, static_cast<unsigned>(grid), C::THREADS, T::SMEM, s, p, tm);
}

template <int LS>
inline cudaError_t launch_tcol_prog(int prog, const ColParams& p, int sms, cudaStream_t s, bool* done) {
  switch (prog) {
    case SC_FIRST: return launch_tcol<LS, 1, 1, false, SD_ROW, EPI_STORE>(p, sms, s, done);
    case SC_MID: return launch_tcol<LS, 2, 2, true, SD_ROW, EPI_STORE>(p, sms, s, done);
    case SC_LAST: return launch_tcol<LS, 1, 0, false, SD_ROW, EPI_GATHER>(p, sms, s, done);
    case SC_SINGLE: return launch_tcol<LS, 3, 7, false, SD_ROW, EPI_GATHER>(p, sms, s, done);
    case SC_VMID: return launch_tcol<LS, 2, 2, true, SD_TILE, EPI_STORE>(p, sms, s, done);
    case SC_VLAST: return launch_tcol<LS, 1, 0, false, SD_ROW, EPI_Y>(p, sms, s, done);
  }
  return cudaErrorInvalidValue;
}

// LS in [5, 9]: one row per thread.  Operands that are not tensor views fall back
// to the cp.async column pass.
inline cudaError_t launch_tcol_ls(int ls, int prog, const ColParams& p, int sms, cudaStream_t s) {
  bool done = false;
  cudaError_t e = cudaErrorInvalidValue;
  switch (ls) {
    case 5: e = launch_tcol_prog<5>(prog, p, sms, s, &done); break;
    case 6: e = launch_tcol_prog<6>(prog, p, sms, s, &done); break;
    case 7: e = launch_tcol_prog<7>(prog, p, sms, s, &done); break;
    case 8: e = launch_tcol_prog<8>(prog, p, sms, s, &done); break;
    case 9: e = launch_tcol_prog<9>(prog, p, sms, s, &done); break;
  }
  if (e != cudaSuccess || done) return e;
  return launch_scol_ls(ls, prog, p, sms, s);
}

}  // namespace spn
