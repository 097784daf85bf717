// Pipelined multi-pass kernels: every tile/segment is staged global->smem with
// cp.async (no registers, zero-filled out of range) and the NEXT tile is requested
// before the current one is computed, so each SM keeps loads in flight while its
// FP32 pipe and smem transposes work.  Diagonals are pre-permuted on the host into
// the exact order each pass consumes (16-B loads with immediate offsets, no per-element
// address arithmetic).  Used by spinner_big.cuh when the pointers are 16-B aligned;
// the register-only kernels there are the fallback.
#pragma once

#include <cstdlib>

#include <cuda_runtime.h>

#include <algorithm>

#include "spinner_vec.cuh"

namespace spn {

// Programmatic dependent launch between consecutive passes of one stream: each pass lets
// its successor start launching immediately and waits for its predecessor's completion
// (and memory flush) before touching data — the successor's launch and prologue overlap
// the predecessor's tail.  Both instructions are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SPN_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class K, class... A>
inline cudaError_t launch_pdl(bool pdl, K kern, unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                              A... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = (pdl && pdl_enabled()) ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// ----------------------------------------------------------------- staged column pass
// Tile = 2^LS rows (transformed sub-index s) x 32 contiguous columns; thread (w, lane)
// holds column lane and R = 32 rows: layout A s = w*R + j, layout B s = j*W + w.
// LS <= 9 so two 64 KB tile buffers fit one SM.
template <int LS_>
struct SColCfg {
  static constexpr int LS = LS_;
  static constexpr int LR = LS < 5 ? LS : 5;
  static constexpr int LW = LS - LR;  // <= 4
  static constexpr int R = 1 << LR, W = 1 << LW, S = 1 << LS;
  static constexpr int THREADS = 32 * W;
  static constexpr size_t SMEM = sizeof(float) * 2 * S * 32;
  // as many CTAs as shared memory allows, but never fewer than 128 registers per thread
  static constexpr int BY_SMEM = (int)((227u * 1024u) / SMEM);
  static constexpr int BY_REGS = 512 / THREADS;
  static constexpr int MIN_CTAS0 = BY_SMEM < BY_REGS ? BY_SMEM : BY_REGS;
  static constexpr int MIN_CTAS = MIN_CTAS0 < 1 ? 1 : MIN_CTAS0;
};

enum SDMode : int { SD_ROW = 0, SD_TILE = 1 };          // broadcast per row / tile-permuted per element
enum SEpi : int { EPI_STORE = 0, EPI_Y = 1, EPI_GATHER = 2 };

template <class C>
__device__ __forceinline__ uint32_t scol_s(bool lay_b, int w, int j) {
  return lay_b ? (uint32_t)(j * C::W + w) : (uint32_t)(w * C::R + j);
}

// 32-bit division by an invariant (Granlund-Montgomery): q = n / d for n < 2^32.
__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint32_t d, uint32_t m, uint32_t l) {
  if (d == 1) return n;
  const uint32_t t = __umulhi(n, m);
  return (t + ((n - t) >> 1)) >> (l - 1);
}

struct TileIdx {
  uint32_t cs, lo, hi, v;
  int64_t e0;
};

// tile = ((v * nhi + hi) * nlo + lo) * nstripes + cs   (nhi, nlo powers of two)
__device__ __forceinline__ TileIdx tile_decode(const ColParams& p, uint32_t tile, int ls) {
  TileIdx t;
  uint32_t q = fdiv(tile, (uint32_t)p.nstripes, p.fd_m, p.fd_l);
  t.cs = tile - q * (uint32_t)p.nstripes;
  t.lo = q & ((1u << p.lg_nlo) - 1u);
  q >>= p.lg_nlo;
  t.hi = q & ((1u << p.lg_nhi) - 1u);
  t.v = q >> p.lg_nhi;
  t.e0 = ((int64_t)t.hi << (p.s0 + ls)) + t.lo;
  return t;
}

// cp.async a 2^LS x 32 tile (row s at base + s*step, 8 chunks of 16 B) into buf[s][32];
// zero fill past the valid columns / elements (ragged d, zero padding of the N axis).
template <class C>
__device__ __forceinline__ void stage_tile(const ColParams& p, const TileIdx& ti, float* buf) {
  const int64_t f0 = ti.e0 * p.src_ld + (int64_t)ti.cs * 32;
  const float* base = p.src + (int64_t)ti.v * p.src_vstride + f0;
  const uint32_t step = (uint32_t)(p.src_ld << p.s0);
  const int64_t lim = p.src_valid - f0;
  const int64_t colrem = p.ncols - (int64_t)ti.cs * 32;
  const bool full = colrem >= 32 && lim >= (int64_t)(C::S - 1) * step + 32;
#pragma unroll
  for (int u = 0; u < (8 * C::S + C::THREADS - 1) / C::THREADS; ++u) {
    const int c = threadIdx.x + C::THREADS * u;
    if (8 * C::S % C::THREADS == 0 || c < 8 * C::S) {
      const int s = c >> 3, q = c & 7;
      const uint32_t off = (uint32_t)s * step + 4u * q;
      if (full) {
        cp_async16(buf + s * 32 + 4 * q, base + off, 16);
      } else {
        const int64_t rem = min(colrem - 4 * q, lim - (int64_t)off);
        const int bytes = rem >= 4 ? 16 : (rem > 0 ? (int)rem * 4 : 0);
        cp_async16(buf + s * 32 + 4 * q, bytes > 0 ? base + off : p.src, bytes);
      }
    }
  }
}

// Pass program: NPARTS H's over the LS bits, diagonal dd[p] before part p when DMASK
// bit p is set, starting in layout B if START_B, epilogue EPI:
//   EPI_STORE  raw store to dst (workspace),
//   EPI_Y      y = relu?(cscale * v) for flat element < rows_valid (config 5 output),
//   EPI_GATHER dst[rowmap[e]][col] = cscale * v (sketch P rows).
// SD_TILE diagonals are host-permuted per tile [cs][w][R/4][lane][4] and must be applied
// in layout A; SD_ROW diagonals are one value per row, [(lo*nhi + hi)*S + s].
template <int LS, int NPARTS, int DMASK, bool START_B, int DMODE, int EPI>
__global__ void __launch_bounds__(SColCfg<LS>::THREADS, SColCfg<LS>::MIN_CTAS) colpass_staged_kernel(const ColParams p) {
  pdl_enter();
  using C = SColCfg<LS>;
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t tiles = (uint32_t)(p.nvec * p.nhi * p.nlo * p.nstripes);
  constexpr bool END_B = C::W > 1 && (START_B ^ ((NPARTS & 1) != 0));
  const uint32_t ostep = (uint32_t)(p.dst_ld << p.s0);
  int cur = 0;
  TileIdx ti{};
  if (blockIdx.x < tiles) {
    ti = tile_decode(p, blockIdx.x, LS);
    stage_tile<C>(p, ti, smem);
  }
  cp_async_commit();
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, cur ^= 1) {
    const TileIdx cti = ti;
    const bool colok = (int64_t)cti.cs * 32 + lane < p.ncols;
    float* buf = smem + cur * (C::S * 32);
    cp_async_wait_all();
    __syncthreads();  // tile in buf visible; everyone is done with the other buffer
    const uint32_t nxt = tile + gridDim.x;
    if (nxt < tiles) {
      ti = tile_decode(p, nxt, LS);
      stage_tile<C>(p, ti, smem + (cur ^ 1) * (C::S * 32));
    }
    cp_async_commit();

    float r[C::R];
    {
      constexpr bool LB = START_B && C::W > 1;
#pragma unroll
      for (int j = 0; j < C::R; ++j) r[j] = buf[scol_s<C>(LB, w, j) * 32 + lane];
    }
    if constexpr (C::W > 1) __syncthreads();  // buf is reused by the transposes
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
          if (!lay_b && C::R >= 4) {
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
        // transpose through this tile's own buffer (the other buffer is being filled)
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
    if constexpr (EPI == EPI_GATHER) {
      const int32_t* rm = p.rowmap + cti.e0;
      float* ob = p.dst + (int64_t)cti.cs * 32 + lane;
#pragma unroll
      for (int j = 0; j < C::R; ++j) {
        const int32_t orow = __ldg(rm + ((int64_t)scol_s<C>(END_B, w, j) << p.s0));
        if (colok && orow >= 0) __stcs(ob + (int64_t)orow * p.ld_out, r[j] * p.cscale);
      }
    } else if constexpr (EPI == EPI_Y) {
      const int64_t f0 = cti.e0 * p.dst_ld + (int64_t)cti.cs * 32 + lane;  // flat index inside the vector
      float* db = p.dst + (int64_t)cti.v * p.dst_vstride + f0;
      const bool all = f0 + (int64_t)(C::S - 1) * ostep < p.rows_valid;
#pragma unroll
      for (int j = 0; j < C::R; ++j) {
        const uint32_t off = scol_s<C>(END_B, w, j) * ostep;
        float o = r[j] * p.cscale;
        if (p.relu) o = fmaxf(o, 0.0f);
        if (colok && (all || f0 + off < p.rows_valid)) __stcs(db + off, o);
      }
    } else {
      float* db = p.dst + (int64_t)cti.v * p.dst_vstride + cti.e0 * p.dst_ld + (int64_t)cti.cs * 32 + lane;
      if (colok) {
#pragma unroll
        for (int j = 0; j < C::R; ++j) db[scol_s<C>(END_B, w, j) * ostep] = r[j];
      }
    }
  }
  cp_async_wait_all();
}

// ------------------------------------------------------------------- staged row pass
// One CTA of T = 2^LT threads per contiguous segment of N = 2^(LR+LT) floats (layouts of
// spinner_vec.cuh: one warp up to 2^11, R = T = 64 at 2^12 — half the registers of a
// single-warp R = 128 segment, c5 row passes 20.5 -> see DESIGN.md).  Diagonals in the
// layout-A float format of spinner_vec.cuh, per segment.
//   RP_FIRST  src -> [D@A] H(A->B) -> dst    (reads the staged segment in layout A)
//   RP_MID    buf -> H(B->A) [D@A] H(A->B) -> buf   (in place)
//   RP_LAST   buf -> H(B->A) -> xpose -> y = relu?(c*v), truncated to rows_valid
enum RowProg : int { RP_FIRST = 0, RP_MID = 1, RP_LAST = 2 };

struct RowParams2 {
  const float* src;       // segment source (RP_FIRST: x, else the workspace)
  int64_t src_vstride, n_in;  // RP_FIRST: zero pad beyond n_in
  float* dst;             // segment destination (workspace or y)
  int64_t dst_vstride;
  int64_t nseg, nvec;     // nseg: power of two
  const float* d;         // diagonal for this pass (RP_FIRST / RP_MID)
  int64_t rows_valid;
  float c;
  int relu;
};

#ifndef SPN_ROW_STAGE_D
#define SPN_ROW_STAGE_D 1
#endif
#ifndef SPN_ROW_DIRECT
#define SPN_ROW_DIRECT 1  // c5: 1.321 -> 1.316 ms (3 A/B pairs)
#endif
template <int PROG>
struct RowCfg {  // direct loads (layout B, no smem staging) for the passes that start in layout B
  static constexpr bool DIRECT = SPN_ROW_DIRECT && PROG != RP_FIRST;
};

template <int LR, int LT, int PROG>
__global__ void __launch_bounds__(1 << LT) rowpass_staged_kernel(const RowParams2 p) {
  pdl_enter();
  using C = VCfg<LR, LT>;
  static_assert(C::GPC == 1, "one segment per CTA");
  constexpr bool DIRECT = RowCfg<PROG>::DIRECT;
  extern __shared__ __align__(16) float smem[];
  float* xb = smem;                          // staging buffer (swizzled 16-B chunks)
  float* sm = DIRECT ? smem : smem + C::N;   // transpose buffer
  // RP_MID: this segment's diagonal slice, copied by each thread (its own float4s, cp.async) at the
  // start of the item so the L2 round trip overlaps the first H half instead of stalling after it
  constexpr bool STAGE_D = SPN_ROW_STAGE_D && DIRECT && PROG == RP_MID;
  float* db = sm + C::N;
  const int t = threadIdx.x;
  const int64_t items = p.nvec * p.nseg;
  const int lgseg = __ffsll(p.nseg) - 1;
  auto stage = [&](int64_t item) {
    const int64_t v = item >> lgseg, seg = item & (p.nseg - 1);
    int64_t valid = C::N;
    if (PROG == RP_FIRST) {
      const int64_t rem = p.n_in - seg * C::N;
      valid = rem < 0 ? 0 : (rem > C::N ? C::N : rem);
    }
    stage_x<C>(xb, p.src + v * p.src_vstride + seg * C::N, valid, t);
  };
  if (!DIRECT && (int64_t)blockIdx.x < items) stage(blockIdx.x);
  cp_async_commit();
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int64_t v = item >> lgseg, seg = item & (p.nseg - 1);
    if constexpr (STAGE_D) {
      const float* dsrc = p.d + seg * C::N;
#pragma unroll
      for (int q = 0; q < C::R / 4; ++q) cp_async16(db + (q * C::T + t) * 4, dsrc + (q * C::T + t) * 4, 16);
      cp_async_commit();
    }
    float r[C::R];
    if constexpr (DIRECT) {
      const float* src = p.src + v * p.src_vstride + seg * C::N + t;
#pragma unroll
      for (int j = 0; j < C::R; ++j) r[j] = __ldcg(src + j * C::T);
    } else {
    cp_async_wait_all();
    group_sync<C>();
    {
      const Swz<C> z(t);
      if constexpr (PROG == RP_FIRST) {
#pragma unroll
        for (int q = 0; q < C::R / 4; ++q) {
          const float4 xv = *reinterpret_cast<const float4*>(xb + z.A(t, q));
          r[4 * q] = xv.x;
          r[4 * q + 1] = xv.y;
          r[4 * q + 2] = xv.z;
          r[4 * q + 3] = xv.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < C::R; ++j) r[j] = xb[z.B(t, j)];
      }
    }
    group_sync<C>();
    if (item + gridDim.x < items) stage(item + gridDim.x);
    cp_async_commit();
    }
    if constexpr (PROG != RP_FIRST) fwht_B_to_A<C>(r, sm, t);
    if constexpr (PROG != RP_LAST) {
      const float4* f = reinterpret_cast<const float4*>(p.d + seg * C::N);
      if constexpr (STAGE_D) cp_async_wait_all();  // this thread's own copies: no barrier needed
#pragma unroll
      for (int q = 0; q < C::R / 4; ++q) {
#ifdef SPN_DBG_NODIAG_ROW  // (bound experiments only: wrong results)
        const float4 dv = make_float4(1.f, -1.f, 1.f, -1.f);
#else
        const float4 dv = STAGE_D ? reinterpret_cast<const float4*>(db)[q * C::T + t] : __ldg(f + q * C::T + t);
#endif
        r[4 * q] *= dv.x;
        r[4 * q + 1] *= dv.y;
        r[4 * q + 2] *= dv.z;
        r[4 * q + 3] *= dv.w;
      }
      fwht_A_to_B<C>(r, sm, t);
      float* row = p.dst + v * p.dst_vstride + seg * C::N;
#pragma unroll
      for (int j = 0; j < C::R; ++j) row[j * C::T + t] = r[j];
    } else {
      xpose_A_to_B<C>(r, sm, t);
      float* yrow = p.dst + v * p.dst_vstride + seg * C::N;
      const bool all = seg * C::N + C::N <= p.rows_valid;
#pragma unroll
      for (int j = 0; j < C::R; ++j) {
        float o = r[j] * p.c;
        if (p.relu) o = fmaxf(o, 0.0f);
        if (all || seg * C::N + j * C::T + t < p.rows_valid) __stcs(yrow + j * C::T + t, o);
      }
    }
  }
  cp_async_wait_all();
}

// ------------------------------------------------------------------------- launch
template <int LS, int NPARTS, int DMASK, bool START_B, int DMODE, int EPI>
inline cudaError_t launch_scol(const ColParams& p_in, int sms, cudaStream_t s) {
  using C = SColCfg<LS>;
  ColParams p = p_in;
  set_tiling(p);
  auto kern = colpass_staged_kernel<LS, NPARTS, DMASK, START_B, DMODE, EPI>;
  static int occ = 0;
  if (occ == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::SMEM));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM);
    if (e != cudaSuccess) return e;
    occ = std::max(occ, 1);
  }
  const int64_t tiles = p.nvec * p.nhi * p.nlo * p.nstripes;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t(sms) * occ));
  return launch_pdl(p.pdl != 0, kern, static_cast<unsigned>(grid), C::THREADS, C::SMEM, s, p);
}

// Programs: sketch P1 ([D] H), sketch P2/P3 (H [D] H), sketch P4 (H, gather), sketch
// single pass (3 H, gather); vectors: P2 (H [D2] H, tile D), P4 (H, y epilogue).
enum SColProg : int { SC_FIRST = 0, SC_MID = 1, SC_LAST = 2, SC_SINGLE = 3, SC_VMID = 4, SC_VLAST = 5 };

template <int LS>
inline cudaError_t launch_scol_prog(int prog, const ColParams& p, int sms, cudaStream_t s) {
  switch (prog) {
    case SC_FIRST: return launch_scol<LS, 1, 1, false, SD_ROW, EPI_STORE>(p, sms, s);
    case SC_MID: return launch_scol<LS, 2, 2, true, SD_ROW, EPI_STORE>(p, sms, s);
    case SC_LAST: return launch_scol<LS, 1, 0, false, SD_ROW, EPI_GATHER>(p, sms, s);
    case SC_SINGLE: return launch_scol<LS, 3, 7, false, SD_ROW, EPI_GATHER>(p, sms, s);
    case SC_VMID: return launch_scol<LS, 2, 2, true, SD_TILE, EPI_STORE>(p, sms, s);
    case SC_VLAST: return launch_scol<LS, 1, 0, false, SD_ROW, EPI_Y>(p, sms, s);
  }
  return cudaErrorInvalidValue;
}

inline cudaError_t launch_scol_ls(int ls, int prog, const ColParams& p, int sms, cudaStream_t s) {
  switch (ls) {
    case 2: return launch_scol_prog<2>(prog, p, sms, s);
    case 3: return launch_scol_prog<3>(prog, p, sms, s);
    case 4: return launch_scol_prog<4>(prog, p, sms, s);
    case 5: return launch_scol_prog<5>(prog, p, sms, s);
    case 6: return launch_scol_prog<6>(prog, p, sms, s);
    case 7: return launch_scol_prog<7>(prog, p, sms, s);
    case 8: return launch_scol_prog<8>(prog, p, sms, s);
    case 9: return launch_scol_prog<9>(prog, p, sms, s);
  }
  return cudaErrorInvalidValue;
}

template <int LR, int LT, int PROG>
inline cudaError_t launch_srow(const RowParams2& p, int sms, cudaStream_t s) {
  using C = VCfg<LR, LT>;
  auto kern = rowpass_staged_kernel<LR, LT, PROG>;
  constexpr size_t smem = sizeof(float) * C::N * (RowCfg<PROG>::DIRECT ? (SPN_ROW_STAGE_D && PROG == RP_MID ? 2 : 1) : 2);
  static int occ = 0;
  if (occ == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::T, smem);
    if (e != cudaSuccess) return e;
    occ = std::max(occ, 1);
  }
  const int64_t items = p.nvec * p.nseg;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(items, int64_t(sms) * occ));
  return launch_pdl(true, kern, static_cast<unsigned>(grid), C::T, smem, s, p);
}

// threads per row segment: one warp up to 2^11 floats, two warps (R = T = 64) at 2^12
inline int row_lt(int lc) { return lc >= 12 ? 6 : 5; }

inline cudaError_t launch_srow_lc(int lc, int prog, const RowParams2& p, int sms, cudaStream_t s) {
  if (lc == 10) {
    if (prog == RP_FIRST) return launch_srow<5, 5, RP_FIRST>(p, sms, s);
    if (prog == RP_MID) return launch_srow<5, 5, RP_MID>(p, sms, s);
    return launch_srow<5, 5, RP_LAST>(p, sms, s);
  }
  if (lc == 11) {
    if (prog == RP_FIRST) return launch_srow<6, 5, RP_FIRST>(p, sms, s);
    if (prog == RP_MID) return launch_srow<6, 5, RP_MID>(p, sms, s);
    return launch_srow<6, 5, RP_LAST>(p, sms, s);
  }
  if (lc == 12) {
    if (prog == RP_FIRST) return launch_srow<6, 6, RP_FIRST>(p, sms, s);
    if (prog == RP_MID) return launch_srow<6, 6, RP_MID>(p, sms, s);
    return launch_srow<6, 6, RP_LAST>(p, sms, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace spn
