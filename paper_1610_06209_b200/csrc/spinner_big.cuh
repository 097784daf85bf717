// Multi-pass split FWHT for transforms that do not fit one CTA, and the
// strided-axis sketch.
//
// H_n factors over any partition of the index bits: with i = r*C + c,
//   H_n = (H_R (x) I_C)(I_R (x) H_C)      and the two factors commute,
// so   H D3 H D2 H D1  =  [Hc3] [Hr3] D3 [Hr2] [Hc2] D2 [Hc1] [Hr1] D1
// regroups into 4 passes instead of 6 (SURVEY.md §7 hard part 2):
//
//   contiguous vectors (n = 2^15..2^20, C = 1024 contiguous "columns"):
//     P1 col-pass  D1, Hr            (r bits, stride C; lanes over contiguous c)
//     P2 row-pass  Hc, D2, Hc        (c bits, one warp per 1024-float segment)
//     P3 col-pass  Hr, D3, Hr
//     P4 row-pass  Hc, epilogue (scale, ReLU, truncate to m, store y)
//   strided sketch of a row-major A[N][d] along N (SketchOperator, newton_sketch.cpp:74-101):
//     P1 (low bits)  D1, H          P2 (high bits) H, D2, H
//     P3 (low bits)  H, D3, H       P4 (high bits) H, gather rows P -> out
// Intermediates live in a workspace sized so a group's working set stays in L2
// (vectors in groups of ~32 MB, sketch columns in groups of ~32 MB).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <mutex>
#include <utility>
#include <vector>

#include "../../include/spinners_b200.h"
#include "errors.hpp"
#include "host_params.hpp"
#include "spinner_vec.cuh"

namespace spn {

// ------------------------------------------------------------- column pass kernel
// A tile is 2^LS "rows" (the transformed sub-index s) x 32 contiguous columns.
// Thread (warp w, lane) holds column col0+lane and R = 2^LR rows:
//   layout A: s = w*R + j      layout B: s = j*W + w
// Loads/stores are 128-B coalesced in both layouts (lanes = columns); the
// transpose goes through smem[s][32] (bank = lane: conflict free).  The pass
// program (number of H parts, where the diagonals go, start layout, epilogue) is
// a template so every address and layout decision folds at compile time; element
// addresses are tile-uniform 64-bit bases + one 32-bit IMAD per element.

template <int LS_>
struct ColCfg {
  static constexpr int LS = LS_;
  static constexpr int LR = LS < 5 ? LS : 5;  // 32 rows per thread
  static constexpr int LW = LS - LR;          // <= 32 warps
  static constexpr int R = 1 << LR, W = 1 << LW, S = 1 << LS;
  static constexpr int THREADS = 32 * W;
  // 1024 resident threads/SM -> <= 64 regs; single-warp tiles get 128 regs (16 CTAs)
  static constexpr int MIN_CTAS = W == 1 ? 16 : (1024 / THREADS > 0 ? 1024 / THREADS : 1);
  static constexpr size_t SMEM = W > 1 ? sizeof(float) * S * 32 : 16;
};

enum DMode : int { DM_PER_ROW = 0, DM_PER_ELEM = 1 };

struct ColParams {
  const float* src;
  int64_t src_ld, src_vstride, src_valid;  // element (v,e,col) valid iff e*src_ld+col < src_valid
  float* dst;
  int64_t dst_ld, dst_vstride;
  int64_t ncols, nstripes;
  int s0;                // bit position of the transformed sub-index inside e
  int64_t nhi, nlo, nvec;
  const float* dd[3];    // D applied before part p (DMASK bit p)
  int64_t d_ld;          // DM_PER_ELEM: dd[p][e*d_ld + col];  DM_PER_ROW: dd[p][(lo*nhi + hi)*S + s]
  const int32_t* rowmap; // GATHER: output row of e, or -1
  int64_t ld_out;
  float cscale;
  int64_t rows_valid;    // EPI_Y: flat elements < rows_valid are stored
  int relu;
  int discard_src;       // EPI_GATHER over a dead workspace: drop each source row's L2 line after the
                         // tile is read (discard.global.L2: no write-back of the workspace to HBM)
  int pdl;               // launch with programmatic dependent launch (vector path: c5 1.366 -> 1.323 ms;
                         // the sketch path measured slightly slower with it, so it stays off there)
  // filled by set_tiling(): fast division by nstripes, log2 of nlo / nhi (powers of two)
  uint32_t fd_m, fd_l;
  int lg_nlo, lg_nhi;
};

// Host: magic numbers for fdiv() and the pow2 logs used by the staged kernels' tile decode.
inline void set_tiling(ColParams& p) {
  const uint32_t d = static_cast<uint32_t>(p.nstripes);
  uint32_t l = 0;
  while ((uint64_t(1) << l) < d) ++l;
  p.fd_l = l;
  p.fd_m = d <= 1 ? 0u : static_cast<uint32_t>(((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1);
  auto lg = [](int64_t x) { int k = 0; while ((int64_t(1) << k) < x) ++k; return k; };
  p.lg_nlo = lg(p.nlo);
  p.lg_nhi = lg(p.nhi);
}

template <int LS>
__device__ __forceinline__ void col_xpose(float (&r)[ColCfg<LS>::R], float* sm, int w, int lane,
                                          bool a_to_b) {
  using C = ColCfg<LS>;
#pragma unroll
  for (int j = 0; j < C::R; ++j) {
    const int s = a_to_b ? (w * C::R + j) : (j * C::W + w);
    sm[s * 32 + lane] = r[j];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < C::R; ++j) {
    const int s = a_to_b ? (j * C::W + w) : (w * C::R + j);
    r[j] = sm[s * 32 + lane];
  }
  __syncthreads();
}

// s held in register j for a layout (compile-time after unrolling).
template <class C>
__device__ __forceinline__ uint32_t col_s(bool lay_b, int w, int j) {
  return lay_b ? (uint32_t)(j * C::W + w) : (uint32_t)(w * C::R + j);
}

template <int LS, int NPARTS, int DMASK, bool START_B, int DMODE, bool GATHER>
__global__ void __launch_bounds__(ColCfg<LS>::THREADS, ColCfg<LS>::MIN_CTAS) colpass_kernel(const ColParams p) {
  using C = ColCfg<LS>;
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t tiles = p.nvec * p.nhi * p.nlo * p.nstripes;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    int64_t tmp = tile;
    const int64_t cs = tmp % p.nstripes;
    tmp /= p.nstripes;
    const int64_t lo = tmp % p.nlo;
    tmp /= p.nlo;
    const int64_t hi = tmp % p.nhi;
    const int64_t v = tmp / p.nhi;
    const bool colok = cs * 32 + lane < p.ncols;
    const int64_t e0 = (hi << (p.s0 + LS)) + lo;

    float r[C::R];
    {
      const float* sb = p.src + v * p.src_vstride + e0 * p.src_ld + cs * 32;
      const uint32_t step = (uint32_t)(p.src_ld << p.s0);
      const int64_t lim = p.src_valid - (e0 * p.src_ld + cs * 32);
      constexpr bool LB = START_B && C::W > 1;
      if (colok && lim >= (int64_t)C::S * step) {
#pragma unroll
        for (int j = 0; j < C::R; ++j) r[j] = __ldg(sb + (col_s<C>(LB, w, j) * step + lane));
      } else {
#pragma unroll
        for (int j = 0; j < C::R; ++j) {
          const uint32_t off = col_s<C>(LB, w, j) * step + lane;
          r[j] = (colok && (int64_t)off < lim) ? __ldg(sb + off) : 0.0f;
        }
      }
    }
#pragma unroll
    for (int part = 0; part < NPARTS; ++part) {
      const bool lay_b = C::W > 1 && (START_B ^ ((part & 1) != 0));
      if ((DMASK >> part) & 1) {
        const float* D = p.dd[part];
        if constexpr (DMODE == DM_PER_ELEM) {
          const float* db = D + e0 * p.d_ld + cs * 32;
          const uint32_t dstep = (uint32_t)(p.d_ld << p.s0);
          if (colok) {
            // 8 loads in flight at a time: all R at once would need R more registers
#pragma unroll
            for (int q = 0; q < C::R; q += 8) {
#pragma unroll
              for (int j = q; j < q + 8 && j < C::R; ++j) r[j] *= __ldg(db + (col_s<C>(lay_b, w, j) * dstep + lane));
              asm volatile("" ::: "memory");
            }
          }
        } else {
          const float* Dt = D + (lo * p.nhi + hi) * C::S;
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
            for (int j = 0; j < C::R; ++j) r[j] *= __ldg(Dt + col_s<C>(lay_b, w, j));
          }
        }
      }
      // one full H over the LS bits of s, switching layout
      reg_fwht<C::R, 0, C::LR>(r);
      if constexpr (C::W > 1) {
        col_xpose<LS>(r, smem, w, lane, !lay_b);
        if (!lay_b)
          reg_fwht<C::R, C::LR - C::LW, C::LR>(r);
        else
          reg_fwht<C::R, 0, C::LW>(r);
      }
    }
    constexpr bool END_B = C::W > 1 && (START_B ^ ((NPARTS & 1) != 0));
    if constexpr (GATHER) {
      const int32_t* rm = p.rowmap + e0;
      const float* unused = nullptr;
      (void)unused;
#pragma unroll
      for (int j = 0; j < C::R; ++j) {
        const int32_t orow = __ldg(rm + ((int64_t)col_s<C>(END_B, w, j) << p.s0));
        if (colok && orow >= 0) __stcs(p.dst + (int64_t)orow * p.ld_out + cs * 32 + lane, r[j] * p.cscale);
      }
    } else {
      float* db = p.dst + v * p.dst_vstride + e0 * p.dst_ld + cs * 32;
      const uint32_t ostep = (uint32_t)(p.dst_ld << p.s0);
      if (colok) {
#pragma unroll
        for (int j = 0; j < C::R; ++j) db[col_s<C>(END_B, w, j) * ostep + lane] = r[j];
      }
    }
  }
}

// --------------------------------------------------------------- row pass kernel
// One warp per 1024-float segment of a vector (VCfg<5,5> layouts of spinner_vec.cuh).
struct RowParams {
  float* buf;            // [nvec][vstride] in place (mid pass) / source (last pass)
  int64_t vstride, nseg, nvec;
  const float* d_mid;    // mid pass: D2 per segment in layout-A float format ([seg][8][32][4])
  float* y;
  int64_t ld_y, rows_valid;
  float c;
  int relu;
};

template <bool LAST>
__global__ void __launch_bounds__(256, 3) rowpass_kernel(const RowParams p) {
  using C = VCfg<5, 5>;
  __shared__ __align__(16) float smem[8 * 1024];
  const int t = threadIdx.x & 31, g = threadIdx.x >> 5;
  float* sm = smem + g * 1024;
  const int64_t items = p.nvec * p.nseg;
  for (int64_t base = (int64_t)blockIdx.x * 8; base < items; base += (int64_t)gridDim.x * 8) {
    const int64_t item = base + g;
    if (item >= items) continue;  // warp-uniform: one segment per warp, warp-level syncs only
    const int64_t v = item / p.nseg, seg = item - v * p.nseg;
    float* row = p.buf + v * p.vstride + seg * 1024;
    float r[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = row[j * 32 + t];
    fwht_B_to_A<C>(r, sm, t);
    if constexpr (!LAST) {
      const float4* f = reinterpret_cast<const float4*>(p.d_mid + seg * 1024);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 dv = __ldg(f + q * 32 + t);
        r[4 * q] *= dv.x;
        r[4 * q + 1] *= dv.y;
        r[4 * q + 2] *= dv.z;
        r[4 * q + 3] *= dv.w;
      }
      fwht_A_to_B<C>(r, sm, t);
#pragma unroll
      for (int j = 0; j < 32; ++j) row[j * 32 + t] = r[j];
    } else {
      xpose_A_to_B<C>(r, sm, t);
      float* yrow = p.y + v * p.ld_y + seg * 1024;
      const bool all = seg * 1024 + 1024 <= p.rows_valid;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float o = r[j] * p.c;
        if (p.relu) o = fmaxf(o, 0.0f);
        if (all || seg * 1024 + j * 32 + t < p.rows_valid) __stcs(yrow + j * 32 + t, o);
      }
    }
  }
}

// ------------------------------------------------------------------- host side

template <int LS, int NPARTS, int DMASK, bool START_B, int DMODE, bool GATHER>
inline cudaError_t launch_col(const ColParams& p, int sms, cudaStream_t s) {
  using C = ColCfg<LS>;
  auto kern = colpass_kernel<LS, NPARTS, DMASK, START_B, DMODE, GATHER>;
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
  kern<<<static_cast<unsigned>(grid), C::THREADS, C::SMEM, s>>>(p);
  return cudaGetLastError();
}

// The pass programs used by the drivers below.
enum ColProg : int {
  CP_FIRST = 0,   // [D] H            start A          (vector P1 / sketch P1)
  CP_MID = 1,     // H [D] H          start B          (vector P3 / sketch P2, P3)
  CP_LAST = 2,    // H, gather rows   start A          (sketch P4)
  CP_SINGLE = 3,  // [D]H[D]H[D]H, gather             (sketch with n <= 2^10)
};

template <int LS>
inline cudaError_t launch_col_prog(int prog, int dmode, const ColParams& p, int sms, cudaStream_t s) {
  if (dmode == DM_PER_ELEM) {
    if (prog == CP_FIRST) return launch_col<LS, 1, 1, false, DM_PER_ELEM, false>(p, sms, s);
    if (prog == CP_MID) return launch_col<LS, 2, 2, true, DM_PER_ELEM, false>(p, sms, s);
    return cudaErrorInvalidValue;
  }
  switch (prog) {
    case CP_FIRST: return launch_col<LS, 1, 1, false, DM_PER_ROW, false>(p, sms, s);
    case CP_MID: return launch_col<LS, 2, 2, true, DM_PER_ROW, false>(p, sms, s);
    case CP_LAST: return launch_col<LS, 1, 0, false, DM_PER_ROW, true>(p, sms, s);
    default: return launch_col<LS, 3, 7, false, DM_PER_ROW, true>(p, sms, s);
  }
}

inline cudaError_t launch_col_ls(int ls, int prog, int dmode, const ColParams& p, int sms, cudaStream_t s) {
  switch (ls) {
    case 1: return launch_col_prog<1>(prog, dmode, p, sms, s);
    case 2: return launch_col_prog<2>(prog, dmode, p, sms, s);
    case 3: return launch_col_prog<3>(prog, dmode, p, sms, s);
    case 4: return launch_col_prog<4>(prog, dmode, p, sms, s);
    case 5: return launch_col_prog<5>(prog, dmode, p, sms, s);
    case 6: return launch_col_prog<6>(prog, dmode, p, sms, s);
    case 7: return launch_col_prog<7>(prog, dmode, p, sms, s);
    case 8: return launch_col_prog<8>(prog, dmode, p, sms, s);
    case 9: return launch_col_prog<9>(prog, dmode, p, sms, s);
    case 10: return launch_col_prog<10>(prog, dmode, p, sms, s);
  }
  return cudaErrorInvalidValue;
}

template <bool LAST>
inline cudaError_t launch_row(const RowParams& p, int sms, cudaStream_t s) {
  static int occ = 0;
  if (occ == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rowpass_kernel<LAST>, 256, 0);
    if (e != cudaSuccess) return e;
    occ = std::max(occ, 1);
  }
  const int64_t ctas = (p.nvec * p.nseg + 7) / 8;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ctas, int64_t(sms) * occ));
  rowpass_kernel<LAST><<<static_cast<unsigned>(grid), 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace spn
#include "spinner_pass.cuh"
#include "spinner_tma.cuh"
#include "sketch_flow.cuh"
namespace spn {

// L2-resident working set per pass group: 24 MB for the vector passes (c5: 1.275 vs
// 1.316 ms at 32 MB), 32 MB for the sketch's column groups (c4: 0.197 ms; 16/48/64 MB
// slower).  SPN_GROUP_MB overrides both (tuning).
inline int64_t group_bytes(bool sketch = false) {
  static const int64_t env = [] {
    const char* e = std::getenv("SPN_GROUP_MB");
    const int64_t mb = e ? std::atoll(e) : 0;
    return mb > 0 ? (mb << 20) : int64_t(0);
  }();
  if (env) return env;
  return sketch ? (int64_t(32) << 20) : (int64_t(24) << 20);
}

// Stream-ordered scratch (cudaMallocFromPoolAsync / cudaFreeAsync) from one pool per device
// that keeps its memory (release threshold = max): per-call workspaces cost no cudaMalloc /
// device-synchronising cudaFree, which matters when plans are short-lived (a fresh sketch
// per Newton iteration).
inline cudaMemPool_t scratch_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&pools[dev], &props) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    uint64_t keep = ~uint64_t(0);
    cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
  }
  return pools[dev];
}

// Per-device library streams: the multi-pass drivers' group streams (shared by every plan on
// the device — plans are short-lived, e.g. a fresh sketch per Newton iteration, and stream
// creation / destruction would cost more than the sketch) and the stream that returns plan
// memory to the pool.
inline cudaStream_t device_stream(int slot) {
  static std::mutex mu;
  static cudaStream_t ss[64][8] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || slot < 0 || slot >= 8) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!ss[dev][slot]) {
    // slot 6 (plan-time realisation) runs at the highest priority: its two CTAs take the
    // first SM slots that free up between the running passes' CTAs
    int lo = 0, hi = 0;
    if (slot != 6 || cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) hi = 0;
    if (cudaStreamCreateWithPriority(&ss[dev][slot], cudaStreamNonBlocking, hi) != cudaSuccess) {
      cudaGetLastError();
      ss[dev][slot] = nullptr;
    }
  }
  return ss[dev][slot];
}
constexpr int kFreeStreamSlot = 7;
constexpr int kRealiseStreamSlot = 6;

inline cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t s) {
  cudaMemPool_t pool = scratch_pool();
  if (!pool) return cudaErrorMemoryAllocation;
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

// Device realisation of a Rademacher (HD3) block's diagonals with the reference's own
// generator (proj/src/spinner.cpp:137-151; common.hpp:61-92): std::mt19937_64 seeded with
// mix_seed(spec_seed, 1) gives D1 then D2 (n draws each), mix_seed(spec_seed, 2) gives D3,
// and rademacher(u) = (u & 1) ? +1 : -1 (common.hpp:86).  One CTA per stream, one thread per
// state word; each 312-word twist runs as its two data-parallel halves (i < 156 reads only
// old words, i >= 156 reads the new words i - 156, and i = 311 the new word 0 — the
// sequential order of the library engine) into the other half of a ping-pong state (two
// barriers per twist), then every thread tempers and emits its word.  Bit-exact with the
// host realisation (tests/test_gpu_parity.py::test_sketch_device_realisation_bit_exact),
// stream-ordered, and launched at plan creation, so a fresh sketch per Newton iteration
// costs no host time.
// Outputs are the sketch layouts: D1, D3 natural, D2 transposed for the high-bit pass
// (f[lo * 2^lsb + s] = D2[(s << lsa) + lo], see build_sketch).
__global__ void __launch_bounds__(320) mt_rademacher_sketch_kernel(uint64_t seed_front, uint64_t seed_tail,
                                                                   int64_t n, int lsa, int lsb, float* d1,
                                                                   float* d2t, float* d3) {
  constexpr int N = 312, M = 156;
  constexpr uint64_t A = 0xB5026F5AA96619E9ULL, UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  __shared__ uint64_t buf[2][N];  // ping-pong states: a twist reads one and writes the other
  const bool front = blockIdx.x == 0;
  const int t = threadIdx.x;  // word t of the state
  if (t == 0) {
    buf[0][0] = front ? seed_front : seed_tail;
    for (int i = 1; i < N; ++i)
      buf[0][i] = 6364136223846793005ULL * (buf[0][i - 1] ^ (buf[0][i - 1] >> 62)) + uint64_t(i);
  }
  __syncthreads();
  const int64_t draws = front ? 2 * n : n;
  const int64_t lo_mask = (int64_t(1) << lsa) - 1;
  int c = 0;
  for (int64_t base = 0; base < draws; base += N, c ^= 1) {
    const uint64_t* cur = buf[c];
    uint64_t* nxt = buf[c ^ 1];
    if (t < M) {  // words 0..155: old words only
      const uint64_t y = (cur[t] & UM) | (cur[t + 1] & LM);
      nxt[t] = cur[t + M] ^ (y >> 1) ^ ((0 - (y & 1)) & A);
    }
    __syncthreads();
    if (t >= M && t < N) {  // words 156..311: new words t - 156 (and new word 0 for t = 311)
      const uint64_t y = (cur[t] & UM) | ((t + 1 < N ? cur[t + 1] : nxt[0]) & LM);
      nxt[t] = nxt[t - M] ^ (y >> 1) ^ ((0 - (y & 1)) & A);
    }
    __syncthreads();
    // temper + emit word t (the next twist writes the other buffer)
    const int64_t k = base + t;
    if (t < N && k < draws) {
      uint64_t y = nxt[t];
      y ^= (y >> 29) & 0x5555555555555555ULL;
      y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
      y ^= (y << 37) & 0xFFF7EEE000000000ULL;
      y ^= y >> 43;
      const float r = (y & 1) ? 1.0f : -1.0f;
      if (!front) {
        d3[k] = r;
      } else if (k < n) {
        d1[k] = r;
      } else {
        const int64_t e = k - n;
        d2t[lsb > 0 ? (e & lo_mask) * (int64_t(1) << lsb) + (e >> lsa) : e] = r;
      }
    }
  }
}

// rowmap[i] = i for i < m (the reference's P = first m rows), -1 beyond
__global__ void rowmap_first_kernel(int32_t* map, int64_t nn, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x)
    map[i] = i < m ? static_cast<int32_t>(i) : -1;
}

// ------------------------------------------------ row epilogues for n > 2^14 (hash / embed)
// The multi-pass path produces y = s * first_m(H D3 H D2 H D1 x) per block; these kernels turn
// the stacked rows into the reference's hash ids and features (one CTA per row, coalesced).

// signed argmax of a row (lsh.cpp:9-21): max |y|, ties to the smallest index, sign(0) = +1;
// id = index + (y < 0 ? k : 0), stored at ids[v * ld_ids + col]
__global__ void __launch_bounds__(256) rows_signed_argmax_kernel(const float* __restrict__ y, int64_t ld_y,
                                                                 int64_t k, int64_t batch, int32_t* __restrict__ ids,
                                                                 int64_t ld_ids, int64_t col) {
  __shared__ float sa[8], sv[8];
  __shared__ int64_t si[8];
  for (int64_t v = blockIdx.x; v < batch; v += gridDim.x) {
    const float* row = y + v * ld_y;
    float ba = -1.0f, bv = 0.0f;
    int64_t bi = INT64_MAX;
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) {  // increasing i: strict '>' keeps the first
      const float val = row[i], a = fabsf(val);
      if (a > ba) {
        ba = a;
        bi = i;
        bv = val;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float oa = __shfl_xor_sync(0xffffffffu, ba, off), ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (oa > ba || (oa == ba && oi < bi)) {
        ba = oa;
        bi = oi;
        bv = ov;
      }
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
      sa[w] = ba;
      si[w] = bi;
      sv[w] = bv;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
        if (sa[q] > ba || (sa[q] == ba && si[q] < bi)) {
          ba = sa[q];
          bi = si[q];
          bv = sv[q];
        }
      ids[v * ld_ids + col] = static_cast<int32_t>(bi + (bv < 0.0f ? k : 0));
    }
    __syncthreads();
  }
}

// embed epilogue in place on rows whose first k entries hold z (kernels.cpp:17-36):
// Gaussian: out[i] = norm cos(z_i / sigma), out[k + i] = norm sin(z_i / sigma); angular:
// out[i] = sign(z_i), sign(0) = +1
__global__ void __launch_bounds__(256) rows_embed_kernel(float* __restrict__ out, int64_t ld_out, int64_t k,
                                                         int64_t batch, int gaussian, float inv_sigma, float norm) {
  for (int64_t v = blockIdx.x; v < batch; v += gridDim.x) {
    float* row = out + v * ld_out;
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) {
      const float z = row[i];
      if (gaussian) {
        float sn, cs;
        sincosf(z * inv_sigma, &sn, &cs);
        row[i] = norm * cs;
        row[k + i] = norm * sn;
      } else {
        row[i] = z < 0.0f ? -1.0f : 1.0f;
      }
    }
  }
}

struct Scratch {  // freed (stream-ordered) on `s` when the scope ends
  void* p = nullptr;
  cudaStream_t s = nullptr;
  cudaError_t alloc(size_t bytes, cudaStream_t st) {
    s = st;
    cudaMemPool_t pool = scratch_pool();
    if (!pool) return cudaErrorMemoryAllocation;
    return cudaMallocFromPoolAsync(&p, bytes, pool, st);
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
};

inline int ilog2_i(int64_t n) {
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  return l;
}

struct BigPlan {
  // contiguous-vector path (n > 2^14): fp32 diagonals [blocks][n]
  int64_t n = 0, tb = 0;
  int L = 0;
  float* dnat[3] = {nullptr, nullptr, nullptr};
  float* drow2 = nullptr;   // D2 in the 1024-wide row-pass layout
  float* srow1 = nullptr;   // staged schedule: D1 / D3 per row segment, D2 per column tile
  float* srow3 = nullptr;
  float* stile2 = nullptr;
  // sketch path (lazy)
  std::mutex mu;
  bool sk_ready = false;
  int sk_lsa = 0, sk_lsb = 0;
  float* sk_d[3] = {nullptr, nullptr, nullptr};
  // Rademacher (HD3) single-block plans realise their sketch diagonals on the device
  // (mt_rademacher_sketch_kernel) instead of uploading host draws
  bool dev_rad = false;
  uint64_t dev_seed = 0;  // spec seed of the block
  // sk_d, sk_d1s and rowmap come from the stream-ordered pool; they go back to it after the
  // last call on every stream that used them (uses), without a device-wide cudaFree
  // synchronisation.  ev_ready marks the device realisation, ev_map the last row-map fill;
  // every call waits for both on its own stream (they may have been made on other streams).
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;
  cudaEvent_t ev_ready = nullptr;  // the device realisation (made on the realisation stream)
  cudaEvent_t ev_map = nullptr;    // the last row-map fill (made on the calling stream)
  cudaError_t note_use(cudaStream_t s) {
    for (auto& u : uses)
      if (u.first == s) return cudaEventRecord(u.second, s);
    cudaEvent_t e = nullptr;
    cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (r != cudaSuccess) return r;
    uses.emplace_back(s, e);
    return cudaEventRecord(e, s);
  }
  cudaError_t wait_uses(cudaStream_t s) {
    for (auto& u : uses)
      if (cudaError_t r = cudaStreamWaitEvent(s, u.second, 0)) return r;
    return cudaSuccess;
  }
  static cudaError_t mark(cudaEvent_t* ev, cudaStream_t s) {
    cudaError_t r = *ev ? cudaSuccess : cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    return r == cudaSuccess ? cudaEventRecord(*ev, s) : r;
  }
  // make s wait for the realisation and the current row map, wherever they were made
  cudaError_t wait_ready(cudaStream_t s) {
    cudaError_t r = cudaSuccess;
    if (ev_ready) r = cudaStreamWaitEvent(s, ev_ready, 0);
    if (r == cudaSuccess && ev_map) r = cudaStreamWaitEvent(s, ev_map, 0);
    return r;
  }
  // scratch
  float* work = nullptr;
  size_t work_bytes = 0;
  int32_t* rowmap = nullptr;
  std::vector<int64_t> rowmap_key;
  // groups alternate between two internal streams so one group's pass tail overlaps the
  // next group's work (each pass is a full-GPU persistent kernel; fill/drain dominate
  // otherwise).  Forked from / joined back into the caller's stream with events.  The
  // streams are the device's library streams (device_stream), shared by all plans.
  static constexpr int kMaxStreams = 4;
  cudaStream_t ss[kMaxStreams] = {};
  cudaEvent_t evf = nullptr, evj[kMaxStreams] = {};
  int64_t rowmap_m = -1;

  void release() {
    for (auto*& q : dnat) {
      if (q) cudaFree(q);
      q = nullptr;
    }
    {
      cudaStream_t fs = device_stream(kFreeStreamSlot);
      if (fs) {
        wait_uses(fs);
        wait_ready(fs);
      }
      auto pfree = [&](void* q) {
        if (!q) return;
        if (!fs || cudaFreeAsync(q, fs) != cudaSuccess) cudaFree(q);
      };
      for (auto*& q : sk_d) {
        pfree(q);
        q = nullptr;
      }
      pfree(rowmap);
      rowmap = nullptr;
      for (auto& u : uses) cudaEventDestroy(u.second);
      uses.clear();
      if (ev_ready) cudaEventDestroy(ev_ready);
      if (ev_map) cudaEventDestroy(ev_map);
      ev_ready = ev_map = nullptr;
    }
    if (drow2) cudaFree(drow2);
    for (float** q : {&srow1, &srow3, &stile2}) {
      if (*q) cudaFree(*q);
      *q = nullptr;
    }
    if (work) cudaFree(work);
    if (evf) cudaEventDestroy(evf);
    for (auto& q : evj)
      if (q) cudaEventDestroy(q);
    drow2 = nullptr;
    work = nullptr;
    rowmap = nullptr;
  }

  static spn_status err(cudaError_t e, const char* what) { return cuda_error(e, what); }

  // number of group streams (default 2; SPN_STREAMS overrides, 1..4)
  static int nstreams() {
    static const int v = [] {
      const char* e = std::getenv("SPN_STREAMS");
      const int k = e ? std::atoi(e) : 2;
      return k < 1 ? 1 : (k > kMaxStreams ? kMaxStreams : k);
    }();
    return v;
  }

  spn_status fork(cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < nstreams() && e == cudaSuccess; ++i) {
      if (!ss[i]) ss[i] = device_stream(i);
      if (!ss[i]) e = cudaErrorInvalidResourceHandle;
      if (e == cudaSuccess && !evj[i]) e = cudaEventCreateWithFlags(&evj[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess && !evf) e = cudaEventCreateWithFlags(&evf, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(evf, s);
    for (int i = 0; i < nstreams() && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(ss[i], evf, 0);
    return e == cudaSuccess ? SPN_OK : err(e, "fork streams");
  }
  spn_status join(cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < nstreams() && e == cudaSuccess; ++i) {
      e = cudaEventRecord(evj[i], ss[i]);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s, evj[i], 0);
    }
    return e == cudaSuccess ? SPN_OK : err(e, "join streams");
  }

  spn_status ensure_work(size_t bytes) {
    if (work_bytes >= bytes) return SPN_OK;
    if (work) cudaFree(work);
    work = nullptr;
    work_bytes = 0;
    cudaError_t e = cudaMalloc(&work, bytes);
    if (e != cudaSuccess) return err(e, "workspace");
    work_bytes = bytes;
    return SPN_OK;
  }

  // row-pass width for the staged schedule: C = 2^lc contiguous floats, lc = max(10, L-8)
  // (<= 12), so the column pass covers <= 8 bits: 32 KB tiles, 256-thread CTAs, two CTAs
  // per SM (c5: 1.464 vs 1.519 ms with lc = L-9 and 64 KB tiles).  SPN_LC_EXTRA shifts it.
  static int staged_lc(int L) {
    static const int extra = [] {
      const char* e = std::getenv("SPN_LC_EXTRA");
      return e ? std::atoi(e) : 0;
    }();
    int lc = (L - 8 > 10 ? L - 8 : 10) + extra;
    if (lc > 12) lc = 12;
    if (lc < 10) lc = 10;
    if (L - lc > 9) lc = L - 9;
    return lc;
  }

  static spn_status upload_f32(const std::vector<float>& f, float** dst) {
    cudaError_t e = cudaMalloc(dst, f.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(*dst, f.data(), f.size() * 4, cudaMemcpyHostToDevice);
    return e == cudaSuccess ? SPN_OK : err(e, "upload diagonals");
  }

  // D permuted per contiguous 2^lc segment into the layout-A float format of
  // VCfg<lc-lt, lt> (lt = log2 threads per segment: 5, or 6 for the two-warp 2^12 rows).
  static std::vector<float> row_perm(const std::vector<double>& d2, int64_t n, int64_t tb, int lc, int lt = 5) {
    const int64_t N = int64_t(1) << lc, T = int64_t(1) << lt, R = N / T;
    std::vector<float> f(static_cast<size_t>(tb * n));
    for (int64_t b = 0; b < tb; ++b)
      for (int64_t seg = 0; seg < n / N; ++seg)
        for (int64_t t = 0; t < T; ++t)
          for (int64_t j = 0; j < R; ++j) {
            const int64_t pos = ((j / 4) * T + t) * 4 + (j % 4);
            f[static_cast<size_t>(b * n + seg * N + pos)] =
                static_cast<float>(d2[static_cast<size_t>(b * n + seg * N + t * R + j)]);
          }
    return f;
  }

  // D permuted per column-pass tile for the staged schedule: tile = 32-column stripe cs of
  // the [2^lr][C] view, [cs][w][R/4][lane][4] with s = w*32 + 4q + k (layout A, R = 32).
  static std::vector<float> tile_perm(const std::vector<double>& d, int64_t n, int64_t tb, int lc) {
    const int64_t C = int64_t(1) << lc, S = n / C, R = S < 32 ? S : 32, W = S / R;
    std::vector<float> f(static_cast<size_t>(tb * n));
    for (int64_t b = 0; b < tb; ++b)
      for (int64_t cs = 0; cs < C / 32; ++cs)
        for (int64_t w = 0; w < W; ++w)
          for (int64_t q = 0; q < R / 4; ++q)
            for (int64_t lane = 0; lane < 32; ++lane)
              for (int64_t k = 0; k < 4; ++k) {
                const int64_t sidx = w * R + 4 * q + k;
                const int64_t pos = (((cs * W + w) * (R / 4) + q) * 32 + lane) * 4 + k;
                f[static_cast<size_t>(b * n + pos)] = static_cast<float>(d[static_cast<size_t>(b * n + sidx * C + cs * 32 + lane)]);
              }
    return f;
  }

  // The apply layouts are built on first use: sketch-only plans (a fresh SketchOperator per
  // Newton iteration, newton_sketch.cpp:155-157) never pay for them.
  const std::vector<double>* dsrc = nullptr;
  bool built = false;
  spn_status build(int64_t n_, int64_t tb_, const std::vector<double>* d, const int*) {
    n = n_;
    tb = tb_;
    L = ilog2_i(n);
    dsrc = d;
    return SPN_OK;
  }
  spn_status build_now() {
    if (built) return SPN_OK;
    const std::vector<double>* d = dsrc;
    std::vector<float> f(static_cast<size_t>(tb * n));
    for (int di = 0; di < 3; ++di) {
      for (size_t i = 0; i < f.size(); ++i) f[i] = static_cast<float>(d[di][i]);
      if (spn_status st = upload_f32(f, &dnat[di])) return st;
    }
    if (spn_status st = upload_f32(row_perm(d[1], n, tb, 10), &drow2)) return st;
    // staged (row-first) schedule: D1, D3 in the row passes, D2 in the column pass
    const int lc = staged_lc(L);
    if (spn_status st = upload_f32(row_perm(d[0], n, tb, lc, row_lt(lc)), &srow1)) return st;
    if (spn_status st = upload_f32(row_perm(d[2], n, tb, lc, row_lt(lc)), &srow3)) return st;
    if (spn_status st = upload_f32(tile_perm(d[1], n, tb, lc), &stile2)) return st;
    built = true;
    return SPN_OK;
  }

  // y = relu?(c * first rows of (H D3 H D2 H D1 x)) for every block (tables == 1).
  // tb0: first (table, block) diagonal set to use — table t of a multi-table plan is tb0 = t * blocks
  spn_status apply(const float* x, int64_t batch, int64_t ld_x, int64_t n_in, float* y, int64_t ld_y,
                   int relu, int64_t k, int64_t m, int64_t blocks, double c, int sms, cudaStream_t s0,
                   int64_t tb0 = 0) {
    if (batch == 0) return SPN_OK;
    std::lock_guard<std::mutex> lock(mu);
    if (spn_status st = build_now()) return st;
    auto al16 = [](const void* q, int64_t ld) { return (reinterpret_cast<uintptr_t>(q) % 16 == 0) && (ld % 4 == 0); };
    // vectors per group: working set ~32 MB (L2-resident passes)
    const int64_t G = std::max<int64_t>(1, std::min<int64_t>(batch, group_bytes() / (n * 4)));
    const bool in_place = blocks == 1 && m == n && k == n && al16(y, ld_y);
    if (!in_place) {
      spn_status st = ensure_work(static_cast<size_t>(nstreams() * G * n * 4));
      if (st) return st;
    }
    if (spn_status st = fork(s0)) return st;
    const bool staged = al16(x, ld_x);
    const int lc = staged ? staged_lc(L) : 10, lr = L - lc;
    const int64_t C = int64_t(1) << lc;
    for (int64_t b = 0; b < blocks; ++b) {
      const int64_t rows_valid = std::min(m, k - b * m);
      int64_t gi = 0;
      for (int64_t v0 = 0; v0 < batch; v0 += G, ++gi) {
        const int si = static_cast<int>(gi % nstreams());
        const cudaStream_t s = ss[si];
        const int64_t nv = std::min(G, batch - v0);
        float* W = in_place ? y + v0 * ld_y : work + si * G * n;
        const int64_t wstride = in_place ? ld_y : n;
        cudaError_t e;
        if (staged) {
          // row-first: P1 row (D1, Hc) | P2 col (Hr, D2, Hr) | P3 row (Hc, D3, Hc) | P4 col (Hr, y)
          RowParams2 rp{};
          rp.src = x + v0 * ld_x;
          rp.src_vstride = ld_x;
          rp.n_in = n_in;
          rp.dst = W;
          rp.dst_vstride = wstride;
          rp.nseg = n / C;
          rp.nvec = nv;
          rp.d = srow1 + (tb0 + b) * n;
          e = launch_srow_lc(lc, RP_FIRST, rp, sms, s);
          if (e != cudaSuccess) return err(e, "rowpass P1");
          ColParams cp{};
          cp.src = W;
          cp.src_ld = C;
          cp.src_vstride = wstride;
          cp.src_valid = n;
          cp.dst = W;
          cp.dst_ld = C;
          cp.dst_vstride = wstride;
          cp.ncols = C;
          cp.nstripes = C / 32;
          cp.s0 = 0;
          cp.nhi = 1;
          cp.nlo = 1;
          cp.nvec = nv;
          cp.pdl = 1;
          cp.dd[1] = stile2 + (tb0 + b) * n;
          const bool tma = lr >= 5 && al16(y, ld_y);
          e = tma ? launch_tcol_ls(lr, SC_VMID, cp, sms, s) : launch_scol_ls(lr, SC_VMID, cp, sms, s);
          if (e != cudaSuccess) return err(e, "colpass P2");
          rp.src = W;
          rp.src_vstride = wstride;
          rp.n_in = n;
          rp.d = srow3 + (tb0 + b) * n;
          e = launch_srow_lc(lc, RP_MID, rp, sms, s);
          if (e != cudaSuccess) return err(e, "rowpass P3");
          cp.dd[1] = nullptr;
          cp.dst = y + v0 * ld_y + b * m;
          cp.dst_vstride = ld_y;
          cp.rows_valid = rows_valid;
          cp.cscale = static_cast<float>(c);
          cp.relu = relu;
          e = tma ? launch_tcol_ls(lr, SC_VLAST, cp, sms, s) : launch_scol_ls(lr, SC_VLAST, cp, sms, s);
          if (e != cudaSuccess) return err(e, "colpass P4");
          continue;
        }
        ColParams cp{};
        cp.src = x + v0 * ld_x;
        cp.src_ld = C;
        cp.src_vstride = ld_x;
        cp.src_valid = n_in;
        cp.dst = W;
        cp.dst_ld = C;
        cp.dst_vstride = wstride;
        cp.ncols = C;
        cp.nstripes = C / 32;
        cp.s0 = 0;
        cp.nhi = 1;
        cp.nlo = 1;
        cp.nvec = nv;
        cp.dd[0] = dnat[0] + (tb0 + b) * n;
        cp.d_ld = C;
        e = launch_col_ls(lr, CP_FIRST, DM_PER_ELEM, cp, sms, s);  // P1: D1, Hr
        if (e != cudaSuccess) return err(e, "colpass P1");
        RowParams rp{};
        rp.buf = W;
        rp.vstride = wstride;
        rp.nseg = n / C;
        rp.nvec = nv;
        rp.d_mid = drow2 + (tb0 + b) * n;
        e = launch_row<false>(rp, sms, s);  // P2: Hc, D2, Hc
        if (e != cudaSuccess) return err(e, "rowpass P2");
        cp.src = W;
        cp.src_vstride = wstride;
        cp.src_valid = n;
        cp.dd[0] = nullptr;
        cp.dd[1] = dnat[2] + (tb0 + b) * n;
        e = launch_col_ls(lr, CP_MID, DM_PER_ELEM, cp, sms, s);  // P3: Hr, D3, Hr
        if (e != cudaSuccess) return err(e, "colpass P3");
        rp.y = y + v0 * ld_y + b * m;
        rp.ld_y = ld_y;
        rp.rows_valid = rows_valid;
        rp.c = static_cast<float>(c);
        rp.relu = relu;
        e = launch_row<true>(rp, sms, s);  // P4: Hc, scale, relu, store
        if (e != cudaSuccess) return err(e, "rowpass P4");
      }
    }
    return join(s0);
  }

  // Rademacher plans: realise the sketch diagonals at plan creation on the library's
  // realisation stream, so the draws overlap whatever the device is running (a Newton
  // solve creates the next iteration's sketch while the current step runs).
  spn_status prefetch_sketch(int64_t nn) {
    if (!dev_rad) return SPN_OK;
    std::lock_guard<std::mutex> lock(mu);
    cudaStream_t rs = device_stream(kRealiseStreamSlot);
    if (!rs) return err(cudaErrorInvalidResourceHandle, "realisation stream");
    return build_sketch(nn, nullptr, rs);
  }

  spn_status build_sketch(int64_t nn, const std::vector<double>* d, cudaStream_t s) {
    if (sk_ready) return SPN_OK;
    const int LL = ilog2_i(nn);
    if (LL <= 10) {
      sk_lsa = LL;
      sk_lsb = 0;
    } else {
      sk_lsa = (LL + 1) / 2;
      sk_lsb = LL / 2;
    }
    if (dev_rad) {
      cudaError_t e = cudaSuccess;
      for (int di = 0; di < 3 && e == cudaSuccess; ++di)
        e = pool_alloc(reinterpret_cast<void**>(&sk_d[di]), static_cast<size_t>(nn) * 4, s);
      if (e == cudaSuccess) {
        mt_rademacher_sketch_kernel<<<2, 320, 0, s>>>(mix_seed(dev_seed, 1), mix_seed(dev_seed, 2), nn, sk_lsa,
                                                      sk_lsb, sk_d[0], sk_d[1], sk_d[2]);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess) e = mark(&ev_ready, s);
      if (e != cudaSuccess) return err(e, "device realisation of the sketch diagonals");
      sk_ready = true;
      return SPN_OK;
    }
    std::vector<float> f(static_cast<size_t>(nn));
    for (int di = 0; di < 3; ++di) {
      const bool transposed = (di == 1 && sk_lsb > 0);  // D2 is applied in the high-bit pass
      if (transposed) {
        const int64_t nlo = int64_t(1) << sk_lsa, S = int64_t(1) << sk_lsb;
        for (int64_t lo = 0; lo < nlo; ++lo)
          for (int64_t s = 0; s < S; ++s) f[static_cast<size_t>(lo * S + s)] = static_cast<float>(d[di][static_cast<size_t>((s << sk_lsa) + lo)]);
      } else {
        for (int64_t i = 0; i < nn; ++i) f[static_cast<size_t>(i)] = static_cast<float>(d[di][static_cast<size_t>(i)]);
      }
      cudaError_t e = pool_alloc(reinterpret_cast<void**>(&sk_d[di]), f.size() * 4, s);
      if (e == cudaSuccess) e = cudaMemcpyAsync(sk_d[di], f.data(), f.size() * 4, cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // f is pageable and goes out of scope
      if (e != cudaSuccess) return err(e, "upload sketch diagonals");
    }
    sk_ready = true;
    return SPN_OK;
  }

  spn_status set_rowmap(int64_t nn, const int64_t* rows, int64_t m_out, cudaStream_t s) {
    std::vector<int64_t> key;
    if (rows) key.assign(rows, rows + m_out);
    if (rowmap && rowmap_m == m_out && key == rowmap_key) return SPN_OK;
    if (!rows) {  // P = first m_out rows: filled on the device, stream-ordered
      cudaError_t e = cudaSuccess;
      if (!rowmap) e = pool_alloc(reinterpret_cast<void**>(&rowmap), static_cast<size_t>(nn) * 4, s);
      else e = wait_uses(s);  // earlier calls (any stream) are done with the old map
      if (e == cudaSuccess) {
        rowmap_first_kernel<<<static_cast<unsigned>(std::min<int64_t>((nn + 255) / 256, 1024)), 256, 0, s>>>(
            rowmap, nn, m_out);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess) e = mark(&ev_map, s);
      if (e != cudaSuccess) return err(e, "row map");
      rowmap_key.clear();
      rowmap_m = m_out;
      return SPN_OK;
    }
    std::vector<int32_t> map(static_cast<size_t>(nn), -1);
    for (int64_t r = 0; r < m_out; ++r) {
      const int64_t i = rows ? rows[r] : r;
      if (map[static_cast<size_t>(i)] != -1) return set_error(SPN_EDIM, "sketch rows must be distinct");
      map[static_cast<size_t>(i)] = static_cast<int32_t>(r);
    }
    cudaError_t e = cudaSuccess;
    if (!rowmap) e = pool_alloc(reinterpret_cast<void**>(&rowmap), static_cast<size_t>(nn) * 4, s);
    else e = wait_uses(s);  // earlier calls (any stream) are done with the old map ...
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // ... once s is
    if (e == cudaSuccess) e = cudaMemcpy(rowmap, map.data(), map.size() * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return err(e, "row map");
    rowmap_key = std::move(key);
    rowmap_m = m_out;
    return SPN_OK;
  }
};

// D1 with a per-row scale folded in (the Newton step's B = diag(h) A, newton_sketch.cpp:63-72,
// sketched in the first pass without materialising B).
__global__ void scale_rows_kernel(const float* __restrict__ d1, const float* __restrict__ h, int64_t n_in,
                                  int64_t nn, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i < n_in ? d1[i] * h[i] : 0.0f;
}

inline spn_status sketch_run(int64_t nn, const std::vector<double>* d, const int* /*dsign*/,
                             const float* a, int64_t n_in, int64_t dcols, int64_t ld_a,
                             const int64_t* rows, int64_t m_out, double cscale, float* out,
                             int64_t ld_out, int sms, cudaStream_t s0, BigPlan* bp,
                             const float* row_scale = nullptr) {
  std::lock_guard<std::mutex> lock(bp->mu);
  if (spn_status st = bp->build_sketch(nn, d, s0)) return st;
  if (spn_status st = bp->set_rowmap(nn, rows, m_out, s0)) return st;
  // the realisation (realisation stream) and the row map (possibly another caller stream)
  if (cudaError_t e = bp->wait_ready(s0)) return BigPlan::err(e, "sketch ready");
  const float* d1 = bp->sk_d[0];
  // D1 times the row scale: per call, from the stream-ordered pool on s0 (freed on s0 after the
  // join), so calls on different streams sharing this plan never overwrite each other's copy
  Scratch d1s;
  if (row_scale) {
    cudaError_t e = d1s.alloc(static_cast<size_t>(nn) * 4, s0);
    if (e != cudaSuccess) return BigPlan::err(e, "scaled D1");
    const int64_t blocks = std::min<int64_t>((nn + 255) / 256, int64_t(sms) * 8);
    scale_rows_kernel<<<static_cast<unsigned>(blocks), 256, 0, s0>>>(bp->sk_d[0], row_scale, n_in, nn,
                                                                       static_cast<float*>(d1s.p));
    e = cudaGetLastError();
    if (e != cudaSuccess) return BigPlan::err(e, "scaled D1");
    d1 = static_cast<const float*>(d1s.p);
  }
  cudaStream_t s = s0;
  const int lsa = bp->sk_lsa, lsb = bp->sk_lsb;
  // pipelined (cp.async double-buffered) column passes when both bit ranges fit them
  const bool staged = (reinterpret_cast<uintptr_t>(a) % 16 == 0) && (ld_a % 4 == 0) && lsa >= 2 && lsa <= 9 &&
                      (lsb == 0 || (lsb >= 2 && lsb <= 9));
  // bulk-copy (TMA) rows when every stripe is full and every row 16-B aligned
  const bool tma = staged && dcols % 32 == 0 && ld_out % 4 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0 &&
                   lsa >= 5 && (lsb == 0 || lsb >= 5);
  auto lcol = [&](int ls, int prog, const ColParams& q) {  // CP_* and SC_FIRST..SC_SINGLE share numbering
    if (tma) return launch_tcol_ls(ls, prog, q, sms, s);
    return staged ? launch_scol_ls(ls, prog, q, sms, s) : launch_col_ls(ls, prog, DM_PER_ROW, q, sms, s);
  };
  ColParams cp{};
  cp.cscale = static_cast<float>(cscale);
  cp.nvec = 1;
  cp.ld_out = ld_out;
  if (lsb == 0) {  // n <= 2^10: the whole chain in one pass
    cp.src = a;
    cp.src_ld = ld_a;
    cp.src_vstride = 0;
    cp.src_valid = n_in * ld_a;
    cp.ncols = dcols;
    cp.nstripes = (dcols + 31) / 32;
    cp.s0 = 0;
    cp.nhi = 1;
    cp.nlo = 1;
    cp.dd[0] = d1;
    cp.dd[1] = bp->sk_d[1];
    cp.dd[2] = bp->sk_d[2];
    cp.rowmap = bp->rowmap;
    cp.dst = out;
    cudaError_t e = lcol(lsa, CP_SINGLE, cp);
    if (e == cudaSuccess) e = bp->note_use(s0);
    return e == cudaSuccess ? SPN_OK : BigPlan::err(e, "sketch single pass");
  }
  // One persistent dataflow launch (sketch_flow.cuh) when the operands are tensor views: every
  // 32-column stripe through the four passes with per-(stripe, pass) dependencies instead of
  // 4 launches per column group.
  if (tma && flow_enabled() && dcols % 32 == 0 && lsa >= 5 && lsa <= 9 && lsb >= 5 && lsb <= 9) {
    FlowParams fp{};
    fp.nstripes = static_cast<int>(dcols / 32);
    fp.G = flow_waves_g();
    static const int nodep = [] { const char* e = std::getenv("SPN_DBG_FLOW_NODEP"); return e ? std::atoi(e) : 0; }();
    fp.nodep = nodep;
    static const int wlast = [] { const char* e = std::getenv("SPN_FLOW_WLAST"); return e ? std::atoi(e) : 1; }();
    fp.wlast = wlast;
    fp.d1 = d1;
    fp.d2t = bp->sk_d[1];
    fp.d3 = bp->sk_d[2];
    fp.rowmap = bp->rowmap;
    fp.wstride = nn * 32;
    fp.out = out;
    fp.ld_out = ld_out;
    fp.cscale = static_cast<float>(cscale);
    Scratch wsp, ctrs;
    if (cudaError_t e = wsp.alloc(static_cast<size_t>(nn) * static_cast<size_t>(dcols) * 4, s0))
      return BigPlan::err(e, "sketch workspace");
    const size_t nctr = 1 + 4 * static_cast<size_t>(fp.nstripes);
    if (cudaError_t e = ctrs.alloc(nctr * 4, s0)) return BigPlan::err(e, "sketch counters");
    if (cudaError_t e = cudaMemsetAsync(ctrs.p, 0, nctr * 4, s0)) return BigPlan::err(e, "sketch counters");
    fp.w = static_cast<float*>(wsp.p);
    fp.ctr = static_cast<uint32_t*>(ctrs.p);
    bool done = false;
    cudaError_t e = launch_flow(lsa, lsb, fp, a, n_in, dcols, ld_a, sms, s0, &done);
    if (e != cudaSuccess) return BigPlan::err(e, "sketch dataflow kernel");
    if (done) {
      if (cudaError_t e2 = bp->note_use(s0)) return BigPlan::err(e2, "sketch use event");
      return SPN_OK;
    }
  }
  // column groups of ~32 MB of workspace
  int64_t dc = std::max<int64_t>(32, (group_bytes(true) / (nn * 4)) / 32 * 32);
  dc = std::min<int64_t>(dc, (dcols + 31) / 32 * 32);
  Scratch scratch;
  if (cudaError_t e = scratch.alloc(static_cast<size_t>(BigPlan::nstreams() * nn * dc * 4), s0))
    return BigPlan::err(e, "sketch workspace");
  float* const work = static_cast<float*>(scratch.p);
  if (spn_status st = bp->fork(s0)) return st;
  int64_t gi = 0;
  const int64_t Sa = int64_t(1) << lsa, Sb = int64_t(1) << lsb;
  for (int64_t c0 = 0; c0 < dcols; c0 += dc, ++gi) {
    const int si = static_cast<int>(gi % BigPlan::nstreams());
    s = bp->ss[si];
    float* W = work + si * nn * dc;
    const int64_t nc = std::min(dc, dcols - c0);
    ColParams pa = cp;  // low-bit passes
    pa.ncols = nc;
    pa.nstripes = (nc + 31) / 32;
    pa.s0 = 0;
    pa.nhi = nn / Sa;
    pa.nlo = 1;
    ColParams pb = pa;  // high-bit passes
    pb.s0 = lsa;
    pb.nhi = 1;
    pb.nlo = Sa;
    // P1: A -> W : D1, H(low)
    pa.src = a + c0;
    pa.src_ld = ld_a;
    pa.src_valid = n_in * ld_a;
    pa.dst = W;
    pa.dst_ld = dc;
    pa.dd[0] = d1;
    cudaError_t e = lcol(lsa, CP_FIRST, pa);
    if (e != cudaSuccess) return BigPlan::err(e, "sketch P1");
    // P2: H(high), D2, H(high)
    pb.src = W;
    pb.src_ld = dc;
    pb.src_valid = nn * dc;
    pb.dst = W;
    pb.dst_ld = dc;
    pb.dd[0] = nullptr;
    pb.dd[1] = bp->sk_d[1];
    e = lcol(lsb, CP_MID, pb);
    if (e != cudaSuccess) return BigPlan::err(e, "sketch P2");
    // P3: H(low), D3, H(low)
    pa.src = W;
    pa.src_ld = dc;
    pa.src_valid = nn * dc;
    pa.dd[0] = nullptr;
    pa.dd[1] = bp->sk_d[2];
    e = lcol(lsa, CP_MID, pa);
    if (e != cudaSuccess) return BigPlan::err(e, "sketch P3");
    // P4: H(high), gather P rows -> out
    pb.dd[0] = nullptr;
    pb.dd[1] = nullptr;
    pb.rowmap = bp->rowmap;
    pb.discard_src = 1;  // W is dead after this pass
    pb.dst = out + c0;
    e = lcol(lsb, CP_LAST, pb);
    if (e != cudaSuccess) return BigPlan::err(e, "sketch P4");
  }
  if (spn_status st = bp->join(s0)) return st;
  if (cudaError_t e = bp->note_use(s0)) return BigPlan::err(e, "sketch use event");
  return SPN_OK;
}

}  // namespace spn
