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
#include <cmath>
#include <mutex>
#include <vector>

#include "../../include/spinners_b200.h"
#include "errors.hpp"
#include "spinner_vec.cuh"

namespace spn {

// ------------------------------------------------------------- column pass kernel
// A tile is 2^LS "rows" (the transformed sub-index s) x 32 contiguous columns.
// Thread (warp w, lane) holds column col0+lane and R = 2^LR rows:
//   layout A: s = w*R + j      layout B: s = j*W + w
// Loads/stores are 128-B coalesced in both layouts (lanes = columns); the
// transpose goes through smem[s][32] (bank = lane: conflict free).

template <int LS_>
struct ColCfg {
  static constexpr int LS = LS_;
  // <= 16 warps per CTA (<= 128 regs/thread at 512 threads): 32 rows per thread up to
  // LS = 9, 64 rows per thread at LS = 10.
  static constexpr int LR = LS <= 5 ? LS : (LS - 4 > 5 ? LS - 4 : 5);
  static constexpr int LW = LS - LR;
  static constexpr int R = 1 << LR, W = 1 << LW, S = 1 << LS;
  static constexpr int THREADS = 32 * W;
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
  int nparts;            // number of H parts (1..3)
  const float* dd[3];    // D applied before part p (nullable)
  int dmode;             // DM_PER_ROW: dd[p][(lo*nhi + hi)*S + s]; DM_PER_ELEM: dd[p][e*d_ld + col]
  int64_t d_ld;
  int start_b;           // start in layout B
  const int32_t* rowmap; // gather epilogue: out row of e, or -1
  int64_t ld_out;
  float cscale;
  int scale_out, relu;
};

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

template <int LS>
__global__ void __launch_bounds__(ColCfg<LS>::THREADS) colpass_kernel(const ColParams p) {
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
    const int64_t col = cs * 32 + lane;
    const bool colok = col < p.ncols;
    // Tile-uniform bases + 32-bit per-element offsets: element s of this tile sits at
    // e = e0 + (s << s0), i.e. base + s * (2^s0 * ld) + lane.
    const int64_t e0 = (hi << (p.s0 + LS)) + lo;
    const float* sb = p.src + v * p.src_vstride + e0 * p.src_ld + cs * 32;
    const uint32_t s_step = (uint32_t)(p.src_ld << p.s0);
    const int64_t s_lim = p.src_valid - (e0 * p.src_ld + cs * 32);
    bool lay_b = p.start_b;
    auto s_of = [&](int j) -> uint32_t { return lay_b ? (uint32_t)(j * C::W + w) : (uint32_t)(w * C::R + j); };

    float r[C::R];
    if (colok && s_lim >= (int64_t)C::S * s_step) {  // whole tile in range (uniform except last stripe)
#pragma unroll
      for (int j = 0; j < C::R; ++j) r[j] = __ldg(sb + (s_of(j) * s_step + lane));
    } else {
#pragma unroll
      for (int j = 0; j < C::R; ++j) {
        const uint32_t off = s_of(j) * s_step + lane;
        r[j] = (colok && (int64_t)off < s_lim) ? __ldg(sb + off) : 0.0f;
      }
    }
    for (int part = 0; part < p.nparts; ++part) {
      const float* D = p.dd[part];
      if (D) {
        if (p.dmode == DM_PER_ELEM) {
          const float* dbase = D + e0 * p.d_ld + cs * 32;
          const uint32_t d_step = (uint32_t)(p.d_ld << p.s0);
#pragma unroll
          for (int j = 0; j < C::R; ++j)
            if (colok) r[j] *= __ldg(dbase + (s_of(j) * d_step + lane));
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
            for (int j = 0; j < C::R; ++j) r[j] *= __ldg(Dt + s_of(j));
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
        lay_b = !lay_b;
      }
    }
    if (p.rowmap) {
      const int32_t* rm = p.rowmap + e0;
#pragma unroll
      for (int j = 0; j < C::R; ++j) {
        const int32_t orow = __ldg(rm + (s_of(j) << p.s0));
        if (colok && orow >= 0) __stcs(p.dst + (int64_t)orow * p.ld_out + col, r[j] * p.cscale);
      }
    } else {
      float* db = p.dst + v * p.dst_vstride + e0 * p.dst_ld + cs * 32;
      const uint32_t o_step = (uint32_t)(p.dst_ld << p.s0);
#pragma unroll
      for (int j = 0; j < C::R; ++j) {
        float o = r[j];
        if (p.scale_out) o *= p.cscale;
        if (p.relu) o = fmaxf(o, 0.0f);
        if (colok) db[s_of(j) * o_step + lane] = o;
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
  int last;              // last pass: store y
  float* y;
  int64_t ld_y, rows_valid;
  float c;
  int relu;
};

__global__ void __launch_bounds__(256) rowpass_kernel(const RowParams p) {
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
    if (!p.last) {
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
      float* yrow = p.y + v * p.ld_y;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int64_t e = seg * 1024 + j * 32 + t;
        float o = r[j] * p.c;
        if (p.relu) o = fmaxf(o, 0.0f);
        if (e < p.rows_valid) __stcs(yrow + e, o);
      }
    }
  }
}

// ------------------------------------------------------------------- host side

template <int LS>
inline cudaError_t launch_col(const ColParams& p, int sms, cudaStream_t s) {
  using C = ColCfg<LS>;
  static int occ = 0;
  if (occ == 0) {
    cudaError_t e = cudaFuncSetAttribute(colpass_kernel<LS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::SMEM));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, colpass_kernel<LS>, C::THREADS, C::SMEM);
    if (e != cudaSuccess) return e;
    occ = std::max(occ, 1);
  }
  const int64_t tiles = p.nvec * p.nhi * p.nlo * p.nstripes;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t(sms) * occ));
  colpass_kernel<LS><<<static_cast<unsigned>(grid), C::THREADS, C::SMEM, s>>>(p);
  return cudaGetLastError();
}

inline cudaError_t launch_col_ls(int ls, const ColParams& p, int sms, cudaStream_t s) {
  switch (ls) {
    case 1: return launch_col<1>(p, sms, s);
    case 2: return launch_col<2>(p, sms, s);
    case 3: return launch_col<3>(p, sms, s);
    case 4: return launch_col<4>(p, sms, s);
    case 5: return launch_col<5>(p, sms, s);
    case 6: return launch_col<6>(p, sms, s);
    case 7: return launch_col<7>(p, sms, s);
    case 8: return launch_col<8>(p, sms, s);
    case 9: return launch_col<9>(p, sms, s);
    case 10: return launch_col<10>(p, sms, s);
  }
  return cudaErrorInvalidValue;
}

inline cudaError_t launch_row(const RowParams& p, int sms, cudaStream_t s) {
  static int occ = 0;
  if (occ == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rowpass_kernel, 256, 0);
    if (e != cudaSuccess) return e;
    occ = std::max(occ, 1);
  }
  const int64_t ctas = (p.nvec * p.nseg + 7) / 8;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ctas, int64_t(sms) * occ));
  rowpass_kernel<<<static_cast<unsigned>(grid), 256, 0, s>>>(p);
  return cudaGetLastError();
}

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
  float* drow2 = nullptr;  // D2 in the row-pass layout
  // sketch path (lazy)
  std::mutex mu;
  bool sk_ready = false;
  int sk_lsa = 0, sk_lsb = 0;
  float* sk_d[3] = {nullptr, nullptr, nullptr};
  // scratch
  float* work = nullptr;
  size_t work_bytes = 0;
  int32_t* rowmap = nullptr;
  std::vector<int64_t> rowmap_key;
  int64_t rowmap_m = -1;

  void release() {
    for (auto*& q : dnat) {
      if (q) cudaFree(q);
      q = nullptr;
    }
    for (auto*& q : sk_d) {
      if (q) cudaFree(q);
      q = nullptr;
    }
    if (drow2) cudaFree(drow2);
    if (work) cudaFree(work);
    if (rowmap) cudaFree(rowmap);
    drow2 = nullptr;
    work = nullptr;
    rowmap = nullptr;
  }

  static spn_status err(cudaError_t e, const char* what) { return cuda_error(e, what); }

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

  spn_status build(int64_t n_, int64_t tb_, const std::vector<double>* d, const int*) {
    n = n_;
    tb = tb_;
    L = ilog2_i(n);
    std::vector<float> f(static_cast<size_t>(tb * n));
    for (int di = 0; di < 3; ++di) {
      for (size_t i = 0; i < f.size(); ++i) f[i] = static_cast<float>(d[di][i]);
      cudaError_t e = cudaMalloc(&dnat[di], f.size() * 4);
      if (e == cudaSuccess) e = cudaMemcpy(dnat[di], f.data(), f.size() * 4, cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return err(e, "upload diagonals");
    }
    // D2 permuted per 1024-segment into the layout-A float format of VCfg<5,5>
    for (int64_t b = 0; b < tb; ++b)
      for (int64_t seg = 0; seg < n / 1024; ++seg)
        for (int t = 0; t < 32; ++t)
          for (int j = 0; j < 32; ++j) {
            const int64_t pos = ((j / 4) * 32 + t) * 4 + (j % 4);
            f[static_cast<size_t>(b * n + seg * 1024 + pos)] =
                static_cast<float>(d[1][static_cast<size_t>(b * n + seg * 1024 + t * 32 + j)]);
          }
    cudaError_t e = cudaMalloc(&drow2, f.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(drow2, f.data(), f.size() * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return err(e, "upload D2");
    return SPN_OK;
  }

  // y = relu?(c * first rows of (H D3 H D2 H D1 x)) for every block (tables == 1).
  spn_status apply(const float* x, int64_t batch, int64_t ld_x, int64_t n_in, float* y, int64_t ld_y,
                   int relu, int64_t k, int64_t m, int64_t blocks, double c, int sms, cudaStream_t s) {
    if (batch == 0) return SPN_OK;
    std::lock_guard<std::mutex> lock(mu);
    const int lc = 10, lr = L - lc;
    const int64_t C = int64_t(1) << lc;
    // vectors per group: working set ~32 MB (L2-resident passes)
    const int64_t G = std::max<int64_t>(1, std::min<int64_t>(batch, (int64_t(32) << 20) / (n * 4)));
    const bool in_place = blocks == 1 && m == n && k == n;
    if (!in_place) {
      spn_status st = ensure_work(static_cast<size_t>(G * n * 4));
      if (st) return st;
    }
    for (int64_t b = 0; b < blocks; ++b) {
      const int64_t rows_valid = std::min(m, k - b * m);
      for (int64_t v0 = 0; v0 < batch; v0 += G) {
        const int64_t nv = std::min(G, batch - v0);
        float* W = in_place ? y + v0 * ld_y : work;
        const int64_t wstride = in_place ? ld_y : n;
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
        cp.nparts = 1;
        cp.dd[0] = dnat[0] + b * n;
        cp.dmode = DM_PER_ELEM;
        cp.d_ld = C;
        cp.start_b = 0;
        cudaError_t e = launch_col_ls(lr, cp, sms, s);  // P1: D1, Hr
        if (e != cudaSuccess) return err(e, "colpass P1");
        RowParams rp{};
        rp.buf = W;
        rp.vstride = wstride;
        rp.nseg = n / C;
        rp.nvec = nv;
        rp.d_mid = drow2 + b * n;
        rp.last = 0;
        e = launch_row(rp, sms, s);  // P2: Hc, D2, Hc
        if (e != cudaSuccess) return err(e, "rowpass P2");
        cp.src = W;
        cp.src_vstride = wstride;
        cp.src_valid = n;
        cp.nparts = 2;
        cp.dd[0] = nullptr;
        cp.dd[1] = dnat[2] + b * n;
        cp.start_b = 1;
        e = launch_col_ls(lr, cp, sms, s);  // P3: Hr, D3, Hr
        if (e != cudaSuccess) return err(e, "colpass P3");
        rp.last = 1;
        rp.y = y + v0 * ld_y + b * m;
        rp.ld_y = ld_y;
        rp.rows_valid = rows_valid;
        rp.c = static_cast<float>(c);
        rp.relu = relu;
        e = launch_row(rp, sms, s);  // P4: Hc, scale, relu, store
        if (e != cudaSuccess) return err(e, "rowpass P4");
      }
    }
    return SPN_OK;
  }

  spn_status build_sketch(int64_t nn, const std::vector<double>* d) {
    if (sk_ready) return SPN_OK;
    const int LL = ilog2_i(nn);
    if (LL <= 10) {
      sk_lsa = LL;
      sk_lsb = 0;
    } else {
      sk_lsa = (LL + 1) / 2;
      sk_lsb = LL / 2;
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
      cudaError_t e = cudaMalloc(&sk_d[di], f.size() * 4);
      if (e == cudaSuccess) e = cudaMemcpy(sk_d[di], f.data(), f.size() * 4, cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return err(e, "upload sketch diagonals");
    }
    sk_ready = true;
    return SPN_OK;
  }

  spn_status set_rowmap(int64_t nn, const int64_t* rows, int64_t m_out, cudaStream_t s) {
    std::vector<int64_t> key;
    if (rows) key.assign(rows, rows + m_out);
    if (rowmap && rowmap_m == m_out && key == rowmap_key) return SPN_OK;
    std::vector<int32_t> map(static_cast<size_t>(nn), -1);
    for (int64_t r = 0; r < m_out; ++r) {
      const int64_t i = rows ? rows[r] : r;
      if (map[static_cast<size_t>(i)] != -1) return set_error(SPN_EDIM, "sketch rows must be distinct");
      map[static_cast<size_t>(i)] = static_cast<int32_t>(r);
    }
    cudaError_t e = cudaSuccess;
    if (!rowmap) e = cudaMalloc(&rowmap, static_cast<size_t>(nn) * 4);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // previous users of the map are done
    if (e == cudaSuccess) e = cudaMemcpy(rowmap, map.data(), map.size() * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return err(e, "row map");
    rowmap_key = std::move(key);
    rowmap_m = m_out;
    return SPN_OK;
  }
};

inline spn_status sketch_run(int64_t nn, const std::vector<double>* d, const int* /*dsign*/,
                             const float* a, int64_t n_in, int64_t dcols, int64_t ld_a,
                             const int64_t* rows, int64_t m_out, double cscale, float* out,
                             int64_t ld_out, int sms, cudaStream_t s, BigPlan* bp) {
  std::lock_guard<std::mutex> lock(bp->mu);
  if (spn_status st = bp->build_sketch(nn, d)) return st;
  if (spn_status st = bp->set_rowmap(nn, rows, m_out, s)) return st;
  const int lsa = bp->sk_lsa, lsb = bp->sk_lsb;
  ColParams cp{};
  cp.dmode = DM_PER_ROW;
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
    cp.nparts = 3;
    cp.dd[0] = bp->sk_d[0];
    cp.dd[1] = bp->sk_d[1];
    cp.dd[2] = bp->sk_d[2];
    cp.rowmap = bp->rowmap;
    cp.dst = out;
    cudaError_t e = launch_col_ls(lsa, cp, sms, s);
    return e == cudaSuccess ? SPN_OK : BigPlan::err(e, "sketch single pass");
  }
  // column groups of ~32 MB of workspace
  int64_t dc = std::max<int64_t>(32, ((int64_t(32) << 20) / (nn * 4)) / 32 * 32);
  dc = std::min<int64_t>(dc, (dcols + 31) / 32 * 32);
  if (spn_status st = bp->ensure_work(static_cast<size_t>(nn * dc * 4))) return st;
  float* W = bp->work;
  const int64_t Sa = int64_t(1) << lsa, Sb = int64_t(1) << lsb;
  for (int64_t c0 = 0; c0 < dcols; c0 += dc) {
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
    pa.nparts = 1;
    pa.dd[0] = bp->sk_d[0];
    pa.start_b = 0;
    cudaError_t e = launch_col_ls(lsa, pa, sms, s);
    if (e != cudaSuccess) return BigPlan::err(e, "sketch P1");
    // P2: H(high), D2, H(high)
    pb.src = W;
    pb.src_ld = dc;
    pb.src_valid = nn * dc;
    pb.dst = W;
    pb.dst_ld = dc;
    pb.nparts = 2;
    pb.dd[0] = nullptr;
    pb.dd[1] = bp->sk_d[1];
    pb.start_b = 1;
    e = launch_col_ls(lsb, pb, sms, s);
    if (e != cudaSuccess) return BigPlan::err(e, "sketch P2");
    // P3: H(low), D3, H(low)
    pa.src = W;
    pa.src_ld = dc;
    pa.src_valid = nn * dc;
    pa.nparts = 2;
    pa.dd[0] = nullptr;
    pa.dd[1] = bp->sk_d[2];
    pa.start_b = 1;
    e = launch_col_ls(lsa, pa, sms, s);
    if (e != cudaSuccess) return BigPlan::err(e, "sketch P3");
    // P4: H(high), gather P rows -> out
    pb.nparts = 1;
    pb.dd[0] = nullptr;
    pb.dd[1] = nullptr;
    pb.start_b = 0;
    pb.rowmap = bp->rowmap;
    pb.dst = out + c0;
    e = launch_col_ls(lsb, pb, sms, s);
    if (e != cudaSuccess) return BigPlan::err(e, "sketch P4");
  }
  return SPN_OK;
}

}  // namespace spn
