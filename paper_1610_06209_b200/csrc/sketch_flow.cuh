// Dataflow sketch: the four strided column passes of a SketchOperator (newton_sketch.cpp:74-101),
// S a = sqrt(N/m) P H D3 H D2 H D1 a for every column a of a row-major A[n_in][d], run as ONE
// persistent kernel instead of 4 launches per column group.
//
// The transform splits the N = 2^(lsa+lsb) index bits into a low half (lsa bits, contiguous rows)
// and a high half (lsb bits), and regroups H D3 H D2 H D1 into four passes (spinner_big.cuh):
//   P0 low  : D1, H(low)            A -> W       (A read from HBM once)
//   P1 high : H(high), D2, H(high)  W -> W
//   P2 low  : H(low), D3, H(low)    W -> W
//   P3 high : H(high), gather P     W -> out     (W's lines discarded from L2: no write-back)
// Work unit = one 64 KB task: a tile of 2^LSM rows x 32 columns (one 32-column "stripe"), or two
// half-height tiles when a pass covers LSM-1 bits.  Tasks are numbered in waves of G stripes —
// P0 of the wave's stripes, then P1, P2, P3 — and fetched by the CTAs in that order from a global
// counter; a task of pass p waits (in the producer warp, before its loads) until every tile of pass
// p-1 of its stripe has been stored, counted by per-(stripe, pass) completion counters.  So there
// are no launch boundaries: the passes of different stripes overlap, nothing fills or drains per
// pass, and every SM keeps NB-1 tile loads in flight (TMA, completing on mbarriers) while its
// consumer warps transform the current tile and store it back with TMA.
//
// Progress: tasks are fetched in dependency order and every CTA consumes its tasks in fetch order,
// so the earliest unfinished task never waits on a later one (no co-residency requirement).
#pragma once

#include <cstdlib>
#include <cstring>

#include "spinner_tma.cuh"

namespace spn {

struct FlowParams {
  int nstripes, G;
  int wlast;  // workspace loads / stores carry an L2 evict-last hint (SPN_FLOW_WLAST)
  int nodep;  // bound experiments only (SPN_DBG_FLOW_NODEP, wrong results): 1 skips the dependency waits, 2 also
              // every load of the two-group kernel (0.1475 / 0.1475 / 0.126 ms at config 4 for 0 / 1 / 2)
  uint32_t ntasks;
  const float* d1;   // [N]
  const float* d2t;  // [N], D2 transposed for the high pass: d2t[lo * 2^lsb + s] = D2[(s << lsa) + lo]
  const float* d3;   // [N]
  const int32_t* rowmap;  // [N]: output row of element e, or -1
  float* w;               // workspace: [stripe][N][32]
  int64_t wstride;        // N * 32
  float* out;
  int64_t ld_out;
  float cscale;
  uint32_t* ctr;  // [0]: next task; [1 + 4*s + p]: stored sub-tiles of (stripe s, pass p)
};

struct FlowMaps {
  CUtensorMap a;    // A   : (col, 1, row, 1)            box {32, 1, 256, 1}
  CUtensorMap wlo;  // W   : (col, 1, row, stripe)       low passes
  CUtensorMap whi;  // W   : (col, lo, hs, stripe)       high passes (row = hs * 2^lsa + lo)
};

__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t cnt) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(cnt) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void bulk_wait_n1() { asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); }
// L2 eviction-priority policy for streamed-once data (A: read by P0 only), so it does not push the
// stripes' live workspace out of L2
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tensor_store4_hint(const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                                   const float* ssrc, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2, %3, %4}], [%5], %6;" ::"l"(
          reinterpret_cast<uint64_t>(m)),
      "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(ssrc)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tensor_load4_hint(float* sdst, const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                                  uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(sdst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <int LSA, int LSB>
struct FlowCfg {
  static constexpr int LSA_ = LSA, LSB_ = LSB;
  static constexpr int LSM = LSA > LSB ? LSA : LSB;
  static constexpr int CTHREADS = 1 << LSM;      // consumers: one row of the task per thread
  static constexpr int THREADS = CTHREADS + 64;  // + the loader warp + the storer warp
  static constexpr size_t TILEB = sizeof(float) * (size_t(1) << LSM) * 32;
  static constexpr size_t DSB = sizeof(float) * (size_t(1) << LSM);
  static constexpr int NB = LSM >= 9 ? 3 : 4;  // buffers: NB-1 loads in flight
  static constexpr size_t SMEM = NB * (TILEB + DSB) + NB * 24 + NB * 4 + 64;
  static constexpr int NSUB_LO = 1 << (LSM - LSA), NSUB_HI = 1 << (LSM - LSB);
  static constexpr int T_LO = (1 << LSB) / NSUB_LO;  // tasks per stripe, low pass
  static constexpr int T_HI = (1 << LSA) / NSUB_HI;  // tasks per stripe, high pass
};

template <class F>
__host__ __device__ constexpr int LSA_of() { return F::LSA_; }

struct FlowTask {
  int stripe, pass, idx;  // idx: task within (stripe, pass)
};

template <class F>
__device__ __forceinline__ FlowTask flow_decode(uint32_t t, const FlowParams& p) {
  const uint32_t per_stripe = 2 * F::T_LO + 2 * F::T_HI;
  const uint32_t wave_tasks = (uint32_t)p.G * per_stripe;
  const uint32_t wv = t / wave_tasks;
  uint32_t r = t - wv * wave_tasks;
  const int g = min(p.G, p.nstripes - (int)wv * p.G);
  FlowTask k;
  k.pass = 0;
  for (int q = 0; q < 4; ++q) {
    const uint32_t n = (uint32_t)g * ((q & 1) ? F::T_HI : F::T_LO);
    if (r < n) {
      k.pass = q;
      break;
    }
    r -= n;
  }
  const uint32_t tp = (k.pass & 1) ? F::T_HI : F::T_LO;
  k.stripe = (int)wv * p.G + (int)(r / tp);
  k.idx = (int)(r % tp);
  return k;
}

// One sub-tile (2^LS rows x 32 columns, row-major in buf) through NPARTS H's over its LS bits,
// D (2^LS floats in smem, one per row) before part 1 when DMASK bit 1 / part 0 when bit 0,
// start layout B if START_B; the result goes back to buf (row-major) scaled by `scale`.
template <class C, int NPARTS, int DMASK, bool START_B>
__device__ __forceinline__ void flow_tile_c(float* buf, const float* dsm, int w, int lane, int bar, float scale) {
  float r[C::R];
  constexpr bool LB = START_B && C::W > 1;
#pragma unroll
  for (int j = 0; j < C::R; ++j) r[j] = buf[scol_s<C>(LB, w, j) * 32 + lane];
  named_bar(bar, C::THREADS);  // the tile is in registers: buf is free for the transposes
#pragma unroll
  for (int part = 0; part < NPARTS; ++part) {
    const bool lay_b = C::W > 1 && (START_B ^ ((part & 1) != 0));
    if ((DMASK >> part) & 1) {  // every D of the sketch passes is applied in layout A (s = w*R + j)
      const float4* dv4 = reinterpret_cast<const float4*>(dsm + w * C::R);
#pragma unroll
      for (int q = 0; q < C::R / 4; ++q) {
        const float4 dv = dv4[q];
        r[4 * q] *= dv.x;
        r[4 * q + 1] *= dv.y;
        r[4 * q + 2] *= dv.z;
        r[4 * q + 3] *= dv.w;
      }
    }
    reg_fwht<C::R, 0, C::LR>(r);
    if constexpr (C::W > 1) {
#pragma unroll
      for (int j = 0; j < C::R; ++j) buf[scol_s<C>(lay_b, w, j) * 32 + lane] = r[j];
      named_bar(bar, C::THREADS);
#pragma unroll
      for (int j = 0; j < C::R; ++j) r[j] = buf[scol_s<C>(!lay_b, w, j) * 32 + lane];
      named_bar(bar, C::THREADS);
      if (!lay_b)
        reg_fwht<C::R, C::LR - C::LW, C::LR>(r);
      else
        reg_fwht<C::R, 0, C::LW>(r);
    }
  }
  constexpr bool END_B = C::W > 1 && (START_B ^ ((NPARTS & 1) != 0));
#pragma unroll
  for (int j = 0; j < C::R; ++j) buf[scol_s<C>(END_B, w, j) * 32 + lane] = r[j] * scale;
  fence_proxy_async();  // generic-proxy smem writes -> visible to the TMA store
  named_bar(bar, C::THREADS);
}

template <int LS, int NPARTS, int DMASK, bool START_B>
__device__ __forceinline__ void flow_tile(float* buf, const float* dsm, int w, int lane, int bar, float scale) {
  flow_tile_c<SColCfg<LS>, NPARTS, DMASK, START_B>(buf, dsm, w, lane, bar, scale);
}

// Roles: consumer warps (one row per thread) transform the tile in slot k; the loader warp
// fetches tasks, waits on their dependencies and issues the TMA loads; the storer warp issues each
// finished tile's TMA stores, frees the slot once the store has read it, and counts the tile for
// its (stripe, pass) once the store is complete.  Loader and storer are separate warps so a loader
// waiting on a dependency never holds up the stores that dependency is waiting for.
template <int LSA, int LSB>
__global__ void __launch_bounds__(FlowCfg<LSA, LSB>::THREADS, 1)
    sketch_flow_kernel(const FlowParams p, const __grid_constant__ FlowMaps mp) {
  using F = FlowCfg<LSA, LSB>;
  constexpr int NB = F::NB;
  extern __shared__ __align__(128) float smem[];
  float* bufs = smem;                                                                   // NB x TILEB
  float* dsl = smem + NB * (F::TILEB / 4);                                              // NB x DSB
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NB * ((F::TILEB + F::DSB) / 4));  // NB: loaded
  uint64_t* ready = full + NB;                                                          // NB: computed
  uint64_t* empty = ready + NB;                                                         // NB: stored (read)
  int* tslot = reinterpret_cast<int*>(empty + NB);                                      // NB task ids
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&ready[b], 1);
      mbar_init(&empty[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (tid == F::CTHREADS) {  // ---------------------------------------------- loader
    const uint64_t pol_a = policy_evict_first();
    for (uint32_t k = 0;; ++k) {
      const int slot = (int)(k % NB);
      // the task fetch and its dependency wait (two L2 round trips) come before the wait for the
      // slot, so only the TMA load itself follows the slot's release
      const uint32_t t = atomicAdd(p.ctr, 1u);
      if (t >= p.ntasks) {
        if (k >= (uint32_t)NB) mbar_wait(&empty[slot], ((k / NB) - 1) & 1u);
        tslot[slot] = -1;
        mbar_arrive(&full[slot]);
        return;
      }
      const FlowTask tk = flow_decode<F>(t, p);
      if (tk.pass > 0 && !p.nodep) {  // every tile of the previous pass of this stripe is stored
        const uint32_t need = (tk.pass & 1) ? (1u << LSB) : (1u << LSA);  // sub-tiles of pass - 1
        const uint32_t* c = p.ctr + 1 + 4 * tk.stripe + (tk.pass - 1);
        // a dependency that never completes is a bug: abort the grid (a CUDA error) rather than hang the GPU
        uint64_t t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while (ld_acquire(c) < need) {
          __nanosleep(100);
          uint64_t t1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
          if (t1 - t0 > 5000000000ull) __trap();
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      if (k >= (uint32_t)NB) mbar_wait(&empty[slot], ((k / NB) - 1) & 1u);
      tslot[slot] = (int)t;
      float* buf = bufs + slot * (F::TILEB / 4);
      float* ds = dsl + slot * (F::DSB / 4);
      const bool low = (tk.pass & 1) == 0;
      const int LS = low ? LSA : LSB;
      const int nsub = low ? F::NSUB_LO : F::NSUB_HI;
      const int box = LS > 8 ? 256 : (1 << LS), nbox = (1 << LS) / box;
      const float* dsrc = tk.pass == 0 ? p.d1 : (tk.pass == 1 ? p.d2t : (tk.pass == 2 ? p.d3 : nullptr));
      const uint32_t bytes = (uint32_t)F::TILEB + (dsrc ? (uint32_t)nsub * (4u << LS) : 0u);
      mbar_arrive_tx(&full[slot], bytes);
      for (int sb = 0; sb < nsub; ++sb) {
        const int ti = tk.idx * nsub + sb;  // low: hi index, high: lo index
        float* sbuf = buf + sb * ((1 << LS) * 32);
        for (int b = 0; b < nbox; ++b) {
          if (tk.pass == 0)
            tensor_load4_hint(sbuf + b * box * 32, &mp.a, tk.stripe * 32, 0, (ti << LSA) + b * box, 0, &full[slot],
                              pol_a);
          else if (low)
            tensor_load4(sbuf + b * box * 32, &mp.wlo, 0, 0, (ti << LSA) + b * box, tk.stripe, &full[slot]);
          else
            tensor_load4(sbuf + b * box * 32, &mp.whi, 0, ti, b * box, tk.stripe, &full[slot]);
        }
        if (dsrc) bulk_load(ds + sb * (1 << LS), dsrc + ((int64_t)ti << LS), 4u << LS, &full[slot]);
      }
    }
  }
  if (tid == F::CTHREADS + 32) {  // ------------------------------------------- storer
    for (uint32_t k = 0;; ++k) {
      const int slot = (int)(k % NB);
      mbar_wait(&ready[slot], (k / NB) & 1u);
      const int t = tslot[slot];
      if (t < 0) break;
      const FlowTask tk = flow_decode<F>((uint32_t)t, p);
      if (tk.pass == 3) {  // gather: the consumers stored their rows and waited for the reads
        mbar_arrive(&empty[slot]);
        continue;
      }
      const bool low = (tk.pass & 1) == 0;
      const int LS = low ? LSA : LSB;
      const int nsub = low ? F::NSUB_LO : F::NSUB_HI;
      const int box = LS > 8 ? 256 : (1 << LS), nbox = (1 << LS) / box;
      float* buf = bufs + slot * (F::TILEB / 4);
      for (int sb = 0; sb < nsub; ++sb) {
        const int ti = tk.idx * nsub + sb;
        float* sbuf = buf + sb * ((1 << LS) * 32);
        for (int b = 0; b < nbox; ++b) {
          if (low)
            tensor_store4(&mp.wlo, 0, 0, (ti << LSA) + b * box, tk.stripe, sbuf + b * box * 32);
          else
            tensor_store4(&mp.whi, 0, ti, b * box, tk.stripe, sbuf + b * box * 32);
        }
      }
      bulk_commit();
      bulk_wait_read();  // the store has read the tile: the slot may be refilled
      mbar_arrive(&empty[slot]);
      bulk_wait_all();   // ... and is complete: count its sub-tiles for the dependent pass
      asm volatile("fence.proxy.async.global;" ::: "memory");
      red_release_add(p.ctr + 1 + 4 * tk.stripe + tk.pass, (uint32_t)nsub);
    }
    return;
  }
  if (tid >= F::CTHREADS) return;

  // ---------------------------------------------------------------------- consumers
  for (uint32_t k = 0;; ++k) {
    const int slot = (int)(k % NB);
    mbar_wait(&full[slot], (k / NB) & 1u);
    const int t = tslot[slot];
    if (t < 0) {
      if (tid == 0) mbar_arrive(&ready[slot]);  // lets the storer see the end
      break;
    }
    const FlowTask tk = flow_decode<F>((uint32_t)t, p);
    float* buf = bufs + slot * (F::TILEB / 4);
    const float* ds = dsl + slot * (F::DSB / 4);
    const bool low = (tk.pass & 1) == 0;
    const int LS = low ? LSA : LSB;
    const int sub = tid >> LS, ltid = tid & ((1 << LS) - 1);
    const int w = ltid >> 5, lane = ltid & 31;
    const int ti = tk.idx * (low ? F::NSUB_LO : F::NSUB_HI) + sub;
    float* sbuf = buf + sub * ((1 << LS) * 32);
    const float* sds = ds + sub * (1 << LS);
    const int bar = 1 + sub;
    switch (tk.pass) {  // P0: D1 H | P1: H D2 H (start B) | P2: H D3 H (start B) | P3: H + gather
      case 0: flow_tile<LSA, 1, 1, false>(sbuf, sds, w, lane, bar, 1.0f); break;
      case 1: flow_tile<LSB, 2, 2, true>(sbuf, sds, w, lane, bar, 1.0f); break;
      case 2: flow_tile<LSA, 2, 2, true>(sbuf, sds, w, lane, bar, 1.0f); break;
      default: flow_tile<LSB, 1, 0, false>(sbuf, sds, w, lane, bar, p.cscale); break;
    }
    if (tk.pass == 3) {  // gather this tile's sampled rows: out[rowmap[e]][stripe*32 + c]
      const int64_t e = (int64_t)ti + ((int64_t)ltid << LSA);
      const int32_t orow = __ldg(p.rowmap + e);
      if (orow >= 0) bulk_store(p.out + (int64_t)orow * p.ld_out + tk.stripe * 32, sbuf + ltid * 32, 128);
      bulk_commit();
      // W's row is dead after this pass: drop it from L2 without a write-back
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(p.w + tk.stripe * p.wstride + e * 32) : "memory");
      bulk_wait_read();
    }
    named_bar(3, F::CTHREADS);  // the whole task is computed (and its gather stores have read smem)
    if (tid == 0) mbar_arrive(&ready[slot]);
  }
  bulk_wait_all();
}

// ------------------------------------------------------------------ two consumer groups
// The one-group kernel above runs its 16 consumer warps in lock step over one task: shared-memory
// phases (tile -> registers, the transposes, registers -> tile: ~384 KB per 64 KB task) and butterfly
// phases alternate, so the SM's shared-memory pipe idles during the butterflies and its FP32 pipe
// during the moves (~6.1 K cycles per task against ~3 K of shared-memory time and ~1.7 K of adds).
// Here the consumers are two independent groups of 8 warps, each transforming a whole 64 KB task with
// 64 rows per thread (SCol2Cfg: 6 register bits, so a 2^9-row tile still needs one transpose per H);
// task k of the CTA's fetch order goes to group k & 1, and the groups drift out of phase so one
// group's moves overlap the other's butterflies.  Same task order, counters, loader and storer.
// (Tried on top of this and dropped: passes 0-2 storing their results straight from registers, one
// 128-B stripe row per warp instruction, with the slot released right after the last transpose read
// and a per-warp release count: correct, a third less shared-memory traffic per task and no storer
// warp, but 0.174 vs 0.147 ms at config 4 — 0.166 even with the release fence removed: the 64 STG
// per thread cost more than the staged TMA store.  And a ring of six 32 KB units instead of three
// 64 KB slots for the 9 + 8 bit split — a high-pass task one 256-row sub-tile in one unit on a whole
// group (8 warps x 32 rows per thread), a low-pass task two units, a published (task, unit) queue —
// so that the high passes hold two units and keep four loading: correct, but 0.179 ms (0.174 without
// dependency waits): at 32 rows per thread the phases between the group barriers are half as long
// and the barriers cost more than the extra loads in flight save.)
template <int LS_>
struct SCol2Cfg {
  static constexpr int LS = LS_;
  static constexpr int LR = LS < 6 ? LS : 6;
  static constexpr int LW = LS - LR;
  static constexpr int R = 1 << LR, W = 1 << LW, S = 1 << LS;
  static constexpr int THREADS = 32 * W;
};

template <int LSA, int LSB>
struct Flow2Cfg {
  using F = FlowCfg<LSA, LSB>;
  static constexpr int NGROUPS = 2;
  static constexpr int GTHREADS = 1 << (F::LSM - 1);  // 64 rows per thread
  static constexpr int CTHREADS = NGROUPS * GTHREADS;
  static constexpr int THREADS = CTHREADS + 64;
  static constexpr bool OK = F::LSM == 9;  // 256-thread groups, three 64 KB slots
};

template <int LS, int NPARTS, int DMASK, bool START_B, bool GATHER, class F>
__device__ __forceinline__ void flow2_task(const FlowParams& p, const FlowTask& tk, float* buf, const float* ds,
                                           int g, int gtid, float scale) {
  using C = SCol2Cfg<LS>;
  constexpr int NSUB = 1 << (F::LSM - LS);
  const int sub = gtid / C::THREADS, ltid = gtid % C::THREADS;
  const int w = ltid >> 5, lane = ltid & 31;
  float* sbuf = buf + sub * (C::S * 32);
  flow_tile_c<C, NPARTS, DMASK, START_B>(sbuf, ds + sub * C::S, w, lane, NSUB > 1 ? 3 + 2 * g + sub : 1 + g, scale);
  if constexpr (GATHER) {  // this sub-tile's sampled rows: out[rowmap[e]][stripe*32 + c], two rows per thread
    const int ti = tk.idx * NSUB + sub;
#pragma unroll
    for (int h = 0; h < C::S / C::THREADS; ++h) {
      const int row = ltid + h * C::THREADS;
      const int64_t e = (int64_t)ti + ((int64_t)row << LSA_of<F>());
      const int32_t orow = __ldg(p.rowmap + e);
      if (orow >= 0) bulk_store(p.out + (int64_t)orow * p.ld_out + tk.stripe * 32, sbuf + row * 32, 128);
      // W's row is dead after this pass: drop it from L2 without a write-back
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(p.w + tk.stripe * p.wstride + e * 32) : "memory");
    }
    bulk_commit();
    bulk_wait_read();
  }
}

template <int LSA, int LSB>
__global__ void __launch_bounds__(Flow2Cfg<LSA, LSB>::THREADS, 1)
    sketch_flow2_kernel(const FlowParams p, const __grid_constant__ FlowMaps mp) {
  using F = FlowCfg<LSA, LSB>;
  using F2 = Flow2Cfg<LSA, LSB>;
  constexpr int NB = F::NB;
  extern __shared__ __align__(128) float smem[];
  float* bufs = smem;
  float* dsl = smem + NB * (F::TILEB / 4);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NB * ((F::TILEB + F::DSB) / 4));
  uint64_t* ready = full + NB;
  uint64_t* empty = ready + NB;
  int* tslot = reinterpret_cast<int*>(empty + NB);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&ready[b], 1);
      mbar_init(&empty[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (tid == F2::CTHREADS) {  // ---------------------------------------------- loader
    const uint64_t pol_a = policy_evict_first();
    const uint64_t pol_w = p.wlast ? policy_evict_last() : 0;
    int ends = 0;
    for (uint32_t k = 0;; ++k) {
      const int slot = (int)(k % NB);
      // the task fetch and its dependency wait (two L2 round trips) come before the wait for the
      // slot, so only the TMA load itself follows the slot's release
      const uint32_t t = ends ? p.ntasks : atomicAdd(p.ctr, 1u);
      if (t >= p.ntasks) {  // one end marker per consumer group (consecutive k: one for each parity)
        if (k >= (uint32_t)NB) mbar_wait(&empty[slot], ((k / NB) - 1) & 1u);
        tslot[slot] = -1;
        mbar_arrive(&full[slot]);
        if (++ends == F2::NGROUPS) return;
        continue;
      }
      const FlowTask tk = flow_decode<F>(t, p);
      if (tk.pass > 0 && !p.nodep) {
        const uint32_t need = (tk.pass & 1) ? (1u << LSB) : (1u << LSA);
        const uint32_t* c = p.ctr + 1 + 4 * tk.stripe + (tk.pass - 1);
        uint64_t t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while (ld_acquire(c) < need) {
          __nanosleep(100);
          uint64_t t1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
          if (t1 - t0 > 5000000000ull) __trap();
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      if (k >= (uint32_t)NB) mbar_wait(&empty[slot], ((k / NB) - 1) & 1u);
      tslot[slot] = (int)t;
      float* buf = bufs + slot * (F::TILEB / 4);
      float* ds = dsl + slot * (F::DSB / 4);
      const bool low = (tk.pass & 1) == 0;
      const int LS = low ? LSA : LSB;
      const int nsub = low ? F::NSUB_LO : F::NSUB_HI;
      const int box = LS > 8 ? 256 : (1 << LS), nbox = (1 << LS) / box;
      const float* dsrc = tk.pass == 0 ? p.d1 : (tk.pass == 1 ? p.d2t : (tk.pass == 2 ? p.d3 : nullptr));
      const uint32_t bytes = (uint32_t)F::TILEB + (dsrc ? (uint32_t)nsub * (4u << LS) : 0u);
      if (p.nodep == 2) {  // bound experiment (wrong results): no loads at all, the slot is "full" at once
        mbar_arrive(&full[slot]);
        continue;
      }
      mbar_arrive_tx(&full[slot], bytes);
      for (int sb = 0; sb < nsub; ++sb) {
        const int ti = tk.idx * nsub + sb;
        float* sbuf = buf + sb * ((1 << LS) * 32);
        for (int b = 0; b < nbox; ++b) {
          if (tk.pass == 0)
            tensor_load4_hint(sbuf + b * box * 32, &mp.a, tk.stripe * 32, 0, (ti << LSA) + b * box, 0, &full[slot],
                              pol_a);
          else if (low) {
            if (p.wlast)
              tensor_load4_hint(sbuf + b * box * 32, &mp.wlo, 0, 0, (ti << LSA) + b * box, tk.stripe, &full[slot], pol_w);
            else
              tensor_load4(sbuf + b * box * 32, &mp.wlo, 0, 0, (ti << LSA) + b * box, tk.stripe, &full[slot]);
          } else {
            if (p.wlast && tk.pass != 3)
              tensor_load4_hint(sbuf + b * box * 32, &mp.whi, 0, ti, b * box, tk.stripe, &full[slot], pol_w);
            else
              tensor_load4(sbuf + b * box * 32, &mp.whi, 0, ti, b * box, tk.stripe, &full[slot]);
          }
        }
        if (dsrc) bulk_load(ds + sb * (1 << LS), dsrc + ((int64_t)ti << LS), 4u << LS, &full[slot]);
      }
    }
  }
  if (tid == F2::CTHREADS + 32) {  // ------------------------------------------- storer
    const uint64_t pol_w = p.wlast ? policy_evict_last() : 0;
    for (uint32_t k = 0;; ++k) {
      const int slot = (int)(k % NB);
      mbar_wait(&ready[slot], (k / NB) & 1u);
      const int t = tslot[slot];
      if (t < 0) break;
      const FlowTask tk = flow_decode<F>((uint32_t)t, p);
      if (tk.pass == 3) {
        mbar_arrive(&empty[slot]);
        continue;
      }
      const bool low = (tk.pass & 1) == 0;
      const int LS = low ? LSA : LSB;
      const int nsub = low ? F::NSUB_LO : F::NSUB_HI;
      const int box = LS > 8 ? 256 : (1 << LS), nbox = (1 << LS) / box;
      float* buf = bufs + slot * (F::TILEB / 4);
      for (int sb = 0; sb < nsub; ++sb) {
        const int ti = tk.idx * nsub + sb;
        float* sbuf = buf + sb * ((1 << LS) * 32);
        for (int b = 0; b < nbox; ++b) {
          if (p.wlast) {
            if (low)
              tensor_store4_hint(&mp.wlo, 0, 0, (ti << LSA) + b * box, tk.stripe, sbuf + b * box * 32, pol_w);
            else
              tensor_store4_hint(&mp.whi, 0, ti, b * box, tk.stripe, sbuf + b * box * 32, pol_w);
          } else if (low)
            tensor_store4(&mp.wlo, 0, 0, (ti << LSA) + b * box, tk.stripe, sbuf + b * box * 32);
          else
            tensor_store4(&mp.whi, 0, ti, b * box, tk.stripe, sbuf + b * box * 32);
        }
      }
      bulk_commit();
      bulk_wait_read();
      mbar_arrive(&empty[slot]);
      bulk_wait_all();  // ... and is complete: count its sub-tiles for the dependent pass
      asm volatile("fence.proxy.async.global;" ::: "memory");
      // (deferring this count by one task when the next task is already computed, so its store is
      // issued first, measured slower: 0.171 vs 0.161 ms with waves of 3 stripes, 0.150 vs 0.149 with 4)
      red_release_add(p.ctr + 1 + 4 * tk.stripe + tk.pass, (uint32_t)nsub);
    }
    return;
  }
  if (tid >= F2::CTHREADS) return;

  // ---------------------------------------------------------------------- consumers
  const int g = tid / F2::GTHREADS, gtid = tid % F2::GTHREADS;
  for (uint32_t k = (uint32_t)g;; k += F2::NGROUPS) {
    const int slot = (int)(k % NB);
    // (one warp polling and the others asleep in the group barrier measured the same: 0.148 ms)
    mbar_wait(&full[slot], (k / NB) & 1u);
    const int t = tslot[slot];
    if (t < 0) {
      if (gtid == 0) mbar_arrive(&ready[slot]);  // lets the storer see the end
      break;
    }
    const FlowTask tk = flow_decode<F>((uint32_t)t, p);
    float* buf = bufs + slot * (F::TILEB / 4);
    const float* ds = dsl + slot * (F::DSB / 4);
    switch (tk.pass) {  // P0: D1 H | P1: H D2 H (start B) | P2: H D3 H (start B) | P3: H + gather
      case 0: flow2_task<LSA, 1, 1, false, false, F>(p, tk, buf, ds, g, gtid, 1.0f); break;
      case 1: flow2_task<LSB, 2, 2, true, false, F>(p, tk, buf, ds, g, gtid, 1.0f); break;
      case 2: flow2_task<LSA, 2, 2, true, false, F>(p, tk, buf, ds, g, gtid, 1.0f); break;
      default: flow2_task<LSB, 1, 0, false, true, F>(p, tk, buf, ds, g, gtid, p.cscale); break;
    }
    named_bar(1 + g, F2::GTHREADS);  // the whole task is computed (and its gather stores have read smem)
    if (gtid == 0) mbar_arrive(&ready[slot]);
  }
  bulk_wait_all();
}

// ------------------------------------------------------------------------- host side
inline int flow_mode();
inline bool flow_enabled() { return flow_mode() != 0; }
// Stripes per wave.  The L2 working set is G stripes of N x 32 floats (16 MB at N = 2^17); a pass of a
// stripe can start only when the stripe's previous pass is complete, so the G - 1 other stripes'
// tasks between them must cover the tasks in flight on the grid (~450: 3 per SM).  Config 4, one
// consumer group: G = 2 0.191 ms, 3 0.174 ms (DRAM 157 MB = 1.15x algorithmic), 4 0.170 ms (290 MB: the
// workspace starts spilling from L2); two consumer groups: G = 2 0.184, 3 0.159, 4 0.148 ms (= the
// time without any dependency wait, SPN_DBG_FLOW_NODEP), 8 0.174 ms.  SPN_FLOW_G overrides (0 = auto).
inline int flow_waves_g() {
  static const int g = [] {
    const char* e = std::getenv("SPN_FLOW_G");
    const int v = e ? std::atoi(e) : 0;
    return v < 0 ? 0 : v;
  }();
  return g;
}
inline int flow_auto_g(int64_t stripe_bytes, int tasks_per_stripe_pass, bool two_groups) {
  const int64_t budget = (two_groups ? 64ll : 48ll) << 20;
  const int by_l2 = (int)(budget / stripe_bytes);
  const int by_dep = 1 + (512 + tasks_per_stripe_pass - 1) / tasks_per_stripe_pass;
  return std::max(2, std::max(by_l2, by_dep));
}

template <int LSA, int LSB>
inline cudaError_t launch_flow_t(FlowParams fp, const float* a, int64_t n_in, int64_t dcols, int64_t ld_a, int sms,
                                 cudaStream_t s, bool* done) {
  using F = FlowCfg<LSA, LSB>;
  *done = false;
  const int64_t nn = int64_t(1) << (LSA + LSB);
  FlowMaps mp;
  std::memset(&mp, 0, sizeof(mp));
  const int box_lo = LSA > 8 ? 256 : (1 << LSA), box_hi = LSB > 8 ? 256 : (1 << LSB);
  if (!encode_view(&mp.a, a, dcols, ld_a, 0, n_in, 1, 0, box_lo)) return cudaSuccess;
  if (!encode_view(&mp.wlo, fp.w, 32, 32, 0, nn, fp.nstripes, fp.wstride, box_lo)) return cudaSuccess;
  if (!encode_view(&mp.whi, fp.w, 32, 32, LSA, int64_t(1) << LSB, fp.nstripes, fp.wstride, box_hi))
    return cudaSuccess;
  fp.ntasks = (uint32_t)fp.nstripes * (2 * F::T_LO + 2 * F::T_HI);
  const bool two = Flow2Cfg<LSA, LSB>::OK && flow_mode() >= 2;
  if (fp.G <= 0) fp.G = flow_auto_g(nn * 32 * 4, std::min(F::T_LO, F::T_HI), two);
  if constexpr (Flow2Cfg<LSA, LSB>::OK) {
    if (two) {  // two consumer groups (one CTA per SM)
      auto kern2 = sketch_flow2_kernel<LSA, LSB>;
      static bool attr2 = false;
      if (!attr2) {
        cudaError_t e = cudaFuncSetAttribute(kern2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F::SMEM);
        if (e != cudaSuccess) return e;
        attr2 = true;
      }
      const int64_t grid2 = std::min<int64_t>(int64_t(sms), fp.ntasks);
      kern2<<<(unsigned)grid2, Flow2Cfg<LSA, LSB>::THREADS, F::SMEM, s>>>(fp, mp);
      *done = true;
      return cudaGetLastError();
    }
  }
  auto kern = sketch_flow_kernel<LSA, LSB>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int occ = 1;
  if (cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, F::THREADS, F::SMEM)) return e;
  occ = occ < 1 ? 1 : occ;
  const int64_t grid = std::min<int64_t>(int64_t(sms) * occ, fp.ntasks);
  kern<<<(unsigned)grid, F::THREADS, F::SMEM, s>>>(fp, mp);
  *done = true;
  return cudaGetLastError();
}

// 2 (default): the dataflow kernel with two consumer groups where it exists (2^9-row tiles, N = 2^17
// and 2^18), else the one-group kernel; 1: the one-group kernel; 0: grouped pass launches.  (A register-direct variant — tiles
// moved global <-> registers with LDG/STG, smem only for transposes, the next tile prefetched into a
// second register set — measured 0.286 vs 0.172 ms at config 4 and was dropped: at 128 registers
// and one 512-thread CTA per SM the direct loads cannot keep enough bytes in flight.)
inline int flow_mode() {
  static const int m = [] {
    const char* e = std::getenv("SPN_FLOW");
    return e ? std::atoi(e) : 2;
  }();
  return m;
}

// lsa = ceil(L/2), lsb = floor(L/2) for N = 2^L, L in [10, 18] (both halves in [5, 9]).
inline cudaError_t launch_flow(int lsa, int lsb, const FlowParams& fp, const float* a, int64_t n_in, int64_t dcols,
                               int64_t ld_a, int sms, cudaStream_t s, bool* done) {
  *done = false;
#define SPN_FLOW_CASE(A, B) \
  if (lsa == A && lsb == B) return launch_flow_t<A, B>(fp, a, n_in, dcols, ld_a, sms, s, done);
  SPN_FLOW_CASE(5, 5) SPN_FLOW_CASE(6, 5) SPN_FLOW_CASE(6, 6) SPN_FLOW_CASE(7, 6) SPN_FLOW_CASE(7, 7)
  SPN_FLOW_CASE(8, 7) SPN_FLOW_CASE(8, 8) SPN_FLOW_CASE(9, 8) SPN_FLOW_CASE(9, 9)
#undef SPN_FLOW_CASE
  return cudaSuccess;
}

}  // namespace spn
