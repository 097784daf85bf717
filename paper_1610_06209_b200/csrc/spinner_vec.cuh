// Fused structured-spinner kernels for n <= 2^14 (one "group" of T threads per vector).
//
// Computes, per vector x (fp32), the reference chain
//     y = scale * first_m( H D3 H D2 H D1 x )          (proj/src/spinner.cpp:186-231)
// with H the normalised Walsh-Hadamard transform (proj/src/transforms.cpp:52-71)
// and fuses the nonlinearity that consumes y:
//     OP_HASH        signed argmax -> int32 bucket id     (proj/src/lsh.cpp:9-30)
//     OP_APPLY       store y (optionally ReLU, optionally + hash ids)
//     OP_EMBED_GAUSS (1/sqrt(k)) [cos(y/sigma) || sin(y/sigma)]   (proj/src/kernels.cpp:27-35)
//     OP_EMBED_ANG   sign(y) with sign(0) = +1                    (proj/src/kernels.cpp:23-26)
//
// Data layout (n = R*T, R = 2^LOG_R registers per thread, T = 2^LOG_T threads):
//   layout B: thread t holds elements i = j*T + t  (j = register) -> coalesced global I/O
//   layout A: thread t holds elements i = t*R + j                  -> 16-B smem vectors
// Every FWHT runs its butterflies on the element bits that currently live in
// registers (packed FADD2 on register pairs), exchanges layouts once through a
// swizzled shared-memory transpose, and finishes the remaining bits.  Three
// H's therefore cost three transposes (plus one for a layout-B epilogue).
// All 1/sqrt(n) factors and the scale are folded into one multiplier.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace spn {

enum Op : int { OP_HASH = 0, OP_APPLY = 1, OP_EMBED_GAUSS = 2, OP_EMBED_ANG = 3, OP_EMBED_GAUSS_P = 4, OP_APPLY_P = 5 };
enum Layout : int { LAY_B = 0, LAY_A = 1 };

// One diagonal position (D1/D2/D3) in one layout, for every (table, block).
struct DiagArrays {
  const uint32_t* sgn;  // ±1 diagonals: [tables*blocks][WORDS][T] bit-packed sign masks
  const float* flt;     // real diagonals: [tables*blocks][R/4][T][4] (fp32)
};

struct VecParams {
  const float* x;
  int64_t ld_x, n_in, batch;
  int64_t m, k;  // rows per block, rows per table
  int blocks, tables;
  DiagArrays d[3][2];  // [diagonal][layout]
  int dsign[3];        // 1: diagonal is ±1 (use sgn), 0: real (use flt)
  float c;             // scale * n^{-3/2}
  float c2;            // OP_EMBED_GAUSS: c / sigma (folded into x once per row)
  float norm;          // OP_EMBED_GAUSS: 1/sqrt(k)
  int32_t* ids;        // OP_HASH / OP_APPLY (optional): [batch][tables]
  float* y;            // OP_APPLY / OP_EMBED_*: output rows
  int64_t ld_y;
  int relu;
  int x_vec_ok;        // x and ld_x 16-B aligned (cp.async staging allowed)
  // fused all-gather (OP_HASH): every id is also stored, at row peer_row0 + v, into each
  // rank's gathered [total][tables] table through peer (CUDA IPC / NVLink) pointers
  int32_t* const* peers;
  int npeers;
  int64_t peer_row0;
  int vec_major;       // OP_HASH: all tables of a vector in one CTA, back to back (see the kernel)
  int perm;            // host: run the apply + ids as OP_APPLY_P (permuted coordinates, 16-B x / y moves)
};

#ifndef SPN_EMBED_WARPS
#define SPN_EMBED_WARPS 24  // n = 1024 embed register budget (resident warps / SM); 20/22/26 measured slower
#endif

#ifndef SPN_APPLY_PREFETCH
#define SPN_APPLY_PREFETCH 1
#endif
#ifndef SPN_TW13
#define SPN_TW13 12  // resident warps / SM the n = 2^13 (R = 128, T = 64) kernels are compiled for
#endif
#ifndef SPN_TW64
#define SPN_TW64 12  // resident warps / SM the R = 64 kernels are compiled for
#endif
#ifndef SPN_XBUF_MAX_LOGN
#define SPN_XBUF_MAX_LOGN 12  // largest n whose embed kernels stage x in a second shared-memory buffer: at
// n = 2^13 / 2^14 the second buffer halves / thirds the resident CTAs (2^14: one 128 KB CTA per SM) and the
// single-block Gaussian features ran 0.44 / 0.41 of HBM; loading x per block like the apply: 0.64 / 0.67
// (with the apply's next-row L2 prefetch on top: 0.65 / 0.63, so the embed kernels go without)
#endif
#ifndef SPN_LOOP_ODD_HASH_MIN_R
#define SPN_LOOP_ODD_HASH_MIN_R 64
#endif
#ifndef SPN_LOOP_ODD_MIN_R
#define SPN_LOOP_ODD_MIN_R 128
#endif
#ifndef SPN_LOOP_MIN_R
#define SPN_LOOP_MIN_R 64
#endif
template <int LOG_R_, int LOG_T_>
struct VCfg {
  static constexpr int LOG_R = LOG_R_, LOG_T = LOG_T_, LOG_N = LOG_R + LOG_T;
  static constexpr int R = 1 << LOG_R, T = 1 << LOG_T, N = 1 << LOG_N;
  static constexpr int THREADS = T >= 32 ? T : 256;          // CTA size
  static constexpr int GPC = THREADS / T;                     // groups (vectors) per CTA
  static constexpr int WORDS = R >= 32 ? R / 32 : 1;          // sign words per thread
  static constexpr int BITS = R >= 32 ? 32 : R;               // valid bits per word
  // swizzle only the 16-B chunk bits inside one thread's layout-A run (bits 2..LOG_R-1)
  static constexpr int XMASK = (R / 4 >= 8 ? 8 : (R / 4 > 0 ? R / 4 : 1)) - 1;
  static constexpr bool MULTI_WARP = T > 32;
  // register budget: resident warps/SM we ask ptxas to allow (R data registers + ~50)
  // R = 32: 28 warps (one wave for config 1's 4096 vectors: 18.6 vs 21.1 us) for hash /
  // apply; the embed kernels keep 24 (80 registers; at 72 they spill: 0.475 vs 0.443 ms)
  static constexpr int TARGET_WARPS = R <= 16 ? 32 : (R == 32 ? 28 : (R == 64 ? SPN_TW64 : (LOG_T == 6 ? SPN_TW13 : 12)));
  __host__ __device__ static constexpr int min_ctas(int op) {
    return (R == 32 && op >= 2 && op <= 4) ? (SPN_EMBED_WARPS / (THREADS / 32) > 0 ? SPN_EMBED_WARPS / (THREADS / 32) : 1)
                                : MIN_CTAS_BASE;
  }
  // looped chain (one copy of the D -> H body, R == T only): keeps the n = 16384 kernel
  // (R = 128, fully unrolled ~57 KB of SASS) inside the 32 KB L1.5 instruction cache.
  // For n = 1024 the unrolled chain fits and measured faster (0.475 vs 0.498 ms); for n = 4096
  // (R = 64) the loop wins: 8-table hash 62.9 -> 77.2 adds/clk/SM, apply 0.62 -> 0.69 of HBM.
  static constexpr bool LOOPED = LOG_R == LOG_T && R >= SPN_LOOP_MIN_R;
  // R == 2T (n = 2^11, 2^13) as a one-body loop too.  The two layouts' register bits overlap in one
  // element bit (LOG_T), so if layout B numbers its registers pb(j) = (j >> 1) | ((j & 1) << (LOG_R-1))
  // (the shared bit on top) both directions run the same code: butterflies over all LOG_R register
  // bits, a transpose (direction chosen at run time: only the transposes have two copies), butterflies
  // over register bits [0, LOG_T).  Loads, stores and the layout-B transposes index registers through
  // pb(); the host packs the all-sign plans' layout-B masks in the same order (build_vec_layouts).
  static constexpr bool LOOPED_ODD = LOG_R == LOG_T + 1 && R >= SPN_LOOP_ODD_MIN_R;
  // n = 2^11 (R = 64, T = 32): the loop is faster for the hash (66.0 -> 71.9 adds/clk/SM) and slower for
  // the apply (0.76 -> 0.72 of HBM), so only the hash kernels take it (the plan keeps its layout-B masks in
  // both orders: spn_plan::vsgnL).
  __host__ __device__ static constexpr bool looped_odd(int op) {
    return LOOPED_ODD || (LOG_R == LOG_T + 1 && R >= SPN_LOOP_ODD_HASH_MIN_R && op == 0 /* OP_HASH */);
  }
  template <bool PI>
  __host__ __device__ static constexpr int pb(int j) {
    return PI ? ((j >> 1) | ((j & 1) << (LOG_R - 1))) : j;
  }
  static constexpr int MIN_CTAS_BASE = TARGET_WARPS / (THREADS / 32) > 0 ? TARGET_WARPS / (THREADS / 32) : 1;
  // per group: transpose buffer (+ an x staging buffer for the embed ops, which reuse
  // x across blocks and prefetch the next row with cp.async)
  __host__ __device__ static constexpr bool xbuf(int op) { return (op == 2 || op == 3 || op == 4) && LOG_N <= SPN_XBUF_MAX_LOGN; }
  __host__ __device__ static constexpr int smem_floats(int op) {
    return GPC * N * (xbuf(op) ? 2 : 1) + (T > 32 ? 4 * (T / 32) : 0);
  }
  __host__ __device__ static constexpr size_t smem_bytes(int op) { return sizeof(float) * (size_t)smem_floats(op); }
};

// 16-B global->shared async copy, zero-filling beyond src_bytes (cp.async, LDGSTS).
__device__ __forceinline__ void cp_async16(float* smem, const float* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// ---------------------------------------------------------------- primitives

// (a0,a1),(b0,b1) <- (a+b, a-b) on packed f32x2 (sm_100a FADD2: one instruction for two adds,
// though it holds the issue port two cycles — the FP32 add rate equals two FADDs).
__device__ __forceinline__ void bfly2(float& a0, float& a1, float& b0, float& b1) {
#ifdef SPN_BFLY_SCALAR  // (microbenchmark only: the same butterflies as four scalar FADDs)
  const float u0 = a0, u1 = a1;
  a0 = u0 + b0;
  a1 = u1 + b1;
  b0 = u0 - b0;
  b1 = u1 - b1;
  return;
#endif
  asm("{\n\t.reg .b64 pa, pb, ps, pd;\n\t"
      "mov.b64 pa, {%0, %1};\n\t"
      "mov.b64 pb, {%2, %3};\n\t"
      "add.rn.f32x2 ps, pa, pb;\n\t"
      "sub.rn.f32x2 pd, pa, pb;\n\t"
      "mov.b64 {%0, %1}, ps;\n\t"
      "mov.b64 {%2, %3}, pd;\n\t}"
      : "+f"(a0), "+f"(a1), "+f"(b0), "+f"(b1));
}

// (a, b) <- (a + b, a - b) inside one register pair as a single packed FFMA2:
// (b, b) * (1, -1) + (a, a) — ptxas encodes the (x, x) operands as .F32 broadcasts.
// fma(b, +-1, a) is exactly the rounded a +- b, so results equal two FADDs.
__device__ __forceinline__ void bfly_inpair(float& a, float& b) {
  asm("{\n\t.reg .b64 pb, pa, pc, pd;\n\t"
      "mov.b64 pb, {%1, %1};\n\t"
      "mov.b64 pa, {%0, %0};\n\t"
      "mov.b64 pc, {%2, %3};\n\t"
      "fma.rn.f32x2 pd, pb, pc, pa;\n\t"
      "mov.b64 {%0, %1}, pd;\n\t}"
      : "+f"(a), "+f"(b)
      : "f"(1.0f), "f"(-1.0f));
}

// Unnormalised butterflies over register bits [BLO, BHI) (transforms.cpp:58-67 restricted
// to the element bits this thread holds).  Register pairs (2q, 2q+1) share one FADD2;
// the in-pair stage (bit 0) is one FFMA2 per pair.
#ifndef SPN_INPAIR_FFMA2_MIN_R
#define SPN_INPAIR_FFMA2_MIN_R 1024
#endif
constexpr int kInpairFfma2MinR = SPN_INPAIR_FFMA2_MIN_R;

template <int R, int BLO, int BHI, bool REV = false>
__device__ __forceinline__ void reg_fwht(float (&r)[R]) {
#pragma unroll
  for (int bb = BLO; bb < BHI; ++bb) {
    const int b = REV ? BLO + BHI - 1 - bb : bb;  // the stages commute: any order
    const int h = 1 << b;
    if (b == 0) {
      // FFMA2 halves the issue slots but occupies the FP32 pipe longer than two FADDs:
      // a win only while the unrolled R = 128 chain was instruction-fetch bound (c3:
      // 312 -> 302 ms); with the looped chain it loses (289 vs 277 ms), and for R = 32
      // too (c2: 0.458 -> 0.479 ms), so it is off by default (SPN_INPAIR_FFMA2_MIN_R).
      if constexpr (R >= kInpairFfma2MinR) {
#pragma unroll
        for (int j = 0; j < R; j += 2) bfly_inpair(r[j], r[j + 1]);
      } else {
#pragma unroll
        for (int j = 0; j < R; j += 2) {
          const float u = r[j], v = r[j + 1];
          r[j] = u + v;
          r[j + 1] = u - v;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < R; j += 2) {
        if (j & h) continue;
        bfly2(r[j], r[j + 1], r[j + h], r[j + h + 1]);
      }
    }
  }
}

template <class C>
__device__ __forceinline__ void group_sync() {
  if constexpr (C::MULTI_WARP)
    __syncthreads();
  else
    __syncwarp();
}

// Swizzled smem slot of element i: the 16-B chunk index (bits 2-4) is XORed with the
// layout-A owner thread, making both the A-side 16-B accesses and the B-side 4-B
// accesses bank-conflict free for R >= 32.
template <class C>
__device__ __forceinline__ int sw(int i) {
  return i ^ (((i >> C::LOG_R) & C::XMASK) << 2);
}

// Swizzled addresses with the runtime part hoisted into 8 base offsets so every
// access is base + immediate (R >= 32 and T >= 32, the performance configurations):
//   A side, chunk q of thread t:  t*R + 4*(q ^ (t&7))            = a[q&7] + 4*(q & ~7)
//   B side, register j:           j*T + (t ^ (((j >> (LOG_R-LOG_T)) & 7) << 2))
template <class C>
struct Swz {
  static constexpr bool FAST = C::R >= 32 && C::T >= 32;
  int a[8], b[8];
  __device__ __forceinline__ explicit Swz(int t) {
    if constexpr (FAST) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        a[c] = t * C::R + 4 * (c ^ (t & 7));
        b[c] = t ^ (c << 2);
      }
    }
  }
  __device__ __forceinline__ int A(int t, int q) const {
    if constexpr (FAST)
      return a[q & 7] + 4 * (q & ~7);
    else
      return sw<C>(t * C::R + 4 * q);
  }
  __device__ __forceinline__ int B(int t, int j) const {
    if constexpr (FAST)
      return j * C::T + b[(j >> (C::LOG_R - C::LOG_T)) & 7];
    else
      return sw<C>(j * C::T + t);
  }
};

// Layout-B side of a transpose as 8x8 b16 matrix moves (ldmatrix / stmatrix .x4): one
// instruction moves four registers of every lane (512 B per warp) where LDS.32 / STS.32
// move one (128 B), cutting the transpose's shared-memory instructions from R + R/4 to
// R/4 + R/4.  For fp32 data an 8x8 b16 matrix is 8 rows of four floats and lane l gets
// word l&3 of row l>>2: with matrix q's rows the eight 16-B chunks of elements
// (j0+q)*T + 32w + [0, 32) (rows supplied by lanes 8q..8q+7), lane l receives element
// (j0+q)*T + 32w + l — exactly register j0+q of layout B.  The swizzle XORs whole 16-B
// chunks inside that 128-B line, so each matrix is still one conflict-free wavefront.
// Needs whole warps per group (T >= 32) and 16-B chunks (R >= 4).
template <class C>
struct MatB {
  static constexpr bool ON = C::T >= 32 && C::R >= 4;
  static constexpr int S = C::LOG_R - C::LOG_T;            // (e >> LOG_R) == (j >> S) on the B side
  static constexpr int P = ((C::XMASK + 1) << S) / 4 > 0 ? ((C::XMASK + 1) << S) / 4 : 1;  // swizzle period in j0/4
  uint32_t off[P];                                          // byte offsets of this lane's row, per j0/4 mod P
  __device__ __forceinline__ MatB(const float* sm, int t) {
    const int l = t & 31, w = t >> 5, q = l >> 3, rho = l & 7;
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int c = ((4 * k + q) >> S) & C::XMASK;
      off[k] = base + 4u * static_cast<uint32_t>((4 * k + q) * C::T + 32 * w + 4 * (rho ^ c));
    }
  }
  __device__ __forceinline__ uint32_t addr(int k) const {  // k = j0 / 4 (compile-time after unrolling)
    return off[k % P] + 16u * static_cast<uint32_t>((k - k % P) * C::T);
  }
};

__device__ __forceinline__ void ldsm_x4(uint32_t a, float& r0, float& r1, float& r2, float& r3) {
  uint32_t u0, u1, u2, u3;
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(u0), "=r"(u1), "=r"(u2), "=r"(u3)
               : "r"(a)
               : "memory");
  r0 = __uint_as_float(u0);
  r1 = __uint_as_float(u1);
  r2 = __uint_as_float(u2);
  r3 = __uint_as_float(u3);
}
__device__ __forceinline__ void stsm_x4(uint32_t a, float r0, float r1, float r2, float r3) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1, %2, %3, %4};\n" ::"r"(a),
               "r"(__float_as_uint(r0)), "r"(__float_as_uint(r1)), "r"(__float_as_uint(r2)),
               "r"(__float_as_uint(r3))
               : "memory");
}

// The same moves for the looped R == 2T chain, whose layout-B registers are numbered pb(j): matrix q of
// quad k carries the standard register pinv(4k + q) = 2 (4k + q) for the first half of the quads and
// 2 (4k + q - R/2) + 1 for the second, so every ldmatrix / stmatrix still fills an aligned register quad
// in physical order (with pb() applied to the destination registers instead, ptxas shuffled every quad
// into place with MOVs).  S = 1, so the swizzle chunk (j >> 1) & 7 is the same for 2m and 2m + 1 and the
// odd half sits one register row (4T bytes) further.
template <class C>
struct MatBP {
  static constexpr int H = C::R / 8;  // quads per half
  uint32_t off[2];
  __device__ __forceinline__ MatBP(const float* sm, int t) {
    const int l = t & 31, w = t >> 5, q = l >> 3, rho = l & 7;
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const int j = 2 * (4 * kk + q);
      const int c = (j >> 1) & C::XMASK;
      off[kk] = base + 4u * static_cast<uint32_t>(j * C::T + 32 * w + 4 * (rho ^ c));
    }
  }
  __device__ __forceinline__ uint32_t addr(int k) const {  // k: physical quad (compile-time after unrolling)
    const int kh = k % H, odd = k / H;
    return off[kh % 2] + 4u * static_cast<uint32_t>(C::T * (8 * (kh - kh % 2) + odd));
  }
};

#ifndef SPN_F1_REV
#define SPN_F1_REV 1
#endif

#ifndef SPN_XPOSE_MATRIX
#define SPN_XPOSE_MATRIX 1
#endif

template <class C, bool PI = false>
__device__ __forceinline__ void xpose_A_to_B(float (&r)[C::R], float* sm, int t) {
  const Swz<C> z(t);
  if constexpr (C::R >= 4) {
#pragma unroll
    for (int q = 0; q < C::R / 4; ++q)
      *reinterpret_cast<float4*>(sm + z.A(t, q)) =
          make_float4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < C::R; ++j) sm[sw<C>(t * C::R + j)] = r[j];
  }
  group_sync<C>();
  if constexpr (MatB<C>::ON && SPN_XPOSE_MATRIX && PI) {
    const MatBP<C> mb(sm, t);
#pragma unroll
    for (int k = 0; k < C::R / 4; ++k) ldsm_x4(mb.addr(k), r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
  } else if constexpr (MatB<C>::ON && SPN_XPOSE_MATRIX) {
    const MatB<C> mb(sm, t);
#pragma unroll
    for (int k = 0; k < C::R / 4; ++k) ldsm_x4(mb.addr(k), r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < C::R; ++j) r[C::template pb<PI>(j)] = sm[z.B(t, j)];
  }
  group_sync<C>();
}

template <class C, bool PI = false>
__device__ __forceinline__ void xpose_B_to_A(float (&r)[C::R], float* sm, int t) {
  const Swz<C> z(t);
  if constexpr (MatB<C>::ON && SPN_XPOSE_MATRIX && PI) {
    const MatBP<C> mb(sm, t);
#pragma unroll
    for (int k = 0; k < C::R / 4; ++k) stsm_x4(mb.addr(k), r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
  } else if constexpr (MatB<C>::ON && SPN_XPOSE_MATRIX) {
    const MatB<C> mb(sm, t);
#pragma unroll
    for (int k = 0; k < C::R / 4; ++k) stsm_x4(mb.addr(k), r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < C::R; ++j) sm[z.B(t, j)] = r[C::template pb<PI>(j)];
  }
  group_sync<C>();
  if constexpr (C::R >= 4) {
#pragma unroll
    for (int q = 0; q < C::R / 4; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(sm + z.A(t, q));
      r[4 * q] = v.x;
      r[4 * q + 1] = v.y;
      r[4 * q + 2] = v.z;
      r[4 * q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < C::R; ++j) r[j] = sm[sw<C>(t * C::R + j)];
  }
  group_sync<C>();
}

// H on a vector whose registers are in layout B; ends in layout A.
template <class C>
__device__ __forceinline__ void fwht_B_to_A(float (&r)[C::R], float* sm, int t) {
  reg_fwht<C::R, 0, C::LOG_R>(r);
  if constexpr (C::T > 1) {
    xpose_B_to_A<C>(r, sm, t);
    reg_fwht<C::R, 0, C::LOG_T>(r);
  }
}

// H on a vector in layout A; ends in layout B.
template <class C>
__device__ __forceinline__ void fwht_A_to_B(float (&r)[C::R], float* sm, int t) {
  reg_fwht<C::R, 0, C::LOG_R>(r);
  if constexpr (C::T > 1) {
    xpose_A_to_B<C>(r, sm, t);
    reg_fwht<C::R, C::LOG_R - C::LOG_T, C::LOG_R>(r);
  }
}

// r <- -r when bit jj of the mask word w is set.  Written as a predicated XOR so ptxas
// turns each 7 bits of w into predicates with one R2P and flips with @P LOP3: ~1.25 ALU
// instructions per element instead of a shift + LOP3 (tools/microbench/fwht_regs.cu,
// R = 128: 82.5 -> 93.4 adds/clk/SM; the plain `(w << (31 - jj)) & 0x80000000` shift even
// compiles to IMAD.SHL on the FMA pipe the butterflies saturate).
__device__ __forceinline__ void flip_if(float& r, uint32_t w, int jj) {
  uint32_t x = __float_as_uint(r);
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
      "and.b32 t, %1, %2;\n\tsetp.ne.u32 p, t, 0;\n\t@p xor.b32 %0, %0, 0x80000000;\n\t}"
      : "+r"(x)
      : "r"(w), "r"(1u << jj));
  r = __uint_as_float(x);
}

// r <- D r, D given in the current layout (diag_matvec, transforms.cpp:228-235).
template <class C>
__device__ __forceinline__ void apply_diag(float (&r)[C::R], const DiagArrays& d, int is_sign,
                                           int64_t tb, int t) {
  if (is_sign) {
    const uint32_t* w = d.sgn + tb * (int64_t)(C::WORDS * C::T);
#pragma unroll
    for (int q = 0; q < C::WORDS; ++q) {
      const uint32_t word = __ldg(w + q * C::T + t);
#pragma unroll
      for (int jj = 0; jj < C::BITS; ++jj) {
        const int j = q * 32 + jj;
        flip_if(r[j], word, jj);
      }
    }
  } else {
    if constexpr (C::R >= 4) {
      const float4* f = reinterpret_cast<const float4*>(d.flt + tb * (int64_t)C::N);
#pragma unroll
      for (int q = 0; q < C::R / 4; ++q) {
        const float4 v = __ldg(f + q * C::T + t);
        r[4 * q] *= v.x;
        r[4 * q + 1] *= v.y;
        r[4 * q + 2] *= v.z;
        r[4 * q + 3] *= v.w;
      }
    } else {
      const float* f = d.flt + tb * (int64_t)C::N;
#pragma unroll
      for (int j = 0; j < C::R; ++j) r[j] *= __ldg(f + j * C::T + t);
    }
  }
}

template <class C>
__device__ __forceinline__ void xor_signs(float (&r)[C::R], const uint32_t (&w)[C::WORDS]) {
#pragma unroll
  for (int q = 0; q < C::WORDS; ++q)
#pragma unroll
    for (int jj = 0; jj < C::BITS; ++jj) {
      const int j = q * 32 + jj;
      flip_if(r[j], w[q], jj);
    }
}

template <class C>
__device__ __forceinline__ void load_words(uint32_t (&w)[C::WORDS], const uint32_t* base, int64_t tb, int t) {
  const uint32_t* s = base + tb * (int64_t)(C::WORDS * C::T);
#pragma unroll
  for (int q = 0; q < C::WORDS; ++q) w[q] = __ldg(s + q * C::T + t);
}

// The three rounds D1 -> H -> D2 -> H -> D3 -> H of one (table, block) on registers r.
// Start layout B (END_B = false) or A (END_B = true); each H flips the layout.
//  * sign diagonals: all three bit-masks are fetched up front so their L1/L2 latency
//    overlaps the first butterflies (they were the top long-scoreboard stall);
//  * LOG_R == LOG_T (n = 4^k, incl. 1024 and 16384): both halves of every H cover
//    all register bits, so the six half-transforms run as a loop over ONE copy of
//    the butterfly code with a runtime transpose direction — a third of the SASS of
//    the unrolled chain, which keeps the n = 16384 kernel inside the instruction cache.
template <class C, bool END_B, bool SIGNS, bool LODD = C::LOOPED_ODD>
__device__ __forceinline__ void spinner_chain(float (&r)[C::R], float* sm, const VecParams& p, int64_t tb,
                                              int t) {
  constexpr int L0 = END_B ? LAY_A : LAY_B, L1 = END_B ? LAY_B : LAY_A;
  if constexpr (SIGNS && C::LOOPED) {
    // R == T: layout A -> B and B -> A are the same (thread, register) swap
    // (thread t register j <-> thread j register t), and both halves of every H cover
    // all register bits, so D -> H is ONE loop body run three times.
    const uint32_t* w1p = p.d[1][L1].sgn;
    const uint32_t* w2p = p.d[2][L0].sgn;
    uint32_t w[C::WORDS];
    load_words<C>(w, p.d[0][L0].sgn, tb, t);
#pragma unroll 1
    for (int h = 0; h < 3; ++h) {
      xor_signs<C>(r, w);
      if (h < 2) load_words<C>(w, h == 0 ? w1p : w2p, tb, t);  // in flight during the butterflies
      reg_fwht<C::R, 0, C::LOG_R, SPN_F1_REV>(r);
#ifndef SPN_DBG_NOXPOSE  // (bound experiments only: wrong results)
      xpose_A_to_B<C>(r, sm, t);
#endif
      reg_fwht<C::R, 0, C::LOG_R>(r);
    }
  } else if constexpr (SIGNS && LODD) {
    // R == 2T: the same loop with layout B's registers numbered pb(j) (see VCfg::LOOPED_ODD)
    const uint32_t* w1p = p.d[1][L1].sgn;
    const uint32_t* w2p = p.d[2][L0].sgn;
    uint32_t w[C::WORDS];
    load_words<C>(w, p.d[0][L0].sgn, tb, t);
#pragma unroll 1
    for (int h = 0; h < 3; ++h) {
      xor_signs<C>(r, w);
      if (h < 2) load_words<C>(w, h == 0 ? w1p : w2p, tb, t);
      reg_fwht<C::R, 0, C::LOG_R, SPN_F1_REV>(r);
      if ((L0 == LAY_A) != ((h & 1) != 0))
        xpose_A_to_B<C, true>(r, sm, t);
      else
        xpose_B_to_A<C, true>(r, sm, t);
      reg_fwht<C::R, 0, C::LOG_T>(r);
    }
  } else if constexpr (SIGNS) {
    uint32_t w0[C::WORDS], w1[C::WORDS], w2[C::WORDS];
    load_words<C>(w0, p.d[0][L0].sgn, tb, t);
    load_words<C>(w1, p.d[1][L1].sgn, tb, t);
    load_words<C>(w2, p.d[2][L0].sgn, tb, t);
    xor_signs<C>(r, w0);
    if constexpr (END_B) fwht_A_to_B<C>(r, sm, t); else fwht_B_to_A<C>(r, sm, t);
    xor_signs<C>(r, w1);
    if constexpr (END_B) fwht_B_to_A<C>(r, sm, t); else fwht_A_to_B<C>(r, sm, t);
    xor_signs<C>(r, w2);
    if constexpr (END_B) fwht_A_to_B<C>(r, sm, t); else fwht_B_to_A<C>(r, sm, t);
  } else {
    apply_diag<C>(r, p.d[0][L0], p.dsign[0], tb, t);
    if constexpr (END_B) fwht_A_to_B<C>(r, sm, t); else fwht_B_to_A<C>(r, sm, t);
    apply_diag<C>(r, p.d[1][L1], p.dsign[1], tb, t);
    if constexpr (END_B) fwht_B_to_A<C>(r, sm, t); else fwht_A_to_B<C>(r, sm, t);
    apply_diag<C>(r, p.d[2][L0], p.dsign[2], tb, t);
    if constexpr (END_B) fwht_A_to_B<C>(r, sm, t); else fwht_B_to_A<C>(r, sm, t);
  }
}

// Load row v in layout B (coalesced), zero padded beyond n_in (dataset.cpp:162-168).
template <class C, bool PI = false>
__device__ __forceinline__ void load_x_B(float (&r)[C::R], const float* __restrict__ xrow,
                                         int64_t n_in, int t) {
  if (n_in >= C::N) {  // uniform fast path: no padding
#pragma unroll
    for (int j = 0; j < C::R; ++j) r[C::template pb<PI>(j)] = __ldg(xrow + j * C::T + t);
  } else {
#pragma unroll
    for (int j = 0; j < C::R; ++j) {
      const int i = j * C::T + t;
      r[C::template pb<PI>(j)] = (i < n_in) ? __ldg(xrow + i) : 0.0f;
    }
  }
}

// Load row v in layout B of PERMUTED coordinates (OP_APPLY_P, R == T, no padding, 16-B aligned rows):
// the kernel's element e' = j*T + t is the real coordinate e = (j & 3) | (t << 2) | ((j >> 2) << (LOG_T + 2))
// (H_n commutes with the bit permutation; the host permutes the diagonals to match, as for
// OP_EMBED_GAUSS_P), so register quad q of lane t is the four consecutive floats at 4t + q * 4T: one
// coalesced 16-B load each (a warp covers 512 contiguous bytes per instruction).
template <class C>
__device__ __forceinline__ void load_x_perm(float (&r)[C::R], const float* __restrict__ xrow, int t) {
#pragma unroll
  for (int q = 0; q < C::R / 4; ++q) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(xrow + q * 4 * C::T + 4 * t));
    r[4 * q] = v.x;
    r[4 * q + 1] = v.y;
    r[4 * q + 2] = v.z;
    r[4 * q + 3] = v.w;
  }
}

// Per-thread signed argmax over this thread's registers, whose element indices
// increase with j (both layouts).  Branch-free: pass 1 takes max |y| (FMNMX on the
// ALU pipe), pass 2 walks j downward so the FIRST register reaching the max wins
// (strict '>' / smallest index, lsh.cpp:13-18).  Elements with index >= rows are
// excluded.  Returns (|y|max, j*, y[j*]) with j* = -1 if nothing valid.
template <class C>
__device__ __forceinline__ void thread_argmax(const float (&r)[C::R], int first_i, int stride_i,
                                              int rows, float& amax, int& jbest, float& vbest) {
  float m = -1.0f;
  if (first_i + (C::R - 1) * stride_i < rows) {
#pragma unroll
    for (int j = 0; j < C::R; ++j) m = fmaxf(m, fabsf(r[j]));
  } else {
#pragma unroll
    for (int j = 0; j < C::R; ++j)
      if (first_i + j * stride_i < rows) m = fmaxf(m, fabsf(r[j]));
  }
  int jb = -1;
  float vb = 0.0f;
#pragma unroll
  for (int j = C::R - 1; j >= 0; --j) {
    const bool hit = fabsf(r[j]) == m;
    jb = hit ? j : jb;
    vb = hit ? r[j] : vb;
  }
  amax = m;
  jbest = (m >= 0.0f) ? jb : -1;
  vbest = vb;
}

// sin/cos for the random-feature epilogue (kernels.cpp:29-34): __sincosf on the angle t
// itself, i.e. the SFU path (FMUL.RZ by 1/2pi + MUFU.SIN/COS) with no explicit range
// reduction.  Its absolute error grows with |t| (tools/microbench/sincos_acc.cu: max abs
// error 2.4e-6 for |t| <= 20; DESIGN.md §3 lists the measured domain).  The Gaussian embed
// at config-2 scale (x in [0,1]^784, sqrt(n)/sigma = 6.4) gives t ~ N(0, 3.2^2), so |t| <= 20
// holds with > 6 sigma margin and the features meet the 1e-5 relative-L2 bar.
// (A 16-B-store variant of this epilogue — angles re-laid through smem so each lane owns
// four consecutive elements — measured 0.577 vs 0.458 ms on config 2 and was dropped.)
// Permuted-coordinate Gaussian embed (OP_EMBED_GAUSS_P): layout-B register j of lane t
// holds element (j & 3) + 4t + 128 (j >> 2); each register quad is stored as one float4
// (a warp store covers 512 contiguous bytes).
template <class C>
__device__ __forceinline__ void embed_store_perm(const float (&r)[C::R], float* __restrict__ yrow,
                                                 const VecParams& p, int t) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float4 s4, c4;
    __sincosf(r[4 * q], &s4.x, &c4.x);
    __sincosf(r[4 * q + 1], &s4.y, &c4.y);
    __sincosf(r[4 * q + 2], &s4.z, &c4.z);
    __sincosf(r[4 * q + 3], &s4.w, &c4.w);
    // (packed FMUL2 for these measured slower: 0.437 vs 0.431 ms)
    c4.x *= p.norm;
    c4.y *= p.norm;
    c4.z *= p.norm;
    c4.w *= p.norm;
    s4.x *= p.norm;
    s4.y *= p.norm;
    s4.z *= p.norm;
    s4.w *= p.norm;
    const int e = 4 * t + 128 * q;
    __stcs(reinterpret_cast<float4*>(yrow + e), c4);
    __stcs(reinterpret_cast<float4*>(yrow + p.k + e), s4);
  }
}

// Embed epilogue in layout B (element i = j*T + t): coalesced 4-B streaming stores.
template <class C, int OP, bool CHECK>
__device__ __forceinline__ void embed_store(const float (&r)[C::R], float* __restrict__ yrow,
                                            const VecParams& p, int t, int rows) {
#pragma unroll
  for (int j = 0; j < C::R; ++j) {
    const int i = j * C::T + t;
    if (CHECK && i >= rows) continue;
    if constexpr (OP == OP_EMBED_GAUSS) {
      // staged x was pre-scaled by scale*n^-1.5/sigma, so r[j] already is the angle t
      // (kernels.cpp:30); the SFU reduces t itself (FMUL.RZ by 1/2pi + MUFU.SIN/COS).
      // Measured max abs error: 2.4e-6 for |t| <= 20 (tools/microbench/sincos_acc.cu).
      float s, co;
      __sincosf(r[j], &s, &co);
      __stcs(yrow + i, co * p.norm);
      __stcs(yrow + p.k + i, s * p.norm);
    } else {  // OP_EMBED_ANG: sign with sign(0) = +1 (kernels.cpp:23-26)
      __stcs(yrow + i, (r[j] * p.c < 0.0f) ? -1.0f : 1.0f);
    }
  }
}

// Running signed-argmax state (lsh.cpp:9-21): max |y|, ties to the smallest row.
struct ArgBest {
  float a;    // |y| (unscaled)
  int gi;     // row within the table
  float val;  // signed unscaled value
};

__device__ __forceinline__ void argbest_update(ArgBest& b, float v, int gi) {
  const float a = fabsf(v);
  if (a > b.a || (a == b.a && gi < b.gi)) {
    b.a = a;
    b.gi = gi;
    b.val = v;
  }
}

__device__ __forceinline__ void argbest_merge(ArgBest& b, float a, int gi, float val) {
  if (a > b.a || (a == b.a && gi < b.gi)) {
    b.a = a;
    b.gi = gi;
    b.val = val;
  }
}

// Reduce the argmax over the T threads of a group; returns the winner in every thread
// of the group (T <= 32) or in thread 0 of the CTA (T > 32).
template <class C>
__device__ __forceinline__ ArgBest group_argmax(ArgBest b, float* red) {
  constexpr int LIM = C::T < 32 ? C::T : 32;
#pragma unroll
  for (int off = LIM / 2; off > 0; off >>= 1) {
    const float oa = __shfl_xor_sync(0xffffffffu, b.a, off);
    const int og = __shfl_xor_sync(0xffffffffu, b.gi, off);
    const float ov = __shfl_xor_sync(0xffffffffu, b.val, off);
    argbest_merge(b, oa, og, ov);
  }
  if constexpr (C::MULTI_WARP) {
    constexpr int W = C::T / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
      red[w] = b.a;
      reinterpret_cast<int*>(red)[W + w] = b.gi;
      red[2 * W + w] = b.val;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 1; q < W; ++q) argbest_merge(b, red[q], reinterpret_cast<int*>(red)[W + q], red[2 * W + q]);
    }
    __syncthreads();
  }
  return b;
}

// ---- signed argmax of a single-block table (lsh.cpp:9-21) without per-element index
// tracking in every warp.  Element i of register j is first_i + j*stride_i (increasing in
// j); elements with i >= rows are excluded.  Keys order candidates so that the reference
// scan's winner (max |y|, strict '>' keeps the FIRST index on ties) wins.

// max |y| over this thread's valid registers (-1 if none); 8 independent FMNMX chains
template <class C>
__device__ __forceinline__ float thread_absmax(const float (&r)[C::R], int first_i, int stride_i, int rows, bool full) {
  constexpr int K = C::R >= 8 ? 8 : C::R;
  float m[K];
#pragma unroll
  for (int k = 0; k < K; ++k) m[k] = -1.0f;
  if (full) {
#pragma unroll
    for (int j = 0; j < C::R; ++j) m[j % K] = fmaxf(m[j % K], fabsf(r[j]));
  } else {
#pragma unroll
    for (int j = 0; j < C::R; ++j)
      if (first_i + j * stride_i < rows) m[j % K] = fmaxf(m[j % K], fabsf(r[j]));
  }
#pragma unroll
  for (int w = K / 2; w > 0; w >>= 1)
#pragma unroll
    for (int k = 0; k < w; ++k) m[k] = fmaxf(m[k], m[k + w]);
  return m[0];
}

// smallest valid register j with |r[j]| == M and its value (4 independent select chains)
template <class C>
__device__ __forceinline__ void thread_first_hit(const float (&r)[C::R], float M, int first_i, int stride_i, int rows,
                                                 bool full, int& jb, float& vb) {
  constexpr int K = C::R >= 16 ? 4 : 1, S = C::R / K;
  int jk[K];
  float vk[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    jk[k] = -1;
    vk[k] = 0.0f;
#pragma unroll
    for (int j = (k + 1) * S - 1; j >= k * S; --j) {
      const bool hit = fabsf(r[j]) == M && (full || first_i + j * stride_i < rows);
      jk[k] = hit ? j : jk[k];
      vk[k] = hit ? r[j] : vk[k];
    }
  }
  jb = jk[K - 1];
  vb = vk[K - 1];
#pragma unroll
  for (int k = K - 2; k >= 0; --k) {
    jb = jk[k] >= 0 ? jk[k] : jb;
    vb = jk[k] >= 0 ? vk[k] : vb;
  }
}

__device__ __forceinline__ int argmax_key(int i, float v, float c) {
  return (i << 1) | ((v * c < 0.0f) ? 1 : 0);  // sign(0) = +1 (lsh.cpp:20)
}
__device__ __forceinline__ int key_to_id(int key, int64_t k) {
  return key == 0x7fffffff ? key : (key >> 1) + ((key & 1) ? (int)k : 0);
}
// Single-warp groups (T <= 32): group max by shuffles, the lanes holding it search their
// registers, then a shuffle min over keys.  Returns the key in every thread of the group.
// QUAD > 0 (permuted coordinates, OP_APPLY_P): register j holds element (j & 3) + first_i + (j >> 2) * QUAD
// (increasing in j); the caller guarantees every element is a valid row.
template <class C, int QUAD = 0>
__device__ __forceinline__ int group_signed_argmax(const float (&r)[C::R], int first_i, int stride_i, int rows,
                                                   float c) {
  const bool full = QUAD > 0 || first_i + (C::R - 1) * stride_i < rows;
  const float m = thread_absmax<C>(r, first_i, stride_i, rows, full);
  constexpr int LIM = C::T < 32 ? C::T : 32;
  float M = m;
#pragma unroll
  for (int off = LIM / 2; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  const bool cand = m == M && m >= 0.0f;
  int key = 0x7fffffff;
  if (__any_sync(0xffffffffu, cand)) {
    int jb;
    float vb;
    if (full)
      thread_first_hit<C>(r, M, first_i, stride_i, rows, true, jb, vb);
    else
      thread_first_hit<C>(r, M, first_i, stride_i, rows, false, jb, vb);
    if (cand) key = argmax_key(QUAD > 0 ? (jb & 3) + first_i + (jb >> 2) * QUAD : first_i + jb * stride_i, vb, c);
  }
#pragma unroll
  for (int off = LIM / 2; off > 0; off >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, off));
  return key;
}

// Multi-warp groups (T > 32, one group per CTA): CTA max of |y| (one barrier), then only
// the warps holding it search, posting their key into smem slot `par` with a shared
// atomicMin and NO trailing barrier — the kernel takes the slot after the next table's
// transposes (their barriers order the atomics), so the argmax adds one barrier to the
// per-table critical path (c3: 283.6 -> 276.2 ms).  Every warp searching against its own
// warp max with a 64-bit atomicMax key (no barrier at all) measured slower (297 ms).
template <class C>
__device__ __forceinline__ void cta_signed_argmax_post(const float (&r)[C::R], int first_i, int stride_i, int rows,
                                                       float c, float* red, int par) {
  constexpr int W = C::T / 32;
  const bool full = first_i + (C::R - 1) * stride_i < rows;
  const float m = thread_absmax<C>(r, first_i, stride_i, rows, full);
  float M = m;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = M;
  __syncthreads();
  M = red[0];
#pragma unroll
  for (int q = 1; q < W; ++q) M = fmaxf(M, red[q]);
  const bool cand = m == M && m >= 0.0f;
  if (__any_sync(0xffffffffu, cand)) {
    int jb;
    float vb;
    if (full)
      thread_first_hit<C>(r, M, first_i, stride_i, rows, true, jb, vb);
    else
      thread_first_hit<C>(r, M, first_i, stride_i, rows, false, jb, vb);
    if (cand) atomicMin(reinterpret_cast<int*>(red) + W + par, argmax_key(first_i + jb * stride_i, vb, c));
  }
}

// Thread 0: take (and reset) the id posted into slot `par` (after a barrier).
template <class C>
__device__ __forceinline__ int cta_signed_argmax_take(float* red, int par, int64_t k) {
  int* s = reinterpret_cast<int*>(red) + C::T / 32 + par;
  const int key = *s;
  *s = 0x7fffffff;
  return key_to_id(key, k);
}
template <class C>
__device__ __forceinline__ void cta_signed_argmax_init(float* red) {
  if (threadIdx.x == 0) {
    reinterpret_cast<int*>(red)[C::T / 32] = 0x7fffffff;
    reinterpret_cast<int*>(red)[C::T / 32 + 1] = 0x7fffffff;
  }
}

// Issue the cp.async copies of one row (n_in valid floats, zero fill to N) into the
// swizzled staging buffer; 16-B chunk c = t + T*u, coalesced across the group.
template <class C>
__device__ __forceinline__ void stage_x(float* xb, const float* __restrict__ xrow, int64_t n_in, int t) {
#pragma unroll
  for (int u = 0; u < C::R / 4; ++u) {
    const int c = t + C::T * u;
    const int64_t rem = n_in - 4 * (int64_t)c;
    const int bytes = rem >= 4 ? 16 : (rem > 0 ? (int)rem * 4 : 0);
    cp_async16(xb + sw<C>(4 * c), bytes > 0 ? xrow + 4 * c : xrow, bytes);
  }
}

// ------------------------------------------------------------------- kernel

template <int LOG_R, int LOG_T, int OP, bool SIGNS>
__global__ void __launch_bounds__(VCfg<LOG_R, LOG_T>::THREADS, VCfg<LOG_R, LOG_T>::min_ctas(OP))
    spinner_vec_kernel(const VecParams p) {
  // programmatic dependent launch (vec_launch.cuh): let the next kernel on the stream launch, then
  // wait for the previous one (a no-op without the launch attribute)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  using C = VCfg<LOG_R, LOG_T>;
  extern __shared__ __align__(16) float smem[];
  constexpr bool END_B = OP != OP_HASH;  // epilogue needs coalesced layout B
  // embed ops reuse x for every block: stage it in smem with cp.async (16-B chunks,
  // zero-filled past n_in, swizzled like the transpose buffer) and prefetch the next
  // row during the last block.  Needs 16-B aligned rows (p.x_vec_ok).
  constexpr bool STAGE_X = C::xbuf(OP) && C::R >= 4;

  const int t = threadIdx.x & (C::T - 1);
  const int g = threadIdx.x >> LOG_T;
  float* sm = smem + g * C::N * (C::xbuf(OP) ? 2 : 1);
  float* xb = sm + C::N;
  float* red = smem + C::smem_floats(OP) - (C::T > 32 ? 4 * (C::T / 32) : 0);

  const int64_t per_vec = (OP == OP_HASH) ? p.tables : 1;
  const int64_t total = p.batch * per_vec;
  const int64_t stride = (int64_t)gridDim.x * C::GPC;
  constexpr bool APPLY = OP == OP_APPLY || OP == OP_APPLY_P;
  constexpr bool PI = SIGNS && C::looped_odd(OP);  // layout B registers numbered pb(j) (looped R == 2T chain)
  constexpr bool PERM = OP == OP_APPLY_P;  // permuted coordinates: 16-B x loads and y stores
  static_assert(!PERM || (LOG_R == LOG_T && LOG_R >= 2), "permuted apply needs R == T");
  const bool want_ids = (OP == OP_HASH) || (APPLY && p.ids != nullptr);
  const bool staged = STAGE_X && p.x_vec_ok;
  // single-block tables take the two-phase argmax (group_signed_argmax / cta_signed_argmax_*);
  // multi-warp groups post each table's winner into smem and write its id one table later
  const bool fast_ids = want_ids && p.blocks == 1;
  constexpr bool DEFER = C::MULTI_WARP;
  int64_t pend_v = -1, pend_tab = 0;
  bool pend_active = false;
  int par = 0;
  if constexpr (DEFER) cta_signed_argmax_init<C>(red);  // visible after the chain's barriers
  auto emit_id = [&](int64_t vv, int64_t tt, int id) {
    if (p.npeers > 0) {
      const int64_t off = (p.peer_row0 + vv) * p.tables + tt;
      for (int q = 0; q < p.npeers; ++q) p.peers[q][off] = id;
    } else {
      p.ids[vv * p.tables + tt] = id;
    }
  };
  // (DEFER) write the previous table's id: its atomics are ordered by the barriers since
  auto flush_pending = [&]() {
    if (pend_v >= 0 && threadIdx.x == 0) {
      const int id = cta_signed_argmax_take<C>(red, par ^ 1, p.k);
      if (pend_active) emit_id(pend_v, pend_tab, id);
    }
    pend_v = -1;
  };

  if constexpr (STAGE_X) {
    const int64_t item0 = (int64_t)blockIdx.x * C::GPC + g;
    if (staged && item0 < total) stage_x<C>(xb, p.x + item0 * p.ld_x, p.n_in, t);
    cp_async_commit();
  }

  // Work order.  Item-major (default): item = (vector, table) pairs dealt round robin over the
  // grid.  Vector-major (multi-table hash with at least one vector per CTA slot, p.vec_major): a
  // CTA takes a vector and runs all its tables back to back, so the vector is read from HBM once
  // and from L2 for the other tables (item-major lets CTAs drift apart over a 2^20-vector batch
  // and re-read x from HBM: 2.4x the algorithmic bytes at config 3).
  const bool vmaj = OP == OP_HASH && p.vec_major;
  const int64_t units = vmaj ? (p.batch + C::GPC - 1) / C::GPC : (total + C::GPC - 1) / C::GPC;
  int64_t sub = 0;
  for (int64_t u = blockIdx.x; u < units;
       vmaj ? (++sub == per_vec ? (sub = 0, u += gridDim.x) : u) : (u += gridDim.x)) {
    const int64_t base = u * C::GPC;
    const int64_t vg = base + g;  // vector-major: this group's vector
    const int64_t item = vmaj ? vg * per_vec + sub : base + g;
    const bool active = vmaj ? vg < p.batch : item < total;
    const int64_t v = active ? (vmaj ? vg : item / per_vec) : 0;
    const int64_t tab = active ? (vmaj ? sub : item - v * per_vec) : 0;
    const float* xrow = p.x + v * p.ld_x;
#if SPN_APPLY_PREFETCH
    // apply at n >= 2^12: one thread asks L2 for the CTA's next row while this one transforms (a CTA
    // idles through its row's load and there is no spare CTA to cover it: 3 per SM at n = 2^14):
    // apply at n = 2^12 / 2^13 / 2^14 0.69 / 0.50 / 0.50 -> 0.70 / 0.57 / 0.52 of the HBM copy peak.  (The
    // same one-instruction prefetch of the next vector in the 8-table hash: 276 vs 250 ms at config 3 —
    // that kernel has no register to spare.)
    if constexpr (OP == OP_APPLY && C::R >= 64 && C::GPC == 1) {
      const int64_t nv = v + gridDim.x;
      if (threadIdx.x == 0 && p.x_vec_ok && nv < p.batch && active) {
        const uint32_t bytes = static_cast<uint32_t>(min(p.n_in, (int64_t)C::N) * 4) & ~15u;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.x + nv * p.ld_x), "r"(bytes) : "memory");
      }
    }
#endif

    float r[C::R];
    if constexpr (STAGE_X) {
      cp_async_wait_all();
      group_sync<C>();
      if constexpr (OP == OP_EMBED_GAUSS_P) {
        // Permuted coordinates (R = T = 32, n = 1024): the kernel runs on v' = P v with
        // e' = P(e) = ((e >> 2) & 31) | ((e & 3) << 5) | (e & 0x380).  H_n commutes with
        // any bit permutation of the index, so H D' H ... on v' is P (H D H ... v) with
        // the host-permuted diagonals D' = D o P^-1.  What it buys: the final layout B in
        // e'-space gives lane t the elements (j & 3) + 4t + 128 (j >> 2), i.e. four
        // CONSECUTIVE outputs per register quad -> 16-B streaming stores (6.2 vs 5.5 TB/s
        // HBM write rate, tools/microbench/wbw.cu) with no extra transpose.
        // Here: scale x by c/sigma and scatter it from natural to e' order (chunk
        // c = t + 32u holds e = 4c .. 4c+3 -> e' = t + 32 i + 128 u; conflict free).
        static_assert(C::R == 32 && C::T == 32, "permuted embed is the n = 1024 kernel");
        if (staged) {
          float xv[C::R];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 v4 = *reinterpret_cast<const float4*>(xb + sw<C>(4 * (t + 32 * u)));
            xv[4 * u] = v4.x * p.c2;
            xv[4 * u + 1] = v4.y * p.c2;
            xv[4 * u + 2] = v4.z * p.c2;
            xv[4 * u + 3] = v4.w * p.c2;
          }
          __syncwarp();
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int i = 0; i < 4; ++i) xb[sw<C>(t + 32 * i + 128 * u)] = xv[4 * u + i];
          __syncwarp();
        }
      }
      if constexpr (OP == OP_EMBED_GAUSS) {
        // fold scale*n^-1.5/sigma into x once per row (the chain is linear), so the
        // four blocks' epilogues feed sin/cos directly; each thread rescales the chunks
        // it staged (chunk c = t + T*u at sw(4c)).
        if (staged) {
#pragma unroll
          for (int u = 0; u < C::R / 4; ++u) {
            float4* q = reinterpret_cast<float4*>(xb + sw<C>(4 * (t + C::T * u)));
            float4 v4 = *q;
            v4.x *= p.c2;
            v4.y *= p.c2;
            v4.z *= p.c2;
            v4.w *= p.c2;
            *q = v4;
          }
          group_sync<C>();
        }
      }
    }

    ArgBest best{-1.0f, 0x7fffffff, 0.0f};
    int fast_key = 0x7fffffff;
    for (int b = 0; b < p.blocks; ++b) {
      if (STAGE_X && staged) {
        if constexpr (STAGE_X) {
          const Swz<C> z(t);
#pragma unroll
          for (int q = 0; q < C::R / 4; ++q) {
            const float4 xv = *reinterpret_cast<const float4*>(xb + z.A(t, q));
            r[4 * q] = xv.x;
            r[4 * q + 1] = xv.y;
            r[4 * q + 2] = xv.z;
            r[4 * q + 3] = xv.w;
          }
          if (b == p.blocks - 1) {  // x consumed: prefetch the next row into xb
            group_sync<C>();
            const int64_t nxt = item + stride;
            if (nxt < total) stage_x<C>(xb, p.x + nxt * p.ld_x, p.n_in, t);
            cp_async_commit();
          }
        }
      } else {
#ifdef SPN_DBG_NOLOAD  // (bound experiments only: wrong results)
        if (base == (int64_t)blockIdx.x * C::GPC) load_x_B<C, PI>(r, xrow, p.n_in, t);
        else {
#pragma unroll
          for (int j = 0; j < C::R; ++j) r[j] = __int_as_float(0x3f800000 + j * 977 + t * 131 + (int)base);
        }
#else
        if constexpr (PERM)
          load_x_perm<C>(r, xrow, t);
        else
          load_x_B<C, PI>(r, xrow, p.n_in, t);
#endif
        if constexpr (END_B) {
          if constexpr (C::T > 1) xpose_B_to_A<C, PI>(r, sm, t);
        }
        if constexpr (OP == OP_EMBED_GAUSS) {
#pragma unroll
          for (int j = 0; j < C::R; ++j) r[j] *= p.c2;
        }
      }
      const int64_t tb = tab * p.blocks + b;
      const int64_t row0 = (int64_t)b * p.m;
      const int64_t rows = min(p.m, p.k - row0);  // valid rows of this block (stacking, spinner.cpp:272-283)
      spinner_chain<C, END_B, SIGNS, C::looped_odd(OP)>(r, sm, p, tb, t);
      if constexpr (PI && END_B) {  // back to the standard layout-B register order for the epilogue
        float rs[C::R];
#pragma unroll
        for (int j = 0; j < C::R; ++j) rs[j] = r[C::template pb<true>(j)];
#pragma unroll
        for (int j = 0; j < C::R; ++j) r[j] = rs[j];
      }
      if constexpr (!END_B) {
        // layout A: element i = t*R + j, increasing j
        if (fast_ids) {
#ifdef SPN_DBG_NOARGMAX  // (bound experiments only: wrong results)
          float acc = 0.0f;
#pragma unroll
          for (int j = 0; j < C::R; ++j) acc += (j & 1) ? r[j] : 0.0f;
          fast_key = __float_as_int(acc) & 0xffff;
#else
          if constexpr (DEFER) {
            flush_pending();
            cta_signed_argmax_post<C>(r, t * C::R, 1, (int)rows, p.c, red, par);
          } else {
            fast_key = group_signed_argmax<C>(r, t * C::R, 1, (int)rows, p.c);
          }
#endif
        } else {
          float am, vb;
          int jb;
          thread_argmax<C>(r, t * C::R, 1, (int)rows, am, jb, vb);
          if (jb >= 0) argbest_merge(best, am, (int)row0 + t * C::R + jb, vb);
        }
      } else {
        // layout B: element i = j*T + t -> coalesced stores
        float* yrow = p.y + v * p.ld_y + row0;
        if constexpr (PERM) {  // full single-block rows (host-checked): 16-B stores, permuted argmax index
          if (want_ids) fast_key = group_signed_argmax<C, 4 * C::T>(r, 4 * t, 0, (int)rows, p.c);
          if (p.y && active) {
#pragma unroll
            for (int q = 0; q < C::R / 4; ++q)
              __stcs(reinterpret_cast<float4*>(yrow + q * 4 * C::T + 4 * t),
                     make_float4(r[4 * q] * p.c, r[4 * q + 1] * p.c, r[4 * q + 2] * p.c, r[4 * q + 3] * p.c));
          }
          continue;
        }
        if constexpr (OP == OP_APPLY) {
          if (fast_ids) {
            if constexpr (DEFER) {
              flush_pending();
              cta_signed_argmax_post<C>(r, t, C::T, (int)rows, p.c, red, par);
            } else {
              fast_key = group_signed_argmax<C>(r, t, C::T, (int)rows, p.c);
            }
          } else if (want_ids) {
            float am, vb;
            int jb;
            thread_argmax<C>(r, t, C::T, (int)rows, am, jb, vb);
            if (jb >= 0) argbest_merge(best, am, (int)row0 + jb * C::T + t, vb);
          }
          if (p.y && active) {
            // the full-block, no-ReLU case without per-element predicates (config 1)
            if (rows >= C::N && !p.relu) {
#pragma unroll
              for (int j = 0; j < C::R; ++j) __stcs(yrow + j * C::T + t, r[j] * p.c);
            } else {
              const int nrows = (int)rows;
#pragma unroll
              for (int j = 0; j < C::R; ++j) {
                const int i = j * C::T + t;
                float out = r[j] * p.c;
                if (p.relu) out = fmaxf(out, 0.0f);
                if (i < nrows) __stcs(yrow + i, out);
              }
            }
          }
          continue;
        }
        if (!active) continue;
        if constexpr (OP == OP_EMBED_GAUSS_P) {
          embed_store_perm<C>(r, yrow, p, t);  // host guarantees full 1024-row blocks
        } else {
          if (rows >= C::N)
            embed_store<C, OP, false>(r, yrow, p, t, (int)rows);
          else
            embed_store<C, OP, true>(r, yrow, p, t, (int)rows);
        }
      }
    }

    if (want_ids) {
      if (fast_ids && DEFER) {
#ifndef SPN_DBG_NOARGMAX
        pend_v = v;
        pend_tab = tab;
        pend_active = active;
        par ^= 1;
        continue;
#endif
      }
      int id;
      if (fast_ids) {
        id = key_to_id(fast_key, p.k);
      } else {
        best = group_argmax<C>(best, red);
        const float yb = best.val * p.c;
        id = best.gi + ((yb < 0.0f) ? (int)p.k : 0);  // sign(0) = +1 (lsh.cpp:20)
      }
      const bool writer = C::MULTI_WARP ? (threadIdx.x == 0) : (t == 0);
      if (writer && active) emit_id(v, tab, id);
    }
  }
  if constexpr (DEFER) {
    if (fast_ids) {
      __syncthreads();
      flush_pending();
    }
  }
}

}  // namespace spn
