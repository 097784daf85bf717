// Launch helpers for spinner_vec_kernel.  Each (OP, all-sign-diagonals) pair's 14 size
// instantiations (n = 2^1 .. 2^14) live in their own translation unit
// (vec_op_<op>_<s|g>.cu) so the build compiles them in parallel.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cstdlib>
#include <utility>

#include "spinner_vec.cuh"

namespace spn {

constexpr int kMaxLogNVec = 14;  // fused single-kernel path: n <= 2^14

using LaunchFn = cudaError_t (*)(const VecParams&, cudaStream_t, int, int64_t);

// signs = 1: every diagonal is ±1 (bit-packed XOR path only, smaller kernel)
LaunchFn vec_launcher_hash(int log_n, int signs);
LaunchFn vec_launcher_apply(int log_n, int signs);
LaunchFn vec_launcher_gauss(int log_n, int signs);
LaunchFn vec_launcher_ang(int log_n, int signs);
// n = 1024 Gaussian embed in permuted coordinates (16-B output stores), sign diagonals
LaunchFn vec_launcher_gauss_perm();
// n = 1024 apply + ids in permuted coordinates (16-B x loads and y stores), sign diagonals
LaunchFn vec_launcher_apply_perm();

// Persistent grid: min(work, SMs x resident CTAs per SM).
template <int LOG_N, int OP, bool SIGNS>
cudaError_t launch_vec(const VecParams& p, cudaStream_t s, int sms, int64_t items) {
  using C = VCfg<(LOG_N + 1) / 2, LOG_N / 2>;
  auto kern = spinner_vec_kernel<C::LOG_R, C::LOG_T, OP, SIGNS>;
  static std::atomic<int> occ_cache{0};
  int occ = occ_cache.load();
  if (occ == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::smem_bytes(OP)));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::smem_bytes(OP));
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    occ_cache.store(occ);
  }
  int64_t ctas = (items + C::GPC - 1) / C::GPC;
  VecParams q = p;
  // multi-table hash over a batch that fills the persistent grid by vectors alone: vector-major
  // order (every table of a vector in one CTA, back to back; the vector stays in L2)
  const int64_t vslots = (p.batch + C::GPC - 1) / C::GPC;
  q.vec_major = OP == OP_HASH && p.tables > 1 && vslots >= int64_t(sms) * occ;
  if (q.vec_major) ctas = vslots;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ctas, int64_t(sms) * occ));
  // programmatic dependent launch: the kernel lets its successor on the stream launch at once (the
  // successor's CTAs take SM slots as ours retire and wait in griddepcontrol.wait for our completion),
  // hiding the launch gap between back-to-back calls (c1 in a CUDA graph)
  static const bool pdl = [] {
    const char* e = std::getenv("SPN_VEC_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::smem_bytes(OP);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, q);
}

template <int OP, bool SIGNS, int... L>
std::array<LaunchFn, sizeof...(L)> make_vec_table(std::integer_sequence<int, L...>) {
  return {{&launch_vec<L + 1, OP, SIGNS>...}};
}

}  // namespace spn
