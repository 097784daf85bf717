// Instantiations of spinner_vec_kernel<*, *, OP_EMBED_GAUSS, SIGNS=false>, n = 2^1 .. 2^14.
#include "vec_launch.cuh"

namespace spn {

LaunchFn vec_launcher_gauss_g(int log_n) {
  static const auto table = make_vec_table<OP_EMBED_GAUSS, false>(std::make_integer_sequence<int, kMaxLogNVec>{});
  return table[static_cast<size_t>(log_n - 1)];
}

}  // namespace spn
