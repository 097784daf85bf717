// Instantiations of spinner_vec_kernel<*, *, OP_EMBED_ANG, SIGNS=true>, n = 2^1 .. 2^14.
#include "vec_launch.cuh"

namespace spn {

LaunchFn vec_launcher_ang_s(int log_n) {
  static const auto table = make_vec_table<OP_EMBED_ANG, true>(std::make_integer_sequence<int, kMaxLogNVec>{});
  return table[static_cast<size_t>(log_n - 1)];
}

}  // namespace spn
