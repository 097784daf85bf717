// Instantiations of spinner_vec_kernel<*, *, OP_HASH, SIGNS=false>, n = 2^1 .. 2^14.
#include "vec_launch.cuh"

namespace spn {

LaunchFn vec_launcher_hash_g(int log_n) {
  static const auto table = make_vec_table<OP_HASH, false>(std::make_integer_sequence<int, kMaxLogNVec>{});
  return table[static_cast<size_t>(log_n - 1)];
}

}  // namespace spn
