// Per-op dispatch between the all-sign and general-diagonal instantiations.
#include "vec_launch.cuh"

namespace spn {

LaunchFn vec_launcher_hash_s(int);
LaunchFn vec_launcher_hash_g(int);
LaunchFn vec_launcher_apply_s(int);
LaunchFn vec_launcher_apply_g(int);
LaunchFn vec_launcher_gauss_s(int);
LaunchFn vec_launcher_gauss_g(int);
LaunchFn vec_launcher_ang_s(int);
LaunchFn vec_launcher_ang_g(int);

LaunchFn vec_launcher_hash(int log_n, int s) { return s ? vec_launcher_hash_s(log_n) : vec_launcher_hash_g(log_n); }
LaunchFn vec_launcher_apply(int log_n, int s) { return s ? vec_launcher_apply_s(log_n) : vec_launcher_apply_g(log_n); }
LaunchFn vec_launcher_gauss(int log_n, int s) { return s ? vec_launcher_gauss_s(log_n) : vec_launcher_gauss_g(log_n); }
LaunchFn vec_launcher_ang(int log_n, int s) { return s ? vec_launcher_ang_s(log_n) : vec_launcher_ang_g(log_n); }
LaunchFn vec_launcher_gauss_perm() { return &launch_vec<10, OP_EMBED_GAUSS_P, true>; }
LaunchFn vec_launcher_apply_perm() { return &launch_vec<10, OP_APPLY_P, true>; }

}  // namespace spn
