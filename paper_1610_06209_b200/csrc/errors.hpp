// Thread-local last-error message shared by the C ABI and the pass drivers.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "../../include/spinners_b200.h"

namespace spn {

inline std::string& last_error() {
  static thread_local std::string msg;
  return msg;
}

inline spn_status set_error(spn_status st, const std::string& msg) {
  last_error() = msg;
  return st;
}

inline spn_status cuda_error(cudaError_t e, const char* where) {
  return set_error(e == cudaErrorMemoryAllocation ? SPN_ENOMEM : SPN_ECUDA,
                   std::string(where) + ": " + cudaGetErrorString(e));
}

}  // namespace spn
