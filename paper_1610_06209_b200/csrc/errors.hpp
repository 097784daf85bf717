// Thread-local last-error message shared by the C ABI and the pass drivers.
#pragma once

#include <cuda_runtime.h>

#include <exception>
#include <new>
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

// Exception barrier for the C ABI: no C++ exception may cross an extern "C" entry point
// (host std::vector growth -> std::bad_alloc, std::thread -> std::system_error, ...).
// Every exported function body is wrapped as  { SPN_TRY ... SPN_CATCH }.
#define SPN_TRY try {
#define SPN_CATCH                                                                              \
  }                                                                                            \
  catch (const std::bad_alloc&) {                                                              \
    return ::spn::set_error(SPN_ENOMEM, "host allocation failed");                             \
  }                                                                                            \
  catch (const std::exception& ex_) {                                                          \
    return ::spn::set_error(SPN_EINVAL, std::string("internal error: ") + ex_.what());          \
  }                                                                                            \
  catch (...) {                                                                                \
    return ::spn::set_error(SPN_EINVAL, "internal error: unknown exception");                  \
  }
