// Entry points shared between translation units of the library (not exported).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/spinners_b200.h"

namespace spn {

int plan_device(const spn_plan* p);
// First-m sketch of diag(row_scale) A by a SketchOperator plan (row_scale: device fp32 [n_in]).
spn_status plan_sketch_scaled(const spn_plan* p, const float* a, int64_t n_in, int64_t d, int64_t ld_a,
                              int64_t m_out, double norm, const float* row_scale, float* out, int64_t ld_out,
                              cudaStream_t s);

}  // namespace spn
