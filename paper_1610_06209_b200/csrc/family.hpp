// Circulant-family variants and the Gaussian dense baseline (family.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/spinners_b200.h"
#include "host_params.hpp"

namespace spn {

struct FamilyPlan;

bool family_variant(int v);
// draw_tail + the front diagonals (spinner.cpp:92-151): d1, d2 [n] (not for dense), tail [n]
// (circulant / skew row, Toeplitz first column), trow [n] (Toeplitz first row), dense [m * n].
void family_realize(int variant, int64_t n, int64_t m, uint64_t spec_seed, double* d1, double* d2, double* tail,
                    double* trow, double* dense);
spn_status family_build(FamilyPlan** out, int variant, int64_t n, int64_t m, int64_t k, int64_t tables,
                        int64_t blocks, const std::vector<double>* d, const std::vector<double>& trow,
                        const std::vector<double>& dense, double scale, int device);
void family_destroy(FamilyPlan* f);
// op: 0 apply (float y [batch][ld_out], relu), 1 hash (int32 ids [batch][tables]),
//     2 gaussian embed (float [batch][ld_out >= 2k]), 3 angular embed (float [batch][ld_out >= k])
spn_status family_run(const FamilyPlan* f, int op, const float* x, int64_t batch, int64_t ld_x, int64_t n_in,
                      void* out, int64_t ld_out, int relu, double sigma, cudaStream_t s);

}  // namespace spn
