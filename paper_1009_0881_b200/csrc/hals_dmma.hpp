// hals_dmma.hpp -- the blocked fp64 tensor-core HALS W sweep (hals_dmma.cu;
// reference: hals_step, solvers.cpp:124-141), non-exact runs at r = 64.
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

namespace mlb {
bool hals_w_dmma_supported(size_t r, size_t n);
// W (64 x n, fp64) columns swept with C (64 x n) and D (64 x 64), fp64
void hals_w_dmma(const double* C, const double* D, double* W, size_t n, int* deg, cudaStream_t s);
// V (m x 64 row-major, fp64) rows swept with A (m x 64) and B (64 x 64): hals_step's V half (solvers.cpp:105-122)
bool hals_v_dmma_supported(size_t r, size_t m);
void hals_v_dmma(const double* A, const double* B, double* V, size_t m, int* deg, cudaStream_t s);
}  // namespace mlb
