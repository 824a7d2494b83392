// hals_dmma.hpp -- the blocked fp64 tensor-core HALS W sweep (hals_dmma.cu;
// reference: hals_step, solvers.cpp:124-141), non-exact runs at r <= 64.
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

namespace mlb {
bool hals_w_dmma_supported(size_t r, size_t n);
// W (r x n, fp64; r <= 64) columns swept with C (r x n) and D (r x r), fp64
void hals_w_dmma(size_t r, const double* C, const double* D, double* W, size_t n, int* deg, cudaStream_t s);
// V (m x r row-major, fp64) rows swept with A (m x r) and B (r x r): hals_step's V half (solvers.cpp:105-122)
bool hals_v_dmma_supported(size_t r, size_t m);
void hals_v_dmma(size_t r, const double* A, const double* B, double* V, size_t m, int* deg, cudaStream_t s);
// MU updates (mu_step, solvers.cpp:79-99) of long factors on the same tiles, non-exact runs
bool mu_dmma_supported(size_t r, size_t count);
void mu_v_dmma(size_t r, const double* A, const double* B, double* V, size_t m, cudaStream_t s);
void mu_w_dmma(size_t r, const double* C, const double* D, double* W, size_t n, cudaStream_t s);
}  // namespace mlb
