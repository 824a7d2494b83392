// hals_reg.hpp -- register-resident HALS sweeps (hals_reg.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace mlb {
bool hals_reg_supported(size_t r);
bool mu_reg_supported(size_t r);
// V (m x r, fp64) rows swept with A (m x r) and B (r x r), fp64; fast
// (non-exact fp32-M runs): interleaved fused dot chains
void hals_v_reg(size_t r, bool fast, const double* A, const double* B, double* V, size_t m, int* deg,
                cudaStream_t s);
// W (r x n, fp64) columns swept with C (r x n) and D (r x r), fp64
void hals_w_reg(size_t r, bool fast, const double* C, const double* D, double* W, size_t n, int* deg,
                cudaStream_t s);
// MU updates (solvers.cpp:79-99), same operands, register-resident rows/columns
void mu_v_reg(size_t r, const double* A, const double* B, double* V, size_t m, cudaStream_t s);
void mu_w_reg(size_t r, const double* C, const double* D, double* W, size_t n, cudaStream_t s);
}  // namespace mlb
