// hals_reg.hpp -- register-resident HALS sweeps (hals_reg.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace mlb {
bool hals_reg_supported(size_t r);
bool mu_reg_supported(size_t r);
// V (m x r, T = f32 ? float : double) rows swept with A (m x r) and B (r x r), fp64;
// fast (fp32 storage, non-exact runs): interleaved fused dot chains
void hals_v_reg(size_t r, bool f32, bool fast, const double* A, const double* B, void* V, size_t m, int* deg,
                cudaStream_t s);
// W (r x n) columns swept with C (r x n) and D (r x r), fp64
void hals_w_reg(size_t r, bool f32, bool fast, const double* C, const double* D, void* W, size_t n, int* deg,
                cudaStream_t s);
// MU updates (solvers.cpp:79-99), same operands, register-resident rows/columns
void mu_v_reg(size_t r, bool f32, const double* A, const double* B, void* V, size_t m, cudaStream_t s);
void mu_w_reg(size_t r, bool f32, const double* C, const double* D, void* W, size_t n, cudaStream_t s);
}  // namespace mlb
