// gram_dmma.hpp -- B = W W^T of a wide fp64 factor on the fp64 tensor-core
// path (gram_dmma.cu; reference: kernels::matmul_abt, kernels.cpp:24-34).
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

namespace mlb {
// r <= 64 and a contraction long enough to fill the GPU
bool gram_dmma_supported(size_t r, size_t K);
// number of split-K partials gram_dmma writes (r x r fp64 each)
int gram_dmma_blocks(size_t K, int sm_count);
// part[b] = the b-th K range's Gram, b < gram_dmma_blocks(K, sm_count).  trans = false: W W^T of W (r x K
// row-major); trans = true: V^T V of V (K x r row-major)
void gram_dmma(const double* W, size_t r, size_t K, int sm_count, double* part, cudaStream_t s, bool trans = false);
}  // namespace mlb
