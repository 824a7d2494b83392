// ix_gemm.hpp -- the two M-streaming products of the fp32-storage path on the
// tcgen05 integer tensor cores (ix_gemm.cu):
//   A (m x r, fp64) = M (m x n) W^T      and      C (r x n, fp64) = V^T M
// with M's fp32 entries and the fp64 factors on per-row 31-bit fixed-point
// grids, split into four signed 8-bit digits; the digit products accumulate
// in int32 TMEM exactly, so the only error is the (unbiased) rounding of
// each operand to its grid (exact for M entries within 2^7 of the row max).
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace mlb {

class TcGemm {
 public:
  virtual ~TcGemm() = default;
  // hash of the work-buffer pointers (engine.cu graph_sig: a captured step
  // graph is valid while they are unchanged)
  virtual uint64_t signature() const = 0;
  // shape supported by the kernels (r <= 64, 16-byte aligned rows)
  virtual bool supports(size_t m, size_t n, size_t r) const = 0;
  // policy: use the tensor path for this level (forced, or large enough)
  virtual bool wants(size_t m, size_t n, size_t r) const = 0;
  // per-level statistics of a (constant) M, once per level: the maximum of
  // every row (m floats) and of every column (n floats).  They fix the
  // fixed-point scale of each MMA row: rows of M in A = M W^T, columns of M
  // in C = V^T M.
  // sqpart (optional): level_stats_blocks(m, n) fp64 partial sums of squares,
  // one per block, whose sum in index order is ||M||_F^2 (the same pass).
  virtual size_t level_stats_blocks(size_t m, size_t n) const = 0;
  virtual void level_stats(const float* M, size_t m, size_t n, float* rowmax, float* colmax, double* sqpart,
                           cudaStream_t s, long* launches) = 0;
  // M fp32 (the streamed operand), factors fp64 (the engine's factor
  // storage; rounded once to the factor's fixed-point grid)
  virtual void mwt(const float* M, const float* rowmax, const double* W, size_t m, size_t n, size_t r, double* A,
                   cudaStream_t s, long* launches) = 0;
  virtual void vtm(const double* V, const float* M, const float* colmax, size_t m, size_t n, size_t r, double* C,
                   cudaStream_t s, long* launches) = 0;
  // fp64 storage of M never takes the tensor path (kept for the templated engine)
  void mwt(const double*, const float*, const double*, size_t, size_t, size_t, double*, cudaStream_t, long*) {}
  void vtm(const double*, const double*, const float*, size_t, size_t, size_t, double*, cudaStream_t, long*) {}
};

// allowed: fp32 storage and not forced to SIMT; forced: the caller demanded
// the tensor path for every supported shape.
TcGemm* make_tc_gemm(bool allowed, bool forced);

}  // namespace mlb
