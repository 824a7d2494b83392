// tc_gemm.hpp -- tcgen05 (5th-gen tensor core) 3xTF32 kernels for the two
// M-streaming products at fp32 storage (tc_gemm.cu):
//   A (m x r, fp64) = M (m x n) W^T      and      C (r x n, fp64) = V^T M.
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace mlb {

// device-allocation epoch (engine.cu): bumped on every buffer (re)allocation
extern std::atomic<uint64_t> g_dev_epoch;

class TcGemm {
 public:
  virtual ~TcGemm() = default;
  virtual bool active() const = 0;
  // shape supported by the kernels (r <= 64, 16-byte aligned rows)
  virtual bool supports(size_t m, size_t n, size_t r) const = 0;
  // policy: use the tensor path for this level (forced, or large enough)
  virtual bool wants(size_t m, size_t n, size_t r) const = 0;
  virtual void mwt(const float* M, const float* W, size_t m, size_t n, size_t r, double* A, cudaStream_t s,
                   long* launches) = 0;
  virtual void vtm(const float* V, const float* M, size_t m, size_t n, size_t r, double* C, cudaStream_t s,
                   long* launches) = 0;
  // ||M - V W||_F^2 into the device scalar out[0] (3xTF32 V W, fp32 residuals
  // summed in fp64); same shape support as the products
  virtual void sqerr(const float* M, const float* V, const float* W, size_t m, size_t n, size_t r, double* out,
                     cudaStream_t s, long* launches) = 0;
  void sqerr(const double*, const double*, const double*, size_t, size_t, size_t, double*, cudaStream_t, long*) {}
  // fp64 storage never takes the tensor path (kept for the templated engine)
  void mwt(const double*, const double*, size_t, size_t, size_t, double*, cudaStream_t, long*) {}
  void vtm(const double*, const double*, size_t, size_t, size_t, double*, cudaStream_t, long*) {}
};

// allowed: fp32 storage and not forced to SIMT; forced: the caller demanded
// tcgen05 for every supported shape.
TcGemm* make_tc_gemm(bool allowed, bool forced);

}  // namespace mlb
