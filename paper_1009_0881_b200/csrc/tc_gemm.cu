// tc_gemm.cu -- tcgen05 3xTF32 M-streaming products (placeholder until the
// kernels land: the engine falls back to the SIMT fp64-accumulating GEMMs;
// forcing the tensor path fails loudly).
#include <stdexcept>

#include "tc_gemm.hpp"

namespace mlb {

TcGemm* make_tc_gemm(bool allowed, bool forced) {
  (void)allowed;
  if (forced) throw std::invalid_argument("tcgen05 path not available in this build");
  return nullptr;
}

}  // namespace mlb
