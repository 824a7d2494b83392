// restrict_tma.hpp -- the TMA-pipelined restriction of all columns of a level
// (restrict_tma.cu; reference: GridHierarchy::build, transfer.cpp:155-174).
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

namespace mlb {

struct RestrictArgs {
  const void* X;       // (h w) x ncols, fp32 or fp64
  void* Y;             // (hc wc) x ncols
  int h, w, hc, wc;
  size_t ncols;
  bool in_f64;         // X is fp64 (then Y is fp64, fp64 math)
  bool out_f64;        // fp32 X restricted into fp64 storage (fp64 math)
  bool f64math;        // fp32 -> fp32 in the reference's unfused fp64 arithmetic (exact mode)
};

// loads the kernels (call once per process, at session creation)
void restrict_tma_prepare();
// 16-byte aligned rows at least four 512-byte slabs wide
bool restrict_tma_supported(const RestrictArgs& a);
// strip: coarse pixel rows per CTA; nslots: ring depth in fine pixel columns
void restrict_tma(const RestrictArgs& a, int strip, int nslots, cudaStream_t s);

}  // namespace mlb
