// gram_dmma.cu -- the r x r Gram of a long fp64 factor, B = W W^T (and D = V^T V, the
// same tiles over V's K-major layout)
// (kernels::matmul_abt with X = Y = W, kernels.cpp:24-34; solvers.cpp:83,106,
// 252), on the fp64 tensor-core path (mma.sync m8n8k4 f64, "DMMA").
//
// W is r x K row-major with K = n_local large (262144 at config 4) and r <= 64:
// 2 r^2 K flops over 8 r K bytes -- compute-bound in fp64 (1.07 G fused
// multiply-adds at config 4; 33 TFLOP/s of DFMA on this chip = 65 us).  The
// SIMT tile kernel spends 0.22 ms there (one 64 x 64 tile per block, 4 x 4
// outputs per thread), a fixed cost of every step at EVERY pyramid level, so
// it weighs most on the coarse levels (config 4, level 4: 0.9 ms per step, of
// which B 0.22 ms).  Here:
//   * one DMMA does 8 x 8 x 4 = 256 fused multiply-adds per warp instruction
//     (8 x fewer instructions than DFMA);
//   * the A fragment (rows 8a .. 8a + 7, k .. k + 3) and the B fragment
//     (k .. k + 3, columns 8b .. 8b + 7 of W^T) of m8n8k4 are the SAME registers
//     when both come from W: lane holds W[8 blk + lane / 4][k + lane % 4];
//   * B is symmetric: only the 36 tiles on or above the diagonal are formed
//     (warp w owns row blocks w and 7 - w: 9 tiles each) and mirrored by the
//     epilogue.  Each product W[i][p] W[j][p] is commutative, so the mirrored
//     entry is bit-identical to the one a full computation would give.
// Split-K over the blocks (each a contiguous K range, 64-column tiles staged
// by cp.async into a double-buffered padded shared-memory tile), fp64 partials
// summed in block order by the caller's deterministic epilogue.
//
// Accumulation order differs from the reference's sequential sum, so exact
// mode keeps the SIMT kernel; non-exact runs hold 1e-10 on the error
// trajectory either way (tests/test_gpu_tc.py::test_gram_w_dmma).
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "gram_dmma.hpp"

namespace mlb {
namespace {

constexpr int kR = 64;        // padded rank (rows of the tile)
constexpr int kKC = 64;       // K columns per tile
constexpr int kLd = kKC + 4;  // padded row (544 B: the half-warp's 4 rows land on distinct bank groups)
constexpr int kThreads = 128;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// One warp's share of a block: row blocks RA (tiles RA .. 7) and RB = 7 - RA
// (tiles RB .. 7), 9 tiles, all indices compile-time (the accumulators stay
// in registers).  Every warp of the block runs the same tile loop and
// barriers; only the tile set differs.
template <int RA, bool TRANS, typename Stage>
__device__ __forceinline__ void warp_tiles(const double* tile, int ntiles, Stage& stage, int lane, int r,
                                           double* __restrict__ out) {
  constexpr int RB = 7 - RA;
  double acc[9][2];
#pragma unroll
  for (int i = 0; i < 9; ++i) acc[i][0] = acc[i][1] = 0.0;
  if (ntiles > 0) stage(0);
  for (int it = 0; it < ntiles; ++it) {
    if (it + 1 < ntiles) {
      stage(it + 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    // tile layout: [factor row i][k] (W, row-major r x K) or [k][factor row i] (TRANS: V, K x r row-major)
    const double* src = tile + (size_t)(it & 1) * kR * kLd +
                        (TRANS ? (lane & 3) * kLd + (lane >> 2) : (lane >> 2) * kLd + (lane & 3));
#pragma unroll 4
    for (int k4 = 0; k4 < kKC / 4; ++k4) {
      double f[8];  // fragment of row block b: X[8 b + lane / 4][4 k4 + lane % 4]
#pragma unroll
      for (int b = 0; b < 8; ++b) f[b] = TRANS ? src[k4 * 4 * kLd + b * 8] : src[b * 8 * kLd + k4 * 4];
#pragma unroll
      for (int j = RA; j < 8; ++j) dmma(acc[j - RA][0], acc[j - RA][1], f[RA], f[j]);
#pragma unroll
      for (int j = RB; j < 8; ++j) dmma(acc[8 - RA + j - RB][0], acc[8 - RA + j - RB][1], f[RB], f[j]);
    }
    __syncthreads();  // the buffer is restaged two tiles later
  }
  // epilogue: C fragment of m8n8k4 -- lane holds (row lane / 4, columns
  // 2 (lane % 4), + 1).  Entries on or above the diagonal are written and
  // mirrored (each below-diagonal entry is written once, by its mirror).
  auto put = [&](int i, int c, double v) {
    if (i < r && c < r && c >= i) {
      out[i * r + c] = v;
      if (c > i) out[c * r + i] = v;
    }
  };
#pragma unroll
  for (int j = RA; j < 8; ++j) {
    const int i = RA * 8 + (lane >> 2), c = j * 8 + 2 * (lane & 3);
    put(i, c, acc[j - RA][0]);
    put(i, c + 1, acc[j - RA][1]);
  }
#pragma unroll
  for (int j = RB; j < 8; ++j) {
    const int i = RB * 8 + (lane >> 2), c = j * 8 + 2 * (lane & 3);
    put(i, c, acc[8 - RA + j - RB][0]);
    put(i, c + 1, acc[8 - RA + j - RB][1]);
  }
}

// part[blockIdx.x][i][j] (r x r) = sum over this block's K range of X[i][p] X[j][p], X[i][p] = W[i K + p]
// (TRANS = false: B = W W^T) or V[p r + i] (TRANS = true: D = V^T V, kernels::matmul_atb, kernels.cpp:36-46)
template <bool TRANS>
__global__ void __launch_bounds__(kThreads) k_gram_dmma(const double* __restrict__ W, int r, size_t K, size_t kchunk,
                                                        double* __restrict__ part) {
  extern __shared__ __align__(16) double tile[];  // [2][kR][kLd]
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const size_t kb = (size_t)blockIdx.x * kchunk;
  const size_t ke = kb + kchunk < K ? kb + kchunk : K;
  const int ntiles = kb < ke ? (int)((ke - kb + kKC - 1) / kKC) : 0;
  const bool vec_ok = ((TRANS ? (size_t)r : K) % 2 == 0) && (reinterpret_cast<uintptr_t>(W) % 16 == 0);

  // stage tile `it` (K indices kb + 64 it ..) into buffer it & 1: 16-byte
  // asynchronous copies where the pair lies inside the range, zeros elsewhere
  auto stage = [&](int it) {
    double* dst = tile + (size_t)(it & 1) * kR * kLd;
    const size_t c0 = kb + (size_t)it * kKC;
    if (!TRANS) {
      for (int e = t; e < kR * (kKC / 2); e += kThreads) {
        const int row = e / (kKC / 2), c2 = (e % (kKC / 2)) * 2;
        const size_t col = c0 + c2;
        double* d = dst + row * kLd + c2;
        if (row < r && vec_ok && col + 1 < ke) {
          const uint32_t sa = (uint32_t)__cvta_generic_to_shared(d);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(W + (size_t)row * K + col) : "memory");
        } else {
          d[0] = (row < r && col < ke) ? W[(size_t)row * K + col] : 0.0;
          d[1] = (row < r && col + 1 < ke) ? W[(size_t)row * K + col + 1] : 0.0;
        }
      }
    } else {
      // tile row = K index p, 64 factor entries (r of them real) of V's row p
      for (int e = t; e < kKC * (kR / 2); e += kThreads) {
        const int pr = e / (kR / 2), i2 = (e % (kR / 2)) * 2;
        const size_t p = c0 + pr;
        double* d = dst + pr * kLd + i2;
        if (p < ke && vec_ok && i2 + 1 < r) {
          const uint32_t sa = (uint32_t)__cvta_generic_to_shared(d);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(W + p * (size_t)r + i2) : "memory");
        } else {
          d[0] = (p < ke && i2 < r) ? W[p * (size_t)r + i2] : 0.0;
          d[1] = (p < ke && i2 + 1 < r) ? W[p * (size_t)r + i2 + 1] : 0.0;
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  switch (warp) {
    case 0: warp_tiles<0, TRANS>(tile, ntiles, stage, lane, r, part + (size_t)blockIdx.x * r * r); break;
    case 1: warp_tiles<1, TRANS>(tile, ntiles, stage, lane, r, part + (size_t)blockIdx.x * r * r); break;
    case 2: warp_tiles<2, TRANS>(tile, ntiles, stage, lane, r, part + (size_t)blockIdx.x * r * r); break;
    default: warp_tiles<3, TRANS>(tile, ntiles, stage, lane, r, part + (size_t)blockIdx.x * r * r); break;
  }
}

}  // namespace

bool gram_dmma_supported(size_t r, size_t K) { return r >= 1 && r <= 64 && K >= 2048; }

int gram_dmma_blocks(size_t K, int sm_count) {
  const size_t target = (size_t)sm_count * 3;  // 3 resident blocks per SM (70 KB of shared memory each)
  const size_t kchunk = ((K + target - 1) / target + kKC - 1) / kKC * kKC;
  return (int)((K + kchunk - 1) / kchunk);
}

void gram_dmma(const double* W, size_t r, size_t K, int sm_count, double* part, cudaStream_t s, bool trans) {
  if (!gram_dmma_supported(r, K)) throw std::invalid_argument("gram_dmma: unsupported shape");
  const size_t target = (size_t)sm_count * 3;
  const size_t kchunk = ((K + target - 1) / target + kKC - 1) / kKC * kKC;
  const int blocks = (int)((K + kchunk - 1) / kchunk);
  const size_t smem = 2 * (size_t)kR * kLd * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_gram_dmma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_gram_dmma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " (gram_dmma)");
    attr = true;
  }
  if (trans) k_gram_dmma<true><<<blocks, kThreads, smem, s>>>(W, (int)r, K, kchunk, part);
  else k_gram_dmma<false><<<blocks, kThreads, smem, s>>>(W, (int)r, K, kchunk, part);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " (gram_dmma)");
}

}  // namespace mlb
