// hals_dmma.cu -- the HALS sweeps at the config-4 rank (r = 64) for wide / tall
// factors (written for W; the V half is the same kernel over V's layout), blocked onto the fp64 tensor-core path (hals_step's W half,
// proj/src/solvers.cpp:124-141), non-exact runs only.
//
// Per column j of W the reference runs r sequential projected updates
//     w_k <- max(0, (C_kj + D_kk w_k - sum_l D_kl w_l) / D_kk)
//          = max(0, (C_kj - sum_{l != k} D_kl w_l) / D_kk),        k = 0 .. r-1
// (Gauss-Seidel: w_l already updated for l < k).  The thread-per-column
// register sweep (hals_reg.cu) issues r^2 = 4096 dependent-chain DFMAs and
// half as many shared-memory loads per column and runs latency- and
// instruction-fetch-bound: 0.45 ms per sweep at n = 262144 -- a fixed cost of
// every step at every pyramid level.  Here the updates are taken in blocks of
// 8: for block b the contributions of all l OUTSIDE the block,
//     T_kj = C_kj - sum_{l not in block} D_kl w_l        (8 k x 8 columns x 56 l)
// are 14 DMMAs (mma.sync m8n8k4 f64) per 8-column tile, and only the 8 x 8
// inside of the block stays sequential.
//
// Layout.  The product is formed transposed, (8 columns x 4 l) . (4 l x 8 k):
// the A fragment is the lane's own w registers (lane holds column lane / 4,
// l = 4 q + lane % 4 for the 16 chunks q), the B fragment is -D from shared
// memory, and the C fragment puts T_kj for column lane / 4 and k = 2 (lane % 4),
// + 1 in the same QUAD of lanes that holds the column's w: the sequential
// part of a block is two DFMAs, a quad reduction (two shuffles) and a select
// per update, the warp's column tiles interleaved.  A warp owns 16 columns (2
// tiles), a lane 32 doubles of W.
//
// Measured (r02, n = 262144, same box): 0.28 ms against 0.45-0.47 ms for the
// register sweep (0.39-0.41 ms with 4 tiles per warp: ncu, profiles/README.md,
// showed 242 registers, 8 warps per SM, stalls on the block's C loads and the
// fixed-latency chain of the in-block updates -- it is occupancy that pays); an up-front L2 prefetch of the warp's C
// slice measured slower (0.42 ms) and is not kept.
//
// The accumulation order differs from the reference's (and from the FAST
// register sweep's); exact mode and fp64 sessions never take this kernel.
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "hals_dmma.hpp"

namespace mlb {
namespace {

constexpr int R = 64;
constexpr int kLd = R + 4;  // padded -D row: a half-warp's 4 rows on distinct bank groups
// 8-column tiles per warp.  Measured r02 (W sweep, n = 262144, same box): 4 tiles (242 registers, 8 warps
// per SM) 0.41 ms; 3 tiles 0.38; 2 tiles (135 registers, 12 warps) 0.28; 1 tile 0.29-0.32; forcing 4 or 6
// blocks per SM through launch bounds 0.30-0.35.
constexpr int kTiles = 2;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// IS_W: the factor is W (64 x n, element (l, column j) at l n + j) with H = C (64 x n) and G = D;
// otherwise V (m x 64 row-major: "column" = row i of V, element (l, i) at i 64 + l) with H = A (m x 64)
// and G = B, whose entry for update k and term l is B[l][k] (the -G tile is stored transposed then).
template <bool IS_W>
__global__ void __launch_bounds__(128) k_hals_dmma(const double* __restrict__ Cm, const double* __restrict__ D,
                                                   double* __restrict__ W, size_t n, int r,
                                                   int* __restrict__ degenerate) {
  // r <= 64: the factor's rows r .. 63 are zero padding (never loaded or stored; their updates are skipped)
  auto at = [n, r](int l, size_t j) { return IS_W ? (size_t)l * n + j : j * (size_t)r + (size_t)l; };
  __shared__ double nD[R * kLd];  // -D with a zero diagonal
  __shared__ double inv[R];       // 1 / D_kk, 0 where D_kk <= 0 (the update is skipped, solvers.cpp:127)
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int e = t; e < R * R; e += blockDim.x) {
    const int k = e / R, l = e % R;
    nD[(IS_W ? k * kLd + l : l * kLd + k)] = (k == l || k >= r || l >= r) ? 0.0 : -D[k * r + l];
  }
  if (t < R) {
    const double d = t < r ? D[t * r + t] : 0.0;
    inv[t] = d > 0.0 ? 1.0 / d : 0.0;
    if (t < r && !(d > 0.0) && degenerate && blockIdx.x == 0) atomicAdd(degenerate, 1);
  }
  __syncthreads();
  const int lr = lane >> 2, lc = lane & 3;  // column within a tile, l (and k pair) within a chunk
  const size_t j0 = ((size_t)blockIdx.x * 4 + warp) * (8 * kTiles);
  size_t col[kTiles];
  bool act[kTiles];
#pragma unroll
  for (int ti = 0; ti < kTiles; ++ti) {
    col[ti] = j0 + (size_t)ti * 8 + lr;
    act[ti] = col[ti] < n;
  }
  // w[ti][q]: column col[ti], element l = 4 q + lc
  double w[kTiles][16];
#pragma unroll
  for (int ti = 0; ti < kTiles; ++ti)
#pragma unroll
    for (int q = 0; q < 16; ++q) w[ti][q] = (act[ti] && 4 * q + lc < r) ? W[at(4 * q + lc, col[ti])] : 0.0;

#pragma unroll
  for (int b = 0; b < 8; ++b) {
    if (8 * b >= r) break;  // padding blocks (warp-uniform)
    // T = C - sum over l outside the block: accumulators start at C (k = 8 b + 2 lc, + 1)
    double acc[kTiles][2];
#pragma unroll
    for (int ti = 0; ti < kTiles; ++ti) {
      acc[ti][0] = (act[ti] && 8 * b + 2 * lc < r) ? Cm[at(8 * b + 2 * lc, col[ti])] : 0.0;
      acc[ti][1] = (act[ti] && 8 * b + 2 * lc + 1 < r) ? Cm[at(8 * b + 2 * lc + 1, col[ti])] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (q == 2 * b || q == 2 * b + 1) continue;
      if (4 * q >= r) continue;  // all-zero padding chunk (warp-uniform)
      const double bf = nD[(8 * b + lr) * kLd + 4 * q + lc];  // B fragment: -D[k = 8 b + lane / 4][l = 4 q + lane % 4]
#pragma unroll
      for (int ti = 0; ti < kTiles; ++ti) dmma(acc[ti][0], acc[ti][1], w[ti][q], bf);
    }
    // the block's 8 sequential updates
#pragma unroll
    for (int kl = 0; kl < 8; ++kl) {
      const int k = 8 * b + kl;
      const double d0 = nD[k * kLd + 8 * b + lc], d1 = nD[k * kLd + 8 * b + 4 + lc];  // -D[k][the lane's two l]
      const double ik = inv[k];
      double tot[kTiles];
#pragma unroll
      for (int ti = 0; ti < kTiles; ++ti) {
        double p = lc == kl / 2 ? acc[ti][kl & 1] : 0.0;  // the lane holding T_k contributes it
        p = fma(d0, w[ti][2 * b], p);
        p = fma(d1, w[ti][2 * b + 1], p);
        p += __shfl_xor_sync(0xffffffffu, p, 1);
        p += __shfl_xor_sync(0xffffffffu, p, 2);
        tot[ti] = p;
      }
#pragma unroll
      for (int ti = 0; ti < kTiles; ++ti) {
        const double q = tot[ti] * ik;
        const double wn = q > 0.0 ? q : 0.0;
        // the lane holding w_k (l = k: chunk 2 b + kl / 4, lc = kl % 4) takes the new value
        if (lc == (kl & 3) && ik != 0.0) w[ti][2 * b + kl / 4] = wn;
      }
    }
  }
#pragma unroll
  for (int ti = 0; ti < kTiles; ++ti)
    if (act[ti])
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (4 * q + lc < r) W[at(4 * q + lc, col[ti])] = w[ti][q];
}

// MU (mu_step, solvers.cpp:79-99) through the same tiles: the update
//     f_k <- f_k H_k / max((G f)_k, 1e-16)        (Jacobi: the old f throughout)
// has no sequential part at all -- (G f) for the warp's 16 columns is 16 x 8 DMMAs, and the quad
// shuffles bring each sum to the lane that holds f_k.  IS_W as above (W against D, V against B).
template <bool IS_W>
__global__ void __launch_bounds__(128) k_mu_dmma(const double* __restrict__ H, const double* __restrict__ G,
                                                 double* __restrict__ F, size_t n, int r) {
  __shared__ double Gs[R * kLd];  // Gs[k][l] = the Gram entry of output k and term l
  auto at = [n, r](int l, size_t j) { return IS_W ? (size_t)l * n + j : j * (size_t)r + (size_t)l; };
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int e = t; e < R * R; e += blockDim.x) {
    const int k = e / R, l = e % R;
    Gs[k * kLd + l] = (k >= r || l >= r) ? 0.0 : (IS_W ? G[k * r + l] : G[l * r + k]);
  }
  __syncthreads();
  const int lr = lane >> 2, lc = lane & 3;
  const size_t j0 = ((size_t)blockIdx.x * 4 + warp) * (8 * kTiles);
  size_t col[kTiles];
  bool act[kTiles];
#pragma unroll
  for (int ti = 0; ti < kTiles; ++ti) {
    col[ti] = j0 + (size_t)ti * 8 + lr;
    act[ti] = col[ti] < n;
  }
  double w[kTiles][16];
#pragma unroll
  for (int ti = 0; ti < kTiles; ++ti)
#pragma unroll
    for (int q = 0; q < 16; ++q) w[ti][q] = (act[ti] && 4 * q + lc < r) ? F[at(4 * q + lc, col[ti])] : 0.0;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    if (8 * b >= r) break;
    double acc[kTiles][2];
#pragma unroll
    for (int ti = 0; ti < kTiles; ++ti) acc[ti][0] = acc[ti][1] = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (4 * q >= r) continue;
      const double bf = Gs[(8 * b + lr) * kLd + 4 * q + lc];
#pragma unroll
      for (int ti = 0; ti < kTiles; ++ti) dmma(acc[ti][0], acc[ti][1], w[ti][q], bf);
    }
    // the lane's two elements of the block: k = 8 b + 4 h + lc, h = 0, 1; their sums sit in quad lane
    // 2 h + lc / 2, register lc % 2
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int src = (lane & ~3) | (2 * h + (lc >> 1));
      const int k = 8 * b + 4 * h + lc;
#pragma unroll
      for (int ti = 0; ti < kTiles; ++ti) {
        const double s0 = __shfl_sync(0xffffffffu, acc[ti][0], src), s1 = __shfl_sync(0xffffffffu, acc[ti][1], src);
        const double sk = (lc & 1) ? s1 : s0;
        if (act[ti] && k < r) {
          const size_t a = at(k, col[ti]);
          F[a] = w[ti][2 * b + h] * (H[a] / (sk < 1e-16 ? 1e-16 : sk));
        }
      }
    }
  }
}

}  // namespace

// r = 64 from a few hundred rows / columns; smaller ranks (zero-padded to 64: config 3's r = 49 spends a
// quarter of the tensor work on padding) where the factor is long enough to pay for it
bool hals_w_dmma_supported(size_t r, size_t n) { return r >= 8 && r <= 64 && n >= 4096; }
bool hals_v_dmma_supported(size_t r, size_t m) { return r >= 8 && r <= 64 && ((r == 64 && m >= 256) || m >= 4096); }

void hals_w_dmma(size_t r, const double* C, const double* D, double* W, size_t n, int* deg, cudaStream_t s) {
  const unsigned blocks = (unsigned)((n + 32 * kTiles - 1) / (32 * kTiles));
  k_hals_dmma<true><<<blocks, 128, 0, s>>>(C, D, W, n, (int)r, deg);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " (hals_w_dmma)");
}

void hals_v_dmma(size_t r, const double* A, const double* B, double* V, size_t m, int* deg, cudaStream_t s) {
  const unsigned blocks = (unsigned)((m + 32 * kTiles - 1) / (32 * kTiles));
  k_hals_dmma<false><<<blocks, 128, 0, s>>>(A, B, V, m, (int)r, deg);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " (hals_v_dmma)");
}

}  // namespace mlb

namespace mlb {
bool mu_dmma_supported(size_t r, size_t count) { return r >= 8 && r <= 64 && count >= 4096; }
void mu_v_dmma(size_t r, const double* A, const double* B, double* V, size_t m, cudaStream_t s) {
  k_mu_dmma<false><<<(unsigned)((m + 32 * kTiles - 1) / (32 * kTiles)), 128, 0, s>>>(A, B, V, m, (int)r);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " (mu_v_dmma)");
}
void mu_w_dmma(size_t r, const double* C, const double* D, double* W, size_t n, cudaStream_t s) {
  k_mu_dmma<true><<<(unsigned)((n + 32 * kTiles - 1) / (32 * kTiles)), 128, 0, s>>>(C, D, W, n, (int)r);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " (mu_w_dmma)");
}
}  // namespace mlb
