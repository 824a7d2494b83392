// hals_reg.cu -- register-resident HALS sweeps at a compile-time rank
// (hals_step, proj/src/solvers.cpp:101-141).  Kept in their own translation
// unit: the fully unrolled r x r sweeps take minutes to compile.
#include <cuda_runtime.h>

#include <cstddef>
#include <stdexcept>
#include <string>

#include "hals_reg.hpp"

namespace mlb {
namespace {

template <typename T>
__device__ __forceinline__ T to_t(double v);
template <>
__device__ __forceinline__ float to_t<float>(double v) { return __double2float_rn(v); }
template <>
__device__ __forceinline__ double to_t<double>(double v) { return v; }
// reference: `s -= a * b` (solvers.cpp:118,136), unfused
__device__ __forceinline__ double msub(double acc, double a, double b) { return __dsub_rn(acc, __dmul_rn(a, b)); }

// FAST sweeps: kChains independent fused dot chains per update (the l-sum is
// latency-bound at 12 warps per SM and 168 registers), summed pairwise.
// Measured r02, W sweep at n = 262144: 4 chains + a per-thread reciprocal
// 0.49-0.52 ms; 8 chains + per-block reciprocals 0.43-0.47 ms.  Not kept: the
// Gram as constant-bank / uniform-register operand (LDCU.128 per pair: 0.56
// ms), one 384-thread block per SM with a barrier per update against
// instruction-fetch stalls (no_instructions is ncu's top stall reason on the
// ~160 KB unrolled sweep: neutral for W, worse for V).
constexpr int kChains = 8;
__device__ __forceinline__ double chain_sum(const double (&p)[kChains]) {
  double s[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) s[c] = p[c];
#pragma unroll
  for (int w = kChains; w > 1; w /= 2)
#pragma unroll
    for (int c = 0; c < w / 2; ++c) s[c] = s[2 * c] + s[2 * c + 1];
  return s[0];
}

// Register-resident HALS sweeps for a compile-time rank R (the config-4 rank):
// the factor row / column lives in R registers instead of shared memory, the
// Gram row for update k is read as broadcast from shared memory, and both k
// and l loops are unrolled.  Same arithmetic and operation order as k_hals_v /
// k_hals_w (the reference's, unfused), so results are bitwise identical;
// ~10x fewer shared-memory accesses.
// FAST (non-exact runs): the l-sum as kChains interleaved fused chains and the
// division by a per-block reciprocal -- the reference-order chain is 2R
// dependent fp64 operations per update (~1000 cycles of latency at R = 64),
// the interleaved one R / kChains fused ones.
template <typename T, int R, bool FAST = false>
__global__ void __launch_bounds__(128) k_hals_v_reg(const double* __restrict__ A, const double* __restrict__ B,
                                                    T* __restrict__ V, size_t m, int* __restrict__ degenerate) {
  __shared__ double Bt[R * R];  // Bt[k][l] = B[l][k]: row k is the column the update reads
  __shared__ double inv[R];     // FAST: reciprocal pivots, once per block (a per-thread fp64 division per k
                                // was a quarter of the sweep's instructions, ncu r02)
  const int t = threadIdx.x;
  for (int e = t; e < R * R; e += blockDim.x) Bt[e] = B[(e % R) * R + e / R];
  if (FAST && t < R) {
    const double d = B[t * R + t];
    inv[t] = d > 0.0 ? 1.0 / d : 0.0;
  }
  __syncthreads();
  const size_t i = (size_t)blockIdx.x * blockDim.x + t;
  const bool act = i < m;
  double v[R];
#pragma unroll
  for (int l = 0; l < R; ++l) v[l] = act ? (double)V[i * R + l] : 0.0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const double bkk = Bt[k * R + k];
    if (bkk <= 0.0) {
      if (degenerate && blockIdx.x == 0 && t == 0) atomicAdd(degenerate, 1);
      continue;
    }
    const double a = act ? A[i * R + k] : 0.0;
    double q;
    if (FAST) {
      double p[kChains];
#pragma unroll
      for (int c = 0; c < kChains; ++c) p[c] = 0.0;
#pragma unroll
      for (int l = 0; l < R; ++l) p[l % kChains] = fma(v[l], Bt[k * R + l], p[l % kChains]);
      q = (fma(v[k], bkk, a) - chain_sum(p)) * inv[k];
    } else {
      double num = __dadd_rn(a, __dmul_rn(v[k], bkk));
#pragma unroll
      for (int l = 0; l < R; ++l) num = msub(num, v[l], Bt[k * R + l]);
      q = num / bkk;
    }
    v[k] = q > 0.0 ? q : 0.0;
  }
  if (act)
#pragma unroll
    for (int l = 0; l < R; ++l) V[i * R + l] = to_t<T>(v[l]);
}

template <typename T, int R, bool FAST = false>
__global__ void __launch_bounds__(128) k_hals_w_reg(const double* __restrict__ Cm, const double* __restrict__ D,
                                                    T* __restrict__ W, size_t n, int* __restrict__ degenerate) {
  __shared__ double Ds[R * R];
  __shared__ double inv[R];  // FAST: reciprocal pivots, once per block
  const int t = threadIdx.x;
  for (int e = t; e < R * R; e += blockDim.x) Ds[e] = D[e];
  if (FAST && t < R) {
    const double d = D[t * R + t];
    inv[t] = d > 0.0 ? 1.0 / d : 0.0;
  }
  __syncthreads();
  const size_t j = (size_t)blockIdx.x * blockDim.x + t;
  const bool act = j < n;
  double w[R];
#pragma unroll
  for (int l = 0; l < R; ++l) w[l] = act ? (double)W[(size_t)l * n + j] : 0.0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const double dkk = Ds[k * R + k];
    if (dkk <= 0.0) {
      if (degenerate && blockIdx.x == 0 && t == 0) atomicAdd(degenerate, 1);
      continue;
    }
    const double c = act ? Cm[(size_t)k * n + j] : 0.0;
    double q;
    if (FAST) {
      double p[kChains];
#pragma unroll
      for (int cc = 0; cc < kChains; ++cc) p[cc] = 0.0;
#pragma unroll
      for (int l = 0; l < R; ++l) p[l % kChains] = fma(Ds[k * R + l], w[l], p[l % kChains]);
      q = (fma(dkk, w[k], c) - chain_sum(p)) * inv[k];
    } else {
      double num = __dadd_rn(c, __dmul_rn(dkk, w[k]));
#pragma unroll
      for (int l = 0; l < R; ++l) num = msub(num, Ds[k * R + l], w[l]);
      q = num / dkk;
    }
    w[k] = q > 0.0 ? q : 0.0;
  }
  if (act)
#pragma unroll
    for (int l = 0; l < R; ++l) W[(size_t)l * n + j] = to_t<T>(w[l]);
}


// MU (solvers.cpp:79-99) at a compile-time rank, same unfused arithmetic and
// order as k_mu_v / k_mu_w: V(i,:) *= A(i,:) / max(V(i,:) B, 1e-16) with the
// row's old values (Jacobi within the half) held in registers.
__device__ __forceinline__ double mu_floor(double v) { return v < 1e-16 ? 1e-16 : v; }

template <typename T, int R>
__global__ void __launch_bounds__(128) k_mu_v_reg(const double* __restrict__ A, const double* __restrict__ B,
                                                  T* __restrict__ V, size_t m) {
  __shared__ double Bt[R * R];  // Bt[j][p] = B[p][j]
  const int t = threadIdx.x;
  for (int e = t; e < R * R; e += blockDim.x) Bt[e] = B[(e % R) * R + e / R];
  __syncthreads();
  const size_t i = (size_t)blockIdx.x * blockDim.x + t;
  if (i >= m) return;
  double v[R];
#pragma unroll
  for (int l = 0; l < R; ++l) v[l] = (double)V[i * R + l];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < R; ++q) s = __dadd_rn(s, __dmul_rn(v[q], Bt[j * R + q]));
    V[i * R + j] = to_t<T>(__dmul_rn(v[j], A[i * R + j] / mu_floor(s)));
  }
}

template <typename T, int R>
__global__ void __launch_bounds__(128) k_mu_w_reg(const double* __restrict__ Cm, const double* __restrict__ D,
                                                  T* __restrict__ W, size_t n) {
  __shared__ double Ds[R * R];
  const int t = threadIdx.x;
  for (int e = t; e < R * R; e += blockDim.x) Ds[e] = D[e];
  __syncthreads();
  const size_t j = (size_t)blockIdx.x * blockDim.x + t;
  if (j >= n) return;
  double w[R];
#pragma unroll
  for (int l = 0; l < R; ++l) w[l] = (double)W[(size_t)l * n + j];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < R; ++q) s = __dadd_rn(s, __dmul_rn(Ds[k * R + q], w[q]));
    W[(size_t)k * n + j] = to_t<T>(__dmul_rn(w[k], Cm[(size_t)k * n + j] / mu_floor(s)));
  }
}

template <int R>
void launch_v(bool fast, const double* A, const double* B, double* V, size_t m, int* deg, cudaStream_t s) {
  const dim3 g((unsigned)((m + 127) / 128));
  if (fast) k_hals_v_reg<double, R, true><<<g, 128, 0, s>>>(A, B, V, m, deg);
  else k_hals_v_reg<double, R><<<g, 128, 0, s>>>(A, B, V, m, deg);
}
template <int R>
void launch_w(bool fast, const double* C, const double* D, double* W, size_t n, int* deg, cudaStream_t s) {
  const dim3 g((unsigned)((n + 127) / 128));
  if (fast) k_hals_w_reg<double, R, true><<<g, 128, 0, s>>>(C, D, W, n, deg);
  else k_hals_w_reg<double, R><<<g, 128, 0, s>>>(C, D, W, n, deg);
}

void check(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " (hals_reg)");
}

}  // namespace

// compiled rank: the config-4 rank (an r = 49 instantiation gained ~3 % on
// config 3 for +1.5 min of build time, so it is not built)
bool hals_reg_supported(size_t r) { return r == 64; }
bool mu_reg_supported(size_t r) { return r == 64; }

void mu_v_reg(size_t r, const double* A, const double* B, double* V, size_t m, cudaStream_t s) {
  if (r != 64) throw std::invalid_argument("mu_v_reg: unsupported rank");
  const dim3 g((unsigned)((m + 127) / 128));
  k_mu_v_reg<double, 64><<<g, 128, 0, s>>>(A, B, V, m);
  check(cudaGetLastError());
}

void mu_w_reg(size_t r, const double* C, const double* D, double* W, size_t n, cudaStream_t s) {
  if (r != 64) throw std::invalid_argument("mu_w_reg: unsupported rank");
  const dim3 g((unsigned)((n + 127) / 128));
  k_mu_w_reg<double, 64><<<g, 128, 0, s>>>(C, D, W, n);
  check(cudaGetLastError());
}

void hals_v_reg(size_t r, bool fast, const double* A, const double* B, double* V, size_t m, int* deg,
                cudaStream_t s) {
  if (r == 64) launch_v<64>(fast, A, B, V, m, deg, s);
  else throw std::invalid_argument("hals_v_reg: unsupported rank");
  check(cudaGetLastError());
}

void hals_w_reg(size_t r, bool fast, const double* C, const double* D, double* W, size_t n, int* deg,
                cudaStream_t s) {
  if (r == 64) launch_w<64>(fast, C, D, W, n, deg, s);
  else throw std::invalid_argument("hals_w_reg: unsupported rank");
  check(cudaGetLastError());
}

}  // namespace mlb
