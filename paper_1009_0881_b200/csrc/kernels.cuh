// kernels.cuh -- SIMT CUDA kernels of the multilevel NMF solver path (sm_100a).
//
// Storage type T is float or double (M, V, W); every accumulation and every
// r x r / m x r / r x n intermediate (A = M W^T, B = W W^T, C = V^T M,
// D = V^T V) is fp64.  fp32 products are exact in fp64, so the fp32 path is
// "fp64 arithmetic on fp32 storage" (the most accurate
// fp32 variant).
//
// EXACT = true reproduces the reference's floating-point operation order
// (no FMA contraction, sequential K accumulation, no split-K), so an fp64 run
// is bit-identical to the reference CPU build (proj/src/kernels.cpp,
// solvers.cpp, transfer.cpp).  EXACT = false uses FMA and split-K for
// parallelism; parity is then within the stated tolerance.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace mlb {

template <typename T>
__device__ __forceinline__ T to_t(double v);
template <>
__device__ __forceinline__ float to_t<float>(double v) { return __double2float_rn(v); }
template <>
__device__ __forceinline__ double to_t<double>(double v) { return v; }

template <bool EXACT>
__device__ __forceinline__ double madd(double acc, double a, double b) {
  if constexpr (EXACT) return __dadd_rn(acc, __dmul_rn(a, b));
  else return fma(a, b, acc);
}

// reference: `s -= a * b` (solvers.cpp:118,136) -- always unfused, these are
// O((m+n) r^2) sweeps, not the hot GEMMs.
__device__ __forceinline__ double msub(double acc, double a, double b) {
  return __dsub_rn(acc, __dmul_rn(a, b));
}

// ---------------------------------------------------------------------------
// SplitMix64 (proj/include/mlnmf/matrix.hpp:76-95), counter form: the c-th
// (0-based) output of Rng(seed) is mix(seed + (c+1) * gamma).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t sm64_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ double sm64_uniform(uint64_t seed, uint64_t c) {
  return (double)(sm64_mix(seed + (c + 1) * 0x9E3779B97F4A7C15ULL) >> 11) * 0x1.0p-53;
}

// ---------------------------------------------------------------------------
// Tall-skinny GEMMs.  Tiles 64 x 64 outputs, K step 16 in two stages, 256
// threads, 4x4 outputs per thread; fp64 accumulators; operand tiles staged
// in shared memory as fp64.  Each output accumulates over p in ascending
// order within its K chunk (the EXACT variants follow the reference order).
// ---------------------------------------------------------------------------
constexpr int GT = 64;   // output tile edge
constexpr int GK = 32;   // K granule of the split-K chunking (host side)
constexpr int GKS = 16;  // K step of the two-stage kernels (2 x 2 x 16 x 65 doubles of static smem)

// part[z][i][k] = sum_{p in split z} X[i][p] * Y[k][p]
//   X: rows x K (row-major, ld = K), Y: ny x K (row-major, ld = K).
//   (A = M W^T with X = M, Y = W; B = W W^T with X = Y = W.)
// TC: the output tile's width along Y (32 / 48 / 64; ny = r is narrow)
// Stacked form (one launch for A and B of a half-iteration): rows >= rows0
// come from a second operand X1 (fp64, rows - rows0 rows of length K), so
// X = M, X1 = Y = W gives [A; B] = [M; W] W^T.  rows0 = rows: X alone.
template <typename TX, typename TY, bool EXACT, int TC = GT>
__global__ void __launch_bounds__(256) k_gemm_abt(const TX* __restrict__ X, const double* __restrict__ X1,
                                                  size_t rows0, const TY* __restrict__ Y, size_t rows, size_t ny,
                                                  size_t K, size_t kchunk, double* __restrict__ part) {
  // two stages: the next K step's operands are loaded into registers while
  // the current one is multiplied (one barrier per step; the single-stage
  // version exposed an L2 round trip per 32-wide K step)
  constexpr int NB = TC / 16;             // outputs per thread along Y
  __shared__ double Xs[2][GKS][GT + 1];
  __shared__ double Ys[2][GKS][TC + 1];
  constexpr int PQ = (GT * GKS) / 256;    // X elements per thread and stage
  constexpr int PQY = (TC * GKS) / 256;   // Y elements per thread and stage
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const size_t i0 = (size_t)blockIdx.x * GT, k0 = (size_t)blockIdx.y * TC;
  const size_t kb = (size_t)blockIdx.z * kchunk;
  const size_t ke = kb + kchunk < K ? kb + kchunk : K;
  double acc[4][NB];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[a][b] = 0.0;
  double rx[PQ], ry[PQY];
  auto fetch = [&](size_t p0) {
#pragma unroll
    for (int q = 0; q < PQ; ++q) {
      const int e = tid + 256 * q, rr = e / GKS, pp = e % GKS;
      const size_t p = p0 + pp, gi = i0 + rr;
      rx[q] = (gi < rows && p < ke) ? (gi < rows0 ? (double)X[gi * K + p] : X1[(gi - rows0) * K + p]) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < PQY; ++q) {
      const int e = tid + 256 * q, rr = e / GKS, pp = e % GKS;
      const size_t p = p0 + pp, gk = k0 + rr;
      ry[q] = (gk < ny && p < ke) ? (double)Y[gk * K + p] : 0.0;
    }
  };
  fetch(kb);
  int buf = 0;
  for (size_t p0 = kb; p0 < ke; p0 += GKS, buf ^= 1) {
#pragma unroll
    for (int q = 0; q < PQ; ++q) {
      const int e = tid + 256 * q, rr = e / GKS, pp = e % GKS;
      Xs[buf][pp][rr] = rx[q];
    }
#pragma unroll
    for (int q = 0; q < PQY; ++q) {
      const int e = tid + 256 * q, rr = e / GKS, pp = e % GKS;
      Ys[buf][pp][rr] = ry[q];
    }
    __syncthreads();
    if (p0 + GKS < ke) fetch(p0 + GKS);
#pragma unroll
    for (int kk = 0; kk < GKS; ++kk) {
      double xa[4], yb[NB];
#pragma unroll
      for (int a = 0; a < 4; ++a) xa[a] = Xs[buf][kk][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < NB; ++b) yb[b] = Ys[buf][kk][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b) acc[a][b] = madd<EXACT>(acc[a][b], xa[a], yb[b]);
    }
  }
  double* out = part + (size_t)blockIdx.z * rows * ny;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const size_t gi = i0 + ty + 16 * a;
    if (gi >= rows) continue;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const size_t gk = k0 + tx + 16 * b;
      if (gk < ny) out[gi * ny + gk] = acc[a][b];
    }
  }
}

// part[z][k][j] = sum_{i in split z} V[i][k] * X[i][j]
//   V: K x r (row-major), X: K x ncols (row-major).
//   (C = V^T M with X = M; D = V^T V with X = V, ncols = r.)
// TR: the output tile's height along r (32 / 48 / 64)
// Stacked form (one launch for C and D): columns >= ncols0 come from a second
// operand X1 (fp64, K x (ncols - ncols0)), so X = M, X1 = V gives
// [C | D] = V^T [M | V].  ncols0 = ncols: X alone.
template <typename TV, typename TX, bool EXACT, int TR = GT>
__global__ void __launch_bounds__(256) k_gemm_atb(const TV* __restrict__ V, const TX* __restrict__ X,
                                                  const double* __restrict__ X1, size_t ncols0, size_t K, size_t r,
                                                  size_t ncols, size_t kchunk, double* __restrict__ part) {
  constexpr int NA = TR / 16;            // outputs per thread along r
  __shared__ double Xs[2][GKS][GT + 1];  // two stages, as k_gemm_abt
  __shared__ double Vs[2][GKS][TR + 1];
  constexpr int PQ = (GT * GKS) / 256;
  constexpr int PQV = (TR * GKS) / 256;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const size_t j0 = (size_t)blockIdx.x * GT, k0 = (size_t)blockIdx.y * TR;
  const size_t ib = (size_t)blockIdx.z * kchunk;
  const size_t ie = ib + kchunk < K ? ib + kchunk : K;
  double acc[NA][4];
#pragma unroll
  for (int a = 0; a < NA; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  double rx[PQ], rv[PQV];
  auto fetch = [&](size_t p0) {
#pragma unroll
    for (int q = 0; q < PQ; ++q) {
      const int e = tid + 256 * q, ii = e / GT, cc = e % GT;
      const size_t i = p0 + ii, gj = j0 + cc;
      rx[q] = (i < ie && gj < ncols)
                  ? (gj < ncols0 ? (double)X[i * ncols0 + gj] : X1[i * (ncols - ncols0) + (gj - ncols0)])
                  : 0.0;
    }
#pragma unroll
    for (int q = 0; q < PQV; ++q) {
      const int e = tid + 256 * q, ii = e / TR, cc = e % TR;
      const size_t i = p0 + ii, gk = k0 + cc;
      rv[q] = (i < ie && gk < r) ? (double)V[i * r + gk] : 0.0;
    }
  };
  fetch(ib);
  int buf = 0;
  for (size_t p0 = ib; p0 < ie; p0 += GKS, buf ^= 1) {
#pragma unroll
    for (int q = 0; q < PQ; ++q) {
      const int e = tid + 256 * q, ii = e / GT, cc = e % GT;
      Xs[buf][ii][cc] = rx[q];
    }
#pragma unroll
    for (int q = 0; q < PQV; ++q) {
      const int e = tid + 256 * q, ii = e / TR, cc = e % TR;
      Vs[buf][ii][cc] = rv[q];
    }
    __syncthreads();
    if (p0 + GKS < ie) fetch(p0 + GKS);
#pragma unroll
    for (int ii = 0; ii < GKS; ++ii) {
      double va[NA], xb[4];
#pragma unroll
      for (int a = 0; a < NA; ++a) va[a] = Vs[buf][ii][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) xb[b] = Xs[buf][ii][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < NA; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = madd<EXACT>(acc[a][b], va[a], xb[b]);
    }
  }
  double* out = part + (size_t)blockIdx.z * r * ncols;
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    const size_t gk = k0 + ty + 16 * a;
    if (gk >= r) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const size_t gj = j0 + tx + 16 * b;
      if (gj < ncols) out[gk * ncols + gj] = acc[a][b];
    }
  }
}

// out[e] = sum_z part[z][e], z ascending (deterministic split-K epilogue).
__global__ void k_reduce_splits(const double* __restrict__ part, size_t count, int splits,
                                double* __restrict__ out) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (size_t)gridDim.x * blockDim.x) {
    double s = part[e];
    for (int z = 1; z < splits; ++z) s += part[(size_t)z * count + e];
    out[e] = s;
  }
}

// The stacked products' epilogue: element e = row * rl + col of the stacked
// partials goes to out0 or out1.  by_row: rows < cut form out0 (cut x rl),
// the rest out1 ([A; B]); otherwise columns < cut form out0 (rows x cut),
// the rest out1 (rows x (rl - cut)) ([C | D]).
__device__ __forceinline__ double* stacked_dst(size_t e, size_t rl, size_t cut, int by_row, double* out0,
                                               double* out1) {
  if (by_row) return e < cut * rl ? out0 + e : out1 + (e - cut * rl);
  const size_t row = e / rl, col = e - row * rl;
  return col < cut ? out0 + row * cut + col : out1 + row * (rl - cut) + (col - cut);
}
// z ascending, as k_reduce_splits
__global__ void k_reduce_splits2(const double* __restrict__ part, size_t count, int splits, size_t rl, size_t cut,
                                 int by_row, double* __restrict__ out0, double* __restrict__ out1) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (size_t)gridDim.x * blockDim.x) {
    double s = part[e];
    for (int z = 1; z < splits; ++z) s += part[(size_t)z * count + e];
    *stacked_dst(e, rl, cut, by_row, out0, out1) = s;
  }
}
// 8 groups of splits per output, as k_reduce_splits_wide
__global__ void __launch_bounds__(256) k_reduce_splits2_wide(const double* __restrict__ part, size_t count,
                                                             int splits, size_t rl, size_t cut, int by_row,
                                                             double* __restrict__ out0, double* __restrict__ out1) {
  __shared__ double ps[8][33];
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const size_t e = (size_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (e < count)
    for (int z = q; z < splits; z += 8) s += part[(size_t)z * count + e];
  ps[q][lane] = s;
  __syncthreads();
  if (q == 0 && e < count) {
    double t = ps[0][lane];
    for (int g = 1; g < 8; ++g) t += ps[g][lane];
    *stacked_dst(e, rl, cut, by_row, out0, out1) = t;
  }
}

// Same sum with the splits spread over 8 thread groups (many splits, few
// outputs: r x r Grams over long K): block = 32 consecutive outputs x 8
// groups; group q sums splits q, q + 8, ...; the 8 partials are added in
// group order.  Deterministic; a different association than k_reduce_splits.
__global__ void __launch_bounds__(256) k_reduce_splits_wide(const double* __restrict__ part, size_t count,
                                                            int splits, double* __restrict__ out) {
  __shared__ double ps[8][33];
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const size_t e = (size_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (e < count)
    for (int z = q; z < splits; z += 8) s += part[(size_t)z * count + e];
  ps[q][lane] = s;
  __syncthreads();
  if (q == 0 && e < count) {
    double t = ps[0][lane];
    for (int g = 1; g < 8; ++g) t += ps[g][lane];
    out[e] = t;
  }
}

// ---------------------------------------------------------------------------
// HALS sweeps (solvers.cpp:101-141).  One thread per row of V (resp. column
// of W); the r x r Gram in shared memory; the thread's row/column held in
// shared memory as fp64, layout [l][thread] (bank-conflict free).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_hals_v(const double* __restrict__ A, const double* __restrict__ B, T* __restrict__ V,
                         size_t m, int r, int* __restrict__ degenerate, double* __restrict__ gws) {
  // gws (ranks too large for shared memory): the Gram is read from global
  // memory (L2-resident) and the block's rows live in gws[block][l][thread]
  extern __shared__ double sm[];
  const int bd = blockDim.x, t = threadIdx.x;
  const double* Bs = gws ? B : sm;
  double* vs = gws ? gws + (size_t)blockIdx.x * bd * r : sm + (size_t)r * r;
  if (!gws)
    for (int e = t; e < r * r; e += bd) sm[e] = B[e];
  const size_t i = (size_t)blockIdx.x * bd + t;
  const bool act = i < m;
  if (act)
    for (int l = 0; l < r; ++l) vs[l * bd + t] = (double)V[i * r + l];
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    const double bkk = Bs[k * r + k];
    if (bkk <= 0.0) {
      if (degenerate && blockIdx.x == 0 && t == 0) atomicAdd(degenerate, 1);
      continue;
    }
    if (!act) continue;
    double num = __dadd_rn(A[i * r + k], __dmul_rn(vs[k * bd + t], bkk));
    for (int l = 0; l < r; ++l) num = msub(num, vs[l * bd + t], Bs[l * r + k]);
    const double q = num / bkk;
    vs[k * bd + t] = q > 0.0 ? q : 0.0;  // std::max(0.0, q)
  }
  if (act)
    for (int l = 0; l < r; ++l) V[i * r + l] = to_t<T>(vs[l * bd + t]);
}

template <typename T>
__global__ void k_hals_w(const double* __restrict__ Cm, const double* __restrict__ D, T* __restrict__ W,
                         size_t n, int r, int* __restrict__ degenerate, double* __restrict__ gws) {
  extern __shared__ double sm[];
  const int bd = blockDim.x, t = threadIdx.x;
  const double* Ds = gws ? D : sm;
  double* ws = gws ? gws + (size_t)blockIdx.x * bd * r : sm + (size_t)r * r;
  if (!gws)
    for (int e = t; e < r * r; e += bd) sm[e] = D[e];
  const size_t j = (size_t)blockIdx.x * bd + t;
  const bool act = j < n;
  if (act)
    for (int l = 0; l < r; ++l) ws[l * bd + t] = (double)W[(size_t)l * n + j];
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    const double dkk = Ds[k * r + k];
    if (dkk <= 0.0) {
      if (degenerate && blockIdx.x == 0 && t == 0) atomicAdd(degenerate, 1);
      continue;
    }
    if (!act) continue;
    double num = __dadd_rn(Cm[(size_t)k * n + j], __dmul_rn(dkk, ws[k * bd + t]));
    for (int l = 0; l < r; ++l) num = msub(num, Ds[k * r + l], ws[l * bd + t]);
    const double q = num / dkk;
    ws[k * bd + t] = q > 0.0 ? q : 0.0;
  }
  if (act)
    for (int l = 0; l < r; ++l) W[(size_t)l * n + j] = to_t<T>(ws[l * bd + t]);
}

// Warp-per-row / warp-per-column HALS sweeps for few rows / columns (non-exact
// runs on the small configs, where one thread per column leaves the GPU idle:
// config 3 has n = 165).  Lanes hold elements l and l + 32 (r <= 64); each of
// the r sequential updates is a warp-wide dot product (shuffle reduction) --
// a different association than the reference's sequential sum, so exact mode
// keeps the thread-per-row kernels.
__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// rows of V (m x r): x_k <- max(0, (A_ik + x_k G_kk - sum_l x_l G_lk) / G_kk)
// One warp per row, or per pair of rows interleaved when there are more rows
// than resident warps: each sequential k step is a shuffle-reduction chain
// (~200 cycles of latency), so a second independent row fills the gaps.  Lanes hold x_l and A_il for l = lane, lane + 32;
// the blocks are persistent over row pairs so the Gram and its diagonal
// reciprocals are staged once per block, and the rows of A are loaded before
// the k loop.  Non-exact mode only (tree-reduced dots, reciprocal of G_kk).
// The W half is the same update on columns of W with C and D (CT = true:
// element (k, j) at k * n + j).
template <typename T, bool CT, bool TWO>
__device__ __forceinline__ void hals_warp_rows(const double* __restrict__ A, const double* Gs, const double* Ginv,
                                               T* __restrict__ V, size_t m, int r, size_t i, size_t i2) {
  const int lane = threadIdx.x & 31;
  auto at = [&](size_t row, int k) -> size_t { return CT ? (size_t)k * m + row : row * (size_t)r + k; };
  double x0 = lane < r ? (double)V[at(i, lane)] : 0.0;
  double x1 = lane + 32 < r ? (double)V[at(i, lane + 32)] : 0.0;
  double y0 = TWO && lane < r ? (double)V[at(i2, lane)] : 0.0;
  double y1 = TWO && lane + 32 < r ? (double)V[at(i2, lane + 32)] : 0.0;
  const double a0 = lane < r ? A[at(i, lane)] : 0.0;
  const double a1 = lane + 32 < r ? A[at(i, lane + 32)] : 0.0;
  const double b0 = TWO && lane < r ? A[at(i2, lane)] : 0.0;
  const double b1 = TWO && lane + 32 < r ? A[at(i2, lane + 32)] : 0.0;
  for (int k = 0; k < r; ++k) {
    const double gkk = Gs[k * r + k];
    if (gkk <= 0.0) continue;
    // column k of G for rows of V, row k of D for columns of W
    const double g0 = lane < r ? (CT ? Gs[k * r + lane] : Gs[lane * r + k]) : 0.0;
    const double g1 = lane + 32 < r ? (CT ? Gs[k * r + lane + 32] : Gs[(lane + 32) * r + k]) : 0.0;
    double pa = fma(x1, g1, x0 * g0), pb = TWO ? fma(y1, g1, y0 * g0) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      pa += __shfl_xor_sync(0xffffffffu, pa, o);
      if (TWO) pb += __shfl_xor_sync(0xffffffffu, pb, o);
    }
    const int src = k & 31;
    const double xk = __shfl_sync(0xffffffffu, k < 32 ? x0 : x1, src);
    const double ak = __shfl_sync(0xffffffffu, k < 32 ? a0 : a1, src);
    const double qa = (ak + xk * gkk - pa) * Ginv[k];
    double qb = 0.0;
    if (TWO) {
      const double yk = __shfl_sync(0xffffffffu, k < 32 ? y0 : y1, src);
      const double bk = __shfl_sync(0xffffffffu, k < 32 ? b0 : b1, src);
      qb = (bk + yk * gkk - pb) * Ginv[k];
    }
    if (lane == src) {
      if (k < 32) x0 = qa > 0.0 ? qa : 0.0, y0 = qb > 0.0 ? qb : 0.0;
      else x1 = qa > 0.0 ? qa : 0.0, y1 = qb > 0.0 ? qb : 0.0;
    }
  }
  if (lane < r) V[at(i, lane)] = to_t<T>(x0);
  if (lane + 32 < r) V[at(i, lane + 32)] = to_t<T>(x1);
  if (TWO && lane < r) V[at(i2, lane)] = to_t<T>(y0);
  if (TWO && lane + 32 < r) V[at(i2, lane + 32)] = to_t<T>(y1);
}

// rows i (and i + nw when there are more rows than warps) per warp
template <typename T, bool CT>
__device__ __forceinline__ void hals_warp_pairs(const double* __restrict__ A, const double* Gs, const double* Ginv,
                                                T* __restrict__ V, size_t m, int r) {
  const size_t nw = (size_t)gridDim.x * 8;
  for (size_t i = (size_t)blockIdx.x * 8 + (threadIdx.x >> 5); i < m; i += 2 * nw) {
    if (i + nw < m)
      hals_warp_rows<T, CT, true>(A, Gs, Ginv, V, m, r, i, i + nw);
    else
      hals_warp_rows<T, CT, false>(A, Gs, Ginv, V, m, r, i, i);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_hals_v_warp(const double* __restrict__ A, const double* __restrict__ G,
                                                     T* __restrict__ V, size_t m, int r, int* __restrict__ degenerate) {
  extern __shared__ double Gs[];  // r x r, then r reciprocals of the diagonal
  double* Ginv = Gs + (size_t)r * r;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) Gs[e] = G[e];
  for (int k = threadIdx.x; k < r; k += blockDim.x) Ginv[k] = G[(size_t)k * r + k] > 0.0 ? 1.0 / G[(size_t)k * r + k] : 0.0;
  __syncthreads();
  if (degenerate && blockIdx.x == 0 && threadIdx.x == 0)  // hals_step's count: once per skipped k
    for (int k = 0; k < r; ++k)
      if (Gs[(size_t)k * r + k] <= 0.0) atomicAdd(degenerate, 1);
  hals_warp_pairs<T, false>(A, Gs, Ginv, V, m, r);
}

// columns of W (r x n): the same update with C (r x n) and D (r x r)
template <typename T>
__global__ void __launch_bounds__(256) k_hals_w_warp(const double* __restrict__ Cm, const double* __restrict__ D,
                                                     T* __restrict__ W, size_t n, int r, int* __restrict__ degenerate) {
  extern __shared__ double Ds[];  // r x r, then r reciprocals of the diagonal
  double* Dinv = Ds + (size_t)r * r;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) Ds[e] = D[e];
  for (int k = threadIdx.x; k < r; k += blockDim.x) Dinv[k] = D[(size_t)k * r + k] > 0.0 ? 1.0 / D[(size_t)k * r + k] : 0.0;
  __syncthreads();
  if (degenerate && blockIdx.x == 0 && threadIdx.x == 0)
    for (int k = 0; k < r; ++k)
      if (Ds[(size_t)k * r + k] <= 0.0) atomicAdd(degenerate, 1);
  hals_warp_pairs<T, true>(Cm, Ds, Dinv, W, n, r);
}

// ---------------------------------------------------------------------------
// MU updates (solvers.cpp:79-99).  Jacobi within a half: the denominator uses
// the old factor.  V(i,:) *= A(i,:) / max(V(i,:) B, 1e-16).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double mu_floor(double v) { return v < 1e-16 ? 1e-16 : v; }  // std::max(v, 1e-16)

template <typename T>
__global__ void k_mu_v(const double* __restrict__ A, const double* __restrict__ B, T* __restrict__ V,
                       size_t m, int r, double* __restrict__ gws) {
  extern __shared__ double sm[];
  const int bd = blockDim.x, t = threadIdx.x;
  const double* Bs = gws ? B : sm;
  double* vs = gws ? gws + (size_t)blockIdx.x * bd * r : sm + (size_t)r * r;
  if (!gws)
    for (int e = t; e < r * r; e += bd) sm[e] = B[e];
  const size_t i = (size_t)blockIdx.x * bd + t;
  const bool act = i < m;
  if (act)
    for (int l = 0; l < r; ++l) vs[l * bd + t] = (double)V[i * r + l];
  __syncthreads();
  if (!act) return;
  for (int j = 0; j < r; ++j) {
    double s = 0.0;
    for (int p = 0; p < r; ++p) s = __dadd_rn(s, __dmul_rn(vs[p * bd + t], Bs[p * r + j]));
    V[i * r + j] = to_t<T>(__dmul_rn(vs[j * bd + t], A[i * r + j] / mu_floor(s)));
  }
}

// W(:,j) *= C(:,j) / max(D W(:,j), 1e-16)
template <typename T>
__global__ void k_mu_w(const double* __restrict__ Cm, const double* __restrict__ D, T* __restrict__ W,
                       size_t n, int r, double* __restrict__ gws) {
  extern __shared__ double sm[];
  const int bd = blockDim.x, t = threadIdx.x;
  const double* Ds = gws ? D : sm;
  double* ws = gws ? gws + (size_t)blockIdx.x * bd * r : sm + (size_t)r * r;
  if (!gws)
    for (int e = t; e < r * r; e += bd) sm[e] = D[e];
  const size_t j = (size_t)blockIdx.x * bd + t;
  const bool act = j < n;
  if (act)
    for (int l = 0; l < r; ++l) ws[l * bd + t] = (double)W[(size_t)l * n + j];
  __syncthreads();
  if (!act) return;
  for (int k = 0; k < r; ++k) {
    double s = 0.0;
    for (int p = 0; p < r; ++p) s = __dadd_rn(s, __dmul_rn(Ds[k * r + p], ws[p * bd + t]));
    W[(size_t)k * n + j] = to_t<T>(__dmul_rn(ws[k * bd + t], Cm[(size_t)k * n + j] / mu_floor(s)));
  }
}

// Warp-per-row MU (non-exact: fused multiply-adds in register order) for few
// rows / columns, where one thread per row leaves most SMs idle (config 1's
// W half: 2429 columns -> 19 blocks of the thread kernels).  Lanes own the
// outputs k = lane, lane + 32; the factor row is broadcast by shuffles; the
// Gram sits in shared memory once per persistent block.  CT: columns of W
// (element (k, j) at k * n + j) against D; otherwise rows of V against B.
template <typename T, bool CT>
__global__ void __launch_bounds__(256) k_mu_warp(const double* __restrict__ A, const double* __restrict__ G,
                                                 T* __restrict__ V, size_t m, int r) {
  extern __shared__ double Gs[];
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) Gs[e] = G[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  auto at = [&](size_t row, int k) -> size_t { return CT ? (size_t)k * m + row : row * (size_t)r + k; };
  for (size_t i = (size_t)blockIdx.x * 8 + (threadIdx.x >> 5); i < m; i += (size_t)gridDim.x * 8) {
    const double v0 = lane < r ? (double)V[at(i, lane)] : 0.0;
    const double v1 = lane + 32 < r ? (double)V[at(i, lane + 32)] : 0.0;
    double s0 = 0.0, s1 = 0.0;
    for (int p = 0; p < r; ++p) {
      const double vp = __shfl_sync(0xffffffffu, p < 32 ? v0 : v1, p & 31);
      // V: (V B)_k = sum_p v_p B[p][k];  W: (D W)_k = sum_p D[k][p] w_p
      if (lane < r) s0 = fma(vp, CT ? Gs[lane * r + p] : Gs[p * r + lane], s0);
      if (lane + 32 < r) s1 = fma(vp, CT ? Gs[(lane + 32) * r + p] : Gs[p * r + lane + 32], s1);
    }
    if (lane < r) V[at(i, lane)] = to_t<T>(v0 * (A[at(i, lane)] / mu_floor(s0)));
    if (lane + 32 < r) V[at(i, lane + 32)] = to_t<T>(v1 * (A[at(i, lane + 32)] / mu_floor(s1)));
  }
}

// ---------------------------------------------------------------------------
// Direct residual ||M - VW||^2 per column (kernels.cpp:48-60):
//   part[z][j] = sum_{i in split z} (M_ij - sum_k V_ik W_kj)^2
// 128 columns per block; V rows staged 32 at a time; W column tile in smem.
// ---------------------------------------------------------------------------
template <typename T, bool EXACT, bool GM = false>
__global__ void __launch_bounds__(128) k_col_sqerr(const T* __restrict__ M, const double* __restrict__ V,
                                                   const double* __restrict__ W, size_t m, size_t n, int r,
                                                   size_t rchunk, double* __restrict__ part) {
  // GM (ranks too large for the shared-memory staging): V and W are read
  // from global memory directly, in the same operation order
  extern __shared__ double sm[];
  const int t = threadIdx.x;
  double* Ws = sm;                    // r x 128
  double* Vs = sm + (size_t)r * 128;  // 32 x r
  const size_t j = (size_t)blockIdx.x * 128 + t;
  const bool act = j < n;
  if (!GM)
    for (int k = 0; k < r; ++k) Ws[k * 128 + t] = act ? (double)W[(size_t)k * n + j] : 0.0;
  const size_t ib = (size_t)blockIdx.y * rchunk;
  const size_t ie = ib + rchunk < m ? ib + rchunk : m;
  double acc = 0.0;
  for (size_t i0 = ib; i0 < ie; i0 += 32) {
    if (!GM) {
      __syncthreads();
      for (int e = t; e < 32 * r; e += 128) {
        const size_t i = i0 + e / r;
        Vs[e] = i < ie ? (double)V[i * r + (e % r)] : 0.0;
      }
      __syncthreads();
    }
    if (!act) continue;
    const int cnt = (int)((ie - i0) < 32 ? (ie - i0) : 32);
    for (int ii = 0; ii < cnt; ++ii) {
      double pred = 0.0;
      for (int k = 0; k < r; ++k)
        pred = GM ? madd<EXACT>(pred, V[(i0 + ii) * r + k], W[(size_t)k * n + j])
                  : madd<EXACT>(pred, Vs[ii * r + k], Ws[k * 128 + t]);
      const double d = EXACT ? __dsub_rn((double)M[(i0 + ii) * n + j], pred) : (double)M[(i0 + ii) * n + j] - pred;
      acc = madd<EXACT>(acc, d, d);
    }
  }
  if (act) part[(size_t)blockIdx.y * n + j] = acc;
}

// Register-tiled direct residual for non-exact runs: block = 128 (i) x 128 (j)
// tile of M - V W, 256 threads x (8 x 8) outputs, V and W slices staged in
// shared memory (k-major), the prediction accumulated in T with FMA (round-to-
// nearest, unbiased), the squared residual in fp64.  One fp64 partial per
// block (deterministic).  FMA-bound: m n r FMAs, ~20x faster than k_col_sqerr.
__device__ __forceinline__ void ld4_shared(const float* p, float* o) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  o[0] = v.x, o[1] = v.y, o[2] = v.z, o[3] = v.w;
}
__device__ __forceinline__ void ld4_shared(const double* p, double* o) {
  const double2 u = *reinterpret_cast<const double2*>(p), v = *reinterpret_cast<const double2*>(p + 2);
  o[0] = u.x, o[1] = u.y, o[2] = v.x, o[3] = v.y;
}

// Persistent: block b takes tiles b, b + grid, ... (tile = (column block,
// row block), column blocks fastest) and writes one fp64 partial.  `gate`
// (optional, device): a block returns at once, writing 0, unless *gate != 0
// (the tensor path's sample runs this only when the Gram identity cancels
// too much, engine.cu sample_t).
template <typename T>
__global__ void __launch_bounds__(256, 2) k_sqerr_tiled(const T* __restrict__ M, const double* __restrict__ V,
                                                     const double* __restrict__ W, size_t m, size_t n, int r,
                                                     double* __restrict__ part, const double* __restrict__ gate) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* Vs = reinterpret_cast<T*>(smraw);  // [r][128]
  T* Ws = Vs + (size_t)r * 128;         // [r][128]
  __shared__ double red[8];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  if (gate && *gate == 0.0) {
    if (t == 0) part[blockIdx.x] = 0.0;
    return;
  }
  const size_t cbk = (n + 127) / 128, ntiles = cbk * ((m + 127) / 128);
  double s = 0.0;
  for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
  const size_t i0 = (tile / cbk) * 128, j0 = (tile % cbk) * 128;
  __syncthreads();  // the previous tile's shared-memory reads are done
  for (int e = t; e < r * 128; e += 256) {
    const int k = e >> 7, c = e & 127;
    Ws[e] = (j0 + c < n) ? (T)W[(size_t)k * n + j0 + c] : T(0);
  }
  for (int e = t; e < r * 128; e += 256) {
    const int row = e / r, k = e % r;  // coalesced along V's rows
    Vs[(size_t)k * 128 + row] = (i0 + row < m) ? (T)V[(i0 + row) * r + k] : T(0);
  }
  __syncthreads();
  T acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = T(0);
  // thread rows: (a >> 2) * 64 + ty * 4 + (a & 3); columns likewise with tx:
  // four consecutive k-major values per 16-byte (fp32) shared-memory load
  for (int k = 0; k < r; ++k) {
    T va[8], wb[8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      ld4_shared(Vs + k * 128 + h * 64 + ty * 4, va + 4 * h);
      ld4_shared(Ws + k * 128 + h * 64 + tx * 4, wb + 4 * h);
    }
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[a][b] = fma(va[a], wb[b], acc[a][b]);
  }
  // squared residuals: each row's 8 terms summed in T, then in fp64 (the
  // per-element fp64 convert + FMA would make the kernel fp64-pipe bound)
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const size_t i = i0 + (a >> 2) * 64 + ty * 4 + (a & 3);
    if (i >= m) continue;
    T sr = T(0);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const size_t j = j0 + (b >> 2) * 64 + tx * 4 + (b & 3);
      if (j < n) {
        const T d = M[i * n + j] - acc[a][b];
        sr = fma(d, d, sr);
      }
    }
    s += (double)sr;
  }
  }  // tiles
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((t & 31) == 0) red[t >> 5] = s;
  __syncthreads();
  if (t == 0) {
    double tot = 0.0;
    for (int w = 0; w < 8; ++w) tot += red[w];
    part[blockIdx.x] = tot;
  }
}

// ---------------------------------------------------------------------------
// Deterministic reductions.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// partials[block] = sum over a grid-stride slice of a[e] * b[e] (b may be null => a[e]^2)
// sum of squares of an fp32 array (||M_l||^2, once per level): float4 loads
// and four independent accumulators per thread keep enough bytes in flight
// to stream at the HBM rate (the scalar k_dot_partial loop ran at ~1.3 TB/s:
// 52 ms for config 4's 64 GiB).  count % 4 == 0, 16-byte aligned.
__global__ void __launch_bounds__(256) k_sq_partial_v4(const float4* __restrict__ a, size_t count4,
                                                       double* __restrict__ partials) {
  __shared__ double ws[8];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  const size_t stride = (size_t)gridDim.x * 256;
  size_t e = (size_t)blockIdx.x * 256 + threadIdx.x;
  for (; e + stride < count4; e += 2 * stride) {
    const float4 x = __ldcs(a + e), y = __ldcs(a + e + stride);
    s0 = fma((double)x.x, (double)x.x, s0);
    s1 = fma((double)x.y, (double)x.y, s1);
    s2 = fma((double)x.z, (double)x.z, s2);
    s3 = fma((double)x.w, (double)x.w, s3);
    s0 = fma((double)y.x, (double)y.x, s0);
    s1 = fma((double)y.y, (double)y.y, s1);
    s2 = fma((double)y.z, (double)y.z, s2);
    s3 = fma((double)y.w, (double)y.w, s3);
  }
  if (e < count4) {
    const float4 x = __ldcs(a + e);
    s0 = fma((double)x.x, (double)x.x, s0);
    s1 = fma((double)x.y, (double)x.y, s1);
    s2 = fma((double)x.z, (double)x.z, s2);
    s3 = fma((double)x.w, (double)x.w, s3);
  }
  double s = (s0 + s1) + (s2 + s3);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += ws[w];
    partials[blockIdx.x] = t;
  }
}

template <typename TA, typename TB>
__global__ void __launch_bounds__(256) k_dot_partial(const TA* __restrict__ a, const TB* __restrict__ b,
                                                     size_t count, double* __restrict__ partials) {
  __shared__ double ws[8];
  double s = 0.0;
  for (size_t e = (size_t)blockIdx.x * 256 + threadIdx.x; e < count; e += (size_t)gridDim.x * 256) {
    const double x = (double)a[e];
    s = fma(x, b ? (double)b[e] : x, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += ws[w];
    partials[blockIdx.x] = t;
  }
}

// out[0] = sum_{e<count} v[e] (single block, fixed order).  serial=true sums
// strictly left to right on one thread (reference order, matrix.cpp:39-40).
__global__ void k_sum_final(const double* __restrict__ v, size_t count, double* __restrict__ out, int serial) {
  __shared__ double ws[32];
  if (serial) {
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (size_t e = 0; e < count; ++e) s += v[e];
      out[0] = s;
    }
    return;
  }
  double s = 0.0;
  for (size_t e = threadIdx.x; e < count; e += blockDim.x) s += v[e];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    out[0] = t;
  }
}

// column sums of part[z][j] then the per-column values: out[j] = sum_z part[z][j]
// (already provided by k_reduce_splits).

// sample record: error = sqrt(max(e2, 0)) with e2 assembled from scalars:
//   gram:   e2 = s[0] - 2 s[1] + s[2]   (||M||^2, <C,W>, <D,WW^T>)
//   direct: e2 = s[0]
struct SampleRec {
  double error;
  unsigned long long t_ns;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_write_sample(const double* __restrict__ s, int gram, SampleRec* __restrict__ out) {
  double e2 = gram ? (s[0] - 2.0 * s[1] + s[2]) : s[0];
  out->error = sqrt(e2 > 0.0 ? e2 : 0.0);
  out->t_ns = globaltimer();
}

__global__ void k_set1(double* out, double v) { *out = v; }

// A whole Gram-identity sample in one launch (small problems, one rank):
// s[0] = ||M||^2 (argument), s[1] = <C, W> (count_cw elements), s[2] =
// <D, B> (count_db), each a fixed-order strided sum over the block's threads
// and a fixed tree; rec = sqrt(max(s0 - 2 s1 + s2, 0)) and the time stamp.
// (The general path takes 5 launches and a host-to-device copy.)
__global__ void __launch_bounds__(1024) k_gram_sample(const double* __restrict__ C, const double* __restrict__ W,
                                                      size_t count_cw, const double* __restrict__ D,
                                                      const double* __restrict__ B, size_t count_db, double norm2,
                                                      double* __restrict__ s, SampleRec* __restrict__ rec) {
  __shared__ double w1[32], w2[32];
  double a = 0.0, b = 0.0;
  for (size_t e = threadIdx.x; e < count_cw; e += blockDim.x) a = fma(C[e], W[e], a);
  for (size_t e = threadIdx.x; e < count_db; e += blockDim.x) b = fma(D[e], B[e], b);
  a = warp_sum(a);
  b = warp_sum(b);
  if ((threadIdx.x & 31) == 0) w1[threadIdx.x >> 5] = a, w2[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s1 = 0.0, s2 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s1 += w1[w], s2 += w2[w];
    s[0] = norm2, s[1] = s1, s[2] = s2;
    const double e2 = norm2 - 2.0 * s1 + s2;
    rec->error = sqrt(e2 > 0.0 ? e2 : 0.0);
    rec->t_ns = globaltimer();
  }
}

// s[0] = ||M||^2 - 2 <C, W> + <D, B>, clamped at 0 (Gram identity)
__global__ void k_gram_combine(double* s) {
  const double e2 = s[0] - 2.0 * s[1] + s[2];
  s[0] = e2 > 0.0 ? e2 : 0.0;
}

// Tensor-path samples: the Gram identity cancels ||M||^2 / e^2-fold, so the
// products' input rounding (~1e-9 .. 1e-10 of ||M||^2 on <C, W>) is
// amplified near a tight fit.  s[6] = the Gram e^2; s[7] = 1 when
// e^2 < tau ||M||^2 (the direct residual is then computed and used).
__global__ void k_gram_check(double* s, double tau) {
  const double e2 = s[0] - 2.0 * s[1] + s[2];
  s[6] = e2 > 0.0 ? e2 : 0.0;
  s[7] = e2 < tau * s[0] ? 1.0 : 0.0;
}
// s[0] = s[7] ? s[8] (direct) : s[6] (Gram)
__global__ void k_gram_select(double* s) { s[0] = s[7] != 0.0 ? s[8] : s[6]; }

__global__ void k_timestamp(unsigned long long* out) { *out = globaltimer(); }

// ---------------------------------------------------------------------------
// Transfer operators (transfer.cpp:17-33): Y[o,:] = sum_e w_e X[idx_e,:],
// entries in the reference's order, unfused multiply-add, fp64 math.
// ---------------------------------------------------------------------------
template <typename T, typename TO = T>
__global__ void k_csr_apply(const int* __restrict__ rowptr, const int* __restrict__ idx,
                            const double* __restrict__ wt, const T* __restrict__ X, TO* __restrict__ Y,
                            size_t out_rows, size_t ncols, size_t colblocks) {
  const size_t o = blockIdx.x / colblocks;
  const size_t c = (blockIdx.x % colblocks) * blockDim.x + threadIdx.x;
  if (o >= out_rows || c >= ncols) return;
  const int eb = rowptr[o], ee = rowptr[o + 1];
  double y = 0.0;
  for (int e = eb; e < ee; ++e) y = __dadd_rn(y, __dmul_rn(wt[e], (double)X[(size_t)idx[e] * ncols + c]));
  Y[o * ncols + c] = to_t<TO>(y);
}

// Restriction of many columns (GridHierarchy::build, transfer.cpp:155-174):
// Y = R X for an h x w grid, X (h w rows) x ncols row-major.  The CSR entries
// of R and their order are the reference's (k_csr_apply applies them as a
// gather, re-reading every fine row up to four times).  Here a CTA owns a
// SLABB-byte column slab and a STRIP of `strip` coarse pixel rows
// (blockIdx.y), and walks the coarse pixel columns cj in order, keeping the
// strip's 2 strip + 1 fine pixel rows of the three fine pixel columns
// 2cj - 1 .. 2cj + 1 in a shared-memory ring (NS x (2 strip + 1) x SLABB
// bytes; NS = 5 prefetches the next two columns by cp.async while cj is
// computed).  Every fine element is read from HBM once (plus one shared row
// per strip boundary: 1 / (2 strip)), every coarse element written once, and
// -- the point of the strips -- each fine row is fetched as one SLABB-byte
// piece: strips keep the ring small enough for 256- and 512-byte pieces
// (whole-column rings allowed 64 bytes, one DRAM burst pair per row).  Entry e
// is pre-decoded as code[e] = i * 4 + (dj + 1) (fine row i within its pixel
// column, column offset dj).  Threads: VEC columns each (one 16-byte vector;
// VEC = 1 when ncols is not a multiple of 16 B), SLABB / 16 threads per pixel
// row.  F64MATH: the reference's unfused fp64 sum in entry order
// (bit-identical to k_csr_apply); otherwise fp32 FMA in the same order (fp32
// storage, non-exact runs: within an ulp of the fp64 result).
template <typename T, typename TO, int VEC, bool F64MATH, int SLABB = 64, int NS = 3>
__global__ void __launch_bounds__(256) k_restrict_slab(const int* __restrict__ rowptr, const int* __restrict__ code,
                                                       const double* __restrict__ wt, const T* __restrict__ X,
                                                       TO* __restrict__ Y, int h, int w, int hc, int wc,
                                                       size_t ncols, int strip) {
  constexpr int SLAB = SLABB / (int)sizeof(T);  // columns per CTA
  constexpr int TPR = SLAB / VEC;               // threads per pixel row
  // NS ring slots: columns 2cj-1 .. 2cj+1 (+ the next two, prefetched, when NS = 5)
  extern __shared__ __align__(16) unsigned char smraw[];
  T* ring = reinterpret_cast<T*>(smraw);  // [NS][2 strip + 1][SLAB]
  const int t = threadIdx.x, part = t % TPR, grp = t / TPR, ngrp = blockDim.x / TPR;
  const size_t c0 = (size_t)blockIdx.x * SLAB + (size_t)part * VEC;
  const int nact = c0 >= ncols ? 0 : (int)min((size_t)VEC, ncols - c0);
  // the strip: coarse rows [ca, cb), fine rows [i0, i0 + hs)
  const int ca = (int)blockIdx.y * strip, cb = min(ca + strip, hc);
  const int i0 = max(2 * ca - 1, 0), hs = min(2 * (cb - 1) + 1, h - 1) - i0 + 1;
  const size_t slot = (size_t)(2 * strip + 1) * SLAB;
  // fine pixel column j -> its ring slot: asynchronous 16-byte copies (or
  // plain loads on the unaligned path), committed as one group
  auto fetch = [&](int j) {
    T* dst = ring + (size_t)(j % NS) * slot + part * VEC;
    const T* src = X + ((size_t)j * h + i0) * ncols + c0;
    for (int i = grp; i < hs; i += ngrp) {
      if (VEC > 1 && nact == VEC) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + (size_t)i * SLAB);
        asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(sa), "l"(src + (size_t)i * ncols)
                     : "memory");
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) dst[(size_t)i * SLAB + v] = v < nact ? src[(size_t)i * ncols + v] : T(0);
      }
    }
  };
  fetch(0);
  if (w > 1) fetch(1);
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int cj = 0; cj < wc; ++cj) {
    if (NS == 5) {
      // prefetch coarse column cj + 1's new fine columns during this one
      if (2 * cj + 2 < w) fetch(2 * cj + 2);
      if (2 * cj + 3 < w) fetch(2 * cj + 3);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // this column's group has landed
    } else {
      if (cj > 0) {
        if (2 * cj < w) fetch(2 * cj);
        if (2 * cj + 1 < w) fetch(2 * cj + 1);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    // ring slot of fine column 2 cj + dj, dj = -1, 0, 1 (rows relative to i0)
    const T* sl[3] = {ring + (size_t)((2 * cj + NS - 1) % NS) * slot - (size_t)i0 * SLAB,
                      ring + (size_t)((2 * cj) % NS) * slot - (size_t)i0 * SLAB,
                      ring + (size_t)((2 * cj + 1) % NS) * slot - (size_t)i0 * SLAB};
    for (int ci = ca + grp; ci < cb; ci += ngrp) {
      const size_t o = (size_t)cj * hc + ci;
      const int eb = rowptr[o], ee = rowptr[o + 1];
      double yd[VEC];
      float yf[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) yd[v] = 0.0, yf[v] = 0.f;
      for (int e = eb; e < ee; ++e) {
        const int cd = code[e];
        const T* xs = sl[cd & 3] + (size_t)(cd >> 2) * SLAB + part * VEC;
        T xv[VEC];
        if (VEC > 1) {
          *reinterpret_cast<uint4*>(xv) = *reinterpret_cast<const uint4*>(xs);
        } else {
          xv[0] = xs[0];
        }
        if (F64MATH) {
          const double we = wt[e];
#pragma unroll
          for (int v = 0; v < VEC; ++v) yd[v] = __dadd_rn(yd[v], __dmul_rn(we, (double)xv[v]));
        } else {
          const float we = (float)wt[e];
#pragma unroll
          for (int v = 0; v < VEC; ++v) yf[v] = fmaf(we, (float)xv[v], yf[v]);
        }
      }
      TO* yo = Y + o * ncols + c0;
      if (VEC > 1 && nact == VEC) {
        // one vector store (ncols sizeof(T) % 16 == 0 aligns every row of Y)
        struct alignas(sizeof(TO) * VEC) Pack {
          TO v[VEC];
        } pk;
#pragma unroll
        for (int v = 0; v < VEC; ++v) pk.v[v] = F64MATH ? to_t<TO>(yd[v]) : (TO)yf[v];
        *reinterpret_cast<Pack*>(yo) = pk;
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          if (v < nact) yo[v] = F64MATH ? to_t<TO>(yd[v]) : (TO)yf[v];
      }
    }
    __syncthreads();  // slots of columns 2cj - 1 and 2cj are refilled by the next prefetch
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// smoothness numerator, transfer.cpp:133-139: sum_ij (M_f - P M_c)_ij^2 with
// M_c = R M_f (the next level's resident data), P applied on the fly in the
// reference's entry order, so P R M is never stored.  Grid (colblocks, ry):
// column-coalesced, rows strided by ry; one fp64 partial per CTA.
template <typename TC, typename TF>
__global__ void __launch_bounds__(256) k_csr_residual(const int* __restrict__ rowptr, const int* __restrict__ idx,
                                                      const double* __restrict__ wt, const TC* __restrict__ Mc,
                                                      const TF* __restrict__ Mf, size_t rows, size_t ncols,
                                                      double* __restrict__ part) {
  __shared__ double ws[8];
  const size_t c = (size_t)blockIdx.x * 256 + threadIdx.x;
  double s = 0.0;
  if (c < ncols)
    for (size_t o = blockIdx.y; o < rows; o += gridDim.y) {
      const int eb = rowptr[o], ee = rowptr[o + 1];
      double y = 0.0;
      for (int e = eb; e < ee; ++e) y = __dadd_rn(y, __dmul_rn(wt[e], (double)Mc[(size_t)idx[e] * ncols + c]));
      const double d = (double)Mf[o * ncols + c] - y;
      s = fma(d, d, s);
    }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += ws[w];
    part[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------
// random_init (matrix.cpp:51-60) on the device: V row-major first, then W,
// one SplitMix64 stream.  W is this rank's column slice [col0, col0+n_loc)
// of an n_total-column W, so the stream counter jumps to m*r + k*n_total + j.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_random_init(T* __restrict__ V, T* __restrict__ W, size_t m, size_t r, size_t n_loc,
                              size_t n_total, size_t col0, uint64_t seed) {
  const size_t nv = m * r, nw = r * n_loc;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < nv + nw;
       e += (size_t)gridDim.x * blockDim.x) {
    if (e < nv) {
      V[e] = to_t<T>(sm64_uniform(seed, e));
    } else {
      const size_t f = e - nv, k = f / n_loc, jl = f % n_loc;
      W[f] = to_t<T>(sm64_uniform(seed, nv + k * n_total + col0 + jl));
    }
  }
}

template <typename T>
__global__ void k_convert(const double* __restrict__ src, T* __restrict__ dst, size_t count) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (size_t)gridDim.x * blockDim.x)
    dst[e] = to_t<T>(src[e]);
}
template <typename T>
__global__ void k_widen(const T* __restrict__ src, double* __restrict__ dst, size_t count) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (size_t)gridDim.x * blockDim.x)
    dst[e] = (double)src[e];
}

// ---------------------------------------------------------------------------
// Synthetic data generator (BASELINE.json configs; spec DESIGN.md section 3).
// Counter-based SplitMix64 streams: a column slice generates independently.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t gen_key(uint64_t seed, uint64_t tag) {
  return sm64_mix(seed ^ (0xA0761D6478BD642FULL * tag));
}

// V0[px][k] = sum_b amp_kb exp(-((ix - ci)^2 + (jx - cj)^2) / (2 sigma^2)), px = jx*h + ix
__global__ void k_gen_basis(double* __restrict__ V0, size_t h, size_t w, int r, int blobs, double smin,
                            double smax, uint64_t key) {
  const size_t total = h * w * (size_t)r;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const size_t px = e / r, k = e % r, jx = px / h, ix = px % h;
    double s = 0.0;
    for (int b = 0; b < blobs; ++b) {
      const uint64_t c0 = 4 * (k * (uint64_t)blobs + b);
      const double ci = sm64_uniform(key, c0) * (double)h;
      const double cj = sm64_uniform(key, c0 + 1) * (double)w;
      const double sg = smin + sm64_uniform(key, c0 + 2) * (smax - smin);
      const double amp = 0.5 + 0.5 * sm64_uniform(key, c0 + 3);
      const double di = (double)ix - ci, dj = (double)jx - cj;
      s += amp * exp(-(di * di + dj * dj) / (2.0 * sg * sg));
    }
    V0[px * r + k] = s;
  }
}

// W0[k][jl] = Exp(1) with probability 1/2 else 0, global column col0 + jl
__global__ void k_gen_wcols(double* __restrict__ W0, int r, size_t n_loc, size_t n_total, size_t col0,
                            uint64_t key) {
  const size_t total = (size_t)r * n_loc;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const size_t k = e / n_loc, jl = e % n_loc;
    const uint64_t c = 2 * ((uint64_t)k * n_total + col0 + jl);
    W0[e] = sm64_uniform(key, c) < 0.5 ? 0.0 : -log1p(-sm64_uniform(key, c + 1));
  }
}

// M[px][jl] = max(sum_k V0[px][k] W0[k][jl] + noise, 0).  mode 0: store;
// mode 1: only block maxima into bmax[]; mode 2: store value / div.
template <typename T>
__global__ void __launch_bounds__(128) k_gen_m(T* __restrict__ M, const double* __restrict__ V0,
                                               const double* __restrict__ W0, size_t m, size_t n_loc, int r,
                                               size_t col0, uint64_t keyn, int noise_kind, double noise_scale,
                                               int mode, double div, double* __restrict__ bmax) {
  extern __shared__ double sm[];
  double* Ws = sm;                    // r x 128
  double* Vs = sm + (size_t)r * 128;  // 32 x r
  __shared__ double red[4];
  const int t = threadIdx.x;
  const size_t jl = (size_t)blockIdx.x * 128 + t;
  const bool act = jl < n_loc;
  for (int k = 0; k < r; ++k) Ws[k * 128 + t] = act ? W0[(size_t)k * n_loc + jl] : 0.0;
  const size_t p0 = (size_t)blockIdx.y * 32;
  for (int e = t; e < 32 * r; e += 128) {
    const size_t px = p0 + e / r;
    Vs[e] = px < m ? V0[px * r + (e % r)] : 0.0;
  }
  __syncthreads();
  double mx = 0.0;
  if (act) {
    const int cnt = (int)((m - p0) < 32 ? (m - p0) : 32);
    for (int ii = 0; ii < cnt; ++ii) {
      const size_t px = p0 + ii;
      double s = 0.0;
      for (int k = 0; k < r; ++k) s = __dadd_rn(s, __dmul_rn(Vs[ii * r + k], Ws[k * 128 + t]));
      const uint64_t e = (uint64_t)(col0 + jl) * m + px;
      double noise;
      if (noise_kind == 0) {
        noise = noise_scale * sm64_uniform(keyn, e);
      } else {
        const double u1 = sm64_uniform(keyn, 2 * e), u2 = sm64_uniform(keyn, 2 * e + 1);
        noise = noise_scale * sqrt(-2.0 * log1p(-u1)) * cos(6.283185307179586 * u2);
      }
      const double v0 = __dadd_rn(s, noise);
      const double v = v0 > 0.0 ? v0 : 0.0;
      if (mode == 0) M[px * n_loc + jl] = to_t<T>(v);
      else if (mode == 2) M[px * n_loc + jl] = to_t<T>(v / div);
      else mx = v > mx ? v : mx;
    }
  }
  if (mode == 1) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((t & 31) == 0) red[t >> 5] = mx;
    __syncthreads();
    if (t == 0) bmax[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = fmax(fmax(red[0], red[1]), fmax(red[2], red[3]));
  }
}

__global__ void k_max_final(const double* __restrict__ v, size_t count, double* __restrict__ out) {
  __shared__ double ws[32];
  double s = 0.0;
  for (size_t e = threadIdx.x; e < count; e += blockDim.x) s = fmax(s, v[e]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, ws[w]);
    out[0] = t;
  }
}

// validation: flag |= 1 if any entry is negative or non-finite
template <typename T>
__global__ void k_validate(const T* __restrict__ M, size_t count, int* __restrict__ flag) {
  bool bad = false;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (size_t)gridDim.x * blockDim.x) {
    const double v = (double)M[e];
    bad |= !(v >= 0.0) || !isfinite(v);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

}  // namespace mlb
