// nnls.cuh -- batched active-set NNLS for ANLS (sm_100a).
//
// Restates nnls_active_set (proj/src/solvers.cpp:143-243) with
// cholesky_solve (:24-51) and solve_passive (:55-75) as ONE WARP PER
// SUBPROBLEM: min_{x>=0} x'Gx/2 - h'x with the shared r x r Gram G in shared
// memory, the passive-set Cholesky factor (packed lower) in the warp's shared
// memory slice, lanes parallel over rows.  Control flow is warp-uniform.
// The Cholesky and the forward substitution keep the reference's operation
// order exactly (right-looking forward substitution performs the same
// subtraction sequence per element); EXACT = true also runs the backward
// substitution in the reference's order on one lane, so fp64 results are
// bit-identical to the reference.
//
// Error reporting: *err |= 1 on exchange-cap overflow (NnlsCapExceeded),
// |= 2 on a passive system singular after 8 ridge attempts (runtime_error;
// anls_step maps both to NnlsCapExceeded, solvers.cpp:262-267,289-294).
#pragma once
#include <cstdint>
#include "kernels.cuh"

namespace mlb {

struct NnlsWarpMem {
  double* L;     // p(p+1)/2 packed lower, p <= r
  double* b;     // r (right-hand side, then the solution z)
  double* b0;    // r (saved right-hand side for ridge retries)
  double* x;     // r
  double* h;     // r
  int* passive;  // r
  int* kept;     // r
  unsigned char* inp;  // r
};

__host__ __device__ inline size_t nnls_warp_bytes(int r) {
  size_t d = (size_t)r * (r + 1) / 2 + 4 * (size_t)r;
  return d * 8 + 2 * (size_t)r * 4 + (((size_t)r + 15) / 16) * 16;
}

// Cholesky of the packed lower p x p matrix in place; false on a non-positive
// or non-finite pivot (solvers.cpp:26-37).  !EXACT: the column is scaled by
// one reciprocal of the pivot (an fp64 division is a ~100-cycle dependent
// MUFU + Newton sequence; ncu put the divisions among the hottest spots of
// the batched NNLS), and the diagonal holds 1 / L[k][k] for the
// substitutions, which then multiply instead of divide.
template <bool EXACT>
__device__ inline bool warp_cholesky(double* L, int p, int lane) {
  // 32-bit packed-row offsets and 4-way unrolled dot products: the kernel is
  // issue-bound (ncu: 62 % issue-active, ~42k warp instructions per
  // subproblem), and 64-bit index math plus loop overhead were most of the
  // inner loops' instructions.  The subtraction order is unchanged.
  // EXACT: the reference's unfused d - a * b; otherwise one fused multiply-add
  auto sub = [](double acc, double a, double b) { return EXACT ? msub(acc, a, b) : fma(-a, b, acc); };
  for (int k = 0; k < p; ++k) {
    const double* Lk = L + (unsigned)(k * (k + 1) / 2);
    // Column k in one pass: lane j takes row i = k + j, so lane 0's "row" is
    // the pivot itself -- d = G_kk - sum_q L_kq^2 is the same chain of
    // subtractions as a row's s = G_ik - sum_q L_iq L_kq with i = k.  The
    // pivot dot used to run first, on every lane, before the rows: 2 k
    // dependent operations per column instead of k (same per-element order:
    // results unchanged bit for bit).
    const int i0 = k + lane;
    double s0 = 0.0;
    double* Li0 = L + (unsigned)(i0 * (i0 + 1) / 2);
    if (i0 < p) {
      s0 = Li0[k];
      int qq = 0;
      for (; qq + 4 <= k; qq += 4) {
        s0 = sub(s0, Li0[qq], Lk[qq]);
        s0 = sub(s0, Li0[qq + 1], Lk[qq + 1]);
        s0 = sub(s0, Li0[qq + 2], Lk[qq + 2]);
        s0 = sub(s0, Li0[qq + 3], Lk[qq + 3]);
      }
      for (; qq < k; ++qq) s0 = sub(s0, Li0[qq], Lk[qq]);
    }
    const double d = __shfl_sync(0xffffffffu, s0, 0);
    if (d <= 0.0 || !isfinite(d)) {
      __syncwarp();
      return false;
    }
    const double lkk = sqrt(d);
    const double ilkk = EXACT ? 0.0 : 1.0 / lkk;
    __syncwarp();  // every lane has read row k before its diagonal is overwritten
    if (lane == 0) Li0[k] = EXACT ? lkk : ilkk;
    else if (i0 < p) Li0[k] = EXACT ? s0 / lkk : s0 * ilkk;
    for (int i = i0 + 32; i < p; i += 32) {  // rows beyond the first 32 (p - k > 32: the first columns only)
      double* Li = L + (unsigned)(i * (i + 1) / 2);
      double s = Li[k];
      int qq = 0;
      for (; qq + 4 <= k; qq += 4) {
        s = sub(s, Li[qq], Lk[qq]);
        s = sub(s, Li[qq + 1], Lk[qq + 1]);
        s = sub(s, Li[qq + 2], Lk[qq + 2]);
        s = sub(s, Li[qq + 3], Lk[qq + 3]);
      }
      for (; qq < k; ++qq) s = sub(s, Li[qq], Lk[qq]);
      Li[k] = EXACT ? s / lkk : s * ilkk;
    }
    __syncwarp();
  }
  return true;
}

template <bool EXACT>
__device__ inline void warp_substitute(const double* L, double* b, int p, int lane) {
  // forward: L y = b (solvers.cpp:39-43), right-looking, same per-element order
  for (int q = 0; q < p; ++q) {
    const size_t rq = (size_t)q * (q + 1) / 2;
    const double bq = EXACT ? b[q] / L[rq + q] : b[q] * L[rq + q];  // !EXACT: diagonal holds 1 / L[q][q]
    __syncwarp();
    if (lane == 0) b[q] = bq;
    for (int i = q + 1 + lane; i < p; i += 32)
      b[i] = EXACT ? msub(b[i], L[(size_t)i * (i + 1) / 2 + q], bq) : fma(-L[(size_t)i * (i + 1) / 2 + q], bq, b[i]);
    __syncwarp();
  }
  // backward: L^T x = y (solvers.cpp:44-48)
  if (EXACT) {
    if (lane == 0) {
      for (int ii = p - 1; ii >= 0; --ii) {
        double s = b[ii];
        for (int q = ii + 1; q < p; ++q) s = msub(s, L[(size_t)q * (q + 1) / 2 + ii], b[q]);
        b[ii] = s / L[(size_t)ii * (ii + 1) / 2 + ii];
      }
    }
    __syncwarp();
  } else {
    for (int q = p - 1; q >= 0; --q) {
      const double bq = b[q] * L[(size_t)q * (q + 1) / 2 + q];
      __syncwarp();
      if (lane == 0) b[q] = bq;
      const size_t rq = (size_t)q * (q + 1) / 2;
      for (int ii = lane; ii < q; ii += 32) b[ii] = fma(-L[rq + ii], bq, b[ii]);
      __syncwarp();
    }
  }
}

// solve_passive: z (in wm.b) = G_PP^{-1} h_P with the ridge fallback.
template <bool EXACT>
__device__ inline bool warp_solve_passive(const double* Gs, int r, const NnlsWarpMem& wm, int p, int lane,
                                          double ridge0) {
  for (int a = lane; a < p; a += 32) {
    wm.b[a] = wm.h[wm.passive[a]];
    wm.b0[a] = wm.b[a];
  }
  double ridge = 0.0;
  for (int attempt = -1; attempt < 8; ++attempt) {
    for (int a = 0; a < p; ++a) {
      const size_t ra = (size_t)a * (a + 1) / 2;
      const int pa = wm.passive[a];
      for (int c = lane; c <= a; c += 32) {
        double g = Gs[(size_t)pa * r + wm.passive[c]];
        if (attempt >= 0 && c == a) g += ridge;
        wm.L[ra + c] = g;
      }
    }
    for (int a = lane; a < p; a += 32) wm.b[a] = wm.b0[a];
    __syncwarp();
    if (warp_cholesky<EXACT>(wm.L, p, lane)) {
      warp_substitute<EXACT>(wm.L, wm.b, p, lane);
      return true;
    }
    ridge = attempt < 0 ? ridge0 : ridge * 100.0;
  }
  return false;
}

// One warp per problem.  Problem q has h[k] = H[q*hi + k*he] and warm start /
// output x[k] = X[q*xi + k*xe]; counts[q] receives the exchange count.
template <typename T, bool EXACT>
__global__ void k_nnls_batch(const double* __restrict__ G, int r, size_t nprob, const double* __restrict__ H,
                             size_t hi, size_t he, T* __restrict__ X, size_t xi, size_t xe,
                             int* __restrict__ counts, int* __restrict__ err, unsigned char* __restrict__ gws) {
  // gws (ranks too large for shared memory): the Gram is read from global
  // memory and each warp's workspace is gws + (global warp) * nnls_warp_bytes
  extern __shared__ __align__(16) unsigned char smraw[];
  const double* Gs = gws ? G : reinterpret_cast<const double*>(smraw);
  const int nwarps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (!gws)
    for (int e = threadIdx.x; e < r * r; e += blockDim.x) reinterpret_cast<double*>(smraw)[e] = G[e];
  __syncthreads();
  // ridge base: 1e-12 * tr(G) / r (solvers.cpp:64-67)
  double trace = 0.0;
  for (int k = 0; k < r; ++k) trace += Gs[(size_t)k * r + k];
  double ridge0 = 1e-12 * trace / (double)r;
  if (ridge0 <= 0.0) ridge0 = 1e-12;

  unsigned char* base = gws ? gws + ((size_t)blockIdx.x * nwarps + warp) * nnls_warp_bytes(r)
                            : smraw + (size_t)r * r * 8 + (size_t)warp * nnls_warp_bytes(r);
  NnlsWarpMem wm;
  wm.L = reinterpret_cast<double*>(base);
  wm.b = wm.L + (size_t)r * (r + 1) / 2;
  wm.b0 = wm.b + r;
  wm.x = wm.b0 + r;
  wm.h = wm.x + r;
  wm.passive = reinterpret_cast<int*>(wm.h + r);
  wm.kept = wm.passive + r;
  wm.inp = reinterpret_cast<unsigned char*>(wm.kept + r);

  const uint64_t cap = r < 50 ? 3ull * (1ull << r) + 10ull * (uint64_t)r : ~0ull;

  for (size_t q = (size_t)blockIdx.x * nwarps + warp; q < nprob; q += (size_t)gridDim.x * nwarps) {
    // scale and tol (solvers.cpp:149-152)
    double scale = 1.0;
    for (int k = lane; k < r; k += 32) {
      const double hk = H[q * hi + (size_t)k * he];
      wm.h[k] = hk;
      scale = fmax(scale, fmax(fabs(hk), Gs[(size_t)k * r + k]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
    const double tol = 1e-10 * scale;
    // warm start from supp(x0) (solvers.cpp:158-167), passive in index order
    int np = 0;
    for (int k0 = 0; k0 < r; k0 += 32) {
      const int k = k0 + lane;
      double xv = 0.0;
      bool pos = false;
      if (k < r) {
        xv = (double)X[q * xi + (size_t)k * xe];
        pos = xv > 0.0;
        wm.x[k] = pos ? xv : 0.0;
        wm.inp[k] = pos ? 1 : 0;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, pos);
      if (pos) wm.passive[np + __popc(bal & ((1u << lane) - 1u))] = k;
      np += __popc(bal);
    }
    __syncwarp();
    uint64_t exchanges = 0;
    int fail = 0;
    for (;;) {
      while (np > 0) {
        if (!warp_solve_passive<EXACT>(Gs, r, wm, np, lane, ridge0)) {
          fail = 2;
          break;
        }
        // feasibility and the step length alpha (solvers.cpp:180-189)
        bool infeas = false;
        double alpha = 1.0;
        for (int a = lane; a < np; a += 32) {
          const double za = wm.b[a];
          if (za <= 0.0) {
            infeas = true;
            const double xi_ = wm.x[wm.passive[a]];
            const double denom = xi_ - za;
            const double cand = denom > 0.0 ? xi_ / denom : 0.0;
            alpha = cand < alpha ? cand : alpha;
          }
        }
        infeas = __any_sync(0xffffffffu, infeas);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double oa = __shfl_xor_sync(0xffffffffu, alpha, o);
          alpha = oa < alpha ? oa : alpha;
        }
        if (!infeas) {
          for (int a = lane; a < np; a += 32) wm.x[wm.passive[a]] = wm.b[a];
          __syncwarp();
          break;
        }
        for (int a = lane; a < np; a += 32) {
          const int i = wm.passive[a];
          wm.x[i] = __dadd_rn(wm.x[i], __dmul_rn(alpha, __dsub_rn(wm.b[a], wm.x[i])));
        }
        __syncwarp();
        // drop coordinates that hit zero, keeping order (solvers.cpp:198-209)
        int nk = 0, ndrop = 0;
        for (int a0 = 0; a0 < np; a0 += 32) {
          const int a = a0 + lane;
          bool drop = false, keep = false;
          if (a < np) {
            const int i = wm.passive[a];
            drop = wm.b[a] <= 0.0 && wm.x[i] <= tol * 1e-2;
            keep = !drop;
            if (drop) {
              wm.x[i] = 0.0;
              wm.inp[i] = 0;
            }
          }
          const unsigned kb = __ballot_sync(0xffffffffu, keep);
          if (keep) wm.kept[nk + __popc(kb & ((1u << lane) - 1u))] = wm.passive[a];
          nk += __popc(kb);
          ndrop += __popc(__ballot_sync(0xffffffffu, drop));
        }
        __syncwarp();
        exchanges += (uint64_t)ndrop;
        if (exchanges > cap) {
          fail = 1;
          break;
        }
        if (nk == np) {
          // numerical stall: force out the first most negative z (:210-219)
          double zb = INFINITY;
          int wb = 0x7fffffff;
          for (int a = lane; a < np; a += 32)
            if (wm.b[a] < zb) {
              zb = wm.b[a];
              wb = a;
            }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double oz = __shfl_xor_sync(0xffffffffu, zb, o);
            const int ow = __shfl_xor_sync(0xffffffffu, wb, o);
            if (oz < zb || (oz == zb && ow < wb)) {
              zb = oz;
              wb = ow;
            }
          }
          if (wb == 0x7fffffff) wb = 0;  // all-NaN z: the reference keeps worst = 0
          const int iw = wm.passive[wb];
          __syncwarp();
          if (lane == 0) {
            wm.x[iw] = 0.0;
            wm.inp[iw] = 0;
          }
          int nxt[4], cnt = 0;  // r <= 128: at most 4 positions per lane
          for (int a = wb + lane; a + 1 < nk; a += 32) nxt[cnt++] = wm.kept[a + 1];
          __syncwarp();
          cnt = 0;
          for (int a = wb + lane; a + 1 < nk; a += 32) wm.kept[a] = nxt[cnt++];
          __syncwarp();
          --nk;
          if (++exchanges > cap) {
            fail = 1;
            break;
          }
        }
        for (int a = lane; a < nk; a += 32) wm.passive[a] = wm.kept[a];
        __syncwarp();
        np = nk;
      }
      if (fail) break;
      // outer optimality: w = h - G x on the active set (solvers.cpp:223-235)
      double bw = tol;
      int bi = r;
      for (int i = lane; i < r; i += 32) {
        if (wm.inp[i]) continue;
        double gx = 0.0;
        for (int qq = 0; qq < r; ++qq) gx = __dadd_rn(gx, __dmul_rn(Gs[(size_t)i * r + qq], wm.x[qq]));
        const double wv = wm.h[i] - gx;
        if (wv > bw) {
          bw = wv;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ow = __shfl_xor_sync(0xffffffffu, bw, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ow > bw || (ow == bw && oi < bi)) {
          bw = ow;
          bi = oi;
        }
      }
      if (bi >= r) break;
      __syncwarp();
      if (lane == 0) {
        wm.inp[bi] = 1;
        wm.passive[np] = bi;
      }
      __syncwarp();
      ++np;
      if (++exchanges > cap) {
        fail = 1;
        break;
      }
    }
    if (fail) {
      if (lane == 0) atomicOr(err, fail);
    }
    for (int k = lane; k < r; k += 32) X[q * xi + (size_t)k * xe] = to_t<T>(wm.x[k]);
    if (lane == 0 && counts) counts[q] = (int)exchanges;
    __syncwarp();
  }
}

}  // namespace mlb
