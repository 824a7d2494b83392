// restrict_tma.cu -- restriction of every column (image) of a level,
// Y = R X (GridHierarchy::build, transfer.cpp:155-174; the operator R of
// build_restriction, transfer.cpp:61-85), as a TMA-fed, warp-specialised
// stream for sm_100a.
//
// X is (h w) x ncols row-major, pixel (i, j) of an h x w image at row j h + i;
// Y is (hc wc) x ncols.  Output row o = cj hc + ci sums the fine rows
// (2 ci + di, 2 cj + dj), di, dj in {-1, 0, 1}, that lie inside the image,
// in the reference's entry order (di outer, dj inner) with the reference's
// renormalised weights (a 16-class table rebuilt in shared memory by the same
// fp64 operations as the reference: class_weights).
//
// A CTA owns a 512-byte column slab and a strip of `strip` coarse pixel rows
// and walks the coarse pixel columns cj in order.  The strip's 2 strip + 1
// fine pixel rows of fine pixel column j are ONE 3-D TMA box (512 B x
// (2 strip + 1) rows x 1 pixel column; rows outside the image are zero-filled
// and never referenced) landing in slot j % NS of a shared-memory ring:
//   warp 0 (one lane): the producer -- waits for a slot to be released, arms
//           its mbarrier with the box bytes, issues the box; runs up to NS - 3
//           pixel columns ahead of the consumers
//   warps 1..8: consumers -- step cj waits for columns 2cj and 2cj + 1
//           (2cj - 1 was awaited by the previous step), computes the strip's
//           coarse rows (warp v takes ci = ca + v, ca + v + 8, ...; a lane
//           owns one 16-byte column vector), releases columns 2cj - 1 and 2cj.
// No __syncthreads in the loop: the warps drift apart by up to the ring
// depth, and every fine element is read from HBM once (plus one shared pixel
// row per strip boundary, 1 / (2 strip)) in 512-byte pieces; every coarse
// element is written once, 512 B (fp32) or 1 KB (fp64 out) per warp store.
//
// F64MATH: the reference's unfused fp64 multiply-add chain in entry order
// (bit-identical to the reference; fp64 sessions, exact mode, and fp32 levels
// restricted into fp64 storage); otherwise fp32 FMA in the same order (fp32
// storage, non-exact runs).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "restrict_tma.hpp"

namespace mlb {
namespace rt {

constexpr int kSlabBytes = 512;
constexpr int kConsumers = 8;  // consumer warps
constexpr int kThreads = 32 * (1 + kConsumers);
constexpr int kMaxSlots = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t mbar_try(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok;
}
// bounded wait: a pipeline bug traps instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  if (mbar_try(a, parity)) return;
  const long long t0 = clock64();
  for (uint32_t i = 1;; ++i) {
    if (mbar_try(a, parity)) return;
    if ((i & 255) == 0 && clock64() - t0 > (1ll << 33)) __trap();
  }
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t mbar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(mbar), "l"(pol)
      : "memory");
}

template <typename T>
struct Vec;  // one lane's 16-byte column vector
template <>
struct Vec<float> {
  static constexpr int N = 4;
  float v[4];
};
template <>
struct Vec<double> {
  static constexpr int N = 2;
  double v[2];
};
template <typename T>
__device__ __forceinline__ Vec<T> lds_vec(uint32_t a);
template <>
__device__ __forceinline__ Vec<float> lds_vec<float>(uint32_t a) {
  Vec<float> x;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(x.v[0]), "=f"(x.v[1]), "=f"(x.v[2]), "=f"(x.v[3])
               : "r"(a)
               : "memory");
  return x;
}
template <>
__device__ __forceinline__ Vec<double> lds_vec<double>(uint32_t a) {
  Vec<double> x;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x.v[0]), "=d"(x.v[1]) : "r"(a) : "memory");
  return x;
}

template <typename TO>
__device__ __forceinline__ TO cast_out(double v);
template <>
__device__ __forceinline__ double cast_out<double>(double v) {
  return v;
}
template <>
__device__ __forceinline__ float cast_out<float>(double v) {
  return __double2float_rn(v);
}

struct Params {
  int h, w, hc, wc;
  int strip;   // coarse pixel rows per CTA
  int nslots;  // ring depth (>= 4)
  unsigned long long ncols;
};

// The renormalised weights of one coarse pixel, by validity class: bit 0 of a
// class = the -1 neighbour exists, bit 1 = the +1 neighbour exists (rows:
// class a, columns: class b).  Entry k of a pixel is its k-th VALID
// (di, dj) in the reference's order (di outer, dj inner), its weight
// (wgt / 16) / s with s the sum of the pixel's wgt / 16 in entry order --
// the same fp64 operations as build_restriction + normalize_row
// (transfer.cpp:61-85, :9-15), so the table equals the reference's CSR
// weights bit for bit (tests: restriction parity against the reference).
__device__ __forceinline__ void class_weights(int a, int b, double* out9) {
  double wv[9];
  int n = 0;
  double s = 0.0;
  for (int di = -1; di <= 1; ++di)
    for (int dj = -1; dj <= 1; ++dj) {
      if ((di == -1 && !(a & 1)) || (di == 1 && !(a & 2))) continue;
      if ((dj == -1 && !(b & 1)) || (dj == 1 && !(b & 2))) continue;
      const double wgt = (di == 0 && dj == 0) ? 4.0 : (di == 0 || dj == 0) ? 2.0 : 1.0;
      wv[n] = wgt / 16.0;
      s = __dadd_rn(s, wv[n]);
      ++n;
    }
  for (int k = 0; k < 9; ++k) out9[k] = k < n ? __ddiv_rn(wv[k], s) : 0.0;
}

template <typename T, typename TO, bool F64MATH>
__global__ void __launch_bounds__(kThreads) k_restrict_tma(const __grid_constant__ CUtensorMap map_x, TO* __restrict__ Y,
                                                           const Params p) {
  constexpr int N = Vec<T>::N;                   // columns per lane
  constexpr int SLAB = kSlabBytes / (int)sizeof(T);  // columns per CTA
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* ring = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const int rows = 2 * p.strip + 1;              // fine pixel rows per slot
  const uint32_t slot_bytes = (uint32_t)rows * kSlabBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)p.nslots * slot_bytes);
  uint64_t* empty = full + kMaxSlots;
  double* wtab = reinterpret_cast<double*>(empty + kMaxSlots);  // [4 row classes][4 column classes][9]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NS = p.nslots;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
  }
  if (threadIdx.x >= 32 && threadIdx.x < 48) {
    const int cls = threadIdx.x - 32;
    class_weights(cls >> 2, cls & 3, wtab + cls * 9);
  }
  __syncthreads();

  const int ca = (int)blockIdx.y * p.strip, cb = min(ca + p.strip, p.hc);
  const int i_first = 2 * ca - 1;  // fine pixel row of slot row 0 (may be -1: zero-filled)
  const int col0 = (int)blockIdx.x * SLAB;

  if (warp == 0) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int s = 0;
      uint32_t ph = 1u;  // a fresh barrier passes the parity-1 wait
      for (int j = 0; j < p.w; ++j) {
        mbar_wait(smem_u32(&empty[s]), ph);
        const uint32_t fb = smem_u32(&full[s]);
        mbar_expect_tx(fb, slot_bytes);
        tma_load_3d(smem_u32(ring + (size_t)s * slot_bytes), &map_x, col0, i_first, j, fb, pol);
        if (++s == NS) s = 0, ph ^= 1u;
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int v = warp - 1;
  const size_t c = (size_t)col0 + (size_t)lane * N;
  const int nact = c >= p.ncols ? 0 : (int)min((unsigned long long)N, p.ncols - c);
  const uint32_t ring_a = smem_u32(ring) + (uint32_t)lane * 16u;
  // ring slots / barrier phases of columns 2cj - 1, 2cj, 2cj + 1, advanced by two per step
  int sl_m = NS - 1, sl_0 = 0, sl_p = 1 % NS;
  uint32_t ph_0 = 0, ph_p = (uint32_t)(1 / NS) & 1u;
  for (int cj = 0; cj < p.wc; ++cj) {
    const int j0 = 2 * cj;
    const bool vjm = j0 > 0, vjp = j0 + 1 < p.w;
    mbar_wait(smem_u32(&full[sl_0]), ph_0);
    if (vjp) mbar_wait(smem_u32(&full[sl_p]), ph_p);
    const uint32_t sm = ring_a + (uint32_t)sl_m * slot_bytes, s0 = ring_a + (uint32_t)sl_0 * slot_bytes,
                   sp = ring_a + (uint32_t)sl_p * slot_bytes;
    const int clsb = (vjm ? 1 : 0) | (vjp ? 2 : 0);
    for (int ci = ca + v; ci < cb; ci += kConsumers) {
      const size_t o = (size_t)cj * p.hc + ci;
      const bool vim = ci > 0, vip = 2 * ci + 1 < p.h;
      const double* we = wtab + (((vim ? 1 : 0) | (vip ? 2 : 0)) * 4 + clsb) * 9;
      double yd[N];
      float yf[N];
#pragma unroll
      for (int k = 0; k < N; ++k) yd[k] = 0.0, yf[k] = 0.f;
#pragma unroll
      for (int di = -1; di <= 1; ++di) {
        if (di == -1 ? !vim : (di == 1 ? !vip : false)) continue;  // warp-uniform
        const uint32_t ro = (uint32_t)(2 * ci + di - i_first) * kSlabBytes;
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj) {
          if (dj == -1 ? !vjm : (dj == 1 ? !vjp : false)) continue;  // warp-uniform
          const Vec<T> x = lds_vec<T>((dj == -1 ? sm : (dj == 0 ? s0 : sp)) + ro);
          const double wgt = *we++;
          if (F64MATH) {
#pragma unroll
            for (int k = 0; k < N; ++k) yd[k] = __dadd_rn(yd[k], __dmul_rn(wgt, (double)x.v[k]));
          } else {
            const float wf = (float)wgt;
#pragma unroll
            for (int k = 0; k < N; ++k) yf[k] = fmaf(wf, (float)x.v[k], yf[k]);
          }
        }
      }
      TO* yo = Y + o * p.ncols + c;
      if (nact == N) {
        struct alignas(sizeof(TO) * N) Pack {
          TO q[N];
        } pk;
#pragma unroll
        for (int k = 0; k < N; ++k) pk.q[k] = F64MATH ? cast_out<TO>(yd[k]) : (TO)yf[k];
        *reinterpret_cast<Pack*>(yo) = pk;
      } else {
#pragma unroll
        for (int k = 0; k < N; ++k)
          if (k < nact) yo[k] = F64MATH ? cast_out<TO>(yd[k]) : (TO)yf[k];
      }
    }
    // columns 2cj - 1 and 2cj are dead after this step (2cj + 1 is the next
    // step's 2cj' - 1)
    __syncwarp();
    if (lane == 0) {
      if (vjm) mbar_arrive(smem_u32(&empty[sl_m]));
      mbar_arrive(smem_u32(&empty[sl_0]));
    }
    sl_m = sl_p;
    sl_0 += 2;
    if (sl_0 >= NS) sl_0 -= NS, ph_0 ^= 1u;
    sl_p += 2;
    if (sl_p >= NS) sl_p -= NS, ph_p ^= 1u;
  }
}

}  // namespace rt

namespace {

#define RT_CK(x)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess)                                                                        \
      throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e_) + " at " +    \
                               __FILE__ + ":" + std::to_string(__LINE__));                        \
  } while (0)

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    RT_CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

template <typename T, typename TO, bool F64MATH>
void run(const RestrictArgs& a, int strip, int nslots, cudaStream_t s) {
  const size_t es = sizeof(T);
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)a.ncols, (cuuint64_t)a.h, (cuuint64_t)a.w};
  cuuint64_t strides[2] = {(cuuint64_t)a.ncols * es, (cuuint64_t)a.ncols * es * (cuuint64_t)a.h};
  cuuint32_t box[3] = {(cuuint32_t)(rt::kSlabBytes / es), (cuuint32_t)(2 * strip + 1), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&map, es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                                 const_cast<void*>(a.X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (restriction) failed: " + std::to_string((int)r));
  rt::Params p{};
  p.h = a.h, p.w = a.w, p.hc = a.hc, p.wc = a.wc;
  p.strip = strip;
  p.nslots = nslots;
  p.ncols = a.ncols;
  const size_t smem = 128 + (size_t)nslots * (2 * strip + 1) * rt::kSlabBytes + 2 * rt::kMaxSlots * 8 + 16 * 9 * 8;
  auto kern = rt::k_restrict_tma<T, TO, F64MATH>;
  RT_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const dim3 g((unsigned)((a.ncols * es + rt::kSlabBytes - 1) / rt::kSlabBytes), (unsigned)((a.hc + strip - 1) / strip));
  kern<<<g, rt::kThreads, smem, s>>>(map, static_cast<TO*>(a.Y), p);
  RT_CK(cudaGetLastError());
}

}  // namespace

// Loads the four instantiations (CUDA loads a kernel lazily at its first
// launch or attribute call) and fetches the tensor-map encoder: done at
// session creation, the first pyramid build of a process that has already run
// solver steps otherwise pays ~0.1 s of module loading inside its timed region
// (measured r02: 120 ms instead of 25 ms for the config-4 pyramid).
void restrict_tma_prepare() {
  const int smem = 128 + 16 * 17 * rt::kSlabBytes;  // any valid size: the call itself loads the function
  RT_CK(cudaFuncSetAttribute(rt::k_restrict_tma<double, double, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  RT_CK(cudaFuncSetAttribute(rt::k_restrict_tma<float, double, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  RT_CK(cudaFuncSetAttribute(rt::k_restrict_tma<float, float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  RT_CK(cudaFuncSetAttribute(rt::k_restrict_tma<float, float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  (void)encode_fn();
}

bool restrict_tma_supported(const RestrictArgs& a) {
  const size_t es = a.in_f64 ? 8 : 4;
  return a.h >= 2 && a.w >= 2 && (a.ncols * es) % 16 == 0 && reinterpret_cast<uintptr_t>(a.X) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(a.Y) % 32 == 0 && a.ncols * es >= 2048 && a.ncols < (1ull << 31);
}

void restrict_tma(const RestrictArgs& a, int strip, int nslots, cudaStream_t s) {
  if (!restrict_tma_supported(a)) throw std::invalid_argument("restrict_tma: unsupported shape");
  if (strip < 1) strip = 1;
  if (strip > a.hc) strip = a.hc;
  if (2 * strip + 1 > 256) strip = 127;  // TMA box rows <= 256
  if (nslots < 4) nslots = 4;
  if (nslots > rt::kMaxSlots) nslots = rt::kMaxSlots;
  if (a.in_f64) {
    run<double, double, true>(a, strip, nslots, s);
  } else if (a.out_f64) {
    run<float, double, true>(a, strip, nslots, s);
  } else if (a.f64math) {
    run<float, float, true>(a, strip, nslots, s);
  } else {
    run<float, float, false>(a, strip, nslots, s);
  }
}

}  // namespace mlb
