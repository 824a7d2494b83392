// ix_gemm.cu -- the two M-streaming products of the fp32-storage path on the
// 5th-generation tensor cores (tcgen05, sm_100a), integer digits, exact
// accumulation:
//
//   product 1 (TRANS = false):  A (m x r)   = M (m x n) . W^T    (kernels.cpp:24-34; solvers.cpp:82,105,252)
//   product 2 (TRANS = true):   C^T (n x r) = M^T (n x m) . V    (kernels.cpp:36-46; solvers.cpp:91,124,273)
//
// Number format (tests/ixmodel.py is its numpy model).  Every fp32 entry x
// of an MMA row of M (a row for product 1, a column for product 2) is scaled
// by a power of two s chosen from the row maximum (max * s in [2^30, 2^31))
// and rounded once (half-even, one F2I) to X = round(x s): a 31-bit fixed
// point on which every fp32 entry within 2^7 of the maximum is EXACT.  Every
// fp64 factor entry f (a row of W, a column of V; the factors are fp64 on the
// device) is likewise rounded to Y = round(f s_f) on its row's 31-bit grid.
// Both are split into balanced base-256 digits
//     X = d1 2^24 + d2 2^16 + d3 2^8 + d4,   Y = e1 2^24 + e2 2^16 + e3 2^8 + e4
// (d1, e1 in [0, 127]; the others in [-128, 127]: the bytes of X + 0x808080).
// The digit products d_i e_j of weight classes c = i + j - 2 <= 3 are summed
// over K per class in int32 TMEM by `tcgen05.mma.kind::i8` -- exactly, in
// any order -- and
//     sum x f ~= 2^24 (G0 2^24 + G1 2^16 + G2 2^8 + G3) / (s s_f)
// (the bracket exact in int64, then one fp64 rounding).  Classes 4..6
// (d2 e4, d3 e3, d4 e2, d3 e4, d4 e3, d4 e4) are <= 2^-32 of the largest
// product and are not formed.  The products are then accurate to ~1e-9
// (tests), and whole fp32 runs through this path track the fp64 reference
// (fed the same fp32 M) as closely as the fp64-accumulating SIMT path does:
// 5e-8 single-level / 1.6e-6 five-level FMG on the config-4 slice
// (tests/test_gpu_tc_config4.py; the FMG floor is the fp32 storage of the
// restricted pyramid, not the products).
// History (r02, measured): a 3-digit M x 3-digit factor split keeping six
// products drifted 1e-4 from the reference (a small factor entry, leading
// digit d2 or d3, kept ~16 bits); all nine products 1.4e-5; a 23-bit factor
// grid let the Gram-identity error samples cancel 5e-5 at coarse levels.
//
// MMA shape: the four factor digit planes are STACKED along N in shared
// memory ([e1; e2; e3; e4], r_pad rows each), and M digit plane d_i (TMEM,
// the A operand) multiplies the prefix [e1 .. e_(5-i)] (N = (5 - i) r_pad)
// into the accumulator window starting at class group i - 1: block j lands
// on group i + j - 2, so the overlapping windows do the class sums.  4 MMAs
// per 32-wide chunk (N = 4, 3, 2, 1 x r_pad; 320 tensor cycles per 128-row
// chunk at r_pad = 64, ~40 % of the chunk's HBM time at 1.9 GHz).
//
// The kernel (persistent, warp-specialised, one CTA per SM, 736 threads):
//   warp 0: TMA producer of M slices (16 KB, issued and released in pairs;
//           product 1 fetches a chunk pair as one 3-D box of 128 rows x 256 B)
//   warp 1: MMA issuer (allocates TMEM): per chunk PAIR one wait on the
//           pair's staging slots, 8 MMAs, one commit; the factor stage (a
//           chunk QUAD) is waited for by a quad's first pair and released by
//           its second.  One accumulator set (4 classes x r_pad int32
//           columns) per work unit, drained and zeroed by the epilogue
//           between units (the MMAs always accumulate).
//   warp 2: TMA producer of factor digit quads (4 r_pad rows x 128 B =
//           4 chunks of the stacked planes, SWIZZLE_128B)
//   warps 3-18: converters (four groups of 4 warps, chunk g -> group g % 4):
//           fp32 slice from shared memory -> FMUL + F2I + IADD per element ->
//           byte permutes into the digit planes d1 | d2 | d3 | d4 ->
//           tcgen05.st into a staging slot (thread = MMA row = TMEM lane)
//   warps 19-22: epilogue: drains a unit's four class accumulators once
//           (units of <= kMaxUnitChunks chunks keep int32 exact), converts to
//           fp64, writes the split-K partial, re-zeroes.
// TMEM (512 columns): the accumulator set at 0 (class c at c r_pad), staging
// slots at 256 + 32 s, s < 8 (d1 | d2 | d3 | d4, 8 columns each); chunk g
// uses slot g % 8, chunk pair h the slot pair h % 4.  Work units hold a
// multiple of 4 chunks (zero chunks pad a ragged K: TMA zero-fills M beyond
// the matrix, the factor digits are zero there).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "ix_gemm.hpp"

namespace mlb {
namespace ix {

constexpr int kChunk = 32;             // K elements per pipeline chunk
constexpr int kMStages = 8;            // M-slice ring (TMA -> converters), 16 KB each
constexpr int kMGroup = 2;             // the ring is filled and released in pairs of slices (one TMA each; 4 measured slower, r02)
constexpr int kMGroups = kMStages / kMGroup;
constexpr int kBStages = 2;            // factor digit ring (TMA -> MMA), one chunk QUAD per stage
constexpr int kBStageBytes = 32768;    // 4 planes x r_pad (<= 64) rows x 128 B (= 4 chunks x 32 K)
constexpr int kQuad = 4;               // chunks per factor stage
constexpr int kSlots = 8;              // TMEM staging slots: four pairs (chunk g -> slot g % 8)
constexpr int kPairs = kSlots / 2;
constexpr int kSlotCols = 32;          // columns per slot (24 used)
constexpr int kGroupCols = 64;         // columns per accumulator group (r_pad <= 64)
constexpr int kClasses = 4;            // digit-product weight classes 2^40, 2^32, 2^24, 2^16
constexpr int kAccCols = kClasses * kGroupCols;
constexpr int kStg0 = 256;             // staging slots after the (single) accumulator set
static_assert(kQuad % kMGroup == 0, "units (whole quads) hold whole M groups");
static_assert(kAccCols <= kStg0 && kStg0 + kSlots * kSlotCols <= 512, "TMEM map");
// factor fixed point: 31 bits (four digits e1 e2 e3 e4, e1 in [0, 127])
constexpr double kFBias = 8421504.0;   // 0x808080: balanced low three digits
// chunks per work unit: class G3 sums four digit products (|d e| <= 2^14) per
// K element, so an int32 accumulator is exact for K <= 2^31 / 2^16 = 32768
// = 1024 chunks
constexpr int kMaxUnitChunks = 1024;
constexpr int kConvGroups = 4;         // converter groups (4 warps each), chunk g -> group g % 4
constexpr int kEpiWarps = 4;           // epilogue: one warp per TMEM lane quarter
constexpr int kWarpM = 0, kWarpMma = 1, kWarpB = 2, kWarpConv0 = 3;
constexpr int kWarpEpi0 = kWarpConv0 + 4 * kConvGroups;
constexpr int kThreads = (kWarpEpi0 + kEpiWarps) * 32;
constexpr int kMTileBytes = 128 * kChunk * 4;  // 16 KB
// the row maximum's grid position: max * s_hi <= kXMax (then x * 256 s_hi < 2^31 - 0x808080)
constexpr float kXMax = 8355711.0f;            // 2^23 - 0x8080 - 1

#define IX_CK(x)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess)                                                                        \
      throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e_) + " at " +    \
                               __FILE__ + ":" + std::to_string(__LINE__));                        \
  } while (0)

// ----------------------------------------------------------------------------
// PTX helpers
// ----------------------------------------------------------------------------
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
// Bounded wait: a pipeline bug traps (kernel error) after ~2^34 cycles
// instead of hanging the GPU.
template <int SLEEP_NS = 0>
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  if (mbar_try(a, parity)) return;
  const long long t0 = clock64();
  for (uint32_t i = 1;; ++i) {
    if (SLEEP_NS) __nanosleep(SLEEP_NS);
    if (mbar_try(a, parity)) return;
    if ((i & 255) == 0 && clock64() - t0 > (1ll << 34)) __trap();
  }
}
__device__ __forceinline__ void lds128(uint32_t a, float& x, float& y, float& z, float& w) {
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a) : "memory");
}
__device__ __forceinline__ float lds32(uint32_t a) {
  float x;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(a) : "memory");
  return x;
}
// L2 policies: the M stream is read once (evict_first) and must not push out
// the factor digit slices, which every CTA working on the same K range reads
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t mbar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(mbar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t mbar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(mbar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// warp-wide call; one elected lane commits
__device__ __forceinline__ void tc_commit(uint32_t mbar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(mbar)
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor: K-major, SWIZZLE_128B, 8-row atoms of
// 128 B (SBO = 1024 B), Blackwell version bit.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;            // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024u >> 4) << 32;  // SBO
  d |= (uint64_t)1u << 46;            // version = 1 (sm_100)
  d |= (uint64_t)2u << 61;            // SWIZZLE_128B
  return d;
}
// Instruction descriptor: D s32, A/B s8, K-major both, N, M = 128.
__host__ __device__ constexpr uint32_t idesc_s8(int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// The fixed-point multiplier 2^e of a row with maximum mx: mx * 2^e lies in
// [2^21, kXMax] (a power of two: x * 2^e is exact in fp32).
__host__ __device__ __forceinline__ float scale_of(float mx) {
  if (!(mx > 0.f)) return 1.f;
  int e;
  (void)frexpf(mx, &e);  // mx = f 2^e, f in [0.5, 1)
  int k = 23 - e;
  k = k > 125 ? 125 : (k < -125 ? -125 : k);
  float s = ldexpf(1.f, k);
  if (mx * s > kXMax) s *= 0.5f;
  return s;
}

// The factor's fixed-point multiplier: mx * s in [2^29, 2^30) (power of two,
// fp64; mx is the fp32 row maximum rounded up), so X + 0x808080 < 2^31.
__host__ __device__ __forceinline__ double fscale_of(float mx) {
  if (!(mx > 0.f)) return 1.0;
  int e;
  (void)frexpf(mx, &e);
  return ldexp(1.0, 30 - e);
}

// One chunk's 3 MMAs (K = 32 each) on staging slot S: M digit plane d_i
// (TMEM, 128 rows) times a prefix of the STACKED factor digit planes
// [e1; e2; e3; e4] (shared memory, r_pad rows each), written to the
// accumulator window starting at class group i - 1.  Block j of MMA i lands
// on group i + j - 2, so the windows' overlap sums every digit product
// d_i e_j into its weight class c = i + j - 2 (weight 2^(40 - 8c)):
//   G0 = d1 e1;  G1 = d1 e2 + d2 e1;  G2 = d1 e3 + d2 e2 + d3 e1;
//   G3 = d1 e4 + d2 e3 + d3 e2
// (d1: N = 4 r_pad, d2: 3 r_pad, d3: 2 r_pad), exact in int32.  Not formed:
// d2 e4, d3 e3, d3 e4 (classes 4 and 5, <= 2^-32 of the largest product):
// measured on sparse coarse-level factors they change no product beyond
// 1e-12 relative, and they would cost a third more tensor work -- which
// the board's power limit turns into SM clock (ncu r02c: 12 products ran
// the tensor pipe at 70-80 % and the clock at 1.24-1.34 GHz).  The leading
// six of a 3 x 3 split were NOT enough: a small factor entry (leading digit
// d2 or d3, common in sparse NMF factors) kept ~16 bits and the config-4 FMG
// trajectory drifted 1e-4 from the reference; the factor's fourth digit
// (grid 2^-31 of the row maximum) fixed the Gram-identity samples at coarse
// levels.  The accumulators always accumulate (the epilogue zeroes them
// after each drain).
template <int S>
__device__ __forceinline__ void issue_chunk(uint64_t bd, uint32_t id4, uint32_t id3, uint32_t id2, uint32_t id1,
                                            uint32_t rp) {
  constexpr uint32_t a1 = kStg0 + S * kSlotCols, a2 = a1 + 8, a3 = a1 + 16, a4 = a1 + 24;
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%4], %8, %9, 1;\n\t"    // d1 [e1..e4] -> G0..G3
      "@e tcgen05.mma.cta_group::1.kind::i8 [%1], [%5], %8, %10, 1;\n\t"   // d2 [e1..e3] -> G1..G3
      "@e tcgen05.mma.cta_group::1.kind::i8 [%2], [%6], %8, %11, 1;\n\t"   // d3 [e1, e2] -> G2..G3
      "@e tcgen05.mma.cta_group::1.kind::i8 [%3], [%7], %8, %12, 1;\n\t}"  // d4 [e1]     -> G3
      ::"r"(0u), "r"(rp), "r"(2u * rp), "r"(3u * rp), "r"(a1), "r"(a2), "r"(a3), "r"(a4), "l"(bd), "r"(id4),
      "r"(id3), "r"(id2), "r"(id1)
      : "memory");
}
// A chunk pair: slots 2 PS and 2 PS + 1 (factor columns at bd0 / bd1)
template <int PS>
__device__ __forceinline__ void issue_pair(uint64_t bd0, uint64_t bd1, uint32_t id4, uint32_t id3, uint32_t id2,
                                           uint32_t id1, uint32_t rp) {
  issue_chunk<2 * PS>(bd0, id4, id3, id2, id1, rp);
  issue_chunk<2 * PS + 1>(bd1, id4, id3, id2, id1, rp);
}

// M entries on a 31-bit grid: X = round(x s) (half-even, one F2I), s =
// 256 s_hi a power of two (x * s exact: fp32 entries within 2^7 of the row
// maximum are represented exactly, x s <= 256 kXMax < 2^31 - 0x808080), as
// four balanced digits X = d1 2^24 + d2 2^16 + d3 2^8 + d4: the bytes of
// X + 0x808080 are d1 | d2 + 128 | d3 + 128 | d4 + 128 (3..0).  The four
// planes of 4 consecutive elements (element t in byte t) by byte permutes.
__device__ __forceinline__ void planes_of(const uint32_t (&w)[4], uint32_t& p1, uint32_t& p2, uint32_t& p3,
                                          uint32_t& p4) {
  const uint32_t t01 = __byte_perm(w[0], w[1], 0x5140), t23 = __byte_perm(w[2], w[3], 0x5140);
  const uint32_t u01 = __byte_perm(w[0], w[1], 0x7362), u23 = __byte_perm(w[2], w[3], 0x7362);
  p4 = __byte_perm(t01, t23, 0x5410) ^ 0x80808080u;
  p3 = __byte_perm(t01, t23, 0x7632) ^ 0x80808080u;
  p2 = __byte_perm(u01, u23, 0x5410) ^ 0x80808080u;
  p1 = __byte_perm(u01, u23, 0x7632);
}
__device__ __forceinline__ void planes4x(float x0, float x1, float x2, float x3, float s, uint32_t& p1,
                                         uint32_t& p2, uint32_t& p3, uint32_t& p4) {
  const uint32_t w[4] = {(uint32_t)__float2int_rn(x0 * s) + 0x808080u, (uint32_t)__float2int_rn(x1 * s) + 0x808080u,
                         (uint32_t)__float2int_rn(x2 * s) + 0x808080u, (uint32_t)__float2int_rn(x3 * s) + 0x808080u};
  planes_of(w, p1, p2, p3, p4);
}

struct Params {
  int rows;        // MMA-M extent: m (product 1) or n (product 2)
  int kdim;        // K extent: n (product 1) or m (product 2)
  int r;           // true rank
  int rp;          // padded rank (multiple of 16, <= 64)
  int tiles;       // ceil(rows / 128)
  int splits;      // K ranges
  int chunks_per_split;
  int nchunks;     // ceil(kdim / 32)
  int wide;        // product 1: a chunk pair is one 3-D TMA box of 128 rows x 256 B
  const float* rowmax;  // per MMA row: the maximum of its M row (product 1) / column (product 2)
  const float* fmax;    // per output column k: the maximum of factor row k
  double* part;    // [splits][...] fp64 partial outputs
};

// Work units: unit u = (tile u % tiles, K range u / tiles), dealt round-robin
// to the persistent CTAs (concurrent CTAs hold consecutive tiles of the same
// K range, so they read the same factor slices from L2 at about the same time).
struct Unit {
  int tile, split, c0, n;
};
__device__ __forceinline__ Unit unit_of(const Params& p, int u) {
  Unit x;
  x.tile = u % p.tiles;
  x.split = u / p.tiles;
  x.c0 = x.split * p.chunks_per_split;
  x.n = min(x.c0 + p.chunks_per_split, p.nchunks) - x.c0;
  return x;
}

template <bool TRANS>
__global__ void __launch_bounds__(kThreads, 1)
    k_ix_product(const __grid_constant__ CUtensorMap map_m, const __grid_constant__ CUtensorMap map_b,
                 const Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sm_m = base;                                   // kMStages x 16 KB
  unsigned char* sm_b = base + kMStages * kMTileBytes;          // kBStages x 8 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm_b + kBStages * kBStageBytes);
  uint64_t* mfull = bars;                  // [kMGroups]  TMA -> converters
  uint64_t* mempty = mfull + kMGroups;     // [kMGroups]  converters -> TMA
  uint64_t* ready = mempty + kMGroups;     // [kPairs]    converters -> MMA (slot pair written)
  uint64_t* sdone = ready + kPairs;        // [kPairs]    MMA commit -> converters (slot pair free)
  uint64_t* bfull = sdone + kPairs;        // [kBStages]  TMA -> MMA
  uint64_t* bempty = bfull + kBStages;     // [kBStages]  MMA commit -> TMA
  uint64_t* afull = bempty + kBStages;     // [2]         MMA commit -> epilogue (unit done)
  uint64_t* aempty = afull + 2;            // [2]         epilogue -> MMA (accumulators drained)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(aempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kMGroups; ++i) {
      mbar_init(smem_u32(&mfull[i]), 1);
      mbar_init(smem_u32(&mempty[i]), 4 * kMGroup);  // the 4 converter warps of each slice
    }
    for (int i = 0; i < kPairs; ++i) {
      mbar_init(smem_u32(&ready[i]), 4 * 2);  // the 4 converter warps of each of the pair's chunks
      mbar_init(smem_u32(&sdone[i]), 1);
    }
    for (int i = 0; i < kBStages; ++i) {
      mbar_init(smem_u32(&bfull[i]), 1);
      mbar_init(smem_u32(&bempty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&afull[i]), 1);
      mbar_init(smem_u32(&aempty[i]), kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_m)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == kWarpMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if (tmem != 0) __trap();  // one CTA per SM owning all 512 columns: base is lane 0, column 0

  const int total_units = p.tiles * p.splits;
  const int u0 = blockIdx.x, ustep = gridDim.x;

  if (warp == kWarpM) {
    // ======================= TMA producer: M slices =======================
    if (lane == 0) {
      int g = 0, npend = 0;
      int pt[kMGroup] = {}, pc[kMGroup] = {};
      const uint64_t pol = l2_evict_first();
      auto issue_group = [&]() {
        const int pg = g / kMGroup, ps = pg % kMGroups;
        mbar_wait(smem_u32(&mempty[ps]), ((uint32_t)(pg / kMGroups) & 1u) ^ 1u);
        const uint32_t fm = smem_u32(&mfull[ps]);
        mbar_expect_tx(fm, npend * kMTileBytes);
        unsigned char* dst = sm_m + ps * kMGroup * kMTileBytes;
        if (!TRANS && p.wide && npend == kMGroup) {
          // chunks c .. c + 3 of one tile: each row's 512 contiguous bytes
          // in one request stream, one 3-D box
          tma_load_3d(smem_u32(dst), &map_m, 0, pc[0], pt[0] * 128, fm, pol);
        } else {
          for (int k = 0; k < npend; ++k) {
            if (!TRANS)
              tma_load_2d(smem_u32(dst + k * kMTileBytes), &map_m, pc[k] * kChunk, pt[k] * 128, fm, pol);
            else
              tma_load_2d(smem_u32(dst + k * kMTileBytes), &map_m, pt[k] * 128, pc[k] * kChunk, fm, pol);
          }
        }
        g += kMGroup;
        npend = 0;
      };
      for (int u = u0; u < total_units; u += ustep) {
        const Unit x = unit_of(p, u);
        for (int i = 0; i < x.n; ++i) {
          pt[npend] = x.tile, pc[npend] = x.c0 + i;
          if (++npend == kMGroup) issue_group();
        }
      }
      if (npend > 0) issue_group();
    }
  } else if (warp == kWarpB) {
    // ======================= TMA producer: factor digit slices =======================
    if (lane == 0) {
      const uint64_t pol = l2_evict_last();
      const uint32_t bytes = 4u * (uint32_t)p.rp * 128u;
      int qc = 0;  // chunk quad counter
      for (int u = u0; u < total_units; u += ustep) {
        const Unit x = unit_of(p, u);
        for (int i = 0; i < x.n; i += kQuad, ++qc) {
          const int bs = qc % kBStages;
          mbar_wait(smem_u32(&bempty[bs]), ((uint32_t)(qc / kBStages) & 1u) ^ 1u);
          const uint32_t fb = smem_u32(&bfull[bs]);
          mbar_expect_tx(fb, bytes);
          tma_load_2d(smem_u32(sm_b + bs * kBStageBytes), &map_b, 0, ((x.c0 + i) / kQuad) * 4 * p.rp, fb, pol);
        }
      }
    }
  } else if (warp == kWarpMma) {
    // ======================= MMA issuer =======================
    // The whole warp runs the (warp-uniform) loop so every operand stays in
    // the uniform datapath; one elected lane issues each tcgen05 instruction.
    // Per chunk PAIR (the issue loop of this one warp is the serial path of
    // the whole pipeline: one ready wait, 6 MMAs, one commit; the factor
    // stage -- a chunk quad -- is waited for by a quad's first pair and
    // released by its second)
    const uint64_t bdesc0 = sdesc_sw128(smem_u32(sm_b));
    const uint32_t id4 = idesc_s8(4 * p.rp), id3 = idesc_s8(3 * p.rp), id2 = idesc_s8(2 * p.rp),
                   id1 = idesc_s8(p.rp);
    const uint32_t rp = (uint32_t)p.rp;
    int h = 0, uc = 0;
    for (int u = u0; u < total_units; u += ustep, ++uc) {
      const int n_u = unit_of(p, u).n;
      // the single accumulator set: drained and zeroed by the epilogue
      // (phase 0 = the initial zeroing)
      mbar_wait(smem_u32(&aempty[0]), (uint32_t)uc & 1u);
      for (int i = 0; i < n_u; i += 2, ++h) {
        const int ps = h % kPairs, qc = h >> 1, bs = qc % kBStages;
        mbar_wait(smem_u32(&ready[ps]), (uint32_t)(h / kPairs) & 1u);
        if (!(h & 1)) mbar_wait(smem_u32(&bfull[bs]), (uint32_t)(qc / kBStages) & 1u);
        tc_fence_after();
        // chunk (2h) % 4 of the quad: its K columns at byte 32 (2h % 4)
        const uint64_t bd = bdesc0 + ((uint64_t)(bs * kBStageBytes) >> 4) + (uint64_t)(4 * (h & 1));
        switch (ps) {
          case 0: issue_pair<0>(bd, bd + 2, id4, id3, id2, id1, rp); break;
          case 1: issue_pair<1>(bd, bd + 2, id4, id3, id2, id1, rp); break;
          case 2: issue_pair<2>(bd, bd + 2, id4, id3, id2, id1, rp); break;
          default: issue_pair<3>(bd, bd + 2, id4, id3, id2, id1, rp); break;
        }
        tc_commit(smem_u32(&sdone[ps]));                // slot pair reusable once these MMAs finish
        if (h & 1) tc_commit(smem_u32(&bempty[bs]));  // ... and, after a quad's second pair, its factor stage
        __syncwarp();
      }
      tc_commit(smem_u32(&afull[0]));  // the unit's accumulators are final
      __syncwarp();
    }
    // no tcgen05.commit arrival may land after the CTA exits: wait for the
    // last commit on every slot pair and stage (pair h' / quad q' = last use)
    for (int k = 0; k < kPairs && k < h; ++k) {
      const int hl = k + ((h - 1 - k) / kPairs) * kPairs;
      mbar_wait(smem_u32(&sdone[k]), (uint32_t)(hl / kPairs) & 1u);
    }
    const int nq = h >> 1;
    for (int k = 0; k < kBStages && k < nq; ++k) {
      const int ql = k + ((nq - 1 - k) / kBStages) * kBStages;
      mbar_wait(smem_u32(&bempty[k]), (uint32_t)(ql / kBStages) & 1u);
    }
  } else if (warp < kWarpEpi0) {
    // ======================= converters: fp32 -> digit planes in TMEM =======================
    // Group grp takes the chunks g with g % 2 == grp; within a group warp q
    // owns TMEM lane quarter q (access rule), thread = MMA row.
    const int grp = (warp - kWarpConv0) >> 2;
    const int q = warp & 3;
    const int row = q * 32 + lane;
    int g = 0;
    for (int u = u0; u < total_units; u += ustep) {
      const Unit x = unit_of(p, u);
      const int gi = x.tile * 128 + row;
      const float s = 256.f * scale_of(gi < p.rows ? p.rowmax[gi] : 0.f);  // the row's 31-bit grid
      for (int c = 0; c < x.n; ++c, ++g) {
        if (g % kConvGroups != grp) continue;
        const int pg = g / kMGroup, ps = pg % kMGroups, slot = g % kSlots, sp = (g >> 1) % kPairs;
        const uint32_t mph = (uint32_t)(pg / kMGroups) & 1u, sphase = (uint32_t)(g / kSlots) & 1u;
        mbar_wait(smem_u32(&mfull[ps]), mph);
        // digit planes d1 (words 0..7) | d2 (8..15) | d3 (16..23) | d4 (24..31);
        // word j holds elements 4j .. 4j + 3, element t of the word in byte t
        uint32_t pl[32];
        const uint32_t tile = smem_u32(sm_m) + (uint32_t)((ps * kMGroup + g % kMGroup) * kMTileBytes);
        if (!TRANS && p.wide) {
          // group buffer [row][chunk][32] (SWIZZLE_128B per 128-byte line):
          // this chunk's row is line kMGroup row + c, 16-byte piece j at
          // j ^ (line & 7); lanes 4..7 of each quarter-warp walk the pieces
          // flipped (j ^ 1) to spread the wavefront over the bank groups;
          // the planes of adjacent pieces are swapped back afterwards
          const uint32_t pairb = smem_u32(sm_m) + (uint32_t)(ps * kMGroup * kMTileBytes);
          const uint32_t line = (uint32_t)kMGroup * (uint32_t)row + (uint32_t)(g % kMGroup);
          const int flip = (lane >> 2) & 1;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float a0, a1, a2, a3;
            lds128(pairb + line * 128 + ((((uint32_t)(j ^ flip)) ^ (line & 7)) << 4), a0, a1, a2, a3);
            planes4x(a0, a1, a2, a3, s, pl[j], pl[8 + j], pl[16 + j], pl[24 + j]);
          }
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const uint32_t e0 = pl[j], e1 = pl[j + 1];
            pl[j] = flip ? e1 : e0;
            pl[j + 1] = flip ? e0 : e1;
          }
        } else if (!TRANS) {
          // row `row` of a 128 x 32 SWIZZLE_128B tile: 16-byte piece j at j ^ (row & 7)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float a0, a1, a2, a3;
            lds128(tile + row * 128 + ((j ^ (row & 7)) << 4), a0, a1, a2, a3);
            planes4x(a0, a1, a2, a3, s, pl[j], pl[8 + j], pl[16 + j], pl[24 + j]);
          }
        } else {
          // column `row` of a 32 x 128 (k x j) tile, no swizzle
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t b0 = tile + (uint32_t)((4 * j * 128 + row) * 4);
            planes4x(lds32(b0), lds32(b0 + 512), lds32(b0 + 1024), lds32(b0 + 1536), s, pl[j], pl[8 + j], pl[16 + j],
                     pl[24 + j]);
          }
        }
        // generic-proxy reads of the slice before the async-proxy (TMA) refill
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&mempty[ps]));
        mbar_wait(smem_u32(&sdone[sp]), sphase ^ 1);
        tc_fence_after();
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + kStg0 + slot * kSlotCols;
        tmem_st16(ta, reinterpret_cast<const uint32_t(&)[16]>(pl[0]));
        tmem_st16(ta + 16, reinterpret_cast<const uint32_t(&)[16]>(pl[16]));
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&ready[sp]));
      }
    }
  } else {
    // ======================= epilogue: int32 groups -> fp64 =======================
    // 4 warps: lane quarter q (TMEM access rule), all r_pad columns.
    const int q = warp & 3;
    const int row = q * 32 + lane;
    // output column k's 1 / s_f: lane holds columns lane and 32 + lane
    // (broadcast by shuffles)
    const double cinv0 = lane < p.r ? 1.0 / fscale_of(p.fmax[lane]) : 0.0;
    const double cinv1 = 32 + lane < p.r ? 1.0 / fscale_of(p.fmax[32 + lane]) : 0.0;
    // class c of output column k is TMEM column c r_pad + k (8-column blocks
    // below r_pad)
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t zero[16] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    auto zero_acc = [&]() {
#pragma unroll
      for (int c = 0; c < kClasses; ++c)
#pragma unroll
        for (int h = 0; h < kGroupCols / 8; ++h)
          if (h * 8 < p.rp) tmem_st8(tq + c * p.rp + h * 8, reinterpret_cast<const uint32_t(&)[8]>(zero[0]));
      tmem_wait_st();
    };
    // the accumulators start at zero and are re-zeroed after every drain:
    // the MMAs always accumulate (aempty phase 0 = this initial zeroing)
    zero_acc();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&aempty[0]));
    int uc = 0;
    for (int u = u0; u < total_units; u += ustep, ++uc) {
      const Unit x = unit_of(p, u);
      const int gi = x.tile * 128 + row;
      const double rinv = 1.0 / (double)scale_of(gi < p.rows ? p.rowmax[gi] : 0.f);
      mbar_wait<256>(smem_u32(&afull[0]), (uint32_t)uc & 1u);
      tc_fence_after();
      {
#pragma unroll
        for (int h = 0; h < kGroupCols / 8; ++h) {  // 8 columns at a time
          if (h * 8 >= p.rp) break;
          uint32_t g[kClasses][8];
#pragma unroll
          for (int c = 0; c < kClasses; ++c) tmem_ld8(tq + c * p.rp + h * 8, g[c]);
          tmem_wait_ld();
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int k = h * 8 + kk;
            const double ck = __shfl_sync(0xffffffffu, k < 32 ? cinv0 : cinv1, k & 31);  // all lanes
            // sum X Y = 2^24 (G0 2^24 + G1 2^16 + G2 2^8 + G3), the bracket
            // exact in int64 (|G0| < 2^14 K <= 2^29 for a unit's K <= 32768),
            // then one fp64 rounding; X = x * 256 s_hi, so the 2^24 / 256
            // folds into 2^16
            const long long S =
                (((long long)(int)g[0][kk] * 256ll + (int)g[1][kk]) * 256ll + (int)g[2][kk]) * 256ll + (int)g[3][kk];
            const double v = (double)S * 65536.0 * rinv * ck;
            if (gi < p.rows && k < p.r) {
              if (!TRANS)
                p.part[(size_t)x.split * p.rows * p.r + (size_t)gi * p.r + k] = v;
              else
                p.part[(size_t)x.split * p.r * p.rows + (size_t)k * p.rows + gi] = v;
            }
          }
        }
        zero_acc();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&aempty[0]));
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kWarpMma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// ----------------------------------------------------------------------------
// Per-level statistics of M (once per level): row and column maxima, as
// float bit patterns combined with atomicMax (M >= 0: nonnegative floats
// order like their bit patterns).  Block: 256 threads x float4 = 1024
// columns, kStatRows rows; row maxima reduced per row through shared memory.
// ----------------------------------------------------------------------------
constexpr int kStatRows = 512;
__global__ void __launch_bounds__(256) k_mstats(const float* __restrict__ M, size_t m, size_t n,
                                                unsigned* __restrict__ rowmax, unsigned* __restrict__ colmax,
                                                double* __restrict__ sqpart) {
  __shared__ float part[kStatRows][8];
  __shared__ double sqw[8];
  double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0;  // the block's share of ||M||_F^2 (fp64, as k_sq_partial_v4)
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const size_t j = (size_t)blockIdx.x * 1024 + (size_t)t * 4;
  const size_t i0 = (size_t)blockIdx.y * kStatRows;
  const int nr = (int)std::min<size_t>(kStatRows, m - i0);
  float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
  for (int ii = 0; ii < nr; ++ii) {
    float tm = 0.f;
    if (j < n) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(M + (i0 + ii) * n + j));
      c0 = fmaxf(c0, v.x), c1 = fmaxf(c1, v.y), c2 = fmaxf(c2, v.z), c3 = fmaxf(c3, v.w);
      tm = fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w));
      if (sqpart) {
        q0 = fma((double)v.x, (double)v.x, q0), q1 = fma((double)v.y, (double)v.y, q1);
        q2 = fma((double)v.z, (double)v.z, q2), q3 = fma((double)v.w, (double)v.w, q3);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, o));
    if (lane == 0) part[ii][warp] = tm;
  }
  if (j < n) {
    atomicMax(colmax + j, __float_as_uint(c0));
    atomicMax(colmax + j + 1, __float_as_uint(c1));
    atomicMax(colmax + j + 2, __float_as_uint(c2));
    atomicMax(colmax + j + 3, __float_as_uint(c3));
  }
  __syncthreads();
  for (int ii = t; ii < nr; ii += 256) {
    float tm = part[ii][0];
#pragma unroll
    for (int w = 1; w < 8; ++w) tm = fmaxf(tm, part[ii][w]);
    atomicMax(rowmax + i0 + ii, __float_as_uint(tm));
  }
  if (sqpart) {  // one partial per block, summed in block order by the caller (deterministic)
    double q = (q0 + q1) + (q2 + q3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    if (lane == 0) sqw[warp] = q;
    __syncthreads();
    if (t == 0) {
      double tot = 0.0;
      for (int w = 0; w < 8; ++w) tot += sqw[w];
      sqpart[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = tot;
    }
  }
}

// Factor maxima: row k of F (fp64) over its K elements, rounded UP to fp32
// (the scale chosen from it must keep every rounded entry <= kXMax).  F is
// either row-major r x K (W; trans = 0) or K x r (V; trans = 1).
__global__ void __launch_bounds__(256) k_fmax(const double* __restrict__ F, int r, size_t K, int trans,
                                              unsigned* __restrict__ fmax) {
  __shared__ double red[256];
  const int t = threadIdx.x;
  if (!trans) {
    // block (k, segment): a strided pass over row k
    const int k = blockIdx.x % r;
    const size_t seg = blockIdx.x / r, nseg = gridDim.x / r;
    double mx = 0.0;
    for (size_t e = seg * 256 + t; e < K; e += nseg * 256) mx = ::fmax(mx, F[(size_t)k * K + e]);
    red[t] = mx;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (t < o) red[t] = ::fmax(red[t], red[t + o]);
      __syncthreads();
    }
    if (t == 0) atomicMax(fmax + k, __float_as_uint(fmaxf(__double2float_ru(red[0]), 0.f)));
  } else {
    // rows i of V, thread (lane group gq, column k): k = t % 64, 4 row lanes
    const int k = t & 63, gq = t >> 6;
    double mx = 0.0;
    if (k < r)
      for (size_t i = (size_t)blockIdx.x * 4 + gq; i < K; i += (size_t)gridDim.x * 4) mx = ::fmax(mx, F[i * r + k]);
    red[t] = mx;
    __syncthreads();
    if (t < 64 && k < r) {
      const double v = ::fmax(::fmax(red[t], red[t + 64]), ::fmax(red[t + 128], red[t + 192]));
      atomicMax(fmax + k, __float_as_uint(fmaxf(__double2float_ru(v), 0.f)));
    }
  }
}

// Factor digit slices (fp64 factor), one 4 r_pad-row block per chunk QUAD
// (K elements 128 q .. 128 q + 127): row j r_pad + k holds digit plane e_(j+1)
// of factor row k, 128 bytes = 4 chunks x 32 elements (the MMA's stacked B
// operand: N = 4 r_pad rows, chunk cq at byte 32 cq).  Zero for k >= r or
// beyond K.  Thread (q, k, cq, qd): 4 consecutive elements -> one word of
// each plane row.
__global__ void __launch_bounds__(256) k_fdigits(const double* __restrict__ F, int r, int rp, size_t K,
                                                 size_t nquads, int trans, const float* __restrict__ fmax,
                                                 uint32_t* __restrict__ D) {
  const size_t total = nquads * (size_t)rp * 32;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    size_t q;
    int k, w;  // w = cq * 8 + qd: the word within the 128-byte row
    if (!trans) {  // words fastest: 32 threads read 128 consecutive elements of one W row
      w = (int)(e & 31);
      k = (int)((e >> 5) % rp);
      q = (e >> 5) / rp;
    } else {       // factor rows fastest: consecutive threads read consecutive V entries
      k = (int)(e % rp);
      w = (int)((e / rp) & 31);
      q = (e / rp) >> 5;
    }
    uint32_t wv[4] = {0u, 0u, 0u, 0u};
    bool any = false;
    if (k < r) {
      const double s = fscale_of(fmax[k]);
      const size_t j0 = q * 128 + (size_t)w * 4;
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      if (!trans && j0 + 3 < K) {  // K % 4 == 0: 16-byte aligned pairs
        const double2 a = *reinterpret_cast<const double2*>(F + (size_t)k * K + j0);
        const double2 b = *reinterpret_cast<const double2*>(F + (size_t)k * K + j0 + 2);
        v[0] = a.x, v[1] = a.y, v[2] = b.x, v[3] = b.y;
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (j0 + t < K) v[t] = trans ? F[(j0 + t) * r + k] : F[(size_t)k * K + j0 + t];
      }
      // the fp64 entry rounded once (half-even) to its row's 31-bit grid:
      // X + 0x808080 = e1 | e2 + 128 | e3 + 128 | e4 + 128 (bytes 3..0)
#pragma unroll
      for (int t = 0; t < 4; ++t) wv[t] = (uint32_t)(long long)(rint(v[t] * s) + kFBias);
      any = true;
    }
    uint32_t p1 = 0u, p2 = 0u, p3 = 0u, p4 = 0u;
    if (any) planes_of(wv, p1, p2, p3, p4);  // byte t of plane j = digit j of element t
    uint32_t* rowq = D + (q * 4 * rp + k) * 32 + w;  // plane j's row: + j rp rows
    rowq[0] = p1;
    rowq[(size_t)rp * 32] = p2;
    rowq[(size_t)2 * rp * 32] = p3;
    rowq[(size_t)3 * rp * 32] = p4;
  }
}

// out[e] = sum_z part[z][e], z ascending (deterministic split-K epilogue)
__global__ void k_split_reduce(const double* __restrict__ part, size_t count, int splits, double* __restrict__ out) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (size_t)gridDim.x * blockDim.x) {
    double s = part[e];
    for (int z = 1; z < splits; ++z) s += part[(size_t)z * count + e];
    out[e] = s;
  }
}

}  // namespace ix

// ============================================================================
// host side
// ============================================================================
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    IX_CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

void encode(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* ptr, const cuuint64_t* dims,
            const cuuint64_t* strides, const cuuint32_t* box, bool swz) {
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(m, dt, rank, const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           // 128-byte L2 promotion: 256 B measured 1.5-2 % slower on both products (r02, three
                           // alternations on one box; 64 B and none equal 128 B)
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

// 2-D fp32 map: inner extent `inner`, outer `outer`, row stride inner * 4 B
CUtensorMap map_f32(const void* ptr, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo, bool swz) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 4};
  cuuint32_t box[2] = {bi, bo};
  encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ptr, dims, strides, box, swz);
  return m;
}
// 3-D view of a row-major fp32 matrix (n % (32 kMGroup) == 0): (32 columns,
// n / 32 column blocks, m rows), box (32, kMGroup, 128): one 128-row x
// (128 kMGroup)-byte slab laid out [row][block][32] with the 128-byte swizzle.
CUtensorMap map_rows3(const void* ptr, uint64_t n, uint64_t m) {
  CUtensorMap map;
  cuuint64_t dims[3] = {32, n / 32, m};
  cuuint64_t strides[2] = {128, n * 4};
  cuuint32_t box[3] = {32, (cuuint32_t)ix::kMGroup, 128};
  encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims, strides, box, true);
  return map;
}
// factor digit slices: rows of 128 bytes, box = the 4 r_pad rows of a chunk quad
CUtensorMap map_digits(const void* ptr, uint64_t rows, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {128, rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {128, box_rows};
  encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, ptr, dims, strides, box, true);
  return m;
}

size_t cdiv(size_t a, size_t b) { return (a + b - 1) / b; }

class IxGemm final : public TcGemm {
 public:
  explicit IxGemm(bool forced) : forced_(forced) {
    int dev = 0;
    IX_CK(cudaGetDevice(&dev));
    IX_CK(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev));
  }
  ~IxGemm() override {
    for (void* p : {digits_, part_, fmax_})
      if (p) cudaFree(p);
  }
  uint64_t signature() const override {
    uint64_t h = 1469598103934665603ull;
    for (const void* p : {digits_, part_, fmax_}) h = (h ^ (uint64_t)(uintptr_t)p) * 1099511628211ull;
    return h;
  }
  bool supports(size_t m, size_t n, size_t r) const override {
    return r >= 1 && r <= 64 && m % 4 == 0 && n % 4 == 0 && m >= 128 && n >= 128 && m < (1u << 31) &&
           n < (1u << 31);
  }
  bool wants(size_t m, size_t n, size_t r) const override {
    if (!supports(m, n, r)) return false;
    return forced_ || m * n >= ((size_t)1 << 24);
  }

  size_t level_stats_blocks(size_t m, size_t n) const override { return cdiv(n, 1024) * cdiv(m, ix::kStatRows); }
  void level_stats(const float* M, size_t m, size_t n, float* rowmax, float* colmax, double* sqpart, cudaStream_t s,
                   long* launches) override {
    IX_CK(cudaMemsetAsync(rowmax, 0, m * 4, s));
    IX_CK(cudaMemsetAsync(colmax, 0, n * 4, s));
    dim3 g((unsigned)cdiv(n, 1024), (unsigned)cdiv(m, ix::kStatRows));
    ix::k_mstats<<<g, 256, 0, s>>>(M, m, n, reinterpret_cast<unsigned*>(rowmax), reinterpret_cast<unsigned*>(colmax),
                                   sqpart);
    IX_CK(cudaGetLastError());
    ++*launches;
  }

  void mwt(const float* M, const float* rowmax, const double* W, size_t m, size_t n, size_t r, double* A,
           cudaStream_t s, long* launches) override {
    run<false>(M, rowmax, W, m, n, r, A, s, launches);
  }
  void vtm(const double* V, const float* M, const float* colmax, size_t m, size_t n, size_t r, double* C,
           cudaStream_t s, long* launches) override {
    run<true>(M, colmax, V, m, n, r, C, s, launches);
  }

 private:
  template <bool TRANS>
  void run(const float* M, const float* rowmax, const double* F, size_t m, size_t n, size_t r, double* out,
           cudaStream_t s, long* launches) {
    if (!supports(m, n, r)) throw std::invalid_argument("tcgen05 path: unsupported shape");
    const int rp = (int)cdiv(r, 16) * 16;
    const size_t K = TRANS ? m : n;     // contraction
    const size_t rows = TRANS ? n : m;  // MMA-M extent
    // chunks are processed in quads (the factor stage) of pairs (the MMA
    // loop): a ragged tail is padded with zero chunks (TMA zero-fills M
    // beyond K, the factor digits are zero there)
    const size_t nchunks = cdiv(cdiv(K, ix::kChunk), ix::kQuad) * ix::kQuad;
    const size_t nquads = nchunks / ix::kQuad;
    // factor: row maxima, then digit slices [nchunks][rp][128 B]
    ensure(&fmax_, &fmax_bytes_, 64 * 4);
    ensure(&digits_, &digits_bytes_, nchunks * rp * 128);  // = nquads x 4 rp rows x 128 B
    IX_CK(cudaMemsetAsync(fmax_, 0, 64 * 4, s));
    {
      const unsigned g = TRANS ? (unsigned)std::min<size_t>(cdiv(K, 4), (size_t)sms_ * 4)
                               : (unsigned)(r * std::max<size_t>(1, std::min<size_t>(cdiv(K, 4096), 32)));
      ix::k_fmax<<<g, 256, 0, s>>>(F, (int)r, K, TRANS ? 1 : 0, static_cast<unsigned*>(fmax_));
      const size_t tot = nquads * rp * 32;
      ix::k_fdigits<<<(unsigned)std::min<size_t>(cdiv(tot, 256), 16384), 256, 0, s>>>(
          F, (int)r, rp, K, nquads, TRANS ? 1 : 0, static_cast<const float*>(fmax_), static_cast<uint32_t*>(digits_));
      IX_CK(cudaGetLastError());
      *launches += 2;
    }
    ix::Params p{};
    p.rows = (int)rows;
    p.kdim = (int)K;
    p.r = (int)r;
    p.rp = rp;
    p.tiles = (int)cdiv(rows, 128);
    p.nchunks = (int)nchunks;
    p.wide = (!TRANS && n % (32 * ix::kMGroup) == 0) ? 1 : 0;
    p.rowmax = rowmax;
    p.fmax = static_cast<const float*>(fmax_);
    // split-K: units (tile, K range) are dealt round-robin to the persistent
    // CTAs, so the kernel lasts ceil(units / SMs) units.  Pick the split
    // factor that maximises the balanced fraction units / (ceil(units / SMs)
    // SMs), charging each extra split its fp64 partial-output traffic (write
    // + reduce read, 16 B per output element) against the M bytes streamed;
    // a unit holds at most kMaxUnitChunks chunks (exact int32 accumulation).
    const int smin = (int)cdiv(nchunks, ix::kMaxUnitChunks);
    int splits = smin;
    {
      double best = -1.0;
      const int smax = std::max(smin, std::min<int>((int)nchunks / 8, 64));
      for (int sp = smin; sp <= smax; ++sp) {
        int cps = (int)cdiv(nchunks, sp);
        cps = (int)cdiv(cps, ix::kQuad) * ix::kQuad;  // whole chunk quads per unit
        if (cps > ix::kMaxUnitChunks) continue;
        const int spr = (int)cdiv(nchunks, cps);
        const double units = (double)p.tiles * spr;
        const double rounds = std::ceil(units / sms_);
        const double balance = units / (rounds * sms_);
        const double extra = spr > 1 ? (double)spr * rows * r * 16.0 / ((double)rows * K * 4.0) : 0.0;
        const double score = balance / (1.0 + extra);
        if (score > best + 1e-9) best = score, splits = sp;
      }
    }
    p.chunks_per_split = (int)cdiv(nchunks, splits);
    p.chunks_per_split = (int)cdiv(p.chunks_per_split, ix::kQuad) * ix::kQuad;
    p.splits = (int)cdiv(nchunks, p.chunks_per_split);
    const size_t out_count = rows * r;
    double* dst = out;
    if (p.splits > 1) {
      ensure(&part_, &part_bytes_, (size_t)p.splits * out_count * 8);
      dst = static_cast<double*>(part_);
    }
    p.part = dst;
    const CUtensorMap mm = TRANS    ? map_f32(M, n, m, 128, ix::kChunk, false)
                           : p.wide ? map_rows3(M, n, m)
                                    : map_f32(M, n, m, ix::kChunk, 128, true);
    const CUtensorMap mb = map_digits(digits_, nchunks * rp, 4u * (uint32_t)rp);
    const size_t smem = 1024 + ix::kMStages * ix::kMTileBytes + ix::kBStages * ix::kBStageBytes + 256;
    auto kern = TRANS ? ix::k_ix_product<true> : ix::k_ix_product<false>;
    if (!attr_set_[TRANS ? 1 : 0]) {
      IX_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr_set_[TRANS ? 1 : 0] = true;
    }
    const int units = p.tiles * p.splits;
    const int grid = std::min(units, sms_);
    kern<<<grid, ix::kThreads, smem, s>>>(mm, mb, p);
    IX_CK(cudaGetLastError());
    ++*launches;
    if (p.splits > 1) {
      const unsigned g = (unsigned)std::min<size_t>(cdiv(out_count, 256), 4096);
      ix::k_split_reduce<<<g, 256, 0, s>>>(static_cast<const double*>(part_), out_count, p.splits, out);
      IX_CK(cudaGetLastError());
      ++*launches;
    }
  }

  static void ensure(void** p, size_t* have, size_t need) {
    if (need <= *have) return;
    if (*p) IX_CK(cudaFree(*p));
    *p = nullptr;
    IX_CK(cudaMalloc(p, need));
    *have = need;
  }

  bool forced_;
  int sms_ = 148;
  void* digits_ = nullptr;
  size_t digits_bytes_ = 0;
  void* part_ = nullptr;
  size_t part_bytes_ = 0;
  void* fmax_ = nullptr;
  size_t fmax_bytes_ = 0;
  bool attr_set_[2] = {false, false};
};

}  // namespace

TcGemm* make_tc_gemm(bool allowed, bool forced) {
  if (!allowed) {
    if (forced) throw std::invalid_argument("the tensor-core path needs fp32 storage");
    return nullptr;
  }
  return new IxGemm(forced);
}

}  // namespace mlb
