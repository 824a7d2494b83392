// tc_gemm.cu -- the two M-streaming products on the 5th-generation tensor
// cores (tcgen05, sm_100a), fp32 storage, 3xTF32 precision:
//
//   product 1 (TRANS = false):  A (m x r)  = M (m x n) . W^T       (solvers.cpp:82,105,252)
//   product 2 (TRANS = true):   C^T (n x r) = M^T (n x m) . V      (solvers.cpp:91,124,273)
//
// Both stream M from HBM exactly once.  MMA operand roles (M = 128 rows of the
// MMA, N = r_pad, K = 8 per tcgen05.mma, kind::tf32):
//   A operand: a 128 x 32 slice of M (product 1) or of M^T (product 2), split
//              by the converter warps into tf32 hi = rna(x) and lo = rna(x - hi)
//              and written straight into a TMEM staging slot (tcgen05.st).
//   B operand: [F_hi ; F_lo] (2 r_pad x 32, K-major, SWIZZLE_128B) where F is
//              W (product 1) or V^T (product 2), pre-split once per step by a
//              small kernel and brought in by TMA.
// K3 form (default): per 32-K chunk, 12 MMAs of N = r_pad accumulate
//   D[:, 0:r) += [A_hi A_lo A_hi] . [F_hi F_hi F_lo]^T = A_hi F_hi + A_lo F_hi + A_hi F_lo
// (3xTF32) into an r-column accumulator; A_hi is re-read from the slot, F_hi /
// F_lo are rows 0..r_pad / r_pad..2 r_pad of the factor stage.  (The stacked
// form, 4 MMAs of N = 2 r_pad + 4 of N = r_pad into 2 r_pad columns, is kept
// behind MLB_TC_K3=0.)
// fp32 TMEM accumulation is limited to windows of kWindow chunks; the
// epilogue warps drain each window into fp64 registers and write fp64 split-K
// partials that a deterministic reduce sums in fixed order.
// Why windows: the tensor core's fp32 accumulate truncates toward zero, so on
// the all-nonnegative NMF operands the error is a one-sided bias that grows
// linearly with the accumulation length (per chunk ~2.4e-7 relative in the
// stacked form, ~3e-7 in K3; tools/tc_check.py: window 64 -> 1.6e-5, 8 ->
// 1.9e-6, 1 -> 2.0e-7).  kWindow = 6 keeps the products ~2e-6 of fp64.
//
// Warp roles (640 threads, one persistent CTA per SM, 512 TMEM columns =
// 2 MMA warps x 2 accumulator buffers x r_pad + 4 staging slots x 64):
//   warp 0: TMA producer (M slices, issued and released in pairs)
//   warps 1, 2: MMA issuers for even / odd chunks, each into its own pair of
//               accumulator buffers (windows alternate buffers, so a warp
//               never waits for a drain); warp 1 allocates TMEM
//   warps 3-10: converters (two groups of 4: even / odd chunks)
//   warps 11-18: epilogue (lane quarter x column half), drains all windows
//   warp 19: TMA producer (factor slices, one thread, stream order)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "tc_gemm.hpp"

namespace mlb {
namespace tc {

// nanosleep (ns) between failed barrier polls of the TMA producers and of
// the converters (0: spin); spinning warps take issue slots and power
#ifndef MLB_TC_ST64
#define MLB_TC_ST64 0  // one 64-column tcgen05.st per chunk instead of two of 32
#endif
#ifndef MLB_TC_PSLEEP
#define MLB_TC_PSLEEP 0
#endif
#ifndef MLB_TC_CSLEEP
#define MLB_TC_CSLEEP 0
#endif
#ifndef MLB_TC_MSTAGES
#define MLB_TC_MSTAGES 8
#endif
constexpr int kMStages = MLB_TC_MSTAGES;  // M-slice ring (TMA -> converters), 16 KB each
#ifndef MLB_TC_MGROUP
#define MLB_TC_MGROUP 2
#endif
constexpr int kMGroup = MLB_TC_MGROUP;       // the ring is filled and released in groups of slices
constexpr int kMGroups = kMStages / kMGroup;
static_assert(kMStages % kMGroup == 0, "M ring: whole groups");
#ifndef MLB_TC_K3
#define MLB_TC_K3 1
#endif
// K3 form: D[:, 0:r) += [A_hi A_lo A_hi] . [F_hi F_hi F_lo]^T as one r-column
// accumulation (12 N = r MMAs per chunk); else the stacked form
// D[:, 0:2r) += A_hi [F_hi;F_lo]^T, D[:, 0:r) += A_lo F_hi^T (2r columns).
constexpr bool kK3 = MLB_TC_K3 != 0;
#ifndef MLB_TC_ACCBUFS
#define MLB_TC_ACCBUFS 2
#endif
// accumulator buffers per MMA warp: with 2, a warp starts its next window
// while the epilogue drains the previous one (K3 form only: 4 x r_pad columns)
constexpr int kAccBufs = kK3 ? MLB_TC_ACCBUFS : 1;
constexpr int kSlots = kK3 ? (512 - 2 * kAccBufs * 64) / 64 : 4;  // TMEM staging slots (hi|lo, 64 columns each)
#ifndef MLB_TC_BSINGLE
#define MLB_TC_BSINGLE 1  // one thread issues every factor slice in stream order
#endif
#ifndef MLB_TC_BSTAGES
#define MLB_TC_BSTAGES 6
#endif
// factor-slice ring: deeper than the staging slots, because a slice can only be
// refilled after the MMAs reading it complete and the refill's TMA latency
// (~1-2k cycles) must be covered (traced: a 4-deep ring lockstepped with the
// slots left the MMA warps waiting ~1000 cycles per chunk for B).
constexpr int kBStages = MLB_TC_BSTAGES;
#ifndef MLB_TC_BPREFETCH
#define MLB_TC_BPREFETCH 0
#endif
constexpr int kBPrefetch = MLB_TC_BPREFETCH;  // factor slices prefetched into L2 this many chunks ahead
static_assert(MLB_TC_BSINGLE || kBStages % 2 == 0, "B ring: even/odd chunk producers own alternate stages");
constexpr int kBStageBytes = 16384;  // fixed stride (2 r_pad x 128 B <= 16 KB)
constexpr int kAccStride = kK3 ? 64 : 128;  // TMEM columns per accumulator (r_pad or 2 r_pad)
constexpr int kStgCol0 = 2 * kAccBufs * kAccStride;  // staging slots follow the accumulators
static_assert(kStgCol0 + kSlots * 64 == 512, "TMEM map: accumulators + staging = 512 columns");
constexpr int kChunk = 32;        // K elements per pipeline chunk (128 B rows)
#ifndef MLB_TC_WINDOW
#define MLB_TC_WINDOW 6
#endif
constexpr int kWindow = MLB_TC_WINDOW;  // chunks per fp32 accumulation window
constexpr int kConvGroups = 2;    // converter groups of 4 warps (alternate chunks)
constexpr int kWarpM = 0;                            // TMA producer: M slices
constexpr int kWarpMma0 = 1, kWarpMma1 = 2;           // MMA issuers (even / odd chunks); 1 allocates TMEM
constexpr int kWarpConv0 = 3;                        // converter groups
constexpr int kWarpEpi0 = kWarpConv0 + 4 * kConvGroups;  // 8 epilogue warps
constexpr int kWarpB = kWarpEpi0 + 8;                // TMA producers: factor slices (lanes 0 / 1)
constexpr int kThreads = (kWarpB + 1) * 32;
constexpr int kMTileBytes = 128 * kChunk * 4;  // 16 KB

#define TC_CK(x)                                                                                  \
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
// Bounded wait: a pipeline bug traps (kernel error) after ~2^34 cycles instead
// of hanging the GPU.
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
template <int SLEEP_NS = 0>
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  if (mbar_try(a, parity)) return;
  const long long t0 = clock64();
  for (uint32_t i = 1;; ++i) {
    if (SLEEP_NS) __nanosleep(SLEEP_NS);  // off-critical-path waiters yield issue slots
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
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}
// TMA load with an L2 cache-policy hint (createpolicy): the M stream is read
// once (evict_first) and must not push out the factor slices, which every CTA
// of the split re-reads (evict_last).
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d_hint(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t mbar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(mbar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_hint(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint32_t mbar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(mbar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// CTA pairs (cta_group::2): the peer-visible address of a shared-memory
// location in CTA `cta` of the cluster, and a release arrive on it
__device__ __forceinline__ uint32_t cluster_addr(uint32_t local, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(cta));
  return r;
}
// (default .release.cta semantics, as CUTLASS's ClusterBarrier::arrive: a
// .cluster-scope release compiles to a MEMBAR that stalled the converters and
// the epilogue ~100k samples in ncu and made the pair kernel 1.6x slower)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t caddr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA into this CTA's shared memory, completion counted on an mbarrier that
// may live in the peer CTA of the pair (the leader's)
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t mbar_c,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(mbar_c), "l"(pol)
      : "memory");
}
// pair commit: arrives on the barrier at this offset in both CTAs
__device__ __forceinline__ void tc_commit_pair(uint32_t mbar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(mbar),
      "h"((uint16_t)3)
      : "memory");
}
// warp-wide call; one elected lane commits
__device__ __forceinline__ void tc_commit(uint32_t mbar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(mbar)
      : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]^T, kind::tf32, M = 128; warp-wide call, one
// elected lane issues.
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

#define TC_REG32(v) \
  "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), \
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),          \
      "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]),           \
      "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
#define TC_OREG32(v)                                                                                           \
  "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), \
      "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),  \
      "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), \
      "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      TC_REG32(v)
      : "memory");
}
// 64 consecutive columns (hi | lo of a staging slot) in one instruction
__device__ __forceinline__ void tmem_st64(uint32_t taddr, const uint32_t (&a)[32], const uint32_t (&b)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, "
      "%37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, "
      "%59, %60, %61, %62, %63, %64};" ::"r"(taddr),
      TC_REG32(a), TC_REG32(b)
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
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : TC_OREG32(v)
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor: K-major, SWIZZLE_128B, 8-row atoms of
// 128 B (SBO = 1024 B), Blackwell version bit.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;                 // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024u >> 4) << 32;       // SBO
  d |= (uint64_t)1u << 46;                 // version = 1 (sm_100)
  d |= (uint64_t)2u << 61;                 // SWIZZLE_128B
  return d;
}
// Instruction descriptor: D f32, A/B tf32, K-major both, N, M (128; 256 for
// a CTA pair).
__host__ __device__ constexpr uint32_t idesc_tf32(int N, int M = 128) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// One pipeline chunk (K = 32, four K-steps of 8) on staging slot S into
// accumulator ACC, issued by one elected lane in a single asm block:
//   D[:, 0:2r) (+)= A_hi [F_hi;F_lo]^T   and   D[:, 0:r) += A_lo F_hi^T.
// The four N = 2r MMAs go first, then the four N = r ones: alternating the two
// shapes on overlapping accumulator columns serialises every MMA on the
// previous one's result (measured ~2x slower issue).
// TMEM addresses and the B-descriptor offsets are compile-time constants
// (TMEM base 0, fixed strides), so the operands sit in uniform registers
// without per-chunk R2UR traffic.  `first` clears the accumulator (window start).
template <int S, int ACC>
__device__ __forceinline__ void issue_chunk(uint64_t bdesc, uint32_t id_full, uint32_t id_hi, uint32_t first) {
  constexpr uint32_t d = ACC * kAccStride;
  constexpr uint32_t a_hi = kStgCol0 + S * 64, a_lo = a_hi + 32;
  constexpr uint64_t boff = 0;  // bdesc addresses the factor-slice stage
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .pred p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.eq.u32 p, %13, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %5, %9, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%3], %6, %9, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%11], %7, %9, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%14], %8, %9, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %5, %10, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%4], %6, %10, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%12], %7, %10, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%15], %8, %10, 1;\n\t}" ::"r"(d),
      "r"(a_hi), "r"(a_lo), "r"(a_hi + 8), "r"(a_lo + 8), "l"(bdesc + boff), "l"(bdesc + boff + 2),
      "l"(bdesc + boff + 4), "l"(bdesc + boff + 6), "r"(id_full), "r"(id_hi), "r"(a_hi + 16), "r"(a_lo + 16),
      "r"(first), "r"(a_hi + 24), "r"(a_lo + 24)
      : "memory");
}

// K3 chunk: the accumulator holds only the r output columns; the three 3xTF32
// terms are one K = 96 accumulation, A = [A_hi A_lo A_hi] from the TMEM slot
// (A_hi re-read, not stored twice), B = [F_hi F_hi F_lo] from the factor slice
// (rows 0..r_pad of the stage, then rows r_pad..2 r_pad).  Half the TMEM
// columns of the stacked form, so 6 staging slots fit and the epilogue drains
// half as much.
#define MLB_ISSUE3(CG)                                                                                        \
  asm volatile(                                                                                              \
      "{\n\t.reg .pred e;\n\t.reg .pred p;\n\t"                                                              \
      "elect.sync _|e, 0xffffffff;\n\t"                                                                      \
      "setp.eq.u32 p, %12, 0;\n\t"                                                                           \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%1], %3, %11, p;\n\t"                              \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%13], %4, %11, 1;\n\t"                             \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%14], %5, %11, 1;\n\t"                             \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%15], %6, %11, 1;\n\t"                             \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%2], %3, %11, 1;\n\t"                              \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%16], %4, %11, 1;\n\t"                             \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%17], %5, %11, 1;\n\t"                             \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%18], %6, %11, 1;\n\t"                             \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%1], %7, %11, 1;\n\t"                              \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%13], %8, %11, 1;\n\t"                             \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%14], %9, %11, 1;\n\t"                             \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%15], %10, %11, 1;\n\t}" ::"r"(d),                \
      "r"(a_hi), "r"(a_lo), "l"(bd), "l"(bd + 2), "l"(bd + 4), "l"(bd + 6), "l"(bd_lo), "l"(bd_lo + 2),      \
      "l"(bd_lo + 4), "l"(bd_lo + 6), "r"(id), "r"(first), "r"(a_hi + 8), "r"(a_hi + 16), "r"(a_hi + 24),   \
      "r"(a_lo + 8), "r"(a_lo + 16), "r"(a_lo + 24)                                                         \
      : "memory")
// PAIR: the same 12 MMAs as one CTA-pair instruction stream (cta_group::2,
// M = 256: A from each CTA's own TMEM slot, B rows split r_pad / 2 per CTA)
// timing experiment (wrong results): MLB_TC_EXP_TERMS = 2 drops the A_lo F_hi
// MMAs, 1 also the A_hi F_lo ones -- the speed a split with fewer MMA passes
// per chunk could reach
#define MLB_ISSUE_N(CG, NT)                                                                             \
  asm volatile(                                                                                       \
      "{\n\t.reg .pred e;\n\t.reg .pred p;\n\t"                                                      \
      "elect.sync _|e, 0xffffffff;\n\t"                                                               \
      "setp.eq.u32 p, %8, 0;\n\t"                                                                     \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%1], %2, %7, p;\n\t"                        \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%9], %3, %7, 1;\n\t"                        \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%10], %4, %7, 1;\n\t"                       \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%11], %5, %7, 1;\n\t" NT "}" ::"r"(d),     \
      "r"(a_hi), "l"(bd), "l"(bd + 2), "l"(bd + 4), "l"(bd + 6), "l"(bd_lo), "r"(id), "r"(first),      \
      "r"(a_hi + 8), "r"(a_hi + 16), "r"(a_hi + 24), "l"(bd_lo + 2), "l"(bd_lo + 4), "l"(bd_lo + 6)    \
      : "memory")
#define MLB_HI_LO_TERM                                                                                 \
  "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %6, %7, 1;\n\t"                                  \
  "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%9], %12, %7, 1;\n\t"                                 \
  "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%10], %13, %7, 1;\n\t"                                \
  "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%11], %14, %7, 1;\n\t"
// MIXED: the two 3xTF32 cross terms A_lo F_hi + A_hi F_lo (each ~2^-11 of the
// result, so ~2^-11 relative accuracy suffices) as ONE K = 64 bf16 product
// [A_lo | A_hi] . [F_hi ; F_lo]: 4 kind::f16 MMAs (K = 16) instead of 8
// kind::tf32 ones (K = 8), next to the 4 tf32 MMAs of A_hi F_hi.  Same TMEM
// slot and factor-slice bytes: the converters store bf16 pairs in the lo
// half of the slot, k_split_factor writes the F_lo rows as bf16 [F_hi | F_lo]
// per 32-wide chunk (the same 128 bytes per row the TMA box fetches).
// Selected per launch (K % 32 == 0, no CTA pairs); MLB_TC_MIXED=0 disables it.
__host__ __device__ constexpr uint32_t idesc_bf16(int N, int M = 128) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
#ifndef MLB_TC_EXP_TERMS
#define MLB_TC_EXP_TERMS 3
#endif
#define MLB_ISSUE_MIXED(CG) \
  asm volatile( \
      "{\n\t.reg .pred e;\n\t.reg .pred p;\n\t" \
      "elect.sync _|e, 0xffffffff;\n\t" \
      "setp.eq.u32 p, %12, 0;\n\t" \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%1], %3, %11, p;\n\t" \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%13], %4, %11, 1;\n\t" \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%14], %5, %11, 1;\n\t" \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], [%15], %6, %11, 1;\n\t" \
      "@e tcgen05.mma.cta_group::" CG ".kind::f16 [%0], [%2], %7, %19, 1;\n\t" \
      "@e tcgen05.mma.cta_group::" CG ".kind::f16 [%0], [%16], %8, %19, 1;\n\t" \
      "@e tcgen05.mma.cta_group::" CG ".kind::f16 [%0], [%17], %9, %19, 1;\n\t" \
      "@e tcgen05.mma.cta_group::" CG ".kind::f16 [%0], [%18], %10, %19, 1;\n\t}" ::"r"(d), \
      "r"(a_hi), "r"(a_lo), "l"(bd), "l"(bd + 2), "l"(bd + 4), "l"(bd + 6), "l"(bd_lo), "l"(bd_lo + 2), \
      "l"(bd_lo + 4), "l"(bd_lo + 6), "r"(id), "r"(first), "r"(a_hi + 8), "r"(a_hi + 16), "r"(a_hi + 24), \
      "r"(a_lo + 8), "r"(a_lo + 16), "r"(a_lo + 24), "r"(idx) \
      : "memory")
template <int S, int ACC, bool PAIR = false, bool MIXED = false>
__device__ __forceinline__ void issue_chunk3(uint64_t bd, uint64_t bd_lo, uint32_t id, uint32_t first,
                                             uint32_t idx = 0) {
  constexpr uint32_t d = ACC * kAccStride;
  constexpr uint32_t a_hi = kStgCol0 + S * 64, a_lo = a_hi + 32;
  if constexpr (MIXED) {  // idx: the bf16 instruction descriptor (N = r_pad; M = 256 for a pair)
    if constexpr (PAIR)
      MLB_ISSUE_MIXED("2");
    else
      MLB_ISSUE_MIXED("1");
  return;
  }
#if MLB_TC_EXP_TERMS == 3
  if constexpr (PAIR)
    MLB_ISSUE3("2");
  else
    MLB_ISSUE3("1");
#elif MLB_TC_EXP_TERMS == 2
  (void)a_lo;
  MLB_ISSUE_N("1", MLB_HI_LO_TERM);
#else
  (void)a_lo;
  MLB_ISSUE_N("1", "");
#endif
}

// Optional event trace of CTA 0 (build with -DMLB_TC_TRACE=1; tools/tc_trace.py).
#if MLB_TC_TRACE
constexpr int kTraceChunks = 4096;
__device__ long long g_tctrace[8][kTraceChunks];
#define TCT(ev, gidx)                                                                        \
  do {                                                                                       \
    if (blockIdx.x == 0 && (gidx) < kTraceChunks && (threadIdx.x & 31) == 0) g_tctrace[ev][gidx] = clock64(); \
  } while (0)
#else
#define TCT(ev, gidx)
#endif

struct Params {
  int rows;        // MMA-M extent: m (product 1) or n (product 2)
  int kdim;        // K extent: n (product 1) or m (product 2)
  int r;           // true rank
  int rp;          // padded rank (multiple of 16, <= 64)
  int tiles;       // ceil(rows / 128)
  int splits;      // split-K factor
  int chunks_per_split;
  int nchunks;     // ceil(kdim / 32)
  int interleave;  // unit order: interleaved phases of one tile (see unit_of)
  int rotate;      // blocked order: rotate each tile's chunk order
  int wide;        // product 1: a chunk pair is one 3-D TMA box of 128 rows x 256 B
                   // (smem [row][half][32]); chunks_per_split even, n % 64 == 0
  double* part;    // [splits][...] fp64 partial outputs
};

// ----------------------------------------------------------------------------
// The persistent warp-specialised kernel
// ----------------------------------------------------------------------------
// Chunks are numbered g = 0, 1, 2, ... in the order a CTA streams them (all of
// its units, in order).  Parity w = g & 1 selects the converter group, the MMA
// warp, the factor-slice producer and the accumulator; g % kSlots the TMEM
// staging slot and B stage.  Within a unit, the chunks of parity w are
// i = i0(w), i0(w) + 2, ... with i0(w) = (w - g0) & 1.
__device__ __forceinline__ int own_first(int g0, int w) { return (w - g0) & 1; }
__device__ __forceinline__ int own_count(int g0, int n_u, int w) {
  const int i0 = own_first(g0, w);
  return n_u > i0 ? (n_u - i0 + 1) >> 1 : 0;
}

// Work units.  Blocked order (product 2, and product 1 at small strides):
// unit u = (tile u % tiles, K range u / tiles), chunks c_beg .. c_beg + n - 1;
// concurrent CTAs hold consecutive tiles (for product 2 adjacent column blocks
// of the same M rows).  Interleaved order (product 1 at >= 1 MiB row strides):
// unit u = (tile u / S, phase u % S), chunks phase, phase + S, ...; the S CTAs
// that run a tile concurrently fetch neighbouring 128-byte segments of the
// same rows.  (With whole-tile K ranges per CTA, 148 concurrent tiles at the
// same column offset hit the same DRAM channels: a pure TMA stream in that
// order tops out at ~4.7 TB/s against 7.4 TB/s with all CTAs on one tile --
// tools/stream_probe.cu -- but in the product kernel the interleaved order
// measured slower, so it is opt-in.)
struct Unit {
  int tile, split, n;
};
__device__ __forceinline__ Unit unit_of(const Params& p, int u) {
  Unit x;
  if (p.interleave == 1) {
    x.tile = u / p.splits;
    x.split = u % p.splits;
    x.n = (p.nchunks - x.split + p.splits - 1) / p.splits;
  } else {
    // 0: split-major (concurrent CTAs on consecutive tiles, same K range);
    // 2: tile-major (the splits of one tile run concurrently)
    x.tile = p.interleave == 2 ? u / p.splits : u % p.tiles;
    x.split = p.interleave == 2 ? u % p.splits : u / p.tiles;
    const int c_beg = x.split * p.chunks_per_split;
    x.n = min(c_beg + p.chunks_per_split, p.nchunks) - c_beg;
  }
  return x;
}
// chunk index of the i-th chunk of unit x.  With `rotate`, a blocked unit
// starts at a tile-dependent chunk (concurrent tiles then sit at different
// column offsets; +2-3 % for product 1 at 1 MiB row strides).
__device__ __forceinline__ int unit_chunk(const Params& p, const Unit& x, int i) {
  if (p.interleave == 1) return x.split + i * p.splits;
  if (p.rotate) {
    const int k = i + (int)(((long long)x.tile * 97) % x.n);
    i = k >= x.n ? k - x.n : k;
  }
  return x.split * p.chunks_per_split + i;
}

// MMA issuer for the chunks of parity W into accumulator W.  Two such warps
// run concurrently: the tensor pipe accepts an MMA only when it has room, so a
// single issuing warp stalls inside the MMAs and its per-chunk waits and
// commits leave the pipe idle; with two, one warp's bookkeeping overlaps the
// other's MMAs.
template <int W, bool PAIR, bool MIXED>
__device__ __forceinline__ void mma_role(const Params& p, int total_units, int u0, int ustep, bool issue,
                                         uint64_t bdesc0, uint64_t* ready,
                                         uint64_t* sdone, uint64_t* bfull, uint64_t* bempty, uint64_t* afull,
                                         uint64_t* aempty) {
  const uint32_t id_full = idesc_tf32(2 * p.rp), id_hi = idesc_tf32(p.rp, PAIR ? 256 : 128);
  const uint32_t id_x = idesc_bf16(p.rp, PAIR ? 256 : 128);  // MIXED cross terms
  int g = 0;
  int wc = 0;  // windows this warp has opened (all units): buffer wc % kAccBufs
  int lastph[kSlots / 2];    // parity of the last commit on this warp's slots W, W + 2, ...
#pragma unroll
  for (int k = 0; k < kSlots / 2; ++k) lastph[k] = -1;
  int lastb[kBStages];       // ... and on the factor-slice stages this warp used
#pragma unroll
  for (int k = 0; k < kBStages; ++k) lastb[k] = -1;
  // CTA pairs: K3 form only (the host never selects pairs otherwise)
  for (int u = u0; u < total_units; u += ustep) {
    const int n_u = unit_of(p, u).n;
    for (int i = own_first(g, W), j = 0; i < n_u; i += 2, ++j) {
      const int gg = g + i, slot = gg % kSlots;
      const uint32_t sph = (uint32_t)(gg / kSlots) & 1u;
      // accumulator 1's windows are offset by half a window (its first one
      // is kWindow / 2 long), so the two accumulators fill -- and stall their
      // warps for the drain -- at alternating times, not together
      const int wpos = (j + W * (kWindow / 2)) % kWindow;
      const int abuf = wc % kAccBufs, abar = W * kAccBufs + abuf;
      const int bs = gg % kBStages;
      if (!issue) {
        // peer CTA of a pair: no MMAs here, only the bookkeeping of the
        // leader's multicast commits for the drain below
        lastph[slot >> 1] = (int)sph;
        lastb[bs] = (int)((gg / kBStages) & 1);
        if (wpos == kWindow - 1 || i + 2 >= n_u) ++wc;
        continue;
      }
      if (wpos == 0 || j == 0) mbar_wait(smem_u32(&aempty[abar]), ((uint32_t)(wc / kAccBufs) & 1u) ^ 1u);
      mbar_wait(smem_u32(&ready[slot]), sph);
      mbar_wait(smem_u32(&bfull[bs]), (uint32_t)(gg / kBStages) & 1u);
      TCT(4, gg);
      tc_fence_after();
      const uint32_t first = (wpos == 0 || j == 0) ? 1u : 0u;
      const uint64_t bd = bdesc0 + ((uint64_t)(bs * kBStageBytes) >> 4);
      TCT(7, gg);  // issue start (after the waits and the fence)
      if constexpr (kK3) {
        // F_lo rows of the stage (PAIR: each CTA holds r_pad / 2 rows of each)
        const uint64_t bd_lo = bd + ((uint64_t)((PAIR ? p.rp / 2 : p.rp) * 128) >> 4);
        constexpr int A0 = W * kAccBufs, A1 = W * kAccBufs + (kAccBufs > 1 ? 1 : 0);
        const int sidx = slot >> 1;  // this warp's slots are W, W + 2, ...
#ifndef MLB_TC_EXP_NOMMA  // timing experiment: no MMAs (wrong results)
        if (abuf == 0) {
          if (sidx == 0) issue_chunk3<W, A0, PAIR, MIXED>(bd, bd_lo, id_hi, first, id_x);
          else if (sidx == 1) issue_chunk3<(W + 2) % kSlots, A0, PAIR, MIXED>(bd, bd_lo, id_hi, first, id_x);
          else issue_chunk3<(W + 4) % kSlots, A0, PAIR, MIXED>(bd, bd_lo, id_hi, first, id_x);
        } else {
          if (sidx == 0) issue_chunk3<W, A1, PAIR, MIXED>(bd, bd_lo, id_hi, first, id_x);
          else if (sidx == 1) issue_chunk3<(W + 2) % kSlots, A1, PAIR, MIXED>(bd, bd_lo, id_hi, first, id_x);
          else issue_chunk3<(W + 4) % kSlots, A1, PAIR, MIXED>(bd, bd_lo, id_hi, first, id_x);
        }
#else
        (void)sidx, (void)bd_lo;
#endif
      } else {
        if (slot == W)
          issue_chunk<W, W>(bd, id_full, id_hi, first);
        else
          issue_chunk<(W + 2) % kSlots, W>(bd, id_full, id_hi, first);
      }
      if (PAIR) {  // both CTAs' slots and factor halves
        tc_commit_pair(smem_u32(&sdone[slot]));
        tc_commit_pair(smem_u32(&bempty[bs]));
      } else {
        tc_commit(smem_u32(&sdone[slot]));   // staging slot reusable once these MMAs finish
        tc_commit(smem_u32(&bempty[bs]));    // ... and the factor-slice stage
      }
      lastph[slot >> 1] = (int)sph;
      lastb[bs] = (int)((gg / kBStages) & 1);
      TCT(5, gg);
      if (wpos == kWindow - 1 || i + 2 >= n_u) {
        if (PAIR)
          tc_commit_pair(smem_u32(&afull[abar]));
        else
          tc_commit(smem_u32(&afull[abar]));
        ++wc;
      }
      __syncwarp();
    }
    g += n_u;
  }
  // drain: no tcgen05.commit arrival may land after the CTA exits
  for (int k = 0; k < kSlots / 2; ++k)
    if (lastph[k] >= 0) mbar_wait(smem_u32(&sdone[W + 2 * k]), (uint32_t)lastph[k]);
  for (int k = 0; k < kBStages; ++k)
    if (lastb[k] >= 0) mbar_wait(smem_u32(&bempty[k]), (uint32_t)lastb[k]);
}

// PAIR: CTA pairs (clusters of 2 on one TPC) share a 256-row tile: each CTA
// streams and converts its own 128 rows into its own TMEM, loads half of
// each factor slice (r_pad / 2 rows of F_hi and of F_lo), and the leader
// (rank 0) issues cta_group::2 MMAs (M = 256) for both; its commits are
// multicast to both CTAs' barriers, and the peer's converters / epilogue
// arrive on the leader's barriers.  Per SM this halves the factor-slice
// traffic (TMA and MMA reads of shared memory) and the MMA issue work.
template <bool TRANS, bool PAIR, bool MIXED>
__global__ void __launch_bounds__(kThreads, 1)
    k_tc_product(const __grid_constant__ CUtensorMap map_m, const __grid_constant__ CUtensorMap map_b,
                 const Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // carve: [M ring: kMStages x 16 KB][B ring: kBStages x 16 KB][barriers]
  // The rings are separate so an M slice is released as soon as the
  // converters have read it (more HBM bytes in flight), while a factor slice
  // lives until the MMAs reading it complete.
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int b_bytes = 2 * p.rp * 128;      // bytes TMA writes per factor slice
  unsigned char* sm_m = base;
  unsigned char* sm_b = base + kMStages * kMTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm_b + kBStages * kBStageBytes);
  uint64_t* mfull = bars;                  // [kMGroups]  TMA -> converters (a group of slices)
  uint64_t* mempty = mfull + kMGroups;     // [kMGroups]  converters -> TMA
  uint64_t* ready = mempty + kMGroups;     // [kSlots]    converters -> MMA (TMEM slot s written)
  uint64_t* sdone = ready + kSlots;        // [kSlots]    MMA commit -> converters (slot s free)
  uint64_t* bfull = sdone + kSlots;        // [kBStages]  TMA -> MMA (factor slice)
  uint64_t* bempty = bfull + kBStages;     // [kBStages]  MMA commit -> TMA
  uint64_t* afull = bempty + kBStages;     // [2 x kAccBufs] MMA warp w commit -> epilogue
  uint64_t* aempty = afull + 2 * kAccBufs; // [2 x kAccBufs] epilogue -> MMA warp w
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(aempty + 2 * kAccBufs);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kTileRows = PAIR ? 256 : 128;
  static_assert(!PAIR || MLB_TC_BSINGLE, "CTA pairs: single factor-slice producer");
  const uint32_t crank = PAIR ? cluster_rank() : 0u;
  const int row0 = (int)crank * 128;  // this CTA's rows within a tile
  const int u0 = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int ustep = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kMGroups; ++i) {
      mbar_init(smem_u32(&mfull[i]), 1);
      mbar_init(smem_u32(&mempty[i]), 4 * kMGroup);  // 4 converter warps per slice
    }
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(smem_u32(&ready[i]), PAIR ? 8 : 4);  // the 4 converter warps (of both CTAs)
      mbar_init(smem_u32(&sdone[i]), 1);
    }
    for (int i = 0; i < kBStages; ++i) {
      mbar_init(smem_u32(&bfull[i]), 1);
      mbar_init(smem_u32(&bempty[i]), 1);
    }
    for (int i = 0; i < 2 * kAccBufs; ++i) {
      mbar_init(smem_u32(&afull[i]), 1);
      mbar_init(smem_u32(&aempty[i]), PAIR ? 16 : 8);  // the 8 epilogue warps (of both CTAs)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_m)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == kWarpMma0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (PAIR)
    cluster_sync_all();  // both CTAs' barriers initialised before any cross-CTA arrive
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if (tmem != 0) __trap();  // one CTA per SM owning all 512 columns: base is lane 0, column 0

  const int total_units = p.tiles * p.splits;

  if (warp == kWarpM) {
    // ======================= TMA producer: M slices =======================
    if (lane == 0) {
      // Slices go out in groups of kMGroup consecutive chunks on one barrier,
      // back to back: for product 1 the 128-byte row segments of consecutive
      // chunks are adjacent in DRAM, so issuing them together keeps DRAM pages
      // open (+2-3% over single slices).
      int g = 0, npend = 0;
      int pt[kMGroup] = {}, pc[kMGroup] = {};
      const uint64_t pol_m = l2_policy_evict_first();
      auto issue_group = [&]() {
        const int pg = g / kMGroup, ps = pg % kMGroups;
        mbar_wait<MLB_TC_PSLEEP>(smem_u32(&mempty[ps]), ((uint32_t)(pg / kMGroups) & 1u) ^ 1u);
        const uint32_t fm = smem_u32(&mfull[ps]);
        mbar_expect_tx(fm, npend * kMTileBytes);
        for (int k = 0; k < npend; ++k) TCT(0, g + k);
        unsigned char* dst = sm_m + ps * kMGroup * kMTileBytes;
        if (!TRANS && p.wide) {
          // pair (c, c + 1), c even, same tile: each row's 256 contiguous bytes
          // in one request stream (a 2-D box per chunk fetches 128 B per row
          // and DRAM serves that pattern at ~4.6 TB/s; 256 B rows ~7 TB/s --
          // tools/stream_probe.cu)
          tma_load_3d_hint(smem_u32(dst), &map_m, 0, pc[0], pt[0] * kTileRows + row0, fm, pol_m);
        } else {
          for (int k = 0; k < npend; ++k) {
            if (!TRANS)
              tma_load_2d_hint(smem_u32(dst + k * kMTileBytes), &map_m, pc[k] * kChunk, pt[k] * kTileRows + row0, fm,
                               pol_m);
            else
              tma_load_2d_hint(smem_u32(dst + k * kMTileBytes), &map_m, pt[k] * kTileRows + row0, pc[k] * kChunk, fm,
                               pol_m);
          }
        }
        g += kMGroup;
        npend = 0;
      };
      for (int u = u0; u < total_units; u += ustep) {
        const Unit x = unit_of(p, u);
        for (int i = 0; i < x.n; ++i) {
          pt[npend] = x.tile, pc[npend] = unit_chunk(p, x, i);
          if (++npend == kMGroup) issue_group();
        }
      }
      if (npend > 0) issue_group();
    }
  } else if (warp == kWarpB) {
    // ======================= TMA producers: factor slices (lanes 0 / 1: even / odd chunks) =======================
    // Own warp: the B ring (freed only when a chunk's MMAs complete) must not
    // throttle the M stream, and one parity's stall must not block the other.
#if MLB_TC_BSINGLE
    if (lane == 0) {
      // one thread, all chunks in stream order, spin without sleeping
      const uint64_t pol_b = l2_policy_evict_last();
      int g = 0;
      for (int u = u0; u < total_units; u += ustep) {
        const Unit x = unit_of(p, u);
        const int n_u = x.n;
        for (int i = 0; i < n_u; ++i) {
          const int gg = g + i, bs = gg % kBStages;
          mbar_wait<MLB_TC_PSLEEP>(smem_u32(&bempty[bs]), ((uint32_t)(gg / kBStages) & 1u) ^ 1u);
          const uint32_t fb = smem_u32(&bfull[bs]);
          if (PAIR) {
            // this CTA's halves: rows [crank * rp/2, +rp/2) of F_hi and of F_lo,
            // counted on the leader's barrier (which expects both CTAs' bytes)
            const uint32_t fbc = cluster_addr(fb, 0);
            const int hr = p.rp / 2;
            if (crank == 0) mbar_expect_tx(fb, b_bytes);
            const uint32_t dst = smem_u32(sm_b + bs * kBStageBytes);
            tma_load_2d_pair(dst, &map_b, unit_chunk(p, x, i) * kChunk, (int)crank * hr, fbc, pol_b);
            tma_load_2d_pair(dst + hr * 128, &map_b, unit_chunk(p, x, i) * kChunk, p.rp + (int)crank * hr, fbc, pol_b);
          } else {
            mbar_expect_tx(fb, b_bytes);
            tma_load_2d_hint(smem_u32(sm_b + bs * kBStageBytes), &map_b, unit_chunk(p, x, i) * kChunk, 0, fb, pol_b);
          }
          if (kBPrefetch > 0 && i + kBPrefetch < n_u) tma_prefetch_2d(&map_b, unit_chunk(p, x, i + kBPrefetch) * kChunk, 0);
          TCT(6, gg);
        }
        g += n_u;
      }
    }
#else
    const int w = lane;
    if (lane < 2) {
      int g = 0;
      for (int u = u0; u < total_units; u += ustep) {
        const Unit x = unit_of(p, u);
        const int n_u = x.n;
        for (int i = own_first(g, w); i < n_u; i += 2) {
          const int gg = g + i, bs = gg % kBStages;
          mbar_wait<64>(smem_u32(&bempty[bs]), ((uint32_t)(gg / kBStages) & 1u) ^ 1u);
          const uint32_t fb = smem_u32(&bfull[bs]);
          mbar_expect_tx(fb, b_bytes);
          tma_load_2d(smem_u32(sm_b + bs * kBStageBytes), &map_b, unit_chunk(p, x, i) * kChunk, 0, fb);
          if (kBPrefetch > 0 && i + kBPrefetch < n_u) tma_prefetch_2d(&map_b, unit_chunk(p, x, i + kBPrefetch) * kChunk, 0);
          TCT(6, gg);
        }
        g += n_u;
      }
    }
#endif
  } else if (warp == kWarpMma0 || warp == kWarpMma1) {
    // ======================= MMA issuers (one per parity) =======================
    // The whole warp runs the (warp-uniform) loop so every MMA operand stays in
    // the uniform datapath; one elected lane issues each tcgen05 instruction.
    const uint64_t bdesc0 = sdesc_sw128(smem_u32(sm_b));
    const bool issue = !PAIR || crank == 0;  // in a pair only the leader issues
    if (warp == kWarpMma0)
      mma_role<0, PAIR, MIXED>(p, total_units, u0, ustep, issue, bdesc0, ready, sdone, bfull, bempty, afull, aempty);
    else
      mma_role<1, PAIR, MIXED>(p, total_units, u0, ustep, issue, bdesc0, ready, sdone, bfull, bempty, afull, aempty);
  } else if (warp < kWarpEpi0) {
    // ======================= converters: fp32 -> tf32 hi/lo into TMEM =======================
    // kConvGroups groups of 4 warps take alternate chunks (more chunks in
    // flight); within a group warp q owns TMEM lane quarter q (access rule).
    const int grp = (warp - kWarpConv0) >> 2;
    const int q = warp & 3;
    const int row = q * 32 + lane;   // MMA row (= TMEM lane) owned by this thread
    int g = 0;                       // global chunk sequence number
    for (int u = u0; u < total_units; u += ustep) {
      const int n_u = unit_of(p, u).n;
      for (int c = 0; c < n_u; ++c, ++g) {
        if (g % kConvGroups != grp) continue;
        const int pg = g / kMGroup, ps = pg % kMGroups, slot = g % kSlots;
        const uint32_t mph = (uint32_t)(pg / kMGroups) & 1u, sphase = (uint32_t)(g / kSlots) & 1u;
        mbar_wait<MLB_TC_CSLEEP>(smem_u32(&mfull[ps]), mph);
        if (q == 0) TCT(1, g);
        // the thread's 32 values of this chunk (its MMA row / TMEM lane)
        float x[32];
        // shared-window address of the slice (explicit ld.shared: a generic
        // pointer here compiles to slower generic LD.E)
        const uint32_t tile = smem_u32(sm_m) + (uint32_t)((ps * kMGroup + g % kMGroup) * kMTileBytes);
        if (!TRANS && p.wide) {
          // pair buffer [row][half][32] (SWIZZLE_128B per 128-byte line):
          // this chunk's row is line 2 row + h; 16-byte piece jj at
          // jj ^ (line & 7).  Lanes 4..7 of each quarter-warp walk the pieces
          // in a flipped order (jj = j ^ 1), so the 8 lanes of a wavefront hit
          // 8 distinct bank groups.
          const uint32_t pairb = smem_u32(sm_m) + (uint32_t)(ps * kMGroup * kMTileBytes);
          const uint32_t line = 2u * (uint32_t)row + (uint32_t)(g & 1);
          const int flip = (lane >> 2) & 1;
          float y[32];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            lds128(pairb + line * 128 + ((((uint32_t)(j ^ flip)) ^ (line & 7)) << 4), y[4 * j], y[4 * j + 1],
                   y[4 * j + 2], y[4 * j + 3]);
          // y holds piece j ^ flip in slot j: swap adjacent pieces back when flipped
#pragma unroll
          for (int k = 0; k < 32; ++k) x[k] = flip ? y[k ^ 4] : y[k];
        } else if (!TRANS) {
          // row `row` of a 128 x 32 SWIZZLE_128B tile: 16-byte chunk j at j ^ (row & 7)
#pragma unroll
          for (int j = 0; j < 8; ++j)
            lds128(tile + row * 128 + ((j ^ (row & 7)) << 4), x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
        } else {
          // column `row` of a 32 x 128 (k x j) tile, no swizzle
#pragma unroll
          for (int k = 0; k < 32; ++k) x[k] = lds32(tile + (uint32_t)((k * 128 + row) * 4));
        }
        // tf32 split in registers before waiting for the staging slot:
        // hi = rna(x), lo = rna(x - hi); x - hi is exact in fp32 (bit-pattern
        // round-to-nearest-away == cvt.rna.tf32)
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) hi[k] = (__float_as_uint(x[k]) + 0x1000u) & 0xFFFFE000u;
        if (MIXED) {
          // lo half of the slot: bf16 pairs [x - hi (32) | hi (32)], element 2j in the low 16 bits
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const __nv_bfloat162 l2 = __floats2bfloat162_rn(x[2 * j] - __uint_as_float(hi[2 * j]),
                                                            x[2 * j + 1] - __uint_as_float(hi[2 * j + 1]));
            const __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(hi[2 * j]), __uint_as_float(hi[2 * j + 1]));
            lo[j] = *reinterpret_cast<const uint32_t*>(&l2);
            lo[16 + j] = *reinterpret_cast<const uint32_t*>(&h2);
          }
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k)
            lo[k] = (__float_as_uint(x[k] - __uint_as_float(hi[k])) + 0x1000u) & 0xFFFFE000u;
        }
        // The slice was read through the generic proxy and the refill is an
        // async-proxy (TMA) write: order the two before releasing the stage
        // (without this fence a refill can land before lanes' reads retire --
        // seen as ~1e-3 product errors once the M ring runs far ahead).
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&mempty[ps]));  // slice consumed: TMA may refill the group
        mbar_wait<MLB_TC_CSLEEP>(smem_u32(&sdone[slot]), sphase ^ 1);
        if (q == 0) TCT(2, g);
        tc_fence_after();
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + kStgCol0 + slot * 64;
#ifndef MLB_TC_EXP_NOST  // timing experiment: no TMEM stores (wrong results)
#if MLB_TC_ST64
        tmem_st64(ta, hi, lo);
#else
        tmem_st32(ta, hi);
        tmem_st32(ta + 32, lo);
#endif
#endif
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR)
            mbar_arrive_cluster(cluster_addr(smem_u32(&ready[slot]), 0));  // the leader issues the MMAs
          else
            mbar_arrive(smem_u32(&ready[slot]));
        }
        if (q == 0) TCT(3, g);
      }
    }
  } else {
    // ======================= epilogue: fp32 windows -> fp64 =======================
    // 8 warps: lane quarter q (TMEM access rule), column half cb = 0 / 32.
    // Per unit, windows are drained in a fixed order (window k of accumulator
    // 1, then of accumulator 0 -- their completion order), so the fp64 sums
    // are deterministic.
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int cb = ((warp - kWarpEpi0) >> 2) * 32;
    const bool live = cb < p.rp;
    int wcnt[2] = {0, 0};  // windows drained per accumulator warp (all units)
    int g = 0;
    double sum[32];
    for (int u = u0; u < total_units; u += ustep) {
      const Unit x = unit_of(p, u);
      const int tile = x.tile, split = x.split, n_u = x.n;
      const int c1 = own_count(g, n_u, 1);
      const int nw0 = (own_count(g, n_u, 0) + kWindow - 1) / kWindow;
      const int nw1 = c1 > 0 ? (c1 + kWindow / 2 + kWindow - 1) / kWindow : 0;  // first window is half length
#pragma unroll
      for (int k = 0; k < 32; ++k) sum[k] = 0.0;
      for (int k = 0; k < max(nw0, nw1); ++k) {
#pragma unroll
        for (int ww = 0; ww < 2; ++ww) {
          const int w = 1 - ww;  // window k of accumulator 1 completes before window k of accumulator 0
          if (k >= (w ? nw1 : nw0)) continue;
          const int ab = wcnt[w] % kAccBufs, abar = w * kAccBufs + ab;
          mbar_wait<256>(smem_u32(&afull[abar]), (uint32_t)(wcnt[w] / kAccBufs) & 1u);
          tc_fence_after();
          if (live) {
            const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + abar * kAccStride + cb;
#pragma unroll
            for (int h = 0; h < (kK3 ? 2 : 4); ++h) {  // 16 cols each (stacked form: then the F_lo part)
              uint32_t v[16];
              tmem_ld16(ta + (h >> 1) * p.rp + (h & 1) * 16, v);
              tmem_wait_ld();
#pragma unroll
              for (int kk = 0; kk < 16; ++kk) sum[(h & 1) * 16 + kk] += (double)__uint_as_float(v[kk]);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (PAIR)
              mbar_arrive_cluster(cluster_addr(smem_u32(&aempty[abar]), 0));
            else
              mbar_arrive(smem_u32(&aempty[abar]));
          }
          ++wcnt[w];
        }
      }
      g += n_u;
      const int gi = tile * kTileRows + row0 + row;
      if (live && gi < p.rows) {
        if (!TRANS) {
          double* out = p.part + (size_t)split * p.rows * p.r + (size_t)gi * p.r + cb;
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (cb + k < p.r) out[k] = sum[k];
        } else {
          double* out = p.part + (size_t)split * p.r * p.rows + (size_t)cb * p.rows + gi;
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (cb + k < p.r) out[(size_t)k * p.rows] = sum[k];
        }
      }
    }
  }

  tc_fence_before();
  if (PAIR)
    cluster_sync_all();  // the peer's TMEM is read by the leader's MMAs until the end
  else
    __syncthreads();
  if (warp == kWarpMma0) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// F (rows x ld, row-major, rows <= r) -> S (2 rp x K): S[k] = rna(F[k]),
// S[rp + k] = rna(F[k] - S[k]); padding rows zero.  trans: F is K x r
// (V, row-major) and row k of S is column k of F.
// S rows have pitch Kp = K rounded up to whole 32-wide chunks (zero tail), so
// the last chunk's bf16 [F_hi | F_lo] block stays inside its row.
template <bool MIXED>
__global__ void k_split_factor(const float* __restrict__ F, float* __restrict__ S, int r, int rp, size_t K,
                               size_t Kp, int trans) {
  const size_t total = (size_t)rp * Kp;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const size_t k = e / Kp, j = e % Kp;
    float hi = 0.f, lo = 0.f;
    if ((int)k < r && j < K) {
      const float x = trans ? F[j * r + k] : F[k * K + j];
      const uint32_t h = tf32_rna(x);
      hi = __uint_as_float(h);
      lo = __uint_as_float(tf32_rna(x - hi));
    }
    S[k * Kp + j] = hi;
    if (MIXED) {
      // row k of the lo region as bf16 [F_hi (32) | F_lo (32)] per 32-wide chunk:
      // the same 128 bytes per row that fp32 columns [32c, 32c + 32) occupy
      __nv_bfloat16* Sx = reinterpret_cast<__nv_bfloat16*>(S + ((size_t)rp + k) * Kp);
      const size_t c = j / 32, t = j % 32;
      Sx[64 * c + t] = __float2bfloat16_rn(hi);
      Sx[64 * c + 32 + t] = __float2bfloat16_rn(lo);
    } else {
      S[((size_t)rp + k) * Kp + j] = lo;
    }
  }
}

// out[0] = sum of part[0..count) in a fixed order (one block)
__global__ void k_sum_parts(const double* __restrict__ part, int count, double* __restrict__ out) {
  __shared__ double ws[32];
  double s = 0.0;
  for (int e = threadIdx.x; e < count; e += blockDim.x) s += part[e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    out[0] = t;
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


// ----------------------------------------------------------------------------
// Direct residual ||M - V W||_F^2 on the tensor cores (frobenius_error,
// proj/src/matrix.cpp:37-42; the trace sample of run_solver_phase).
// Per tile (128 columns J of M) x (64 rows I of M):
//   P^T[j][i] = sum_k W[k][j] V[i][k]   (3xTF32: W^T_hi V_hi + W^T_hi V_lo + W^T_lo V_hi)
// in TMEM (M_mma = 128 columns j, N = 64 rows i, K = r_pad), then the epilogue
// sums (M[i][j] - P[i][j])^2 in fp32 per 32 and fp64 across.  Operands come
// pre-split (k_split_rows), K-major, row width 2 * rpa (hi | lo), rpa = r_pad
// rounded up to whole 128-byte swizzle atoms.
//   A operand (W^T tile, 128 j x 2 rpa): loaded once per J tile by the
//     epilogue warps, global -> registers -> a TMEM buffer (double-buffered
//     across J tiles): TS form, so the MMAs read only V from shared memory
//     (SS at N = 64 is shared-memory bound, 48 vs 32 cycles per MMA:
//     tools/mma_probe2.cu).
//   V slices (64 i x 2 rpa, L2) and M tiles (TMA, 4 boxes of 64 rows x 128 B,
//     HBM, evict-first) stream through separate rings, released by the MMA
//     commit and by the epilogue respectively.
//   Two MMA warps take alternate I tiles (own V stage and accumulator), so one
//     warp's barrier waits and commits overlap the other's MMAs (with a single
//     MMA warp and no memory traffic at all the kernel ran at ~50 % of the
//     tensor rate).
// Config-4 slice (n = 65536): SS form 4.9 ms -> TS + separate rings 3.8 ms.
// (Per-lane global loads of M ran at 0.9 TB/s; the TMA-staged tile reads it
// at the HBM rate.)
// ----------------------------------------------------------------------------
// warps: 0 TMA (V), 1 MMA (1 allocates TMEM), 2 .. 2 + kREpi - 1 epilogue,
// then TMA (M), then (optional) a second MMA warp taking the odd I tiles
#ifndef MLB_TC_RES_EPI
#define MLB_TC_RES_EPI 8
#endif
#ifndef MLB_TC_RES_MMA2
#define MLB_TC_RES_MMA2 0
#endif
constexpr int kREpi = MLB_TC_RES_EPI;        // epilogue warps: 4 lane quarters x kREpi / 4 row groups
constexpr int kRRows = 64 / (kREpi / 4);     // rows i per epilogue warp and tile
constexpr int kRMmaWarps = MLB_TC_RES_MMA2 ? 2 : 1;
constexpr int kRWarpM = 2 + kREpi, kRWarpMma1 = 3 + kREpi;
constexpr int kRThreads = (3 + kREpi + (kRMmaWarps - 1)) * 32;
static_assert(kREpi == 8 || kREpi == 16, "epilogue: 2 or 4 row groups per lane quarter");
constexpr int kResAcol0 = 256;  // TMEM: accumulators at columns 0 / 64, A buffers at 256 / 384
#ifndef MLB_TC_RES_VS
#define MLB_TC_RES_VS 2
#endif
constexpr int kRVS = MLB_TC_RES_VS;  // V stages (tile t uses stage t % kRVS)
static_assert(kRVS % 2 == 0, "V ring: whole pairs (accumulator / MMA-warp parity)");
#ifndef MLB_TC_RES_MS
#define MLB_TC_RES_MS 4
#endif
constexpr int kRMS = MLB_TC_RES_MS;  // M stages
constexpr int kRAcc = 2;             // accumulators (one per MMA warp)
constexpr int kResTmemCols = 512;
constexpr int kRAtomBytes = 128 * 128;  // one 128-row x 32-fp32 SW128 box
constexpr int kRMBytes = 64 * 128 * 4;   // M tile: 64 rows i x 128 columns j

// X -> S (rows x 2 rpa): [rna(x) | rna(x - rna(x))], zero padded.  trans: X is
// r x rows (W, row-major) and row j of S comes from column j of X.
// MIXED (the residual's bf16 cross terms): the lo half of each S row holds
// bf16 [hi | lo] (V, the B operand) or [lo | hi] (W^T, the A operand) packed
// in the same rpa 32-bit words, so [W_lo | W_hi] . [V_hi ; V_lo] is one K = 2
// rpa bf16 product.
// (the bf16 halves are r_pad long -- the K extent the MMAs cover -- so the
// pair is [x (rp) | y (rp)] within the 2 rpa bf16 slots; k >= rp is padding)
__device__ __forceinline__ void put_split(float* row, int rpa, int rp, int k, float x, bool mixed, bool lo_first) {
  const float hi = __uint_as_float(tf32_rna(x));
  row[k] = hi;
  if (mixed) {
    __nv_bfloat16* bx = reinterpret_cast<__nv_bfloat16*>(row + rpa);
    const __nv_bfloat16 bh = __float2bfloat16_rn(hi), bl = __float2bfloat16_rn(x - hi);
    if (k < rp) {
      bx[k] = lo_first ? bl : bh;
      bx[rp + k] = lo_first ? bh : bl;
    } else if (rp + k < 2 * rpa) {
      bx[rp + k] = __float2bfloat16_rn(0.f);  // zero the tail beyond 2 rp
    }
  } else {
    row[rpa + k] = __uint_as_float(tf32_rna(x - hi));
  }
}

__global__ void k_split_rows(const float* __restrict__ X, float* __restrict__ S, int r, int rpa, int rp,
                             size_t rows, int trans, int mixed) {
  const size_t total = (size_t)rows * rpa;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    size_t j, k;
    if (trans) k = e / rows, j = e % rows;  // coalesced reads of W rows
    else j = e / rpa, k = e % rpa;
    const float x = (int)k < r ? (trans ? X[k * rows + j] : X[j * r + k]) : 0.f;
    put_split(S + j * 2 * rpa, rpa, rp, (int)k, x, mixed != 0, trans != 0);
  }
}

// The transposed case (W, r x rows -> S rows x 2 rpa) through a shared-memory
// tile: 64 columns of W read row by row (coalesced), written as 64 contiguous
// S rows (coalesced); the element-wise version scattered 4-byte writes at a
// 2 rpa stride (0.35 ms per error sample at config 4).
__global__ void __launch_bounds__(256) k_split_rows_t(const float* __restrict__ X, float* __restrict__ S, int r,
                                                      int rpa, int rp, size_t rows, int mixed) {
  __shared__ float tile[64][65];  // [k][j], k < rpa <= 64
  const size_t j0 = (size_t)blockIdx.x * 64;
  const int t = threadIdx.x, tj = t & 63, tk = t >> 6;  // 4 k-rows per pass
  for (int k = tk; k < rpa; k += 4) {
    const size_t j = j0 + tj;
    tile[k][tj] = (k < r && j < rows) ? X[(size_t)k * rows + j] : 0.f;
  }
  __syncthreads();
  // each warp writes whole S rows: lanes over k (hi then lo)
  const int warp = t >> 5, lane = t & 31;
  for (int jj = warp; jj < 64; jj += 8) {
    const size_t j = j0 + jj;
    if (j >= rows) break;
    float* row = S + j * 2 * (size_t)rpa;
    for (int k = lane; k < rpa; k += 32) put_split(row, rpa, rp, k, tile[k][jj], mixed != 0, true);
  }
}

struct RParams {
  const float* M;
  const float* wsplit;     // W^T split rows: n x 2 rpa, [hi | lo]
  int m, n, r, rp, atoms;  // atoms = rpa / 32
  int tj, ti;              // tile counts along n (J) and m (I)
  double* part;            // [gridDim.x] per-CTA sums
};

// The MMAs of one tile: K = KS x 8 (KS = 0: runtime p.rp / 8), A = TMEM
// columns [ta, ta + rpa) (hi) and [ta + rpa, ...) (lo), B = the V stage.
__device__ __forceinline__ void mma_ts_bf16(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
template <int KS, bool MIXED>
__device__ __forceinline__ void res_tile_mmas(uint32_t d, uint32_t ta, int rpa, uint64_t dbs, uint64_t lo_b,
                                              uint32_t id, uint32_t idx, int ks_rt) {
  const int ksteps = KS > 0 ? KS : ks_rt;
#pragma unroll
  for (int kk = 0; kk < (KS > 0 ? KS : 16); ++kk) {
    if (KS == 0 && kk >= ksteps) break;
    const uint64_t ob = (uint64_t)(((kk >> 2) * (kRAtomBytes / 2) + (kk & 3) * 32) >> 4);
    mma_ts(d, ta + kk * 8, dbs + ob, id, kk > 0 ? 1u : 0u);  // W_hi V_hi
    if (MIXED) {
      // K = 16 bf16 of [W_lo | W_hi] . [V_hi ; V_lo] (the same 32-byte step)
      mma_ts_bf16(d, ta + rpa + kk * 8, dbs + lo_b + ob, idx, 1u);
    } else {
      mma_ts(d, ta + kk * 8, dbs + lo_b + ob, id, 1u);  // W_hi V_lo
      mma_ts(d, ta + rpa + kk * 8, dbs + ob, id, 1u);   // W_lo V_hi
    }
  }
}

template <bool MIXED>
__global__ void __launch_bounds__(kRThreads, 1)
    k_tc_residual(const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_m,
                  const RParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int opb = p.atoms * kRAtomBytes;  // V slice: 64 i x 2 rpa
  unsigned char* sm_v = base;                // kRVS V stages
  unsigned char* sm_m = sm_v + kRVS * opb;   // kRMS M stages (64 i x 128 j, four 32-column boxes)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm_m + kRMS * kRMBytes);
  uint64_t* vfull = bars;              // [kRVS] V slice landed
  uint64_t* vempty = vfull + kRVS;     // [kRVS] MMAs reading it done (commit)
  uint64_t* mfull = vempty + kRVS;     // [kRMS] M tile landed
  uint64_t* mempty = mfull + kRMS;     // [kRMS] epilogue done with it (8 warps)
  uint64_t* cfull = mempty + kRMS;     // [kRAcc] accumulator ready for the epilogue
  uint64_t* cempty = cfull + kRAcc;    // [kRAcc] epilogue done with the accumulator
  uint64_t* aready = cempty + kRAcc;   // [2] W^T tile stored in TMEM A buffer b (8 epilogue warps)
  uint64_t* tfree = aready + 2;        // [2] both MMA warps done with TMEM A buffer b
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tfree + 2);
  __shared__ double red[kREpi];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kRVS; ++i) {
      mbar_init(smem_u32(&vfull[i]), 1);
      mbar_init(smem_u32(&vempty[i]), 1);
    }
    for (int i = 0; i < kRMS; ++i) {
      mbar_init(smem_u32(&mfull[i]), 1);
      mbar_init(smem_u32(&mempty[i]), kREpi);
    }
    for (int i = 0; i < kRAcc; ++i) {
      mbar_init(smem_u32(&cfull[i]), 1);
      mbar_init(smem_u32(&cempty[i]), kREpi);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&aready[i]), kREpi);
      mbar_init(smem_u32(&tfree[i]), kRMmaWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(kResTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  double s64 = 0.0;

  if (warp == 0) {
    // ---- TMA producer: V slices ----
    if (lane == 0) {
      int tc_ = 0;
      for (int jt = blockIdx.x; jt < p.tj; jt += gridDim.x)
        for (int it = 0; it < p.ti; ++it, ++tc_) {
          const int st = tc_ % kRVS;
          unsigned char* sb = sm_v + st * opb;
          mbar_wait(smem_u32(&vempty[st]), ((uint32_t)(tc_ / kRVS) & 1u) ^ 1u);
#ifdef MLB_TC_RES_EXP_NOV
          if (tc_ >= kRVS) {  // timing experiment only: reuse the first V slices (wrong results)
            mbar_arrive(smem_u32(&vfull[st]));
            continue;
          }
#endif
          mbar_expect_tx(smem_u32(&vfull[st]), (uint32_t)opb);
          for (int h = 0; h < 2; ++h)
            for (int a = 0; a < p.atoms; ++a)
              tma_load_2d(smem_u32(sb + (h * p.atoms + a) * (kRAtomBytes / 2)), &map_v, h * p.atoms * 32 + a * 32,
                          it * 64, smem_u32(&vfull[st]));
        }
    }
  } else if (warp == kRWarpM) {
    // ---- TMA producer: M tiles ----
    if (lane == 0) {
      const uint64_t pol_m = l2_policy_evict_first();  // M is read once; keep the V / W slices in L2
      int tc_ = 0;
      for (int jt = blockIdx.x; jt < p.tj; jt += gridDim.x)
        for (int it = 0; it < p.ti; ++it, ++tc_) {
          const int st = tc_ % kRMS;
          unsigned char* sb = sm_m + st * kRMBytes;
          mbar_wait(smem_u32(&mempty[st]), ((uint32_t)(tc_ / kRMS) & 1u) ^ 1u);
#ifdef MLB_TC_RES_EXP_NOM
          if (tc_ >= kRMS) {  // timing experiment only: reuse the first M tiles (wrong results)
            mbar_arrive(smem_u32(&mfull[st]));
            continue;
          }
#endif
          mbar_expect_tx(smem_u32(&mfull[st]), (uint32_t)kRMBytes);
          for (int b = 0; b < 4; ++b)  // M rows i of the tile, 32 columns j per box
            tma_load_2d_hint(smem_u32(sb + b * (kRMBytes / 4)), &map_m, jt * 128 + b * 32, it * 64,
                             smem_u32(&mfull[st]), pol_m);
        }
    }
  } else if (warp == 1 || (kRMmaWarps == 2 && warp == kRWarpMma1)) {
    // ---- MMA issuer(s): with two, warp w takes the I tiles with tc_ % 2 == w ----
    const int w = warp == 1 ? 0 : 1;
    const uint32_t id = idesc_tf32(64);
    const uint64_t ds = sdesc_sw128(smem_u32(sm_v));
    const uint64_t lo_b = (uint64_t)((p.atoms * kRAtomBytes / 2) >> 4);
    const int rpa = p.atoms * 32, ks_rt = p.rp / 8;
    int jc = 0, tc_ = 0, lastv[kRVS];
    for (int k = 0; k < kRVS; ++k) lastv[k] = -1;
    int lastt[2] = {-1, -1};
    for (int jt = blockIdx.x; jt < p.tj; jt += gridDim.x, ++jc) {
      const uint32_t ab = (uint32_t)jc & 1u;
      const uint32_t ta = kResAcol0 + ab * 128;  // TMEM A buffer: W^T hi in [ta, ta + rpa), lo after
      mbar_wait(smem_u32(&aready[ab]), (uint32_t)(jc >> 1) & 1u);
      for (int it = 0; it < p.ti; ++it, ++tc_) {
        if (kRMmaWarps == 2 && (tc_ & 1) != w) continue;
        const int sa = tc_ & 1, sv = tc_ % kRVS;        // accumulator = tile parity; V stage
        const uint32_t ph = (uint32_t)(tc_ >> 1) & 1u;  // tile tc_ is use tc_ / 2 of accumulator sa
        const uint32_t vph = (uint32_t)(tc_ / kRVS) & 1u;
        mbar_wait(smem_u32(&cempty[sa]), ph ^ 1u);
        mbar_wait(smem_u32(&vfull[sv]), vph);
        tc_fence_after();
        const uint32_t d = (uint32_t)(sa * 64);
        const uint64_t dbs = ds + (uint64_t)((sv * opb) >> 4);
        if (ks_rt == 8)
          res_tile_mmas<8, MIXED>(d, ta, rpa, dbs, lo_b, id, idesc_bf16(64), ks_rt);
        else
          res_tile_mmas<0, MIXED>(d, ta, rpa, dbs, lo_b, id, idesc_bf16(64), ks_rt);
        tc_commit(smem_u32(&vempty[sv]));  // V slice free (the M tile is released by the epilogue)
        tc_commit(smem_u32(&cfull[sa]));
        lastv[sv] = (int)vph;
        __syncwarp();
      }
      tc_commit(smem_u32(&tfree[ab]));  // this warp is done with TMEM A buffer ab (count 2)
      lastt[ab] = (jc >> 1) & 1;
      __syncwarp();
    }
    // no commit arrival may land after exit
    for (int k = 0; k < kRVS; ++k)
      if (lastv[k] >= 0) mbar_wait(smem_u32(&vempty[k]), (uint32_t)lastv[k]);
    for (int b = 0; b < 2; ++b)
      if (lastt[b] >= 0) mbar_wait(smem_u32(&tfree[b]), (uint32_t)lastt[b]);
  } else {
    // ---- epilogue: lane quarter q (TMEM lane = column j of M), row group h (kRRows rows i of the tile) ----
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int rpa = p.atoms * 32;
    int tc_ = 0, jc = 0;
    for (int jt = blockIdx.x; jt < p.tj; jt += gridDim.x, ++jc) {
      const int jl = q * 32 + lane, j = jt * 128 + jl;
      const int b = jl >> 5, jb = jl & 31;  // M box and column within it
      {
        // W^T row jl of this J tile -> TMEM A buffer (lane jl), straight from
        // the (L2-resident) split buffer: the row's 2 x atoms 32-column pieces
        // (hi atoms, then lo atoms) are shared out over the kREpi / 4 warps of
        // the lane quarter
        const uint32_t ab = (uint32_t)jc & 1u;
        const float4* src = reinterpret_cast<const float4*>(p.wsplit + (size_t)j * 2 * rpa);
        bool waited = jc < 2;
        for (int pc = h; pc < 2 * p.atoms; pc += kREpi / 4) {
          uint4 wv[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 x = j < p.n ? __ldg(src + pc * 8 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
            wv[c] = make_uint4(__float_as_uint(x.x), __float_as_uint(x.y), __float_as_uint(x.z), __float_as_uint(x.w));
          }
          if (!waited) mbar_wait<64>(smem_u32(&tfree[ab]), (uint32_t)((jc >> 1) - 1) & 1u), waited = true;
          tc_fence_after();
          tmem_st32(tmem + ((uint32_t)(q * 32) << 16) + kResAcol0 + ab * 128 + (uint32_t)(pc * 32),
                    reinterpret_cast<const uint32_t(&)[32]>(wv));
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&aready[ab]));
      }
      for (int it = 0; it < p.ti; ++it, ++tc_) {
        const int acc = tc_ & 1, st = tc_ % kRMS;
        const uint32_t ph = (uint32_t)(tc_ >> 1) & 1u;
        mbar_wait<128>(smem_u32(&cfull[acc]), ph);
        tc_fence_after();
        uint32_t v[32];
        if (kRRows == 32)
          tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * 64 + h * 32, v);
        else
          tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc * 64 + h * kRRows,
                    reinterpret_cast<uint32_t(&)[16]>(v));
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&cempty[acc]));
        // M[i][j] from the staged tile (SW128 rows of 32 fp32: a warp reads one
        // 128-byte row per load, conflict-free)
        mbar_wait<64>(smem_u32(&mfull[st]), (uint32_t)(tc_ / kRMS) & 1u);
        const uint32_t mt = smem_u32(sm_m + st * kRMBytes + b * (kRMBytes / 4));
        const int i0 = it * 64 + h * kRRows;
        float s32 = 0.f;  // one fp32 chain (four independent chains measured 3 % slower)
#pragma unroll
        for (int ii = 0; ii < kRRows; ++ii) {
          const int il = h * kRRows + ii;
          const float mval = lds32(mt + il * 128 + ((((jb >> 2) ^ (il & 7)) << 4) | ((jb & 3) << 2)));
          const float dlt = mval - __uint_as_float(v[ii]);
          s32 = (j < p.n && i0 + ii < p.m) ? fmaf(dlt, dlt, s32) : s32;
        }
        s64 += (double)s32;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the TMA refill
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&mempty[st]));  // M tile read
      }
    }
  }
  // per-CTA sum (fixed order: deterministic)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s64 += __shfl_xor_sync(0xffffffffu, s64, o);
  if (warp >= 2 && warp < 2 + kREpi && lane == 0) red[warp - 2] = s64;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kREpi; ++w) t += red[w];
    p.part[blockIdx.x] = t;
  }
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kResTmemCols) : "memory");
  }
}

}  // namespace tc

// ============================================================================
// host side
// ============================================================================
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    TC_CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D fp32 tensor map: inner extent `inner`, outer extent `outer`, row stride
// inner*4 bytes, box (bi x bo), optional 128-byte swizzle.
CUtensorMap make_map(const void* ptr, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo, bool swz) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 4};
  cuuint32_t box[2] = {bi, bo};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

// 3-D view of a row-major fp32 matrix (n % 64 == 0): (32 columns, n / 32
// column blocks, m rows), box (32, 2, 128): one 128-row x 256-byte slab, laid
// out [row][block][32] with the 128-byte swizzle.
CUtensorMap make_map3_rows(const void* ptr, uint64_t n, uint64_t m) {
  CUtensorMap map;
  cuuint64_t dims[3] = {32, n / 32, m};
  cuuint64_t strides[2] = {128, n * 4};
  cuuint32_t box[3] = {32, 2, 128};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (3-D) failed: " + std::to_string((int)r));
  return map;
}

size_t cdiv(size_t a, size_t b) { return (a + b - 1) / b; }

class TcGemmImpl final : public TcGemm {
 public:
  explicit TcGemmImpl(bool forced) : forced_(forced) {
    int dev = 0;
    TC_CK(cudaGetDevice(&dev));
    TC_CK(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev));
  }
  ~TcGemmImpl() override {
    if (split_) cudaFree(split_);
    if (part_) cudaFree(part_);
    if (rv_) cudaFree(rv_);
    if (rw_) cudaFree(rw_);
  }
  bool active() const override { return true; }
  bool supports(size_t m, size_t n, size_t r) const override {
    return r >= 1 && r <= 64 && m % 4 == 0 && n % 4 == 0 && m >= 128 && n >= 128 && m < (1u << 31) &&
           n < (1u << 31);
  }
  bool wants(size_t m, size_t n, size_t r) const override {
    if (!supports(m, n, r)) return false;
    return forced_ || m * n >= ((size_t)1 << 24);
  }

  void mwt(const float* M, const float* W, size_t m, size_t n, size_t r, double* A, cudaStream_t s,
           long* launches) override {
    run<false>(M, W, m, n, r, A, s, launches);
  }
  void vtm(const float* V, const float* M, size_t m, size_t n, size_t r, double* C, cudaStream_t s,
           long* launches) override {
    run<true>(M, V, m, n, r, C, s, launches);
  }

  void sqerr(const float* M, const float* V, const float* W, size_t m, size_t n, size_t r, double* out,
             cudaStream_t s, long* launches) override {
    if (!supports(m, n, r)) throw std::invalid_argument("tcgen05 residual: unsupported shape");
    const int rp = (int)cdiv(r, 16) * 16;
    const int rpa = (int)cdiv(rp, 32) * 32;
    ensure(&rv_, &rv_bytes_, (size_t)m * 2 * rpa * 4);
    ensure(&rw_, &rw_bytes_, (size_t)n * 2 * rpa * 4);
    {
      const unsigned gv = (unsigned)std::min<size_t>(cdiv((size_t)m * rpa, 256), 16384);
      tc::k_split_rows<<<gv, 256, 0, s>>>(V, static_cast<float*>(rv_), (int)r, rpa, rp, m, 0, mixed_ ? 1 : 0);
      tc::k_split_rows_t<<<(unsigned)cdiv(n, 64), 256, 0, s>>>(W, static_cast<float*>(rw_), (int)r, rpa, rp, n,
                                                               mixed_ ? 1 : 0);
      TC_CK(cudaGetLastError());
      *launches += 2;
    }
    tc::RParams p{};
    p.M = M;
    p.wsplit = static_cast<const float*>(rw_);
    p.m = (int)m;
    p.n = (int)n;
    p.r = (int)r;
    p.rp = rp;
    p.atoms = rpa / 32;
    p.tj = (int)cdiv(n, 128);
    p.ti = (int)cdiv(m, 64);
    const int grid = std::min(p.tj, sms_);
    ensure(&part_, &part_bytes_, (size_t)grid * 8);
    p.part = static_cast<double*>(part_);
    const CUtensorMap mv = make_map(rv_, (uint64_t)2 * rpa, m, 32, 64, true);
    const CUtensorMap mm = make_map(M, n, m, 32, 64, true);
    // V stages (64 rows x 2 rpa) + M stages + barriers; the launch is one CTA
    // per SM at every rank (512 TMEM columns)
    const size_t smem = 1024 + (size_t)tc::kRVS * p.atoms * tc::kRAtomBytes + tc::kRMS * tc::kRMBytes + 256;
    if (!resid_attr_) {
      const size_t smax = 1024 + (size_t)tc::kRVS * 2 * tc::kRAtomBytes + tc::kRMS * tc::kRMBytes + 256;
      TC_CK(cudaFuncSetAttribute(tc::k_tc_residual<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax));
      TC_CK(cudaFuncSetAttribute(tc::k_tc_residual<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax));
      resid_attr_ = true;
    }
    if (mixed_)
      tc::k_tc_residual<true><<<grid, tc::kRThreads, smem, s>>>(mv, mm, p);
    else
      tc::k_tc_residual<false><<<grid, tc::kRThreads, smem, s>>>(mv, mm, p);
    TC_CK(cudaGetLastError());
    tc::k_sum_parts<<<1, 256, 0, s>>>(static_cast<const double*>(part_), grid, out);
    TC_CK(cudaGetLastError());
    *launches += 2;
  }

 private:
  template <bool TRANS>
  void run(const float* M, const float* F, size_t m, size_t n, size_t r, double* out, cudaStream_t s,
           long* launches) {
    if (!supports(m, n, r)) throw std::invalid_argument("tcgen05 path: unsupported shape");
    const int rp = (int)cdiv(r, 16) * 16;
    const size_t K = TRANS ? m : n;        // contraction
    const size_t rows = TRANS ? n : m;     // MMA-M extent
    // split factor F -> [F_hi ; F_lo] (2 rp x K)
    const size_t Kp = cdiv(K, tc::kChunk) * tc::kChunk;  // split row pitch: whole chunks
    ensure(&split_, &split_bytes_, (size_t)2 * rp * Kp * 4);
    const bool mixed = mixed_;
    {
      const size_t tot = (size_t)rp * K;
      const unsigned g = (unsigned)std::min<size_t>(cdiv(tot, 256), 16384);
      if (mixed)
        tc::k_split_factor<true><<<g, 256, 0, s>>>(F, static_cast<float*>(split_), (int)r, rp, K, Kp, TRANS ? 1 : 0);
      else
        tc::k_split_factor<false><<<g, 256, 0, s>>>(F, static_cast<float*>(split_), (int)r, rp, K, Kp, TRANS ? 1 : 0);
      TC_CK(cudaGetLastError());
      ++*launches;
    }
    // CTA pairs (cta_group::2, 256-row tiles): r_pad in {32, 64} (N split in
    // halves of >= 16 rows), an even SM count, enough tiles to fill the pairs
    const bool pair = tc::kK3 && pair_ && (rp == 32 || rp == 64) && sms_ >= 2 && cdiv(rows, 256) >= 8;
    const int slots = pair ? sms_ / 2 : sms_;  // persistent schedulers: pairs or CTAs
    tc::Params p{};
    p.rows = (int)rows;
    p.kdim = (int)K;
    p.r = (int)r;
    p.rp = rp;
    p.tiles = (int)cdiv(rows, pair ? 256 : 128);
    p.nchunks = (int)cdiv(K, tc::kChunk);
    p.wide = (!TRANS && tc::kMGroup == 2 && n % 64 == 0) ? 1 : 0;
    if (const char* e = getenv("MLB_TC_WIDE")) p.wide = p.wide && atoi(e);  // debug override
    // unit order (see unit_of): split-major blocked.  The interleaved (1) and
    // tile-major (2) orders read M in DRAM-friendlier patterns
    // (tools/stream_probe.cu) but lose the cross-CTA L2 sharing of factor
    // slices and measured slower in the kernel; they stay opt-in.
    p.interleave = 0;
    p.rotate = 0;  // measured within noise (+-2 %) at config 4; opt-in
    if (const char* e = getenv("MLB_TC_INTERLEAVE")) p.interleave = atoi(e);  // debug override
    if (const char* e = getenv("MLB_TC_ROTATE")) p.rotate = atoi(e);          // debug override
    // split-K: units (tile, K range) are dealt round-robin to the persistent
    // CTAs, so the kernel lasts ceil(units / SMs) units.  Pick the split factor
    // that maximises the balanced fraction units / (ceil(units / SMs) * SMs),
    // charging each extra split its fp64 partial-output traffic (write + reduce
    // read, 16 B per output element) against the M bytes streamed.
    int splits = 1;
    {
      double best = -1.0;
      const int smax = std::max(1, std::min(p.nchunks / 8, 64));
      for (int sp = p.interleave == 1 ? std::min(4, smax) : 1; sp <= smax; ++sp) {
        int cps = (int)cdiv(p.nchunks, sp);
        if (p.wide) cps += cps & 1;  // whole chunk pairs per unit
        const int spr = (int)cdiv(p.nchunks, cps);
        const double units = (double)p.tiles * spr;
        const double rounds = std::ceil(units / slots);
        const double balance = units / (rounds * slots);
        const double extra = spr > 1 ? (double)spr * rows * r * 16.0 / ((double)rows * K * 4.0) : 0.0;
        const double score = balance / (1.0 + extra);
        if (score > best + 1e-9) best = score, splits = sp;
      }
    }
    if (const char* e = getenv("MLB_TC_SPLITS")) splits = std::max(1, atoi(e));  // debug override
    splits = std::min(splits, p.nchunks);
    p.chunks_per_split = (int)cdiv(p.nchunks, splits);
    if (p.wide) {
      p.chunks_per_split += p.chunks_per_split & 1;
      if (p.interleave == 1) p.interleave = 0;  // pairs must stay (c even, c + 1)
      p.rotate = 0;
    }
    p.splits = p.interleave == 1 ? splits : (int)cdiv(p.nchunks, p.chunks_per_split);
    const size_t out_count = rows * r;
    double* dst = out;
    if (p.splits > 1) {
      ensure(&part_, &part_bytes_, (size_t)p.splits * out_count * 8);
      dst = static_cast<double*>(part_);
    }
    p.part = dst;
    const CUtensorMap mm = TRANS    ? make_map(M, n, m, 128, tc::kChunk, false)
                           : p.wide ? make_map3_rows(M, n, m)
                                    : make_map(M, n, m, tc::kChunk, 128, true);
    // factor slices: the whole [F_hi; F_lo] (2 rp rows) per chunk, or per CTA
    // of a pair its rp / 2 rows of each half (two boxes)
    const CUtensorMap mb = make_map(split_, Kp, 2 * rp, tc::kChunk, pair ? rp / 2 : 2 * rp, true);
    const size_t smem = 1024 + tc::kMStages * tc::kMTileBytes + tc::kBStages * tc::kBStageBytes + 512;
    auto kern = pair ? (mixed ? tc::k_tc_product<TRANS, true, true> : tc::k_tc_product<TRANS, true, false>)
                : mixed ? tc::k_tc_product<TRANS, false, true> : tc::k_tc_product<TRANS, false, false>;
    const int ak = (TRANS ? 1 : 0) + (pair ? 2 : 0) + (mixed ? 4 : 0);
    if (!attr_set_[ak]) {
      TC_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr_set_[ak] = true;
    }
    const int units = p.tiles * p.splits;
    int grid = std::min(units, slots);
    if (const char* e = getenv("MLB_TC_GRID")) grid = std::max(1, std::min(grid, atoi(e)));  // debug override
    if (pair) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2 * grid);
      cfg.blockDim = dim3(tc::kThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2, attr[0].val.clusterDim.y = 1, attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      TC_CK(cudaLaunchKernelEx(&cfg, kern, mm, mb, p));
    } else {
      kern<<<grid, tc::kThreads, smem, s>>>(mm, mb, p);
    }
    TC_CK(cudaGetLastError());
#if MLB_TC_TRACE
    if (const char* path = getenv("MLB_TC_TRACE_OUT")) {
      static long long h[8][tc::kTraceChunks];
      TC_CK(cudaStreamSynchronize(s));
      TC_CK(cudaMemcpyFromSymbol(h, tc::g_tctrace, sizeof(h)));
      std::string f = std::string(path) + (TRANS ? ".C" : ".A");
      if (FILE* fp = fopen(f.c_str(), "wb")) {
        fwrite(h, sizeof(h), 1, fp);
        fclose(fp);
      }
    }
#endif

    ++*launches;
    if (p.splits > 1) {
      const unsigned g = (unsigned)std::min<size_t>(cdiv(out_count, 256), 4096);
      tc::k_split_reduce<<<g, 256, 0, s>>>(static_cast<const double*>(part_), out_count, p.splits, out);
      TC_CK(cudaGetLastError());
      ++*launches;
    }
  }

  static void ensure(void** p, size_t* have, size_t need) {
    if (need <= *have) return;
    g_dev_epoch.fetch_add(1);  // invalidates captured step graphs holding the old pointer
    if (*p) TC_CK(cudaFree(*p));
    *p = nullptr;
    TC_CK(cudaMalloc(p, need));
    *have = need;
  }

  bool forced_;
  int sms_ = 148;
  void* split_ = nullptr;
  size_t split_bytes_ = 0;
  void* part_ = nullptr;
  size_t part_bytes_ = 0;
  bool attr_set_[8] = {false, false, false, false, false, false, false, false};
  // bf16 cross terms (MLB_TC_MIXED=0 keeps all three terms in tf32)
  bool mixed_ = [] {
    const char* e = getenv("MLB_TC_MIXED");
    return e == nullptr || atoi(e) != 0;
  }();
  // CTA-pair products (MLB_TC_PAIR=1 to enable; see k_tc_product)
  bool pair_ = [] {
    const char* e = getenv("MLB_TC_PAIR");
    return e != nullptr && atoi(e) != 0;
  }();
  void* rv_ = nullptr;  // residual operands: V and W^T split into [hi | lo] rows
  void* rw_ = nullptr;
  size_t rv_bytes_ = 0, rw_bytes_ = 0;
  bool resid_attr_ = false;
};

}  // namespace

TcGemm* make_tc_gemm(bool allowed, bool forced) {
  if (!allowed) {
    if (forced) throw std::invalid_argument("tcgen05 path needs fp32 storage");
    return nullptr;
  }
  return new TcGemmImpl(forced);
}

}  // namespace mlb
