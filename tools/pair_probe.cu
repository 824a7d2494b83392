// pair_probe.cu -- tcgen05.mma.cta_group::2 (CTA pair, M = 256) kind::tf32 in
// the TS form with N = 64: which shared-memory B rows each CTA supplies, that
// the A operand comes from each CTA's own TMEM lanes, and that a multicast
// commit reaches both CTAs.  One cluster of 2 CTAs, K = 8 (one MMA).
//   A (TMEM, each CTA its 128 rows): A[c][i][k] = ((c * 128 + i) % 7) + 0.5 k
//   B (smem, K-major SW128): CTA c holds 32 rows, B[c][n'][k] = (c * 32 + n') % 5 + k
// Expectation checked: D[c][i][n] = sum_k A[c][i][k] * Bfull[n][k] with
// Bfull[n] = CTA (n / 32)'s row n % 32 (hypothesis H1), or Bfull = CTA 0's
// rows only (H0).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pair_probe pair_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int N, int M) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(float* D) {
  __shared__ __align__(1024) unsigned char sb[4096];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // B half of this CTA: 32 rows x 32 fp32 (k < 8 nonzero), K-major SW128
  for (int e = t; e < 32 * 32; e += 128) {
    const int n = e / 32, k = e % 32;
    const float v = k < 8 ? (float)(((int)rank * 32 + n) % 5 + k) : 0.f;
    *(float*)(sb + n * 128 + (((k >> 2) ^ (n & 7)) << 4) + (k & 3) * 4) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = holder;
  // A: columns 64..71 of this CTA's TMEM, lane i = row i
  {
    uint32_t v[8];
    const int i = warp * 32 + lane;
    for (int k = 0; k < 8; ++k) v[k] = __float_as_uint((float)(((int)rank * 128 + i) % 7) + 0.5f * k);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
                     tmem + ((uint32_t)(warp * 32) << 16) + 64),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (rank == 0 && warp == 0) {
    const uint32_t id = idesc(64, 256);
    const uint64_t bd = desc(smem_u32(sb));
    asm volatile(
        "{.reg .pred p; .reg .pred e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0;"
        " @e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;}" ::"r"(tmem),
        "r"(tmem + 64), "l"(bd), "r"(id), "r"(0));
    asm volatile(
        "{.reg .pred e; elect.sync _|e, 0xffffffff;"
        " @e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;}" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)3));
  }
  uint32_t ok = 0;
  for (long long it = 0; !ok && it < (1ll << 26); ++it)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}"
                 : "=r"(ok)
                 : "r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[32];
  for (int h = 0; h < 2; ++h) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16) + h * 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int n = 0; n < 32; ++n) D[((int)rank * 128 + warp * 32 + lane) * 64 + h * 32 + n] = __uint_as_float(v[n]);
  }
  if (t == 0 && !ok) D[0] = -1.f;
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(tmem));
  }
}

int main() {
  float* dD;
  cudaMalloc(&dD, 256 * 64 * 4);
  cudaMemset(dD, 0, 256 * 64 * 4);
  probe<<<2, 128>>>(dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  static float hD[256 * 64];
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  int ok1 = 0, ok0 = 0;
  for (int row = 0; row < 256; ++row)
    for (int n = 0; n < 64; ++n) {
      double e1 = 0, e0 = 0;
      for (int k = 0; k < 8; ++k) {
        const double a = (row % 7) + 0.5 * k;  // row = c * 128 + i
        e1 += a * (double)(n % 5 + k);          // B row n from CTA n / 32: ((n/32)*32 + n%32) % 5 = n % 5
        e0 += a * (double)((n % 32) % 5 + k);   // only CTA 0's rows (n mod 32)
      }
      ok1 += hD[row * 64 + n] == (float)e1;
      ok0 += hD[row * 64 + n] == (float)e0;
    }
  printf("cta_group::2 TS N=64: of %d outputs, H1 (B rows split 32/32 across the pair) %d, H0 (CTA 0 rows) %d; "
         "D[0][0]=%g D[128][33]=%g\n",
         256 * 64, ok1, ok0, hD[0], hD[128 * 64 + 33]);
  return 0;
}
