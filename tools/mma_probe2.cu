// mma_probe2.cu -- tcgen05.mma.kind::tf32 issue rate with warp-uniform,
// compile-time operands (TMEM base 0 after a 512-column allocation).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16; d |= (uint64_t)(1024u >> 4) << 32; d |= (uint64_t)1u << 46; d |= (uint64_t)2u << 61;
  return d;
}
template <int N> __host__ __device__ constexpr uint32_t idesc() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
template <int N, int NACC, bool TS>
__global__ void __launch_bounds__(128, 1) probe(int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    const uint32_t sbase = smem_u32(sm);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t d = (uint32_t)((j % NACC) * N);
        const uint64_t bd = sdesc(sbase + (j & 3) * 32);
        if (TS) {
          const uint32_t a = 384u + (uint32_t)(j & 3) * 8;
          asm volatile("{.reg .pred p; .reg .pred e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}"
                       ::"r"(d), "r"(a), "l"(bd), "r"(idesc<N>()), "r"(1));
        } else {
          const uint64_t ad = sdesc(sbase + 16384 + (j & 3) * 32);
          asm volatile("{.reg .pred p; .reg .pred e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}"
                       ::"r"(d), "l"(ad), "l"(bd), "r"(idesc<N>()), "r"(1));
        }
      }
    }
    if (lane == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    __syncwarp();
    long long t1 = clock64();
    uint32_t ok = 0;
    do {
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    } while (!ok);
    long long t2 = clock64();
    if (blockIdx.x == 0 && lane == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(holder));
  }
}

template <int N, int NACC, bool TS>
void run(long long* d, int grid) {
  const int iters = 512;
  cudaFuncSetAttribute(probe<N, NACC, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<N, NACC, TS><<<grid, 128, 64 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double mmas = iters * 16.0, macs = mmas * 128.0 * N * 8;
  printf("tf32 M=128 N=%3d nacc=%d %s grid=%d: issue %.1f cyc/mma, total %.1f cyc/mma, %.0f MAC/cyc/SM\n", N, NACC,
         TS ? "TS" : "SS", grid, h[0] / mmas, h[1] / mmas, macs / h[1]);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<256, 1, false>(d, 148);
  run<256, 2, false>(d, 148);
  run<128, 1, false>(d, 148);
  run<64, 1, false>(d, 148);
  run<256, 1, true>(d, 148);
  run<128, 1, true>(d, 148);
  run<64, 4, true>(d, 148);
  run<256, 1, false>(d, 1);
  // one accumulation chain vs independent accumulators at N = 64 (TS)
  run<64, 1, true>(d, 148);
  run<64, 2, true>(d, 148);
  run<64, 3, true>(d, 148);
  run<128, 1, true>(d, 148);
  return 0;
}
