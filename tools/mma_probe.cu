// mma_probe.cu -- microbenchmark of tcgen05.mma.kind::tf32 issue/throughput
// on sm_100a (A from TMEM = TS, or from shared memory = SS), to size the
// M-streaming product pipeline.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
// Each CTA (one per SM): warp 0 lane 0 issues `iters` groups of MMAs
//   group = `per` MMAs (N = n) rotating over `nacc` independent accumulators,
//   then a tcgen05.commit every `commit_every` groups and a wait on it every
//   `wait_every` groups.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int N, int kind, int M) {
  // kind 0: tf32 (fmt 2), kind 1: bf16 (fmt 1)
  return (1u << 4) | ((kind ? 1u : 2u) << 7) | ((kind ? 1u : 2u) << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__global__ void __launch_bounds__(128, 1) probe(int iters, int per, int n, int nacc, int ts, int commit_every,
                                                int wait_every, int kind, int M, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
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
  const uint32_t tmem = holder;
  if (warp == 0) {
    const uint32_t id = idesc(n, kind, M);
    const uint64_t bd = sdesc(smem_u32(base));
    const uint64_t ad = sdesc(smem_u32(base + 16384));
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int j = 0; j < per; ++j) {
        const uint32_t d = tmem + (uint32_t)((j % nacc) * n);
        const uint32_t a = tmem + 384 + (uint32_t)(j % 4) * 8;
        const uint32_t acc = it > 0 ? 1u : 0u;
        if (kind == 0) {
          if (ts)
            asm volatile("{.reg .pred p; .reg .pred e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}"
                         ::"r"(d), "r"(a), "l"(bd), "r"(id), "r"(acc));
          else
            asm volatile("{.reg .pred p; .reg .pred e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}"
                         ::"r"(d), "l"(ad), "l"(bd), "r"(id), "r"(acc));
        } else {
          if (ts)
            asm volatile("{.reg .pred p; .reg .pred e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}"
                         ::"r"(d), "r"(a), "l"(bd), "r"(id), "r"(acc));
          else
            asm volatile("{.reg .pred p; .reg .pred e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                         ::"r"(d), "l"(ad), "l"(bd), "r"(id), "r"(acc));
        }
      }
      if (commit_every > 0 && (it + 1) % commit_every == 0) {
        // commit and wait: a full MMA round trip every commit_every groups
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        uint32_t ok = 0;
        do {
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                       : "=r"(ok) : "r"(smem_u32(&bar)), "r"(phase));
        } while (!ok);
        phase ^= 1;
      }
    }
    if (lane == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    __syncwarp();
    long long t1 = clock64();
    // final wait for all MMAs
    uint32_t ok = 0;
    int tries = 0;
    while (tries < 1 << 28) {
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                   : "=r"(ok) : "r"(smem_u32(&bar)), "r"(phase));
      if (ok) break;
      ++tries;
    }
    long long t2 = clock64();
    if (blockIdx.x == 0 && lane == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main(int argc, char** argv) {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  struct Cfg { int per, n, nacc, ts, ce, we, kind, M; } cfgs[] = {
      {8, 256, 1, 0, 0, 0, 0, 128}, {8, 256, 2, 0, 0, 0, 0, 128}, {8, 128, 1, 0, 0, 0, 0, 128},
      {8, 64, 1, 0, 0, 0, 0, 128}, {8, 256, 1, 0, 0, 0, 1, 128}, {8, 256, 1, 1, 0, 0, 0, 128},
      {32, 256, 1, 0, 0, 0, 0, 128}, {8, 256, 1, 0, 0, 0, 0, 64},
      {12, 64, 1, 1, 0, 0, 0, 128}, {12, 64, 1, 0, 0, 0, 0, 128}, {12, 64, 2, 1, 0, 0, 0, 128},
      {12, 64, 2, 0, 0, 0, 0, 128}, {12, 128, 1, 1, 0, 0, 0, 128}, {12, 128, 1, 0, 0, 0, 0, 128},
  };
  const int iters = 1024;
  for (auto c : cfgs) {
    long long h[2];
    probe<<<148, 128, 64 * 1024>>>(iters, c.per, c.n, c.nacc, c.ts, c.ce, c.we, c.kind, c.M, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double mmas = (double)iters * c.per;
    const double macs = mmas * (double)c.M * c.n * (c.kind ? 16 : 8);
    printf("%s M=%d per=%2d N=%3d nacc=%d %s commit_every=%d wait_every=%d : issue %.1f cyc/mma, total %.1f cyc/mma, %.0f MAC/cyc\n",
           c.kind ? "bf16" : "tf32", c.M, c.per, c.n, c.nacc, c.ts ? "TS" : "SS", c.ce, c.we, h[0] / mmas, h[1] / mmas, macs / h[1]);
  }
  return 0;
}
