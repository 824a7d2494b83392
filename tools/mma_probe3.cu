// mma_probe3.cu -- the M-streaming product's MMA issue pattern in isolation:
// per chunk 4 x (N=128 into D1, N=64 into D2), TS operands, then optional
// tcgen05.commit to `commits` mbarriers and an optional fence.  Cycles/chunk.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16; d |= (uint64_t)(1024u >> 4) << 32; d |= (uint64_t)1u << 46; d |= (uint64_t)2u << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{.reg .pred p; .reg .pred e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}"
               ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff; @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}" ::"r"(bar));
}
template <int S>
__device__ __forceinline__ void chunk(uint32_t sb, int same_acc) {
  const uint32_t a_hi = 256 + S * 64, a_lo = a_hi + 32;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const uint64_t bd = sdesc(sb + S * 16384 + kk * 32);
    mma_ts(0, a_hi + kk * 8, bd, idesc(128), 1);
    mma_ts(128, a_lo + kk * 8, bd, idesc(64), 1);
  }
}
__global__ void __launch_bounds__(256, 1) probe(int iters, int commits, int fence, int same_acc, int stwarps, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
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
    const uint32_t sb = smem_u32(sm);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      switch (it & 3) {
        case 0: chunk<0>(sb, same_acc); break;
        case 1: chunk<1>(sb, same_acc); break;
        case 2: chunk<2>(sb, same_acc); break;
        default: chunk<3>(sb, same_acc); break;
      }
      for (int c = 0; c < commits; ++c) commit(smem_u32(&bar[c]));
      if (fence) asm volatile("tcgen05.fence::after_thread_sync;");
      for (int w = 0; w < same_acc; ++w) {  // vote-waits on a never-arrived barrier's previous phase (passes)
        uint32_t ok;
        do {
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1; selp.u32 %0, 1, 0, p;}"
                       : "=r"(ok) : "r"(smem_u32(&bar[6])));
        } while (!__all_sync(0xffffffffu, ok));
      }
    }
    commit(smem_u32(&bar[7]));
    long long t1 = clock64();
    uint32_t ok = 0;
    do {
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}"
                   : "=r"(ok) : "r"(smem_u32(&bar[7])));
    } while (!ok);
    long long t2 = clock64();
    if (blockIdx.x == 0 && lane == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  } else if (warp >= 4 && warp < 4 + stwarps) {
    // converter-like TMEM store traffic: 64 columns per "chunk" per warp into rotating slots
    const int q = warp & 3;
    uint32_t v[32];
    for (int k = 0; k < 32; ++k) v[k] = k * lane;
    for (int it = 0; it < iters; ++it) {
      const uint32_t ta = ((uint32_t)(q * 32) << 16) + 256 + (it & 3) * 64;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
        ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
        ::"r"(ta + 32), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
      asm volatile("tcgen05.wait::st.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(holder));
  }
}
int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  const int iters = 2048;
  int cfg[][4] = {{0, 0, 0, 0}, {0, 0, 2, 0}, {0, 1, 2, 0}, {1, 1, 2, 4}, {1, 1, 3, 4}};
  for (auto& c : cfg) {
    probe<<<148, 256, 80 * 1024>>>(iters, c[0], c[1], c[2], c[3], d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("commits=%d fence=%d vote_waits=%d st_warps=%d : issue %.1f cyc/chunk, total %.1f cyc/chunk (ideal 384)\n", c[0], c[1],
           c[2], c[3], (double)h[0] / iters, (double)h[1] / iters);
  }
  return 0;
}
