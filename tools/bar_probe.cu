// bar_probe.cu -- latency of mbarrier.try_wait vs test_wait on an already
// completed phase (warp-wide, vote exit), sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE>
__global__ void probe(int iters, long long* out) {
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  long long t0 = clock64();
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    uint32_t ok;
    if (MODE == 0)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1; selp.u32 %0, 1, 0, p;}" : "=r"(ok) : "r"(smem_u32(&bar)));
    else if (MODE == 1)
      asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], 1; selp.u32 %0, 1, 0, p;}" : "=r"(ok) : "r"(smem_u32(&bar)));
    else
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 p, [%1], 1; selp.u32 %0, 1, 0, p;}" : "=r"(ok) : "r"(smem_u32(&bar)));
    acc += __all_sync(0xffffffffu, ok);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = acc; }
}
template <int M> void run(long long* d, const char* name) {
  probe<M><<<148, 32>>>(4096, d);
  cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%-28s %.1f cycles/wait (ok=%lld)\n", name, h[0] / 4096.0, h[1]);
}
int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<0>(d, "try_wait (acquire)");
  run<1>(d, "test_wait (acquire)");
  run<2>(d, "try_wait.relaxed");
  return 0;
}
