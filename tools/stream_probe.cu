// stream_probe.cu -- read-only TMA streaming ceiling for the product kernels'
// access patterns (no compute): persistent CTAs stream an m x n fp32 matrix
// as 2-D boxes through a shared-memory ring; one consumer warp only releases
// stages.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool tryw(uint32_t a, uint32_t ph) {
  uint32_t ok;
  asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(a), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void wait(uint32_t a, uint32_t ph) { while (!tryw(a, ph)) {} }

template <int STAGES, int BYTES>
__global__ void __launch_bounds__(64, 1) k_stream(const __grid_constant__ CUtensorMap map, int ntiles_outer, int nchunks, int rowmode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const long total = (long)ntiles_outer * nchunks;
  if (warp == 0 && lane == 0) {
    int s = 0; uint32_t ph = 0;
    for (long u = blockIdx.x; u < total; u += gridDim.x) {
      const int t = (int)(u / nchunks), c = (int)(u % nchunks);
      wait(su(&empty[s]), ph ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(BYTES));
      const int c0 = rowmode ? c * 32 : t * 128, c1 = rowmode ? t * 128 : c * 32;
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su(sm + s * BYTES)), "l"((uint64_t)&map), "r"(c0), "r"(c1), "r"(su(&full[s])) : "memory");
      if (++s == STAGES) s = 0, ph ^= 1;
    }
  } else if (warp == 1 && lane == 0) {
    int s = 0; uint32_t ph = 0;
    for (long u = blockIdx.x; u < total; u += gridDim.x) {
      wait(su(&full[s]), ph);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])));
      if (++s == STAGES) s = 0, ph ^= 1;
    }
  }
}

int main() {
  const size_t m = 65536, n = 262144;
  float* M; cudaMalloc(&M, m * n * 4); cudaMemset(M, 0, m * n * 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  for (int mode = 1; mode >= 0; --mode) {  // 1: 128 rows x 32 cols (product A), 0: 32 rows x 128 cols (product C)
    CUtensorMap map;
    cuuint64_t dims[2] = {n, m}; cuuint64_t str[1] = {n * 4};
    cuuint32_t box[2] = {mode ? 32u : 128u, mode ? 128u : 32u}; cuuint32_t es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, M, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        mode ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int outer = mode ? (int)(m / 128) : (int)(n / 128), nch = mode ? (int)(n / 32) : (int)(m / 32);
    auto k = k_stream<12, 16384>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384 + 1024);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      k<<<148, 64, 12 * 16384 + 1024>>>(map, outer, nch, mode);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("%s: %.3f ms  %.0f GB/s  (%s)\n", mode ? "128x32 boxes (A)" : "32x128 boxes (C)", ms, m * n * 4 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
