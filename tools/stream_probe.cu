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
__global__ void __launch_bounds__(64, 1) k_stream(const __grid_constant__ CUtensorMap map, int ntiles_outer, int nchunks, int rowmode, int rot, int boxw) {
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
  const long total = (long)ntiles_outer * nchunks + (rowmode == 2 ? 148L * 8192 : 0);  // mode 2 breaks by unit count
  if (warp == 0 && lane == 0) {
    int s = 0; uint32_t ph = 0;
    for (long u = blockIdx.x; u < total; u += gridDim.x) {
      int t, c;
      if (rowmode == 2) {  // product-kernel order: units (tile, split) dealt round-robin, 13 splits
        const int splits = 13, cps = (nchunks + splits - 1) / splits;
        const long k = (u - blockIdx.x) / gridDim.x;   // k-th chunk of this CTA
        const long unit = blockIdx.x + (k / cps) * gridDim.x;
        if (unit >= (long)ntiles_outer * splits) break;
        const int tt = rot == 2 ? (int)(unit / splits) : (int)(unit % ntiles_outer);
        const int sp = rot == 2 ? (int)(unit % splits) : (int)(unit / ntiles_outer);
        const int i = (int)(k % cps);
        const int ii = rot == 1 ? (int)((i + (long)tt * 97) % cps) : i;
        t = tt; c = sp * cps + ii;
      } else {
        t = (int)(u / nchunks); c = (int)(u % nchunks);
      }
      wait(su(&empty[s]), ph ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(BYTES));
      const int c0 = rowmode ? c * boxw : t * 128, c1 = rowmode ? t * 128 : c * 32;  // mode 2 = row boxes
      if (boxw == 0)
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(su(sm + s * BYTES)), "l"((uint64_t)&map), "r"(0), "r"(c * 2), "r"(t * 128), "r"(su(&full[s])) : "memory");
      else
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su(sm + s * BYTES)), "l"((uint64_t)&map), "r"(c0), "r"(c1), "r"(su(&full[s])) : "memory");
      if (++s == STAGES) s = 0, ph ^= 1;
    }
  } else if (warp == 1 && lane == 0) {
    int s = 0; uint32_t ph = 0;
    for (long u = blockIdx.x; u < total; u += gridDim.x) {
      if (rowmode == 2) {
        const int splits = 13, cps = (nchunks + splits - 1) / splits;
        const long k = (u - blockIdx.x) / gridDim.x;
        if (blockIdx.x + (k / cps) * gridDim.x >= (long)ntiles_outer * splits) break;
      }
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
  for (int mode = 6; mode >= 5; --mode) {  // 1: 128 rows x 32 cols (product A), 0: 32 rows x 128 cols (product C)
    CUtensorMap map;
    if (mode == 6) {
      cuuint64_t d3[3] = {32, n / 32, m}; cuuint64_t s3[2] = {128, n * 4};
      cuuint32_t b3[3] = {32, 2, 128}; cuuint32_t e3[3] = {1, 1, 1};
      enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, M, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    cuuint64_t dims[2] = {n, m}; cuuint64_t str[1] = {n * 4};
    cuuint32_t box[2] = {mode == 5 ? 64u : mode ? 32u : 128u, mode ? 128u : 32u}; cuuint32_t es[2] = {1, 1};  // mode 5: 256 B rows
    if (mode != 6) enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, M, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        (mode && mode != 5) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int outer = mode ? (int)(m / 128) : (int)(n / 128), nch = mode >= 5 ? (int)(n / 64) : mode ? (int)(n / 32) : (int)(m / 32);
    auto run = [&](auto kern, int stages) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, stages * 16384 + 1024);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      float best = 1e9f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        kern<<<148, 64, stages * 16384 + 1024>>>(map, outer, nch, mode >= 2 ? 2 : mode, mode == 3 ? 1 : mode == 4 ? 2 : 0, mode == 6 ? 0 : mode == 5 ? 64 : 32);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      printf("%s stages %2d (%3d KB in flight): %.3f ms  %.0f GB/s  (%s)\n", mode == 6 ? "3-D (32,2,128) SW128 boxes, A order" : mode == 5 ? "128x64 per-CTA tiles (256 B rows, A order)" : mode == 4 ? "128x32 tile-major blocked (13 K ranges/tile)" : mode == 3 ? "128x32 per-CTA tiles, rotated" : mode == 2 ? "128x32 per-CTA tiles (A order)" : mode ? "128x32 boxes (A)" : "32x128 boxes (C)", stages,
             stages * 16, best, m * n * 4 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    if (mode >= 5) {
      run(k_stream<3, 32768>, 6);
      run(k_stream<6, 32768>, 12);
    } else {
      run(k_stream<4, 16384>, 4);
      run(k_stream<8, 16384>, 8);
    }
  }
  return 0;
}
