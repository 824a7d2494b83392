// ss_probe.cu -- tcgen05.mma.kind::tf32 with A read from SHARED memory as raw
// fp32 (SS form): (1) how the tensor core converts an fp32 smem operand to
// tf32 (truncate or round), (2) that a K-major SWIZZLE_128B tile and an
// MN-major SWIZZLE_128B tile (4 MN atoms at LBO) are addressed as assumed.
// B = identity (exact), so D[i][n] = tf32(A[i][n]) exactly.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ss_probe ss_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// D f32, A/B tf32, N, M = 128; a_mn: A MN-major (bit 15)
__host__ __device__ constexpr uint32_t idesc(int N, int a_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}

// mode 0: A K-major; mode 1: A MN-major (LBO = MN atom stride 4096, SBO = 1024);
// mode 2: A MN-major with LBO / SBO swapped; mode 3: A K-major, B flagged
// MN-major (the identity has the same bytes in both layouts)
__global__ void __launch_bounds__(128, 1) probe(const float* A, int mode, float* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  unsigned char* sa = base;           // 16 KB
  unsigned char* sb = base + 16384;   // 32 rows x 128 B = 4 KB (N = 32)
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // A[i][k], i < 128, k < 32
  for (int e = t; e < 128 * 32; e += 128) {
    const int i = e / 32, k = e % 32;
    uint32_t off;
    if (mode == 0 || mode == 3)
      off = i * 128 + (((k >> 2) ^ (i & 7)) << 4) + (k & 3) * 4;
    else {
      const int b = i >> 5, w = i & 31;
      off = b * 4096 + k * 128 + (((w >> 2) ^ (k & 7)) << 4) + (w & 3) * 4;
    }
    *(float*)(sa + off) = A[e];
  }
  // B[n][k] = (n == k), N = 32, K-major SW128
  for (int e = t; e < 32 * 32; e += 128) {
    const int n = e / 32, k = e % 32;
    *(float*)(sb + n * 128 + (((k >> 2) ^ (n & 7)) << 4) + (k & 3) * 4) = n == k ? 1.0f : 0.0f;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = holder;
  if (warp == 0) {
    const uint32_t id = idesc(32, mode == 1 || mode == 2) | (mode == 3 ? (1u << 16) : 0u);
    for (int s = 0; s < 4; ++s) {
      uint64_t ad;
      if (mode == 0 || mode == 3)
        ad = desc(smem_u32(sa) + s * 32, 16, 1024);
      else if (mode == 1)
        ad = desc(smem_u32(sa) + s * 1024, 4096, 1024);
      else
        ad = desc(smem_u32(sa) + s * 1024, 1024, 4096);
      const uint64_t bd = mode == 3 ? desc(smem_u32(sb) + s * 1024, 4096, 1024) : desc(smem_u32(sb) + s * 32, 16, 1024);
      const uint32_t acc = s > 0;
      asm volatile(
          "{.reg .pred p; .reg .pred e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0;"
          " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(id), "r"(acc));
    }
    asm volatile(
        "{.reg .pred e; elect.sync _|e, 0xffffffff;"
        " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}" ::"r"(smem_u32(&bar)));
  }
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}"
                 : "=r"(ok)
                 : "r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int n = 0; n < 32; ++n) D[(warp * 32 + lane) * 32 + n] = __uint_as_float(v[n]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
  }
}

static float bits(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static uint32_t ubits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}

int main() {
  const int NE = 128 * 32;
  float* hA = (float*)malloc(NE * 4);
  float* hD = (float*)malloc(NE * 4);
  srand(1);
  for (int e = 0; e < NE; ++e) {
    // random fp32 in [0.5, 2) with all 23 mantissa bits random; some negatives
    uint32_t m = ((uint32_t)rand() << 8 ^ (uint32_t)rand()) & 0x7FFFFFu;
    uint32_t ex = 126 + (rand() & 1);
    uint32_t s = (e % 7 == 3) ? 0x80000000u : 0;
    hA[e] = bits(s | ex << 23 | m);
  }
  float *dA, *dD;
  cudaMalloc(&dA, NE * 4);
  cudaMalloc(&dD, NE * 4);
  cudaMemcpy(dA, hA, NE * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  const char* names[] = {"K-major SW128", "MN-major SW128 (LBO=4096 MN atoms, SBO=1024)",
                         "MN-major SW128 (LBO=1024, SBO=4096)", "A K-major, B MN-major"};
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(dD, 0, NE * 4);
    probe<<<1, 128, 32 * 1024>>>(dA, mode, dD);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
      printf("%s: error %s\n", names[mode], cudaGetErrorString(err));
      return 1;
    }
    cudaMemcpy(hD, dD, NE * 4, cudaMemcpyDeviceToHost);
    int n_trunc = 0, n_rna = 0, n_rne = 0, n_bad = 0;
    for (int e = 0; e < NE; ++e) {
      const uint32_t u = ubits(hA[e]);
      const float tr = bits(u & 0xFFFFE000u);
      const float rna = bits((u + 0x1000u) & 0xFFFFE000u);
      const uint32_t lsb = (u >> 13) & 1u;
      const float rne = bits((u + 0xFFFu + lsb) & 0xFFFFE000u);
      const float d = hD[e];
      const bool t = d == tr, a = d == rna, r = d == rne;
      n_trunc += t, n_rna += a, n_rne += r;
      if (!t && !a && !r) ++n_bad;
    }
    printf("%s: of %d: trunc %d, rna %d, rne %d, none %d  (D[0]=%.9g A[0]=%.9g)\n", names[mode], NE, n_trunc, n_rna,
           n_rne, n_bad, hD[0], hA[0]);
  }
  return 0;
}
