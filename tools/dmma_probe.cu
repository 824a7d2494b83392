// dmma_probe.cu -- fp64 throughput on sm_100a: mma.sync m8n8k4 f64 (DMMA)
// vs plain DFMA, independent accumulators, all SMs.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dmma(int iters, double* out) {
  double d[8][2] = {};
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
  if (s == 12345.0) out[0] = s;
}
__global__ void k_dfma(int iters, double* out) {
  double d[16] = {};
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) d[j] = fma(a, b, d[j]);
  }
  double s = 0;
  for (int j = 0; j < 16; ++j) s += d[j];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, blocks = 148 * 4, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k_dmma<<<blocks, threads>>>(iters, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32);
    printf("DMMA m8n8k4: %.2f TFLOP/s\n", flops / ms / 1e9);
    cudaEventRecord(e0); k_dfma<<<blocks, threads>>>(iters, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * iters * (double)blocks * threads;
    printf("DFMA:        %.2f TFLOP/s\n", flops / ms / 1e9);
  }
  return 0;
}
