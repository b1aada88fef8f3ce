// Do DMMA (FP64 tensor) and DFMA (FP64 ALU) share issue capacity on B200?
// Each CTA runs W warps; warps with (warp % 2 == 0) issue DMMA.8x8x4, the others
// DFMA (mode 2), or all DMMA (mode 0), or all DFMA (mode 1).  Prints TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>
__device__ double sink;
__global__ void mixed(int iters, int mode) {
  const int warp = threadIdx.x >> 5;
  const bool use_mma = mode == 0 || (mode == 2 && (warp & 1) == 0);
  double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-12;
  double s = 0;
  if (use_mma) {
    double c[8][2] = {};
    for (int i = 0; i < iters; i++) {
#pragma unroll
      for (int j = 0; j < 8; j++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
    for (int j = 0; j < 8; j++) s += c[j][0] + c[j][1];
  } else {
    double c[16] = {};
    for (int i = 0; i < 2 * iters; i++) {
#pragma unroll
      for (int j = 0; j < 16; j++) c[j] = fma(a, c[j], b);
    }
    for (int j = 0; j < 16; j++) s += c[j];
  }
  if (s == 12345.0) sink = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount, tpb = 512, blocks = sms * 4, iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    mixed<<<blocks, tpb>>>(16, mode); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    mixed<<<blocks, tpb>>>(iters, mode);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)blocks * tpb / 32;
    const double mma_w = mode == 0 ? warps : (mode == 1 ? 0 : warps / 2);
    const double fma_w = warps - mma_w;
    const double flops = mma_w * 8.0 * iters * 512 + fma_w * 32 * 16.0 * 2 * iters * 2;
    printf("{\"probe\":\"fp64_mix\",\"mode\":\"%s\",\"tflops\":%.2f,\"ms\":%.3f}\n",
           mode == 0 ? "dmma" : (mode == 1 ? "dfma" : "half_dmma_half_dfma"), flops / ms * 1e-9, ms);
  }
  return 0;
}
