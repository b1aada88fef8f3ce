// DMMA issue-rate probe: TFLOP/s vs warps per SM and independent accumulator chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void dmma_chains(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-12;
  double c[CH][2] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < CH; j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};" : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int j = 0; j < CH; j++) s += c[j][0] + c[j][1];
  if (s == 12345.0) out[0] = s;
}
template <int CH> void run(double* d, int warps_per_sm) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int tpb = 32 * warps_per_sm; int blocks = 148; int iters = 32768 / CH;
  dmma_chains<CH><<<blocks, tpb>>>(d, 16); cudaDeviceSynchronize();
  cudaEventRecord(e0); dmma_chains<CH><<<blocks, tpb>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 256 * CH * (double)iters * blocks * warps_per_sm;
  printf("{\"probe\":\"dmma_issue\",\"warps_per_sm\":%d,\"chains\":%d,\"tflops\":%.2f}\n", warps_per_sm, CH, fl / ms * 1e-9);
}
int main() {
  double* d; cudaMalloc(&d, 1024);
  for (int w : {1, 2, 4, 8, 16}) { run<1>(d, w); run<2>(d, w); run<4>(d, w); run<8>(d, w); run<16>(d, w); }
  return 0;
}
