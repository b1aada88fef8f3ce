// Latency probe: dependent fp64 ops, MUFU fp64 approximations, block barriers (B200).
#include <cstdio>
#include <cuda_runtime.h>
__device__ double sink;
__global__ void k_dfma(int iters, long long* out) {
  double x = threadIdx.x * 1e-3 + 1.0, y = 0.999999;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) { x = fma(x, y, 1e-7); x = fma(x, y, 1e-7); x = fma(x, y, 1e-7); x = fma(x, y, 1e-7); }
  long long t1 = clock64();
  if (x == 123.0) sink = x;
  if (threadIdx.x == 0) out[0] = (t1 - t0) / (4LL * iters);
}
__global__ void k_rcp(int iters, long long* out) {
  double x = threadIdx.x * 1e-3 + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) { double y; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y + 0.5; }
  long long t1 = clock64();
  if (x == 123.0) sink = x;
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}
__global__ void k_rsq(int iters, long long* out) {
  double x = threadIdx.x * 1e-3 + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y + 1.5; }
  long long t1 = clock64();
  if (x == 123.0) sink = x;
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}
__global__ void k_div(int iters, long long* out) {
  double x = threadIdx.x * 1e-3 + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) { x = 1.0 / x + 0.5; }
  long long t1 = clock64();
  if (x == 123.0) sink = x;
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}
__global__ void k_sqrt(int iters, long long* out) {
  double x = threadIdx.x * 1e-3 + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) { x = sqrt(x) + 0.5; }
  long long t1 = clock64();
  if (x == 123.0) sink = x;
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}
__global__ void k_bar(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}
__global__ void k_lds(int iters, long long* out) {
  __shared__ int buf[1024];
  buf[threadIdx.x] = (threadIdx.x + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) p = buf[p];
  long long t1 = clock64();
  if (p == 12345) sink = p;
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}
__global__ void k_shfl(int iters, long long* out) {
  double x = threadIdx.x * 1e-3 + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) x += __shfl_xor_sync(0xffffffffu, x, 1);
  long long t1 = clock64();
  if (x == 123.0) sink = x;
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}
int main() {
  long long* d; cudaMalloc(&d, 8); long long h;
  auto run = [&](const char* name, void (*k)(int, long long*), int threads) {
    k<<<1, threads>>>(100, d); cudaDeviceSynchronize();
    k<<<1, threads>>>(10000, d); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("{\"probe\":\"%s\",\"threads\":%d,\"cycles\":%lld}\n", name, threads, h);
  };
  run("dfma_latency", k_dfma, 32);
  run("rcp_approx_f64_latency", k_rcp, 32);
  run("rsqrt_approx_f64_latency", k_rsq, 32);
  run("div_f64_latency", k_div, 32);
  run("sqrt_f64_latency", k_sqrt, 32);
  run("lds_latency", k_lds, 32);
  run("shfl_f64_plus_dadd_latency", k_shfl, 32);
  for (int t : {32, 64, 128, 256, 512, 1024}) run("bar_sync", k_bar, t);
  return 0;
}
