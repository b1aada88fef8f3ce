// Barrier-cost probe: cycles per round of {warp 0 (or all warps) issues S shared
// stores; __syncthreads()} for W warps per CTA, optionally with an LDS→use
// dependency after the barrier (B200).
#include <cstdio>
#include <cuda_runtime.h>
__device__ double sink;
template <int S>
__global__ void k_round(int iters, int all_store, int dep, long long* out) {
  __shared__ double buf[4096];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v = threadIdx.x;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (warp == 0 || all_store) {
#pragma unroll
      for (int s = 0; s < S; ++s) buf[(warp * 32 + lane + s * 131) & 4095] = v + s;
    }
    __syncthreads();
    if (dep) v += buf[(lane * 3 + it) & 4095];
  }
  long long t1 = clock64();
  if (v == -1.0) sink = v;
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}
int main() {
  long long* d;
  cudaMalloc(&d, 8);
  const int warps[] = {1, 4, 8, 16, 32};
  for (int dep = 0; dep < 2; ++dep)
    for (int all = 0; all < 2; ++all)
      for (int w : warps) {
        long long h[4];
        k_round<0><<<1, 32 * w>>>(2000, all, dep, d); cudaMemcpy(&h[0], d, 8, cudaMemcpyDeviceToHost);
        k_round<1><<<1, 32 * w>>>(2000, all, dep, d); cudaMemcpy(&h[1], d, 8, cudaMemcpyDeviceToHost);
        k_round<4><<<1, 32 * w>>>(2000, all, dep, d); cudaMemcpy(&h[2], d, 8, cudaMemcpyDeviceToHost);
        k_round<11><<<1, 32 * w>>>(2000, all, dep, d); cudaMemcpy(&h[3], d, 8, cudaMemcpyDeviceToHost);
        printf("{\"probe\":\"bar_round\",\"warps\":%d,\"all_warps_store\":%d,\"lds_dep\":%d,\"cycles_sts0\":%lld,\"sts1\":%lld,\"sts4\":%lld,\"sts11\":%lld}\n",
               w, all, dep, h[0], h[1], h[2], h[3]);
      }
  return 0;
}
