// Round-cost probe (B200): one CTA of 16 warps; per round the last warp loads
// 18 doubles from shared memory (ping-pong buffers), runs a short FP64 chain and
// stores 9 results into the other buffer; every warp then hits __syncthreads().
// The address span (mask) is varied: small spans mimic small Jacobi matrices.
#include <cstdio>
#include <cuda_runtime.h>
__device__ double sink;
__global__ void k_round(int iters, int lanes, int mask, int store, long long* out) {
  __shared__ double buf[2][2048];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i >> 11][i & 2047] = 1.0 + i * 1e-6;
  __syncthreads();
  long long t0 = clock64();
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    const double* A = buf[it & 1];
    double* An = buf[(it + 1) & 1];
    if (warp == 15 && lane < lanes) {
      double v[18];
#pragma unroll
      for (int j = 0; j < 18; ++j) v[j] = A[(lane * 17 + j * 5) & mask];
      double r[9];
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        double x = v[2 * j] * v[(2 * j + 3) % 18] - v[2 * j + 1] * v[(2 * j + 5) % 18];
        r[j] = x * 0.25 + 0.75;
      }
      if (store) {
#pragma unroll
        for (int j = 0; j < 9; ++j) An[(lane * 17 + j * 7 + 3) & mask] = r[j];
      } else {
#pragma unroll
        for (int j = 0; j < 9; ++j) acc += r[j];
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (acc == -1.0) sink = acc;
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}
int main() {
  long long* d;
  cudaMalloc(&d, 8);
  for (int lanes : {4, 32})
    for (int mask : {63, 255, 1023, 2047}) {
      long long h[2];
      for (int st = 0; st < 2; ++st) {
        k_round<<<1, 512>>>(4000, lanes, mask, st, d);
        cudaMemcpy(&h[st], d, 8, cudaMemcpyDeviceToHost);
      }
      printf("{\"probe\":\"round_span\",\"active_lanes\":%d,\"span_doubles\":%d,\"no_store\":%lld,\"store\":%lld}\n", lanes,
             mask + 1, h[0], h[1]);
    }
  return 0;
}
