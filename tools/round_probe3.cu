// Jacobi-round skeleton probe (B200): 16 warps; warp 15 ("pivot") loads P
// values, optionally runs a dependent FP64 chain of C steps, arrives on named
// barrier 1 after its loads (when NB) and stores S values; warps 0-14
// ("workers") wait on barrier 1 (when NB), load 6 values, do 16 FP64 ops, store
// 4 values; then __syncthreads().  Ping-pong buffers as in the real kernel.
#include <cstdio>
#include <cuda_runtime.h>
__device__ double sink;
template <int C, bool NB, bool WORK>
__global__ void k_round(int iters, long long* out) {
  __shared__ double buf[2][2048];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i >> 11][i & 2047] = 1.0 + i * 1e-6;
  __syncthreads();
  long long t0 = clock64();
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    const double* A = buf[it & 1];
    double* An = buf[(it + 1) & 1];
    if (warp == 15) {
      double v[18];
#pragma unroll
      for (int j = 0; j < 18; ++j) v[j] = A[(lane * 67 + j * 131) & 2047];
      if (NB) asm volatile("bar.arrive 1, 512;" ::: "memory");
      double x = v[0];
#pragma unroll
      for (int c = 0; c < C; ++c) x = fma(x, v[1 + (c % 17)], 0.5);
#pragma unroll
      for (int j = 0; j < 9; ++j) An[(lane * 67 + j * 131 + 5) & 2047] = x * v[j] + v[j + 9];
    } else {
      if (NB) asm volatile("bar.sync 1, 512;" ::: "memory");
      if (WORK) {
        const int base = (warp * 32 + lane) * 4;
        double a0 = A[base & 2047], a1 = A[(base + 1) & 2047], a2 = A[(base + 2) & 2047], a3 = A[(base + 3) & 2047];
        double c0 = A[(warp * 7) & 2047], c1 = A[(lane * 3 + 64) & 2047];
        double b0 = c0 * a0 - c1 * a1, b1 = c0 * a2 - c1 * a3, b2 = c1 * a0 + c0 * a1, b3 = c1 * a2 + c0 * a3;
        double d0 = c0 * b0 - c1 * b1, d1 = c1 * b0 + c0 * b1, d2 = c0 * b2 - c1 * b3, d3 = c1 * b2 + c0 * b3;
        An[(base + 7) & 2047] = d0; An[(base + 8) & 2047] = d1; An[(base + 9) & 2047] = d2; An[(base + 10) & 2047] = d3;
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
  long long h;
#define RUN(C, NB, W)                                                                                      \
  k_round<C, NB, W><<<1, 512>>>(4000, d);                                                                  \
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);                                                            \
  printf("{\"probe\":\"jacobi_round_skeleton\",\"pivot_chain_fma\":%d,\"named_barrier\":%d,\"workers\":%d,\"cycles\":%lld}\n", \
         C, NB, W, h);
  RUN(0, false, false) RUN(0, true, false) RUN(0, false, true) RUN(0, true, true)
  RUN(16, true, true) RUN(32, true, true) RUN(64, true, true)
  return 0;
}
