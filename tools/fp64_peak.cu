// FP64 roofline denominator probe for B200 (sm_100a).
// Measures: DFMA issue-bound peak, DMMA.8x8x4 (mma.sync m8n8k4 f64) peak, and
// cuBLAS DGEMM (yardstick only) at a few shapes including the skinny shapes of
// the stacked sketch GEMMs. Prints one JSON line per measurement.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-12;
  double c[8][2] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int j = 0; j < 8; j++) s += c[j][0] + c[j][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-12;
  double c[16] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 16; j++) c[j] = fma(a, c[j], b);
  }
  double s = 0; for (int j = 0; j < 16; j++) s += c[j];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  double* d; CK(cudaMalloc(&d, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    int iters = 4096;
    dmma_loop<<<blocks, tpb>>>(d, 16); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_loop<<<blocks, tpb>>>(d, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * blocks * (tpb / 32);
    printf("{\"probe\":\"dmma_m8n8k4\",\"tpb\":%d,\"blocks\":%d,\"tflops\":%.3f}\n", tpb, blocks, flops / ms * 1e-9);
    dfma_loop<<<blocks, tpb>>>(d, 16); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_loop<<<blocks, tpb>>>(d, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * (double)iters * blocks * tpb;
    printf("{\"probe\":\"dfma\",\"tpb\":%d,\"blocks\":%d,\"tflops\":%.3f}\n", tpb, blocks, flops / ms * 1e-9);
  }
  cublasHandle_t h; cublasCreate(&h);
  struct S { int m, n, k; int ta, tb; const char* what; };
  std::vector<S> shapes = {{8192, 8192, 8192, 0, 0, "square"},
                           {8192, 64, 8192, 1, 0, "stageA_RxS_TN"},
                           {8192, 64, 8192, 0, 0, "stageC_NxS_NN"},
                           {64, 8192, 8192, 1, 0, "stageE_QxR_TN"}};
  for (auto s : shapes) {
    size_t na = (size_t)s.m * s.k, nb = (size_t)s.k * s.n, nc = (size_t)s.m * s.n;
    double *A, *B, *C; CK(cudaMalloc(&A, na * 8)); CK(cudaMalloc(&B, nb * 8)); CK(cudaMalloc(&C, nc * 8));
    cudaMemset(A, 0, na * 8); cudaMemset(B, 0, nb * 8);
    double al = 1, be = 0;
    int lda = s.ta ? s.k : s.m, ldb = s.tb ? s.n : s.k;
    auto run = [&]() { cublasDgemm(h, s.ta ? CUBLAS_OP_T : CUBLAS_OP_N, s.tb ? CUBLAS_OP_T : CUBLAS_OP_N,
                                   s.m, s.n, s.k, &al, A, lda, B, ldb, &be, C, s.m); };
    for (int i = 0; i < 3; i++) run();
    CK(cudaDeviceSynchronize());
    int reps = 10;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; i++) run();
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * s.m * s.n * (double)s.k * reps;
    printf("{\"probe\":\"cublas_dgemm\",\"shape\":\"%s\",\"m\":%d,\"n\":%d,\"k\":%d,\"tflops\":%.3f}\n", s.what, s.m, s.n, s.k, flops / ms * 1e-9);
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  printf("{\"probe\":\"device\",\"name\":\"%s\",\"sms\":%d,\"clock_khz\":%d}\n", p.name, sms, p.clockRate);
  return 0;
}
