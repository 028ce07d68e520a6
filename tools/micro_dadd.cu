// Microbenchmark: dependent fp64 add chain latency on sm_100a (one thread),
// and the same chain fed from shared memory with gathered addends.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, int iters, double a) {
  double x = 0.0;
  for (int i = 0; i < iters; ++i) x = __dadd_rn(x, a);
  out[0] = x;
}
__global__ void chain_i(long long* out, int iters, long long a) {
  long long x = 0;
  for (int i = 0; i < iters; ++i) x = x + a * (long long)i;
  out[0] = x;
}
__global__ void chain_f(float* out, int iters, float a) {
  float x = 0.0f;
  for (int i = 0; i < iters; ++i) x = __fadd_rn(x, a);
  out[0] = x;
}
int main() {
  double* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 1 << 20;
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); chain<<<1, 1>>>(d, iters, 1.5); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DADD chain: %.2f ns per add\n", ms * 1e6 / iters);
    cudaEventRecord(e0); chain_f<<<1, 1>>>((float*)d, iters, 1.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FADD chain: %.2f ns per add\n", ms * 1e6 / iters);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock %d kHz\n", clk);
  return 0;
}
