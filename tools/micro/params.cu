// Launch cost seen by CUDA events vs kernel-parameter size (empty kernels), B200.
#include <cstdio>
#include <cuda_runtime.h>
template <int B> struct P { unsigned char b[B]; };
template <int B> __global__ void k(const __grid_constant__ P<B> p, int* o) { if (p.b[threadIdx.x % B] == 7 && o) o[0] = 1; }
template <int B> float run(int threads, size_t smem) {
  P<B> p{}; cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaFuncSetAttribute(k<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int i = 0; i < 20; ++i) k<B><<<148, threads, smem>>>(p, nullptr);
  float tot = 0;
  for (int i = 0; i < 200; ++i) {
    cudaEventRecord(a); k<B><<<148, threads, smem>>>(p, nullptr); cudaEventRecord(b);
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); tot += ms;
  }
  return tot / 200 * 1000;
}
int main() {
  printf("params 64B   1024thr smem 0     : %.2f us\n", run<64>(1024, 0));
  printf("params 2688B 1024thr smem 0     : %.2f us\n", run<2688>(1024, 0));
  printf("params 64B   1024thr smem 96KB  : %.2f us\n", run<64>(1024, 96 << 10));
  printf("params 2688B 1024thr smem 96KB  : %.2f us\n", run<2688>(1024, 96 << 10));
  printf("params 2688B 1024thr smem 160KB : %.2f us\n", run<2688>(1024, 160 << 10));
  printf("params 64B   256thr  smem 0     : %.2f us\n", run<64>(256, 0));
}
