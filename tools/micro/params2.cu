// Empty-kernel cost between CUDA events vs CTA shape and parameter bytes (B200).
#include <cstdio>
#include <cuda_runtime.h>
template <int B> struct P { unsigned char b[B]; };
template <int B> __global__ void k(const __grid_constant__ P<B> p, int* o) { if (p.b[threadIdx.x % B] == 7 && o) o[0] = 1; }
template <int B> float run(int grid, int threads) {
  P<B> p{}; cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 20; ++i) k<B><<<grid, threads>>>(p, nullptr);
  float tot = 0;
  for (int i = 0; i < 300; ++i) {
    cudaEventRecord(a); k<B><<<grid, threads>>>(p, nullptr); cudaEventRecord(b);
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); tot += ms;
  }
  return tot / 300 * 1000;
}
int main() {
  int shapes[][2] = {{148, 1024}, {296, 512}, {592, 256}, {148, 512}, {148, 256}, {1, 32}};
  for (auto& s : shapes)
    printf("grid %4d x %4d thr: 64B %.2f us | 1344B %.2f us | 2688B %.2f us\n", s[0], s[1],
           run<64>(s[0], s[1]), run<1344>(s[0], s[1]), run<2688>(s[0], s[1]));
}
