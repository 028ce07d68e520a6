// What the saturating float->int conversions return for NaN / inf / out-of-range on B200.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(const double* x, unsigned* o, int n, double na, double c0) {
  int i = threadIdx.x;
  if (i >= n) return;
  unsigned a, b, c;
  double t = __fma_rn(x[i], na, c0);
  asm("cvt.rzi.u8.f64 %0, %1;" : "=r"(a) : "d"(x[i]));
  asm("cvt.rzi.u8.f64 %0, %1;" : "=r"(b) : "d"(t));
  c = __double2uint_rz(x[i]);
  o[3 * i] = a; o[3 * i + 1] = b; o[3 * i + 2] = c;
}
int main() {
  double h[8] = {NAN, -NAN, INFINITY, -INFINITY, 300.0, -5.0, 7.9, 0.0};
  double* d; unsigned* o; unsigned ho[24];
  cudaMalloc(&d, sizeof h); cudaMalloc(&o, sizeof ho);
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(d, o, 8, -3.0, 2.0);
  cudaMemcpy(ho, o, sizeof ho, cudaMemcpyDeviceToHost);
  const char* nm[8] = {"nan", "-nan", "inf", "-inf", "300", "-5", "7.9", "0"};
  for (int i = 0; i < 8; ++i) printf("%5s: u8(x)=%u u8(fma(x,-3,2))=%u u32(x)=%u\n", nm[i], ho[3*i], ho[3*i+1], ho[3*i+2]);
}
