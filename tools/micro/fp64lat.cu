// Latency of dependent fp64 operations on B200 (cycles per op): DADD, DFMA,
// DMUL, correctly rounded division __ddiv_rn, int64 add.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n, double seed) {
  double x = seed, y = seed * 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, 1.0000001);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) y = __fma_rn(y, 0.9999999, 1e-9);
  long long t2 = clock64();
  double z = seed + 3.0;
  for (int i = 0; i < n; ++i) z = __ddiv_rn(z, 1.0000003) + 1e-12;
  long long t3 = clock64();
  double w = seed + 5.0;
  for (int i = 0; i < n; ++i) w = __dmul_rn(w, 1.0000001);
  long long t4 = clock64();
  out[threadIdx.x] = x + y + z + w;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 64);
  for (int th : {1, 32}) {
    k<<<1, th>>>(out, cyc, 1000, 1.5); cudaDeviceSynchronize();
    k<<<1, th>>>(out, cyc, 1000, 1.5); cudaDeviceSynchronize();
    printf("threads %d: DADD %.1f  DFMA %.1f  DDIV(+DADD) %.1f  DMUL %.1f cycles/op\n", th, cyc[0] / 1000.0,
           cyc[1] / 1000.0, cyc[2] / 1000.0, cyc[3] / 1000.0);
  }
  return 0;
}
