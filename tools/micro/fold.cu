// Latency of Algorithm 1's exact fold on B200: one thread per candidate sums
// serve[site_i] over n samples in index order (a chain of n dependent DADDs),
// with the site bytes and serve table in shared memory. Also a bare DADD chain.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_fold(int n, int nc, double* out, long long* cyc) {
  __shared__ unsigned char sites[16 * 1024];
  __shared__ uint32_t bits[1024];
  __shared__ double serve[32];
  for (int i = threadIdx.x; i < 16 * 1024; i += blockDim.x) sites[i] = (unsigned char)((i * 7) % 7);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) bits[i] = i * 2654435761u;
  if (threadIdx.x < 32) serve[threadIdx.x] = 1.0 + threadIdx.x * 0.37;
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x < nc) {
    const unsigned char* st = sites + threadIdx.x * 1024;
    double ms = 0; long long ok = 0;
    for (int i0 = 0; i0 < n; i0 += 8) {
      const uint2 sw = *reinterpret_cast<const uint2*>(st + i0);
      double add[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int site = ((q < 4 ? sw.x : sw.y) >> (8 * (q & 3))) & 0xFF;
        ok += (bits[i0 + q] >> site) & 1u;
        add[q] = serve[site];
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) ms = __dadd_rn(ms, add[q]);
    }
    out[threadIdx.x] = ms + ok;
  }
  __syncthreads();
  long long t1 = clock64();
  // software-pipelined fold: the serve values of step k+1 are loaded before step k's adds
  if (threadIdx.x < nc) {
    const unsigned char* st = sites + threadIdx.x * 1024;
    double ms = 0; long long ok = 0;
    double cur[8], nxt[8];
    uint2 sw = *reinterpret_cast<const uint2*>(st);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int site = ((q < 4 ? sw.x : sw.y) >> (8 * (q & 3))) & 0xFF;
      ok += (bits[q] >> site) & 1u;
      cur[q] = serve[site];
    }
    for (int i0 = 0; i0 < n; i0 += 8) {
      const int i1 = i0 + 8 < n ? i0 + 8 : i0;
      sw = *reinterpret_cast<const uint2*>(st + i1);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int site = ((q < 4 ? sw.x : sw.y) >> (8 * (q & 3))) & 0xFF;
        if (i1 != i0) ok += (bits[i1 + q] >> site) & 1u;
        nxt[q] = serve[site];
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) ms = __dadd_rn(ms, cur[q]);
#pragma unroll
      for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
    }
    out[32 + threadIdx.x] = ms + ok;
  }
  __syncthreads();
  long long t15 = clock64();
  if (threadIdx.x == 0) cyc[2] = t15 - t1;
  t1 = t15;
  // bare chain
  double x = out[0] * 1e-300;
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, 1.0000001);
    out[63] = x;
  }
  __syncthreads();
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 64 * 8); cudaMallocManaged(&cyc, 32);
  for (int n : {128, 1000}) {
    k_fold<<<1, 512>>>(n, 6, out, cyc); cudaDeviceSynchronize();
    k_fold<<<1, 512>>>(n, 6, out, cyc); cudaDeviceSynchronize();
    printf("n=%d fold %lld cycles (%.1f per sample), pipelined %lld (%.1f), bare DADD chain %lld cycles (%.1f per add)\n", n,
           cyc[0], (double)cyc[0] / n, cyc[2], (double)cyc[2] / n, cyc[1], (double)cyc[1] / n);
  }
}
