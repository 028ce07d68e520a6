// Microbenchmark: shared-memory histogram increments on sm_100a.
// Measures throughput of per-CTA smem atomicAdd with random bins (12 x 65 bins,
// one copy per CTA or one per warp) to size the diagonal-family histogram path.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int COPIES>
__global__ void k_hist(const uint8_t* __restrict__ keys, int64_t n, int r, unsigned* out) {
  __shared__ unsigned h[COPIES][12 * 65 + 1];
  for (int i = threadIdx.x; i < COPIES * (12 * 65 + 1); i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const int copy = (threadIdx.x / 32) % COPIES;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t* k = keys + i * 12;
    uint4 v = *reinterpret_cast<const uint4*>(keys + (i * 12 & ~15ll));  // touch
    (void)v;
#pragma unroll
    for (int j = 0; j < 12; ++j) atomicAdd(&h[copy][j * 65 + (k[j] & 63)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 12 * 65; i += blockDim.x) {
    unsigned s = 0;
    for (int c = 0; c < COPIES; ++c) s += h[c][i];
    atomicAdd(out + i, s);
  }
}

int main() {
  const int64_t n = 1 << 20;
  uint8_t* keys;
  unsigned* out;
  cudaMalloc(&keys, n * 12 + 16);
  cudaMalloc(&out, 12 * 65 * 4);
  uint8_t* hk = (uint8_t*)malloc(n * 12);
  uint64_t x = 88172645463325252ull;
  for (int64_t i = 0; i < n * 12; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; hk[i] = (uint8_t)(x % 65); }
  cudaMemcpy(keys, hk, n * 12, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int blocks_per_sm : {2, 4, 8}) {
    float ms1 = 0, ms8 = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      k_hist<1><<<sms * blocks_per_sm, 256>>>(keys, n, 12, out);
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms1, a, b);
      cudaEventRecord(a);
      k_hist<8><<<sms * blocks_per_sm, 256>>>(keys, n, 12, out);
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms8, a, b);
    }
    printf("blocks/SM %d: 1 copy %.1f us (%.2f G atom/s), 8 copies %.1f us (%.2f G atom/s)\n", blocks_per_sm,
           ms1 * 1e3, n * 12 / (ms1 * 1e6), ms8 * 1e3, n * 12 / (ms8 * 1e6));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
