// Microbenchmark of the primitives the diagonal-sweep redesign depends on:
// shared atomics vs. non-atomic RMW vs. MATCH.ANY, in SM cycles per warp-op.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
template <int MODE, int ACTIVE>
__global__ void k(unsigned* out, unsigned seed) {
  extern __shared__ int h[];
  for (int i = threadIdx.x; i < 48 * 1024; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned x = seed * 2654435761u + threadIdx.x * 40503u;
  unsigned acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    x = x * 1664525u + 1013904223u;
    const bool act = lane < ACTIVE;
    if (MODE == 0) {  // ATOMS, distinct addresses (bank = lane), per-warp region
      int* a = h + warp * 1024 + ((x >> 20) & 31) * 32 + lane - (warp >= 16 ? 16 * 1024 : 0);
      if (act) atomicAdd(a, 1);
    } else if (MODE == 1) {  // ATOMS, random addresses within per-warp 1690-int region
      int* a = h + (warp % 16) * 2048 + ((x >> 16) % 1690);
      if (act) atomicAdd(a, 1);
    } else if (MODE == 2) {  // lane-private RMW (plain LDS/STS), random cell in own row of 130
      int* a = h + warp * 32 * 130 / 4 * 0 + (warp * 32 + lane) * 33 + ((x >> 16) % 33);
      if (act) { int v = *(volatile int*)a; *(volatile int*)a = v + 1; }
    } else if (MODE == 3) {  // MATCH.ANY over a 6-bit key
      unsigned m = __match_any_sync(0xffffffffu, (x >> 26));
      acc += m;
    } else if (MODE == 4) {  // VOTE.ballot
      acc += __ballot_sync(0xffffffffu, x & 0x100);
    } else if (MODE == 5) {  // ATOMS, random addr, concentrated (8 distinct cells)
      int* a = h + (warp % 16) * 2048 + ((x >> 29) & 7) * 65;
      if (act) atomicAdd(a, 1);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x * 2] = (unsigned)(t1 - t0);
  if (acc == 0x12345) out[1] = acc;
}

template <int MODE, int ACTIVE>
void run(const char* name, int warps) {
  unsigned* d;
  cudaMalloc(&d, 1024 * 8);
  cudaFuncSetAttribute(k<MODE, ACTIVE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608);
  k<MODE, ACTIVE><<<1, warps * 32, 196608>>>(d, 1);
  cudaDeviceSynchronize();
  k<MODE, ACTIVE><<<1, warps * 32, 196608>>>(d, 2);
  unsigned h;
  cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
  printf("%-44s warps=%2d active=%2d: %7.2f cyc per warp-op (SM-wide), %6.3f cyc per lane-op\n", name,
         warps, ACTIVE, (double)h / ITERS / warps, (double)h / ITERS / warps / ACTIVE);
  cudaFree(d);
}

int main() {
  for (int w : {4, 8, 16, 32}) {
    run<0, 32>("ATOMS distinct banks", w);
    run<1, 32>("ATOMS random in 1690", w);
    run<1, 8>("ATOMS random in 1690", w);
    run<5, 32>("ATOMS 8 hot cells", w);
    run<2, 32>("lane-private LDS+STS RMW", w);
    run<3, 32>("MATCH.ANY 6-bit key", w);
    run<4, 32>("VOTE.ballot", w);
  }
  return 0;
}
