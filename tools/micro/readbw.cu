// Read-only HBM bandwidth on B200 for the sweep's access pattern: how fast can
// 97.5 MB (1M x 12 f64 + 1M u32) be streamed by 147-148 1024-thread CTAs with
// one or two 3 KB warp-chunks in flight, vs a plain grid-stride uint4 reader.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int R = 12;
template <int DEPTH>
__global__ void __launch_bounds__(1024, 1) k_chunks(const double* s, const uint32_t* bits, int64_t n, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nchunks = n >> 5, G = (int64_t)gridDim.x * 32;
  double acc = 0;
  double2 v[DEPTH][R / 2];
  uint32_t cb[DEPTH];
  int64_t ch = (int64_t)blockIdx.x * 32 + warp;
  auto load = [&](int d, int64_t c) {
    if (c >= nchunks) return;
    const double2* src = reinterpret_cast<const double2*>(s + (c << 5) * R);
#pragma unroll
    for (int k = 0; k < R / 2; ++k) v[d][k] = __ldcs(src + k * 32 + lane);
    cb[d] = __ldcs(bits + (c << 5) + lane);
  };
#pragma unroll
  for (int d = 0; d < DEPTH; ++d) load(d, ch + d * G);
  for (; ch < nchunks; ch += DEPTH * G) {
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      if (ch + d * G < nchunks) {
#pragma unroll
        for (int k = 0; k < R / 2; ++k) acc += v[d][k].x + v[d][k].y;
        acc += cb[d];
        load(d, ch + (d + DEPTH) * G);
      }
    }
  }
  if (acc == 1234.5) out[0] = acc;
}
__global__ void k_plain(const uint4* p, int64_t n16, double* out) {
  uint32_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 t = __ldcs(p + i);
    acc ^= t.x ^ t.y ^ t.z ^ t.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
int main() {
  const int64_t n = 1000000;
  const int copies = 4;
  const size_t sb = n * R * 8, bb = n * 4;
  char* base; cudaMalloc(&base, copies * (sb + bb));
  cudaMemset(base, 0, copies * (sb + bb));
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto launch) {
    for (int i = 0; i < 20; ++i) launch(i % copies);
    cudaDeviceSynchronize();
    const int K = 400;
    cudaEventRecord(a);
    for (int i = 0; i < K; ++i) launch(i % copies);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1000 / K;
    printf("%-44s %7.2f us/pass  %7.1f GB/s\n", name, us, (sb + bb) / (us * 1e-6) / 1e9);
  };
  for (int grid : {147, 148}) {
    char nm[64];
    snprintf(nm, 64, "chunks depth1 grid %d", grid);
    timeit(nm, [&](int c) { char* p = base + c * (sb + bb); k_chunks<1><<<grid, 1024>>>((double*)p, (uint32_t*)(p + sb), n, out); });
    snprintf(nm, 64, "chunks depth2 grid %d", grid);
    timeit(nm, [&](int c) { char* p = base + c * (sb + bb); k_chunks<2><<<grid, 1024>>>((double*)p, (uint32_t*)(p + sb), n, out); });
  }
  for (int g : {148, 296, 592, 1184}) {
    char nm[64]; snprintf(nm, 64, "plain uint4 grid %d x 512", g);
    timeit(nm, [&](int c) { char* p = base + c * (sb + bb); k_plain<<<g, 512>>>((const uint4*)p, (int64_t)((sb + bb) / 16), out); });
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
