// pool.cuh — global average pooling for the wide-head ramps (the A operand of
// the tcgen05 GEMM in gemm_tc2.cuh). Included by eeb200.cu.
#pragma once

namespace pool {

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(uint16_t v) { return __uint_as_float((uint32_t)v << 16); }

// global average pool NCHW [B, C, HW] (fp32 or bf16) -> bf16 [B, C] (GEMM A operand)
template <typename T>
__global__ void k_pool_bf16(const T* __restrict__ x, int64_t BC, int HW,
                            uint16_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t bc = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); bc < BC;
       bc += (int64_t)gridDim.x * (blockDim.x / 32)) {
    float acc = 0.f;
    for (int p = lane; p < HW; p += 32) acc += to_f32(__ldg(x + bc * HW + p));
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const float m = acc / (float)HW;
      // round to nearest even bf16
      uint32_t u = __float_as_uint(m);
      u += 0x7FFF + ((u >> 16) & 1);
      out[bc] = (uint16_t)(u >> 16);
    }
  }
}

// global average pool of a channels_last map [B, HW, C] -> bf16 [B, C]:
// CTA (b, 64-channel block); 16 x 16 threads, thread (ty, tx) sums channels
// 4 tx .. 4 tx + 3 over positions ty, ty + 16, ...; rows meet in shared memory.
template <typename T>
__global__ void __launch_bounds__(256) k_pool_nhwc(const T* __restrict__ x, int C, int HW,
                                                   uint16_t* __restrict__ out) {
  __shared__ float part[16][64 + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int b = blockIdx.y, c0 = blockIdx.x * 64 + 4 * tx;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  if (c0 < C) {
    const T* base = x + ((int64_t)b * HW) * C + c0;
    using V = typename std::conditional<sizeof(T) == 2, uint2, float4>::type;
    auto add = [&](const V& v) {
      if constexpr (sizeof(T) == 2) {
        a0 += __uint_as_float(v.x << 16);
        a1 += __uint_as_float(v.x & 0xffff0000u);
        a2 += __uint_as_float(v.y << 16);
        a3 += __uint_as_float(v.y & 0xffff0000u);
      } else {
        a0 += v.x, a1 += v.y, a2 += v.z, a3 += v.w;
      }
    };
    constexpr int DEPTH = 8;  // loads issued before any is consumed
    int p = ty;
    for (; p + (DEPTH - 1) * 16 < HW; p += DEPTH * 16) {
      V v[DEPTH];
#pragma unroll
      for (int i = 0; i < DEPTH; ++i) v[i] = __ldcs(reinterpret_cast<const V*>(base + (int64_t)(p + 16 * i) * C));
#pragma unroll
      for (int i = 0; i < DEPTH; ++i) add(v[i]);
    }
    for (; p < HW; p += 16) add(__ldcs(reinterpret_cast<const V*>(base + (int64_t)p * C)));
  }
  part[ty][4 * tx] = a0;
  part[ty][4 * tx + 1] = a1;
  part[ty][4 * tx + 2] = a2;
  part[ty][4 * tx + 3] = a3;
  __syncthreads();
  if (threadIdx.x < 64 && blockIdx.x * 64 + (int)threadIdx.x < C) {
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < 16; ++r) acc += part[r][threadIdx.x];
    uint32_t u = __float_as_uint(acc / (float)HW);
    u += 0x7FFF + ((u >> 16) & 1);  // round to nearest even bf16
    out[(int64_t)b * C + blockIdx.x * 64 + threadIdx.x] = (uint16_t)(u >> 16);
  }
}

// Small channels_last maps (HW <= 64, e.g. the 7 x 7 layer4 output of a
// ResNet-50), bf16, C % 8 == 0: a CTA covers 256 channels of one image as 32
// groups of 8 channels (one 16-byte load per position) x 8 position slices;
// every slice's loads (<= 8 positions) are in flight at once and the slices
// meet in shared memory in slice order. The generic kernel above spends
// 8192 tiny CTAs on a 256 x 2048 x 7 x 7 map with a dependent load chain each.
__global__ void __launch_bounds__(256) k_pool_nhwc_small(const uint16_t* __restrict__ x, int C, int HW,
                                                         uint16_t* __restrict__ out) {
  __shared__ float part[8][256 + 4];
  const int g = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int b = blockIdx.y, c0 = blockIdx.x * 256 + 8 * g;
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c0 < C) {
    const uint16_t* base = x + ((int64_t)b * HW) * C + c0;
    uint4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int p = sl + 8 * i;
      v[i] = p < HW ? __ldcs(reinterpret_cast<const uint4*>(base + (int64_t)p * C)) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a[2 * e] += __uint_as_float(w[e] << 16);
        a[2 * e + 1] += __uint_as_float(w[e] & 0xffff0000u);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) part[sl][8 * g + e] = a[e];
  __syncthreads();
  const int c = blockIdx.x * 256 + (int)threadIdx.x;
  if (c < C) {
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < 8; ++r) acc += part[r][threadIdx.x];
    uint32_t u = __float_as_uint(acc / (float)HW);
    u += 0x7FFF + ((u >> 16) & 1);  // round to nearest even bf16
    out[(int64_t)b * C + c] = (uint16_t)(u >> 16);
  }
}

}  // namespace pool
