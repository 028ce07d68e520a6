// conv_aux.cuh — the two NHWC passes a ResNet stem needs around the tcgen05
// GEMM. Included by eeb200.cu.
//
// k_im2col_nhwc: a convolution whose input channels are too few for the
//   implicit-GEMM kernel's 64-channel TMA im2col tiles (the 3-channel ImageNet
//   stem) gets its A operand written out once: row m = output pixel (n, oh, ow),
//   column k = (kh, kw, c) (the channels_last weight's memory order), zero past
//   kh*kw*c up to kp (a multiple of 64) and outside the image. One 16-byte chunk
//   (8 columns) per thread; the gathers hit L2 (the input is read ~kh*kw/s^2
//   times).
// k_maxpool_nhwc: max pooling of an NHWC bf16 map, 8 channels per 16-byte
//   vector per thread, padding = -inf (PyTorch's semantics).
#pragma once

namespace convaux {

__global__ void k_im2col_nhwc(const uint16_t* __restrict__ x, int h, int w, int c, int kh, int kw,
                              int stride, int pad, int ho, int wo, int64_t m, int kp,
                              uint4* __restrict__ out) {
  const int chunks = kp / 8;
  const int K = kh * kw * c;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < m * chunks;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = v / chunks;
    const int k0 = (int)(v - row * chunks) * 8;
    const int64_t img = row / ((int64_t)ho * wo);
    const int rem = (int)(row - img * ho * wo);
    const int oh = rem / wo, ow = rem - oh * wo;
    uint32_t o[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int k = k0 + e;
      if (k >= K) break;
      const int tap = k / c, ch = k - tap * c;
      const int r = tap / kw, s = tap - r * kw;
      const int ih = oh * stride - pad + r, iw = ow * stride - pad + s;
      if (ih < 0 || ih >= h || iw < 0 || iw >= w) continue;
      const uint32_t val = __ldg(x + ((img * h + ih) * w + iw) * c + ch);
      o[e >> 1] |= val << (16 * (e & 1));
    }
    out[v] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

__device__ __forceinline__ float bf_f(uint32_t w, int hi) {
  return __uint_as_float(hi ? (w & 0xffff0000u) : (w << 16));
}

__global__ void k_maxpool_nhwc(const uint4* __restrict__ x, int h, int w, int cv, int k, int stride,
                               int pad, int ho, int wo, int64_t nvec, uint4* __restrict__ out) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = v / cv;
    const int cc = (int)(v - pix * cv);
    const int64_t img = pix / ((int64_t)ho * wo);
    const int rem = (int)(pix - img * ho * wo);
    const int oh = rem / wo, ow = rem - oh * wo;
    float mx[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) mx[e] = -INFINITY;
    for (int r = 0; r < k; ++r) {
      const int ih = oh * stride - pad + r;
      if (ih < 0 || ih >= h) continue;
      for (int s = 0; s < k; ++s) {
        const int iw = ow * stride - pad + s;
        if (iw < 0 || iw >= w) continue;
        const uint4 q = __ldg(x + ((img * h + ih) * w + iw) * cv + cc);
        const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) mx[e] = fmaxf(mx[e], bf_f(qw[e >> 1], e & 1));
      }
    }
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)  // maxima of bf16 values are bf16 values: exact
      o[e] = (__float_as_uint(mx[2 * e]) >> 16) | (__float_as_uint(mx[2 * e + 1]) & 0xffff0000u);
    out[v] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace convaux
