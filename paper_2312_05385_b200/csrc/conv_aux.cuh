// conv_aux.cuh — the two NHWC passes a ResNet stem needs around the tcgen05
// GEMM. Included by eeb200.cu.
//
// k_im2col_nhwc: a convolution whose input channels are too few for the
//   implicit-GEMM kernel's 64-channel TMA im2col tiles (the 3-channel ImageNet
//   stem) gets its A operand written out once: row m = output pixel (n, oh, ow),
//   column (r, s, c) at r * seg + s * c + c (seg = kw * c rounded up to 8), zero
//   in the gaps, past kh * seg up to kp (a multiple of 64) and outside the image.
// k_maxpool_nhwc: max pooling of an NHWC bf16 map, 8 channels per 16-byte
//   vector per thread, padding = -inf (PyTorch's semantics).
#pragma once

namespace convaux {

// One CTA per output row (n, oh): the kh input rows it needs (zero rows outside
// the image, zero columns for the horizontal padding) are staged in shared
// memory. Column layout: filter row r owns the `seg`-wide segment
// [r * seg, r * seg + kw * c) (seg = kw * c rounded up to 8; the weight is laid
// out the same way, zeros in the gaps), so every 16-byte output chunk copies up
// to 8 CONTIGUOUS elements of one staged row: no division per element, and
// the wo x kp block is written as consecutive coalesced chunks.
constexpr int IM2COL_THREADS = 256;
__global__ void __launch_bounds__(IM2COL_THREADS)
    k_im2col_nhwc(const uint16_t* __restrict__ x, int h, int w, int c, int kh, int kw, int stride,
                  int pad, int ho, int wo, int kp, int seg, uint4* __restrict__ out) {
  extern __shared__ uint16_t srow[];  // [kh][wp * c], wp = w + 2 pad (padded row)
  const int wp = w + 2 * pad;
  const int rowlen = wp * c;
  const int64_t img = blockIdx.x / ho;
  const int oh = (int)(blockIdx.x - img * ho);
  for (int q = threadIdx.x; q < kh * rowlen; q += IM2COL_THREADS) {
    const int r = q / rowlen, col = q - r * rowlen;
    const int ih = oh * stride - pad + r;
    const int iw = col / c - pad;
    uint16_t v = 0;
    if (ih >= 0 && ih < h && iw >= 0 && iw < w) v = __ldg(x + ((img * h + ih) * w) * c + (int64_t)iw * c + col % c);
    srow[q] = v;
  }
  __syncthreads();
  const int chunks = kp / 8, segc = seg / 8, span = kw * c;
  uint4* dst = out + (int64_t)blockIdx.x * wo * chunks;
  for (int q = threadIdx.x; q < wo * chunks; q += IM2COL_THREADS) {
    const int ow = q / chunks, ch = q - ow * chunks;
    const int r = ch / segc, e0 = (ch - r * segc) * 8;  // filter row, first element in its segment
    uint32_t o[4] = {0u, 0u, 0u, 0u};
    if (r < kh) {
      const uint16_t* src = srow + r * rowlen + ow * stride * c + e0;
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (e0 + e < span) o[e >> 1] |= (uint32_t)src[e] << (16 * (e & 1));
    }
    dst[q] = make_uint4(o[0], o[1], o[2], o[3]);
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
