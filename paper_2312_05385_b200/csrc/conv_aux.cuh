// conv_aux.cuh — the two NHWC passes a ResNet stem needs around the tcgen05
// GEMM. Included by eeb200.cu.
//
// k_im2col_nhwc: a convolution whose input channels are too few for the
//   implicit-GEMM kernel's 64-channel TMA im2col tiles (the 3-channel ImageNet
//   stem) gets its A operand written out once: row m = output pixel (n, oh, ow),
//   column (r, s, c) at r * seg + s * c + c (seg = kw * c rounded up to 8; the
//   gap columns meet zero weights), zero past kh * seg up to kp (a multiple of
//   8) and outside the image.
// k_maxpool_nhwc: max pooling of an NHWC bf16 map, 8 channels per 16-byte
//   vector per thread, padding = -inf (PyTorch's semantics).
#pragma once

namespace convaux {

// One CTA per output row (n, oh). The kh input rows it needs are staged in
// shared memory with 16-byte copies, each behind lp >= pad * c zero elements
// (lp a multiple of 8, so the copies stay aligned) and followed by zeros for
// the right padding; rows outside the image stay zero. Column layout of the
// output: filter row r owns the `seg`-wide segment [r * seg, r * seg + kw * c)
// (seg = kw * c rounded up to 8; the weight is laid out the same way, zero in
// the gaps), so each 16-byte output chunk is 8 CONTIGUOUS staged elements:
// five 32-bit shared loads and a funnel shift, no per-element index math. The
// gap columns pick up neighbouring (finite) staged values, which meet zero
// weights. Thread t writes chunk t % chunks of pixels t / chunks, + PIX, ...:
// consecutive threads write consecutive 16-byte chunks.
constexpr int IM2COL_THREADS = 256;
__global__ void __launch_bounds__(IM2COL_THREADS)
    k_im2col_nhwc(const uint16_t* __restrict__ x, int h, int w, int c, int kh, int kw, int stride,
                  int pad, int ho, int wo, int kp, int seg, int lp, int rowlen,
                  uint4* __restrict__ out) {
  extern __shared__ __align__(16) uint16_t srow[];  // [kh][rowlen]
  const int64_t img = blockIdx.x / ho;
  const int oh = (int)(blockIdx.x - img * ho);
  uint4* s4 = reinterpret_cast<uint4*>(srow);
  const int n4 = kh * rowlen / 8;
  for (int q = threadIdx.x; q < n4; q += IM2COL_THREADS) s4[q] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  const int v_row = w * c / 8;  // 16-byte vectors per input row
  for (int q = threadIdx.x; q < kh * v_row; q += IM2COL_THREADS) {
    const int r = q / v_row, v = q - r * v_row;
    const int ih = oh * stride - pad + r;
    if (ih < 0 || ih >= h) continue;
    const uint4* src = reinterpret_cast<const uint4*>(x + (img * h + ih) * (int64_t)w * c);
    s4[(r * rowlen + lp) / 8 + v] = __ldg(src + v);
  }
  __syncthreads();
  const int chunks = kp / 8, segc = seg / 8;
  const int PIX = IM2COL_THREADS / chunks;
  const int ci = threadIdx.x % chunks, pix0 = threadIdx.x / chunks;
  if (pix0 >= PIX) return;
  const int r = ci / segc, e0 = (ci - r * segc) * 8;
  const uint32_t* s32 = reinterpret_cast<const uint32_t*>(srow);
  const int obase = r * rowlen + lp - pad * c + e0;  // staged element of (ow = 0, this chunk)
  uint4* dst = out + (int64_t)blockIdx.x * wo * chunks + ci;
  for (int ow = pix0; ow < wo; ow += PIX) {
    uint4 o = make_uint4(0u, 0u, 0u, 0u);
    if (r < kh) {
      const int e = obase + ow * stride * c;
      const uint32_t* wp = s32 + (e >> 1);
      const uint32_t a0 = wp[0], a1 = wp[1], a2 = wp[2], a3 = wp[3];
      if (e & 1) {
        const uint32_t a4 = wp[4];
        o = make_uint4(__funnelshift_r(a0, a1, 16), __funnelshift_r(a1, a2, 16),
                       __funnelshift_r(a2, a3, 16), __funnelshift_r(a3, a4, 16));
      } else {
        o = make_uint4(a0, a1, a2, a3);
      }
    }
    dst[(int64_t)ow * chunks] = o;
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

// k_maxpool_nhwc for a fixed K x K window (the ResNet stem's 3 x 3): every tap's
// 16-byte load is issued before the first max (the generic loop above waits on
// one load per tap); taps outside the image are skipped in the same order, so
// the result is the same bits.
template <int K>
__global__ void __launch_bounds__(256) k_maxpool_nhwc_k(const uint4* __restrict__ x, int h, int w, int cv,
                                                        int stride, int pad, int ho, int wo, int64_t nvec,
                                                        uint4* __restrict__ out) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = v / cv;
    const int cc = (int)(v - pix * cv);
    const int64_t img = pix / ((int64_t)ho * wo);
    const int rem = (int)(pix - img * ho * wo);
    const int oh = rem / wo, ow = rem - oh * wo;
    uint4 q[K * K];
    bool ok[K * K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int ih = oh * stride - pad + r;
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const int iw = ow * stride - pad + s;
        ok[r * K + s] = ih >= 0 && ih < h && iw >= 0 && iw < w;
        q[r * K + s] = ok[r * K + s] ? __ldg(x + ((img * h + ih) * w + iw) * cv + cc) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
    float mx[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) mx[e] = -INFINITY;
#pragma unroll
    for (int t = 0; t < K * K; ++t) {
      const uint32_t qw[4] = {q[t].x, q[t].y, q[t].z, q[t].w};
#pragma unroll
      for (int e = 0; e < 8; ++e) mx[e] = ok[t] ? fmaxf(mx[e], bf_f(qw[e >> 1], e & 1)) : mx[e];
    }
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      o[e] = (__float_as_uint(mx[2 * e]) >> 16) | (__float_as_uint(mx[2 * e + 1]) & 0xffff0000u);
    out[v] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace convaux
