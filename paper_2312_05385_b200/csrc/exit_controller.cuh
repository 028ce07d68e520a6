// exit_controller.cuh — fused ramp head + exit controller + batch compactor
// (north star (2)). Included by eeb200.cu.
//
// For one ramp over a batch of B rows:
//   pool   global average over HW of the ramp input (NCHW [B, C, HW] or
//          NHWC [B, HW, C]; HW = 1 means already pooled, e.g. a BERT token-0
//          hidden state)                                   fp32 accumulate
//   logits W[K, C] @ pooled + bias                          fp32
//   err    1 - max softmax  (conf = 0)                      fp32
//          or H(p) / ln K   (conf = 1, the paper's entropy rule)
//   label  argmax (first maximum, like torch.argmax)
//   exit   (double)err < threshold  — the reference exit rule, strict
//          (engine.py:207), applied only to rows still alive
// then one CTA (the last to finish) compacts the batch: surviving rows are
// listed in ascending row order (stable), and every exiting row's
// (label, err, site) is scattered to its request slot.
//
// One CTA per row; the weights stay in L2 across CTAs. For large K (ImageNet
// heads) the logits come from the tensor-core GEMM and ee_exit_from_logits
// runs the same epilogue.
#pragma once

#include <cooperative_groups.h>

namespace exitc {

namespace cg = cooperative_groups;

constexpr int THREADS = 256;
constexpr int MAXK_FUSED = 256;

struct Out {
  float* err;        // [B] per row (all rows)
  int32_t* label;    // [B]
  uint8_t* exits;    // [B] 1 = exits here
  float* logits;     // [B, K] optional
  int32_t* keep;     // [B] compacted surviving rows (ascending)
  int32_t* n_keep;   // [1]
  const int32_t* slot;  // [B] request slot of each row (nullable = identity)
  int32_t* slot_label;  // [slots] scatter targets (nullable)
  float* slot_err;
  int32_t* slot_site;
  int32_t site;
  unsigned* done;    // grid completion counter (zero on entry; the last CTA leaves it zero)
};

__device__ __forceinline__ float bf16_to_f32(uint16_t h) {
  return __uint_as_float(((uint32_t)h) << 16);
}

template <typename T>
__device__ __forceinline__ float ld_f32(const T* p, int64_t i);
template <>
__device__ __forceinline__ float ld_f32<float>(const float* p, int64_t i) {
  return __ldg(p + i);
}
template <>
__device__ __forceinline__ float ld_f32<uint16_t>(const uint16_t* p, int64_t i) {
  return bf16_to_f32(__ldg(p + i));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// softmax confidence over logits l[0..K) in shared memory (one warp)
__device__ __forceinline__ void confidence(const float* l, int K, int conf, float* err_out,
                                           int* label_out) {
  const int lane = threadIdx.x & 31;
  float mx = -INFINITY;
  int arg = 0x7fffffff;
  for (int k = lane; k < K; k += 32) {
    const float v = l[k];
    if (v > mx || (v == mx && k < arg)) {
      mx = v;
      arg = k;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, mx, o);
    const int a2 = __shfl_xor_sync(0xffffffffu, arg, o);
    if (m2 > mx || (m2 == mx && a2 < arg)) {
      mx = m2;
      arg = a2;
    }
  }
  float se = 0.f, sle = 0.f;
  for (int k = lane; k < K; k += 32) {
    const float d = l[k] - mx;
    const float e = expf(d);
    se += e;
    sle += d * e;
  }
  se = warp_sum(se);
  sle = warp_sum(sle);
  float err;
  if (conf == 0) {
    err = 1.f - 1.f / se;  // max p = exp(0) / sum
  } else {
    // H = log(sum) - sum_k d_k e_k / sum ; normalised by ln K
    const float H = logf(se) - sle / se;
    err = K > 1 ? H / logf((float)K) : 0.f;
  }
  err = fminf(fmaxf(err, 0.f), 1.f);  // err in [0, 1] (trace.py:93)
  *err_out = err;
  *label_out = arg;
}

// last CTA: stable compaction of the survivors (the exiting rows were already
// scattered to their request slots by the CTA or warp that owns the row)
__device__ void compact_and_scatter(int64_t B, const uint8_t* alive_in, const Out& o) {
  // alive_in already has this launch's exits cleared (keep = alive after the ramp)
  __shared__ int warp_tot[THREADS / 32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t r0 = 0; r0 < B; r0 += THREADS) {
    const int64_t row = r0 + threadIdx.x;
    const bool valid = row < B;
    const uint8_t ex = valid ? __ldcg(o.exits + row) : 0;
    const bool alive = valid && (alive_in ? __ldcg(alive_in + row) != 0 : true);
    const bool keep = alive && !ex;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) warp_tot[wid] = __popc(m);
    __syncthreads();
    int off = base;
    for (int w = 0; w < wid; ++w) off += warp_tot[w];
    if (keep) o.keep[off + __popc(m & ((1u << lane) - 1))] = (int32_t)row;
    __syncthreads();
    if (threadIdx.x == 0)
      for (int w = 0; w < THREADS / 32; ++w) base += warp_tot[w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *o.n_keep = base;
    *o.done = 0u;  // every other CTA has counted: ready for the next launch
  }
}

// an exiting row's (label, err, site) -> its request slot
__device__ __forceinline__ void scatter_row(const Out& o, int64_t row, int32_t label, float err) {
  if (!o.slot_label) return;
  const int32_t s = o.slot ? o.slot[row] : (int32_t)row;
  o.slot_label[s] = label;
  o.slot_err[s] = err;
  o.slot_site[s] = o.site;
}

// `arrivals` CTAs count in (default: the whole grid; the clustered head: one per row)
__device__ __forceinline__ bool last_cta(unsigned* done, unsigned arrivals = 0u) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == (arrivals ? arrivals : gridDim.x) - 1;
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// pool + FC + confidence + compare for one row per CLUSTER of S CTAs, K <= MAXK_FUSED.
// The row's HW positions are split into S contiguous slices, one per CTA of the
// cluster, so a large map (a CIFAR stem: 64 x 32 x 32 bf16 = 128 KB per row) is
// read by S SMs at once instead of one; each CTA leaves its slice's channel
// sums in its own shared memory and the cluster's rank 0 adds them over DSMEM
// in rank order (deterministic, and independent of the batch size since S
// depends on the row shape only), then runs the FC / confidence / compare.
template <typename TF, typename TW>
__global__ void __launch_bounds__(THREADS)
    k_exit_fused(const TF* __restrict__ feat, int64_t B, int C, int HW, int nhwc,
                 const TW* __restrict__ W, const float* __restrict__ bias, int K, int conf,
                 double threshold, const double* __restrict__ d_threshold,
                 uint8_t* __restrict__ alive_in, Out o, int S) {
  if (d_threshold) threshold = *d_threshold;
  extern __shared__ float sh[];  // pooled[C], logits[K]
  float* pooled = sh;
  float* logits = sh + C;
  const int64_t row = blockIdx.x / S;
  const int rank = (int)(blockIdx.x % S);
  const int p_begin = (int)((int64_t)HW * rank / S), p_end = (int)((int64_t)HW * (rank + 1) / S);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const float inv = 1.f / (float)HW;
  if ((nhwc || HW == 1) && C % 4 == 0 && C <= 4 * THREADS &&
      (reinterpret_cast<uintptr_t>(feat) & (4 * sizeof(TF) - 1)) == 0) {
    // channels contiguous: a thread owns 4 channels (one 8/16-byte load per
    // position) and the CTA's threads split the slice's positions into
    // THREADS / (C/4) sub-slices, so every thread keeps loads in flight;
    // sub-slices meet in shared memory
    __shared__ float4 part[THREADS];
    const int G = C / 4, SS = THREADS / G;
    const int g = threadIdx.x % G, sl = threadIdx.x / G;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (sl < SS) {
      const TF* base = feat + row * (int64_t)HW * C + 4 * g;
      using V = typename std::conditional<sizeof(TF) == 2, uint2, float4>::type;
      auto add = [&](const V& v) {
        if constexpr (sizeof(TF) == 2) {
          acc.x += __uint_as_float(v.x << 16);
          acc.y += __uint_as_float(v.x & 0xffff0000u);
          acc.z += __uint_as_float(v.y << 16);
          acc.w += __uint_as_float(v.y & 0xffff0000u);
        } else {
          acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
        }
      };
      // DEPTH loads issued before any is consumed; the last batch is predicated
      // (zeros for absent positions leave the fp32 sums unchanged) so a short
      // slice is one round of loads, not a dependent load per position
      constexpr int DEPTH = 8;
      for (int p = p_begin + sl; p < p_end; p += DEPTH * SS) {
        V v[DEPTH];
#pragma unroll
        for (int i = 0; i < DEPTH; ++i)
          v[i] = p + i * SS < p_end ? __ldg(reinterpret_cast<const V*>(base + (int64_t)(p + i * SS) * C)) : V{};
#pragma unroll
        for (int i = 0; i < DEPTH; ++i) add(v[i]);
      }
    }
    part[threadIdx.x] = acc;
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += THREADS) {
      const int gc = c / 4, k = c % 4;
      float t = 0.f;
      for (int q = 0; q < SS; ++q) {
        const float4 v = part[q * G + gc];
        t += k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
      }
      pooled[c] = t;
    }
  } else if (nhwc || HW == 1) {
    // channels contiguous: threads over channels, loop over positions
    const TF* base = feat + row * (int64_t)HW * C;
    for (int c = threadIdx.x; c < C; c += THREADS) {
      float acc = 0.f;
      for (int p = p_begin; p < p_end; ++p) acc += ld_f32(base, (int64_t)p * C + c);
      pooled[c] = acc;
    }
  } else if (HW <= 64) {
    // NCHW, small planes (late CNN stages, 4x4 .. 8x8): a thread per channel,
    // no per-channel warp reduction on the load-latency chain
    const TF* base = feat + row * (int64_t)C * HW;
    for (int c = threadIdx.x; c < C; c += THREADS) {
      float acc = 0.f;
      for (int p = p_begin; p < p_end; ++p) acc += ld_f32(base, (int64_t)c * HW + p);
      pooled[c] = acc;
    }
  } else {
    // NCHW: one warp per channel, lanes over the contiguous slice of the plane
    const TF* base = feat + row * (int64_t)C * HW;
    for (int c = wid; c < C; c += THREADS / 32) {
      float acc = 0.f;
      for (int p = p_begin + lane; p < p_end; p += 32) acc += ld_f32(base, (int64_t)c * HW + p);
      acc = warp_sum(acc);
      if (lane == 0) pooled[c] = acc;
    }
  }
  if (S > 1) {
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();  // every slice's sums are in its CTA's shared memory
    if (rank == 0) {
      for (int c = threadIdx.x; c < C; c += THREADS) {
        float t = pooled[c];
        for (int q = 1; q < S; ++q) t += cluster.map_shared_rank(pooled, q)[c];
        pooled[c] = t * inv;
      }
    }
    cluster.sync();  // the other ranks' shared memory stays alive until read
    if (rank != 0) return;
  } else {
    for (int c = threadIdx.x; c < C; c += THREADS) pooled[c] *= inv;
  }
  __syncthreads();
  // logits: one warp per output class, lanes over channels
  for (int k = wid; k < K; k += THREADS / 32) {
    float acc = 0.f;
    for (int c = lane; c < C; c += 32) acc += ld_f32(W, (int64_t)k * C + c) * pooled[c];
    acc = warp_sum(acc);
    if (lane == 0) logits[k] = acc + (bias ? bias[k] : 0.f);
  }
  __syncthreads();
  if (o.logits)
    for (int k = threadIdx.x; k < K; k += THREADS) o.logits[row * K + k] = logits[k];
  if (wid == 0) {
    float err;
    int label;
    confidence(logits, K, conf, &err, &label);
    if (lane == 0) {
      const bool alive = alive_in ? alive_in[row] != 0 : true;
      const bool ex = alive && (double)err < threshold;
      o.err[row] = err;
      o.label[row] = label;
      o.exits[row] = ex ? 1 : 0;
      if (ex && alive_in) alive_in[row] = 0;  // exited rows stop being alive
      if (ex) scatter_row(o, row, label, err);
    }
  }
  if (o.keep && last_cta(o.done, (unsigned)B)) compact_and_scatter(B, alive_in, o);
}

// confidence() with the row held in registers (NPL values per lane, K <= 32
// NPL): every load is issued before the first compare, instead of one L2 round
// trip per 32 logits per pass. Same per-lane order and reductions, so the same
// bits as confidence().
template <int NPL>
__device__ __forceinline__ void confidence_reg(const float* __restrict__ l, int K, int conf,
                                               float* err_out, int* label_out) {
  const int lane = threadIdx.x & 31;
  float v[NPL];
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int k = lane + 32 * i;
    v[i] = k < K ? __ldg(l + k) : 0.f;
  }
  float mx = -INFINITY;
  int arg = 0x7fffffff;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int k = lane + 32 * i;
    if (k < K && (v[i] > mx || (v[i] == mx && k < arg))) {
      mx = v[i];
      arg = k;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, mx, o);
    const int a2 = __shfl_xor_sync(0xffffffffu, arg, o);
    if (m2 > mx || (m2 == mx && a2 < arg)) {
      mx = m2;
      arg = a2;
    }
  }
  float se = 0.f, sle = 0.f;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    if (lane + 32 * i < K) {
      const float d = v[i] - mx;
      const float e = expf(d);
      se += e;
      sle += d * e;
    }
  }
  se = warp_sum(se);
  sle = warp_sum(sle);
  float err;
  if (conf == 0) {
    err = 1.f - 1.f / se;
  } else {
    const float H = logf(se) - sle / se;
    err = K > 1 ? H / logf((float)K) : 0.f;
  }
  err = fminf(fmaxf(err, 0.f), 1.f);
  *err_out = err;
  *label_out = arg;
}

// confidence + compare + compaction from precomputed logits [B, K] (fp32);
// NPL > 0: the row is held in registers (K <= 32 NPL)
template <int NPL>
__global__ void __launch_bounds__(THREADS)
    k_exit_logits(const float* __restrict__ logits_in, int64_t B, int K, int conf,
                  double threshold, const double* __restrict__ d_threshold,
                  uint8_t* __restrict__ alive_in, Out o) {
  if (d_threshold) threshold = *d_threshold;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t row = (int64_t)blockIdx.x * (THREADS / 32) + wid;  // one warp per row
  if (row < B) {
    float err;
    int label;
    if constexpr (NPL > 0)
      confidence_reg<NPL>(logits_in + row * K, K, conf, &err, &label);
    else
      confidence(logits_in + row * K, K, conf, &err, &label);
    if (lane == 0) {
      const bool alive = alive_in ? alive_in[row] != 0 : true;
      const bool ex = alive && (double)err < threshold;
      o.err[row] = err;
      o.label[row] = label;
      o.exits[row] = ex ? 1 : 0;
      if (ex && alive_in) alive_in[row] = 0;
      if (ex) scatter_row(o, row, label, err);
    }
  }
  if (o.keep && last_cta(o.done)) compact_and_scatter(B, alive_in, o);
}

// Wide heads (an LM-head ramp: K = 50257): one CTA per row, block-wide
// reductions. Same two passes and tie-breaks as confidence(): first maximum
// (label), then sum exp(l - max) and sum (l - max) exp(l - max).
constexpr int ROW_THREADS = 512;
__global__ void __launch_bounds__(ROW_THREADS)
    k_exit_logits_row(const float* __restrict__ logits_in, int64_t B, int K, int conf,
                      double threshold, const double* __restrict__ d_threshold,
                      uint8_t* __restrict__ alive_in, Out o) {
  if (d_threshold) threshold = *d_threshold;
  constexpr int NW = ROW_THREADS / 32;
  __shared__ float s_mx[NW], s_se[NW], s_sle[NW];
  __shared__ int s_arg[NW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t row = blockIdx.x;
  const float* l = logits_in + row * K;
  float mx = -INFINITY;
  int arg = 0x7fffffff;
  for (int k = threadIdx.x; k < K; k += ROW_THREADS) {
    const float v = __ldg(l + k);
    if (v > mx || (v == mx && k < arg)) {
      mx = v;
      arg = k;
    }
  }
#pragma unroll
  for (int of = 16; of; of >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, mx, of);
    const int a2 = __shfl_xor_sync(0xffffffffu, arg, of);
    if (m2 > mx || (m2 == mx && a2 < arg)) mx = m2, arg = a2;
  }
  if (lane == 0) s_mx[wid] = mx, s_arg[wid] = arg;
  __syncthreads();
  mx = s_mx[0];
  arg = s_arg[0];
  for (int w = 1; w < NW; ++w)
    if (s_mx[w] > mx || (s_mx[w] == mx && s_arg[w] < arg)) mx = s_mx[w], arg = s_arg[w];
  float se = 0.f, sle = 0.f;
  for (int k = threadIdx.x; k < K; k += ROW_THREADS) {
    const float d = __ldg(l + k) - mx;
    const float e = expf(d);
    se += e;
    sle += d * e;
  }
  se = warp_sum(se);
  sle = warp_sum(sle);
  if (lane == 0) s_se[wid] = se, s_sle[wid] = sle;
  __syncthreads();
  if (threadIdx.x == 0) {
    se = 0.f;
    sle = 0.f;
    for (int w = 0; w < NW; ++w) se += s_se[w], sle += s_sle[w];
    float err;
    if (conf == 0) {
      err = 1.f - 1.f / se;
    } else {
      const float H = logf(se) - sle / se;
      err = K > 1 ? H / logf((float)K) : 0.f;
    }
    err = fminf(fmaxf(err, 0.f), 1.f);
    const bool alive = alive_in ? alive_in[row] != 0 : true;
    const bool ex = alive && (double)err < threshold;
    o.err[row] = err;
    o.label[row] = arg;
    o.exits[row] = ex ? 1 : 0;
    if (ex && alive_in) alive_in[row] = 0;
    if (ex) scatter_row(o, row, arg, err);
  }
  if (o.keep && last_cta(o.done)) compact_and_scatter(B, alive_in, o);
}

// gather surviving rows into a dense buffer (downstream blocks skip exited rows)
__global__ void k_compact_rows(const uint8_t* __restrict__ src, int64_t row_bytes,
                               const int32_t* __restrict__ keep, const int32_t* __restrict__ n_keep,
                               uint8_t* __restrict__ dst) {
  const int64_t nk = *n_keep;
  for (int64_t r = blockIdx.x; r < nk; r += gridDim.x) {
    const uint4* s = reinterpret_cast<const uint4*>(src + (int64_t)keep[r] * row_bytes);
    uint4* d = reinterpret_cast<uint4*>(dst + r * row_bytes);
    for (int64_t q = threadIdx.x; q < row_bytes / 16; q += blockDim.x) d[q] = __ldg(s + q);
  }
}

// the survivors' bookkeeping for the next compacted stage (capacity cap rows):
// request slot of each dense row (dummy past n_keep), its alive byte, and a
// persistent copy of n_keep the host reads
__global__ void k_compact_meta(const int32_t* __restrict__ keep, const int32_t* __restrict__ n_keep,
                               const int32_t* __restrict__ rows_in, int64_t cap, int32_t dummy,
                               int32_t* __restrict__ rows_out, uint8_t* __restrict__ alive_out,
                               int32_t* __restrict__ n_out) {
  const int64_t nk = *n_keep;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x) {
    const bool live = i < nk;
    rows_out[i] = live ? (rows_in ? rows_in[keep[i]] : keep[i]) : dummy;
    alive_out[i] = live ? 1 : 0;
    if (i == 0 && n_out) *n_out = (int32_t)nk;
  }
}

// a compacted batch's ramp signals into the per-request tables (one launch for
// both, no index conversion): table[rows[i]] = value[i]
__global__ void k_scatter_signals(const float* __restrict__ err, const int32_t* __restrict__ label,
                                  const int32_t* __restrict__ rows, int64_t n, float* __restrict__ err_tab,
                                  int32_t* __restrict__ label_tab) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = rows[i];
    err_tab[s] = err[i];
    label_tab[s] = label[i];
  }
}

// In-place compaction of a batch buffer: the survivors already below n_keep
// stay where they are and only the survivors at or above n_keep move, in
// ascending order, into the exited rows' places below n_keep (ascending), so
// a batch where few rows exited moves only those few rows instead of copying
// every survivor (the stable gather of k_compact_rows). Every CTA rebuilds the
// (hole, source) pairing from `keep` in shared memory (rows <= FILL_MAX_ROWS),
// then the CTAs copy 16-byte words of the pairs' rows; CTA 0 writes the new
// row -> request slot map and alive bytes. Sources (>= n_keep) and holes
// (< n_keep) never overlap.
constexpr int FILL_MAX_ROWS = 8192;
__global__ void __launch_bounds__(256)
    k_compact_fill(uint8_t* __restrict__ buf, int64_t row_bytes, const int32_t* __restrict__ keep,
                   const int32_t* __restrict__ n_keep, int rows, const int32_t* __restrict__ rows_in,
                   int32_t dummy, int32_t* __restrict__ rows_out, uint8_t* __restrict__ alive_out,
                   int32_t* __restrict__ n_out) {
  __shared__ uint8_t mark[FILL_MAX_ROWS];
  __shared__ int16_t hole[FILL_MAX_ROWS];  // hole rank -> position (< n_keep <= FILL_MAX_ROWS)
  __shared__ int wsum[8];
  __shared__ int s_m;
  const int nk = min(*n_keep, rows);
  for (int i = threadIdx.x; i < nk; i += blockDim.x) mark[i] = 0;
  if (threadIdx.x == 0) s_m = 0;
  __syncthreads();
  int mine = 0;
  for (int t = threadIdx.x; t < nk; t += blockDim.x)
    if (keep[t] < nk) mark[keep[t]] = 1, ++mine;
  atomicAdd(&s_m, mine);
  __syncthreads();
  const int m = s_m;  // survivors below n_keep: keep[0 .. m), the rest keep[m .. nk)
  // rank the holes (positions < nk not marked), 256 positions per step
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int base = 0;
  for (int p0 = 0; p0 < nk; p0 += 256) {
    const int p = p0 + threadIdx.x;
    const bool h = p < nk && !mark[p];
    const unsigned b = __ballot_sync(0xffffffffu, h);
    if (lane == 0) wsum[wid] = __popc(b);
    __syncthreads();
    int off = base;
    for (int w = 0; w < wid; ++w) off += wsum[w];
    if (h) hole[off + __popc(b & ((1u << lane) - 1))] = (int16_t)p;
    int tot = 0;
    for (int w = 0; w < 8; ++w) tot += wsum[w];
    base += tot;
    __syncthreads();
  }
  const int npairs = nk - m;
  if (blockIdx.x == 0) {
    // new order: position p < nk holds p itself (a survivor) or the source its hole got
    for (int p = threadIdx.x; p < rows; p += blockDim.x) {
      if (p < nk) {
        rows_out[p] = rows_in ? rows_in[p] : p;
        alive_out[p] = 1;
      } else {
        rows_out[p] = dummy;
        alive_out[p] = 0;
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < npairs; t += blockDim.x) {
      const int src = keep[m + t];
      rows_out[hole[t]] = rows_in ? rows_in[src] : src;
    }
    if (threadIdx.x == 0 && n_out) *n_out = nk;
  }
  // the copies: (pair, 16-byte word) items over the whole grid
  const int64_t words = row_bytes / 16;
  const int64_t items = (int64_t)npairs * words;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(it / words);
    const int64_t w = it - (int64_t)t * words;
    const uint4* src = reinterpret_cast<const uint4*>(buf + (int64_t)keep[m + t] * row_bytes) + w;
    uint4* dst = reinterpret_cast<uint4*>(buf + (int64_t)hole[t] * row_bytes) + w;
    *dst = __ldcs(src);
  }
}

}  // namespace exitc
