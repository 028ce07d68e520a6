// gemm.cu — 5th-generation tensor-core GEMMs for the backbone contractions and
// the wide ramp heads (north star (1)):
//
//     C[M, N] (bf16 or fp32) = act(A[M, K] (bf16, K-major) * W[N, K]^T (bf16) + bias[N]
//                                  [+ R[M, N] (bf16 residual, e.g. a ResNet shortcut)])
//
// W is an nn.Linear weight (out_features x in_features, row-major), so both
// operands are K-major and the whole contraction is one tcgen05 "TN" GEMM.
// Two kernels, picked per shape by the host (dispatch below):
//
// k_gemm_pair  (M > 256: BERT encoder projections, GPT-2 prefill)
//   Persistent, one CTA pair (cluster of 2, cta_group::2) per two SMs. A pair
//   owns 256 x BN output tiles (BN = 256 or 128); CTA r loads A rows
//   [m0 + 128r, +128) and W rows [n0 + BN/2 r, +BN/2) into its own half of a
//   STAGES-deep ring (TMA, SWIZZLE_128B), and the leader's single thread issues
//   tcgen05.mma.cta_group::2 M=256 over both halves. Accumulators are double
//   buffered in TMEM (2 x BN fp32 columns), so the pair's 8 epilogue warps
//   drain tile i (tcgen05.ld -> bias/activation -> bf16 -> swizzled smem ->
//   TMA store) while the tensor cores already run tile i+1.
//
// k_gemm_swap  (M <= 256: decode steps, ramp heads on a batch)
//   Weight streaming. The roles of the operands swap: W is the MMA's M side
//   (128 output features per CTA) and up to 256 activation rows are its N side
//   (32 / 64 / 128 / 256, so the weights stream once per call). The K range is split
//   over a cluster of S CTAs along x: each CTA writes its fp32 partial tile to
//   an L2-resident workspace slot, one cluster barrier (release/acquire at
//   cluster scope), then rank s sums activation rows s, s + S, ... over the S
//   slots in rank order (deterministic), adds the bias, applies the activation
//   and stores. S = 1 stores straight from the TMEM registers. One launch, no
//   second reduction kernel. (Pushing the partials through DSMEM stores
//   measured 3-4x slower end to end: ~0.15 us per column per CTA.)
//
// Both: warp 0 = TMA producer (one lane), warp 1 = TMEM allocator + MMA issuer
// (one lane), warps 2..5 = epilogue (warp w owns TMEM lanes 32*(w%4)..).
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

namespace gemm3 {

constexpr int BK = 64;  // bf16 per k-tile row = 128 B = one SWIZZLE_128B atom row
constexpr int THREADS = 192;       // swap kernel: producer, MMA, 4 epilogue warps
constexpr int PAIR_THREADS = 320;  // pair kernel: producer, MMA, 8 epilogue warps
constexpr int SMEM_LIMIT = 232448;  // 227 KB opt-in per CTA on sm_100
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;  // shared::cluster address of the pair's rank 0

enum Act { ACT_NONE = 0, ACT_GELU_ERF = 1, ACT_GELU_TANH = 2, ACT_RELU = 3 };

// implicit-GEMM convolution (k_gemm_pair<..., true>): GEMM row m = output pixel
// (n, oh, ow) of an NHWC map, k = (kh, kw, c) with 64-channel blocks
struct ConvGeom {
  int hw_out;   // Ho * Wo
  int wo;       // Wo
  int kw;       // filter width
  int cblocks;  // C / 64
  int stride, pad;
  // split-K (both the plain and the implicit GEMM): tile t covers k-tile range
  // split t / (mt * nt) and writes fp32 partials to rows split * m_pad + m of
  // the output map; ee_splitk_epilogue sums the splits in order
  int ksplit, m_pad;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// UMMA shared-memory descriptor, K-major SWIZZLE_128B: 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor: fp32 accumulate, bf16 x bf16, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// arrive on the pair leader's copy of this barrier (same smem offset, rank 0)
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                   smem_u32(bar) & PEER_MASK)
               : "memory");
}

// TMA 2D load into this CTA's smem, completion bytes on `bar` (this CTA's)
__device__ __forceinline__ void tma_load(void* smem, const CUtensorMap* map, uint64_t* bar, int x,
                                         int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
// pair form: data lands in this CTA's smem, completion bytes on the leader's barrier
__device__ __forceinline__ void tma_load_pair(void* smem, const CUtensorMap* map, uint64_t* bar,
                                              int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & PEER_MASK), "r"(x), "r"(y)
      : "memory");
}
// pair form of an im2col load (implicit-GEMM convolution): 128 consecutive
// output pixels x 64 channels of the NHWC input for filter tap (ow_off, oh_off);
// (c, w, h, n) is the input position of the first pixel's window corner
__device__ __forceinline__ void tma_load_im2col_pair(void* smem, const CUtensorMap* map, uint64_t* bar,
                                                     int c, int w, int h, int n, int ow_off, int oh_off) {
  const uint16_t ow16 = (uint16_t)ow_off, oh16 = (uint16_t)oh_off;
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & PEER_MASK), "r"(c), "r"(w), "r"(h),
      "r"(n), "h"(ow16), "h"(oh16)
      : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap* map, const void* smem, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(smem)), "r"(x), "r"(y)
               : "memory");
}

template <int CG>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t id,
                                     uint32_t acc) {
  if constexpr (CG == 1)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(id), "r"(acc));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(id), "r"(acc));
}
// MMA completion -> mbarrier arrive (cta_group::2: on both CTAs of the pair)
template <int CG>
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  if constexpr (CG == 1)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
  else
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}
template <int CG>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t cols) {
  if constexpr (CG == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  } else {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc(uint32_t base, uint32_t cols) {
  if constexpr (CG == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols));
  else
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols));
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 32 lanes x 32 consecutive fp32 columns (one TMEM row per lane); no wait
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t bf16x2(float lo, float hi) {  // RNE, lo in the low half
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// erf-GELU 0.5 x (1 + erf(z)), z = x / sqrt(2), in one branch-free chain:
// erfc(|z|) = 2^(p(|z|) - |z|^2 log2 e) with p a degree-7 fit of log2(erfcx) on
// [0, 4.5] (|z| clamped there: erfc(4.5) = 2e-10), so
//   x >= 0:  x (1 - erfc(|z|) / 2)        x < 0:  x erfc(|z|) / 2
// 13 FP ops + one MUFU.EX2 per element instead of erff's two-branch
// coefficient selects. Max relative error 6.3e-6 over |gelu| > 1e-6 (fp64
// check of this exact fp32 sequence: tools/gelu_fit.py), three orders below a
// bf16 output's rounding step. The epilogue of an N = 3072, K = 768 layer
// (BERT FFN1) is issue-bound on this function.
__device__ __forceinline__ float gelu_erf(float x) {
  const float a = fminf(fabsf(x * 0.70710678118654752f), 4.5f);
  float p = -2.045430483e-05f;
  p = fmaf(p, a, 4.882906796e-04f);
  p = fmaf(p, a, -5.237843376e-03f);
  p = fmaf(p, a, 3.395731747e-02f);
  p = fmaf(p, a, -1.525138170e-01f);
  p = fmaf(p, a, 5.256913900e-01f);
  p = fmaf(p, a, -1.628095508e+00f);
  p = fmaf(p, a, 3.896280305e-06f);
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fmaf(-a * a, 1.4426950408889634f, p)));
  const float h = 0.5f * e;
  return x * (x >= 0.f ? 1.f - h : h);  // +inf -> +inf, NaN -> NaN
}

template <int ACT>
__device__ __forceinline__ float act(float x) {
  if constexpr (ACT == ACT_GELU_ERF) return gelu_erf(x);
  if constexpr (ACT == ACT_GELU_TANH) {
    const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
    return 0.5f * x * (1.f + tanhf(u));
  }
  if constexpr (ACT == ACT_RELU) return fmaxf(x, 0.f);
  return x;
}

// ===========================================================================
// k_gemm_pair: persistent, CTA pair, 256 x BN tiles, double-buffered TMEM.
// ===========================================================================
template <int BN>
struct PairCfg {
  static constexpr int A_BYTES = 128 * BK * 2;         // this CTA's 128 rows of A
  static constexpr int B_BYTES = (BN / 2) * BK * 2;    // this CTA's BN/2 rows of W
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int EPI = 8 * 2 * 32 * 128;         // 8 warps x 2 buffers x 32 rows x 128 B
  static constexpr int BIAS = 8 * 64 * 4;              // one 64-float bias row per epilogue warp
  // dynamic = alignment slack + ring + staging + bias; ~1 KB of static barriers
  static constexpr int STAGES = std::min(8, (SMEM_LIMIT - 1024 - 1024 - EPI - BIAS) / STAGE);
  static constexpr int SMEM = 1024 + STAGES * STAGE + EPI + BIAS;
};

template <int BN, int ACT, bool OUT_BF16, bool IM2COL = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PAIR_THREADS, 1)
    k_gemm_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmR,
                const float* __restrict__ bias,
                const uint16_t* __restrict__ res, int M, int N, int K, const ConvGeom G) {
  using Cfg = PairCfg<BN>;
  constexpr int ST = Cfg::STAGES;
  constexpr int CW = OUT_BF16 ? 64 : 32;  // output columns per 128-byte staging row
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* epi_smem = smem + ST * Cfg::STAGE;
  float* bias_smem = reinterpret_cast<float*>(epi_smem + Cfg::EPI);
  __shared__ __align__(8) uint64_t full_bar[8], empty_bar[8], tfull_bar[2], tempty_bar[2];
  __shared__ __align__(8) uint64_t rbar[16];  // residual box landed: epilogue warp x staging buffer
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int mt = (M + 255) / 256, nt = (N + BN - 1) / BN;
  const int kt_n = (K + BK - 1) / BK;
  const int nsplit = G.ksplit > 1 ? G.ksplit : 1;
  const int mn = mt * nt, tiles = mn * nsplit;
  const int kpt = (kt_n + nsplit - 1) / nsplit;  // k-tiles per split (every split non-empty: host)
  // tile t -> (m tile, n tile, k-tile range, output row offset)
  auto tile_m = [&](int t) { return (t % mn) % mt; };
  auto tile_n = [&](int t) { return (t % mn) / mt; };
  auto tile_k0 = [&](int t) { return (t / mn) * kpt; };
  auto tile_k1 = [&](int t) { return min(kt_n, (t / mn) * kpt + kpt); };
  auto tile_rowoff = [&](int t) { return (t / mn) * G.m_pad; };
  const int pair = blockIdx.x >> 1, pairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmC)) : "memory");
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full_bar[s], 1);   // the leader's expect_tx; both CTAs' bytes
      mbar_init(&empty_bar[s], 1);  // one multicast MMA commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);   // one multicast MMA commit
      mbar_init(&tempty_bar[a], 16);  // the 16 epilogue warps of the pair (leader's copy used)
    }
    for (int b = 0; b < 16; ++b) mbar_init(&rbar[b], 1);  // lane 0's expect_tx
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  constexpr uint32_t TMEM_COLS = 2 * BN <= 256 ? 256 : 512;  // power of two >= 2 accumulators
  if (warp == 1) tmem_alloc<2>(&tmem_base, TMEM_COLS);
  fence_before();
  cluster_sync();
  fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer (both CTAs; bytes land on the leader's barrier)
      uint32_t it = 0;
      for (int t = pair; t < tiles; t += pairs) {
        const int m0 = tile_m(t) * 256 + (int)rank * 128;
        const int n0 = tile_n(t) * BN + (int)rank * (BN / 2);
        // implicit GEMM: the input window corner of this CTA's first output pixel
        int img = 0, hb = 0, wb = 0;
        if constexpr (IM2COL) {
          img = m0 / G.hw_out;
          const int rem = m0 - img * G.hw_out;
          const int oh = rem / G.wo;
          hb = oh * G.stride - G.pad;
          wb = (rem - oh * G.wo) * G.stride - G.pad;
        }
        for (int kt = tile_k0(t); kt < tile_k1(t); ++kt, ++it) {
          const int s = it % ST;
          mbar_wait(&empty_bar[s], ((it / ST) & 1) ^ 1);
          if (rank == 0) mbar_expect_tx(&full_bar[s], 2 * Cfg::STAGE);
          unsigned char* sa = smem + s * Cfg::STAGE;
          if constexpr (IM2COL) {
            const int tap = kt / G.cblocks, cb = kt - tap * G.cblocks;
            const int kh = tap / G.kw;
            tma_load_im2col_pair(sa, &tmA, &full_bar[s], cb * BK, wb, hb, img, tap - kh * G.kw, kh);
          } else {
            tma_load_pair(sa, &tmA, &full_bar[s], kt * BK, m0);
          }
          tma_load_pair(sa + Cfg::A_BYTES, &tmB, &full_bar[s], kt * BK, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ===== MMA issuer (leader only)
      constexpr uint32_t id = idesc(256, BN);
      uint32_t it = 0, ai = 0;
      for (int t = pair; t < tiles; t += pairs, ++ai) {
        const uint32_t a = ai & 1;
        mbar_wait(&tempty_bar[a], ((ai >> 1) & 1) ^ 1);
        fence_after();
        const uint32_t d = tmem + a * BN;
        const int k0 = tile_k0(t);
        for (int kt = k0; kt < tile_k1(t); ++kt, ++it) {
          const int s = it % ST;
          mbar_wait(&full_bar[s], (it / ST) & 1);
          fence_after();
          const uint32_t a0 = smem_u32(smem + s * Cfg::STAGE), b0 = a0 + Cfg::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma<2>(d, desc_sw128(a0 + k * 32), desc_sw128(b0 + k * 32), id, (kt != k0 || k) ? 1u : 0u);
          umma_commit<2>(&empty_bar[s]);
        }
        umma_commit<2>(&tfull_bar[a]);
      }
    }
  } else {  // ===== epilogue: warps 2..9; TMEM lane quarter q = warp % 4, column half h
    const int q = warp & 3, h = (warp - 2) >> 2;
    unsigned char* stage0 = epi_smem + (warp - 2) * 2 * 4096;  // two 32 x 128 B staging boxes
    float* bias_row = bias_smem + (warp - 2) * 64;
    uint32_t ai = 0;
    int buf = 0;
    constexpr int NCH = BN / CW;  // chunks per tile; half h takes chunks [h*NCH/2 ...)
    const int c_lo = h * (NCH / 2) * CW, c_hi = h ? BN : (NCH / 2) * CW;
    // Residual (a ResNet shortcut, bf16 output only): lane 0 TMA-loads the next
    // chunk's 32 x 64 residual box into the staging buffer that chunk will use
    // (swizzled exactly like the output this warp writes there), one chunk ahead,
    // so the residual arrives as one bulk request while this chunk drains; each
    // lane then reads its own row from shared memory and overwrites it with the
    // output. Every chunk alternates the two staging buffers.
    const bool tres = res != nullptr && OUT_BF16;
    uint64_t* rb = rbar + (warp - 2) * 2;
    uint32_t rpar = 0;  // bit b: parity of the next wait on rb[b]
    auto issue_res = [&](int t, int c0, int b) {  // lane 0
      mbar_expect_tx(&rb[b], 4096);
      tma_load(stage0 + b * 4096, &tmR, &rb[b], tile_n(t) * BN + c0,
               tile_m(t) * 256 + (int)rank * 128 + q * 32);
    };
    if (tres && pair < tiles && c_lo < c_hi && lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmR)) : "memory");
      issue_res(pair, c_lo, 0);
    }
    for (int t = pair; t < tiles; t += pairs, ++ai) {
      const uint32_t a = ai & 1;
      const int row0 = tile_m(t) * 256 + (int)rank * 128 + q * 32;
      const int n0 = tile_n(t) * BN;
      const int rowoff = tile_rowoff(t);  // split-K: this split's region of the partial map
      mbar_wait(&tfull_bar[a], (ai >> 1) & 1);
      fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + a * BN;
      if (c_lo >= c_hi) {  // a one-chunk tile (BN = 64, bf16): half 0 only releases TMEM
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tempty_bar[a]);
        continue;
      }
#pragma unroll 1
      for (int c0 = c_lo; c0 < c_hi; c0 += CW) {
        uint32_t v[CW];
        if (tres && lane == 0) {  // the next chunk's residual into the other buffer
          const bool last = c0 + CW >= c_hi;
          const int tn = last ? t + pairs : t;
          // the store that last read that buffer (two chunks ago) must be done with it
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          if (tn < tiles) issue_res(tn, last ? c_lo : c0 + CW, buf ^ 1);
        }
        if constexpr (CW == 64) {
          tmem_ld32_nowait(tbase + c0, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
          tmem_ld32_nowait(tbase + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
        } else {
          tmem_ld32_nowait(tbase + c0, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
        }
        tmem_wait_ld();
        const uint32_t sb = smem_u32(stage0 + buf * 4096 + lane * 128);
        if (tres) {  // v += residual (fp32), before the bias / activation
          mbar_wait(&rb[buf], (rpar >> buf) & 1u);
          rpar ^= 1u << buf;
#pragma unroll
          for (int c = 0; c < CW / 8; ++c) {
            uint32_t w4[4];
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(w4[0]), "=r"(w4[1]), "=r"(w4[2]), "=r"(w4[3])
                         : "r"(sb + ((c ^ (lane & 7)) << 4))
                         : "memory");
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              v[8 * c + 2 * e] = __float_as_uint(__uint_as_float(v[8 * c + 2 * e]) + __uint_as_float(w4[e] << 16));
              v[8 * c + 2 * e + 1] =
                  __float_as_uint(__uint_as_float(v[8 * c + 2 * e + 1]) + __uint_as_float(w4[e] & 0xffff0000u));
            }
          }
        }
        if (c0 + CW >= c_hi) {  // this warp's columns drained: the MMA may reuse them
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_leader(&tempty_bar[a]);
        }
        if (n0 + c0 >= N) {  // fully out of range (TMA would clip anyway)
          // with a residual every chunk alternates the buffers (its zero-filled
          // box was consumed above); without one only stored chunks do
          if (tres) buf ^= 1;
          continue;
        }
        // bias for these CW columns through a warp-private smem row, read back
        // as broadcast float4s
        float f[CW];
        if (bias) {
          const int cA = n0 + c0 + lane, cB = cA + 32;
          bias_row[lane] = cA < N ? __ldg(bias + cA) : 0.f;
          if (CW == 64) bias_row[lane + 32] = cB < N ? __ldg(bias + cB) : 0.f;
          __syncwarp();
#pragma unroll
          for (int j = 0; j < CW; j += 4) {
            const float4 b4 = *reinterpret_cast<const float4*>(bias_row + j);
            f[j] = act<ACT>(__uint_as_float(v[j]) + b4.x);
            f[j + 1] = act<ACT>(__uint_as_float(v[j + 1]) + b4.y);
            f[j + 2] = act<ACT>(__uint_as_float(v[j + 2]) + b4.z);
            f[j + 3] = act<ACT>(__uint_as_float(v[j + 3]) + b4.w);
          }
          __syncwarp();
        } else {
#pragma unroll
          for (int j = 0; j < CW; ++j) f[j] = act<ACT>(__uint_as_float(v[j]));
        }
        // the staging buffer we are about to overwrite: its store must have read it
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 8; ++c) {  // 16-byte chunk c of this row, SWIZZLE_128B position
          uint4 w;
          if constexpr (OUT_BF16) {
            w.x = bf16x2(f[8 * c + 0], f[8 * c + 1]);
            w.y = bf16x2(f[8 * c + 2], f[8 * c + 3]);
            w.z = bf16x2(f[8 * c + 4], f[8 * c + 5]);
            w.w = bf16x2(f[8 * c + 6], f[8 * c + 7]);
          } else {
            w.x = __float_as_uint(f[4 * c + 0]);
            w.y = __float_as_uint(f[4 * c + 1]);
            w.z = __float_as_uint(f[4 * c + 2]);
            w.w = __float_as_uint(f[4 * c + 3]);
          }
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sb + ((c ^ (lane & 7)) << 4)),
                       "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w)
                       : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          tma_store(&tmC, stage0 + buf * 4096, n0 + c0, rowoff + row0);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        buf ^= 1;
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  fence_before();
  cluster_sync();  // neither CTA frees TMEM / exits while the pair still uses it
  if (warp == 1) tmem_dealloc<2>(tmem, TMEM_COLS);
}

// ===========================================================================
// k_gemm_swap: C^T tiles = W (128 features) x A^T (NP <= 256 rows), split-K
// over a cluster of S CTAs, DSMEM reduction in rank order.
// ===========================================================================
template <int NP>
struct SwapCfg {
  static_assert(NP == 32 || NP == 64 || NP == 128 || NP == 256, "activation rows per CTA");
  static constexpr int W_BYTES = 128 * BK * 2;
  static constexpr int A_BYTES = NP * BK * 2;
  static constexpr int STAGE = W_BYTES + A_BYTES;
  // NP = 32: two CTAs per SM (more weight bytes in flight per SM; one CTA's
  // prologue/epilogue overlaps the other's stream)
  static constexpr int CTAS_PER_SM = NP <= 32 ? 2 : 1;
  static constexpr int STAGES_MAX = (SMEM_LIMIT / CTAS_PER_SM - 2048) / STAGE;
  static constexpr int STAGES = STAGES_MAX > 8 ? 8 : STAGES_MAX;
  static constexpr int SMEM = 1024 + STAGES * STAGE;
  static constexpr int TMEM_COLS = NP <= 32 ? 32 : NP <= 64 ? 64 : NP <= 128 ? 128 : 256;
};

template <int NP, int ACT, bool OUT_BF16>
__global__ void __launch_bounds__(THREADS, SwapCfg<NP>::CTAS_PER_SM)
    k_gemm_swap(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmA,
                const float* __restrict__ bias, const uint16_t* __restrict__ res,
                void* __restrict__ C, int M, int N, int K, int kt_per, float* __restrict__ part) {
  using Cfg = SwapCfg<NP>;
  constexpr int ST = Cfg::STAGES;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[8], empty_bar[8], done_bar;
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = gridDim.x;  // cluster size = split count (the cluster spans x)
  const int s_rank = blockIdx.x;
  const int f0 = blockIdx.y * 128;  // output features of this CTA
  const int r0 = blockIdx.z * NP;   // activation rows of this CTA
  const int rows = min(NP, M - r0);
  const int kt_n = (K + BK - 1) / BK;
  const int kt0 = s_rank * kt_per, kt1 = min(kt_n, kt0 + kt_per);
  const int nkt = max(0, kt1 - kt0);
  // this cluster's S partial tiles [S][NP cols][128 features] in the workspace
  float* cpart = part ? part + (size_t)(blockIdx.z * gridDim.y + blockIdx.y) * S * NP * 128 : nullptr;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc<1>(&tmem_base, Cfg::TMEM_COLS);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nkt; ++i) {
        const int s = i % ST;
        if (i >= ST) mbar_wait(&empty_bar[s], ((i / ST) - 1) & 1);
        unsigned char* sw = smem + s * Cfg::STAGE;
        mbar_expect_tx(&full_bar[s], Cfg::STAGE);
        tma_load(sw, &tmW, &full_bar[s], (kt0 + i) * BK, f0);
        tma_load(sw + Cfg::W_BYTES, &tmA, &full_bar[s], (kt0 + i) * BK, r0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id = idesc(128, NP);
      for (int i = 0; i < nkt; ++i) {
        const int s = i % ST;
        mbar_wait(&full_bar[s], (i / ST) & 1);
        fence_after();
        const uint32_t w0 = smem_u32(smem + s * Cfg::STAGE), a0 = w0 + Cfg::W_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          umma<1>(tmem, desc_sw128(w0 + k * 32), desc_sw128(a0 + k * 32), id, (i | k) ? 1u : 0u);
        umma_commit<1>(&empty_bar[s]);
      }
      umma_commit<1>(&done_bar);
    }
  } else {
    // epilogue warps: TMEM lane = feature f0 + 32q + lane (fixed per thread),
    // TMEM column = activation row. S == 1: bias + activation + store straight
    // from the registers; S > 1: the fp32 partial goes to this rank's slot of
    // the cluster's workspace tile (lanes on consecutive features: 128-byte
    // coalesced stores, L2-resident).
    const int q = warp & 3;
    const int feat = q * 32 + lane;
    const int f = f0 + feat;
    const float bf = (S == 1 && bias && f < N) ? __ldg(bias + f) : 0.f;
    if (nkt > 0) mbar_wait(&done_bar, 0);
    fence_after();
#pragma unroll 1
    for (int c0 = 0; c0 < rows; c0 += 32) {
      uint32_t v[32];
      if (nkt > 0) {
        tmem_ld32_nowait(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0u;
      }
      if (S == 1) {
        if (f < N) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < rows) {
              const int64_t o = (int64_t)(r0 + c0 + j) * N + f;
              const float rr = res ? __uint_as_float((uint32_t)__ldg(res + o) << 16) : 0.f;
              const float y = act<ACT>((__uint_as_float(v[j]) + rr) + bf);
              if constexpr (OUT_BF16)
                static_cast<uint16_t*>(C)[o] = (uint16_t)(bf16x2(y, 0.f) & 0xFFFFu);
              else
                static_cast<float*>(C)[o] = y;
            }
        }
      } else {
        float* dst = cpart + ((size_t)s_rank * NP + c0) * 128 + feat;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c0 + j < rows) dst[j * 128] = __uint_as_float(v[j]);
      }
    }
  }
  if (S > 1) {
    // all S partials of this cluster are in L2 (release/acquire at cluster
    // scope orders the global stores); rank s then reduces activation rows
    // s, s + S, ... in rank order (deterministic), adds the bias, applies the
    // activation and stores (consecutive threads: consecutive features)
    cluster_sync();
    // float4 groups of 4 features, two groups per thread per round: up to 2 x S
    // independent 16-byte L2 loads in flight before the first add
    const int mine = (rows - s_rank + S - 1) / S;
    const int groups = mine * 32;
    for (int g0 = threadIdx.x; g0 < groups; g0 += 2 * THREADS) {
      float4 xs[2][8];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int g = g0 + u * THREADS;
        const int col = s_rank + (g >> 5) * S;
        const float4* src = reinterpret_cast<const float4*>(cpart + (size_t)col * 128 + (g & 31) * 4);
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (g < groups && r < S) xs[u][r] = __ldcg(src + (size_t)r * NP * 32);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int g = g0 + u * THREADS;
        if (g >= groups) continue;
        const int col = s_rank + (g >> 5) * S;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (r < S) {  // rank order: deterministic
            acc.x += xs[u][r].x;
            acc.y += xs[u][r].y;
            acc.z += xs[u][r].z;
            acc.w += xs[u][r].w;
          }
        const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
        const int fb = f0 + (g & 31) * 4;
        const int64_t o = (int64_t)(r0 + col) * N + fb;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (fb + e >= N) break;
          const float rr = res ? __uint_as_float((uint32_t)__ldg(res + o + e) << 16) : 0.f;
          const float y = act<ACT>((a4[e] + rr) + (bias ? __ldg(bias + fb + e) : 0.f));
          if constexpr (OUT_BF16)
            static_cast<uint16_t*>(C)[o + e] = (uint16_t)(bf16x2(y, 0.f) & 0xFFFFu);
          else
            static_cast<float*>(C)[o + e] = y;
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<1>(tmem, Cfg::TMEM_COLS);
}

}  // namespace gemm3

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// row-major [rows, cols] tensor, box {box_cols, box_rows}, 128-byte swizzle
bool make_map(CUtensorMap* m, const void* ptr, CUtensorMapDataType dt, int esize, int64_t rows,
              int64_t cols, int box_cols, int box_rows) {
  auto enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * esize};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

PFN_cuTensorMapEncodeIm2col_v12000 encoder_im2col() {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(p);
  });
  return fn;
}

// im2col view of an NHWC bf16 map [n, h, w, c] for a kh x kw / stride / pad
// convolution: each load is 128 consecutive output pixels (w fastest, then h,
// then n) x 64 channels of one filter tap, zero outside the image (SWIZZLE_128B,
// the same smem layout as a 2D K-major tile)
bool make_im2col_map(CUtensorMap* m, const void* x, int n, int h, int w, int c, int kh, int kw,
                     int stride, int pad) {
  auto enc = encoder_im2col();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)c * 2, (cuuint64_t)w * c * 2, (cuuint64_t)h * w * c * 2};
  int lower[2] = {-pad, -pad};                          // (w, h)
  int upper[2] = {pad - (kw - 1), pad - (kh - 1)};      // Wo = (w + upper - lower - 1) / s + 1
  cuuint32_t estr[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
  if (enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, lower, upper,
          (cuuint32_t)gemm3::BK, 128, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  // drivers up to 13.1 mis-set one descriptor bit for tensors under 128 KB
  // (the same workaround as CUTLASS's im2col copy traits)
  int drv = 0;
  cudaDriverGetVersion(&drv);
  if (drv <= 13010 && (uint64_t)n * h * w * c * 2 < 131072)
    reinterpret_cast<uint64_t*>(m)[1] &= ~(1ull << 21);
  return true;
}

cudaError_t set_smem(const void* fn, int smem) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;  // (fn, device)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  for (auto& d : done)
    if (d.first == fn && d.second == dev) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) done.push_back({fn, dev});
  return e;
}

int device_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

// how many CTA pairs of k_gemm_pair can be resident at once (cached per kernel)
template <class Kern>
int max_pairs(Kern kern, int smem) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, int>> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const void* key = reinterpret_cast<const void*>(kern);
  {
    std::lock_guard<std::mutex> g(mu);
    for (auto& c : cache)
      if (c.first.first == key && c.first.second == dev) return c.second;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * 74, 1, 1);
  cfg.blockDim = dim3(gemm3::PAIR_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (void*)kern, &cfg) != cudaSuccess || n <= 0)
    n = device_sms() / 2;
  std::lock_guard<std::mutex> g(mu);
  cache.push_back({{key, dev}, n});
  return n;
}

template <int BN, int ACT, bool BF>
cudaError_t launch_pair(const void* a, const void* w, const float* bias, const uint16_t* res, void* c,
                        int m, int n, int k, cudaStream_t st) {
  using Cfg = gemm3::PairCfg<BN>;
  auto kern = gemm3::k_gemm_pair<BN, ACT, BF>;
  cudaError_t e = set_smem(reinterpret_cast<const void*>(kern), Cfg::SMEM);
  if (e != cudaSuccess) return e;
  CUtensorMap ta, tb, tc;
  if (!make_map(&ta, a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, m, k, gemm3::BK, 128) ||
      !make_map(&tb, w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n, k, gemm3::BK, BN / 2) ||
      !make_map(&tc, c, BF ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                BF ? 2 : 4, m, n, BF ? 64 : 32, 32))
    return cudaErrorInvalidValue;
  const int tiles = ((m + 255) / 256) * ((n + BN - 1) / BN);
  const int pairs = std::max(1, std::min(tiles, max_pairs(kern, Cfg::SMEM)));
  CUtensorMap tr = tc;  // the residual [m, n] bf16, boxed like the output
  if (res && BF && !make_map(&tr, res, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, m, n, 64, 32))
    return cudaErrorInvalidValue;
  kern<<<dim3(2 * pairs), gemm3::PAIR_THREADS, Cfg::SMEM, st>>>(ta, tb, tc, tr, bias, res, m, n, k,
                                                                 gemm3::ConvGeom{0, 0, 0, 0, 0, 0, 1, 0});
  return cudaGetLastError();
}

// split-K epilogue: y[m, n] = act(sum_s part[s * m_pad + m, n] + bias[n] (+ res[m, n]))
// in bf16, the splits summed in order (deterministic); 8 columns per thread
__global__ void k_splitk_epilogue(const float* __restrict__ part, int S, int64_t m_pad, int64_t M,
                                  int N, const float* __restrict__ bias, const uint16_t* __restrict__ res,
                                  int act, uint16_t* __restrict__ y) {
  const int nv = N / 8;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < M * nv;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = v / nv;
    const int c0 = (int)(v - m * nv) * 8;
    float f[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = 0.f;
    for (int s = 0; s < S; ++s) {
      const float4* src = reinterpret_cast<const float4*>(part + (s * m_pad + m) * N + c0);
      const float4 a = __ldcs(src), b = __ldcs(src + 1);
      f[0] += a.x, f[1] += a.y, f[2] += a.z, f[3] += a.w, f[4] += b.x, f[5] += b.y, f[6] += b.z, f[7] += b.w;
    }
    uint32_t rw[4] = {0u, 0u, 0u, 0u};
    if (res) {
      const uint4 r4 = *reinterpret_cast<const uint4*>(res + m * N + c0);
      rw[0] = r4.x, rw[1] = r4.y, rw[2] = r4.z, rw[3] = r4.w;
    }
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float lo = f[2 * e] + (res ? __uint_as_float(rw[e] << 16) : 0.f);
      float hi = f[2 * e + 1] + (res ? __uint_as_float(rw[e] & 0xffff0000u) : 0.f);
      if (bias) lo += __ldg(bias + c0 + 2 * e), hi += __ldg(bias + c0 + 2 * e + 1);
      if (act == gemm3::ACT_RELU) lo = fmaxf(lo, 0.f), hi = fmaxf(hi, 0.f);
      o[e] = gemm3::bf16x2(lo, hi);
    }
    *reinterpret_cast<uint4*>(y + m * N + c0) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// Few output tiles over a long K (late layers of a small batch): split K so the
// tiles x splits fill the SM pairs (fp32 partials, then one epilogue pass), when
// at least 3 splits fit (below that the extra pass costs what the split saves)
int conv_splits(int m, int cout, int k, int bn, int avail) {
  const int tiles = ((m + 255) / 256) * ((cout + bn - 1) / bn);
  const int kt_n = (k + gemm3::BK - 1) / gemm3::BK;
  if (kt_n < 12 || tiles * 3 > avail) return 1;
  int S = std::min({avail / tiles, kt_n / 4, 8});
  const int kpt = (kt_n + S - 1) / S;
  S = (kt_n + kpt - 1) / kpt;  // no empty split
  return S >= 3 ? S : 1;
}

template <int BN, int ACT>
cudaError_t launch_conv(const void* x, const void* w, const float* bias, const uint16_t* res, void* y,
                        int n, int h, int wd, int c, int cout, int kh, int kw, int stride, int pad,
                        void* work, size_t work_bytes, cudaStream_t st) {
  using Cfg = gemm3::PairCfg<BN>;
  const int ho = (h + 2 * pad - kh) / stride + 1, wo = (wd + 2 * pad - kw) / stride + 1;
  const int m = n * ho * wo, k = kh * kw * c;
  const int mt = (m + 255) / 256, tiles = mt * ((cout + BN - 1) / BN);
  const int S = conv_splits(m, cout, k, BN, device_sms() / 2);
  CUtensorMap ta, tb, tc;
  if (!make_im2col_map(&ta, x, n, h, wd, c, kh, kw, stride, pad) ||
      !make_map(&tb, w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, cout, k, gemm3::BK, BN / 2))
    return cudaErrorInvalidValue;
  const gemm3::ConvGeom g{ho * wo, wo, kw, c / gemm3::BK, stride, pad, S, mt * 256};
  if (S == 1) {
    auto kern = gemm3::k_gemm_pair<BN, ACT, true, true>;
    cudaError_t e = set_smem(reinterpret_cast<const void*>(kern), Cfg::SMEM);
    if (e != cudaSuccess) return e;
    if (!make_map(&tc, y, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, m, cout, 64, 32)) return cudaErrorInvalidValue;
    const int pairs = std::max(1, std::min(tiles, max_pairs(kern, Cfg::SMEM)));
    CUtensorMap tr = tc;
    if (res && !make_map(&tr, res, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, m, cout, 64, 32))
      return cudaErrorInvalidValue;
    kern<<<dim3(2 * pairs), gemm3::PAIR_THREADS, Cfg::SMEM, st>>>(ta, tb, tc, tr, bias, res, m, cout, k, g);
    return cudaGetLastError();
  }
  auto kern = gemm3::k_gemm_pair<BN, 0, false, true>;  // fp32 partials, no epilogue math
  cudaError_t e = set_smem(reinterpret_cast<const void*>(kern), Cfg::SMEM);
  if (e != cudaSuccess) return e;
  // the caller's workspace (ee_conv_workspace_size bytes)
  float* part = static_cast<float*>(work);
  const size_t part_b = (size_t)S * mt * 256 * cout * 4;
  if (!part || work_bytes < part_b) return cudaErrorInvalidValue;
  if (!make_map(&tc, part, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (int64_t)S * mt * 256, cout, 32, 32))
    return cudaErrorInvalidValue;
  const int pairs = std::max(1, std::min(tiles * S, max_pairs(kern, Cfg::SMEM)));
  kern<<<dim3(2 * pairs), gemm3::PAIR_THREADS, Cfg::SMEM, st>>>(ta, tb, tc, tc, nullptr, nullptr, m, cout, k, g);
  e = cudaGetLastError();
  if (e == cudaSuccess) {
    const int64_t nv = (int64_t)m * (cout / 8);
    const unsigned blocks = (unsigned)std::min<int64_t>((nv + 255) / 256, (int64_t)device_sms() * 8);
    k_splitk_epilogue<<<blocks, 256, 0, st>>>(part, S, (int64_t)mt * 256, m, cout, bias, res, ACT,
                                              static_cast<uint16_t*>(y));
    e = cudaGetLastError();
  }
  return e;
}

// how one call runs (host-side plan; the workspace query uses the same one)
struct Plan {
  bool swap = false;
  int np = 32;       // swap: activation rows per CTA (32 / 64 / 128 / 256)
  int S = 1;         // swap: split count = cluster size
  int per = 1;       // swap: k-tiles per split
  int bn = 256;      // pair: tile width
  size_t work = 0;   // swap with S > 1: fp32 partial tiles
};

int pick_bn(int m, int n, int pairs);

Plan make_plan(int m, int n, int k, int splits, int path, bool bf) {
  Plan p;
  // TMA stores need 16-byte output rows; otherwise (e.g. the 50257-wide LM
  // head) the swap kernel's plain stores take any shape
  const bool c_ok = (n * (bf ? 2 : 4)) % 16 == 0;
  p.swap = path == 1 || path == 6 || (path == 0 && m <= 256) || !c_ok;
  if (!p.swap) {
    p.bn = path == 3 ? 128 : path == 2 ? 256 : path == 4 ? 192 : path == 5 ? 64 : pick_bn(m, n, device_sms() / 2);
    return p;
  }
  // one z tile up to 256 rows (the weights stream once per call), unless the
  // output is wide enough that 32-row z tiles still fit one wave at two CTAs
  // per SM: their deeper weight ring (8 stages, 2 CTAs) beats the single wider
  // tile and the repeated weight reads come from L2 (tools/sweep_np.py: M = 160,
  // N = 3072 / 4096, K = 1024: 7.7 / 10.1 us vs 8.9 / 15.1 us)
  const int ft = (n + 127) / 128;
  p.np = path == 6 ? 32 : m <= 32 ? 32 : m <= 64 ? 64 : m <= 128 ? 128 : 256;
  if (path == 0 && m > 64 && ft >= 16 && ((m + 31) / 32) * ft <= 2 * device_sms()) p.np = 32;
  const int zt = (m + p.np - 1) / p.np;
  const int kt_n = (k + gemm3::BK - 1) / gemm3::BK;
  int S = splits;
  if (S <= 0) {  // the largest power of two with <= ~96 CTAs in all, S <= 8 and
                 // >= 2 k-tiles per split: the measured optimum on B200
                 // (tools/sweep_swap.py); beyond it the reduction and the
                 // per-CTA latency chain cost more than the shorter K loop saves
    S = 1;
    while (S * 2 * ft * zt <= 96 && S * 2 <= 8 && S * 2 * 2 <= kt_n) S *= 2;
  }
  S = std::max(1, std::min({S, 8, kt_n}));  // the reduction keeps <= 8 partials in registers
  p.per = (kt_n + S - 1) / S;
  p.S = (kt_n + p.per - 1) / p.per;  // no empty split
  if (p.S > 1) p.work = (size_t)p.S * ft * zt * p.np * 128 * 4;
  return p;
}

template <int NP, int ACT, bool BF>
cudaError_t launch_swap(const Plan& p, const void* a, const void* w, const float* bias,
                        const uint16_t* res, void* c, int m, int n, int k, void* work, cudaStream_t st) {
  using Cfg = gemm3::SwapCfg<NP>;
  auto kern = gemm3::k_gemm_swap<NP, ACT, BF>;
  cudaError_t e = set_smem(reinterpret_cast<const void*>(kern), Cfg::SMEM);
  if (e != cudaSuccess) return e;
  CUtensorMap tw, ta;
  if (!make_map(&tw, w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n, k, gemm3::BK, 128) ||
      !make_map(&ta, a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, m, k, gemm3::BK, NP))
    return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.S, (n + 127) / 128, (m + NP - 1) / NP);
  cfg.blockDim = dim3(gemm3::THREADS, 1, 1);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.S;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (p.S == 1 || work)
    return cudaLaunchKernelEx(&cfg, kern, tw, ta, bias, res, c, m, n, k, p.per, (float*)work);
  // no caller workspace: stream-ordered pool memory (capturable: inside a CUDA
  // graph it becomes an allocation node)
  float* part = nullptr;
  e = cudaMallocAsync(reinterpret_cast<void**>(&part), p.work, st);
  if (e != cudaSuccess) return e;
  e = cudaLaunchKernelEx(&cfg, kern, tw, ta, bias, res, c, m, n, k, p.per, part);
  cudaError_t e2 = cudaFreeAsync(part, st);
  return e != cudaSuccess ? e : e2;
}

// 256 x BN tiles: waves x the measured relative cost of one tile of that width
// (B200, K-bound tiles: a 128-wide tile costs 0.76 of a 256-wide one, a
// 192-wide one 0.853: the narrower MMAs leave the tensor pipe partly idle);
// ties go to the wider tile
int pick_bn(int m, int n, int pairs) {
  const int bns[4] = {256, 192, 128, 64};
  const double rel[4] = {1.0, 0.853, 0.76, 0.6};
  int best = 256;
  double best_cost = 1e30;
  for (int i = 0; i < (n <= 64 ? 4 : 3); ++i) {
    const int64_t tiles = (int64_t)((m + 255) / 256) * ((n + bns[i] - 1) / bns[i]);
    const double cost = (double)((tiles + pairs - 1) / pairs) * rel[i];
    if (cost < best_cost * 0.97) best = bns[i], best_cost = cost;
  }
  return best;
}

template <int ACT, bool BF>
cudaError_t dispatch(const Plan& p, const void* a, const void* w, const float* bias,
                     const uint16_t* res, void* c, int m, int n, int k, void* work, cudaStream_t st) {
  if (p.swap) {
    if (p.np == 32) return launch_swap<32, ACT, BF>(p, a, w, bias, res, c, m, n, k, work, st);
    if (p.np == 64) return launch_swap<64, ACT, BF>(p, a, w, bias, res, c, m, n, k, work, st);
    if (p.np == 128) return launch_swap<128, ACT, BF>(p, a, w, bias, res, c, m, n, k, work, st);
    return launch_swap<256, ACT, BF>(p, a, w, bias, res, c, m, n, k, work, st);  // z tiles of 256 rows
  }
  if (p.bn == 256) return launch_pair<256, ACT, BF>(a, w, bias, res, c, m, n, k, st);
  if (p.bn == 192) return launch_pair<192, ACT, BF>(a, w, bias, res, c, m, n, k, st);
  if (p.bn == 64) return launch_pair<64, ACT, BF>(a, w, bias, res, c, m, n, k, st);
  return launch_pair<128, ACT, BF>(a, w, bias, res, c, m, n, k, st);
}

}  // namespace

// Implicit-GEMM convolution entry (ee_conv_bf16, eeb200.cu): NHWC bf16 x
// [n, h, w, c], weight [cout, kh, kw, c], y [n, ho, wo, cout] = act(conv + bias
// (+ res)); c % 64 == 0, cout % 8 == 0, act 0 or 3.
size_t ee_conv3_workspace(int n, int h, int wd, int c, int cout, int kh, int kw, int stride, int pad) {
  const int ho = (h + 2 * pad - kh) / stride + 1, wo = (wd + 2 * pad - kw) / stride + 1;
  const int m = n * ho * wo;
  const int bn = pick_bn(m, cout, device_sms() / 2);
  const int S = conv_splits(m, cout, kh * kw * c, bn, device_sms() / 2);
  return S > 1 ? (size_t)S * ((m + 255) / 256) * 256 * cout * 4 : 0;
}

cudaError_t ee_conv3_launch(const void* x, const void* w, const float* bias, const void* res, void* y,
                            int n, int h, int wd, int c, int cout, int kh, int kw, int stride, int pad,
                            int act, void* work, size_t work_bytes, cudaStream_t st) {
  const auto* r = static_cast<const uint16_t*>(res);
  const int ho = (h + 2 * pad - kh) / stride + 1, wo = (wd + 2 * pad - kw) / stride + 1;
  const int bn = pick_bn(n * ho * wo, cout, device_sms() / 2);
  if (act == 3) {
    if (bn == 256) return launch_conv<256, 3>(x, w, bias, r, y, n, h, wd, c, cout, kh, kw, stride, pad, work, work_bytes, st);
    if (bn == 192) return launch_conv<192, 3>(x, w, bias, r, y, n, h, wd, c, cout, kh, kw, stride, pad, work, work_bytes, st);
    if (bn == 64) return launch_conv<64, 3>(x, w, bias, r, y, n, h, wd, c, cout, kh, kw, stride, pad, work, work_bytes, st);
    return launch_conv<128, 3>(x, w, bias, r, y, n, h, wd, c, cout, kh, kw, stride, pad, work, work_bytes, st);
  }
  if (bn == 256) return launch_conv<256, 0>(x, w, bias, r, y, n, h, wd, c, cout, kh, kw, stride, pad, work, work_bytes, st);
  if (bn == 192) return launch_conv<192, 0>(x, w, bias, r, y, n, h, wd, c, cout, kh, kw, stride, pad, work, work_bytes, st);
  if (bn == 64) return launch_conv<64, 0>(x, w, bias, r, y, n, h, wd, c, cout, kh, kw, stride, pad, work, work_bytes, st);
  return launch_conv<128, 0>(x, w, bias, r, y, n, h, wd, c, cout, kh, kw, stride, pad, work, work_bytes, st);
}

// Internal entries used by ee_gemm_bf16_ex / ee_gemm_workspace_size
// (eeb200.cu). path: 0 auto, 1 swap-AB split-K, 2 / 4 / 3 / 5 pair with BN =
// 256 / 192 / 128 / 64 (tests pin each path).
size_t ee_gemm3_workspace(int m, int n, int k, int splits, int path, int out_bf16) {
  return make_plan(m, n, k, splits, path, out_bf16 != 0).work;
}

cudaError_t ee_gemm3_launch(const void* a, const void* w, const float* bias, const void* res, void* c,
                            int out_bf16, int act, int m, int n, int k, int splits, int path, void* work,
                            size_t work_bytes, cudaStream_t st) {
  const auto* r = static_cast<const uint16_t*>(res);
  const Plan p = make_plan(m, n, k, splits, path, out_bf16 != 0);
  if (work && work_bytes < p.work) return cudaErrorInvalidValue;
  switch (act * 2 + (out_bf16 ? 1 : 0)) {
    case 0: return dispatch<0, false>(p, a, w, bias, r, c, m, n, k, work, st);
    case 1: return dispatch<0, true>(p, a, w, bias, r, c, m, n, k, work, st);
    case 2: return dispatch<1, false>(p, a, w, bias, r, c, m, n, k, work, st);
    case 3: return dispatch<1, true>(p, a, w, bias, r, c, m, n, k, work, st);
    case 4: return dispatch<2, false>(p, a, w, bias, r, c, m, n, k, work, st);
    case 5: return dispatch<2, true>(p, a, w, bias, r, c, m, n, k, work, st);
    case 6: return dispatch<3, false>(p, a, w, bias, r, c, m, n, k, work, st);
    case 7: return dispatch<3, true>(p, a, w, bias, r, c, m, n, k, work, st);
    default: return cudaErrorInvalidValue;
  }
}
