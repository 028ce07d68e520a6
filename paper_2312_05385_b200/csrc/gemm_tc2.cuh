// gemm_tc2.cuh — warp-specialized 5th-generation tensor-core GEMM for the ramp
// heads and backbone contractions (north star (1)):
//
//     C[M, N] (fp32 or bf16) = A[M, K] (bf16, K-major) * B[N, K]^T (bf16) + bias[N]
//
// The canonical sm_100 structure (blackwell_cuda_programming.md, "Anatomy"):
//   warp 0 (one lane)  TMA producer: cp.async.bulk.tensor.2d of the A and B
//                      k-tiles (64 bf16 = 128 B per row, SWIZZLE_128B) into a
//                      STAGES-deep ring; mbarrier complete_tx signals "full"
//   warp 1             TMEM allocation; one lane issues tcgen05.mma (M = 128,
//                      N = BN, K = 16 per instruction, fp32 accumulators in
//                      TMEM) and tcgen05.commit frees each stage ("empty") and
//                      finally signals the epilogue
//   warps 2..5         epilogue: tcgen05.ld 32 columns at a time from their TMEM
//                      lane quarter, bias, convert, store
// Split-K (blockIdx.z) writes fp32 partial tiles that k_splitk_sum2 adds in
// split order: results are deterministic.
#pragma once

#include <cudaTypedefs.h>

namespace gemm2 {

constexpr int BM = 128;
constexpr int BK = 64;      // bf16 elements per k-tile row = 128 B (one swizzle atom row)
constexpr int THREADS = 192;
// two CTAs per SM (~97 KB of shared memory each): one CTA's epilogue overlaps
// the other's MMAs; the epilogue staging tiles reuse the drained stage ring
template <int BN>
__host__ __device__ constexpr int stages() { return BN == 256 ? 2 : 3; }
template <int BN>
__host__ __device__ constexpr int smem_bytes() { return stages<BN>() * (BM + BN) * BK * 2 + 1024; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// sm_100 UMMA shared-memory descriptor (cute/arch/mma_sm100_desc.hpp): start >> 4
// [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46), version 1 [46,48), layout type
// [61,64) = 2 (SWIZZLE_128B). K-major SW128: 8-row atoms of 1024 B (SBO), LBO unused.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                      // LBO (ignored for swizzled K-major)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;  // SBO = 1024 B between 8-row groups
  d |= (uint64_t)1 << 46;                       // version (sm_100)
  d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
  return d;
}

// instruction descriptor: F32 accumulate, BF16 x BF16, both K-major, M x N
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
__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t id,
                                     uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint16_t f2bf(float f) {  // round to nearest even
  uint32_t u = __float_as_uint(f);
  u += 0x7FFF + ((u >> 16) & 1);
  return (uint16_t)(u >> 16);
}

template <int BN, bool OUT_BF16>
__global__ void __launch_bounds__(THREADS, 2)
    k_gemm2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
            const float* __restrict__ bias, void* __restrict__ C, int M, int N, int K,
            int k_tiles_per_split, float* __restrict__ partials) {
  constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr int STAGES = stages<BN>();
  static_assert(STAGES * STAGE_BYTES >= 4 * 32 * 33 * 4, "epilogue tiles live in the ring");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for SWIZZLE_128B
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[4], empty_bar[4], done_bar;
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kt_total = (K + BK - 1) / BK;
  const int kt0 = blockIdx.z * k_tiles_per_split;
  const int kt1 = min(kt_total, kt0 + k_tiles_per_split);
  const int nkt = kt1 - kt0;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // BN fp32 columns x 128 lanes of TMEM
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer
      for (int i = 0; i < nkt; ++i) {
        const int s = i % STAGES;
        if (i >= STAGES) mbar_wait(&empty_bar[s], ((i / STAGES) - 1) & 1);
        unsigned char* sa = smem + s * STAGE_BYTES;
        mbar_expect_tx(&full_bar[s], STAGE_BYTES);
        tma_load_2d(sa, &tmA, &full_bar[s], (kt0 + i) * BK, m0);
        tma_load_2d(sa + A_BYTES, &tmB, &full_bar[s], (kt0 + i) * BK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer
      constexpr uint32_t id = idesc(BM, BN);
      for (int i = 0; i < nkt; ++i) {
        const int s = i % STAGES;
        mbar_wait(&full_bar[s], (i / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = smem_u32(smem + s * STAGE_BYTES), b0 = a0 + A_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)  // K = 16 per MMA: 32 B along the swizzled row
          umma(tmem, desc_sw128(a0 + k * 32), desc_sw128(b0 + k * 32), id, (i | k) ? 1u : 0u);
        umma_commit(&empty_bar[s]);  // the stage is free once these MMAs have read it
      }
      umma_commit(&done_bar);  // all MMAs complete -> epilogue
    }
  } else {  // ===== epilogue: warps 2..5 own TMEM lane quarters (warp % 4)
    // TMEM holds one output row per lane; each 32 x 32 block goes through a
    // padded shared-memory tile so that a warp then writes one row per
    // instruction with consecutive lanes on consecutive columns (coalesced).
    const int q = warp & 3;
    float* stile = reinterpret_cast<float*>(smem) + q * 32 * 33;  // ring is drained by now
    const int rbase = m0 + q * 32;
    if (nkt > 0) mbar_wait(&done_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const bool partial = partials != nullptr;
    for (int c0 = 0; c0 < BN; c0 += 32) {
      if (n0 + c0 >= N) break;  // warp-uniform
      uint32_t r[32];
      if (nkt > 0) {
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + c0, r);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = 0u;
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) stile[lane * 33 + j] = __uint_as_float(r[j]);
      __syncwarp();
      const int col = n0 + c0 + lane;
      const float bv = (!partial && bias && col < N) ? __ldg(bias + col) : 0.f;
      for (int rr = 0; rr < 32; ++rr) {
        const int row = rbase + rr;
        if (row >= M) break;
        if (col < N) {
          const float v = stile[rr * 33 + lane];
          const int64_t idx = (int64_t)row * N + col;
          if (partial)
            partials[(int64_t)blockIdx.z * M * N + idx] = v;
          else if (OUT_BF16)
            static_cast<uint16_t*>(C)[idx] = f2bf(v + bv);
          else
            static_cast<float*>(C)[idx] = v + bv;
        }
      }
      __syncwarp();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
}

// deterministic split-K reduction (split order) with bias and optional bf16 output
template <bool OUT_BF16>
__global__ void k_splitk_sum2(const float* __restrict__ partials, int splits, int64_t MN, int N,
                              const float* __restrict__ bias, void* __restrict__ C) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < MN;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < splits; ++s) acc += partials[(int64_t)s * MN + i];
    acc += bias ? bias[i % N] : 0.f;
    if (OUT_BF16)
      static_cast<uint16_t*>(C)[i] = f2bf(acc);
    else
      static_cast<float*>(C)[i] = acc;
  }
}

}  // namespace gemm2
