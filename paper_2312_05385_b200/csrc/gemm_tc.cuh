// gemm_tc.cuh — 5th-generation tensor-core GEMM (tcgen05.mma, TMEM
// accumulators) for ramp heads: C[M, N] (fp32) = A[M, K] (bf16, K-major) *
// B[N, K]^T (bf16, K-major) + bias[N]. Included by eeb200.cu.
//
// Per CTA: one 128 x BN output tile, accumulated in TMEM (128 lanes x BN fp32
// columns). Operands are staged in shared memory in the canonical K-major
// no-swizzle UMMA layout (8-row x 16-byte core matrices; LBO = 128 B between
// the two K-halves of an MMA, SBO = 1024 B between 8-row groups), two stages
// deep: all 128 threads load k-tile t+1 while the single elected thread's
// MMAs on k-tile t run; tcgen05.commit arrives on a per-stage mbarrier that
// guards reuse of the stage. Split-K CTAs write fp32 partial tiles that a
// second pass sums in fixed order, so results are deterministic.
#pragma once

namespace gemmtc {

constexpr int BM = 128;
constexpr int BK = 64;  // bf16 elements per k-tile (128 bytes per row)
constexpr int THREADS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (layout type 0),
// version 1 (sm_100): start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// instruction descriptor: F32 accumulate, BF16 x BF16, both K-major, M x N
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4)                       // c_format = F32
         | (1u << 7)                     // a_format = BF16
         | (1u << 10)                    // b_format = BF16
         | ((uint32_t)(N >> 3) << 17)    // n_dim
         | ((uint32_t)(M >> 4) << 24);   // m_dim
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

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = __uint_as_float(r[q]);
}

// canonical no-swizzle K-major offset of element (row, k) inside a tile
__device__ __forceinline__ uint32_t tile_off(int row, int kchunk) {
  return (uint32_t)((row >> 3) * 1024 + kchunk * 128 + (row & 7) * 16);
}

// stage a ROWS x BK bf16 tile (rows row0.., k-cols k0..) into shared memory;
// rows >= nrows and columns >= K are zero-filled
template <int ROWS>
__device__ __forceinline__ void load_tile(const uint16_t* __restrict__ g, int64_t ld, int row0,
                                          int nrows, int k0, int K, unsigned char* s) {
  constexpr int CHUNKS = ROWS * (BK / 8);  // 16-byte chunks
  for (int c = threadIdx.x; c < CHUNKS; c += THREADS) {
    const int row = c >> 3, q = c & 7;
    const int gr = row0 + row, gk = k0 + q * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (gr < nrows) {
      if (gk + 8 <= K) {
        v = __ldg(reinterpret_cast<const uint4*>(g + (int64_t)gr * ld + gk));
      } else if (gk < K) {
        uint16_t tmp[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) tmp[e] = gk + e < K ? g[(int64_t)gr * ld + gk + e] : 0;
        v = *reinterpret_cast<uint4*>(tmp);
      }
    }
    *reinterpret_cast<uint4*>(s + tile_off(row, q)) = v;
  }
}

template <int BN>
__global__ void __launch_bounds__(THREADS, 1)
    k_gemm_bf16(const uint16_t* __restrict__ A, const uint16_t* __restrict__ B,
                const float* __restrict__ bias, float* __restrict__ C, int M, int N, int K,
                int k_tiles_per_split, float* __restrict__ partials) {
  constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sA[2] = {smem, smem + A_BYTES + B_BYTES};
  unsigned char* sB[2] = {smem + A_BYTES, smem + 2 * A_BYTES + B_BYTES};
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int split = blockIdx.z;
  const int kt_total = (K + BK - 1) / BK;
  const int kt0 = split * k_tiles_per_split;
  const int kt1 = min(kt_total, kt0 + k_tiles_per_split);

  if (warp == 0) {  // one warp owns TMEM: BN fp32 columns x 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  constexpr uint32_t idesc = make_idesc(BM, BN);

  uint32_t phase[2] = {0, 0};
  if (kt0 < kt1) {
    load_tile<BM>(A, K, m0, M, kt0 * BK, K, sA[0]);
    load_tile<BN>(B, K, n0, N, kt0 * BK, K, sB[0]);
  }
  for (int kt = kt0; kt < kt1; ++kt) {
    const int st = (kt - kt0) & 1;
    // make this thread's generic-proxy smem writes visible to the tensor core
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = smem_u32(sA[st]), b0 = smem_u32(sB[st]);
#pragma unroll
      for (int s = 0; s < BK / 16; ++s) {
        const uint64_t da = make_desc(a0 + s * 256, 128, 1024);
        const uint64_t db = make_desc(b0 + s * 256, 128, 1024);
        umma_bf16(tmem, da, db, idesc, (kt > kt0 || s > 0) ? 1u : 0u);
      }
      umma_commit(&mbar[st]);  // arrives when these MMAs have read the stage
    }
    // overlap: stage the next k-tile into the other buffer while the MMAs run
    if (kt + 1 < kt1) {
      const int nx = st ^ 1;
      if (kt > kt0) {  // the other stage was last read by k-tile kt-1's MMAs
        mbar_wait(&mbar[nx], phase[nx]);
        phase[nx] ^= 1;
      }
      load_tile<BM>(A, K, m0, M, (kt + 1) * BK, K, sA[nx]);
      load_tile<BN>(B, K, n0, N, (kt + 1) * BK, K, sB[nx]);
    }
  }
  // wait for the last commit (covers every earlier MMA)
  if (kt1 > kt0) {
    const int last = (kt1 - 1 - kt0) & 1;
    mbar_wait(&mbar[last], phase[last]);
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // epilogue: warp w reads TMEM lanes 32w..32w+31 = output rows m0+32w+lane
  const int row = m0 + warp * 32 + lane;
  float* dst = partials ? partials + ((int64_t)split * M) * N : C;
  for (int c0 = 0; c0 < BN; c0 += 8) {
    float v[8];
    if (kt1 > kt0) {
      tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = 0.f;
    }
    if (row < M) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int col = n0 + c0 + q;
        if (col < N) dst[(int64_t)row * N + col] = v[q] + ((!partials && bias) ? bias[col] : 0.f);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
}

// deterministic split-K reduction: C = bias + sum_s partials[s] in split order
__global__ void k_splitk_sum(const float* __restrict__ partials, int splits, int64_t MN, int N,
                             const float* __restrict__ bias, float* __restrict__ C) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < MN;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < splits; ++s) acc += partials[(int64_t)s * MN + i];
    C[i] = acc + (bias ? bias[i % N] : 0.f);
  }
}

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

}  // namespace gemmtc
