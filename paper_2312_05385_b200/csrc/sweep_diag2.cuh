// sweep_diag2.cuh — k_diag2: the diagonal-family sweep (every candidate row
// repeats one threshold on all ramps) re-laid-out for the
// B200 memory pipes. Same difference-array algebra as k_diag
// (sweep_diag.cuh:4-18): with b_j = #{u_k <= prefix-min_j}, sample i exits at
// site j for positions b_j <= p < b_{j-1}, so every drop of b contributes
// +1 at (j, b_j) and -1 at (j, b_{j-1}) in a per-site difference array split by
// the correctness bit of that site.
//
// What changed against k_diag, from the ncu capture in profiles/ and the
// primitive costs measured by tools/micro/prims.cu on B200:
//  * Loads are warp-coalesced: lane l reads 16 B at chunk offset 16*(32k+l)
//    (4 L1 wavefronts per LDG.128 instead of 24 for a 96-byte-stride row load).
//    Each lane turns its two doubles into two 7-bit keys; keys are transposed
//    through a per-warp byte buffer so that afterwards lane s owns sample s.
//  * key(x) = #{u_k <= x} is one conflict-free LDS.32 plus one fp64 compare:
//    a 256-bin grid (one FMA, saturating F2I.U32, clamp) indexes a
//    table replicated 32 times so lane l always reads bank l. The entry holds
//    lo = #thresholds below the bin and the byte offset of the bin's own
//    threshold (or of a NaN sentinel, which every lane without one reads as a
//    broadcast), so key = lo + (u_cmp <= x) with no branch.
//  * Difference-array updates are straight-line ATOMS: lanes without a drop
//    aim at one dummy word per row (same-address lanes merge in the ATOMS
//    unit). An ATOMS costs ~2-4 SM cycles per instruction on B200 whatever
//    the active-lane count (tools/micro/prims.cu); a predicated one made ptxas
//    emit BSSY/BSYNC reconvergence around every update, and adding 0 from
//    every lane at its own cell tripled the bank conflicts.
//  * The no-exit site r needs no updates for rows whose bit r is 1 (the
//    engine always sets it, engine.py:159): its histogram is n minus the other
//    sites, and only samples with bit r = 0 feed Z(p) = #{c_r = 0, b_{r-1} > p}.
//  * Thresholds, the bin grid and the serve table travel as kernel parameters
//    and the global accumulator is left zeroed by the last CTA, so one sweep is
//    exactly one launch (no memset, no H2D copy on the stream).
// The first chunk's loads are issued before the prologue builds the tables,
// so table construction overlaps the first HBM round trip.
#pragma once

namespace diag2 {

constexpr int THREADS = 1024;
constexpr int WARPS = THREADS / 32;
constexpr int MAX_M = 127;  // distinct thresholds (7-bit keys)
constexpr int NB = 256;     // bins
constexpr int W = 128;      // positions per difference-array row (p = m is the sink)
constexpr int RMAX = 16;
constexpr int MAX_POS = 512;  // candidate -> position map carried in the parameters
constexpr int ROWB = 2 * W + 32;  // ints per site row: [p][correct] + one dummy word per lane
// global accumulator gD: u64 [RMAX + 1][W] per-position counts, one 64-bit RED
// carrying (incorrect, correct) as two 32-bit halves (site r: -Z), + corr + done
constexpr int CORR_IDX = (RMAX + 1) * W;
constexpr int ACC_WORDS = CORR_IDX + 2;
constexpr int SENT = MAX_M;                  // su[SENT] is a NaN sentinel (never <= x)
// Thresholds are replicated 16x (entry t, copy q at byte 128 t + 8 q) and lane l
// reads copy l % 16: a half-warp's 64-bit loads then hit 16 distinct bank pairs
// whatever thresholds its lanes need (one copy measured ~50 conflict wavefronts
// per warp-chunk, the largest item on the shared-memory pipe).
constexpr int SU_REP = 16;
constexpr int SU_STRIDE = SU_REP * 8;  // bytes per threshold

// dynamic shared memory layout (compile-time offsets -> immediate addressing)
constexpr int OFF_TAB = 0;                       // u32 [NB][32]: lo | (8*cmp) << 16
constexpr int OFF_SU = OFF_TAB + NB * 32 * 4;    // f64 [MAX_M + 1][SU_REP]
constexpr int OFF_KEY = OFF_SU + (MAX_M + 1) * SU_STRIDE;  // u8 [WARPS][32 R]
template <int R>
__host__ __device__ constexpr int off_d() { return OFF_KEY + WARPS * 32 * R; }
template <int R>
__host__ __device__ constexpr int sd_bytes() {  // difference rows + the last CTA's correct counts
  return (R + 1) * ROWB * 4 + R * MAX_M * 8;
}
template <int R>
__host__ __device__ constexpr int fin_bytes() {  // last CTA: hist/pr/pe [R+1][M+1], ok/acc/sav [M+1]
  return 3 * (R + 1) * (MAX_M + 1) * 8 + 3 * (MAX_M + 1) * 8;
}
template <int R>
__host__ __device__ constexpr int smem_bytes() {
  return off_d<R>() + sd_bytes<R>() + fin_bytes<R>();
}

struct Params {
  const double* s;
  const uint32_t* bits;
  int64_t n;
  long long* gD;   // [CORR_IDX + 1] zero on entry, left zero on exit
  unsigned* done;  // [2]: loops finished, merges published; zero on entry, left zero
  int64_t* hist;
  int64_t* ok;
  double* acc;
  double* sav;
  const unsigned char* pos_dev;  // used when C > MAX_POS
  int64_t C;
  double a, c0;  // bin(x) = min(cvt.rzi.u32(fma(x, a, c0)), 255), a > 0
  int m;
  double vanilla;
  double serve[RMAX + 1];
  double u[MAX_M + 1];
  uint32_t tab[NB];  // bin k: lo = #{u < bin k} | (SU_STRIDE * index of the bin's own threshold, or SENT) << 16
  unsigned char pos[MAX_POS];  // position of candidate c in u, 255 = NaN row
  unsigned long long* trace;   // optional: per-CTA %globaltimer stamps [grid][6] (profiling)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Shared by host (grid choice, single-threshold check) and device; monotone
// in x. On B200 the saturating F2I.U32 maps NaN to 2^31 (measured,
// tools/micro/cvt.cu), so after the clamp NaN shares bin 255 with +inf and
// everything above the last threshold: key m, the "never exits" key a NaN
// score must get (strict <). The host guarantees bin 255 holds no threshold
// (no +inf threshold; finite thresholds land in bins [2, 253]).
__host__ __device__ inline unsigned bin_of(double x, double a, double c0) {
#ifdef __CUDA_ARCH__
  const unsigned k = __double2uint_rz(__fma_rn(x, a, c0));
#else
  const double t = std::fma(x, a, c0);
  unsigned k;
  if (!(t == t))
    k = 2147483648u;
  else if (t <= 0.0)
    k = 0u;
  else if (t >= 4294967295.0)
    k = 4294967295u;
  else
    k = (unsigned)t;
#endif
  return k < 255u ? k : 255u;
}

// compile-time unrolled loop: the body sees j as a constant expression
template <int N, int I = 0>
struct Unroll {
  template <class F>
  __device__ __forceinline__ static void run(F&& f) {
    if constexpr (I < N) {
      f(std::integral_constant<int, I>{});
      Unroll<N, I + 1>::run(f);
    }
  }
};

// 32-bit shared-window accesses: the register part of the address stays one
// IMAD/LEA and the per-ramp row offset rides in the instruction's immediate.
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
template <int OFF>
__device__ __forceinline__ void red_shared(uint32_t a, int v) {
  asm volatile("red.shared.add.s32 [%0+%2], %1;" ::"r"(a), "r"(v), "n"(OFF) : "memory");
}

// UPD selects how a lane without a drop sits out an update: 0 = branch around
// the atomic (ptxas emits BSSY/BSYNC), 1 = aim at the lane's own dummy word
// (straight-line; dummies sit in bank = lane).
template <int R, int UPD>
__global__ void __launch_bounds__(THREADS, 1) k_diag2(const __grid_constant__ Params P) {
  static_assert(R % 2 == 0 && R >= 2 && R <= RMAX, "even R only");
  constexpr int DSTRIDE = (R + 1) * ROWB;
  constexpr int NW = (R + 3) / 4;
  constexpr int OFF_D = off_d<R>();
  extern __shared__ __align__(16) unsigned char sm[];
  const int m = P.m;
  uint32_t* stab = reinterpret_cast<uint32_t*>(sm + OFF_TAB);
  double* su = reinterpret_cast<double*>(sm + OFF_SU);
  unsigned char* skey = sm + OFF_KEY;
  int* sD = reinterpret_cast<int*>(sm + OFF_D);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned FULL = 0xffffffffu;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);

  const int64_t n = P.n;
  const int64_t nchunks = (n + 31) >> 5;
  const int64_t G = (int64_t)gridDim.x * WARPS;
  int64_t ch = (int64_t)blockIdx.x * WARPS + warp;
  double2 v[R / 2];
  uint32_t cb = 0;
  auto load = [&](int64_t c) {
    if (c >= nchunks) return;
    const int64_t s0 = c << 5;
    const double2* src = reinterpret_cast<const double2*>(P.s + s0 * R);
    if (s0 + 32 <= n) {
#pragma unroll
      for (int k = 0; k < R / 2; ++k) v[k] = __ldcs(src + k * 32 + lane);
      cb = __ldcs(P.bits + s0 + lane);
    } else {
      const int64_t npairs = (n - s0) * (R / 2);
#pragma unroll
      for (int k = 0; k < R / 2; ++k) {
        const int t = k * 32 + lane;
        v[k] = t < npairs ? __ldcs(src + t) : make_double2(INF, INF);  // key m: no events
      }
      cb = s0 + lane < n ? __ldcs(P.bits + s0 + lane) : 0u;
    }
  };
  if (P.trace && tid == 0) P.trace[blockIdx.x * 6 + 0] = gtimer();
  load(ch);  // first HBM round trip overlaps the prologue

  // ---- prologue: thresholds, the replicated bin table (built on the host), zeroed counters
  for (int i = tid; i < (MAX_M + 1) * SU_REP; i += THREADS) {
    const int t = i / SU_REP;
    su[i] = t < m ? P.u[t] : __longlong_as_double(0x7ff8000000000000LL);
  }
  for (int i = tid; i < DSTRIDE; i += THREADS) sD[i] = 0;
#pragma unroll
  for (int q = tid; q < NB * 32; q += THREADS) stab[q] = P.tab[q >> 5];  // warp-uniform LDC
  __syncthreads();

  const double pa = P.a, pc0 = P.c0;
  const uint32_t smb = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t tb = smb + OFF_TAB + (uint32_t)lane * 4;  // this lane's bank of the table
  const uint32_t sub = smb + OFF_SU + (uint32_t)(lane % SU_REP) * 8;  // this lane's copy
  const uint32_t dB = smb + OFF_D;  // 16-byte aligned: bit 2 is free for the correct column
  const uint32_t dummy = dB + 2 * W * 4 + (uint32_t)lane * 4;  // + row offset
  // key(x) = #{u_k <= x} (7 bits; garbage above bit 7 is dropped by the byte pack)
  auto keyof = [&](double x) -> uint32_t {
    uint32_t e = lds_u32(tb + bin_of(x, pa, pc0) * 128u);
    const double t = lds_f64(sub + (e >> 16));
    asm("{\n\t.reg .pred p;\n\tsetp.le.f64 p, %1, %2;\n\t@p add.u32 %0, %0, 1;\n\t}"
        : "+r"(e)
        : "d"(t), "d"(x));
    return e;
  };

  unsigned char* kb = skey + warp * 32 * R;
  unsigned corr = 0;
  if (P.trace && tid == 0) P.trace[blockIdx.x * 6 + 1] = gtimer();
  for (; ch < nchunks; ch += G) {
    __syncwarp();  // previous chunk's key reads are done
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      const uint32_t k0 = keyof(v[k].x), k1 = keyof(v[k].y);
      *reinterpret_cast<unsigned short*>(kb + 2 * (k * 32 + lane)) =
          (unsigned short)__byte_perm(k0, k1, 0x0040);
    }
    const uint32_t cbc = cb;
    load(ch + G);  // next chunk in flight while this one is counted
    __syncwarp();
    uint32_t kw[NW];
    if constexpr (R % 16 == 0) {
#pragma unroll
      for (int q = 0; q < NW / 4; ++q) {
        const uint4 t = reinterpret_cast<const uint4*>(kb + lane * R)[q];
        kw[4 * q] = t.x, kw[4 * q + 1] = t.y, kw[4 * q + 2] = t.z, kw[4 * q + 3] = t.w;
      }
    } else if constexpr (R % 8 == 0) {
#pragma unroll
      for (int q = 0; q < NW / 2; ++q) {
        const uint2 t = reinterpret_cast<const uint2*>(kb + lane * R)[q];
        kw[2 * q] = t.x, kw[2 * q + 1] = t.y;
      }
    } else if constexpr (R % 4 == 0) {
#pragma unroll
      for (int q = 0; q < NW; ++q) kw[q] = reinterpret_cast<const uint32_t*>(kb + lane * R)[q];
    } else {
#pragma unroll
      for (int q = 0; q < NW; ++q) kw[q] = 0;
#pragma unroll
      for (int h = 0; h < R / 2; ++h)
        kw[h >> 1] |= (uint32_t)reinterpret_cast<const unsigned short*>(kb + lane * R)[h]
                      << (16 * (h & 1));
    }
    // difference-array updates, straight-line: lanes without a drop hit the
    // row's dummy word (all of them the same address, which ATOMS merges)
    uint32_t prev = (uint32_t)m;
    const uint32_t cb4 = cbc << 2;
    Unroll<R>::run([&](auto jc) {
      constexpr int j = decltype(jc)::value;
      const uint32_t kj = __byte_perm(kw[j >> 2], 0, 0x4440 | (j & 3));
      const bool drop = kj < prev;
      const uint32_t b = drop ? kj : prev;
      const uint32_t rowc = ((cb4 >> j) & 4u) | dB;  // + 4 for the correct column
      if constexpr (UPD == 1) {
        red_shared<j * ROWB * 4>(drop ? rowc + 8u * b : dummy, 1);
        if constexpr (j > 0)  // j = 0: prev = m is the sink
          red_shared<j * ROWB * 4>(drop ? rowc + 8u * prev : dummy, -1);
      } else if (drop) {
        red_shared<j * ROWB * 4>(rowc + 8u * b, 1);
        if constexpr (j > 0) red_shared<j * ROWB * 4>(rowc + 8u * prev, -1);
      }
      prev = b;
    });
    const unsigned cr = (cbc >> R) & 1u;
    corr += cr;
    if (__any_sync(FULL, cr == 0u))  // Z(p) = #{c_r = 0, b_{r-1} > p}: -1 at b_{r-1}
      red_shared<R * ROWB * 4>(cr == 0u ? dB + 8u * prev : dummy, -1);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) corr += __shfl_xor_sync(FULL, corr, o);
  if (P.trace && lane == 0) atomicMax(P.trace + blockIdx.x * 6 + 2, gtimer());  // last warp out
  // Back-to-back sweeps over resident windows (EE_MODE_FLAG_RESIDENT): the next
  // sweep on the stream may be scheduled once every CTA has left its loop, so
  // its CTAs take the SMs this grid frees and stream their window while our last
  // CTA finalises. Everything before this point only reads immutable inputs;
  // every global side effect below sits after griddepcontrol.wait (= the
  // previous sweep has fully completed and its memory is visible). Both are
  // no-ops for a normal launch.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __syncthreads();
  // per-CTA counts, in place: prefix over p of this CTA's difference rows
  // (non-negative for sites < r; site r holds -Z's partial, only -1 events)
  for (int site = warp; site <= R; site += WARPS) {
    int* row = sD + site * ROWB;
    int c0 = 0, c1 = 0;
    for (int p0 = 0; p0 < m; p0 += 32) {
      const int p = p0 + lane;
      int x0 = 0, x1 = 0;
      if (p < m) {
        const int2 t = *reinterpret_cast<const int2*>(row + 2 * p);
        x0 = t.x;
        x1 = t.y;
      }
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y0 = __shfl_up_sync(FULL, x0, o), y1 = __shfl_up_sync(FULL, x1, o);
        if (lane >= o) x0 += y0, x1 += y1;
      }
      x0 += c0;
      x1 += c1;
      if (p < m) *reinterpret_cast<int2*>(row + 2 * p) = make_int2(x0, x1);
      c0 = __shfl_sync(FULL, x0, 31);
      c1 = __shfl_sync(FULL, x1, 31);
    }
  }
  __shared__ unsigned s_last;
  __shared__ unsigned long long s_corr;
  if (tid == 0) s_corr = 0;
  __syncthreads();
  if (lane == 0 && corr) atomicAdd(&s_corr, (unsigned long long)corr);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // previous sweep done: gD/done/outputs are ours
  if (tid == 0) s_last = atomicAdd(P.done, 1u) == gridDim.x - 1;  // loops finished
  if (P.trace && tid == 0) P.trace[blockIdx.x * 6 + 3] = gtimer();
  __syncthreads();
  if (!s_last) {
    // publish: (incorrect, correct) as one 64-bit RED per (site, p) — the halves
    // never carry (totals < 2^32); site r sends Z's partial negated (>= 0)
    for (int site = warp; site <= R; site += WARPS) {
      const int* row = sD + site * ROWB;
      for (int p = lane; p < m; p += 32) {
        const int2 t = *reinterpret_cast<const int2*>(row + 2 * p);
        const unsigned long long v =
            site < R ? ((unsigned long long)(uint32_t)t.x | ((unsigned long long)(uint32_t)t.y << 32))
                     : (unsigned long long)(uint32_t)(-t.x);
        if (v) atomicAdd(reinterpret_cast<unsigned long long*>(P.gD + site * W + p), v);
      }
    }
    if (tid == 0 && s_corr) atomicAdd(reinterpret_cast<unsigned long long*>(P.gD + CORR_IDX), s_corr);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    __syncthreads();
    if (tid == 0) atomicAdd(P.done + 1, 1u);  // merged
    return;
  }

  // ---- the last CTA to finish its loop: fold its own counts in from shared
  // memory (no RED / fence on the critical path), wait for the others' merges
  if (tid == 0) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(P.done + 1) : "memory");
    } while (v < gridDim.x - 1);
  }
  __syncthreads();
  if (P.trace && tid == 0) P.trace[blockIdx.x * 6 + 1] = gtimer();  // (last CTA: reuses slot 1)
  const int M1 = m + 1;  // positions + the NaN row (p = m)
  // scratch: hist i64 [R+1][M1], ok i64 [M1], pr/pe f64 [R+1][M1], acc/sav [M1]
  long long* hst = reinterpret_cast<long long*>(sm + OFF_D + sd_bytes<R>());
  long long* okp = hst + (R + 1) * M1;
  double* prs = reinterpret_cast<double*>(okp + M1);
  double* pes = prs + (R + 1) * M1;
  double* accp = pes + (R + 1) * M1;
  double* savp = accp + M1;
  long long* c1s = reinterpret_cast<long long*>(sD + (R + 1) * ROWB);  // i64 [R][m] correct counts
  __shared__ long long s_corr_all;
  if (tid == 0) {
    s_corr_all = (long long)(__ldcg(P.gD + CORR_IDX) + s_corr);
    P.gD[CORR_IDX] = 0;
    P.done[0] = 0u;
    P.done[1] = 0u;
  }
  for (int i = tid; i < (R + 1) * m; i += THREADS) {  // read, add own, zero for the next launch
    const int site = i / m, p = i - site * m;
    const unsigned long long g = (unsigned long long)__ldcg(P.gD + site * W + p);
    P.gD[site * W + p] = 0;
    const int2 own = *reinterpret_cast<const int2*>(sD + site * ROWB + 2 * p);
    if (site < R) {
      const long long c0 = (long long)(g & 0xffffffffull) + own.x;
      const long long c1 = (long long)(g >> 32) + own.y;
      hst[site * M1 + p] = c0 + c1;
      c1s[site * m + p] = c1;
    } else {
      hst[R * M1 + p] = (long long)(g & 0xffffffffull) - own.x;  // #{c_r = 0, b_{r-1} <= p}
    }
  }
  __syncthreads();
  const long long corrR = s_corr_all;
  for (int p = tid; p < M1; p += THREADS) {  // no-exit site and correct counts per position
    if (p == m) {  // NaN threshold row: nothing exits
      for (int site = 0; site < R; ++site) hst[site * M1 + p] = 0;
      hst[R * M1 + p] = n;
      okp[p] = corrR;
      continue;
    }
    long long tot = 0, okc = 0;
    for (int site = 0; site < R; ++site) {
      tot += hst[site * M1 + p];
      okc += c1s[site * m + p];
    }
    const long long hr = n - tot;
    // Z(p) = #{c_r = 0, b_{r-1} > p} = (n - corrR) - #{c_r = 0, b_{r-1} <= p}
    okc += hr - ((n - corrR) - hst[R * M1 + p]);
    hst[R * M1 + p] = hr;
    okp[p] = okc;
  }
  __syncthreads();
  for (int i = tid; i < (R + 1) * M1; i += THREADS) {  // error-free products, all in parallel
    const int site = i / M1;
    const double x = (double)hst[i];
    const double pr = __dmul_rn(x, P.serve[site]);
    prs[i] = pr;
    pes[i] = __fma_rn(x, P.serve[site], -pr);
  }
  __syncthreads();
  for (int p = tid; p < M1; p += THREADS) {  // the ordered TwoSum chain of k_finalize
    double hi = 0.0, lo = 0.0;
#pragma unroll
    for (int site = 0; site <= R; ++site) {
      double s2, e;
      two_sum(hi, prs[site * M1 + p], s2, e);
      hi = s2;
      lo = __dadd_rn(lo, __dadd_rn(e, pes[site * M1 + p]));
    }
    double tot2, e;
    two_sum(hi, lo, tot2, e);
    const double dn = (double)n;
    accp[p] = __ddiv_rn((double)okp[p], dn);
    savp[p] = __dsub_rn(P.vanilla, __ddiv_rn(tot2, dn));
  }
  __syncthreads();
  auto posof = [&](int64_t c) -> int {
    const int q = P.C <= MAX_POS ? P.pos[c] : P.pos_dev[c];
    return q == 255 ? m : q;
  };
  if (P.hist)
    for (int64_t i = tid; i < P.C * (R + 1); i += THREADS) {
      const int64_t c = i / (R + 1);
      const int site = (int)(i - c * (R + 1));
      P.hist[i] = hst[site * M1 + posof(c)];
    }
  for (int64_t c = tid; c < P.C; c += THREADS) {
    const int p = posof(c);
    if (P.ok) P.ok[c] = okp[p];
    if (P.acc) {
      P.acc[c] = accp[p];
      P.sav[c] = savp[p];
    }
  }
  if (P.trace) {
    __syncthreads();
    if (tid == 0) P.trace[blockIdx.x * 6 + 4] = gtimer();
  }
}

}  // namespace diag2
