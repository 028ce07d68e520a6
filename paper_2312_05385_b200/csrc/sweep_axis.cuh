// sweep_axis.cuh — the single-coordinate ("axis") candidate family in one pass:
// every candidate row equals a base vector b except in at most one column j,
// where it holds a value v from one shared sorted set V (|V| <= 64). SURVEY
// §8(d)'s C = 768 family (b = 0.3, ramp j swept over 64 points) is this shape.
//
// Per sample, with below_t = s_t < b_t (fp64, the reference's strict compare),
// f = first t with below_t and f2 = the next one (R if none): a candidate (j, v)
// exits at f when f < j; otherwise at j when s_j < v, else at g_j (g_j = f when
// f > j, f2 when f = j). With key_j = #{v in V : v <= s_j}, "s_j < v_k" is
// "key_j <= k", so per column j the k-dependence is a cumulative count over
// key_j, split by the site g_j the sample would otherwise reach:
//   hist[t < j]  = B[t]                    (B[t] = #{f = t})
//   hist[j](k)   = sum_s F_j(k, s)          (F_j(k, s) = #{f >= j, g_j = s, key_j <= k})
//   hist[s > j]  = B[s] + E[j][s] - F_j(k, s)   (E[j][s] = #{f = j, f2 = s})
//   ok(k) = sum_{t<j} Bc[t] + sum_{s>j} (Bc[s] + Ec[j][s]) + sum_s D_j(k, s)
// where Bc/Ec count the correct bit of the site reached and D_j accumulates
// c_j - c_{g_j} over the same cells as F_j. Per sample: one update of B, one of
// E, and one of (j, key_j, g_j) for every column j <= f, packed as
// count | delta << 16 (B/E: count | correct << 16) in shared memory.
//
// k_axis writes each CTA's cells to a partial buffer; k_axis_reduce sums the
// partials into 64-bit totals; k_axis_fin (one CTA per column) takes the
// prefix over keys and finalises every candidate of its column exactly as
// k_finalize does. Envelope (else the generic path): even R <= 16, |V| <= 64,
// C <= 1024, at most 32767 samples per CTA (the packed halves stay exact).
#pragma once

namespace axis {

constexpr int THREADS = 1024;
constexpr int WARPS = THREADS / 32;
constexpr int MAX_M = 64;
constexpr int CELLS = MAX_M + 1;       // keys 0..m (m: never exits at j)
constexpr int MAX_C = 1024;
constexpr int MAX_CTA_CHUNKS = 1023;   // 32-sample chunks per CTA: <= 32736 samples
constexpr int REDUCE_SPLIT = 16;       // partial-sum slices per cell in k_axis_reduce

struct Params {
  const double* s;
  const uint32_t* bits;
  int64_t n;
  uint32_t* part;  // [grid][ncell] per-CTA packed cells
  int ncell;
  double a, c0;  // bin grid of V (diag2::bin_of)
  int m;         // |V|
  double base[diag2::RMAX];
  double u[diag2::MAX_M + 1];  // V, then NaN (slot SENT)
  uint32_t tab[diag2::NB];
};

struct FinParams {
  const unsigned long long* tot_cnt;  // [ncell]
  const long long* tot_x;             // [ncell] delta (C3) or correct (B/E)
  int64_t n;
  int m;
  int64_t C;
  double vanilla;
  double serve[diag2::RMAX + 1];
  int64_t* hist;
  int64_t* ok;
  double* acc;
  double* sav;
  uint16_t code[MAX_C];  // candidate c: column << 8 | position in V (255 = NaN value)
};

// cell layout (partials and totals): C3 [R][m][R+1], then B [R+1], then E [R][R+1]
__host__ __device__ constexpr int ncell(int R, int m) { return R * m * (R + 1) + (R + 1) + R * (R + 1); }

template <int R>
struct Layout {
  static constexpr int R1 = R + 1;
  static constexpr int OFF_BASE = diag2::off_d<R>();  // after table, thresholds, key buffer
  static constexpr int OFF_C3 = OFF_BASE + diag2::RMAX * 8;
  static constexpr int OFF_B = OFF_C3 + (R * CELLS * R1 * 4 + 15) / 16 * 16;  // lane-private [R1][32]
  static constexpr int OFF_E = OFF_B + R1 * 32 * 4;          // lane-private [R][R1][32]
  static constexpr int OFF_DUM = OFF_E + R * R1 * 32 * 4;    // one dummy word per lane
  static constexpr int SMEM = OFF_DUM + 32 * 4;
};

// NANCHK: V holds +inf, which shares bin 255 with NaN, so NaN is keyed explicitly.
template <int R, bool NANCHK>
__global__ void __launch_bounds__(THREADS, 1) k_axis(const __grid_constant__ Params P) {
  static_assert(R % 2 == 0 && R >= 2 && R <= diag2::RMAX, "even R only");
  using L = Layout<R>;
  constexpr int R1 = L::R1;
  constexpr int NW = (R + 3) / 4;
  using diag2::lds_f64;
  using diag2::lds_u32;
  using diag2::Unroll;
  extern __shared__ __align__(16) unsigned char sm[];
  const int m = P.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  const int64_t n = P.n;
  const int64_t nchunks = (n + 31) >> 5;
  const int64_t c_end = (int64_t)(blockIdx.x + 1) * nchunks / gridDim.x;
  int64_t ch = (int64_t)blockIdx.x * nchunks / gridDim.x + warp;

  // parameters first (their constant-bank misses must not queue behind the window)
  const uint32_t te0 = P.tab[tid >> 3], te1 = P.tab[(tid + THREADS) >> 3];
  const int tu = tid / (diag2::SU_REP / 2);
  const double ue = tu < m ? P.u[tu] : __longlong_as_double(0x7ff8000000000000LL);
  double2 v[R / 2];
  uint32_t cb = 0;
  if (ch < c_end) {
    const int64_t s0 = ch << 5;
    const double2* src = reinterpret_cast<const double2*>(P.s + s0 * R);
    const int64_t npairs = (n - s0) * (R / 2);
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      const int t = k * 32 + lane;
      v[k] = t < npairs ? __ldcs(src + t) : make_double2(INF, INF);
    }
    cb = s0 + lane < n ? __ldcs(P.bits + s0 + lane) : 0u;
  }
  {
    uint4* t4 = reinterpret_cast<uint4*>(sm + diag2::OFF_TAB);
    t4[tid] = make_uint4(te0, te0, te0, te0);
    t4[tid + THREADS] = make_uint4(te1, te1, te1, te1);
    reinterpret_cast<double2*>(sm + diag2::OFF_SU)[tid] = make_double2(ue, ue);
    if (tid < R) reinterpret_cast<double*>(sm + L::OFF_BASE)[tid] = P.base[tid];
    uint4* z = reinterpret_cast<uint4*>(sm + L::OFF_C3);
    for (int q = tid; q < (L::OFF_DUM + 32 * 4 - L::OFF_C3) / 16; q += THREADS) z[q] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();

  const double pa = P.a, pc0 = P.c0;
  const uint32_t smb = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t tb = smb + diag2::OFF_TAB + (uint32_t)lane * 4;
  const uint32_t sub = smb + diag2::OFF_SU + (uint32_t)(lane % diag2::SU_REP) * 8;
  const uint32_t sbase = smb + L::OFF_BASE;
  const uint32_t sC3 = smb + L::OFF_C3;
  const uint32_t sB = smb + L::OFF_B + (uint32_t)lane * 4;
  const uint32_t sE = smb + L::OFF_E + (uint32_t)lane * 4;
  const uint32_t dummy = smb + L::OFF_DUM + (uint32_t)lane * 4;
  // key (7 bits) | below-base bit << 7 for the score x of ramp j
  auto code_of = [&](double x, uint32_t j) -> uint32_t {
    uint32_t e = lds_u32(tb + diag2::bin_of(x, pa, pc0) * 128u);
    const double t = lds_f64(sub + (e >> 16));
    const double b = lds_f64(sbase + j * 8u);
    uint32_t key = e & 0xffffu;
    asm("{\n\t.reg .pred p;\n\tsetp.le.f64 p, %1, %2;\n\t@p add.u32 %0, %0, 1;\n\t}"
        : "+r"(key)
        : "d"(t), "d"(x));
    if constexpr (NANCHK) key = x != x ? (uint32_t)m : key;  // NaN never exits
    return key | (x < b ? 0x80u : 0u);
  };
  unsigned char* kb = sm + diag2::OFF_KEY + warp * 32 * R;
  for (; ch < c_end; ch += WARPS) {
    __syncwarp();
    const int64_t nx = ch + WARPS;
    const int64_t s1 = nx << 5;
    const double2* src = reinterpret_cast<const double2*>(P.s + s1 * R);
    const int64_t npairs = nx < c_end ? (n - s1) * (R / 2) : 0;
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      const uint32_t j0 = (uint32_t)((2 * (k * 32 + lane)) % R);
      const uint32_t k0 = code_of(v[k].x, j0), k1 = code_of(v[k].y, j0 + 1);
      *reinterpret_cast<unsigned short*>(kb + 2 * (k * 32 + lane)) =
          (unsigned short)__byte_perm(k0, k1, 0x0040);
      const int t = k * 32 + lane;
      if (npairs >= 32 * (R / 2))
        v[k] = __ldcs(src + t);
      else if (npairs > 0)
        v[k] = t < npairs ? __ldcs(src + t) : make_double2(INF, INF);
    }
    const uint32_t cbc = cb;
    if (nx < c_end) cb = s1 + lane < n ? __ldcs(P.bits + s1 + lane) : 0u;
    __syncwarp();
    uint32_t kw[NW];
#pragma unroll
    for (int q = 0; q < NW; ++q) kw[q] = 0;
#pragma unroll
    for (int h = 0; h < R / 2; ++h)
      kw[h >> 1] |= (uint32_t)reinterpret_cast<const unsigned short*>(kb + lane * R)[h] << (16 * (h & 1));
    uint32_t mask = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) mask |= ((kw[j >> 2] >> (8 * (j & 3) + 7)) & 1u) << j;
    const uint32_t rest = mask & (mask - 1);
    const uint32_t f = mask ? (uint32_t)(__ffs(mask) - 1) : (uint32_t)R;
    const uint32_t f2 = rest ? (uint32_t)(__ffs(rest) - 1) : (uint32_t)R;
    const uint32_t cf = (cbc >> f) & 1u, cf2 = (cbc >> f2) & 1u;
    const bool live = (ch << 5) + lane < n;  // the last chunk's padding lanes count nowhere
    diag2::red_shared<0>(live ? sB + f * 128u : dummy, (int)(1u + (cf << 16)));
    diag2::red_shared<0>(live && f < (uint32_t)R ? sE + (f * R1 + f2) * 128u : dummy,
                         (int)(1u + (cf2 << 16)));
    Unroll<R>::run([&](auto jc) {
      constexpr int j = decltype(jc)::value;
      const uint32_t key = (kw[j >> 2] >> (8 * (j & 3))) & 0x7fu;
      const uint32_t g = (uint32_t)j < f ? f : f2;
      const int d = (int)((cbc >> j) & 1u) - (int)((cbc >> g) & 1u);
      const uint32_t addr = live && j <= (int)f ? sC3 + ((j * CELLS + key) * R1 + g) * 4u : dummy;
      diag2::red_shared<0>(addr, 1 + d * 65536);
    });
  }
  __syncthreads();
  // this CTA's cells -> its partial row (plain coalesced stores); lane copies folded
  uint32_t* out = P.part + (int64_t)blockIdx.x * P.ncell;
  const uint32_t* c3 = reinterpret_cast<const uint32_t*>(sm + L::OFF_C3);
  const uint32_t* bl = reinterpret_cast<const uint32_t*>(sm + L::OFF_B);
  const int n3 = R * m * R1;
  for (int q = tid; q < P.ncell; q += THREADS) {
    uint32_t w;
    if (q < n3) {
      const int j = q / (m * R1), rem = q - j * (m * R1);  // rem = key * R1 + s
      w = c3[j * CELLS * R1 + rem];
    } else {
      const uint32_t* cell = bl + (q - n3) * 32;  // B then E rows, 32 lane copies each
      uint32_t lo = 0, hi = 0;
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const uint32_t x = cell[(k + lane) & 31];
        lo += x & 0xffffu;
        hi += x >> 16;
      }
      w = lo | (hi << 16);
    }
    out[q] = w;
  }
}

// totals[q] = sum over CTAs of the partials (counts unsigned; C3 deltas signed)
__global__ void k_axis_reduce(const uint32_t* __restrict__ part, int grid, int ncell, int n3,
                              unsigned long long* __restrict__ tot_cnt, long long* __restrict__ tot_x) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ncell) return;
  const int g0 = (int)((int64_t)blockIdx.y * grid / gridDim.y), g1 = (int)((int64_t)(blockIdx.y + 1) * grid / gridDim.y);
  unsigned long long c = 0;
  long long x = 0;
#pragma unroll 4
  for (int g = g0; g < g1; ++g) {
    const uint32_t w = __ldcg(part + (int64_t)g * ncell + q);
    c += w & 0xffffu;
    x += q < n3 ? (long long)(short)(w >> 16) : (long long)(w >> 16);
  }
  if (c) atomicAdd(tot_cnt + q, c);
  if (x) atomicAdd(reinterpret_cast<unsigned long long*>(tot_x + q), (unsigned long long)x);
}

// one CTA per column j: prefix over keys, then every candidate of column j
template <int R>
__global__ void __launch_bounds__(512) k_axis_fin(const __grid_constant__ FinParams P) {
  constexpr int R1 = R + 1;
  const int j = blockIdx.x, m = P.m, tid = threadIdx.x;
  __shared__ long long pc[MAX_M * R1], pd[MAX_M * R1];
  __shared__ long long sB[R1], sBc[R1], sE[R1], sEc[R1];
  const int n3 = R * m * R1;
  for (int q = tid; q < m * R1; q += blockDim.x) {
    pc[q] = (long long)P.tot_cnt[j * m * R1 + q];
    pd[q] = P.tot_x[j * m * R1 + q];
  }
  if (tid < R1) {
    sB[tid] = (long long)P.tot_cnt[n3 + tid];
    sBc[tid] = P.tot_x[n3 + tid];
    sE[tid] = (long long)P.tot_cnt[n3 + R1 + j * R1 + tid];
    sEc[tid] = P.tot_x[n3 + R1 + j * R1 + tid];
  }
  __syncthreads();
  {  // prefix over keys, one warp per site s (shuffle scans, 32 keys per step)
    const int lane = tid & 31;
    for (int srow = tid >> 5; srow < R1; srow += blockDim.x >> 5) {
      long long ca = 0, cd = 0;
      for (int k0 = 0; k0 < m; k0 += 32) {
        const int k = k0 + lane;
        long long a = k < m ? pc[k * R1 + srow] : 0, b = k < m ? pd[k * R1 + srow] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const long long ya = __shfl_up_sync(0xffffffffu, a, o), yb = __shfl_up_sync(0xffffffffu, b, o);
          if (lane >= o) a += ya, b += yb;
        }
        a += ca;
        b += cd;
        if (k < m) pc[k * R1 + srow] = a, pd[k * R1 + srow] = b;
        ca = __shfl_sync(0xffffffffu, a, 31);
        cd = __shfl_sync(0xffffffffu, b, 31);
      }
    }
  }
  __syncthreads();
  for (int64_t c = tid; c < P.C; c += blockDim.x) {
    const int code = P.code[c];
    if ((code >> 8) != j) continue;
    const int k = code & 0xff;  // 255: NaN value, never exits at j
    long long h[R1];
    long long okc = 0, here = 0;
#pragma unroll
    for (int t = 0; t < R1; ++t) {
      if (t < j) {
        h[t] = sB[t];
        okc += sBc[t];
      } else if (t > j) {
        const long long F = k == 255 ? 0 : pc[k * R1 + t];
        h[t] = sB[t] + sE[t] - F;
        here += F;
        okc += sBc[t] + sEc[t] + (k == 255 ? 0 : pd[k * R1 + t]);
      }
    }
    h[j] = here;
    double hi = 0.0, lo = 0.0;
#pragma unroll
    for (int t = 0; t < R1; ++t) {  // the ordered TwoSum chain of k_finalize
      if (P.hist) P.hist[c * R1 + t] = h[t];
      const double x = (double)h[t];
      const double p = __dmul_rn(x, P.serve[t]);
      const double pe = __fma_rn(x, P.serve[t], -p);
      double s2, e;
      two_sum(hi, p, s2, e);
      hi = s2;
      lo = __dadd_rn(lo, __dadd_rn(e, pe));
    }
    double tot, e;
    two_sum(hi, lo, tot, e);
    const double dn = (double)P.n;
    if (P.ok) P.ok[c] = okc;
    if (P.acc) {
      P.acc[c] = __ddiv_rn((double)okc, dn);
      P.sav[c] = __dsub_rn(P.vanilla, __ddiv_rn(tot, dn));
    }
  }
}

}  // namespace axis
