// sweep_diag3.cuh — k_diag3: the diagonal-family sweep with lane-private
// cumulative counters. Same inputs, planning (diag2::Params) and outputs as
// k_diag2; what changes is how a sample is counted.
//
// With b_j = min(b_{j-1}, key_j) (b_{-1} = m) the sample exits at site j for
// positions b_j <= p < b_{j-1}. Because b is non-increasing,
//   1[b_j <= p < b_{j-1}] = 1[b_j <= p] - 1[b_{j-1} <= p],
// so with F_j(p) = #{i : b_j(i) <= p} (a cumulative count of b_j)
//   hist_j(p) = F_j(p) - F_{j-1}(p),   hist_r(p) = n - F_{r-1}(p),
// and, collecting the correctness bits c_j by the same identity,
//   ok(p) = #{c_r = 1} + sum_j #{i : b_j(i) <= p} weighted by (c_j - c_{j+1}).
// Every (sample, ramp) is therefore ONE shared-memory update at cell b_j of
// ramp j: +1 in the low half-word (the count) and c_j - c_{j+1} in the high
// half-word. The count never reaches 2^16, so nothing carries out of the low
// half and the high half holds the exact signed sum modulo 2^16 (|sum| < 2^15).
// k_diag2 needs two updates per drop and its updates collide in shared-memory
// banks (ncu: 2.8 wavefronts per ATOMS, 69 of the ~120 wavefronts per warp-chunk);
// here every lane owns its own copy of each cell (cell p, lane l at word
// 32 p + l, i.e. bank l), so each update instruction is exactly one wavefront
// and no lane ever waits for a dummy or a branch.
//
// Envelope (else the host runs k_diag2): m <= 64 distinct thresholds (cells
// 0..m, cell m is the "never exits" sink), and at most 32767 samples per
// lane copy per CTA (n <= ~154M at 147 CTAs) so the half-words stay exact.
#pragma once

namespace diag3 {

using diag2::Params;
constexpr int MAX_M = 64;
constexpr int CELLS = MAX_M + 1;  // positions 0..m (m = sink)

// Shape of one variant: NT threads per CTA; CP copies of every cell and of the
// bin table (lane l uses copy l % CP). CP = 32 makes every update and table
// read conflict-free; CP = 16 halves that shared memory (lanes l and l + 16
// share a copy, at most 2-way conflicts) so two 512-thread CTAs fit one SM and
// one CTA's prologue / fold overlaps the other's streaming.
template <int NT, int CP>
struct Cfg {
  static constexpr int THREADS = NT;
  static constexpr int WARPS = NT / 32;
  static constexpr int OFF_TAB = 0;                                   // u32 [NB][CP]
  static constexpr int OFF_SU = OFF_TAB + diag2::NB * CP * 4;         // f64 [128][SU_REP]
  static constexpr int OFF_KEY = OFF_SU + (diag2::MAX_M + 1) * diag2::SU_STRIDE;  // u8 [WARPS][32 R]
  static constexpr int ROWC = CELLS * CP * 4;                         // bytes per ramp: [cell][copy]
  // updates per copy of a cell: 32 / CP lanes x one per chunk, kept < 2^15
  static constexpr int MAX_CTA_CHUNKS = 32767 / (32 / CP);
  template <int R>
  __host__ __device__ static constexpr int off_c() { return OFF_KEY + WARPS * 32 * R; }
  template <int R>
  __host__ __device__ static constexpr int smem_bytes() { return off_c<R>() + R * ROWC; }
  template <int R>  // last CTA: finalisation scratch over the cell rows
  __host__ __device__ static constexpr int fin_bytes() { return 3 * (R + 1) * CELLS * 8 + 3 * CELLS * 8; }
};
using Big = Cfg<1024, 32>;   // one CTA per SM
using Pair = Cfg<512, 16>;   // two CTAs per SM

// Finalise one window from its merged per-position totals gD (+ this CTA's own
// unmerged sums cF / osum / own_corr when given): prefix over positions, exact
// histograms and correct counts, the k_finalize TwoSum chain, outputs per
// candidate. zero_acc leaves gD and the completion counters zeroed.
template <int R, int THREADS>
__device__ void finalize_window(const Params& P, unsigned char* scratch, long long* gD, const int* cF,
                                const int* osum, unsigned long long own_corr, bool zero_acc,
                                int64_t n, int64_t* hist_out, int64_t* ok_out, double* acc_out,
                                double* sav_out) {
  constexpr int WARPS = THREADS / 32;
  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = P.m;
  const int M1 = m + 1;
  long long* hst = reinterpret_cast<long long*>(scratch);  // [R+1][M1] (F_j first)
  long long* okp = hst + (R + 1) * M1;
  double* prs = reinterpret_cast<double*>(okp + M1);
  double* pes = prs + (R + 1) * M1;
  double* accp = pes + (R + 1) * M1;
  double* savp = accp + M1;
  __shared__ long long s_corr_all;
  if (tid == 0) {
    s_corr_all = (long long)(__ldcg(gD + diag2::CORR_IDX) + own_corr);
    if (zero_acc) {
      gD[diag2::CORR_IDX] = 0;
      P.done[0] = 0u;
      P.done[1] = 0u;
    }
  }
  for (int q = tid; q < (R + 1) * m; q += THREADS) {  // global + own (+ zero for the next launch)
    const int j = q / m, p = q - j * m;
    const long long g = __ldcg(gD + j * diag2::W + p);
    if (zero_acc) gD[j * diag2::W + p] = 0;
    const long long own = !cF ? 0 : j < R ? (long long)cF[j * MAX_M + p] : (long long)osum[p];
    hst[j * M1 + p] = g + own;
  }
  __syncthreads();
  for (int row = warp; row <= R; row += WARPS) {  // inclusive prefix over p < m: F_j(p), O(p)
    long long* a = hst + row * M1;
    long long carry = 0;
    for (int p0 = 0; p0 < m; p0 += 32) {
      const int p = p0 + lane;
      long long x = p < m ? a[p] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
      }
      x += carry;
      if (p < m) a[p] = x;
      carry = __shfl_sync(FULL, x, 31);
    }
  }
  __syncthreads();
  const long long corrR = s_corr_all;
  for (int p = tid; p < M1; p += THREADS) {  // F -> histograms, O -> correct counts
    if (p == m) {  // NaN threshold row: nothing exits
      for (int j = 0; j < R; ++j) hst[j * M1 + p] = 0;
      hst[R * M1 + p] = n;
      okp[p] = corrR;
      continue;
    }
    okp[p] = corrR + hst[R * M1 + p];
    long long fprev = 0;
    for (int j = 0; j < R; ++j) {
      const long long f = hst[j * M1 + p];
      hst[j * M1 + p] = f - fprev;
      fprev = f;
    }
    hst[R * M1 + p] = n - fprev;
  }
  __syncthreads();
  for (int i = tid; i < (R + 1) * M1; i += THREADS) {  // error-free products
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
    const int q = P.C <= diag2::MAX_POS ? P.pos[c] : P.pos_dev[c];
    return q == 255 ? m : q;
  };
  if (hist_out)
    for (int64_t i = tid; i < P.C * (R + 1); i += THREADS) {
      const int64_t c = i / (R + 1);
      const int site = (int)(i - c * (R + 1));
      hist_out[i] = hst[site * M1 + posof(c)];
    }
  for (int64_t c = tid; c < P.C; c += THREADS) {
    const int p = posof(c);
    if (ok_out) ok_out[c] = okp[p];
    if (acc_out) {
      acc_out[c] = accp[p];
      sav_out[c] = savp[p];
    }
  }
}

// Finalise one window whose accumulator already holds PREFIX sums over positions
// (k_diag3<DIST>: every CTA scanned its own counts before merging, and the scan
// is linear): gD[j][p] = F_j(p), gD[R][p] = O(p). One thread per position turns
// its column into the histogram, the correct count and the k_finalize TwoSum
// chain in registers (the operations of finalize_window, in the same order, so
// the same bits); the accumulator is read once and left zeroed.
template <int R, int THREADS>
__device__ void finalize_prefixed(const Params& P, unsigned char* scratch, long long* gD, int64_t n) {
  const int tid = threadIdx.x;
  const int m = P.m;
  const int M1 = m + 1;
  long long* hst = reinterpret_cast<long long*>(scratch);  // [R+1][M1]: F_j, then histograms
  long long* okp = hst + (R + 1) * M1;
  double* accp = reinterpret_cast<double*>(okp + M1);
  double* savp = accp + M1;
  __shared__ long long s_corr_all;
  if (tid == THREADS - 1) {
    s_corr_all = (long long)__ldcg(gD + diag2::CORR_IDX);
    gD[diag2::CORR_IDX] = 0;
  }
  for (int q = tid; q < (R + 1) * m; q += THREADS) {
    const int j = q / m, p = q - j * m;
    hst[j * M1 + p] = __ldcg(gD + j * diag2::W + p);
    gD[j * diag2::W + p] = 0;
  }
  __syncthreads();
  const long long corrR = s_corr_all;
  for (int p = tid; p < M1; p += THREADS) {
    long long h[R + 1];
    long long ok;
    if (p == m) {  // NaN threshold row: nothing exits
#pragma unroll
      for (int j = 0; j < R; ++j) h[j] = 0;
      h[R] = n;
      ok = corrR;
    } else {
      ok = corrR + hst[R * M1 + p];
      long long fprev = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const long long f = hst[j * M1 + p];
        h[j] = f - fprev;
        fprev = f;
      }
      h[R] = n - fprev;
    }
    double hi = 0.0, lo = 0.0;
#pragma unroll
    for (int site = 0; site <= R; ++site) {
      const double x = (double)h[site];
      const double pr = __dmul_rn(x, P.serve[site]);
      const double pe = __fma_rn(x, P.serve[site], -pr);
      double s2, e;
      two_sum(hi, pr, s2, e);
      hi = s2;
      lo = __dadd_rn(lo, __dadd_rn(e, pe));
      hst[site * M1 + p] = h[site];
    }
    double tot2, e;
    two_sum(hi, lo, tot2, e);
    const double dn = (double)n;
    okp[p] = ok;
    accp[p] = __ddiv_rn((double)ok, dn);
    savp[p] = __dsub_rn(P.vanilla, __ddiv_rn(tot2, dn));
  }
  __syncthreads();
  auto posof = [&](int64_t c) -> int {
    const int q = P.C <= diag2::MAX_POS ? P.pos[c] : P.pos_dev[c];
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
}

// DIST = false: the CTA elected first-to-finish-streaming last waits for every
// other CTA's merge, then finalises the whole window (finalize_window: scan,
// histograms, products, chain in separate block-wide phases).
// DIST = true: each CTA folds its lane copies with 16-byte reads, scans its own
// counts over positions, merges the prefix sums and takes a ticket; the last
// ticket finalises with one thread per position (finalize_prefixed). Nobody
// waits on anybody: the tail is fold + scan + merge + one parallel finalise.
template <int R, int NT, int CP, bool DIST = false>
__global__ void __launch_bounds__(NT, 1024 / NT) k_diag3(const __grid_constant__ Params P) {
  using C = Cfg<NT, CP>;
  constexpr int THREADS = C::THREADS, WARPS = C::WARPS, ROWC = C::ROWC;
  constexpr int OFF_TAB = C::OFF_TAB, OFF_SU = C::OFF_SU, OFF_KEY = C::OFF_KEY;
  static_assert(R % 2 == 0 && R >= 2 && R <= diag2::RMAX, "even R only");
  static_assert(C::template fin_bytes<R>() <= R * ROWC, "finalisation scratch fits the cell rows");
  static_assert(R * MAX_M * 4 <= WARPS * 32 * R, "per-CTA sums fit the key buffer");
  constexpr int NW = (R + 3) / 4;
  constexpr int OFF_C = C::template off_c<R>();
  using diag2::lds_f64;
  using diag2::lds_u32;
  using diag2::Unroll;
  extern __shared__ __align__(16) unsigned char sm[];
  const int m = P.m;
  uint32_t* stab = reinterpret_cast<uint32_t*>(sm + OFF_TAB);
  double* su = reinterpret_cast<double*>(sm + OFF_SU);
  unsigned char* skey = sm + OFF_KEY;
  uint32_t* cells = reinterpret_cast<uint32_t*>(sm + OFF_C);
  __shared__ unsigned s_last;
  __shared__ unsigned long long s_corr;
  __shared__ int s_osum[MAX_M];  // sum over ramps of the O cells, per position
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned FULL = 0xffffffffu;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);

  const int64_t n = P.n;
  const int64_t nchunks = (n + 31) >> 5;
  // Each CTA streams one contiguous, equal share of the chunks (212-213 at
  // config 4) and its warps interleave over it: a grid-stride split gave 7
  // chunks per warp to two thirds of the CTAs and 6 to the rest.
  const int64_t c_end = (int64_t)(blockIdx.x + 1) * nchunks / gridDim.x;
  int64_t ch = (int64_t)blockIdx.x * nchunks / gridDim.x + warp;
  constexpr int64_t G = WARPS;
  double2 v[R / 2];
  uint32_t cb = 0;
  auto load = [&](int64_t c) {
    if (c >= c_end) return;
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
        v[k] = t < npairs ? __ldcs(src + t) : make_double2(INF, INF);  // key m: the sink
      }
      cb = s0 + lane < n ? __ldcs(P.bits + s0 + lane) : 0u;
    }
  };
  if (P.trace && tid == 0) P.trace[blockIdx.x * 6 + 0] = diag2::gtimer();
  // Parameter reads first: a constant-bank miss issued after the window's
  // loads queues behind them (measured: a 2 us prologue).
  constexpr int TQ = diag2::NB * CP / 4 / THREADS;                        // table uint4 per thread
  constexpr int SQ = (diag2::MAX_M + 1) * diag2::SU_REP / 2 / THREADS;    // threshold pairs per thread
  static_assert(TQ * THREADS * 4 == diag2::NB * CP && SQ * THREADS * 2 == (diag2::MAX_M + 1) * diag2::SU_REP,
                "whole table / threshold pairs per thread");
  uint32_t te[TQ];
  double ue[SQ];
#pragma unroll
  for (int i = 0; i < TQ; ++i) te[i] = P.tab[(tid + i * THREADS) / (CP / 4)];
#pragma unroll
  for (int i = 0; i < SQ; ++i) {
    const int tu = (tid + i * THREADS) / (diag2::SU_REP / 2);
    ue[i] = tu < m ? P.u[tu] : __longlong_as_double(0x7ff8000000000000LL);
  }
  load(ch);  // first HBM round trip overlaps the prologue

  // ---- prologue (vector stores): zeroed cells, replicated bin table and thresholds
  {
    uint4* c4 = reinterpret_cast<uint4*>(cells);
    const int per_ramp = (m + 1) * CP / 4;  // uint4 per ramp row in use (cells 0..m)
    for (int q = tid; q < R * per_ramp; q += THREADS) {
      const int j = q / per_ramp;
      c4[j * CELLS * CP / 4 + (q - j * per_ramp)] = make_uint4(0u, 0u, 0u, 0u);
    }
    if (tid < MAX_M) s_osum[tid] = 0;
    if (tid == 0) s_corr = 0;
    uint4* t4 = reinterpret_cast<uint4*>(stab);  // CP / 4 uint4 per bin
#pragma unroll
    for (int i = 0; i < TQ; ++i) t4[tid + i * THREADS] = make_uint4(te[i], te[i], te[i], te[i]);
#pragma unroll
    for (int i = 0; i < SQ; ++i) reinterpret_cast<double2*>(su)[tid + i * THREADS] = make_double2(ue[i], ue[i]);
  }
  __syncthreads();

  const double pa = P.a, pc0 = P.c0;
  const uint32_t smb = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t tb = smb + OFF_TAB + (uint32_t)(lane % CP) * 4;
  const uint32_t sub = smb + OFF_SU + (uint32_t)(lane % diag2::SU_REP) * 8;
  const uint32_t cB = smb + OFF_C + (uint32_t)(lane % CP) * 4;  // this lane's copy of every cell
  auto keyof = [&](double x) -> uint32_t {
    uint32_t e = lds_u32(tb + diag2::bin_of(x, pa, pc0) * (CP * 4u));
    const double t = lds_f64(sub + (e >> 16));
    asm("{\n\t.reg .pred p;\n\tsetp.le.f64 p, %1, %2;\n\t@p add.u32 %0, %0, 1;\n\t}"
        : "+r"(e)
        : "d"(t), "d"(x));
    return e;
  };

  unsigned char* kb = skey + warp * 32 * R;
  unsigned corr = 0;
  if (P.trace && tid == 0) P.trace[blockIdx.x * 6 + 1] = diag2::gtimer();
  for (; ch < c_end; ch += G) {
    __syncwarp();  // previous chunk's key reads are done
    // Each pair's registers are refilled with the next chunk as soon as its two
    // keys are taken, so the next chunk's loads leave during the keying (ncu:
    // the top-of-loop wait on the loads was the largest stall).
    const int64_t nx = ch + G;
    const int64_t s1 = nx << 5;
    const double2* src = reinterpret_cast<const double2*>(P.s + s1 * R);
    const int64_t npairs = nx < c_end ? (n - s1) * (R / 2) : 0;  // valid pairs of the next chunk
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      const uint32_t k0 = keyof(v[k].x), k1 = keyof(v[k].y);
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
    // one update per ramp: cell b_j += 1 + ((c_j - c_{j+1}) << 16)
    uint32_t prev = (uint32_t)m;
    Unroll<R>::run([&](auto jc) {
      constexpr int j = decltype(jc)::value;
      const uint32_t kj = __byte_perm(kw[j >> 2], 0, 0x4440 | (j & 3));
      prev = kj < prev ? kj : prev;
      const uint32_t val = 1u + ((cbc << (16 - j)) & 0x10000u) - ((cbc << (15 - j)) & 0x10000u);
      diag2::red_shared<j * ROWC>(cB + prev * (CP * 4u), (int)val);
    });
    corr += (cbc >> R) & 1u;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) corr += __shfl_xor_sync(FULL, corr, o);
  if (P.trace && lane == 0) atomicMax(P.trace + blockIdx.x * 6 + 2, diag2::gtimer());
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // see sweep_diag2.cuh
  asm volatile("griddepcontrol.wait;" ::: "memory");  // previous sweep done: gD/done/outputs are ours
  __syncthreads();
  // Elect the last CTA now; the round trip overlaps the fold below (the last
  // thread has no cell to fold unless R * m = 1024).
  if constexpr (!DIST)
    if (tid == THREADS - 1) s_last = atomicAdd(P.done, 1u) == gridDim.x - 1;
  if (lane == 0 && corr) atomicAdd(&s_corr, (unsigned long long)corr);

  // ---- per-CTA sums: fold the lane copies of each cell. F stays per ramp; O is
  // summed over ramps.
  int* cF = reinterpret_cast<int*>(skey);  // F [R][MAX_M] raw per-position counts
  {
    // 16-byte reads of 4 copies at a time, the chunk order rotated by thread so
    // the CP / 4 threads of a group cover all 32 banks (4 wavefronts per warp
    // read, the minimum for 512 bytes) with a dependent chain of CP / 4 loads.
    // Under DIST the prefix over positions follows per CTA; otherwise it is
    // linear, so only the last CTA takes it, on totals.
    constexpr int NQ = CP / 4;
    for (int q = tid; q < R * m; q += THREADS) {
      const int j = q / m, p = q - j * m;
      const uint4* cell = reinterpret_cast<const uint4*>(cells + (j * CELLS + p) * CP);
      int lo = 0, hi = 0;
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        const uint4 w = cell[(k + tid) % NQ];
        lo += (int)(w.x & 0xffffu) + (int)(w.y & 0xffffu) + (int)(w.z & 0xffffu) + (int)(w.w & 0xffffu);
        // each copy's high half is its exact signed sum mod 2^16
        hi += (int)(short)(w.x >> 16) + (int)(short)(w.y >> 16) + (int)(short)(w.z >> 16) +
              (int)(short)(w.w >> 16);
      }
      cF[j * MAX_M + p] = lo;
      if (hi) atomicAdd(&s_osum[p], hi);
    }
  }
  __syncthreads();
  if (P.trace && tid == 0) P.trace[blockIdx.x * 6 + 3] = diag2::gtimer();
  if constexpr (DIST) {
    // this CTA's inclusive prefix over positions (warp j < R: row j, warp R: O)
    if (warp <= R) {
      int* a = warp < R ? cF + warp * MAX_M : s_osum;
      int carry = 0;
      for (int p0 = 0; p0 < m; p0 += 32) {
        const int p = p0 + lane;
        int x = p < m ? a[p] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(FULL, x, o);
          if (lane >= o) x += y;
        }
        x += carry;
        if (p < m) a[p] = x;
        carry = __shfl_sync(FULL, x, 31);
      }
    }
    __syncthreads();
    long long* gD = P.gD;
    for (int q = tid; q < (R + 1) * m; q += THREADS) {
      const int j = q / m, p = q - j * m;
      const long long x = j < R ? (long long)cF[j * MAX_M + p] : (long long)s_osum[p];
      if (x) atomicAdd(reinterpret_cast<unsigned long long*>(gD + j * diag2::W + p), (unsigned long long)x);
    }
    if (tid == 0 && s_corr)
      atomicAdd(reinterpret_cast<unsigned long long*>(gD + diag2::CORR_IDX), s_corr);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    __syncthreads();
    if (P.trace && tid == 0) P.trace[blockIdx.x * 6 + 5] = diag2::gtimer();
    if (tid == 0) {
      unsigned t;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(P.done) : "memory");
      s_last = t == gridDim.x - 1;
      if (s_last) P.done[0] = 0u;  // the next launch counts after its griddepcontrol.wait
    }
    __syncthreads();
    if (!s_last) return;
    if (P.trace && tid == 0) P.trace[blockIdx.x * 6 + 1] = diag2::gtimer();
    finalize_prefixed<R, THREADS>(P, sm + OFF_C, gD, n);
    if (P.trace) {
      __syncthreads();
      if (tid == 0) P.trace[blockIdx.x * 6 + 4] = diag2::gtimer();
    }
    return;
  }
  long long* gD = P.gD;  // [j * W + p]: F_j[p] for j < R, row R: sum_j O_j[p] (two's complement)
  if (!s_last) {
    for (int q = tid; q < (R + 1) * m; q += THREADS) {
      const int j = q / m, p = q - j * m;
      const long long x = j < R ? (long long)cF[j * MAX_M + p] : (long long)s_osum[p];
      if (x) atomicAdd(reinterpret_cast<unsigned long long*>(gD + j * diag2::W + p),
                       (unsigned long long)x);
    }
    if (tid == 0 && s_corr)
      atomicAdd(reinterpret_cast<unsigned long long*>(gD + diag2::CORR_IDX), s_corr);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    __syncthreads();
    if (tid == 0) atomicAdd(P.done + 1, 1u);
    return;
  }

  // ---- the last CTA: wait for the others' merges, fold its own sums in, finalise
  if (tid == 0) {
    unsigned v2;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v2) : "l"(P.done + 1) : "memory");
    } while (v2 < gridDim.x - 1);
  }
  __syncthreads();
  if (P.trace && tid == 0) P.trace[blockIdx.x * 6 + 1] = diag2::gtimer();
  finalize_window<R, THREADS>(P, sm + OFF_C, gD, cF, s_osum, s_corr, /*zero_acc=*/true, n, P.hist,
                              P.ok, P.acc, P.sav);
  if (P.trace) {
    __syncthreads();
    if (tid == 0) P.trace[blockIdx.x * 6 + 4] = diag2::gtimer();
  }
}


// ---------------------------------------------------------------------------
// k_diag3_windows_db: the k_diag3 sweep over nwin windows (same n, r and
// candidate rows) in one persistent launch, with the per-window fold taken off
// the streaming path. Tables are built once. Two cell buffers (16 lane copies each, so both fit beside the tables):
// 30 "stream" warps count window w into buffer w & 1 while 2 "fold" warps fold
// window w - 1 out of the other buffer (sum the copies, zero them, merge the
// per-CTA sums into that window's accumulator). Named barriers hand buffers
// over: FULL[b] (stream arrive, fold sync) when a window is counted, ZERO[b]
// (fold arrive, stream sync) when its buffer is clean again, so at most one
// generation of each barrier is ever pending. The per-window fold / merge no
// longer stalls the SM's HBM stream (the single-buffer version, where every
// CTA folded each window itself, ran at 18.7 us per window against 16.7 us
// here). Totals per window land in accw; k_diag3_windows_fin finalises them.
// ---------------------------------------------------------------------------
namespace dbw {
constexpr int THREADS = 1024, SW = 30, FW = 2, CP = 16;
constexpr int ROWC = CELLS * CP * 4;                                 // bytes per ramp per buffer
constexpr int OFF_TAB = 0;                                           // u32 [NB][CP]
constexpr int OFF_SU = OFF_TAB + diag2::NB * CP * 4;                 // f64 [128][SU_REP]
constexpr int OFF_KEY = OFF_SU + (diag2::MAX_M + 1) * diag2::SU_STRIDE;  // u8 [SW][32 R]
template <int R>
__host__ __device__ constexpr int off_c() { return OFF_KEY + ((SW * 32 * R + 15) & ~15); }
template <int R>
__host__ __device__ constexpr int smem_bytes() { return off_c<R>() + 2 * R * ROWC; }
// updates per copy of a cell: 2 lanes x one per chunk, kept < 2^15
constexpr int MAX_CTA_CHUNKS = 32767 / 2;
}  // namespace dbw

template <int R>
__global__ void __launch_bounds__(dbw::THREADS, 1) k_diag3_windows_db(
    const __grid_constant__ Params P, const double* const* __restrict__ s_list,
    const uint32_t* const* __restrict__ b_list, int nwin, long long* __restrict__ accw) {
  using namespace dbw;
  constexpr int NW = (R + 3) / 4;
  constexpr int OFF_C = off_c<R>();
  constexpr int BUF = R * ROWC;  // bytes per cell buffer
  using diag2::lds_f64;
  using diag2::lds_u32;
  using diag2::Unroll;
  extern __shared__ __align__(16) unsigned char sm[];
  const int m = P.m;
  uint32_t* stab = reinterpret_cast<uint32_t*>(sm + OFF_TAB);
  double* su = reinterpret_cast<double*>(sm + OFF_SU);
  unsigned char* skey = sm + OFF_KEY;
  __shared__ unsigned long long s_corr[2];
  __shared__ int s_osum[MAX_M];
  __shared__ int s_cF[R * MAX_M];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned FULL = 0xffffffffu;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  const int64_t n = P.n;
  const int64_t nchunks = (n + 31) >> 5;
  const int64_t c_end = (int64_t)(blockIdx.x + 1) * nchunks / gridDim.x;
  const int64_t c_begin = (int64_t)blockIdx.x * nchunks / gridDim.x + warp;
  double2 v[R / 2];
  uint32_t cb = 0;
  auto load = [&](const double* S, const uint32_t* BITS, int64_t c) {
    if (c >= c_end) return;
    const int64_t s0 = c << 5;
    const double2* src = reinterpret_cast<const double2*>(S + s0 * R);
    const int64_t npairs = (n - s0) * (R / 2);
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      const int t = k * 32 + lane;
      v[k] = t < npairs ? __ldcs(src + t) : make_double2(INF, INF);
    }
    cb = s0 + lane < n ? __ldcs(BITS + s0 + lane) : 0u;
  };
  if (warp < SW) load(s_list[0], b_list[0], c_begin);
  {  // tables once, both cell buffers zero
    uint4* t4 = reinterpret_cast<uint4*>(stab);
    for (int q = tid; q < diag2::NB * CP / 4; q += THREADS) {
      const uint32_t e = P.tab[q / (CP / 4)];
      t4[q] = make_uint4(e, e, e, e);
    }
    for (int q = tid; q < (diag2::MAX_M + 1) * diag2::SU_REP / 2; q += THREADS) {
      const int tu = q / (diag2::SU_REP / 2);
      const double x = tu < m ? P.u[tu] : __longlong_as_double(0x7ff8000000000000LL);
      reinterpret_cast<double2*>(su)[q] = make_double2(x, x);
    }
    uint4* c4 = reinterpret_cast<uint4*>(sm + OFF_C);
    for (int q = tid; q < 2 * BUF / 16; q += THREADS) c4[q] = make_uint4(0u, 0u, 0u, 0u);
    if (tid < 2) s_corr[tid] = 0ull;
  }
  __syncthreads();
  const uint32_t smb = (uint32_t)__cvta_generic_to_shared(sm);
  if (warp < SW) {
    // ======================= stream warps =======================
    const double pa = P.a, pc0 = P.c0;
    const uint32_t tb = smb + OFF_TAB + (uint32_t)(lane % CP) * 4;
    const uint32_t sub = smb + OFF_SU + (uint32_t)(lane % diag2::SU_REP) * 8;
    auto keyof = [&](double x) -> uint32_t {
      uint32_t e = lds_u32(tb + diag2::bin_of(x, pa, pc0) * (CP * 4u));
      const double t = lds_f64(sub + (e >> 16));
      asm("{\n\t.reg .pred p;\n\tsetp.le.f64 p, %1, %2;\n\t@p add.u32 %0, %0, 1;\n\t}"
          : "+r"(e)
          : "d"(t), "d"(x));
      return e;
    };
    unsigned char* kb = skey + warp * 32 * R;
    for (int w = 0; w < nwin; ++w) {
      const int bi = w & 1;
      const double* S = s_list[w];
      const uint32_t* BITS = b_list[w];
      if (w >= 2) asm volatile("bar.sync %0, %1;" ::"r"(3 + bi), "r"(THREADS) : "memory");  // buffer bi clean
      const uint32_t cB = smb + OFF_C + bi * BUF + (uint32_t)(lane % CP) * 4;
      unsigned corr = 0;
      for (int64_t ch = c_begin; ch < c_end; ch += SW) {
        __syncwarp();
        const int64_t nx = ch + SW;
        const int64_t s1 = nx << 5;
        const double2* src = reinterpret_cast<const double2*>(S + s1 * R);
        const int64_t npairs = nx < c_end ? (n - s1) * (R / 2) : 0;
#pragma unroll
        for (int k = 0; k < R / 2; ++k) {
          const uint32_t k0 = keyof(v[k].x), k1 = keyof(v[k].y);
          *reinterpret_cast<unsigned short*>(kb + 2 * (k * 32 + lane)) =
              (unsigned short)__byte_perm(k0, k1, 0x0040);
          const int t = k * 32 + lane;
          if (npairs >= 32 * (R / 2))
            v[k] = __ldcs(src + t);
          else if (npairs > 0)
            v[k] = t < npairs ? __ldcs(src + t) : make_double2(INF, INF);
        }
        const uint32_t cbc = cb;
        if (nx < c_end) cb = s1 + lane < n ? __ldcs(BITS + s1 + lane) : 0u;
        __syncwarp();
        uint32_t kw[NW];
#pragma unroll
        for (int q = 0; q < NW; ++q) kw[q] = 0;
#pragma unroll
        for (int hq = 0; hq < R / 2; ++hq)
          kw[hq >> 1] |= (uint32_t)reinterpret_cast<const unsigned short*>(kb + lane * R)[hq]
                         << (16 * (hq & 1));
        uint32_t prev = (uint32_t)m;
        Unroll<R>::run([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          const uint32_t kj = __byte_perm(kw[j >> 2], 0, 0x4440 | (j & 3));
          prev = kj < prev ? kj : prev;
          const uint32_t val = 1u + ((cbc << (16 - j)) & 0x10000u) - ((cbc << (15 - j)) & 0x10000u);
          diag2::red_shared<j * ROWC>(cB + prev * (CP * 4u), (int)val);
        });
        corr += (cbc >> R) & 1u;
      }
      if (w + 1 < nwin) load(s_list[w + 1], b_list[w + 1], c_begin);  // next window in flight
#pragma unroll
      for (int o = 16; o; o >>= 1) corr += __shfl_xor_sync(FULL, corr, o);
      if (lane == 0 && corr) atomicAdd(&s_corr[bi], (unsigned long long)corr);
      asm volatile("bar.arrive %0, %1;" ::"r"(1 + bi), "r"(THREADS) : "memory");  // window w counted
    }
    return;
  }
  // ======================= fold warps =======================
  const int ft = tid - SW * 32;  // 0 .. FW * 32 - 1
  constexpr int FT = FW * 32;
  constexpr int NQ = CP / 4;
  for (int w = 0; w < nwin; ++w) {
    const int bi = w & 1;
    asm volatile("bar.sync %0, %1;" ::"r"(1 + bi), "r"(THREADS) : "memory");  // window w counted
    for (int q = ft; q < MAX_M; q += FT) s_osum[q] = 0;
    asm volatile("bar.sync 5, %0;" ::"r"(FT) : "memory");
    uint32_t* cells = reinterpret_cast<uint32_t*>(sm + OFF_C + bi * BUF);
    for (int q = ft; q < R * (m + 1); q += FT) {  // fold cells 0..m-1, zero 0..m (m = the sink)
      const int j = q / (m + 1), p = q - j * (m + 1);
      uint4* cell = reinterpret_cast<uint4*>(cells + (j * CELLS + p) * CP);
      if (p < m) {
        int lo = 0, hi = 0;
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
          const uint4 x = cell[(k + ft) % NQ];
          lo += (int)(x.x & 0xffffu) + (int)(x.y & 0xffffu) + (int)(x.z & 0xffffu) + (int)(x.w & 0xffffu);
          hi += (int)(short)(x.x >> 16) + (int)(short)(x.y >> 16) + (int)(short)(x.z >> 16) +
                (int)(short)(x.w >> 16);
        }
        s_cF[j * MAX_M + p] = lo;
        if (hi) atomicAdd(&s_osum[p], hi);
      }
#pragma unroll
      for (int k = 0; k < NQ; ++k) cell[k] = make_uint4(0u, 0u, 0u, 0u);
    }
    asm volatile("bar.sync 5, %0;" ::"r"(FT) : "memory");
    long long* gD = accw + (int64_t)w * diag2::ACC_WORDS;
    for (int q = ft; q < (R + 1) * m; q += FT) {
      const int j = q / m, p = q - j * m;
      const long long x = j < R ? (long long)s_cF[j * MAX_M + p] : (long long)s_osum[p];
      if (x) atomicAdd(reinterpret_cast<unsigned long long*>(gD + j * diag2::W + p), (unsigned long long)x);
    }
    if (ft == 0) {
      const unsigned long long c = s_corr[bi];
      s_corr[bi] = 0ull;
      if (c) atomicAdd(reinterpret_cast<unsigned long long*>(gD + diag2::CORR_IDX), c);
    }
    asm volatile("bar.sync 5, %0;" ::"r"(FT) : "memory");  // s_cF / s_osum free again
    asm volatile("bar.arrive %0, %1;" ::"r"(3 + bi), "r"(THREADS) : "memory");  // buffer bi clean
  }
}

// one CTA per window: finalise from the totals k_diag3_windows_db left in accw
template <int R>
__global__ void __launch_bounds__(1024, 1) k_diag3_windows_fin(const __grid_constant__ Params P,
                                                              long long* __restrict__ accw,
                                                              double* __restrict__ acc_out,
                                                              double* __restrict__ sav_out) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int w = blockIdx.x;
  finalize_window<R, 1024>(P, sm, accw + (int64_t)w * diag2::ACC_WORDS, nullptr, nullptr, 0ull,
                           /*zero_acc=*/false, P.n, nullptr, nullptr, acc_out + w * P.C,
                           sav_out + w * P.C);
}
}  // namespace diag3
