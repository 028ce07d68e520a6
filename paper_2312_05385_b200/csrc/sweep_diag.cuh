// sweep_diag.cuh — HBM-bound sweep for the diagonal candidate family
// (every candidate row repeats one threshold on all ramps: t_c * 1, SURVEY §7
// step 4, the config-4 "64-point grid"). Included by eeb200.cu.
//
// With u_0 < ... < u_{M-1} the distinct non-NaN thresholds, sample i's exit
// site under threshold u_p is the first ramp whose score is < u_p, i.e. the
// first j whose prefix minimum m_j (NaN-skipping fmin) is < u_p. With
// b_j = #{k : u_k <= m_j} (M when m_j is NaN), b is non-increasing in j and
//     site(p) = j   <=>   b_j <= p < b_{j-1}         (b_{-1} := M)
//     site(p) = R   <=>   p < b_{R-1}
// so each sample contributes one interval of candidate positions per ramp at
// which its prefix minimum drops: +1/-1 at the ends of that interval in a
// difference array D[site][p]. Correct releases are the union of intervals
// over correct ramps (runs of consecutive correct ramps merge into one
// interval). Per-warp shared-memory copies of the difference arrays absorb the
// updates; prefix sums over p then give, for every candidate, the exact
// integer histogram and correct count — the same numbers k_count produces —
// after reading each fp64 score exactly once.
#pragma once

namespace diag {

constexpr int THREADS = 256;
constexpr int MAX_M = 256;   // distinct thresholds supported by this path
constexpr int NBINS = 2048;  // bucket grid resolution

// O(1) bucket lookup: b(x) = #{k : u[k] <= x}. A uniform grid over the finite
// threshold range gives bin(x) (monotone in x); lo[k] counts the thresholds
// whose own bin is < k — all of them are < x — and th[k] = u[lo[k]] is the
// only other threshold that can still be <= x when every bin holds at most one
// threshold (SINGLE, checked on the host with the same arithmetic). Otherwise
// a short scan finishes the count; u[m] is a NaN sentinel that stops it.
struct Grid {
  double base, inv_w;
  int top;  // nbins - 1
  int nbins;
};

// cvt.rzi.s32.f64 semantics (truncate, saturate, NaN -> 0) on host and device,
// then clamp to [0, top]: monotone in x.
__host__ __device__ __forceinline__ int grid_bin(const Grid& g, double x) {
#ifdef __CUDA_ARCH__
  const int k = __double2int_rz(__dmul_rn(__dsub_rn(x, g.base), g.inv_w));
#else
  volatile double d = x - g.base;
  volatile double q = d * g.inv_w;
  const double t = q;
  const int k = t != t ? 0 : t >= 2147483647.0 ? 2147483647 : t <= -2147483648.0 ? (-2147483647 - 1) : (int)t;
#endif
  return k < 0 ? 0 : (k > g.top ? g.top : k);
}

template <bool SINGLE>
__device__ __forceinline__ int bucket(const double* __restrict__ u,
                                      const unsigned short* __restrict__ lo,
                                      const double* __restrict__ th, const Grid& g, double x) {
  const int k = grid_bin(g, x);
  int b = lo[k];
  if constexpr (SINGLE) {
    return b + (th[k] <= x);
  } else {
    while (u[b] <= x) ++b;
    return b;
  }
}

// Difference arrays per copy: one row of W (p) x 2 (correct) counters per
// site, interleaved as [p][c] (position p = m is a sink for interval ends,
// never read back). Splitting by the correctness of the exit ramp makes the
// correct-release count fall out of the same two updates:
// hist[site] = D[site][.][0] + D[site][.][1], ok = sum_site D[site][.][1].
template <int RMAX, int W, bool EVEN, bool SINGLE>
__global__ void __launch_bounds__(THREADS)
    k_diag(const double* __restrict__ s, const uint32_t* __restrict__ bits, int64_t n, int r,
           const double* __restrict__ utab, const unsigned short* __restrict__ lotab,
           const double* __restrict__ thtab, Grid g,
           int m, int copies, long long* __restrict__ gD, unsigned* __restrict__ done,
           const int* __restrict__ pos, int64_t C, const double* __restrict__ serve,
           double vanilla, int64_t* __restrict__ hist_out, int64_t* __restrict__ ok_out,
           double* __restrict__ acc, double* __restrict__ sav) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sth = reinterpret_cast<double*>(smem_raw);                   // [nbins]
  double* su = sth + g.nbins;                                          // [m+1]
  unsigned short* slo = reinterpret_cast<unsigned short*>(su + m + 1);  // [nbins]
  int* sD = reinterpret_cast<int*>(slo + ((g.nbins + 7) & ~7));        // [copies][dstride]
  const int rows = 2 * (r + 1);
  const int dstride = rows * W;
  for (int k = threadIdx.x; k <= m; k += THREADS) su[k] = utab[k];
  for (int k = threadIdx.x; k < g.nbins; k += THREADS) {
    slo[k] = lotab[k];
    sth[k] = thtab[k];
  }
  for (int k = threadIdx.x; k < copies * dstride; k += THREADS) sD[k] = 0;
  __syncthreads();
  int* D = sD + ((threadIdx.x >> 5) % copies) * dstride;
  unsigned corrR = 0;

  const int64_t stride = (int64_t)gridDim.x * THREADS;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  // software pipeline: the next sample's row is in flight while this one is binned
  double vn[RMAX];
  uint32_t cbn = 0;
  auto load = [&](int64_t i) {
    const double* row = s + i * r;
    if (EVEN) {
#pragma unroll
      for (int j = 0; j < RMAX; j += 2) {
        double2 x = make_double2(inf, inf);
        if (j < r) x = __ldg(reinterpret_cast<const double2*>(row + j));
        vn[j] = x.x;
        vn[j + 1] = x.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < RMAX; ++j) vn[j] = j < r ? __ldg(row + j) : inf;
    }
    cbn = __ldg(bits + i);
  };
  int64_t i = (int64_t)blockIdx.x * THREADS + threadIdx.x;
  if (i < n) load(i);
  for (; i < n; i += stride) {
    double v[RMAX];
#pragma unroll
    for (int j = 0; j < RMAX; ++j) v[j] = vn[j];
    const uint32_t cb = cbn;
    if (i + stride < n) load(i + stride);
    corrR += (cb >> r) & 1u;
    // b only moves when the (NaN-skipping) prefix minimum does, so the table
    // lookup and the two interval updates run only on new-minimum ramps:
    // inactive lanes put no traffic on the shared-memory banks.
    double mn = inf;  // +inf start: an all-NaN or empty prefix keeps b = m
    int prev = m;     // b_{j-1}
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
      if (v[j] < mn) {  // false for NaN and for the +inf padding past r
        mn = v[j];
        const int b = bucket<SINGLE>(su, slo, sth, g, mn);
        if (b < prev) {
          int* row = D + j * 2 * W + ((cb >> j) & 1u);  // columns interleave (p, correct)
          atomicAdd(row + 2 * b, 1);
          atomicAdd(row + 2 * prev, -1);
          prev = b;
        }
      }
    }
    // no-exit site r: interval [0, b_{r-1})
    int* rowr = D + r * 2 * W + ((cb >> r) & 1u);
    if (prev > 0) {
      atomicAdd(rowr, 1);
      atomicAdd(rowr + 2 * prev, -1);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) corrR += __shfl_xor_sync(0xffffffffu, corrR, o);
  if ((threadIdx.x & 31) == 0 && corrR)
    atomicAdd(reinterpret_cast<unsigned long long*>(gD + dstride), (unsigned long long)corrR);
  __syncthreads();
  for (int k = threadIdx.x; k < dstride; k += THREADS) {
    long long a = 0;
    for (int c = 0; c < copies; ++c) a += sD[c * dstride + k];
    if (a) atomicAdd(reinterpret_cast<unsigned long long*>(gD + k), (unsigned long long)a);
  }
  // last CTA to finish turns the difference arrays into per-candidate results
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  long long* cum = reinterpret_cast<long long*>(sD);  // [rows][m] (fits: copies*dstride*4 >= rows*m*8 checked on host)
  // cum[(2*site + c) * m + p] from the interleaved layout gD[site*2W + 2p + c]
  for (int k = threadIdx.x; k < rows * m; k += THREADS) {
    const int rr = k / m, p = k % m;
    cum[k] = __ldcg(gD + (rr >> 1) * 2 * W + 2 * p + (rr & 1));
  }
  __syncthreads();
  for (int rr = threadIdx.x; rr < rows; rr += THREADS) {
    long long run = 0;
    for (int p = 0; p < m; ++p) {
      run += cum[rr * m + p];
      cum[rr * m + p] = run;
    }
  }
  __syncthreads();
  for (int64_t c = threadIdx.x; c < C; c += THREADS) {
    const int p = pos[c];
    double hi = 0.0, lo = 0.0;
    long long ok = 0;
    for (int site = 0; site <= r; ++site) {
      long long cnt;
      if (p < 0) {  // NaN threshold row: nothing ever exits
        cnt = site == r ? n : 0;
      } else {
        const long long cc = cum[(2 * site + 1) * m + p];
        cnt = cum[2 * site * m + p] + cc;
        ok += cc;
      }
      if (hist_out) hist_out[c * (r + 1) + site] = cnt;
      const double x = (double)cnt;
      const double pr = __dmul_rn(x, serve[site]);
      const double pe = __fma_rn(x, serve[site], -pr);
      double sm, e;
      two_sum(hi, pr, sm, e);
      hi = sm;
      lo = __dadd_rn(lo, __dadd_rn(e, pe));
    }
    if (p < 0) ok = __ldcg(gD + dstride);  // never-exiting row: #samples with bit r set
    double tot, e;
    two_sum(hi, lo, tot, e);
    if (ok_out) ok_out[c] = ok;
    if (acc) {
      const double dn = (double)n;
      acc[c] = __ddiv_rn((double)ok, dn);
      sav[c] = __dsub_rn(vanilla, __ddiv_rn(tot, dn));
    }
  }
}

}  // namespace diag
