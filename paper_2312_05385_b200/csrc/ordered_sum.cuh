// ordered_sum.cuh — the reference's sequential fp64 sum, (((S + a0) + a1) + ...)
// with every addition rounded (the Cython loop of _exitcore.pyx:43-53), computed
// by a warp bit for bit but 128 addends at a time. Included by eeb200.cu.
//
// While the running sum S stays in one binade [2^E, 2^(E+1)), every result is a
// multiple of u = 2^(E-52), S = N u with N in [2^52, 2^53), and for an addend
// a >= 0 with a / u = q + f (q integer, 0 <= f < 1):
//   fl(S + a) = (N + q + [f > 1/2]) u        unless f = 1/2 (a tie: the even
//                                             neighbour, which depends on N).
// So without ties the integer increments q + [f > 1/2] are independent of S and
// a warp prefix-sums them; the first addend whose N would reach 2^53 (the sum
// leaves the binade, the grid coarsens) is added with one real __dadd_rn from
// the exact sum before it, and the scan restarts from there. A chunk with a
// tie, a negative or non-finite addend, or a subnormal / zero S runs as the
// plain __dadd_rn chain. The sum crosses ~log2(n) binades, so nearly every
// chunk takes the parallel path.
#pragma once

namespace osum {

constexpr int PER_LANE = 4;  // addends per lane per chunk: 128 per warp step (2 and 8 measured slower)

// get(i) -> addend i (0 <= i < n); every lane of the warp must call this with
// the same S and n. Returns the sequential sum on every lane.
template <class Get>
__device__ __forceinline__ double warp_ordered_sum(double S, int n, Get get) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const long long TOP = 1LL << 53;
  int i0 = 0;
  while (i0 < n) {
    const int cnt = min(32 * PER_LANE, n - i0);
    double a[PER_LANE];
#pragma unroll
    for (int e = 0; e < PER_LANE; ++e) {
      const int i = lane * PER_LANE + e;
      a[e] = i < cnt ? get(i0 + i) : 0.0;
    }
    if (S == 0.0) {  // the first addend lands exactly; the grid exists from then on
      S = __dadd_rn(S, __shfl_sync(FULL, a[0], 0));
      i0 += 1;
      continue;
    }
    const unsigned long long sb = (unsigned long long)__double_as_longlong(S);
    const int ex = (int)((sb >> 52) & 0x7ff);
    bool fine = ex > 100 && ex < 0x7ff && !(sb >> 63);  // S normal, finite, positive, not tiny
#pragma unroll
    for (int e = 0; e < PER_LANE; ++e) fine = fine && a[e] >= 0.0 && a[e] < 1e300;  // NaN fails
    // u = 2^(E-52) and 1/u, both exact powers of two
    const double u = __longlong_as_double((long long)(ex - 52) << 52);
    const double inv_u = __longlong_as_double((long long)(1023 + 1023 + 52 - ex) << 52);
    long long x[PER_LANE];
    bool big[PER_LANE];
    bool tie = false;
#pragma unroll
    for (int e = 0; e < PER_LANE; ++e) {
      const double as = a[e] * inv_u;  // exact scaling
      big[e] = !(as < 4.0e15);         // this addend leaves the binade on its own
      const double fl = floor(big[e] ? 0.0 : as);
      const double fr = (big[e] ? 0.0 : as) - fl;  // exact
      tie = tie || fr == 0.5;
      x[e] = (long long)fl + (fr > 0.5 ? 1 : 0);
    }
    if (!__all_sync(FULL, fine) || __any_sync(FULL, tie)) {  // the plain chain for this chunk
      for (int i = 0; i < cnt; ++i) {
        const double ai = __shfl_sync(FULL, a[i % PER_LANE], i / PER_LANE);
        S = __dadd_rn(S, ai);
      }
      i0 += cnt;
      continue;
    }
    // lane-local inclusive prefix, then a warp scan of the lane totals
    long long p[PER_LANE];
    long long acc = 0;
#pragma unroll
    for (int e = 0; e < PER_LANE; ++e) p[e] = (acc += x[e]);
    long long incl = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const long long N0 = (long long)(S * inv_u);  // exact, in [2^52, 2^53)
    const long long base = N0 + incl - acc;       // N before this lane's first addend
    int first = PER_LANE;                         // this lane's first leaving addend
#pragma unroll
    for (int e = PER_LANE - 1; e >= 0; --e)
      if (lane * PER_LANE + e < cnt && (big[e] || base + p[e] >= TOP)) first = e;
    const unsigned cross = __ballot_sync(FULL, first < PER_LANE);
    if (!cross) {
      const int last = cnt - 1;
      const long long nl = __shfl_sync(FULL, base + acc, last / PER_LANE);  // lanes past cnt add 0
      S = (double)nl * u;
      i0 += cnt;
      continue;
    }
    const int k = __ffs(cross) - 1;
    const int e = __shfl_sync(FULL, first, k);
    // the exact sum before addend (k, e) (N of the addend before it: < 2^53,
    // exact as a double) plus that addend, rounded once, as the chain would
    long long before = base;
    double ak = 0.0;
#pragma unroll
    for (int q = 0; q < PER_LANE; ++q) {
      if (q + 1 == first) before = base + p[q];
      if (q == first) ak = a[q];
    }
    const long long nb = __shfl_sync(FULL, before, k);
    ak = __shfl_sync(FULL, ak, k);
    S = __dadd_rn((double)nb * u, ak);
    i0 += k * PER_LANE + e + 1;
  }
  return S;
}

}  // namespace osum
