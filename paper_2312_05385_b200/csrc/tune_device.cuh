// tune_device.cuh — Algorithm 1 (threshold hill climbing, reference
// pkg/src/eesim/tuner.py:97-171) run entirely on the device: one CTA keeps the
// hill-climb state in shared memory, every round's tentative increments are
// scored with the exact (Cython-order) evaluation, and thread 0 applies the
// reference's selection rule with the same IEEE operations. The host sees one
// launch and one copy-back instead of a Python round trip per round
// (SURVEY §8f #2). Included by eeb200.cu.
#pragma once

namespace tunedev {

constexpr int THREADS = 512;
constexpr int MAXR = 31;
constexpr double ACC_EPS = 1e-12;

struct Params {
  double budget, init_step, min_step;
  int max_rounds;  // reference raises after 200000
  int trace_cap;   // rows of `trace` available (r doubles each)
  double serve[MAXR + 1];  // serve table (by value: no staging copy)
  long long* prof;         // optional: clock64 cycles per phase [8] (ee_tune_profile)
};

// out_d: [0, r) thresholds, r: savings, r+1: accuracy
// out_i: 0 rounds, 1 evals, 2 trace rows written, 3 status (0 ok, 1 budget violated,
//        2 did not terminate)
template <int RB>  // register slots for one sample's scores (RB >= r)
__global__ void __launch_bounds__(THREADS, 1)
    k_tune(const double* __restrict__ s, const uint32_t* __restrict__ bits, int n, int r,
           double vanilla, const __grid_constant__ Params p,
           double* __restrict__ vals, double* __restrict__ out_d, int* __restrict__ out_i,
           double* __restrict__ trace, int window_in_smem, int rows_in_smem) {
  // Every round re-scans the window and folds the addend rows sequentially, so
  // both live in shared memory when they fit: [addends f64 (r+1) x n8][bits u32 n][window]
  extern __shared__ __align__(16) unsigned char sdyn[];
  const int n8s = (n + 7) & ~7;
  const double* win = s;
  int64_t wsi = r, wsj = 1;  // score (i, j) at win[i * wsi + j * wsj]
  const uint32_t* wbits = bits;
  if (rows_in_smem) {
    vals = reinterpret_cast<double*>(sdyn);
    uint32_t* sb = reinterpret_cast<uint32_t*>(sdyn + (size_t)(r + 1) * n8s * 8);
    for (int k = threadIdx.x; k < n; k += THREADS) sb[k] = bits[k];
    wbits = sb;
    if (window_in_smem) {
      double* sw = reinterpret_cast<double*>(sdyn + (size_t)(r + 1) * n8s * 8 + (size_t)n8s * 4);
      // transposed [r][n8]: a warp's lanes (consecutive samples) read consecutive words
      for (int64_t k = threadIdx.x; k < (int64_t)n * r; k += THREADS) {
        const int64_t i = k / r, j = k - i * r;
        sw[j * n8s + i] = s[k];
      }
      win = sw;
      wsi = 1;
      wsj = n8s;
    }
  }
  __shared__ double th[MAXR], steps[MAXR], cand[MAXR + 1][MAXR], accs[MAXR + 1], savs[MAXR + 1];
  __shared__ double sserve[MAXR + 1];
  __shared__ int elig[MAXR], posof[MAXR], nelig, done;
  __shared__ double acc_cur, sav_cur;
  __shared__ int n_evals, n_rows, status;
  const int tid = threadIdx.x;
  for (int j = tid; j <= r; j += THREADS) sserve[j] = p.serve[j];
  if (tid < r) {
    th[tid] = 0.0;
    steps[tid] = p.init_step;
  }
  __syncthreads();

  // exact evaluation of rows cand[0..nc): every sample's first exit in parallel,
  // written as its serve value (the fold's addend) while the correct counts are
  // summed with ballots (integer sums are order-free); then one warp per
  // candidate folds the addends in index order (same order and the same
  // roundings as _exitcore.pyx:43-53; osum::warp_ordered_sum).
  const int n8 = (n + 7) & ~7;
  __shared__ unsigned okc[MAXR + 1];  // n <= EE_TUNE_N_MAX: 32-bit counts, native shared atomics
  // optional phase profile (thread 0's clock): 0 candidates, 1 scan, 2 fold, 3 select, 4 update
  long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tc = clock64();
  auto mark = [&](int k) {
    if (p.prof && tid == 0) {
      const long long t = clock64();
      ph[k] += t - tc;
      tc = t;
    }
  };
  // delta: candidate c is the current thresholds th with only ramp elig[c]
  // raised (every round after the first), so its exit site is the current one
  // unless that ramp now fires first: site_c = (site0 > i && x_i < up_i) ? i : site0
  auto evaluate = [&](int nc, bool delta) {
    if (tid <= MAXR) okc[tid] = 0;
    __syncthreads();
    const int lane = tid & 31;
    // (candidate, sample) pairs flattened over all threads: a warp's 32 pairs
    // share one candidate (samples padded to 32), so small windows use every warp
    if (n >= THREADS) {
      // large windows: a thread per sample; its scores are read once into registers
      // (RB >= r, the extra slots predicated off) and scanned for every candidate
      for (int i0 = 0; i0 < n; i0 += THREADS) {  // warp-uniform trip count for the ballots
        const int i = i0 + tid;
        const bool valid = i < n;
        double x[RB];
#pragma unroll
        for (int j = 0; j < RB; ++j) x[j] = (valid && j < r) ? win[(int64_t)i * wsi + j * wsj] : 0.0;
        const uint32_t wb = valid ? wbits[i] : 0u;
        auto emit = [&](int c, int site) {
          unsigned hit = 0;
          if (valid) {
            vals[(int64_t)c * n8 + i] = sserve[site];
            hit = (wb >> site) & 1u;
          }
          const unsigned b = __ballot_sync(0xffffffffu, hit);
          if (lane == 0 && b) atomicAdd(&okc[c], (unsigned)__popc(b));
        };
        if (delta) {
          int site0 = r;
#pragma unroll
          for (int j = RB - 1; j >= 0; --j)
            if (j < r && x[j] < th[j]) site0 = j;
          // one candidate per eligible ramp: loop over the ramps (static
          // register indices), candidate slot posof[j] (-1: not eligible)
#pragma unroll
          for (int j = 0; j < RB; ++j) {
            if (j >= r) break;
            const int c = posof[j];
            if (c < 0) continue;
            emit(c, (site0 > j && x[j] < cand[c][j]) ? j : site0);
          }
        } else {
          for (int c = 0; c < nc; ++c) {
            int site = r;
#pragma unroll
            for (int j = RB - 1; j >= 0; --j)
              if (j < r && x[j] < cand[c][j]) site = j;
            emit(c, site);
          }
        }
      }
    } else {
    const int n32 = (n + 31) & ~31;
    const int total = nc * n32;
    for (int t0 = 0; t0 < total; t0 += THREADS) {  // warp-uniform trip count for the ballot
      const int t = t0 + tid;
      const int c = t / n32, i = t - c * n32;
      unsigned hit = 0;
      if (c < nc && i < n) {
        const double* row = win + (int64_t)i * wsi;
        int site = r;
        for (int j = r - 1; j >= 0; --j)  // branch-free: every score is read, earliest hit wins
          if (row[j * wsj] < cand[c][j]) site = j;
        vals[(int64_t)c * n8 + i] = sserve[site];
        hit = (wbits[i] >> site) & 1u;
      }
      const unsigned b = __ballot_sync(0xffffffffu, hit);
      if (lane == 0 && b) atomicAdd(&okc[c], (unsigned)__popc(b));
    }
    }
    __syncthreads();
    mark(1);
    // the fold: a warp per candidate sums the addends in index order, bit for
    // bit the sequential chain, 128 at a time (osum::warp_ordered_sum)
    for (int c = tid >> 5; c < nc; c += THREADS / 32) {
      const double* vr = vals + (int64_t)c * n8;
      const double ms = osum::warp_ordered_sum(0.0, n, [&](int i) { return vr[i]; });
      if (lane == 0) {
        const double dn = (double)n;
        accs[c] = __ddiv_rn((double)okc[c], dn);
        savs[c] = __dsub_rn(vanilla, __ddiv_rn(ms, dn));
      }
    }
    __syncthreads();
    mark(2);
  };

  if (tid < r) cand[0][tid] = 0.0;
  __syncthreads();
  evaluate(1, false);
  const double floor = __dsub_rn(1.0, p.budget);
  const double floor_eps = __dsub_rn(floor, ACC_EPS);
  if (tid == 0) {
    acc_cur = accs[0];
    sav_cur = savs[0];
    done = 0;
    // counters live in shared memory; out_i / trace may be mapped host memory
    // (ee_tune), which the kernel only ever writes
    n_evals = 1;
    n_rows = 0;
    status = 0;
    if (p.trace_cap > 0) {
      for (int j = 0; j < r; ++j) trace[j] = steps[j];
      n_rows = 1;
    }
  }
  __syncthreads();
  int rounds = 0;
  while (true) {
    ++rounds;
    if (tid < 32) {  // eligible ramps in index order (r <= 31: one warp)
      const bool e = tid < r && th[tid] < 1.0;
      const unsigned m = __ballot_sync(0xffffffffu, e);
      const int pos = __popc(m & ((1u << tid) - 1));
      if (e) elig[pos] = tid;
      if (tid < MAXR) posof[tid] = e ? pos : -1;
      if (tid == 0) nelig = __popc(m);
    }
    __syncthreads();
    if (nelig == 0) break;
    for (int q = tid; q < nelig * r; q += THREADS) {  // candidate rows, all entries in parallel
      const int pos = q / r, j = q - pos * r;
      const int i = elig[pos];
      double v = th[j];
      if (j == i) {
        const double up = __dadd_rn(th[i], steps[i]);
        v = up < 1.0 ? up : 1.0;
      }
      cand[pos][j] = v;
    }
    __syncthreads();
    mark(0);
    evaluate(nelig, true);
    __shared__ int s_best;
    __shared__ unsigned s_viol;
    __shared__ bool s_allmin;
    if (tid < 32) {
      // every eligible increment scored by its own lane; key (1, dsav, -i) when
      // it loses no accuracy, else (0, dsav / dloss, dsav, -i)
      const int pos = tid;
      const bool valid = pos < nelig;
      const int i = valid ? elig[pos] : 0;
      const bool viol_me = valid && accs[pos] < floor_eps;
      bool ok = valid && !viol_me;
      int k0 = 0;
      double k1 = 0.0, k2 = 0.0;
      if (ok) {
        const double dsav = __dsub_rn(savs[pos], sav_cur);
        const double dloss = __dsub_rn(acc_cur, accs[pos]);
        if (dloss <= ACC_EPS) {
          k0 = 1;
          k1 = dsav;
        } else {
          k1 = __ddiv_rn(dsav, dloss);
          k2 = dsav;
        }
      }
      mark(5);
      // lane 0 scans the keys in index order keeping the first maximum: the
      // reference's in-order scan itself (tuner.py:141-153)
      __shared__ double s_k1[MAXR], s_k2[MAXR];
      __shared__ int s_k0[MAXR], s_ok[MAXR];
      if (valid) {
        s_ok[pos] = ok;
        s_k0[pos] = k0;
        s_k1[pos] = k1;
        s_k2[pos] = k2;
      }
      __syncwarp();
      int best = -1;
      if (pos == 0) {
        int b0 = 0;
        double b1 = 0.0, b2 = 0.0;
        for (int q = 0; q < nelig; ++q) {
          if (!s_ok[q]) continue;
          const int c0 = s_k0[q];
          const double c1 = s_k1[q], c2 = s_k2[q];
          bool take = best < 0;
          if (!take) {
            if (c0 != b0)
              take = c0 > b0;
            else if (c1 != b1)
              take = c1 > b1;
            else if (c0 == 0 && c2 != b2)
              take = c2 > b2;
            // equal keys: the earlier index (larger -i) wins
          }
          if (take) best = q, b0 = c0, b1 = c1, b2 = c2;
        }
      }
      mark(6);
      unsigned vm = viol_me ? 1u << i : 0u;
#pragma unroll
      for (int o = 16; o; o >>= 1) vm |= __shfl_xor_sync(0xffffffffu, vm, o);
      const bool at_min = !valid || steps[i] <= __dadd_rn(p.min_step, ACC_EPS);
      const bool all_min = __all_sync(0xffffffffu, at_min);
      if (tid == 0) {
        s_best = best;
        s_viol = vm;
        s_allmin = all_min;
      }
    }
    __syncwarp();
    mark(3);
    if (tid == 0) {
      n_evals += nelig;
      const int best = s_best;
      const unsigned viol = s_viol;
      if (best >= 0) {
        const int i = elig[best];
        const double up = __dadd_rn(th[i], steps[i]);
        th[i] = up < 1.0 ? up : 1.0;
        acc_cur = accs[best];
        sav_cur = savs[best];
        steps[i] = __dmul_rn(steps[i], 2.0);
      } else if (s_allmin) {
        done = 1;
      }
      if (!done) {
        for (int i = 0; i < r; ++i)
          if (viol & (1u << i)) {
            const double h = __ddiv_rn(steps[i], 2.0);
            steps[i] = p.min_step > h ? p.min_step : h;  // Python max(min_step, h)
          }
        if (n_rows < p.trace_cap) {
          for (int j = 0; j < r; ++j) trace[n_rows * r + j] = steps[j];
          n_rows += 1;
        }
        if (rounds > p.max_rounds) {
          done = 1;
          status = 2;
        }
      }
    }
    __syncthreads();
    mark(4);
    if (done) break;
  }
  if (p.prof && tid == 0)
    for (int k = 0; k < 8; ++k) p.prof[k] = ph[k];
  if (tid == 0) {
    if (status == 0 && acc_cur < __dsub_rn(floor, 1e-9)) status = 1;
    out_i[0] = rounds;
    out_i[1] = n_evals;
    out_i[2] = n_rows;
    out_i[3] = status;
    for (int j = 0; j < r; ++j) out_d[j] = th[j];
    out_d[r] = sav_cur;
    out_d[r + 1] = acc_cur;
  }
}

}  // namespace tunedev
