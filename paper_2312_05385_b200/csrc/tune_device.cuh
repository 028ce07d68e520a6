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
};

// out_d: [0, r) thresholds, r: savings, r+1: accuracy
// out_i: 0 rounds, 1 evals, 2 trace rows written, 3 status (0 ok, 1 budget violated,
//        2 did not terminate)
__global__ void __launch_bounds__(THREADS, 1)
    k_tune(const double* __restrict__ s, const uint32_t* __restrict__ bits, int n, int r,
           const double* __restrict__ serve, double vanilla, Params p,
           unsigned char* __restrict__ sites, double* __restrict__ out_d, int* __restrict__ out_i,
           double* __restrict__ trace, int window_in_smem, int rows_in_smem) {
  // Every round re-scans the window and folds the site rows sequentially, so
  // both live in shared memory when they fit: [bits u32 n][sites (r+1) x n8][window]
  extern __shared__ __align__(16) unsigned char sdyn[];
  const int n8s = (n + 7) & ~7;
  const double* win = s;
  const uint32_t* wbits = bits;
  if (rows_in_smem) {
    uint32_t* sb = reinterpret_cast<uint32_t*>(sdyn);
    for (int k = threadIdx.x; k < n; k += THREADS) sb[k] = bits[k];
    wbits = sb;
    sites = sdyn + (size_t)n8s * 4;
    if (window_in_smem) {
      double* sw = reinterpret_cast<double*>(sdyn + (size_t)n8s * 4 + (size_t)(r + 1) * n8s);
      for (int64_t k = threadIdx.x; k < (int64_t)n * r; k += THREADS) sw[k] = s[k];
      win = sw;
    }
  }
  __shared__ double th[MAXR], steps[MAXR], cand[MAXR + 1][MAXR], accs[MAXR + 1], savs[MAXR + 1];
  __shared__ double sserve[MAXR + 1];
  __shared__ int elig[MAXR], nelig, done;
  __shared__ double acc_cur, sav_cur;
  const int tid = threadIdx.x;
  for (int j = tid; j <= r; j += THREADS) sserve[j] = serve[j];
  if (tid < r) {
    th[tid] = 0.0;
    steps[tid] = p.init_step;
  }
  __syncthreads();

  // exact evaluation of rows cand[0..nc): sites in parallel, then one thread per
  // candidate folds samples in index order (same order as _exitcore.pyx:43-53)
  // per-candidate site rows, padded to 8 samples so the fold reads 8 at a time
  const int n8 = (n + 7) & ~7;
  auto evaluate = [&](int nc) {
    for (int c = 0; c < nc; ++c) {
      for (int i = tid; i < n; i += THREADS) {
        const double* row = win + (int64_t)i * r;
        int site = r;
        for (int j = r - 1; j >= 0; --j)  // branch-free: every score is read, earliest hit wins
          if (row[j] < cand[c][j]) site = j;
        sites[(int64_t)c * n8 + i] = (unsigned char)site;
      }
    }
    __syncthreads();
    if (tid < nc) {
      const unsigned char* st = sites + (int64_t)tid * n8;
      long long ok = 0;
      double ms = 0.0;
      const int nfull = n & ~7;
      for (int i0 = 0; i0 < nfull; i0 += 8) {
        // 8 independent shared loads per step; only the fp64 adds form a chain
        const uint2 sw = *reinterpret_cast<const uint2*>(st + i0);
        double add[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int site = ((q < 4 ? sw.x : sw.y) >> (8 * (q & 3))) & 0xFF;
          ok += (wbits[i0 + q] >> site) & 1u;
          add[q] = sserve[site];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) ms = __dadd_rn(ms, add[q]);
      }
      for (int i = nfull; i < n; ++i) {
        const int site = st[i];
        ok += (wbits[i] >> site) & 1u;
        ms = __dadd_rn(ms, sserve[site]);
      }
      const double dn = (double)n;
      accs[tid] = __ddiv_rn((double)ok, dn);
      savs[tid] = __dsub_rn(vanilla, __ddiv_rn(ms, dn));
    }
    __syncthreads();
  };

  if (tid < r) cand[0][tid] = 0.0;
  __syncthreads();
  evaluate(1);
  const double floor = __dsub_rn(1.0, p.budget);
  const double floor_eps = __dsub_rn(floor, ACC_EPS);
  if (tid == 0) {
    acc_cur = accs[0];
    sav_cur = savs[0];
    done = 0;
    out_i[0] = 0;
    out_i[1] = 1;
    out_i[2] = 0;
    out_i[3] = 0;
    if (p.trace_cap > 0) {
      for (int j = 0; j < r; ++j) trace[j] = steps[j];
      out_i[2] = 1;
    }
  }
  __syncthreads();
  int rounds = 0;
  while (true) {
    ++rounds;
    if (tid == 0) {
      int k = 0;
      for (int i = 0; i < r; ++i)
        if (th[i] < 1.0) elig[k++] = i;
      nelig = k;
      for (int pos = 0; pos < k; ++pos) {
        for (int j = 0; j < r; ++j) cand[pos][j] = th[j];
        const int i = elig[pos];
        const double up = __dadd_rn(th[i], steps[i]);
        cand[pos][i] = up < 1.0 ? up : 1.0;
      }
    }
    __syncthreads();
    if (nelig == 0) break;
    evaluate(nelig);
    if (tid == 0) {
      out_i[1] += nelig;
      int best = -1;
      // key: (1, dsav, -i) when the increment loses no accuracy, else
      // (0, dsav / dloss, dsav, -i); lexicographic max (tuner.py:141-153)
      int bk0 = 0;
      double bk1 = 0.0, bk2 = 0.0;
      int bk3 = 0;
      unsigned viol = 0;
      for (int pos = 0; pos < nelig; ++pos) {
        const int i = elig[pos];
        if (accs[pos] < floor_eps) {
          viol |= 1u << i;
          continue;
        }
        const double dsav = __dsub_rn(savs[pos], sav_cur);
        const double dloss = __dsub_rn(acc_cur, accs[pos]);
        int k0;
        double k1, k2;
        if (dloss <= ACC_EPS) {
          k0 = 1;
          k1 = dsav;
          k2 = 0.0;
        } else {
          k0 = 0;
          k1 = __ddiv_rn(dsav, dloss);
          k2 = dsav;
        }
        const int k3 = -i;
        bool better;
        if (best < 0)
          better = true;
        else if (k0 != bk0)
          better = k0 > bk0;
        else if (k1 != bk1)
          better = k1 > bk1;
        else if (k0 == 0 && k2 != bk2)
          better = k2 > bk2;
        else
          better = k3 > bk3;
        if (better) {
          best = pos;
          bk0 = k0;
          bk1 = k1;
          bk2 = k2;
          bk3 = k3;
        }
      }
      if (best >= 0) {
        const int i = elig[best];
        const double up = __dadd_rn(th[i], steps[i]);
        th[i] = up < 1.0 ? up : 1.0;
        acc_cur = accs[best];
        sav_cur = savs[best];
        steps[i] = __dmul_rn(steps[i], 2.0);
      } else {
        bool all_min = true;
        for (int pos = 0; pos < nelig; ++pos)
          if (!(steps[elig[pos]] <= __dadd_rn(p.min_step, ACC_EPS))) all_min = false;
        if (all_min) done = 1;
      }
      if (!done) {
        for (int i = 0; i < r; ++i)
          if (viol & (1u << i)) {
            const double h = __ddiv_rn(steps[i], 2.0);
            steps[i] = p.min_step > h ? p.min_step : h;  // Python max(min_step, h)
          }
        if (out_i[2] < p.trace_cap) {
          for (int j = 0; j < r; ++j) trace[out_i[2] * r + j] = steps[j];
          out_i[2] += 1;
        }
        if (rounds > p.max_rounds) {
          done = 1;
          out_i[3] = 2;
        }
      }
    }
    __syncthreads();
    if (done) break;
  }
  if (tid == 0) {
    out_i[0] = rounds;
    for (int j = 0; j < r; ++j) out_d[j] = th[j];
    out_d[r] = sav_cur;
    out_d[r + 1] = acc_cur;
    if (out_i[3] == 0 && acc_cur < __dsub_rn(floor, 1e-9)) out_i[3] = 1;
  }
}

}  // namespace tunedev
