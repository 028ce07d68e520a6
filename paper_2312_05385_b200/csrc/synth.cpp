// synth.cpp — columnar replay of the reference workload generator
// (pkg/src/eesim/trace.py:164-227) for window ingest at 1M-record scale
// (the per-record Python generator takes ~64 s per 1M).
//
// The caller supplies numpy's raw PCG64 output (Generator.bit_generator
// .random_raw) and this loop consumes it exactly as the reference's calls do:
//   Generator.random()      -> (next64 >> 11) * 2^-53
//   Generator.integers(k)   -> Lemire bounded 32-bit draw; 32-bit halves are
//                              buffered in the bit generator (low half first),
//                              k == 1 draws nothing.
// The replay is checked record-for-record against the Python generator and
// the reference's digests in the tests.
#pragma STDC FP_CONTRACT OFF
#include <cstdint>

#include "../../include/eeb200.h"

namespace {

struct Raw {
  const uint64_t* p;
  int64_t n;
  int64_t pos;
  int32_t has32;
  uint32_t buf;
  bool out;
  uint64_t next64() {
    if (pos >= n) {
      out = true;
      return 0;
    }
    return p[pos++];
  }
  uint32_t next32() {
    if (has32) {
      has32 = 0;
      return buf;
    }
    const uint64_t x = next64();
    has32 = 1;
    buf = (uint32_t)(x >> 32);
    return (uint32_t)x;
  }
  double random() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
  int64_t integers(int64_t k) {
    const uint32_t rng = (uint32_t)(k - 1);
    if (rng == 0) return 0;
    const uint32_t excl = rng + 1;
    uint64_t m = (uint64_t)next32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (0xFFFFFFFFu - rng) % excl;
      while (left < thr && !out) {
        m = (uint64_t)next32() * excl;
        left = (uint32_t)m;
      }
    }
    return (int64_t)(m >> 32);
  }
};

}  // namespace

extern "C" int ee_synth_columns(const uint64_t* raw, int64_t n_raw, int64_t* io_pos,
                                int32_t* io_has32, uint32_t* io_buf, const double* u, int64_t n,
                                int64_t t_begin, int64_t* t_end, double* io_d_prev,
                                int32_t n_sites, const double* agree_early,
                                const double* agree_late, int32_t use_late, double continuity,
                                double miscal, double miscal_late, int32_t n_labels,
                                double* errs, int32_t* labels, int32_t* finals) {
  if (!raw || !io_pos || !io_has32 || !io_buf || !u || !t_end || !io_d_prev || !agree_early ||
      !agree_late || !errs || !labels || !finals || n_sites < 1 || n_labels < 2)
    return EE_ERR_ARG;
  Raw s{raw, n_raw, *io_pos, *io_has32, *io_buf, false};
  double d_prev = *io_d_prev;
  const int64_t half = n / 2;
  int64_t t = t_begin;
  for (; t < n; ++t) {
    const Raw snap = s;
    const double d = t == 0 ? u[0] : continuity * d_prev + (1.0 - continuity) * u[t];
    const double* curve = (t < half || !use_late) ? agree_early : agree_late;
    const double mc = t < half ? miscal : miscal_late;
    const int64_t final_label = s.integers(n_labels);
    double* erow = errs + t * n_sites;
    int32_t* lrow = labels + t * n_sites;
    for (int j = 0; j < n_sites; ++j) {
      const double a = curve[j];
      const double p_agree = a + (1.0 - a) * (1.0 - d);
      const bool agrees = s.random() < p_agree;
      const double low = 0.5 * d * s.random();
      if (agrees) {
        erow[j] = low;
        lrow[j] = (int32_t)final_label;
        continue;
      }
      const int64_t off = s.integers(n_labels - 1);
      lrow[j] = (int32_t)((final_label + 1 + off) % n_labels);
      if (s.random() < mc)
        erow[j] = low;
      else
        erow[j] = 1.0 - 0.5 * (1.0 - d) * s.random();
    }
    if (s.out) {  // buffer ran dry mid-record: roll back, caller refills
      s = snap;
      break;
    }
    finals[t] = (int32_t)final_label;
    d_prev = d;
  }
  *io_pos = s.pos;
  *io_has32 = s.has32;
  *io_buf = s.buf;
  *io_d_prev = d_prev;
  *t_end = t;
  return EE_OK;
}
