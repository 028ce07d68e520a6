/*
 * eeb200.h — C ABI of the B200 (sm_100a) early-exit decision kernels.
 *
 * This is the drop-in boundary for the exit-decision seam of the reference
 * package `eesim` (arXiv 2312.05385, "Apparate"): the module
 * `eesim._kernels` (pkg/src/eesim/_kernels/__init__.py:14-48) exposes two
 * callables, `exit_sites` and `eval_thresholds`, implemented in Cython
 * (pkg/src/eesim/_kernels/_exitcore.pyx:11-56) with a numpy twin
 * (pkg/src/eesim/_kernels/_ref.py:17-62). Every entry point below names the
 * reference function it replaces.
 *
 * Conventions
 *   - Plain C types only. Pointers prefixed d_ are DEVICE pointers (caller
 *     owned, any allocator); pointers prefixed h_ are HOST pointers. Control
 *     data (thresholds, serve table) is host-side: it is at most C*R doubles and
 *     the library derives its device tables from it.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *     Every call is asynchronous with respect to the host unless stated.
 *   - Return value: 0 on success, a negative EE_ERR_* code otherwise;
 *     ee_last_error() returns a thread-local message for the last failure.
 *     Shapes are validated here; nothing is undefined behaviour (the Cython
 *     reference silently reads out of bounds on a short threshold vector).
 *   - Semantics (pkg/src/eesim/_kernels/_ref.py:1-6, _exitcore.pyx:19-21):
 *     a record exits at the first ramp j with scores[i,j] < thresholds[j]
 *     (strict IEEE compare, so NaN never exits); site R means "no exit".
 */
#ifndef EEB200_H
#define EEB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EE_OK 0
#define EE_ERR_ARG (-1)        /* bad shape / size / null pointer */
#define EE_ERR_CUDA (-2)       /* CUDA runtime failure */
#define EE_ERR_NOT_BINARY (-3) /* correct_ext holds a value other than 0.0 / 1.0 */
#define EE_ERR_RAMPS (-4)      /* more ramps than the kernels support (R > 31) */

#define EE_MODE_AUTO 0  /* exact below EE_EXACT_N_MAX samples, histogram above */
#define EE_MODE_EXACT 1 /* per-candidate in-order fp64 sums: bit-identical to _exitcore.pyx:43-55 */
#define EE_MODE_HIST 2  /* integer exit-site histograms; acc exact, sav exactly rounded */
/* OR-ed into `mode`: scores/bits are immutable device buffers (a resident window
 * whose producers completed before this call). The diagonal sweep may then start
 * streaming them while the previous sweep on the stream finishes (programmatic
 * dependent launch); its own side effects still wait for that sweep. */
#define EE_MODE_FLAG_RESIDENT 0x100
#define EE_EXACT_N_MAX 4096

#define EE_MAX_RAMPS 31

typedef struct ee_workspace ee_workspace;

/* Library / device information. */
const char* ee_version(void);
const char* ee_last_error(void);
int ee_device_sm_count(int32_t* out_sms);

/* Scratch owner: device buffers for keys, histograms and threshold tables, a
 * pinned staging area and an event. One workspace per host thread (calls on
 * one workspace are serialised by an internal mutex). */
int ee_workspace_create(ee_workspace** out);
int ee_workspace_destroy(ee_workspace* ws);

/* Replaces _exitcore.exit_sites (pkg/src/eesim/_kernels/_exitcore.pyx:11-24)
 * and _ref.exit_sites (_ref.py:17-27).
 *   d_scores  f64 [n, r] row-major, d_th f64 [r], d_out i64 [n] in [0, r]. */
int ee_exit_sites(const double* d_scores, int64_t n, int32_t r, const double* d_th,
                  int64_t* d_out, void* stream);

/* Packs the reference's correctness matrix correct_ext f64 [n, r1] (r1 = r+1,
 * built at pkg/src/eesim/engine.py:154-159) into one uint32 bit row per
 * sample (bit j = column j). Every entry must be exactly 0.0 or 1.0; any other
 * value sets *d_flag to 1 (the host maps that to EE_ERR_NOT_BINARY). */
int ee_pack_correct(const double* d_correct_ext, int64_t n, int32_t r1, uint32_t* d_bits,
                    int32_t* d_flag, void* stream);

/* Replaces engine.decision_scores (pkg/src/eesim/engine.py:106-121) for k > 1:
 * trailing mean of the last k active-ramp scores via the same cumulative-sum
 * difference, bit-identical to numpy. d_out may alias nothing. */
int ee_decision_scores(const double* d_errs, int64_t n, int32_t r, int32_t k, double* d_out,
                       void* stream);

/* Replaces _exitcore.eval_thresholds (pkg/src/eesim/_kernels/_exitcore.pyx:27-56),
 * _ref.eval_thresholds (_ref.py:30-62) as called by
 * WindowEvaluator.evaluate_many (pkg/src/eesim/engine.py:165-170).
 *   d_scores  f64 [n, r]; d_bits u32 [n] (from ee_pack_correct, r+1 columns)
 *   h_serve   f64 [r+1] (engine._serve_table, engine.py:124-132), vanilla f64
 *   h_th      f64 [c, r] candidate threshold rows
 *   outputs (device; acc/sav may both be NULL in HIST mode with d_hist/d_ok
 *   given — counts only, e.g. before a cross-rank all-reduce):
 *     d_hist  i64 [c, r+1] exit-site histogram (HIST mode only; zero-filled in EXACT)
 *     d_ok    i64 [c]      correct releases
 *     d_acc   f64 [c]      ok / n
 *     d_sav   f64 [c]      vanilla - (sum_i serve[site_i]) / n
 * n == 0 yields NaN acc/sav exactly like the reference's 0/0. */
int ee_eval_thresholds(ee_workspace* ws, const double* d_scores, const uint32_t* d_bits,
                       int64_t n, int32_t r, const double* h_serve, double vanilla,
                       const double* h_th, int64_t c, int32_t mode, int64_t* d_hist,
                       int64_t* d_ok, double* d_acc, double* d_sav, void* stream);

/* The same HIST-mode evaluation over nwin windows at once (same n, r and
 * candidate rows; d_scores_list / d_bits_list are DEVICE arrays of nwin device
 * pointers, each window laid out as for ee_eval_thresholds): one persistent
 * sweep launch that builds its tables once and streams the windows back to
 * back, then one finalisation launch. acc/sav are [nwin, c]. Diagonal
 * candidate rows only (every row repeats one threshold; <= 64 distinct
 * values, c <= 512, even r <= 16); anything else returns EE_ERR_ARG. */
int ee_eval_thresholds_windows(ee_workspace* ws, const double* const* d_scores_list,
                               const uint32_t* const* d_bits_list, int32_t nwin, int64_t n,
                               int32_t r, const double* h_serve, double vanilla, const double* h_th,
                               int64_t c, double* d_acc, double* d_sav, void* stream);

/* The counting half of ee_eval_thresholds_windows, for a caller that reduces
 * across ranks first (one all-reduce per K windows): exact
 * per-window totals into d_accw int64 [nwin, EE_WINDOW_ACC_WORDS] (zeroed here;
 * the all-reduce sums them), then ee_windows_finalize on the reduced totals
 * with the global sample count. */
#define EE_WINDOW_ACC_WORDS 2178
int ee_windows_counts(ee_workspace* ws, const double* const* d_scores_list,
                      const uint32_t* const* d_bits_list, int32_t nwin, int64_t n, int32_t r,
                      const double* h_th, int64_t c, int64_t* d_accw, void* stream);
int ee_windows_finalize(ee_workspace* ws, const int64_t* d_accw, int32_t nwin, int64_t n_total, int32_t r,
                        const double* h_serve, double vanilla, const double* h_th, int64_t c,
                        double* d_acc, double* d_sav, void* stream);

/* The same evaluation from HOST buffers (the reference's own calling
 * convention: numpy arrays in, numpy arrays out, engine.py:165-170):
 * h_scores f64 [n, r], h_correct_ext f64 [n, r+1] (0.0/1.0, else
 * EE_ERR_NOT_BINARY), h_serve f64 [r+1], h_th f64 [c, r] -> h_acc, h_sav f64
 * [c]. correct_ext is packed to 4-byte bit rows on n_threads host threads
 * (<= 0: all cores) while the scores stream to the device, so 8r + 4 bytes
 * per sample cross PCIe instead of 16r + 8. Synchronous. */
int ee_eval_thresholds_host(ee_workspace* ws, const double* h_scores, const double* h_correct_ext,
                            int64_t n, int32_t r, const double* h_serve, double vanilla,
                            const double* h_th, int64_t c, int32_t mode, double* h_acc,
                            double* h_sav, int32_t n_threads, void* stream);

/* The counting half of ee_eval_thresholds_host for a sample shard (SURVEY
 * §8e): the same host staging (bits packed on the CPU, 8r + 4 bytes per sample
 * over PCIe), then exact int64 per-candidate exit histograms d_hist [c, r+1]
 * and correct counts d_ok [c] on the device (HIST mode, no finalisation) —
 * the buffers a rank all-reduces before ee_finalize_hist. Returns once the
 * host inputs are no longer read. */
int ee_eval_counts_host(ee_workspace* ws, const double* h_scores, const double* h_correct_ext,
                        int64_t n, int32_t r, const double* h_th, int64_t c, int64_t* d_hist,
                        int64_t* d_ok, int32_t n_threads, void* stream);

/* Host-side packing of correct_ext f64 [n, r1] into u32 bit rows (bit j =
 * column j) on n_threads threads (<= 0: all cores); EE_ERR_NOT_BINARY if any
 * entry is not exactly 0.0 or 1.0. */
/* Host only (no device work): which sweep family a candidate matrix th [c, r]
 * belongs to, as eval dispatch sees it: *kind = 1 diagonal (every row repeats
 * one threshold; *n_values = distinct non-NaN thresholds), 2 single-coordinate
 * (rows equal a base vector except in at most one column; *n_values = distinct
 * non-NaN varied values; the base is written to base[r] when base is non-null),
 * 0 anything else. Replaces no reference function: it documents and tests the
 * family dispatch in front of _exitcore.eval_thresholds (_exitcore.pyx:27-56). */
int ee_classify_candidates(const double* h_th, int64_t c, int32_t r, int32_t* kind,
                           int32_t* n_values, double* base);

int ee_pack_correct_host(const double* h_correct_ext, int64_t n, int32_t r1, uint32_t* h_bits,
                         int32_t n_threads);

/* Scores the full lattice vals^r in lexicographic (meshgrid 'ij') row order
 * without materialising it — the candidate set of tuner.grid_oracle
 * (pkg/src/eesim/tuner.py:213-223) — and returns acc/sav per lattice point
 * (device, length L^r), computed in EXACT mode. h_vals must be ascending. */
int ee_eval_lattice(ee_workspace* ws, const double* d_scores, const uint32_t* d_bits, int64_t n,
                    int32_t r, const double* h_serve, double vanilla, const double* h_vals,
                    int32_t n_vals, double* d_acc, double* d_sav, void* stream);

/* Device-resident Algorithm 1: the whole threshold hill climb of
 * tuner.tune (pkg/src/eesim/tuner.py:97-171) in one single-CTA launch over a
 * device window (d_scores f64 [n, r], d_bits u32 [n]). Every round's tentative
 * increments are scored in EXACT mode and selected with the reference's key
 * (same IEEE operations), so thresholds, savings, accuracy, rounds, evals and
 * the step trace are bit-identical to the compiled reference.
 * Synchronous. Outputs: h_out f64 [r + 2] = thresholds, savings, accuracy;
 * h_info i32 [4] = rounds, evals, trace rows, status (0 ok, 1 accuracy
 * postcondition violated, 2 exceeded max_rounds); h_trace f64 [trace_cap, r]
 * (step vectors, first row = initial steps). n <= EE_TUNE_N_MAX. */
#define EE_TUNE_N_MAX 65536
int ee_tune(ee_workspace* ws, const double* d_scores, const uint32_t* d_bits, int64_t n, int32_t r,
            const double* h_serve, double vanilla, double acc_loss_budget, double init_step,
            double min_step, int32_t max_rounds, double* h_out, int32_t* h_info, double* h_trace,
            int32_t trace_cap, void* stream);

/* ---- Ramp heads / exit controller / compaction ----
 * One ramp over a batch of b rows, fused in one launch: global-average pool of
 * the ramp input (d_feat: NCHW [b, c, hw] when nhwc == 0, NHWC [b, hw, c]
 * when nhwc == 1; hw == 1 for pre-pooled inputs such as a token-0 hidden
 * state; fp32 or bf16 when feat_bf16), ramp FC (d_w [k, c] fp32/bf16, d_bias
 * [k] fp32 nullable, k <= 256), softmax confidence (conf 0: err = 1 - max p;
 * conf 1: err = H(p)/ln k), argmax label, and the reference exit rule
 * (double)err < threshold (strict, engine.py:207) for rows whose d_alive byte
 * is 1 (d_alive NULL = all alive). A non-NULL d_threshold (one device f64)
 * overrides `threshold`, so a captured CUDA graph picks up retuned
 * thresholds without re-capture. d_alive is updated in place (exiting rows
 * are cleared), so chaining ramps needs no extra launch. Outputs per row: d_err f32, d_label i32,
 * d_exit u8, optional d_logits f32 [b, k]. Then, in the same launch, the
 * surviving (alive, non-exiting) rows are compacted in ascending row order
 * into d_keep with their count in *d_nkeep (both NULL: no compaction, e.g. a
 * feedback-mode batch that keeps every row, and no cross-CTA step at all), and
 * each exiting row's (label, err, site) is scattered to its request slot
 * d_slot[row] (NULL = row index) in d_slot_label / d_slot_err / d_slot_site
 * (all NULL = no scatter). */
int ee_exit_controller(ee_workspace* ws, const void* d_feat, int32_t feat_bf16, int64_t b,
                       int32_t c, int32_t hw, int32_t nhwc, const void* d_w, int32_t w_bf16,
                       const float* d_bias, int32_t k, int32_t conf, double threshold,
                       const double* d_threshold, uint8_t* d_alive, const int32_t* d_slot,
                       int32_t site, float* d_err,
                       int32_t* d_label, uint8_t* d_exit, float* d_logits, int32_t* d_keep,
                       int32_t* d_nkeep, int32_t* d_slot_label, float* d_slot_err,
                       int32_t* d_slot_site, void* stream);

/* Same epilogue from precomputed fp32 logits [b, k] (large heads whose FC runs
 * as a tensor-core GEMM). */
int ee_exit_from_logits(ee_workspace* ws, const float* d_logits, int64_t b, int32_t k,
                        int32_t conf, double threshold, const double* d_threshold,
                        uint8_t* d_alive,
                        const int32_t* d_slot, int32_t site, float* d_err, int32_t* d_label,
                        uint8_t* d_exit, int32_t* d_keep, int32_t* d_nkeep, int32_t* d_slot_label,
                        float* d_slot_err, int32_t* d_slot_site, void* stream);

/* Tensor-core ramp-head GEMM: d_c f32 [m, n] = d_a bf16 [m, k] (row-major) x
 * d_b bf16 [n, k]^T (row-major, i.e. nn.Linear weight layout) + d_bias f32 [n]
 * (nullable). k % 8 == 0. Same kernels as ee_gemm_bf16_ex (act none, auto
 * path); `splits` > 0 pins the swap kernel's split count. Deterministic. */
int ee_gemm_bf16_tn(ee_workspace* ws, const void* d_a, const void* d_b, const float* d_bias,
                    float* d_c, int64_t m, int64_t n, int64_t k, int32_t splits, void* stream);

/* General form: d_c is fp32 [m, n], or bf16 [m, n] (round to nearest even)
 * when out_bf16 != 0 — ee_gemm_bf16_ex with no activation, auto path. */
int ee_gemm_bf16(ee_workspace* ws, const void* d_a, const void* d_b, const float* d_bias,
                 void* d_c, int32_t out_bf16, int64_t m, int64_t n, int64_t k, int32_t splits,
                 void* stream);

/* Backbone / head GEMM with a fused epilogue (csrc/gemm.cu):
 *   d_c [m, n] = act(d_a bf16 [m, k] x d_w bf16 [n, k]^T + d_bias f32 [n])
 * d_c is bf16 (out_bf16 != 0, round to nearest even) or f32. act: 0 none,
 * 1 GELU (erf), 2 GELU (tanh approximation), 3 ReLU. path: 0 auto, 1 swap-AB
 * weight-streaming kernel (cluster split-K, DSMEM reduction, any m), 2 / 4 / 3 / 5
 * the persistent CTA-pair kernel (cta_group::2, 256 x 256 / 192 / 128 / 64 tiles;
 * needs 16-byte output rows). Auto takes the swap kernel for m <= 256. k % 8 == 0,
 * all pointers 16-byte aligned. Results are deterministic. Replaces the
 * library GEMMs the reference's models would call. */
int ee_gemm_bf16_ex(ee_workspace* ws, const void* d_a, const void* d_w, const float* d_bias,
                    void* d_c, int32_t out_bf16, int32_t act, int64_t m, int64_t n, int64_t k,
                    int32_t splits, int32_t path, void* d_work, int64_t work_bytes, void* stream);

/* ee_gemm_bf16_ex with a residual added before the activation:
 *   d_c [m, n] = act(d_a x d_w^T + d_bias + d_res bf16 [m, n])
 * (a ResNet bottleneck's conv3 + shortcut + ReLU as one kernel over NHWC
 * activations). d_res may be NULL; when given, out_bf16 != 0, n % 8 == 0 and
 * d_res is 16-byte aligned. */
int ee_gemm_bf16_res(ee_workspace* ws, const void* d_a, const void* d_w, const float* d_bias,
                     const void* d_res, void* d_c, int32_t out_bf16, int32_t act, int64_t m,
                     int64_t n, int64_t k, int32_t splits, int32_t path, void* d_work,
                     int64_t work_bytes, void* stream);
/* Bytes of device workspace ee_gemm_bf16_ex needs for this call (split-K
 * partial tiles of the swap kernel; 0 when none). Pass a buffer at least this
 * large as d_work, or NULL to let the call take stream-ordered pool memory
 * (cudaMallocAsync). Negative on a bad shape. */
int64_t ee_gemm_workspace_size(int64_t m, int64_t n, int64_t k, int32_t splits, int32_t path,
                               int32_t out_bf16);

/* Global average pool NCHW [b, c, hw] (f32, or bf16 when x_bf16) -> bf16
 * [b, c] (round to nearest even): the A operand of a large ramp head. */
int ee_pool_bf16(const void* d_x, int32_t x_bf16, int64_t b, int32_t c, int32_t hw, void* d_out,
                 void* stream);
/* The same pool for a channels_last (NHWC) map [B, HW, C]: C contiguous, so a
 * CTA reads 64-channel rows and its 16 thread rows split the spatial extent
 * (no NCHW copy first). c must be a multiple of 4, d_x 8-byte aligned. */
int ee_pool_nhwc_bf16(const void* d_x, int32_t x_bf16, int64_t b, int32_t c, int32_t hw,
                      void* d_out, void* stream);

/* Gathers rows d_keep[0 .. *d_nkeep) of d_src (row_bytes each, multiple of
 * 16) into the dense d_dst (capacity max_rows rows): downstream blocks then
 * run only on the non-exited samples (compaction mode). */
/* KV-cache append for the token-level decoder (config 5, the reference's KV
 * fill for skipped layers, generative.py:170-273): qkv bf16 [b, q, 3, h, dh]
 * (a fused QKV projection), pos i64 [b, q] with 0 <= pos < t1; writes K and V
 * of every (b, i) into kv bf16 [2, b, h, t1, dh] at slot pos[b, i]. A warp per
 * (b, i, K|V, head) row; dh must be a multiple of 2 and at most 256. */
/* Token-level early exit (config 5): the reference decoder's deferral
 * schedule (generative.py:217-259) kept on the device, so a decode step is
 * [prefix layers -> ramp -> ee_defer_plan] then [suffix pass -> ee_defer_finish]
 * with no host round trip. All pointers are device memory; B sequences, C =
 * flush_cap + 1 chunk slots, N decode steps (history rows N + 1: row N is the
 * end flush). kind: 0 none, 1 carry, 2 cap, 3 end. */
typedef struct ee_defer_state {
  int32_t* step;      /* [1] current decode step */
  int32_t* n_def;     /* [B] parked tokens */
  int64_t* qpos;      /* [B] next suffix position */
  int32_t* def_step;  /* [B, C] step of the token parked in each slot */
  int32_t* mem_cnt;   /* [B] this step's suffix chunk size */
  int64_t* spos;      /* [B, C] suffix positions, -1 = padding */
  uint8_t* h_exit;    /* [N + 1, B] history: exited */
  float* h_err;       /* [N + 1, B] ramp error score */
  int32_t* h_lab;     /* [N + 1, B] ramp label */
  int32_t* h_final;   /* [N + 1, B] the model's own token */
  int32_t* h_cnt;     /* [N + 1, B] chunk size decided at each step */
  uint8_t* h_kind;    /* [N + 1, B] flush kind */
  int64_t* h_qbase;   /* [N + 1, B] first suffix position of the chunk */
  int32_t n_max;      /* N */
  int32_t pad_;
} ee_defer_state;

/* Park the ramp's hidden state d_h_ramp bf16 [B, d] in the chunk bf16 [B, C, d]
 * behind the parked ones, record (exit, err, label), and decide each sequence's
 * suffix chunk: a non-exiting token carries every parked one, a sequence with
 * flush_cap parked tokens flushes them (cap). d_fixed u8 [N, B] (nullable)
 * overrides the exit decisions (tests). end_mode: every parked token flushes
 * (end). Writes spos / mem_cnt / history; the caller then runs the suffix. */
int ee_defer_plan(const ee_defer_state* st, int32_t b, int32_t c, int32_t d, int32_t cap,
                  const void* d_h_ramp, void* d_chunk, const uint8_t* d_exits, const uint8_t* d_fixed,
                  const float* d_err, const int32_t* d_lab, int32_t end_mode, void* stream);

/* After the suffix pass: each flushed token's own output d_final_label i32
 * [B * C] goes to the history (and, if d_hidden_hist f32 [N + 1, B, C, d] is
 * given, the chunk's final hidden rows d_final_h f32 [B, C, d]); the next input
 * token d_cur i64 [B] is the ramp label of an exit, else the model's; d_ppos
 * and the step advance. */
int ee_defer_finish(const ee_defer_state* st, int32_t b, int32_t c, int32_t d, const int32_t* d_final_label,
                    const int32_t* d_lab, int64_t* d_cur, int64_t* d_ppos, const float* d_final_h,
                    float* d_hidden_hist, int32_t end_mode, void* stream);

int ee_kv_append_bf16(const void* d_qkv, const int64_t* d_pos, int64_t b, int32_t q, int32_t h,
                      int32_t dh, int64_t t1, void* d_kv, void* stream);

/* Fused residual add + LayerNorm for the decoder (config 5): h[r] += y[r]
 * (bf16, rounded like torch's add), then x[r] = LayerNorm(h[r]) * gamma + beta
 * (fp32 statistics, two-pass), bf16 throughout; y may be null (LayerNorm only).
 * One CTA of d / 8 threads per row; d a multiple of 8, at most 8192. */
/* Convolution as an implicit GEMM on the tcgen05 pair kernel (csrc/gemm.cu):
 * y bf16 NHWC [n, ho, wo, cout] = act(conv(x bf16 NHWC [n, h, w, c],
 * w bf16 [cout, kh, kw, c]) + bias f32 [cout] (nullable) + res bf16
 * [n, ho, wo, cout] (nullable)), ho = (h + 2 pad - kh) / stride + 1 (same for
 * wo); act 0 none / 3 ReLU. The A operand is never materialised: each k-tile
 * is one TMA im2col load (128 consecutive output pixels x 64 channels of one
 * filter tap, zero padding by the TMA unit). c % 64 == 0, cout % 8 == 0,
 * 16-byte aligned pointers; d_work / work_bytes: ee_conv_workspace_size bytes
 * (nullable when that is 0). (A ResNet's spatial convolutions.) */
int ee_conv_bf16(ee_workspace* ws, const void* d_x, int64_t n, int32_t h, int32_t w, int32_t c,
                 const void* d_w, int32_t cout, int32_t kh, int32_t kw, int32_t stride, int32_t pad,
                 const float* d_bias, const void* d_res, int32_t act, void* d_y, void* d_work,
                 int64_t work_bytes, void* stream);

/* Bytes of device workspace ee_conv_bf16 needs for this shape: > 0 when the
 * convolution has too few output tiles for the SMs and splits K (fp32
 * partials [splits, m, cout], summed in order by one epilogue pass), else 0. */
int64_t ee_conv_workspace_size(int64_t n, int32_t h, int32_t w, int32_t c, int32_t cout, int32_t kh,
                               int32_t kw, int32_t stride, int32_t pad);

/* The reference's sequential fp64 sum of each row of d_vals [rows, n]
 * (((0 + v0) + v1) + ...), every addition rounded, as _exitcore.pyx:43-53
 * folds serve times), bit for bit, one warp per row; the fold ee_tune uses. */
int ee_sequential_sum(const double* d_vals, int32_t n, int32_t rows, double* d_out, void* stream);

/* im2col of an NHWC bf16 map for a convolution with too few input channels
 * for ee_conv_bf16 (the 3-channel stem): out bf16 [n*ho*wo, kp]; filter row r
 * owns columns [r * seg, r * seg + kw * c) with seg = kw * c rounded up to 8
 * (column r * seg + s * c + ch = tap (r, s), channel ch); the gap columns
 * hold neighbouring finite input values and need ZERO weights; zeros past
 * kh * seg (kp % 8 == 0, kp / 8 <= 256) and outside the image. w * c % 8 == 0
 * and x 16-byte aligned. The GEMM (weights laid out the same way) then runs on
 * ee_gemm_bf16_res. */
int ee_im2col_bf16(const void* d_x, int64_t n, int32_t h, int32_t w, int32_t c, int32_t kh, int32_t kw,
                   int32_t stride, int32_t pad, int32_t kp, void* d_out, void* stream);

/* k x k max pooling (stride, pad; padding = -inf) of an NHWC bf16 map
 * [n, h, w, c] -> [n, ho, wo, c]; c % 8 == 0, 16-byte aligned pointers. */
int ee_maxpool_nhwc_bf16(const void* d_x, int64_t n, int32_t h, int32_t w, int32_t c, int32_t k,
                         int32_t stride, int32_t pad, void* d_out, void* stream);

/* Convolution epilogue over an NHWC bf16 map viewed as [m, c] rows:
 * y = act(x + bias[c] (+ res)) with act 0 none / 3 ReLU, bias f32 (nullable),
 * res bf16 [m, c] (nullable, e.g. a ResNet shortcut). c % 8 == 0, 16-byte
 * aligned pointers; y may alias x. For the convolutions the repo's GEMM does
 * not run (bias, ReLU and shortcut then cost one pass instead of three). */
int ee_bias_act_bf16(const void* d_x, const float* d_bias, const void* d_res, int32_t act, int64_t m,
                     int32_t c, void* d_y, void* stream);

int ee_add_layernorm_bf16(void* d_h, const void* d_y, const void* d_gamma, const void* d_beta,
                          double eps, int64_t rows, int32_t d, void* d_x, void* stream);

/* Length-aware decode attention for the token-level decoder (config 5): for
 * each (b, head) and each of q <= 8 queries (the fused QKV projection qkv bf16
 * [b, q, 3, h, dh]), softmax(q k^T / sqrt(dh)) v over keys 0 .. qpos[b, i] of
 * the layer's cache kv bf16 [2, b, h, t1, dh]: only the visible part of the
 * cache is read. Writes out bf16 [b, q, h, dh] (the o-projection's input).
 * dh = 64, q * t1 <= 51200. */
int ee_decode_attention_bf16(const void* d_qkv, const void* d_kv, const int64_t* d_qpos, int64_t b,
                             int32_t q, int32_t h, int32_t dh, int64_t t1, void* d_out,
                             void* stream);

int ee_compact_rows(const void* d_src, int64_t row_bytes, const int32_t* d_keep,
                    const int32_t* d_nkeep, int64_t max_rows, void* d_dst, void* stream);

/* Per-request signal tables of a compacted batch: d_err_table[d_rows[i]] =
 * d_err[i], d_label_table[d_rows[i]] = d_label[i] for i < n (one launch; the
 * padding rows' dummy slot is a valid table entry). */
int ee_scatter_signals(const float* d_err, const int32_t* d_label, const int32_t* d_rows, int64_t n,
                       float* d_err_table, int32_t* d_label_table, void* stream);

/* In-place compaction of d_buf [rows, row_bytes] (rows <= 8192, row_bytes % 16
 * == 0, 16-byte aligned) to the *d_nkeep survivors d_keep lists (ascending, as
 * the exit controller writes it): survivors below *d_nkeep stay in place and
 * the survivors at or above it move, ascending, into the exited rows' places
 * below it, so only those rows are copied. d_rows_out[p] = d_rows_in[source
 * row of p] (the source row index if d_rows_in is NULL) for p < *d_nkeep, else
 * `dummy`; d_alive_out[p] = p < *d_nkeep; *d_n_out = *d_nkeep when given. All
 * on the device, so it can sit inside a CUDA graph. */
int ee_compact_fill(void* d_buf, int64_t row_bytes, const int32_t* d_keep, const int32_t* d_nkeep,
                    int64_t rows, const int32_t* d_rows_in, int32_t dummy, int32_t* d_rows_out,
                    uint8_t* d_alive_out, int32_t* d_n_out, void* stream);

/* Compaction bookkeeping for the next stage of a compacted batch (capacity cap
 * rows): d_rows_out[i] = d_rows_in[d_keep[i]] (d_keep[i] if d_rows_in is NULL)
 * for i < *d_nkeep, else `dummy`; d_alive_out[i] = i < *d_nkeep; *d_n_out =
 * *d_nkeep when d_n_out is given. Everything stays on the device (no host
 * round trip), so it can sit inside a CUDA graph. */
int ee_compact_meta(const int32_t* d_keep, const int32_t* d_nkeep, const int32_t* d_rows_in,
                    int64_t cap, int32_t dummy, int32_t* d_rows_out, uint8_t* d_alive_out,
                    int32_t* d_n_out, void* stream);

/* Finalises externally reduced histograms (e.g. after an all-reduce across
 * ranks of per-shard d_hist/d_ok from ee_eval_thresholds in HIST mode):
 * d_hist i64 [c, r+1], d_ok i64 [c], n = total samples -> d_acc, d_sav with
 * the same arithmetic as HIST mode (acc = ok/n, exactly rounded savings). */
int ee_finalize_hist(ee_workspace* ws, const int64_t* d_hist, const int64_t* d_ok, int64_t c,
                     int32_t r, int64_t n, const double* h_serve, double vanilla, double* d_acc,
                     double* d_sav, void* stream);

/* Family-specialised sweeps (default on): HIST-mode evaluations whose rows
 * are diagonal (one threshold repeated on every ramp, <= 256 distinct values)
 * run the single-pass difference-array kernel instead of the generic SWAR
 * scan. Results are identical; 0 forces the generic path (tests, A/B). */
int ee_workspace_set_special(ee_workspace* ws, int32_t on);

/* Which diagonal-family kernel runs (default 2): 2 = k_diag2 (coalesced,
 * conflict-free bin table, predicated updates, one launch) wherever it
 * applies (even r <= 16, <= 127 distinct thresholds, 16-byte aligned scores),
 * else k_diag; 1 = k_diag only. Results are identical (A/B, tests). Calls on
 * one workspace must be stream-ordered: k_diag2 keeps a global accumulator in
 * the workspace that every launch leaves zeroed for the next. */
int ee_workspace_set_diag_version(ee_workspace* ws, int32_t version);

/* Benchmark aid: overwrites d_buf (bytes, > L2 size to evict it) with a
 * streaming-store kernel that uses the same max-shared carveout as the sweep
 * kernels, so an L2 flush between timed sweeps does not also reconfigure the
 * SMs' L1/shared split. */
int ee_l2_flush(void* d_buf, int64_t bytes, void* stream);

/* Profiling aid: while d_trace (device u64 [grid * 6], zeroed by the caller)
 * is set, every k_diag2 CTA records %globaltimer stamps (start, prologue done,
 * last warp out of the sweep loop, merged into the accumulator, and, for the
 * last CTA, finalised). NULL turns it off. */
int ee_diag_trace(ee_workspace* ws, uint64_t* d_trace);

/* Profiling aid: while d_cycles (device i64 [8]) is set, ee_tune writes the
 * clock64 cycles its thread 0 spent per phase over the whole hill climb:
 * candidate rows, the exit scan, the ordered fold, the selection, the state
 * update. NULL turns it off. */
int ee_tune_profile(ee_workspace* ws, int64_t* d_cycles);

/* Per-launch timing: while enabled, every kernel launched through `ws` is
 * bracketed by CUDA events on its stream. ee_profile_read synchronises, writes
 * {"kernel": {"launches": L, "ms": T}, ...} (JSON) into buf and resets. */
int ee_profile_enable(ee_workspace* ws, int32_t on);
int ee_profile_read(ee_workspace* ws, char* buf, int64_t cap);

/* Host-side columnar window ingest (no GPU): replays the reference workload
 * generator (pkg/src/eesim/trace.py:164-227) over a caller-provided raw PCG64
 * stream (numpy Generator.bit_generator.random_raw), writing errs f64 [n, s],
 * labels i32 [n, s] and finals i32 [n] for records [t_begin, *t_end). Stops
 * early (returning *t_end < n) when the raw buffer runs out; the io_* stream
 * state is updated so the caller can refill and resume. */
int ee_synth_columns(const uint64_t* raw, int64_t n_raw, int64_t* io_pos, int32_t* io_has32,
                     uint32_t* io_buf, const double* u, int64_t n, int64_t t_begin,
                     int64_t* t_end, double* io_d_prev, int32_t n_sites, const double* agree_early,
                     const double* agree_late, int32_t use_late, double continuity, double miscal,
                     double miscal_late, int32_t n_labels, double* errs, int32_t* labels,
                     int32_t* finals);

/* Device-scheduled compaction: one executable graph that runs a compacted
 * batch's segments back to back with no host round trip. Segment 0 runs
 * graphs[nb - 1] (bucket h_buckets[nb - 1] = the full batch); before segment
 * k >= 1 a one-thread kernel reads d_n_live[k - 1] (the live rows segment
 * k - 1 left, written on the device) and sets a SWITCH conditional node to the
 * smallest bucket >= it, whose body is graphs[k * nb + j] as a child graph
 * (no body when no row is live: the rest of the chain does nothing).
 * graphs: cudaGraph_t [nseg * nb] (NULL = never needed); reset: an optional
 * graph run first. The graphs may contain kernels, memsets and device-to-
 * device copies only (CUDA conditional-body rules); they are cloned. */
typedef struct ee_seg_chain ee_seg_chain;
int ee_seg_chain_create(void* const* graphs, int32_t nseg, int32_t nb, const int32_t* h_buckets,
                        const int32_t* d_n_live, void* reset, ee_seg_chain** out);
int ee_seg_chain_launch(ee_seg_chain* chain, void* stream);
void ee_seg_chain_destroy(ee_seg_chain* chain);

#ifdef __cplusplus
}
#endif

#endif /* EEB200_H */
