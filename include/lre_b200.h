/*
 * lre_b200.h — C ABI of the B200-native LRE (linear-regression-estimation)
 * hot path of arXiv 1602.08604: Pauli outcome counts -> theta -> mu.
 *
 * Every pointer marked (device) is device memory owned by the caller; every
 * call is asynchronous on the given cudaStream_t (pass 0 for the legacy
 * stream) and returns an lre_status.  The library allocates nothing and keeps
 * no hidden state except a launch counter and a per-device cache of the SM
 * count (read-only after the first call); epilogue factors travel with each
 * launch.  lre_generate_counts with exact != 0 synchronises `stream` (it
 * checks that the state is dyadic).  Host code (Python via ctypes, see
 * INTEGRATION.md) owns memory, streams and the NCCL communicator.
 *
 * Layout conventions (reference pauli.py:1-13): qubit 1 is the most
 * significant digit/bit everywhere; counts are row-major (3^n settings, 2^n
 * outcomes); theta is either NATURAL (index = base-4 Pauli digits I,X,Y,Z) or
 * MASK_MAJOR (index = m * 2^n + a, m = X|Y mask, a = Y|Z mask).
 */
#ifndef LRE_B200_H
#define LRE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *lre_stream_t; /* == cudaStream_t */

typedef enum {
    LRE_OK = 0,
    LRE_EINVAL = 1,       /* bad argument; maps to Python ValueError           */
    LRE_ECUDA = 2,        /* CUDA launch/runtime failure; RuntimeError         */
    LRE_ENOMEM = 3,       /* workspace too small; MemoryError                  */
    LRE_EUNSUPPORTED = 4, /* size/dtype not supported by this build            */
    LRE_EOVERFLOW = 5     /* shots too large for the requested count dtype     */
} lre_status;

typedef enum { LRE_U8 = 1, LRE_U16 = 2, LRE_I32 = 3, LRE_I64 = 4 } lre_dtype;

typedef enum { LRE_LAYOUT_NATURAL = 0, LRE_LAYOUT_MASK_MAJOR = 1 } lre_layout;

/*
 * MASK_MAJOR with the X-masks permuted for a chunked exchange over P = 2^logP
 * ranks in K = 2^logK chunks (step (i) outputs only): mask m = (g, c, j), g =
 * m / S (S = 2^n / P), c = (m % S) / (S / K), j = m % (S / K), is stored at
 * mask position (c * P + g) * (S / K) + j, so chunk c of every rank's slice is
 * one contiguous P x (S/K) x 2^n block: reduce-scatter chunk c.
 */
#define LRE_LAYOUT_MASK_CHUNKED(logP, logK) (2 | ((logP) << 8) | ((logK) << 16))

typedef enum {
    LRE_OUT_THETA_F64 = 0, /* finished theta (fp64), requires the full setting range */
    LRE_OUT_NUM_I64 = 1    /* exact int64 numerators N_i (partial sums allowed)     */
} lre_out_kind;

typedef enum {
    LRE_STATE_MAXMIXED = 0,
    LRE_STATE_GHZ = 1,
    LRE_STATE_PRODUCTZ = 2,
    LRE_STATE_W = 3
} lre_state_kind;

/* Human-readable status text. */
const char *lre_strerror(int status);

/* ABI version (major*100 + minor). */
int lre_version(void);

/* Number of kernels this library has launched since load (for benchmarking). */
int64_t lre_launch_count(void);

/*
 * Step (i) workspace size in bytes for settings [w_begin, w_end).
 * Replaces the per-worker private 4^n partials of
 * reference pipeline.py:74-90,128-137 (step_one_least_squares).
 */
int lre_step1_workspace(int n, int64_t shots, int64_t w_begin, int64_t w_end, size_t *bytes);

/*
 * Step (i): counts (device, rows = settings [w_begin, w_end), 2^n columns,
 * dtype `count_dtype`) -> `out` (device).
 *   out_kind == LRE_OUT_THETA_F64: out = double[4^n] theta (needs the full
 *     range [0, 3^n)); theta_i = N_i / shots * 2^{-n/2} / 3^{zc(i)}.
 *   out_kind == LRE_OUT_NUM_I64: out = int64[4^n] exact numerators of this
 *     setting range (summable across ranges/devices).
 * Replaces reference pipeline.py:116-138 (step_one_least_squares) together
 * with _kernels.py:34-56 (accumulate_fast) and pauli.py:153-209.
 * w_begin/w_end must be multiples of lre_shard_quantum(n) (except w_end = 3^n).
 * Contract (as in the reference's MeasurementRecord.validate, records.py:34-56):
 * every row sums to `shots` and no count is negative.  The integer passes size
 * their intermediates from that bound (int16 Y1 low halves when shots*27 <=
 * 32767, int32 while shots*3^q < 2^31); lre_validate_counts checks it on the
 * device.
 */
int lre_step1(const void *counts, int count_dtype, int n, int64_t shots, int64_t w_begin,
              int64_t w_end, void *workspace, size_t workspace_bytes, void *out, int out_kind,
              int layout, lre_stream_t stream);

/* Alignment quantum of setting shards for lre_step1: 3^min(n, 7) (a multiple of every first-pass tile). */
int64_t lre_shard_quantum(int n);

/* Number of fold passes step (i) runs at this size (1 for n <= 7). */
int lre_step1_num_passes(int n, int64_t shots);

/*
 * Streaming form of lre_step1 for records that arrive in setting chunks
 * (host records larger than HBM, pipelined H2D): lre_step1_stage runs the
 * first fold pass of chunk [w_begin, w_end) (rows of `counts`) into a
 * full-range workspace (size from lre_step1_workspace(n, shots, 0, 3^n));
 * after every chunk has been staged once, lre_step1_finish runs the remaining
 * passes.  When lre_step1_num_passes(n, shots) == 1 (n <= 2, 6, 7) the shard
 * quantum is the whole record, so the only chunk is [0, 3^n).
 */
int lre_step1_stage(const void *counts, int count_dtype, int n, int64_t shots, int64_t w_begin, int64_t w_end,
                    void *workspace, size_t workspace_bytes, lre_stream_t stream);
int lre_step1_finish(void *workspace, size_t workspace_bytes, int n, int64_t shots, void *out, int out_kind,
                     int layout, lre_stream_t stream);

/*
 * Step (i) from fp64 frequencies: the reference's source protocol
 * (pipeline.py:42-59,84 — any source with .frequencies(a, b), e.g.
 * ExactFrequencies; records.py:62-64 for counts/shots).  Streaming only:
 * lre_step1_f64_stage folds the chunk of settings [w_begin, w_end) (rows of
 * `freq`, device fp64, 2^n per row; w_begin a multiple of
 * lre_step1_f64_quantum(n), w_end too unless it is 3^n) into `workspace`
 * (its first passes run in `scratch`); after every chunk has been staged once,
 * lre_step1_f64_finish writes theta (fp64, `layout`).  Sizes:
 * lre_step1_f64_workspace(n, max chunk rows, &workspace, &scratch).
 * Replaces pipeline.py:116-138 for non-integer sources.
 */
int lre_step1_f64_workspace(int n, int64_t chunk_rows, size_t *workspace_bytes, size_t *scratch_bytes);
int64_t lre_step1_f64_quantum(int n);
int lre_step1_f64_stage(const double *freq, int n, int64_t w_begin, int64_t w_end, void *workspace,
                        size_t workspace_bytes, void *scratch, size_t scratch_bytes, lre_stream_t stream);
int lre_step1_f64_finish(void *workspace, size_t workspace_bytes, int n, double *theta, int layout,
                         lre_stream_t stream);

/*
 * Exact outcome probabilities (device fp64, rows x 2^n) of settings
 * [w_begin, w_end) for the state with Pauli coefficients theta (device,
 * NATURAL): 2^{-n/2} WHT of theta on each setting's support — the
 * reference's _theta_probability_block / theta_to_probabilities
 * (simulate.py:141-151); clip != 0 clamps to [0, 1] as probabilities_block
 * does for random states (:176-177, i.e. ExactFrequencies.frequencies).
 * n <= 12.
 */
int lre_theta_probabilities(const double *theta, int n, int64_t w_begin, int64_t w_end, int clip, double *out,
                            lre_stream_t stream);

/*
 * int64 numerators (device, entries [begin, end) of `layout`) -> fp64 theta
 * (device, same positions).  Epilogue of reference pipeline.py:138 and
 * records.py:62-64 (frequencies = counts / float(shots)).
 */
int lre_finalize(const int64_t *num, int n, int64_t shots, int layout, int64_t begin, int64_t end,
                 double *theta, lre_stream_t stream);

/* theta relayout NATURAL <-> MASK_MAJOR (device -> device, out of place). */
int lre_theta_relayout(const double *src, int src_layout, int n, double *dst, lre_stream_t stream);

/*
 * Step (ii): theta (device) -> mu (device, complex128 as interleaved
 * doubles) for the X/Y masks [m_begin, m_end).
 *   layout == LRE_LAYOUT_NATURAL:     theta is the full natural-order vector;
 *   layout == LRE_LAYOUT_MASK_MAJOR:  theta is the slice of those masks,
 *                                     theta[(m - m_begin)*2^n + a].
 * S = m_end - m_begin must be a power of two and m_begin a multiple of S; mu
 * is written as d rows x S columns:
 *   mu_out[r*S + c] = mu[r, ((r / S) ^ (m_begin / S)) * S + c]
 * (S = 2^n gives the full row-major matrix).  Replaces reference
 * pipeline.py:141-161 (step_two_assemble) and pauli.py:270-297.
 */
int lre_assemble(const double *theta, int layout, int n, int64_t m_begin, int64_t m_end, double *mu_out,
                 lre_stream_t stream);

/*
 * One chunk of a rank's step (ii): masks [m_begin, m_end) (theta: their
 * mask-major slice) written into the column slab of the masks [slab_begin,
 * slab_begin + slab_masks) laid out as lre_assemble's output for that range:
 *   mu_slab[r*slab_masks + c] = mu[r, ((r / slab_masks) ^ (slab_begin / slab_masks))*slab_masks + c].
 * m_end - m_begin a power of two dividing m_begin; chunks smaller than the slab
 * need n >= 11 and >= 8 masks (LRE_EUNSUPPORTED otherwise).
 */
int lre_assemble_slab(const double *theta, int n, int64_t m_begin, int64_t m_end, int64_t slab_begin,
                      int64_t slab_masks, double *mu_slab, lre_stream_t stream);

/*
 * Record validation (reference records.py:34-56, MeasurementRecord.validate):
 * result (device int64[3]) receives {first row whose sum != shots (or
 * INT64_MAX), that row's sum, minimum count value}.
 */
int lre_validate_counts(const void *counts, int count_dtype, int n, int64_t rows, int64_t shots,
                        int64_t *result, lre_stream_t stream);

/*
 * Device synthetic count generator (north-star item 4; reference
 * simulate.py:167-266).  Rows [w_begin, w_end) of the record of state
 * `kind` (bits = productz basis string) are written to out (device, row 0 =
 * setting w_begin).  exact != 0 writes the noiseless dyadic record
 * (shots must equal 2^n; LRE_EINVAL if the state is not dyadic).
 * Sampling draws `shots` outcomes per setting from a Philox4x32-10 stream
 * keyed on (seed, setting), so records do not depend on sharding.
 */
int lre_generate_counts(int kind, int n, int64_t bits, int64_t shots, uint64_t seed, int exact,
                        int64_t w_begin, int64_t w_end, void *out, int count_dtype,
                        lre_stream_t stream);

/*
 * Outcome-list records (record ingestion at scale): a
 * sampled record as the outcome of every shot, outcomes[(w - w_begin) * shots
 * + k] (uint16, n <= 16) — 2 bytes per shot instead of 2^n counts per setting
 * (n = 14, 1000 shots: 9.6 GB instead of 157 GB of uint16 counts).
 * lre_generate_outcomes draws them with the same Philox stream as
 * lre_generate_counts (so their histogram equals that record);
 * lre_counts_from_outcomes turns `rows` outcome lists (device) into dense
 * counts (device, count_dtype) for lre_step1 / lre_step1_stage.  Replaces
 * the counting inside reference simulate.py:224-242 (sample_counts).
 */
int lre_generate_outcomes(int kind, int n, int64_t bits, int64_t shots, uint64_t seed, int64_t w_begin,
                          int64_t w_end, uint16_t *out, lre_stream_t stream);
int lre_counts_from_outcomes(const uint16_t *outcomes, int n, int64_t shots, int64_t rows, void *counts,
                             int count_dtype, lre_stream_t stream);

/*
 * Arbitrary (dense / mixed) states (reference
 * simulate.py:114-151, :224-242).
 * lre_dense_to_theta: rho (device, row-major 2^n x 2^n complex128, Hermitian)
 *   -> theta (device, 4^n fp64, NATURAL order), the inverse of lre_assemble
 *   (replaces simulate.dense_to_theta).  n <= 12.
 * lre_generate_counts_theta: sampled counts of settings [w_begin, w_end) for
 *   the state with Pauli coefficients theta (device, NATURAL): per setting
 *   the outcome distribution is one WHT of theta on the setting's support
 *   (replaces _theta_probability_block), then `shots` inverse-CDF draws from
 *   a Philox4x32-10 stream keyed on (seed, setting, shot).  n <= 12.
 */
int lre_dense_to_theta(const double *rho, int n, double *theta, lre_stream_t stream);
int lre_generate_counts_theta(const double *theta, int n, int64_t shots, uint64_t seed, int64_t w_begin,
                              int64_t w_end, void *out, int count_dtype, lre_stream_t stream);

/*
 * Error metrics on the device (reference metrics.py).
 *
 * lre_reduce: deterministic fp64 reduction of `count` doubles (device) into
 * out[0]; out (device) must hold 1 + LRE_REDUCE_BLOCKS doubles (out[1..] is
 * scratch).  Bit-reproducible for a given count (fixed grid, fixed order).
 *   LRE_REDUCE_SUM_SQ     sum (a_i - b_i)^2, b may be NULL: squared Hilbert-
 *                         Schmidt distance over a complex matrix viewed as
 *                         2 d^2 doubles (replaces metrics.py:28-35)
 *   LRE_REDUCE_SUM_SQRT   sum sqrt(max(a_i, 0) * scale): with scale = 1/d over
 *                         a spectrum, sqrt of the fidelity with I/d
 *                         (replaces metrics.py:88-92)
 *   LRE_REDUCE_SUM_SQ_ZC  sum 3^zc(i) a_i^2 over a NATURAL theta (count = 4^n,
 *                         zc = identity digits of i) = sum over settings and
 *                         outcomes of p_ws^2 (the dense MSE predictor,
 *                         metrics.py:124-154, in closed form)
 * lre_truth_terms: for the generator's states, out[0] = Re Tr(A rho_true) and
 * out[1] = Tr(rho_true^2), A a row-major 2^n x 2^n complex128 Hermitian
 * matrix (device); squared HS distance to the truth is
 * ||A||^2 - 2 out[0] + out[1], and for a pure truth out[0] is the fidelity
 * <psi|A|psi> (metrics.py:57-85, evaluate_errors :173-201).
 */
#define LRE_REDUCE_BLOCKS 1184
enum { LRE_REDUCE_SUM_SQ = 0, LRE_REDUCE_SUM_SQRT = 1, LRE_REDUCE_SUM_SQ_ZC = 2 };
int lre_reduce(int op, const double *a, const double *b, int64_t count, double scale, double *out,
               lre_stream_t stream);
int lre_truth_terms(const double *a, int n, int kind, int64_t bits, double *out, lre_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* LRE_B200_H */
