// C ABI of liblre_b200 (include/lre_b200.h).  Argument checking and status
// mapping only; the work is in lre_step1.cu / lre_step2.cu / lre_aux.cu /
// lre_gen.cu.
#include <atomic>
#include <cstdio>
#include <vector>

#include "lre_internal.cuh"

namespace lre {
static std::atomic<int64_t> g_launches{0};
void count_launch(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

int num_sms() {
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    int v = cache[dev].load(std::memory_order_relaxed);
    if (!v) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cache[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

int step1_impl(const void *counts, int dtype, int n, int64_t shots, int64_t w_begin, int64_t w_end, void *ws,
               size_t ws_bytes, void *out, int out_kind, int layout, cudaStream_t stream);
size_t step1_workspace(int n, int64_t shots, int64_t w_begin, int64_t w_end);
int step1_stage_impl(const void *counts, int dtype, int n, int64_t shots, int64_t w_begin, int64_t w_end, void *ws,
                     size_t ws_bytes, cudaStream_t stream);
int step1_finish_impl(void *ws, size_t ws_bytes, int n, int64_t shots, void *out, int out_kind, int layout,
                      cudaStream_t stream);
int step1_num_passes(int n, int64_t shots);
size_t step1_f64_workspace(int n);
size_t step1_f64_scratch(int n, int64_t rows);
int64_t step1_f64_quantum(int n);
int step1_f64_stage_impl(const double *freq, int n, int64_t w_begin, int64_t w_end, void *ws, size_t ws_bytes,
                         void *scratch, size_t scratch_bytes, cudaStream_t stream);
int step1_f64_finish_impl(void *ws, size_t ws_bytes, int n, double *theta, int layout, cudaStream_t stream);
int theta_probabilities_impl(const double *theta, int n, int64_t w_begin, int64_t w_end, int clip, double *out,
                             cudaStream_t s);
int64_t shard_quantum(int n, int64_t shots);
int assemble_impl(const double *theta, int layout, int n, int64_t m_begin, int64_t m_end, double *mu, cudaStream_t s);
int assemble_slab_impl(const double *theta, int n, int64_t m_begin, int64_t m_end, int64_t slab_begin,
                       int64_t slab_masks, double *mu, cudaStream_t s);
int validate_impl(const void *counts, int dtype, int n, int64_t rows, int64_t shots, int64_t *result,
                  cudaStream_t s);
int finalize_impl(const int64_t *num, int n, int64_t shots, int layout, int64_t begin, int64_t end, double *theta,
                  cudaStream_t s);
int relayout_impl(const double *src, int src_layout, int n, double *dst, cudaStream_t s);
int generate_impl(int kind, int n, int64_t bits, int64_t shots, uint64_t seed, int exact, int64_t w_begin,
                  int64_t w_end, void *out, int dtype, cudaStream_t s);
int generate_outcomes_impl(int kind, int n, int64_t bits, int64_t shots, uint64_t seed, int64_t w_begin,
                           int64_t w_end, uint16_t *out, cudaStream_t s);
int counts_from_outcomes_impl(const uint16_t *outcomes, int n, int64_t shots, int64_t rows, void *counts, int dtype,
                              cudaStream_t s);
int dense_to_theta_impl(const double *rho, int n, double *theta, cudaStream_t s);
int generate_theta_impl(const double *theta, int n, int64_t shots, uint64_t seed, int64_t w_begin, int64_t w_end,
                        void *out, int dtype, cudaStream_t s);
int reduce_impl(int op, const double *a, const double *b, int64_t count, double scale, double *out, cudaStream_t s);
int truth_terms_impl(const double *a, int n, int kind, int64_t bits, double *out, cudaStream_t s);
}  // namespace lre

static inline int64_t pow3_i(int n) {
    int64_t r = 1;
    for (int i = 0; i < n; ++i) r *= 3;
    return r;
}

static inline int64_t dtype_max(int dtype) {
    switch (dtype) {
    case LRE_U8: return 255;
    case LRE_U16: return 65535;
    case LRE_I32: return 2147483647LL;
    case LRE_I64: return INT64_MAX;
    default: return -1;
    }
}

static inline bool valid_n(int n) { return n >= 1 && n <= 16; }

// NATURAL, MASK_MAJOR, or MASK_CHUNKED(logP, logK) with 2^(logP+logK) <= 2^n masks
static inline bool valid_layout(int layout, int n) {
    if (layout == LRE_LAYOUT_NATURAL || layout == LRE_LAYOUT_MASK_MAJOR) return true;
    if ((layout & 0xff) != 2 || (layout >> 24)) return false;
    const int logP = (layout >> 8) & 0xff, logK = (layout >> 16) & 0xff;
    return logP + logK <= n;
}

extern "C" {

const char *lre_strerror(int status) {
    switch (status) {
    case LRE_OK: return "ok";
    case LRE_EINVAL: return "invalid argument";
    case LRE_ECUDA: return "CUDA error";
    case LRE_ENOMEM: return "workspace too small";
    case LRE_EUNSUPPORTED: return "unsupported size or dtype";
    case LRE_EOVERFLOW: return "shots too large for the count dtype";
    default: return "unknown status";
    }
}

int lre_version(void) { return 200; }

int64_t lre_launch_count(void) { return lre::g_launches.load(); }

int64_t lre_shard_quantum(int n) { return valid_n(n) ? lre::shard_quantum(n, 1) : -1; }

int lre_step1_workspace(int n, int64_t shots, int64_t w_begin, int64_t w_end, size_t *bytes) {
    if (!valid_n(n) || !bytes || shots < 1) return LRE_EINVAL;
    if (w_begin < 0 || w_end > pow3_i(n) || w_begin >= w_end) return LRE_EINVAL;
    *bytes = lre::step1_workspace(n, shots, w_begin, w_end);
    return LRE_OK;
}

int lre_step1(const void *counts, int count_dtype, int n, int64_t shots, int64_t w_begin, int64_t w_end,
              void *workspace, size_t workspace_bytes, void *out, int out_kind, int layout, lre_stream_t stream) {
    if (!valid_n(n) || !counts || !out || shots < 1) return LRE_EINVAL;
    if (dtype_max(count_dtype) < 0) return LRE_EINVAL;
    if (shots > dtype_max(count_dtype) && count_dtype != LRE_I64) return LRE_EOVERFLOW;
    if (w_begin < 0 || w_end > pow3_i(n) || w_begin >= w_end) return LRE_EINVAL;
    if (out_kind != LRE_OUT_THETA_F64 && out_kind != LRE_OUT_NUM_I64) return LRE_EINVAL;
    if (!valid_layout(layout, n)) return LRE_EINVAL;
    if (out_kind == LRE_OUT_THETA_F64 && (w_begin != 0 || w_end != pow3_i(n))) return LRE_EINVAL;
    const int64_t q = lre::shard_quantum(n, shots);
    if (w_begin % q || (w_end % q && w_end != pow3_i(n))) return LRE_EINVAL;
    return lre::step1_impl(counts, count_dtype, n, shots, w_begin, w_end, workspace, workspace_bytes, out, out_kind,
                           layout, reinterpret_cast<cudaStream_t>(stream));
}

int lre_step1_num_passes(int n, int64_t shots) {
    if (!valid_n(n) || shots < 1) return -1;
    return lre::step1_num_passes(n, shots);
}

int lre_step1_stage(const void *counts, int count_dtype, int n, int64_t shots, int64_t w_begin, int64_t w_end,
                    void *workspace, size_t workspace_bytes, lre_stream_t stream) {
    if (!valid_n(n) || !counts || shots < 1) return LRE_EINVAL;
    if (dtype_max(count_dtype) < 0) return LRE_EINVAL;
    if (shots > dtype_max(count_dtype) && count_dtype != LRE_I64) return LRE_EOVERFLOW;
    if (w_begin < 0 || w_end > pow3_i(n) || w_begin >= w_end) return LRE_EINVAL;
    const int64_t q = lre::shard_quantum(n, shots);
    if (w_begin % q || (w_end % q && w_end != pow3_i(n))) return LRE_EINVAL;
    return lre::step1_stage_impl(counts, count_dtype, n, shots, w_begin, w_end, workspace, workspace_bytes,
                                 reinterpret_cast<cudaStream_t>(stream));
}

int lre_step1_finish(void *workspace, size_t workspace_bytes, int n, int64_t shots, void *out, int out_kind,
                     int layout, lre_stream_t stream) {
    if (!valid_n(n) || !out || shots < 1) return LRE_EINVAL;
    if (out_kind != LRE_OUT_THETA_F64 && out_kind != LRE_OUT_NUM_I64) return LRE_EINVAL;
    if (!valid_layout(layout, n)) return LRE_EINVAL;
    return lre::step1_finish_impl(workspace, workspace_bytes, n, shots, out, out_kind, layout,
                                  reinterpret_cast<cudaStream_t>(stream));
}

int lre_step1_f64_workspace(int n, int64_t chunk_rows, size_t *ws_bytes, size_t *scratch_bytes) {
    if (!valid_n(n) || !ws_bytes || !scratch_bytes || chunk_rows < 1) return LRE_EINVAL;
    *ws_bytes = lre::step1_f64_workspace(n);
    *scratch_bytes = lre::step1_f64_scratch(n, chunk_rows);
    return LRE_OK;
}

int64_t lre_step1_f64_quantum(int n) { return valid_n(n) ? lre::step1_f64_quantum(n) : -1; }

int lre_step1_f64_stage(const double *freq, int n, int64_t w_begin, int64_t w_end, void *workspace,
                        size_t workspace_bytes, void *scratch, size_t scratch_bytes, lre_stream_t stream) {
    if (!valid_n(n) || !freq) return LRE_EINVAL;
    if (w_begin < 0 || w_end > pow3_i(n) || w_begin >= w_end) return LRE_EINVAL;
    return lre::step1_f64_stage_impl(freq, n, w_begin, w_end, workspace, workspace_bytes, scratch, scratch_bytes,
                                     reinterpret_cast<cudaStream_t>(stream));
}

int lre_step1_f64_finish(void *workspace, size_t workspace_bytes, int n, double *theta, int layout,
                         lre_stream_t stream) {
    if (!valid_n(n) || !theta) return LRE_EINVAL;
    if (layout != LRE_LAYOUT_NATURAL && layout != LRE_LAYOUT_MASK_MAJOR) return LRE_EINVAL;
    return lre::step1_f64_finish_impl(workspace, workspace_bytes, n, theta, layout,
                                      reinterpret_cast<cudaStream_t>(stream));
}

int lre_theta_probabilities(const double *theta, int n, int64_t w_begin, int64_t w_end, int clip, double *out,
                            lre_stream_t stream) {
    if (!valid_n(n) || !theta || !out || w_begin < 0 || w_end < w_begin || w_end > pow3_i(n)) return LRE_EINVAL;
    return lre::theta_probabilities_impl(theta, n, w_begin, w_end, clip, out, reinterpret_cast<cudaStream_t>(stream));
}

int lre_finalize(const int64_t *num, int n, int64_t shots, int layout, int64_t begin, int64_t end, double *theta,
                 lre_stream_t stream) {
    if (!valid_n(n) || shots < 1 || !num || !theta) return LRE_EINVAL;
    if (begin < 0 || end > ((int64_t)1 << (2 * n))) return LRE_EINVAL;
    return lre::finalize_impl(num, n, shots, layout, begin, end, theta, reinterpret_cast<cudaStream_t>(stream));
}

int lre_theta_relayout(const double *src, int src_layout, int n, double *dst, lre_stream_t stream) {
    if (!valid_n(n) || !src || !dst || src == dst) return LRE_EINVAL;
    if (src_layout != LRE_LAYOUT_NATURAL && src_layout != LRE_LAYOUT_MASK_MAJOR) return LRE_EINVAL;
    return lre::relayout_impl(src, src_layout, n, dst, reinterpret_cast<cudaStream_t>(stream));
}

int lre_assemble(const double *theta, int layout, int n, int64_t m_begin, int64_t m_end, double *mu_out,
                 lre_stream_t stream) {
    if (!valid_n(n) || !theta || !mu_out) return LRE_EINVAL;
    if (layout != LRE_LAYOUT_NATURAL && layout != LRE_LAYOUT_MASK_MAJOR) return LRE_EINVAL;
    return lre::assemble_impl(theta, layout, n, m_begin, m_end, mu_out, reinterpret_cast<cudaStream_t>(stream));
}

int lre_assemble_slab(const double *theta, int n, int64_t m_begin, int64_t m_end, int64_t slab_begin,
                      int64_t slab_masks, double *mu_slab, lre_stream_t stream) {
    if (!valid_n(n) || !theta || !mu_slab) return LRE_EINVAL;
    return lre::assemble_slab_impl(theta, n, m_begin, m_end, slab_begin, slab_masks, mu_slab,
                                   reinterpret_cast<cudaStream_t>(stream));
}

int lre_validate_counts(const void *counts, int count_dtype, int n, int64_t rows, int64_t shots, int64_t *result,
                        lre_stream_t stream) {
    if (!valid_n(n) || !counts || !result || rows < 1) return LRE_EINVAL;
    return lre::validate_impl(counts, count_dtype, n, rows, shots, result, reinterpret_cast<cudaStream_t>(stream));
}

int lre_generate_counts(int kind, int n, int64_t bits, int64_t shots, uint64_t seed, int exact, int64_t w_begin,
                        int64_t w_end, void *out, int count_dtype, lre_stream_t stream) {
    if (!valid_n(n) || !out) return LRE_EINVAL;
    if (dtype_max(count_dtype) < 0) return LRE_EINVAL;
    if (shots > dtype_max(count_dtype)) return LRE_EOVERFLOW;
    if (w_begin < 0 || w_end > pow3_i(n) || w_begin > w_end) return LRE_EINVAL;
    if (kind == LRE_STATE_PRODUCTZ && (bits < 0 || bits >= ((int64_t)1 << n))) return LRE_EINVAL;
    return lre::generate_impl(kind, n, bits, shots, seed, exact, w_begin, w_end, out, count_dtype,
                              reinterpret_cast<cudaStream_t>(stream));
}

int lre_generate_outcomes(int kind, int n, int64_t bits, int64_t shots, uint64_t seed, int64_t w_begin,
                          int64_t w_end, uint16_t *out, lre_stream_t stream) {
    if (!valid_n(n) || !out || shots < 1) return LRE_EINVAL;
    if (w_begin < 0 || w_end > pow3_i(n) || w_begin > w_end) return LRE_EINVAL;
    if (kind == LRE_STATE_PRODUCTZ && (bits < 0 || bits >= ((int64_t)1 << n))) return LRE_EINVAL;
    return lre::generate_outcomes_impl(kind, n, bits, shots, seed, w_begin, w_end, out,
                                       reinterpret_cast<cudaStream_t>(stream));
}

int lre_counts_from_outcomes(const uint16_t *outcomes, int n, int64_t shots, int64_t rows, void *counts,
                             int count_dtype, lre_stream_t stream) {
    if (!valid_n(n) || !outcomes || !counts || shots < 1 || rows < 0) return LRE_EINVAL;
    if (dtype_max(count_dtype) < 0) return LRE_EINVAL;
    if (shots > dtype_max(count_dtype)) return LRE_EOVERFLOW;
    return lre::counts_from_outcomes_impl(outcomes, n, shots, rows, counts, count_dtype,
                                          reinterpret_cast<cudaStream_t>(stream));
}

int lre_dense_to_theta(const double *rho, int n, double *theta, lre_stream_t stream) {
    if (!valid_n(n) || !rho || !theta) return LRE_EINVAL;
    return lre::dense_to_theta_impl(rho, n, theta, reinterpret_cast<cudaStream_t>(stream));
}

int lre_generate_counts_theta(const double *theta, int n, int64_t shots, uint64_t seed, int64_t w_begin,
                              int64_t w_end, void *out, int count_dtype, lre_stream_t stream) {
    if (!valid_n(n) || !theta || !out || shots < 1 || w_begin < 0 || w_end < w_begin || w_end > pow3_i(n))
        return LRE_EINVAL;
    if (dtype_max(count_dtype) < 0) return LRE_EINVAL;
    if (shots > dtype_max(count_dtype)) return LRE_EOVERFLOW;
    return lre::generate_theta_impl(theta, n, shots, seed, w_begin, w_end, out, count_dtype,
                                    reinterpret_cast<cudaStream_t>(stream));
}

int lre_reduce(int op, const double *a, const double *b, int64_t count, double scale, double *out,
               lre_stream_t stream) {
    if (!a || !out || count < 0) return LRE_EINVAL;
    if (op < LRE_REDUCE_SUM_SQ || op > LRE_REDUCE_SUM_SQ_ZC) return LRE_EINVAL;
    return lre::reduce_impl(op, a, b, count, scale, out, reinterpret_cast<cudaStream_t>(stream));
}

int lre_truth_terms(const double *a, int n, int kind, int64_t bits, double *out, lre_stream_t stream) {
    if (!valid_n(n) || !a || !out) return LRE_EINVAL;
    if (kind < LRE_STATE_MAXMIXED || kind > LRE_STATE_W) return LRE_EINVAL;
    if (kind == LRE_STATE_PRODUCTZ && (bits < 0 || bits >= ((int64_t)1 << n))) return LRE_EINVAL;
    return lre::truth_terms_impl(a, n, kind, bits, out, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
