/*
 * CPU oracle for the LRE hot path — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference package's step (i) and step (ii)
 * (/root/reference/pkg/src/pauli_lre).  Used by tests/ as a fast checker at
 * n = 8..12 and by bench.py as the CPU baseline ("kind": "port") and the
 * `--impl reference` arm.  Never linked into the product library.
 *
 * Parallel scheme follows pipeline.py:62-65,104-113,128-137: settings are
 * split into `threads` contiguous chunks (np.linspace bounds), each worker
 * accumulates a private 4**n fp64 partial, partials are merged in worker
 * order, then divided by the Gram diagonal (pipeline.py:138).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_U8 = 1, ORC_U16 = 2, ORC_I32 = 3, ORC_I64 = 4 };

static inline double load_count(const void *base, int dtype, int64_t idx) {
    switch (dtype) {
    case ORC_U8: return (double)((const uint8_t *)base)[idx];
    case ORC_U16: return (double)((const uint16_t *)base)[idx];
    case ORC_I32: return (double)((const int32_t *)base)[idx];
    default: return (double)((const int64_t *)base)[idx];
    }
}

static inline int64_t load_count_i(const void *base, int dtype, int64_t idx) {
    switch (dtype) {
    case ORC_U8: return ((const uint8_t *)base)[idx];
    case ORC_U16: return ((const uint16_t *)base)[idx];
    case ORC_I32: return ((const int32_t *)base)[idx];
    default: return ((const int64_t *)base)[idx];
    }
}

/* place-scaled digits of setting w: digit_k * 4**(n-1-k)  (pipeline.py:79-85) */
static void place_digits(int64_t w, int n, int64_t *out) {
    int64_t place = 1;
    for (int k = n - 1; k >= 0; --k) {
        out[k] = (w % 3 + 1) * place;
        w /= 3;
        place *= 4;
    }
}

/* locs[t] = sum of place digits over the qubits in subset t, by subset-sum
 * doubling (_kernels.py:21-31). */
static void fill_locations(const int64_t *pd, int n, int64_t *locs) {
    locs[0] = 0;
    int64_t size = 1;
    for (int j = 0; j < n; ++j) {
        int64_t w = pd[n - 1 - j];
        for (int64_t t = 0; t < size; ++t) locs[size + t] = locs[t] + w;
        size *= 2;
    }
}

static void wht_inplace(double *buf, int64_t d) {  /* _kernels.py:44-53 */
    for (int64_t h = 1; h < d; h *= 2)
        for (int64_t start = 0; start < d; start += 2 * h)
            for (int64_t j = start; j < start + h; ++j) {
                double top = buf[j], bot = buf[j + h];
                buf[j] = top + bot;
                buf[j + h] = top - bot;
            }
}

static void wht_inplace_i64(int64_t *buf, int64_t d) {
    for (int64_t h = 1; h < d; h *= 2)
        for (int64_t start = 0; start < d; start += 2 * h)
            for (int64_t j = start; j < start + h; ++j) {
                int64_t top = buf[j], bot = buf[j + h];
                buf[j] = top + bot;
                buf[j + h] = top - bot;
            }
}

/*
 * Step (i) raw accumulation (before Gram division) over settings
 * [w_begin, w_end) of a counts block whose first row is setting w_begin.
 * raw_out (4**n doubles) is overwritten.  Frequencies are count/(double)shots
 * (records.py:62-64); scale = 2**(-n/2) (pipeline.py:78).
 */
int lre_oracle_step1_raw(const void *counts, int dtype, int n, int64_t shots,
                         int64_t w_begin, int64_t w_end, int threads, double *raw_out) {
    const int64_t d = (int64_t)1 << n;
    const int64_t size = (int64_t)1 << (2 * n);
    const double scale = pow(2.0, -n / 2.0);
    const double fshots = (double)shots;
    const int64_t total = w_end - w_begin;
    if (threads < 1) threads = 1;
    if (threads > total) threads = (int)(total > 0 ? total : 1);
    double **partials = (double **)calloc((size_t)threads, sizeof(double *));
    if (!partials) return 1;
    int failed = 0;
#pragma omp parallel num_threads(threads)
    {
        int tid = omp_get_thread_num();
        /* np.linspace(0, total, workers+1).astype(int) (pipeline.py:62-65) */
        int64_t a = (int64_t)((double)total * tid / threads);
        int64_t b = (int64_t)((double)total * (tid + 1) / threads);
        double *raw = (double *)calloc((size_t)size, sizeof(double));
        double *buf = (double *)malloc((size_t)d * sizeof(double));
        int64_t *locs = (int64_t *)malloc((size_t)d * sizeof(int64_t));
        int64_t pd[64];
        if (!raw || !buf || !locs) {
#pragma omp atomic write
            failed = 1;
        } else {
            for (int64_t r = a; r < b; ++r) {
                const int64_t row = r * d;
                for (int64_t s = 0; s < d; ++s) buf[s] = load_count(counts, dtype, row + s) / fshots;
                wht_inplace(buf, d);
                place_digits(w_begin + r, n, pd);
                fill_locations(pd, n, locs);
                for (int64_t t = 0; t < d; ++t) raw[locs[t]] += buf[t] * scale;
            }
        }
        partials[tid] = raw;
        free(buf);
        free(locs);
    }
    if (failed) {
        for (int i = 0; i < threads; ++i) free(partials[i]);
        free(partials);
        return 1;
    }
    /* merge in worker order (pipeline.py:135-137) */
    memcpy(raw_out, partials[0], (size_t)size * sizeof(double));
    for (int i = 1; i < threads; ++i) {
        const double *p = partials[i];
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t j = 0; j < size; ++j) raw_out[j] += p[j];
    }
    for (int i = 0; i < threads; ++i) free(partials[i]);
    free(partials);
    return 0;
}

/*
 * Cost model of lre_oracle_step1_raw on `threads` workers for the CPU
 * baseline (bench.py), measured on a sample of settings [w_begin, w_end):
 *   fixed_s      one-time costs of a full run: zero-filling the `threads`
 *                private 4**n partials (calloc pages are faulted in on first
 *                touch; the reference's np.zeros behaves the same) and the
 *                ordered merge (pipeline.py:135-137);
 *   per_row_s    steady-state seconds per setting per worker, measured on the
 *                sample with the partials already touched (in a full run the
 *                page faults are paid once, not per sampled setting).
 * A full run is then fixed_s + per_row_s * settings / threads.
 */
int lre_oracle_step1_cost(const void *counts, int dtype, int n, int64_t shots, int64_t w_begin, int64_t w_end,
                          int threads, double *fixed_s, double *per_row_s) {
    const int64_t d = (int64_t)1 << n;
    const int64_t size = (int64_t)1 << (2 * n);
    const double scale = pow(2.0, -n / 2.0);
    const double fshots = (double)shots;
    const int64_t total = w_end - w_begin;
    if (threads < 1) threads = 1;
    if (threads > total) threads = (int)(total > 0 ? total : 1);
    double **partials = (double **)calloc((size_t)threads, sizeof(double *));
    if (!partials) return 1;
    int failed = 0;
    double t_touch = 0.0, t_rows = 0.0;
#pragma omp parallel num_threads(threads)
    {
        int tid = omp_get_thread_num();
        int64_t a = (int64_t)((double)total * tid / threads);
        int64_t b = (int64_t)((double)total * (tid + 1) / threads);
        double t0 = omp_get_wtime();
        double *raw = (double *)calloc((size_t)size, sizeof(double));
        if (raw) memset(raw, 0, (size_t)size * sizeof(double));  /* fault every page in */
#pragma omp barrier
        double t1 = omp_get_wtime();
        double *buf = (double *)malloc((size_t)d * sizeof(double));
        int64_t *locs = (int64_t *)malloc((size_t)d * sizeof(int64_t));
        int64_t pd[64];
        if (!raw || !buf || !locs) {
#pragma omp atomic write
            failed = 1;
        } else {
            for (int64_t r = a; r < b; ++r) {
                const int64_t row = r * d;
                for (int64_t s = 0; s < d; ++s) buf[s] = load_count(counts, dtype, row + s) / fshots;
                wht_inplace(buf, d);
                place_digits(w_begin + r, n, pd);
                fill_locations(pd, n, locs);
                for (int64_t t = 0; t < d; ++t) raw[locs[t]] += buf[t] * scale;
            }
        }
#pragma omp barrier
        double t2 = omp_get_wtime();
        if (tid == 0) {
            t_touch = t1 - t0;
            t_rows = t2 - t1;
        }
        partials[tid] = raw;
        free(buf);
        free(locs);
    }
    if (failed) {
        for (int i = 0; i < threads; ++i) free(partials[i]);
        free(partials);
        return 1;
    }
    double tm0 = omp_get_wtime();
    for (int i = 1; i < threads; ++i) {
        double *dst = partials[0];
        const double *p = partials[i];
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t j = 0; j < size; ++j) dst[j] += p[j];
    }
    double t_merge = omp_get_wtime() - tm0;
    for (int i = 0; i < threads; ++i) free(partials[i]);
    free(partials);
    *fixed_s = t_touch + t_merge;
    *per_row_s = t_rows / ((double)total / threads);
    return 0;
}

/* Gram diagonal division: theta = raw / 3**zero_count(i) (pipeline.py:138). */
void lre_oracle_gram_divide(double *theta, int n) {
    const int64_t size = (int64_t)1 << (2 * n);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < size; ++i) {
        int zc = 0;
        for (int k = 0; k < n; ++k) zc += ((i >> (2 * k)) & 3) == 0;
        double g = 1.0;
        for (int k = 0; k < zc; ++k) g *= 3.0;
        theta[i] /= g;
    }
}

/* Exact int64 numerators N_i over settings [w_begin, w_end) (integer form of
 * _kernels.accumulate_fast; the B200 bit-exact contract). num_out overwritten. */
int lre_oracle_numerators(const void *counts, int dtype, int n, int64_t w_begin, int64_t w_end,
                          int threads, int64_t *num_out) {
    const int64_t d = (int64_t)1 << n;
    const int64_t size = (int64_t)1 << (2 * n);
    const int64_t total = w_end - w_begin;
    if (threads < 1) threads = 1;
    if (threads > total) threads = (int)(total > 0 ? total : 1);
    int64_t **partials = (int64_t **)calloc((size_t)threads, sizeof(int64_t *));
    if (!partials) return 1;
    int failed = 0;
#pragma omp parallel num_threads(threads)
    {
        int tid = omp_get_thread_num();
        int64_t a = (int64_t)((double)total * tid / threads);
        int64_t b = (int64_t)((double)total * (tid + 1) / threads);
        int64_t *num = (int64_t *)calloc((size_t)size, sizeof(int64_t));
        int64_t *buf = (int64_t *)malloc((size_t)d * sizeof(int64_t));
        int64_t *locs = (int64_t *)malloc((size_t)d * sizeof(int64_t));
        int64_t pd[64];
        if (!num || !buf || !locs) {
#pragma omp atomic write
            failed = 1;
        } else {
            for (int64_t r = a; r < b; ++r) {
                for (int64_t s = 0; s < d; ++s) buf[s] = load_count_i(counts, dtype, r * d + s);
                wht_inplace_i64(buf, d);
                place_digits(w_begin + r, n, pd);
                fill_locations(pd, n, locs);
                for (int64_t t = 0; t < d; ++t) num[locs[t]] += buf[t];
            }
        }
        partials[tid] = num;
        free(buf);
        free(locs);
    }
    if (failed) {
        for (int i = 0; i < threads; ++i) free(partials[i]);
        free(partials);
        return 1;
    }
    memcpy(num_out, partials[0], (size_t)size * sizeof(int64_t));
    for (int i = 1; i < threads; ++i) {
        const int64_t *p = partials[i];
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t j = 0; j < size; ++j) num_out[j] += p[j];
    }
    for (int i = 0; i < threads; ++i) free(partials[i]);
    free(partials);
    return 0;
}

/*
 * Step (ii) for masks [m_begin, m_end) (pipeline.py:93-101,141-161):
 * v[a] = theta[gather(m)[a]] * (-i)^popcount(a&m)  (pauli.py:270-297),
 * complex WHT, * 2**(-n/2); written as out[(m - m_begin) * d + r] = mu[r, r^m].
 * Complex numbers are interleaved (re, im) doubles.
 */
int lre_oracle_step2_masks(const double *theta, int n, int64_t m_begin, int64_t m_end, int threads,
                           double *out) {
    const int64_t d = (int64_t)1 << n;
    const double scale = pow(2.0, -n / 2.0);
    if (threads < 1) threads = 1;
    int failed = 0;
#pragma omp parallel num_threads(threads)
    {
        double *re = (double *)malloc((size_t)d * sizeof(double));
        double *im = (double *)malloc((size_t)d * sizeof(double));
        if (!re || !im) {
#pragma omp atomic write
            failed = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t m = m_begin; m < m_end; ++m) {
                for (int64_t a = 0; a < d; ++a) {
                    /* basis digit per qubit: mask bit clear -> 3*a_k, set -> 1+a_k */
                    int64_t idx = 0;
                    for (int k = 0; k < n; ++k) {
                        int sh = n - 1 - k;
                        int mb = (int)((m >> sh) & 1), ab = (int)((a >> sh) & 1);
                        idx = idx * 4 + (mb ? 1 + ab : 3 * ab);
                    }
                    double v = theta[idx];
                    switch (__builtin_popcountll((unsigned long long)(a & m)) & 3) {
                    case 0: re[a] = v; im[a] = 0.0; break;
                    case 1: re[a] = 0.0; im[a] = -v; break;
                    case 2: re[a] = -v; im[a] = 0.0; break;
                    default: re[a] = 0.0; im[a] = v; break;
                    }
                }
                wht_inplace(re, d);
                wht_inplace(im, d);
                double *o = out + 2 * (m - m_begin) * d;
                for (int64_t r = 0; r < d; ++r) {
                    o[2 * r] = re[r] * scale;
                    o[2 * r + 1] = im[r] * scale;
                }
            }
        }
        free(re);
        free(im);
    }
    return failed;
}

int lre_oracle_max_threads(void) { return omp_get_max_threads(); }

/*
 * Streaming form of lre_oracle_step1_raw for bench.py's reference arm: the
 * workers' private 4**n partials persist across setting shards, so timing the
 * shards of [0, 3**n) one after another and then the ordered merge + Gram
 * division (pipeline.py:133-138) is one full step (i), measured in pieces.
 * Each shard is split over the workers with np.linspace bounds (pipeline.py:62-65).
 */
typedef struct {
    int n, threads;
    int64_t shots;
    double **partials;
} lre_oracle_acc;

void *lre_oracle_acc_new(int n, int64_t shots, int threads) {
    lre_oracle_acc *acc = (lre_oracle_acc *)calloc(1, sizeof(lre_oracle_acc));
    if (!acc) return NULL;
    acc->n = n;
    acc->shots = shots;
    acc->threads = threads < 1 ? 1 : threads;
    acc->partials = (double **)calloc((size_t)acc->threads, sizeof(double *));
    if (!acc->partials) {
        free(acc);
        return NULL;
    }
    return acc;
}

void lre_oracle_acc_free(void *h) {
    lre_oracle_acc *acc = (lre_oracle_acc *)h;
    if (!acc) return;
    for (int i = 0; i < acc->threads; ++i) free(acc->partials[i]);
    free(acc->partials);
    free(acc);
}

/* settings [w_begin, w_end) of a counts block whose first row is w_begin (_step_one_chunk, pipeline.py:74-90) */
int lre_oracle_acc_add(void *h, const void *counts, int dtype, int64_t w_begin, int64_t w_end) {
    lre_oracle_acc *acc = (lre_oracle_acc *)h;
    const int n = acc->n, threads = acc->threads;
    const int64_t d = (int64_t)1 << n;
    const int64_t size = (int64_t)1 << (2 * n);
    const double scale = pow(2.0, -n / 2.0);
    const double fshots = (double)acc->shots;
    const int64_t total = w_end - w_begin;
    int failed = 0;
#pragma omp parallel num_threads(threads)
    {
        int tid = omp_get_thread_num();
        int64_t a = (int64_t)((double)total * tid / threads);
        int64_t b = (int64_t)((double)total * (tid + 1) / threads);
        if (!acc->partials[tid]) acc->partials[tid] = (double *)calloc((size_t)size, sizeof(double));
        double *raw = acc->partials[tid];
        double *buf = (double *)malloc((size_t)d * sizeof(double));
        int64_t *locs = (int64_t *)malloc((size_t)d * sizeof(int64_t));
        int64_t pd[64];
        if (!raw || !buf || !locs) {
#pragma omp atomic write
            failed = 1;
        } else {
            for (int64_t r = a; r < b; ++r) {
                const int64_t row = r * d;
                for (int64_t s = 0; s < d; ++s) buf[s] = load_count(counts, dtype, row + s) / fshots;
                wht_inplace(buf, d);
                place_digits(w_begin + r, n, pd);
                fill_locations(pd, n, locs);
                for (int64_t t = 0; t < d; ++t) raw[locs[t]] += buf[t] * scale;
            }
        }
        free(buf);
        free(locs);
    }
    return failed;
}

/* ordered merge of the partials (pipeline.py:135-137) and the Gram division (:138) */
int lre_oracle_acc_finish(void *h, double *theta_out) {
    lre_oracle_acc *acc = (lre_oracle_acc *)h;
    const int threads = acc->threads;
    const int64_t size = (int64_t)1 << (2 * acc->n);
    if (acc->partials[0]) memcpy(theta_out, acc->partials[0], (size_t)size * sizeof(double));
    else memset(theta_out, 0, (size_t)size * sizeof(double));
    for (int i = 1; i < threads; ++i) {
        const double *p = acc->partials[i];
        if (!p) continue;
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t j = 0; j < size; ++j) theta_out[j] += p[j];
    }
    lre_oracle_gram_divide(theta_out, acc->n);
    return 0;
}

/* step (ii) for masks [m_begin, m_end) scattered into the dense row-major mu
 * (d x d interleaved complex): mu[r, r ^ m] (pipeline.py:154-160) */
int lre_oracle_step2_scatter(const double *theta, int n, int64_t m_begin, int64_t m_end, int threads, double *mu) {
    const int64_t d = (int64_t)1 << n;
    const double scale = pow(2.0, -n / 2.0);
    if (threads < 1) threads = 1;
    int failed = 0;
#pragma omp parallel num_threads(threads)
    {
        double *re = (double *)malloc((size_t)d * sizeof(double));
        double *im = (double *)malloc((size_t)d * sizeof(double));
        if (!re || !im) {
#pragma omp atomic write
            failed = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t m = m_begin; m < m_end; ++m) {
                for (int64_t a = 0; a < d; ++a) {
                    int64_t idx = 0;
                    for (int k = 0; k < n; ++k) {
                        int sh = n - 1 - k;
                        int mb = (int)((m >> sh) & 1), ab = (int)((a >> sh) & 1);
                        idx = idx * 4 + (mb ? 1 + ab : 3 * ab);
                    }
                    double v = theta[idx];
                    switch (__builtin_popcountll((unsigned long long)(a & m)) & 3) {
                    case 0: re[a] = v; im[a] = 0.0; break;
                    case 1: re[a] = 0.0; im[a] = -v; break;
                    case 2: re[a] = -v; im[a] = 0.0; break;
                    default: re[a] = 0.0; im[a] = v; break;
                    }
                }
                wht_inplace(re, d);
                wht_inplace(im, d);
                for (int64_t r = 0; r < d; ++r) {
                    double *o = mu + 2 * (r * d + (r ^ m));
                    o[0] = re[r] * scale;
                    o[1] = im[r] * scale;
                }
            }
        }
        free(re);
        free(im);
    }
    return failed;
}
