// Device synthetic count generator (north-star item 4).
//
// Reference: simulate.py:167-266 (probabilities_block, _setting_rng,
// sample_counts, exact_record).  The reference forms each setting's 2^n
// outcome distribution and draws one numpy Philox multinomial per setting.
// Here every supported state is a bond-dimension-2 state
//     GHZ: u|0..0> + v|1..1>,  W: u|0..0> + v sum_k |1_k>,  product states,
// so each shot is drawn qubit by qubit from exact conditional probabilities
// (projected-state norms) in O(n), with a Philox4x32-10 stream keyed on
// (seed, setting): a record never depends on how settings are sharded.
// Counts ~ Multinomial(shots, p) exactly; bitwise equality with numpy's
// generator is not a goal, parity is always checked
// on identical counts.
#include <algorithm>
#include <cmath>

#include "lre_internal.cuh"

namespace lre {

struct Cplx {
    double re, im;
};
__device__ __forceinline__ Cplx cmul(Cplx a, Cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
__device__ __forceinline__ Cplx cadd(Cplx a, Cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ double cabs2(Cplx a) { return a.re * a.re + a.im * a.im; }

// <e_{axis,s}|0> and <e_{axis,s}|1> for axis 0=X,1=Y,2=Z (conftest.py:19-24)
__device__ __forceinline__ void basis_coeffs(int axis, int s, Cplx &c0, Cplx &c1) {
    const double h = 0.70710678118654752440;
    if (axis == 0) {
        c0 = {h, 0.0};
        c1 = {s ? -h : h, 0.0};
    } else if (axis == 1) {
        c0 = {h, 0.0};
        c1 = {0.0, s ? h : -h};  // conj(+-i)/sqrt2
    } else {
        c0 = {s ? 0.0 : 1.0, 0.0};
        c1 = {s ? 1.0 : 0.0, 0.0};
    }
}

struct Chain {
    Cplx u, v;
};

__device__ __forceinline__ Chain chain_init(int kind, int n) {
    const double h = 0.70710678118654752440;
    if (kind == LRE_STATE_GHZ) return {{h, 0.0}, {h, 0.0}};
    if (kind == LRE_STATE_W) return {{0.0, 0.0}, {1.0 / sqrt((double)n), 0.0}};
    return {{1.0, 0.0}, {0.0, 0.0}};
}

// one qubit step; returns the weight (norm^2 of the projected remaining state)
__device__ __forceinline__ double chain_step(int kind, int64_t bits, int n, int j, int axis, int s, Chain &ch) {
    Cplx c0, c1;
    basis_coeffs(axis, s, c0, c1);
    const int r = n - j - 1;
    if (kind == LRE_STATE_GHZ) {
        ch.u = cmul(ch.u, c0);
        ch.v = cmul(ch.v, c1);
        return r >= 1 ? cabs2(ch.u) + cabs2(ch.v) : cabs2(cadd(ch.u, ch.v));
    }
    if (kind == LRE_STATE_W) {
        const Cplx u2 = cadd(cmul(ch.u, c0), cmul(ch.v, c1));
        ch.v = cmul(ch.v, c0);
        ch.u = u2;
        return cabs2(ch.u) + (double)r * cabs2(ch.v);
    }
    if (kind == LRE_STATE_PRODUCTZ) {
        const int beta = (int)((bits >> (n - 1 - j)) & 1);
        ch.u = cmul(ch.u, beta ? c1 : c0);
        return cabs2(ch.u);
    }
    return 1.0;  // maxmixed
}

// setting digits of w (qubit 1 first; X=0, Y=1, Z=2)
__device__ __forceinline__ void setting_axes(int64_t w, int n, int ax[16]) {
    int64_t x = w;
    for (int k = n - 1; k >= 0; --k) {
        ax[k] = (int)(x % 3);
        x /= 3;
    }
}

// One shot of setting w: outcome bits drawn qubit by qubit from the exact
// conditional probabilities, Philox4x32-10 keyed on (seed), counter (shot,
// qubit group, w) — the same stream whether counts or outcome lists are made.
__device__ __forceinline__ uint32_t sample_outcome(int kind, int n, int64_t bits, int64_t shot, int64_t w, uint2 key,
                                                   const int ax[16]) {
    Chain ch = chain_init(kind, n);
    uint32_t s = 0;
    uint4 rnd = make_uint4(0, 0, 0, 0);
    for (int j = 0; j < n; ++j) {
        if ((j & 3) == 0)
            rnd = Philox::gen(make_uint4((uint32_t)shot, (uint32_t)(j >> 2) | ((uint32_t)(shot >> 32) << 8), (uint32_t)w,
                                         (uint32_t)(w >> 32)),
                              key);
        const uint32_t ru = (j & 3) == 0 ? rnd.x : (j & 3) == 1 ? rnd.y : (j & 3) == 2 ? rnd.z : rnd.w;
        const double U = ((double)ru + 0.5) * 2.3283064365386963e-10;  // (0,1)
        Chain c0 = ch, c1 = ch;
        const double w0 = chain_step(kind, bits, n, j, ax[j], 0, c0);
        const double w1 = chain_step(kind, bits, n, j, ax[j], 1, c1);
        const int bit = (U * (w0 + w1) < w0) ? 0 : 1;
        ch = bit ? c1 : c0;
        s = (s << 1) | (uint32_t)bit;
    }
    return s;
}

template <typename T>
__global__ void __launch_bounds__(256) gen_sampled_kernel(int kind, int n, int64_t bits, int64_t shots, uint64_t seed,
                                                          int64_t w_begin, int64_t w_end, T *__restrict__ out) {
    extern __shared__ unsigned int hist[];
    const int d = 1 << n;
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    for (int64_t w = w_begin + blockIdx.x; w < w_end; w += gridDim.x) {
        for (int j = threadIdx.x; j < d; j += blockDim.x) hist[j] = 0;
        int ax[16];
        setting_axes(w, n, ax);
        __syncthreads();
        for (int64_t shot = threadIdx.x; shot < shots; shot += blockDim.x)
            atomicAdd(&hist[sample_outcome(kind, n, bits, shot, w, key, ax)], 1u);
        __syncthreads();
        T *row = out + (w - w_begin) * (int64_t)d;
        for (int j = threadIdx.x; j < d; j += blockDim.x) row[j] = (T)hist[j];
        __syncthreads();
    }
}

// Outcome-list record: out[(w - w_begin) * shots + shot] = outcome of that shot
__global__ void __launch_bounds__(256) gen_outcomes_kernel(int kind, int n, int64_t bits, int64_t shots, uint64_t seed,
                                                           int64_t w_begin, int64_t w_end, uint16_t *__restrict__ out) {
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    for (int64_t w = w_begin + blockIdx.x; w < w_end; w += gridDim.x) {
        int ax[16];
        setting_axes(w, n, ax);
        for (int64_t shot = threadIdx.x; shot < shots; shot += blockDim.x)
            out[(w - w_begin) * shots + shot] = (uint16_t)sample_outcome(kind, n, bits, shot, w, key, ax);
    }
}

// Outcome lists -> dense counts (record ingestion for sampled data: the host
// ships 2 bytes per shot instead of 2^n counts per setting).  One CTA per
// setting row at a time: shared-memory histogram, then one coalesced row store.
template <typename T>
__global__ void __launch_bounds__(512) counts_from_outcomes_kernel(const uint16_t *__restrict__ outcomes, int n,
                                                                   int64_t shots, int64_t rows, T *__restrict__ out) {
    extern __shared__ unsigned int hist[];
    const int d = 1 << n;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        for (int j = threadIdx.x; j < d; j += blockDim.x) hist[j] = 0;
        __syncthreads();
        const uint16_t *o = outcomes + r * shots;
        for (int64_t k = threadIdx.x; k < shots; k += blockDim.x) {
            const unsigned int s = __ldcs(o + k);
            if (s < (unsigned)d) atomicAdd(&hist[s], 1u);
        }
        __syncthreads();
        T *row = out + r * (int64_t)d;
        if constexpr (sizeof(T) == 2) {
            for (int j = 2 * threadIdx.x; j < d; j += 2 * blockDim.x)
                __stcs(reinterpret_cast<uint32_t *>(row + j), hist[j] | (hist[j + 1] << 16));
        } else {
            for (int j = threadIdx.x; j < d; j += blockDim.x) __stcs(row + j, (T)hist[j]);
        }
        __syncthreads();
    }
}

template <typename T>
__global__ void gen_exact_kernel(int kind, int n, int64_t bits, int64_t shots, int64_t w_begin, int64_t w_end,
                                 T *__restrict__ out, int *__restrict__ err) {
    const int d = 1 << n;
    for (int64_t w = w_begin + blockIdx.x; w < w_end; w += gridDim.x) {
        int ax[16];
        int64_t x = w;
        for (int k = n - 1; k >= 0; --k) {
            ax[k] = (int)(x % 3);
            x /= 3;
        }
        for (int s = threadIdx.x; s < d; s += blockDim.x) {
            double p;
            if (kind == LRE_STATE_MAXMIXED) {
                p = 1.0 / (double)d;
            } else {
                Chain ch = chain_init(kind, n);
                double wgt = 1.0;
                for (int j = 0; j < n; ++j) wgt = chain_step(kind, bits, n, j, ax[j], (s >> (n - 1 - j)) & 1, ch);
                p = wgt;  // after the last qubit the weight is |amplitude|^2
            }
            const double scaled = p * (double)shots;
            const double rounded = rint(scaled);
            if (fabs(scaled - rounded) > 1e-9 * (1.0 + scaled)) atomicExch(err, 1);
            out[(w - w_begin) * (int64_t)d + s] = (T)(int64_t)rounded;
        }
    }
}

template <typename T>
static int gen_t(int kind, int n, int64_t bits, int64_t shots, uint64_t seed, int exact, int64_t w_begin, int64_t w_end,
                 void *out, cudaStream_t s) {
    const int64_t rows = w_end - w_begin;
    if (rows <= 0) return LRE_OK;
    const unsigned blocks = (unsigned)std::min<int64_t>(rows, (int64_t)num_sms() * 16);
    if (exact) {
        int *err = nullptr;
        if (cudaMallocAsync(&err, sizeof(int), s) != cudaSuccess) return LRE_ECUDA;
        cudaMemsetAsync(err, 0, sizeof(int), s);
        gen_exact_kernel<T><<<blocks, 256, 0, s>>>(kind, n, bits, shots, w_begin, w_end, reinterpret_cast<T *>(out), err);
        count_launch();
        int herr = 0;
        cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaFreeAsync(err, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) return LRE_ECUDA;
        return herr ? LRE_EINVAL : LRE_OK;
    }
    const size_t smem = ((size_t)1 << n) * sizeof(unsigned int);
    cudaError_t e = cudaFuncSetAttribute(gen_sampled_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return LRE_ECUDA;
    gen_sampled_kernel<T><<<blocks, 256, smem, s>>>(kind, n, bits, shots, seed, w_begin, w_end, reinterpret_cast<T *>(out));
    count_launch();
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

int generate_outcomes_impl(int kind, int n, int64_t bits, int64_t shots, uint64_t seed, int64_t w_begin,
                           int64_t w_end, uint16_t *out, cudaStream_t s) {
    if (n < 1 || n > 16) return LRE_EUNSUPPORTED;
    if (kind < LRE_STATE_MAXMIXED || kind > LRE_STATE_W || shots < 1) return LRE_EINVAL;
    const int64_t rows = w_end - w_begin;
    if (rows <= 0) return LRE_OK;
    const unsigned blocks = (unsigned)std::min<int64_t>(rows, (int64_t)num_sms() * 16);
    gen_outcomes_kernel<<<blocks, 256, 0, s>>>(kind, n, bits, shots, seed, w_begin, w_end, out);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

template <typename T>
static int hist_t(const uint16_t *outcomes, int n, int64_t shots, int64_t rows, void *counts, cudaStream_t s) {
    const size_t smem = ((size_t)1 << n) * sizeof(unsigned int);
    cudaError_t e = cudaFuncSetAttribute(counts_from_outcomes_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return LRE_ECUDA;
    const int sms = num_sms();
    const int per_sm = std::max(1, std::min(4, (int)((200 * 1024) / smem)));
    const unsigned blocks = (unsigned)std::min<int64_t>(rows, (int64_t)sms * per_sm);
    counts_from_outcomes_kernel<T><<<blocks, 512, smem, s>>>(outcomes, n, shots, rows, reinterpret_cast<T *>(counts));
    count_launch();
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

int counts_from_outcomes_impl(const uint16_t *outcomes, int n, int64_t shots, int64_t rows, void *counts, int dtype,
                              cudaStream_t s) {
    if (n < 1 || n > 16) return LRE_EUNSUPPORTED;
    if (rows <= 0) return LRE_OK;
    switch (dtype) {
    case LRE_U8: return hist_t<uint8_t>(outcomes, n, shots, rows, counts, s);
    case LRE_U16: return hist_t<uint16_t>(outcomes, n, shots, rows, counts, s);
    case LRE_I32: return hist_t<int32_t>(outcomes, n, shots, rows, counts, s);
    case LRE_I64: return hist_t<int64_t>(outcomes, n, shots, rows, counts, s);
    default: return LRE_EINVAL;
    }
}

int generate_impl(int kind, int n, int64_t bits, int64_t shots, uint64_t seed, int exact, int64_t w_begin,
                  int64_t w_end, void *out, int dtype, cudaStream_t s) {
    if (n < 1 || n > 14) return LRE_EUNSUPPORTED;
    if (kind < LRE_STATE_MAXMIXED || kind > LRE_STATE_W) return LRE_EINVAL;
    if (shots < 1) return LRE_EINVAL;
    switch (dtype) {
    case LRE_U8: return gen_t<uint8_t>(kind, n, bits, shots, seed, exact, w_begin, w_end, out, s);
    case LRE_U16: return gen_t<uint16_t>(kind, n, bits, shots, seed, exact, w_begin, w_end, out, s);
    case LRE_I32: return gen_t<int32_t>(kind, n, bits, shots, seed, exact, w_begin, w_end, out, s);
    case LRE_I64: return gen_t<int64_t>(kind, n, bits, shots, seed, exact, w_begin, w_end, out, s);
    default: return LRE_EINVAL;
    }
}

}  // namespace lre
