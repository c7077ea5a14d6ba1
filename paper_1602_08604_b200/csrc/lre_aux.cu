// Auxiliary kernels around the LRE hot path: record validation, numerator
// finalisation, theta relayout.
#include <algorithm>
#include <climits>
#include <cmath>

#include <type_traits>

#include "lre_internal.cuh"

namespace lre {

// ---------------------------------------------------------------------------
// validation (reference records.py:34-56): per-row sums and the minimum count
// ---------------------------------------------------------------------------
template <typename T>
__global__ void validate_kernel(const T *__restrict__ counts, int n, int64_t rows, int64_t shots,
                                long long *__restrict__ result, bool aligned16) {
    const int64_t d = (int64_t)1 << n;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    long long local_min = LLONG_MAX;
    constexpr int VE = 16 / sizeof(T);  // elements per 16-byte load
    const bool vec = aligned16 && (d % (32 * VE)) == 0;  // whole rows of 512-byte warp loads
    for (int64_t r = warp; r < rows; r += nwarps) {
        const T *row = counts + r * d;
        long long s = 0;
        if (vec) {
            const uint4 *row4 = reinterpret_cast<const uint4 *>(row);
            for (int64_t j = lane; j < d / VE; j += 32) {
                const uint4 q = __ldcs(row4 + j);
                const T *e = reinterpret_cast<const T *>(&q);
#pragma unroll
                for (int k = 0; k < VE; ++k) {
                    const long long v = (long long)e[k];
                    s += v;
                    if constexpr (std::is_signed<T>::value) local_min = v < local_min ? v : local_min;
                }
            }
            if constexpr (!std::is_signed<T>::value) local_min = 0;  // unsigned counts are never negative
        } else {
            for (int64_t j = lane; j < d; j += 32) {
                const long long v = (long long)row[j];
                s += v;
                local_min = v < local_min ? v : local_min;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0 && s != shots) atomicMin(&result[0], (long long)r);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long other = __shfl_xor_sync(0xffffffffu, local_min, o);
        local_min = other < local_min ? other : local_min;
    }
    if (lane == 0) atomicMin(&result[2], local_min);
}

template <typename T>
__global__ void row_sum_kernel(const T *__restrict__ counts, int n, long long *__restrict__ result) {
    const long long r = result[0];
    if (r == LLONG_MAX) return;
    const int64_t d = (int64_t)1 << n;
    long long s = 0;
    for (int64_t j = threadIdx.x; j < d; j += blockDim.x) s += (long long)counts[r * d + j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ long long part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += part[i];
        result[1] = t;
    }
}

__global__ void init_result_kernel(long long *result) {
    result[0] = LLONG_MAX;
    result[1] = 0;
    result[2] = LLONG_MAX;
}

template <typename T>
static int validate_t(const void *counts, int n, int64_t rows, int64_t shots, int64_t *result, cudaStream_t s) {
    long long *res = reinterpret_cast<long long *>(result);
    init_result_kernel<<<1, 1, 0, s>>>(res);
    const int64_t warps_needed = rows;
    const int64_t blocks = std::min<int64_t>((warps_needed + 7) / 8, (int64_t)num_sms() * 32);
    const bool aligned16 = (reinterpret_cast<uintptr_t>(counts) & 15) == 0;
    validate_kernel<T><<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(reinterpret_cast<const T *>(counts), n,
                                                                              rows, shots, res, aligned16);
    row_sum_kernel<T><<<1, 256, 0, s>>>(reinterpret_cast<const T *>(counts), n, res);
    count_launch(3);
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

int validate_impl(const void *counts, int dtype, int n, int64_t rows, int64_t shots, int64_t *result,
                  cudaStream_t s) {
    switch (dtype) {
    case LRE_U8: return validate_t<uint8_t>(counts, n, rows, shots, result, s);
    case LRE_U16: return validate_t<uint16_t>(counts, n, rows, shots, result, s);
    case LRE_I32: return validate_t<int32_t>(counts, n, rows, shots, result, s);
    case LRE_I64: return validate_t<int64_t>(counts, n, rows, shots, result, s);
    default: return LRE_EINVAL;
    }
}

// ---------------------------------------------------------------------------
// finalisation: exact numerators -> theta (pipeline.py:138, records.py:62-64)
// ---------------------------------------------------------------------------
__global__ void finalize_kernel(const int64_t *__restrict__ num, int n, int layout, int64_t begin, int64_t end,
                                const Factors fac, double *__restrict__ theta) {
    __shared__ double sfac[33];
    stage_factors(sfac, fac);
    __syncthreads();
    for (int64_t pos = begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < end;
         pos += (int64_t)gridDim.x * blockDim.x) {
        uint32_t m, a;
        if (layout == LRE_LAYOUT_MASK_MAJOR) {
            m = (uint32_t)(pos >> n);
            a = (uint32_t)(pos & (((int64_t)1 << n) - 1));
        } else {
            natural_to_ma((uint64_t)pos, m, a);
        }
        const int zc = n - __popc(m | a);
        // the same epilogue as the last fold pass of lre_step1 (bit-identical theta)
        theta[pos - begin] = (double)num[pos - begin] * sfac[zc];
    }
}

int finalize_impl(const int64_t *num, int n, int64_t shots, int layout, int64_t begin, int64_t end, double *theta,
                  cudaStream_t s) {
    if (end < begin) return LRE_EINVAL;
    if (end == begin) return LRE_OK;
    const int64_t blocks = std::min<int64_t>((end - begin + 255) / 256, (int64_t)num_sms() * 16);
    finalize_kernel<<<(unsigned)blocks, 256, 0, s>>>(num, n, layout, begin, end, make_factors(n, shots), theta);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

// ---------------------------------------------------------------------------
// relayout NATURAL <-> MASK_MAJOR (gather; writes coalesced)
// ---------------------------------------------------------------------------
__global__ void relayout_kernel(const double *__restrict__ src, int src_layout, int n, double *__restrict__ dst) {
    const int64_t total = (int64_t)1 << (2 * n);
    const int64_t dmask = ((int64_t)1 << n) - 1;
    for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < total;
         pos += (int64_t)gridDim.x * blockDim.x) {
        int64_t from;
        if (src_layout == LRE_LAYOUT_NATURAL) {  // dst is mask-major
            from = (int64_t)ma_to_natural((uint32_t)(pos >> n), (uint32_t)(pos & dmask));
        } else {  // dst is natural
            uint32_t m, a;
            natural_to_ma((uint64_t)pos, m, a);
            from = ((int64_t)m << n) | a;
        }
        dst[pos] = src[from];
    }
}

int relayout_impl(const double *src, int src_layout, int n, double *dst, cudaStream_t s) {
    const int64_t total = (int64_t)1 << (2 * n);
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16);
    relayout_kernel<<<(unsigned)blocks, 256, 0, s>>>(src, src_layout, n, dst);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

}  // namespace lre
