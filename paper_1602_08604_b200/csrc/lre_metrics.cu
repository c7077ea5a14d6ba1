// Error metrics on the device (reference metrics.py).
//
// Deterministic fp64 reductions over an estimate already in HBM, so that the
// paper's error sweep (Fig. 3) runs at n = 14 without a host copy of the
// 4 GB estimate:
//   * reduce_partials_kernel / reduce_final_kernel: fixed grid of
//     LRE_REDUCE_BLOCKS CTAs -> per-CTA partials -> one CTA sums them in
//     index order (bit-reproducible for a given count).  HBM-bound: 8 bytes
//     (16 with a second operand) per element.
//       LRE_REDUCE_SUM_SQ        sum (a_i - b_i)^2            (metrics.py:28-35)
//       LRE_REDUCE_SUM_SQRT      sum sqrt(max(a_i, 0) * scale) (metrics.py:88-92)
//       LRE_REDUCE_SUM_SQ_ZC     sum 3^zc(i) a_i^2 over natural theta
//                                (the dense predictor's sum_{w,s} p_ws^2)
//   * truth_terms_kernel: Re Tr(A rho_true) and Tr(rho_true^2) for the
//     generator's states (maxmixed / GHZ / productz / W), whose state vectors
//     have at most n nonzero amplitudes — the cross term of the squared HS
//     distance and the pure-state fidelity <psi|A|psi> (metrics.py:57-85).
#include <cmath>

#include "lre_internal.cuh"

namespace lre {

constexpr int RED_THREADS = 256;

__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    v = 0.0;
    if (warp == 0) {
        v = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    return v;  // valid in thread 0
}

// 3^zc(i) for a natural Pauli index: zc = identity digits
__device__ __forceinline__ double pow3_identities(int64_t i, int n) {
    const uint64_t u = (uint64_t)i;
    const int zc = n - __popcll((u | (u >> 1)) & 0x5555555555555555ull);
    double r = 1.0;
    for (int k = 0; k < zc; ++k) r *= 3.0;
    return r;
}

template <int OP>
__global__ void __launch_bounds__(RED_THREADS) reduce_partials_kernel(const double *__restrict__ a,
                                                                       const double *__restrict__ b, int64_t count,
                                                                       double scale, int n, double *__restrict__ part) {
    __shared__ double sh[32];
    double acc = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const double x = __ldcs(a + i);
        if constexpr (OP == LRE_REDUCE_SUM_SQ) {
            const double d = b ? x - __ldcs(b + i) : x;
            acc = fma(d, d, acc);
        } else if constexpr (OP == LRE_REDUCE_SUM_SQRT) {
            acc += sqrt(fmax(x, 0.0) * scale);
        } else {
            acc = fma(pow3_identities(i, n) * x, x, acc);
        }
    }
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(RED_THREADS) reduce_final_kernel(double *__restrict__ out, int parts) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < parts; i += blockDim.x) acc += out[1 + i];
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) out[0] = s;
}

int reduce_impl(int op, const double *a, const double *b, int64_t count, double scale, double *out,
                cudaStream_t s) {
    if (count < 0) return LRE_EINVAL;
    int n = 0;
    if (op == LRE_REDUCE_SUM_SQ_ZC) {
        while (n < 32 && ((int64_t)1 << (2 * n)) < count) ++n;
        if (((int64_t)1 << (2 * n)) != count) return LRE_EINVAL;
    }
    const int grid = LRE_REDUCE_BLOCKS;
    double *part = out + 1;
    switch (op) {
    case LRE_REDUCE_SUM_SQ:
        reduce_partials_kernel<LRE_REDUCE_SUM_SQ><<<grid, RED_THREADS, 0, s>>>(a, b, count, scale, n, part);
        break;
    case LRE_REDUCE_SUM_SQRT:
        reduce_partials_kernel<LRE_REDUCE_SUM_SQRT><<<grid, RED_THREADS, 0, s>>>(a, b, count, scale, n, part);
        break;
    case LRE_REDUCE_SUM_SQ_ZC:
        reduce_partials_kernel<LRE_REDUCE_SUM_SQ_ZC><<<grid, RED_THREADS, 0, s>>>(a, b, count, scale, n, part);
        break;
    default: return LRE_EINVAL;
    }
    reduce_final_kernel<<<1, RED_THREADS, 0, s>>>(out, grid);
    count_launch(2);
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

// support of the generator's pure states: index k -> (basis state, amplitude)
__device__ __forceinline__ void pure_support(int kind, int n, int64_t bits, int k, int64_t &idx, double &amp) {
    if (kind == LRE_STATE_GHZ) {
        idx = k == 0 ? 0 : ((int64_t)1 << n) - 1;
        amp = 0.70710678118654752440;
    } else if (kind == LRE_STATE_PRODUCTZ) {
        idx = bits;
        amp = 1.0;
    } else {  // W: |2^(n-1-k)> (qubit k+1 excited), amplitude 1/sqrt(n)
        idx = (int64_t)1 << (n - 1 - k);
        amp = rsqrt((double)n);
    }
}

__global__ void __launch_bounds__(RED_THREADS) truth_terms_kernel(const double2 *__restrict__ A, int n, int kind,
                                                                   int64_t bits, double *__restrict__ out) {
    __shared__ double sh[32];
    const int64_t d = (int64_t)1 << n;
    double acc = 0.0;
    double purity;
    if (kind == LRE_STATE_MAXMIXED) {
        for (int64_t i = threadIdx.x; i < d; i += blockDim.x) acc += A[i * d + i].x;
        acc /= (double)d;
        purity = 1.0 / (double)d;
    } else {
        const int m = kind == LRE_STATE_GHZ ? 2 : kind == LRE_STATE_PRODUCTZ ? 1 : n;
        for (int p = threadIdx.x; p < m * m; p += blockDim.x) {
            int64_t i, j;
            double ai, aj;
            pure_support(kind, n, bits, p / m, i, ai);
            pure_support(kind, n, bits, p % m, j, aj);
            acc += ai * aj * A[i * d + j].x;  // imaginary parts cancel for Hermitian A
        }
        purity = 1.0;
    }
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) {
        out[0] = s;
        out[1] = purity;
    }
}

int truth_terms_impl(const double *a, int n, int kind, int64_t bits, double *out, cudaStream_t s) {
    truth_terms_kernel<<<1, RED_THREADS, 0, s>>>(reinterpret_cast<const double2 *>(a), n, kind, bits, out);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

}  // namespace lre
