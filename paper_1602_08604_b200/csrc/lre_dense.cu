// Arbitrary (dense / mixed) states on the device: the inverse of step (ii)
// and a record generator driven by theta ("mixed
// states"; reference simulate.py:114-151 dense_to_theta /
// _theta_probability_block and :224-242 sample_counts).
//
//   dense_to_theta_kernel   rho (2^n x 2^n complex128) -> theta (natural):
//       per X-mask m, v[a] = 2^{-n/2} sum_r rho[r, r^m] (-1)^{a.r}, then
//       theta(m, a) = Re(v[a] i^{pc(a & m)}) — exactly the inverse of the
//       assembly map mu[r, r^m] = 2^{-n/2} sum_a theta(m,a) (-i)^{pc(a&m)} (-1)^{a.r}.
//   gen_theta_kernel        theta -> sampled counts of settings [w_begin, w_end):
//       p_w(s) = 2^{-n/2} sum_{mask} theta[a(w, mask)] (-1)^{pc(s & mask)}
//       (a(w, mask) = setting digit on the mask's qubits, I elsewhere), one
//       shared-memory WHT per setting, clamp + CDF, then `shots` inverse-CDF
//       draws from the (seed, setting, shot)-keyed Philox stream.
#include <algorithm>
#include <cmath>

#include "lre_internal.cuh"

namespace lre {

constexpr int DENSE_THREADS = 256;

// in-place radix-2 WHT of `len` doubles in shared memory (len = 2^logn)
__device__ __forceinline__ void smem_wht(double *x, int logn) {
    const int len = 1 << logn;
    for (int h = 1; h < len; h <<= 1) {
        for (int i = threadIdx.x; i < (len >> 1); i += blockDim.x) {
            const int lo = ((i & ~(h - 1)) << 1) | (i & (h - 1));
            const double a = x[lo], b = x[lo + h];
            x[lo] = a + b;
            x[lo + h] = a - b;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(DENSE_THREADS) dense_to_theta_kernel(const double2 *__restrict__ rho, int n,
                                                                        double *__restrict__ theta) {
    extern __shared__ double dsm[];
    const int d = 1 << n;
    double *re = dsm, *im = dsm + d;
    const double scale = exp2(-0.5 * n);
    for (int m = blockIdx.x; m < d; m += gridDim.x) {
        for (int r = threadIdx.x; r < d; r += blockDim.x) {
            const double2 v = rho[(int64_t)r * d + (r ^ m)];
            re[r] = v.x;
            im[r] = v.y;
        }
        __syncthreads();
        smem_wht(re, n);
        smem_wht(im, n);
        for (int a = threadIdx.x; a < d; a += blockDim.x) {
            const double vr = scale * re[a], vi = scale * im[a];
            double t;
            switch (__popc((unsigned)(a & m)) & 3) {  // Re(v * i^k)
            case 0: t = vr; break;
            case 1: t = -vi; break;
            case 2: t = -vr; break;
            default: t = vi; break;
            }
            theta[ma_to_natural((uint32_t)m, (uint32_t)a)] = t;
        }
        __syncthreads();
    }
}

template <typename T>
__global__ void __launch_bounds__(DENSE_THREADS) gen_theta_kernel(const double *__restrict__ theta, int n, int64_t shots,
                                                                  uint64_t seed, int64_t w_begin, int64_t w_end,
                                                                  T *__restrict__ out) {
    extern __shared__ double gsm[];
    const int d = 1 << n;
    double *p = gsm;                                              // probabilities, then CDF
    unsigned int *hist = reinterpret_cast<unsigned int *>(gsm + d);  // counts
    __shared__ double part[DENSE_THREADS];
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    const double scale = exp2(-0.5 * n);
    const int per = (d + DENSE_THREADS - 1) / DENSE_THREADS;  // CDF chunk per thread
    for (int64_t w = w_begin + blockIdx.x; w < w_end; w += gridDim.x) {
        int ax[16];
        {
            int64_t x = w;
            for (int k = n - 1; k >= 0; --k) {
                ax[k] = (int)(x % 3);
                x /= 3;
            }
        }
        // gather theta on the support of w: mask bit (n-1-k) <-> qubit k carries digit ax[k] + 1
        for (int mask = threadIdx.x; mask < d; mask += blockDim.x) {
            uint64_t nat = 0;
            for (int k = 0; k < n; ++k) {
                const int dig = ((mask >> (n - 1 - k)) & 1) ? ax[k] + 1 : 0;
                nat = (nat << 2) | (uint64_t)dig;
            }
            p[mask] = __ldg(theta + nat);
            hist[mask] = 0u;
        }
        __syncthreads();
        smem_wht(p, n);
        // clamp negatives (rounding of exact zeros), chunk-local inclusive prefix sums
        const int c0 = threadIdx.x * per, c1 = min(d, c0 + per);
        double run = 0.0;
        for (int s = c0; s < c1; ++s) {
            run += fmax(scale * p[s], 0.0);
            p[s] = run;
        }
        part[threadIdx.x] = run;
        __syncthreads();
        if (threadIdx.x == 0) {  // exclusive scan of the chunk totals (fixed order: deterministic)
            double acc = 0.0;
            for (int i = 0; i < DENSE_THREADS; ++i) {
                const double v = part[i];
                part[i] = acc;
                acc += v;
            }
        }
        __syncthreads();
        const double off = part[threadIdx.x];
        for (int s = c0; s < c1; ++s) p[s] += off;
        __syncthreads();
        const double total = p[d - 1];
        for (int64_t shot = threadIdx.x; shot < shots; shot += blockDim.x) {
            const uint4 r = Philox::gen(make_uint4((uint32_t)shot, (uint32_t)(shot >> 32) | 0x80000000u, (uint32_t)w,
                                                   (uint32_t)(w >> 32)),
                                        key);
            // 53-bit uniform in [0, 1)
            const double u = ((double)(((uint64_t)r.x << 21) ^ (uint64_t)r.y) * 0x1.0p-53) * total;
            int lo = 0, hi = d - 1;  // first s with CDF[s] > u
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (p[mid] > u) hi = mid;
                else lo = mid + 1;
            }
            atomicAdd(&hist[lo], 1u);
        }
        __syncthreads();
        T *row = out + (w - w_begin) * (int64_t)d;
        for (int s = threadIdx.x; s < d; s += blockDim.x) row[s] = (T)hist[s];
        __syncthreads();
    }
}

int dense_to_theta_impl(const double *rho, int n, double *theta, cudaStream_t s) {
    if (n < 1 || n > 12) return LRE_EUNSUPPORTED;
    const size_t smem = 2 * ((size_t)1 << n) * sizeof(double);
    if (cudaFuncSetAttribute(dense_to_theta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return LRE_ECUDA;
    const int grid = (int)std::min<int64_t>((int64_t)1 << n, (int64_t)num_sms() * 4);
    dense_to_theta_kernel<<<grid, DENSE_THREADS, smem, s>>>(reinterpret_cast<const double2 *>(rho), n, theta);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

// exact outcome probabilities of settings [w_begin, w_end) (simulate.py:141-151 and
// probabilities_block's random-state branch, :176-177): per setting, theta on the
// setting's support, one WHT, * 2^{-n/2}, clipped to [0, 1]
__global__ void __launch_bounds__(DENSE_THREADS) theta_prob_kernel(const double *__restrict__ theta, int n,
                                                                   int64_t w_begin, int64_t w_end, int clip,
                                                                   double *__restrict__ out) {
    extern __shared__ double psm[];
    const int d = 1 << n;
    const double scale = exp2(-0.5 * n);
    for (int64_t w = w_begin + blockIdx.x; w < w_end; w += gridDim.x) {
        int ax[16];
        {
            int64_t x = w;
            for (int k = n - 1; k >= 0; --k) {
                ax[k] = (int)(x % 3);
                x /= 3;
            }
        }
        for (int mask = threadIdx.x; mask < d; mask += blockDim.x) {
            uint64_t nat = 0;
            for (int k = 0; k < n; ++k) {
                const int dig = ((mask >> (n - 1 - k)) & 1) ? ax[k] + 1 : 0;
                nat = (nat << 2) | (uint64_t)dig;
            }
            psm[mask] = __ldg(theta + nat);
        }
        __syncthreads();
        smem_wht(psm, n);
        double *row = out + (w - w_begin) * (int64_t)d;
        for (int s = threadIdx.x; s < d; s += blockDim.x)
            row[s] = clip ? fmin(fmax(scale * psm[s], 0.0), 1.0) : scale * psm[s];
        __syncthreads();
    }
}

int theta_probabilities_impl(const double *theta, int n, int64_t w_begin, int64_t w_end, int clip, double *out,
                             cudaStream_t s) {
    if (n < 1 || n > 12) return LRE_EUNSUPPORTED;
    if (w_end <= w_begin) return LRE_OK;
    const size_t smem = ((size_t)1 << n) * sizeof(double);
    if (cudaFuncSetAttribute(theta_prob_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return LRE_ECUDA;
    const int grid = (int)std::min<int64_t>(w_end - w_begin, (int64_t)num_sms() * 8);
    theta_prob_kernel<<<grid, DENSE_THREADS, smem, s>>>(theta, n, w_begin, w_end, clip, out);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

template <typename T>
static int gen_theta_t(const double *theta, int n, int64_t shots, uint64_t seed, int64_t w_begin, int64_t w_end,
                       void *out, cudaStream_t s) {
    const size_t smem = ((size_t)1 << n) * (sizeof(double) + sizeof(unsigned int));
    if (cudaFuncSetAttribute(gen_theta_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return LRE_ECUDA;
    const int64_t rows = w_end - w_begin;
    const int grid = (int)std::min<int64_t>(rows, (int64_t)num_sms() * 8);
    gen_theta_kernel<T><<<grid, DENSE_THREADS, smem, s>>>(theta, n, shots, seed, w_begin, w_end,
                                                           reinterpret_cast<T *>(out));
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

int generate_theta_impl(const double *theta, int n, int64_t shots, uint64_t seed, int64_t w_begin, int64_t w_end,
                        void *out, int dtype, cudaStream_t s) {
    if (n < 1 || n > 12) return LRE_EUNSUPPORTED;
    if (w_end <= w_begin) return LRE_OK;
    switch (dtype) {
    case LRE_U8: return gen_theta_t<uint8_t>(theta, n, shots, seed, w_begin, w_end, out, s);
    case LRE_U16: return gen_theta_t<uint16_t>(theta, n, shots, seed, w_begin, w_end, out, s);
    case LRE_I32: return gen_theta_t<int32_t>(theta, n, shots, seed, w_begin, w_end, out, s);
    case LRE_I64: return gen_theta_t<int64_t>(theta, n, shots, seed, w_begin, w_end, out, s);
    default: return LRE_EINVAL;
    }
}

}  // namespace lre
