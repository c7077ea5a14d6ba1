// Step (ii) of the LRE hot path on B200: theta (mask-major) -> mu (XOR-diagonals).
//
// Reference: pipeline.py:93-101,141-161 (step_two_assemble) with
// pauli.py:270-297 (omega_gather_indices / omega_phase_factors).  For every
// X/Y mask m the reference gathers v[a] = theta[(m,a)] * (-i)^popcount(a&m),
// runs a complex WHT of length 2^n and writes mu[r, r^m].
//
// B200 design: with w[a] = theta[(m,a)] * (-1)^floor(pc(a&m)/2)
// and the real WHT F = H w, the complex WHT splits exactly as
//     mu[r, r^m] = 2^{-n/2} ( (F[r] + F[r^m]) / 2  -  i (F[r] - F[r^m]) / 2 ),
// so one real fp64 transform per mask replaces the complex one.  A CTA owns
// MPC consecutive masks, keeps their transforms in shared memory (padded one
// double per 16 to keep radix-16 rounds bank-conflict free) and writes MPC
// adjacent complex columns per row, so rows of mu are written in runs.
#include <algorithm>
#include <cmath>

#include "lre_internal.cuh"

namespace lre {

__device__ __forceinline__ int padix(int i) { return i + (i >> 4); }

template <int NB>
__device__ __forceinline__ void wht_round(double *buf, int Dp, int logd, int mpc, int shift) {
    const int groups = (1 << logd) >> NB;
    const int lowmask = (1 << shift) - 1;
    for (int it = threadIdx.x; it < mpc * groups; it += blockDim.x) {
        const int ml = it / groups, gi = it - ml * groups;
        const int base = (gi & lowmask) | ((gi >> shift) << (shift + NB));
        double *b = buf + ml * Dp;
        double v[1 << NB];
#pragma unroll
        for (int k = 0; k < (1 << NB); ++k) v[k] = b[padix(base + (k << shift))];
#pragma unroll
        for (int h = 1; h < (1 << NB); h <<= 1)
#pragma unroll
            for (int k = 0; k < (1 << NB); ++k)
                if (!(k & h)) {
                    const double x = v[k], y = v[k + h];
                    v[k] = x + y;
                    v[k + h] = x - y;
                }
#pragma unroll
        for (int k = 0; k < (1 << NB); ++k) b[padix(base + (k << shift))] = v[k];
    }
}

__global__ void __launch_bounds__(1024) assemble_kernel(const double *__restrict__ theta, int layout, int logd,
                                                        int64_t m_begin, int64_t S, int mpc, double scale_half,
                                                        double2 *__restrict__ mu) {
    extern __shared__ double sbuf[];
    const int d = 1 << logd;
    const int Dp = d + (d >> 4) + 1;
    const int64_t mloc0 = (int64_t)blockIdx.x * mpc;  // first mask of this CTA, relative to m_begin
    // load + sign twist w[a] = theta[(m,a)] * (-1)^floor(popc(a&m)/2)
    for (int e = threadIdx.x; e < mpc * d; e += blockDim.x) {
        const int ml = e >> logd, a = e & (d - 1);
        const uint32_t m = (uint32_t)(m_begin + mloc0 + ml);
        // NATURAL: full theta, gathered at the natural index of (m, a); the CTA's
        // consecutive masks cover all digits of the low qubits, so the gather
        // reads whole lines.  MASK_MAJOR: the slice of masks [m_begin, m_end).
        const int64_t idx = layout == LRE_LAYOUT_NATURAL ? (int64_t)ma_to_natural(m, (uint32_t)a)
                                                         : (mloc0 + ml) * (int64_t)d + a;
        double v = __ldg(theta + idx);
        if ((__popc((uint32_t)a & m) >> 1) & 1) v = -v;
        sbuf[ml * Dp + padix(a)] = v;
    }
    __syncthreads();
    int shift = 0;
    while (shift < logd) {
        const int nb = logd - shift >= 4 ? 4 : logd - shift;
        switch (nb) {
        case 4: wht_round<4>(sbuf, Dp, logd, mpc, shift); break;
        case 3: wht_round<3>(sbuf, Dp, logd, mpc, shift); break;
        case 2: wht_round<2>(sbuf, Dp, logd, mpc, shift); break;
        default: wht_round<1>(sbuf, Dp, logd, mpc, shift); break;
        }
        shift += nb;
        __syncthreads();
    }
    // mu[r, r^m] for the CTA's masks; consecutive threads take consecutive
    // masks of the same row so each row is written as an mpc-long run.
    for (int e = threadIdx.x; e < mpc * d; e += blockDim.x) {
        const int ml = e % mpc, r = e / mpc;
        const uint32_t m = (uint32_t)(m_begin + mloc0 + ml);
        const double *b = sbuf + ml * Dp;
        const double f1 = b[padix(r)], f2 = b[padix(r ^ m)];
        const int64_t col = (int64_t)((r ^ m) & (uint32_t)(S - 1));
        __stcs(mu + (int64_t)r * S + col, make_double2(scale_half * (f1 + f2), scale_half * (f2 - f1)));
    }
}

int assemble_impl(const double *theta, int layout, int n, int64_t m_begin, int64_t m_end, double *mu,
                  cudaStream_t s) {
    const int64_t S = m_end - m_begin;
    const int64_t d = (int64_t)1 << n;
    if (n < 1 || n > 14) return LRE_EUNSUPPORTED;
    if (S <= 0 || (S & (S - 1)) || m_begin % S || m_end > d) return LRE_EINVAL;
    int mpc = 1;
    while (mpc < 8 && (int64_t)mpc * 2 <= S && ((int64_t)mpc * 2 * d) <= (1 << 14)) mpc *= 2;
    const int Dp = (int)(d + (d >> 4) + 1);
    const size_t smem = (size_t)mpc * Dp * sizeof(double);
    int threads = (int)std::min<int64_t>(1024, std::max<int64_t>(64, mpc * d / 16));
    cudaError_t e = cudaFuncSetAttribute(assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return LRE_ECUDA;
    const double scale_half = 0.5 * pow(2.0, -n / 2.0);
    assemble_kernel<<<(unsigned)(S / mpc), threads, smem, s>>>(theta, layout, n, m_begin, S, mpc, scale_half,
                                                              reinterpret_cast<double2 *>(mu));
    count_launch();
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

}  // namespace lre
