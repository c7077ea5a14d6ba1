// Step (ii) of the LRE hot path on B200: theta -> mu (XOR-diagonals).
//
// Reference: pipeline.py:93-101,141-161 (step_two_assemble) with
// pauli.py:270-297 (omega_gather_indices / omega_phase_factors).  For every
// X/Y mask m the reference gathers v[a] = theta[(m,a)] * (-i)^popcount(a&m),
// runs a complex WHT of length 2^n and writes mu[r, r^m].
//
// B200 design: with w[a] = theta[(m,a)] * (-1)^floor(pc(a&m)/2)
// and the real WHT F = H w, the complex WHT splits exactly as
//     mu[r, r^m] = 2^{-n/2} ( (F[r] + F[r^m]) / 2  -  i (F[r] - F[r^m]) / 2 ),
// so one real fp64 transform per mask replaces the complex one.
//
// A CTA owns a block of B consecutive masks (B = 2^j, the low j mask bits
// vary), keeps their transforms in shared memory (radix-16 rounds, one pad
// double per 16 so rounds are bank-conflict free) and
//   * gathers theta in NATURAL order as runs of 4^j contiguous doubles (the
//     low j qubits take all four Pauli digits across the block), and
//   * writes each row r of mu as B adjacent complex values (the columns
//     r ^ m of an aligned mask block are an aligned column block).
// When one mask fills the shared memory (n >= 13: 2^14 doubles), two CTAs
// form a cluster, each transforms one mask of an aligned pair, and the write
// phase reads the partner's transform through distributed shared memory so
// every row still gets a 32-byte pair.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>

#include "lre_internal.cuh"

namespace lre {

namespace cg = cooperative_groups;

__device__ __forceinline__ int padix(int i) { return i + (i >> 4); }

// 256-bit global accesses (sm_100): one transaction per 32-byte run / row segment
__device__ __forceinline__ void st256_cs(double2 *dst, double2 v0, double2 v1) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "d"(v0.x), "d"(v0.y), "d"(v1.x), "d"(v1.y)
                 : "memory");
}
__device__ __forceinline__ double4 ld256_nc(const double *src) {
    double4 v;
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(src));
    return v;
}

// Cluster barrier without release/acquire semantics: the end-of-iteration
// barrier only has to order the partners' DSMEM reads (already consumed by
// their stores) before this CTA overwrites its buffer.  cluster.sync()'s
// release would also wait for this thread's streaming global stores to
// drain (the "membar" stall in the n = 14 profile).
__device__ __forceinline__ void cluster_sync_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

template <int NB>
__device__ __forceinline__ void wht_round(double *buf, int Dp, int logd, int nm, int shift) {
    const int groups = (1 << logd) >> NB;
    const int lowmask = (1 << shift) - 1;
    for (int it = threadIdx.x; it < nm * groups; it += blockDim.x) {
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

__device__ __forceinline__ void wht_all(double *sbuf, int Dp, int logd, int nm) {
    int shift = 0;
    while (shift < logd) {
        const int nb = logd - shift >= 4 ? 4 : logd - shift;
        switch (nb) {
        case 4: wht_round<4>(sbuf, Dp, logd, nm, shift); break;
        case 3: wht_round<3>(sbuf, Dp, logd, nm, shift); break;
        case 2: wht_round<2>(sbuf, Dp, logd, nm, shift); break;
        default: wht_round<1>(sbuf, Dp, logd, nm, shift); break;
        }
        shift += nb;
        __syncthreads();
    }
}

struct AsmArgs {
    const double *theta;
    int layout;      // LRE_LAYOUT_NATURAL (full theta) or MASK_MAJOR (slice of [m_begin, m_end))
    int logd;        // n
    int logb;        // j: B = 2^j masks per CTA
    int cl;          // CTAs per cluster (1 or 2)
    int64_t m_begin;
    int64_t S;       // masks in the slice (power of two); mu rows are S complex wide
    int64_t groups;  // mask groups of B * cl masks
    double scale_half;
    double2 *mu;
};

// load + sign twist of the CTA's B masks [mloc0, mloc0 + B) into shared memory
__device__ __forceinline__ void asm_load(const AsmArgs &a, double *sbuf, int Dp, int64_t mloc0) {
    const int d = 1 << a.logd;
    const int B = 1 << a.logb;
    if (a.layout == LRE_LAYOUT_NATURAL) {
        // e = a_high * 4^j + d_low: consecutive threads read a contiguous run
        // of 4^j natural indices (the low j qubits' digits).
        const int j = a.logb;
        const uint32_t mhigh = (uint32_t)((a.m_begin + mloc0) >> j);
        for (int e = threadIdx.x; e < B * d; e += blockDim.x) {
            const uint32_t dlow = (uint32_t)e & ((1u << (2 * j)) - 1);
            const uint32_t ahigh = (uint32_t)e >> (2 * j);
            // decode the low digits: digit X/Y -> mask bit, Y/Z -> a bit
            const uint32_t hi = compact_odd(dlow), lo = compact_even(dlow);
            const uint32_t alow = hi, mlow = hi ^ lo;
            const uint32_t m = (mhigh << j) | mlow;
            const uint32_t av = (ahigh << j) | alow;
            const uint64_t nat = ma_to_natural(m, av);
            double v = __ldg(a.theta + nat);
            if ((__popc(av & m) >> 1) & 1) v = -v;
            sbuf[mlow * Dp + padix((int)av)] = v;
        }
    } else {
        for (int e = threadIdx.x; e < B * d; e += blockDim.x) {
            const int ml = e >> a.logd, av = e & (d - 1);
            const uint32_t m = (uint32_t)(a.m_begin + mloc0 + ml);
            double v = __ldg(a.theta + (mloc0 + ml) * (int64_t)d + av);
            if ((__popc((uint32_t)av & m) >> 1) & 1) v = -v;
            sbuf[ml * Dp + padix(av)] = v;
        }
    }
}

__global__ void __launch_bounds__(1024) assemble_kernel(const AsmArgs a) {
    extern __shared__ double sbuf[];
    const int d = 1 << a.logd;
    const int Dp = d + (d >> 4) + 1;
    const int B = 1 << a.logb;
    const int64_t S = a.S;
    for (int64_t grp = blockIdx.x; grp < a.groups; grp += gridDim.x) {
        const int64_t mloc0 = grp * B;  // relative to m_begin
        asm_load(a, sbuf, Dp, mloc0);
        __syncthreads();
        wht_all(sbuf, Dp, a.logd, B);
        // rows of mu as runs of B adjacent complex values
        if (B >= 2) {  // aligned mask pairs -> one 32-byte store per (row, pair)
            const int lp = a.logb - 1;
            for (int e = threadIdx.x; e < (B >> 1) * d; e += blockDim.x) {
                const int mp = e & ((B >> 1) - 1), r = e >> lp;
                const uint32_t m0 = (uint32_t)(a.m_begin + mloc0 + 2 * mp), m1 = m0 + 1;
                const double *b0 = sbuf + (2 * mp) * Dp, *b1 = b0 + Dp;
                const double f01 = b0[padix(r)], f02 = b0[padix(r ^ (int)m0)];
                const double f11 = b1[padix(r)], f12 = b1[padix(r ^ (int)m1)];
                const double2 v0 = make_double2(a.scale_half * (f01 + f02), a.scale_half * (f02 - f01));
                const double2 v1 = make_double2(a.scale_half * (f11 + f12), a.scale_half * (f12 - f11));
                const int64_t c0 = (int64_t)((r ^ m0) & (uint32_t)(S - 1));
                double2 *dst = a.mu + (int64_t)r * S + (c0 & ~(int64_t)1);
                if (c0 & 1) st256_cs(dst, v1, v0);
                else st256_cs(dst, v0, v1);
            }
            __syncthreads();
            continue;
        }
        for (int e = threadIdx.x; e < B * d; e += blockDim.x) {
            const int ml = e & (B - 1), r = e >> a.logb;
            const uint32_t m = (uint32_t)(a.m_begin + mloc0 + ml);
            const double *b = sbuf + ml * Dp;
            const double f1 = b[padix(r)], f2 = b[padix(r ^ (int)m)];
            const int64_t col = (int64_t)((r ^ m) & (uint32_t)(S - 1));
            __stcs(a.mu + (int64_t)r * S + col, make_double2(a.scale_half * (f1 + f2), a.scale_half * (f2 - f1)));
        }
        __syncthreads();
    }
}

// n >= 13: a cluster of two CTAs transforms the aligned mask pair (m0, m0 + 1);
// CTA k writes rows [k d/2, (k+1) d/2) of both masks, reading the partner's
// transform through distributed shared memory -> 32-byte row segments.
template <int NT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1) assemble_pair_kernel(const AsmArgs a) {
    extern __shared__ double sbuf[];
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int d = 1 << a.logd;
    const int Dp = d + (d >> 4) + 1;
    const int64_t S = a.S;
    const double *own = sbuf;
    const double *peer = cluster.map_shared_rank(sbuf, rank ^ 1);
    const double *tr0 = rank == 0 ? own : peer;  // transform of mask m0
    const double *tr1 = rank == 0 ? peer : own;  // transform of mask m0 + 1
    const int64_t ncl = gridDim.x / 2;
    double *dst0 = rank == 0 ? sbuf : cluster.map_shared_rank(sbuf, 0);  // mask m0's buffer
    double *dst1 = rank == 1 ? sbuf : cluster.map_shared_rank(sbuf, 1);  // mask m0 + 1's buffer
    cluster.sync();  // the partner CTA has started before its shared memory is written
    for (int64_t grp = blockIdx.x / 2; grp < a.groups; grp += ncl) {
        const int64_t mloc0 = grp * 2;
        const uint32_t m0 = (uint32_t)(a.m_begin + mloc0);
        if (a.layout == LRE_LAYOUT_NATURAL) {
            // Natural theta of the pair comes in 32-byte runs (the lowest qubit's
            // I, X, Y, Z): I/Z belong to m0 (a_low = 0/1), X/Y to m0 + 1.  CTA k
            // loads the runs of half of the a_high values (8 runs in flight per
            // thread) and stores into both masks' buffers (one via DSMEM).
            const uint32_t mh = m0 >> 1;
            const int half = d >> 2;  // a_high values per CTA
            constexpr int U = 4;
            for (int base = threadIdx.x; base < half; base += U * blockDim.x) {
                double4 q[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int ah = rank * half + base + u * blockDim.x;
                    if (base + u * (int)blockDim.x < half) {
                        const uint64_t run = ma_to_natural(mh, (uint32_t)ah);  // natural index / 4
                        q[u] = ld256_nc(a.theta + 4 * run);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int ah = rank * half + base + u * blockDim.x;
                    if (base + u * (int)blockDim.x < half) {
                        const uint32_t a0 = (uint32_t)ah << 1, a1 = a0 | 1u;
                        const uint32_t m1 = m0 + 1;
                        // I: (m0, a0), Z: (m0, a1), X: (m1, a0), Y: (m1, a1)
                        const double vI = ((__popc(a0 & m0) >> 1) & 1) ? -q[u].x : q[u].x;
                        const double vZ = ((__popc(a1 & m0) >> 1) & 1) ? -q[u].w : q[u].w;
                        const double vX = ((__popc(a0 & m1) >> 1) & 1) ? -q[u].y : q[u].y;
                        const double vY = ((__popc(a1 & m1) >> 1) & 1) ? -q[u].z : q[u].z;
                        dst0[padix((int)a0)] = vI;
                        dst0[padix((int)a1)] = vZ;
                        dst1[padix((int)a0)] = vX;
                        dst1[padix((int)a1)] = vY;
                    }
                }
            }
            cluster.sync();  // both buffers filled (local and remote stores)
        } else {
            asm_load(a, sbuf, Dp, mloc0 + rank);
            __syncthreads();
        }
        wht_all(sbuf, Dp, a.logd, 1);
        cluster.sync();  // both transforms complete
        const uint32_t m1 = m0 + 1;
        for (int r = rank * (d >> 1) + threadIdx.x; r < (rank + 1) * (d >> 1); r += blockDim.x) {
            const double f01 = tr0[padix(r)], f02 = tr0[padix(r ^ (int)m0)];
            const double f11 = tr1[padix(r)], f12 = tr1[padix(r ^ (int)m1)];
            const double2 v0 = make_double2(a.scale_half * (f01 + f02), a.scale_half * (f02 - f01));
            const double2 v1 = make_double2(a.scale_half * (f11 + f12), a.scale_half * (f12 - f11));
            const int64_t c0 = (int64_t)((r ^ m0) & (uint32_t)(S - 1));  // c0 ^ 1 is mask m1's column
            double2 *dst = a.mu + (int64_t)r * S + (c0 & ~(int64_t)1);
            if (c0 & 1) st256_cs(dst, v1, v0);
            else st256_cs(dst, v0, v1);
        }
        cluster_sync_relaxed();  // the partner has finished reading this CTA's transform
    }
}

int assemble_impl(const double *theta, int layout, int n, int64_t m_begin, int64_t m_end, double *mu, cudaStream_t s) {
    const int64_t S = m_end - m_begin;
    const int64_t d = (int64_t)1 << n;
    if (n < 1 || n > 14) return LRE_EUNSUPPORTED;
    if (S <= 0 || (S & (S - 1)) || m_begin % S || m_end > d) return LRE_EINVAL;
    static int num_sms = 0;
    if (!num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int Dp = (int)(d + (d >> 4) + 1);
    // shared-memory budget per CTA (masks per CTA = largest power of two that
    // fits): measured best 40 KB at n <= 11 (several CTAs per SM), 75 KB at
    // n = 12, 150 KB at n = 13 (profiles/README.md); LRE_ASM_BUDGET_KB
    // overrides it for A/B runs
    static const int budget_env = [] {
        const char *v = getenv("LRE_ASM_BUDGET_KB");
        return v ? atoi(v) : 0;
    }();
    const size_t smem_budget = (size_t)(budget_env > 0 ? budget_env : n <= 11 ? 40 : n == 12 ? 75 : 150) * 1024;
    int logb = 0;
    while (logb < 3 && ((int64_t)2 << logb) <= S && (size_t)(2 << logb) * Dp * sizeof(double) <= smem_budget) ++logb;
    AsmArgs a;
    a.theta = theta;
    a.layout = layout;
    a.logd = n;
    a.logb = logb;
    a.m_begin = m_begin;
    a.S = S;
    a.scale_half = 0.5 * pow(2.0, -n / 2.0);
    a.mu = reinterpret_cast<double2 *>(mu);
    const size_t smem = ((size_t)Dp << logb) * sizeof(double);
    const int threads = (int)std::min<int64_t>(1024, std::max<int64_t>(64, (d << logb) / 16));
    cudaError_t e;
    if (logb == 0 && S >= 2) {
        a.cl = 2;
        a.groups = S / 2;
        e = cudaFuncSetAttribute(assemble_pair_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return LRE_ECUDA;
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, assemble_pair_kernel<512>, 512, smem);
        const int64_t grid = 2 * std::min<int64_t>(a.groups, (int64_t)num_sms * std::max(1, per_sm) / 2);
        assemble_pair_kernel<512><<<(unsigned)grid, 512, smem, s>>>(a);
    } else {
        a.cl = 1;
        a.groups = S >> logb;
        e = cudaFuncSetAttribute(assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return LRE_ECUDA;
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, assemble_kernel, threads, smem);
        const int64_t grid = std::min<int64_t>(a.groups, (int64_t)num_sms * std::max(1, per_sm));
        assemble_kernel<<<(unsigned)grid, threads, smem, s>>>(a);
    }
    count_launch();
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

}  // namespace lre
