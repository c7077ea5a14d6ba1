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

// ---------------------------------------------------------------------------
// n >= 11, mask-major theta: assemble_cl8_kernel<LOGD>
//
// The write pattern decides this kernel (profiles/r02_microbench_mu_writes.txt,
// 4.3 GB of XOR-diagonal stores at n = 14): a row segment of 16 B (one mask)
// runs at 1.1 TB/s, 32 B (a mask pair) at 2.9-3.6 TB/s and 64 B at 2.9-4.7
// TB/s depending on whether the CTAs writing the two halves of a 128-byte line
// happen to be in step; only whole 128-byte lines (8 consecutive masks per
// row) hold 4.6 TB/s for any schedule.  One mask's transform is 2^n doubles
// (128 KB at n = 14), so 8 masks cannot share one SM:
//   * a cluster of 8 CTAs owns an aligned block of 8 masks, CTA j the
//     transform of mask m0 + j, in its own shared memory;
//   * theta arrives mask-major (each mask's 2^n coefficients contiguous) by
//     bulk copies (cp.async.bulk, mbarrier completion): the first half of the
//     next mask is prefetched into a staging buffer while the current mask is
//     written out, the second half lands in the transform buffer as soon as
//     the partners have finished reading it;
//   * the fp64 WHT runs in three shared-memory rounds (bits 5-9 with the sign
//     twist, bits 0-4, bits 10..n-1), one pad double per 32 (conflict-free);
//   * after one cluster barrier CTA c writes rows [c d/8, (c+1) d/8): per row
//     16 transform values (two per mask, 14 of them read from the partners
//     through distributed shared memory) -> one 128-byte segment.
// ---------------------------------------------------------------------------
template <int LOGD> struct Cl8 {
    static constexpr int D = 1 << LOGD;
    static constexpr int NT = D / 32;     // threads per CTA
    static constexpr int FP = D + D / 32; // padded transform (doubles)
    static constexpr int HALF = D / 2;    // prefetched first half (doubles)
    static constexpr int FH = HALF + HALF / 32;  // linear landing offset of the second half inside F
    static constexpr size_t SMEM = (size_t)(FP + HALF) * sizeof(double) + 2 * sizeof(uint64_t);
    static constexpr uint32_t HALF_BYTES = (uint32_t)HALF * sizeof(double);
};

__device__ __forceinline__ int pad32(int x) { return x + (x >> 5); }

struct Cl8Args {
    const double *theta;  // mask-major slice: theta[(m - m_begin) * 2^n + a]
    int64_t m_begin;
    int64_t S;            // masks in the slice (power of two >= 8); mu rows are S complex wide
    int64_t units;        // S / 8
    double scale_half;
    double2 *mu;
};

template <int LOGD>
__device__ __forceinline__ void cl8_issue_half(const Cl8Args &a, int64_t u, int rank, int half, double *dst,
                                               uint64_t *bar) {
    using C = Cl8<LOGD>;
    const double *src = a.theta + ((u * 8 + rank) << LOGD) + (int64_t)half * C::HALF;
    constexpr uint32_t CHUNK = C::HALF_BYTES < 16384u ? C::HALF_BYTES : 16384u;
    mbar_expect_tx(bar, C::HALF_BYTES);
#pragma unroll 1
    for (uint32_t off = 0; off < C::HALF_BYTES; off += CHUNK)
        bulk_load(reinterpret_cast<char *>(dst) + off, reinterpret_cast<const char *>(src) + off, CHUNK, bar);
}

template <int LOGD>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(Cl8<LOGD>::NT, LOGD >= 14 ? 1 : LOGD == 13 ? 2 : 4) assemble_cl8_kernel(const Cl8Args a) {
    using C = Cl8<LOGD>;
    constexpr int D = C::D, NT = C::NT;
    extern __shared__ __align__(16) double cl8_smem[];
    double *F = cl8_smem;
    double *Sbuf = cl8_smem + C::FP;
    uint64_t *bars = reinterpret_cast<uint64_t *>(Sbuf + C::HALF);
    uint64_t *barS = bars, *barF = bars + 1;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int t = threadIdx.x;
    const int64_t ncl = gridDim.x / 8;
    const int64_t u0 = blockIdx.x / 8;
    if (t == 0) {
        mbar_init(barS, 1);
        mbar_init(barF, 1);
        fence_mbar_init();
        if (u0 < a.units) {
            cl8_issue_half<LOGD>(a, u0, rank, 0, Sbuf, barS);
            cl8_issue_half<LOGD>(a, u0, rank, 1, F + C::FH, barF);
        }
    }
    __syncthreads();
    uint32_t parity = 0;
    for (int64_t u = u0; u < a.units; u += ncl, parity ^= 1) {
        const uint32_t m = (uint32_t)(a.m_begin + u * 8 + rank);  // this CTA's mask
        // ---- round A: bits 5..9 (+ sign twist), read linear, write padded ----
        {
            const int g = t >> 5, l = t & 31;
            const int base = g * 1024 + l;
            const double *src = base < C::HALF ? Sbuf + base : F + C::FH + (base - C::HALF);
            double v[32];
            mbar_wait(base < C::HALF ? barS : barF, parity);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const uint32_t av = (uint32_t)(base + 32 * j);
                const double x = src[32 * j];
                v[j] = ((__popc(av & m) >> 1) & 1) ? -x : x;
            }
#pragma unroll
            for (int h = 1; h < 32; h <<= 1)
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (!(j & h)) {
                        const double x = v[j], y = v[j + h];
                        v[j] = x + y;
                        v[j + h] = x - y;
                    }
            __syncthreads();  // every read of the second half (landed inside F) precedes the padded writes
#pragma unroll
            for (int j = 0; j < 32; ++j) F[pad32(base + 32 * j)] = v[j];
        }
        __syncthreads();
        // the staging buffer is consumed: prefetch the first half of the next mask
        if (t == 0 && u + ncl < a.units) {
            fence_proxy_async_smem();
            cl8_issue_half<LOGD>(a, u + ncl, rank, 0, Sbuf, barS);
        }
        // ---- round B: bits 0..4 (32 consecutive elements per thread) ----
        {
            double *b = F + 33 * t;
            double v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = b[i];
#pragma unroll
            for (int h = 1; h < 32; h <<= 1)
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (!(i & h)) {
                        const double x = v[i], y = v[i + h];
                        v[i] = x + y;
                        v[i + h] = x - y;
                    }
#pragma unroll
            for (int i = 0; i < 32; ++i) b[i] = v[i];
        }
        __syncthreads();
        // ---- round C: bits 10..LOGD-1 ----
        if constexpr (LOGD > 10) {
            constexpr int K = 1 << (LOGD - 10);
#pragma unroll 1
            for (int bse = t; bse < 1024; bse += NT) {
                double v[K];
#pragma unroll
                for (int j = 0; j < K; ++j) v[j] = F[pad32(bse + 1024 * j)];
#pragma unroll
                for (int h = 1; h < K; h <<= 1)
#pragma unroll
                    for (int j = 0; j < K; ++j)
                        if (!(j & h)) {
                            const double x = v[j], y = v[j + h];
                            v[j] = x + y;
                            v[j + h] = x - y;
                        }
#pragma unroll
                for (int j = 0; j < K; ++j) F[pad32(bse + 1024 * j)] = v[j];
            }
        }
        // ---- all 8 transforms of the cluster complete and visible ----
        cluster.sync();
        // ---- write phase: rows [rank d/8, (rank+1) d/8), one 128-byte segment each ----
        {
            const uint32_t m0 = (uint32_t)(a.m_begin + u * 8);
            const int64_t smask = a.S - 1;
#pragma unroll 1
            for (int k = 0; k < 4; k += 2) {
                // loads: mask j uniform across the warp, lanes on consecutive rows -> each
                // warp access reads one partner's shared memory contiguously
                double2 o[2][8];  // [row][mask j]: mu[r, r ^ (m0 + j)]
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const double *Fj = cluster.map_shared_rank(F, j);
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int r = rank * (D / 8) + t + NT * (k + q);
                        const double f1 = Fj[pad32(r)], f2 = Fj[pad32(r ^ (int)(m0 + j))];
                        o[q][j] = make_double2(a.scale_half * (f1 + f2), a.scale_half * (f2 - f1));
                    }
                }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int r = rank * (D / 8) + t + NT * (k + q);
                    // column slot of mask j is (r & 7) ^ j: permute the register array by
                    // XOR with r & 7 (three conditional swap stages)
#pragma unroll
                    for (int b = 0; b < 3; ++b) {
                        const bool sw = (r >> b) & 1;
#pragma unroll
                        for (int x = 0; x < 8; ++x)
                            if (!(x & (1 << b))) {
                                const double2 lo = o[q][x], hi = o[q][x | (1 << b)];
                                o[q][x] = sw ? hi : lo;
                                o[q][x | (1 << b)] = sw ? lo : hi;
                            }
                    }
                    const int64_t cb = (int64_t)((uint32_t)r ^ m0) & smask & ~(int64_t)7;
                    double2 *dst = a.mu + (int64_t)r * a.S + cb;
#pragma unroll
                    for (int w = 0; w < 4; ++w) st256_cs(dst + 2 * w, o[q][2 * w], o[q][2 * w + 1]);
                }
            }
        }
        // partners have finished reading this CTA's transform (their loads were consumed by stores)
        cluster_sync_relaxed();
        if (t == 0 && u + ncl < a.units) {
            fence_proxy_async_smem();
            cl8_issue_half<LOGD>(a, u + ncl, rank, 1, F + C::FH, barF);
        }
    }
}

template <int LOGD>
static int launch_cl8(const double *theta, int64_t m_begin, int64_t S, double *mu, cudaStream_t s) {
    using C = Cl8<LOGD>;
    auto kern = assemble_cl8_kernel<LOGD>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) != cudaSuccess)
        return LRE_ECUDA;
    Cl8Args a;
    a.theta = theta;
    a.m_begin = m_begin;
    a.S = S;
    a.units = S / 8;
    a.scale_half = 0.5 * pow(2.0, -LOGD / 2.0);
    a.mu = reinterpret_cast<double2 *>(mu);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(8, 1, 1);
    cfg.blockDim = dim3(C::NT, 1, 1);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 8;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int max_clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, (void *)kern, &cfg) != cudaSuccess || max_clusters < 1)
        max_clusters = std::max(1, num_sms() / 8);
    const int64_t clusters = std::min<int64_t>(a.units, max_clusters);
    kern<<<(unsigned)(8 * clusters), C::NT, C::SMEM, s>>>(a);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

// the cluster kernel applies to mask-major slices of >= 8 masks at n >= 11 (one
// round-A group of 1024 coefficients must lie inside one half of a mask)
// (LRE_ASM=legacy selects the round-1 kernels for A/B runs)
static bool use_cl8(int layout, int n, int64_t S) {
    static const bool legacy = [] {
        const char *v = getenv("LRE_ASM");
        return v && !strcmp(v, "legacy");
    }();
    return !legacy && layout == LRE_LAYOUT_MASK_MAJOR && n >= 11 && n <= 14 && S >= 8;
}

static int launch_cl8_n(int n, const double *theta, int64_t m_begin, int64_t S, double *mu, cudaStream_t s) {
    switch (n) {
    case 11: return launch_cl8<11>(theta, m_begin, S, mu, s);
    case 12: return launch_cl8<12>(theta, m_begin, S, mu, s);
    case 13: return launch_cl8<13>(theta, m_begin, S, mu, s);
    case 14: return launch_cl8<14>(theta, m_begin, S, mu, s);
    default: return LRE_EUNSUPPORTED;
    }
}

int assemble_impl(const double *theta, int layout, int n, int64_t m_begin, int64_t m_end, double *mu, cudaStream_t s) {
    const int64_t S = m_end - m_begin;
    const int64_t d = (int64_t)1 << n;
    if (n < 1 || n > 14) return LRE_EUNSUPPORTED;
    if (S <= 0 || (S & (S - 1)) || m_begin % S || m_end > d) return LRE_EINVAL;
    if (use_cl8(layout, n, S)) return launch_cl8_n(n, theta, m_begin, S, mu, s);
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
        const int64_t grid = 2 * std::min<int64_t>(a.groups, (int64_t)num_sms() * std::max(1, per_sm) / 2);
        assemble_pair_kernel<512><<<(unsigned)grid, 512, smem, s>>>(a);
    } else {
        a.cl = 1;
        a.groups = S >> logb;
        e = cudaFuncSetAttribute(assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return LRE_ECUDA;
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, assemble_kernel, threads, smem);
        const int64_t grid = std::min<int64_t>(a.groups, (int64_t)num_sms() * std::max(1, per_sm));
        assemble_kernel<<<(unsigned)grid, threads, smem, s>>>(a);
    }
    count_launch();
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

}  // namespace lre
