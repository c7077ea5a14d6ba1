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
// n >= 11, mask-major theta: assemble_x8_kernel<LOGD>
//
// The write pattern decides this kernel (profiles/r02_microbench_mu_writes.txt,
// 4.3 GB of XOR-diagonal stores at n = 14): a row segment of 16 B (one mask)
// runs at 0.4-1.1 TB/s, 32 B (a mask pair) at 1.4-3.6 TB/s and 64 B at
// 2.4-4.7 TB/s depending on when the other parts of each 128-byte line are
// written (partial lines evicted early are read-modify-written); only whole
// 128-byte lines (8 consecutive masks per row, written by one thread) hold
// 4.5-4.7 TB/s for any schedule.  One mask's transform is 2^n doubles (128 KB
// at n = 14), so the 8 masks of a line live on the 8 CTAs of a cluster.
//
// SPLIT mode (all but ~3% of the mask blocks): the block's masks m0..m0+7
// share three zero bits b0 < b1 < b2 in [3, n).  Every row r and its partner
// r ^ m then agree on those bits, so the transform splits exactly into eighths:
// for r with (r_b0, r_b1, r_b2) = k,
//     F_m[r] = WHT_{n-3}( G_{m,k} )[r'],   G_{m,k}[a'] = sum_s (-1)^{s.k} w_m[a' with s inserted],
// (r', a' = the index with the three bits removed).  CTA j loads its own mask
// m0 + j (contiguous, mask-major theta) straight into registers, applies the
// sign twist and the 3-bit butterfly, and pushes eighth k to CTA k with
// st.async (distributed shared memory, completing on CTA k's mbarrier).  CTA
// k then holds eighth k of all 8 masks (2^n doubles), transforms them locally
// and writes its 2^(n-3) rows as whole 128-byte lines, reading only its own
// shared memory.  One relaxed cluster barrier per block protects the buffers;
// no release fence waits on the streaming mu stores, and the next block's
// theta loads are in flight (registers) during the write phase.
// FULL mode (blocks with fewer than three common zero bits): CTA j bulk-copies
// its mask, transforms all 2^n coefficients, and the write phase pulls the
// partners' values through distributed shared memory.
// ---------------------------------------------------------------------------
template <int LOGD> struct X8 {
    static constexpr int D = 1 << LOGD;
    static constexpr int NT = D / 32;                  // threads per CTA
    static constexpr int L = LOGD - 3;                 // bits of an eighth
    static constexpr int E = 1 << L;                   // eighth length
    static constexpr int EP = E + E / 16 + 2;          // padded eighth stride (2 per 32; even; shifts banks per mask)
    static constexpr int FULLP = D + D / 32;           // FULL mode: one pad double per 32
    static constexpr int FD = 8 * EP > FULLP ? 8 * EP : FULLP;
    static constexpr size_t STAGE = (size_t)8 * NT * 16;  // next block's second a' pair (cp.async)
    static constexpr size_t SMEM = (size_t)FD * sizeof(double) + STAGE + 16;
};

__device__ __forceinline__ int pad32(int x) { return x + (x >> 5); }
__device__ __forceinline__ int pad2_32(int x) { return x + 2 * (x >> 5); }

// insert bit values (s0, s1, s2) at final positions b0 < b1 < b2
__device__ __forceinline__ uint32_t ins3(uint32_t x, int b0, int b1, int b2, uint32_t s) {
    x = ((x >> b0) << (b0 + 1)) | ((s & 1u) << b0) | (x & ((1u << b0) - 1));
    x = ((x >> b1) << (b1 + 1)) | (((s >> 1) & 1u) << b1) | (x & ((1u << b1) - 1));
    x = ((x >> b2) << (b2 + 1)) | (((s >> 2) & 1u) << b2) | (x & ((1u << b2) - 1));
    return x;
}
__device__ __forceinline__ uint32_t del3(uint32_t x, int b0, int b1, int b2) {
    x = ((x >> (b2 + 1)) << b2) | (x & ((1u << b2) - 1));
    x = ((x >> (b1 + 1)) << b1) | (x & ((1u << b1) - 1));
    x = ((x >> (b0 + 1)) << b0) | (x & ((1u << b0) - 1));
    return x;
}

__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_v2(uint32_t raddr, double x, double y, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "d"(x), "d"(y), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ double2 ld_nc_v2(const double *p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }

#ifdef LRE_X8_PROFILE
// phase timestamps of the first 64 blocks of every CTA (debug builds only):
// [cta][block][phase] with phases 0 top, 1 after wait, 2 pushed, 3 data in, 4 WHT done, 5 write done
__device__ unsigned long long g_x8_prof[148 * 2][64][6];
#define X8_T(ph)                                                                           \
    do {                                                                                   \
        if (t == 0 && it_ < 64) {                                                          \
            unsigned long long now_;                                                       \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now_));                      \
            g_x8_prof[blockIdx.x][it_][ph] = now_;                                         \
        }                                                                                  \
    } while (0)
#else
#define X8_T(ph) \
    do {         \
    } while (0)
#endif

struct X8Args {
    const double *theta;  // mask-major slice: theta[(m - m_begin) * 2^n + a]
    int64_t m_begin;
    int64_t S;            // mu rows are S complex wide: the slab of S masks holding [m_begin, m_begin + 8 units)
    int64_t units;        // masks / 8
    double scale_half;
    double2 *mu;
    int order;            // 0: FULL-mode blocks first, round-robin (n = 14); 1: plain stride
};

// zero bits of m0 in [3, n): SPLIT mode needs three
__device__ __forceinline__ int zero_bits(uint32_t m0, int n) { return __popc(~m0 & (((1u << n) - 1) & ~7u)); }

// The clusters' block schedule at n = 14.  A FULL-mode block (fewer than three
// common zero bits, 3% of the blocks) costs ~2.5x a SPLIT block, and a plain
// stride over u hands one cluster nine of them and another none (u mod 15: the
// slowest cluster ran ~6% over the mean).  So the blocks are dealt out
// round-robin, the FULL-mode blocks first (pass 0) and then the SPLIT blocks
// (pass 1), the dealing position carried across the passes: every cluster gets
// the same number of each kind to within one.
struct X8Units {
    int64_t scan, ph, cid, ncl;
    int pass;
    __device__ __forceinline__ int64_t take(const X8Args &a, int n) {
        if (a.order) {  // plain stride
            const int64_t u = scan ? scan : cid;
            scan = u + ncl;
            return u < a.units ? u : a.units;
        }
        for (; pass < 2; ++pass, scan = 0) {
            for (; scan < a.units; ++scan) {
                if ((zero_bits((uint32_t)(a.m_begin + scan * 8), n) >= 3) != (pass == 1)) continue;
                const bool mine = ph == cid;
                if (++ph == ncl) ph = 0;
                if (mine) return scan++;
            }
        }
        return a.units;
    }
};

// three highest zero bits of m0 in [3, n) (b0 < b1 < b2); false if fewer than three
__device__ __forceinline__ bool split_bits(uint32_t m0, int n, int &b0, int &b1, int &b2) {
    uint32_t z = ~m0 & (((1u << n) - 1) & ~7u);
    if (__popc(z) < 3) return false;
    b2 = 31 - __clz(z);
    z &= ~(1u << b2);
    b1 = 31 - __clz(z);
    z &= ~(1u << b1);
    b0 = 31 - __clz(z);
    return true;
}

// the 8 double2 theta loads of one thread's a' pair q for SPLIT block u (8 split combinations)
template <int LOGD>
__device__ __forceinline__ void x8_load(const X8Args &a, int64_t u, int rank, int t, int q, int b0, int b1, int b2,
                                        double2 (&v)[8]) {
    using C = X8<LOGD>;
    const double *src = a.theta + ((u * 8 + rank) << LOGD) + ins3(2u * (uint32_t)(t + C::NT * q), b0, b1, b2, 0u);
    const uint32_t P0 = 1u << b0, P1 = 1u << b1, P2 = 1u << b2;
#pragma unroll
    for (int sc = 0; sc < 8; ++sc)
        v[sc] = ld_nc_v2(src + ((sc & 1 ? P0 : 0u) | (sc & 2 ? P1 : 0u) | (sc & 4 ? P2 : 0u)));
}

// the same 8 pairs as x8_load, copied asynchronously into this thread's stage slots
template <int LOGD>
__device__ __forceinline__ void x8_stage(const X8Args &a, int64_t u, int rank, int t, int q, int b0, int b1, int b2,
                                         double2 *stg) {
    using C = X8<LOGD>;
    const double *src = a.theta + ((u * 8 + rank) << LOGD) + ins3(2u * (uint32_t)(t + C::NT * q), b0, b1, b2, 0u);
    const uint32_t P0 = 1u << b0, P1 = 1u << b1, P2 = 1u << b2;
#pragma unroll
    for (int sc = 0; sc < 8; ++sc)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(stg + sc * C::NT)),
                     "l"(src + ((sc & 1 ? P0 : 0u) | (sc & 2 ? P1 : 0u) | (sc & 4 ? P2 : 0u)))
                     : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int LOGD>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(X8<LOGD>::NT, LOGD >= 14 ? 1 : LOGD == 13 ? 2 : 4)
    assemble_x8_kernel(const X8Args a) {
    using C = X8<LOGD>;
    constexpr int D = C::D, NT = C::NT, E = C::E, EP = C::EP;
    extern __shared__ __align__(16) double x8_smem[];
    double *F = x8_smem;
    uint64_t *barR = reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(x8_smem + C::FD) + C::STAGE);
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int t = threadIdx.x;
    const int64_t ncl = gridDim.x / 8;
    const uint32_t F_s = smem_u32(F), bar_s = smem_u32(barR);

    if (t == 0) {
        mbar_init(barR, 1);
        fence_mbar_init();
    }
    cluster.sync();  // every CTA's mbarrier is initialised before any remote st.async

    X8Units units{0, 0, (int64_t)blockIdx.x / 8, ncl, 0};
    int64_t u = units.take(a, LOGD), un_next = a.units;
    // the next block's a' pairs are in flight during the write phase: pair 0 in
    // registers, pair 1 in a per-thread shared-memory stage (cp.async, [combination][thread])
    double2 v[8];
    double2 *stg = reinterpret_cast<double2 *>(x8_smem + C::FD) + t;
    int b0 = 0, b1 = 0, b2 = 0;
    bool split = false;
    if (u < a.units) {
        split = split_bits((uint32_t)(a.m_begin + u * 8), LOGD, b0, b1, b2);
        if (split) {
            x8_load<LOGD>(a, u, rank, t, 0, b0, b1, b2, v);
            x8_stage<LOGD>(a, u, rank, t, 1, b0, b1, b2, stg);
        }
    }
    uint32_t parity = 0;
    bool first = true;
    int it_ = 0;
    for (; u < a.units; u = un_next, parity ^= 1, ++it_) {
        un_next = units.take(a, LOGD);
        const uint32_t m0 = (uint32_t)(a.m_begin + u * 8);
        const int64_t smask = a.S - 1;
        X8_T(0);
        if (!first) cluster_wait();  // every CTA has finished reading its buffer for the previous block
        first = false;
        X8_T(1);
        if (split) {
            // ---- push: twist + 3-bit butterfly of this CTA's mask, eighth k -> CTA k ----
            if (t == 0) mbar_expect_tx(barR, (uint32_t)D * sizeof(double));
            const uint32_t mj = m0 + (uint32_t)rank;
            double2 v1[8];
            asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
            for (int sc = 0; sc < 8; ++sc) v1[sc] = stg[sc * NT];
            // g[q][e][k]: a' = ap_q + e (ap_q = 2 (t + NT q): q selects the top bit L-1 of a', e bit 0)
            double g[2][2][8];
#pragma unroll
            for (int sc = 0; sc < 8; ++sc) {
                g[0][0][sc] = v[sc].x;
                g[0][1][sc] = v[sc].y;
                g[1][0][sc] = v1[sc].x;
                g[1][1][sc] = v1[sc].y;
            }
            // 3-bit butterfly over the split bits (sc -> eighth k)
#pragma unroll
            for (int h = 1; h < 8; h <<= 1)
#pragma unroll
                for (int sc = 0; sc < 8; ++sc)
                    if (!(sc & h)) {
#pragma unroll
                        for (int q = 0; q < 2; ++q)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const double x = g[q][e][sc], y = g[q][e][sc + h];
                                g[q][e][sc] = x + y;
                                g[q][e][sc + h] = x - y;
                            }
                    }
            // sign twist (-1)^floor(pc(a & m)/2): the split bits are zero in m, so it is one
            // sign per a' for all eight combinations (applied after the linear butterfly)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int pc = __popc(ins3(2u * (uint32_t)(t + NT * q), b0, b1, b2, 0u) & mj);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const uint64_t neg = (uint64_t)(((pc + (e ? (int)(mj & 1u) : 0)) >> 1) & 1) << 63;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        g[q][e][k] = __longlong_as_double(__double_as_longlong(g[q][e][k]) ^ (long long)neg);
                }
            }
            // the WHT stages of a' bits 0 (e) and L-1 (q) are in registers already
#pragma unroll
            for (int k = 0; k < 8; ++k) {
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const double x = g[q][0][k], y = g[q][1][k];
                    g[q][0][k] = x + y;
                    g[q][1][k] = x - y;
                }
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const double x = g[0][e][k], y = g[1][e][k];
                    g[0][e][k] = x + y;
                    g[1][e][k] = x - y;
                }
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint32_t off = (uint32_t)(rank * EP + pad2_32(2 * (t + NT * q))) * sizeof(double);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    st_async_v2(mapa_u32(F_s + off, k), g[q][0][k], g[q][1][k], mapa_u32(bar_s, k));
            }
            X8_T(2);
            mbar_wait(barR, parity);
            X8_T(3);
            // ---- WHT over a' bits 1 .. L-2 of the 8 eighths (this CTA's k = rank) ----
            {  // bits 1..4: 32 consecutive elements per thread (16-byte accesses, conflict-free)
                const int arr = t / (E / 32), blk = t % (E / 32);
                double2 *b = reinterpret_cast<double2 *>(F + arr * EP + 34 * blk);
                double w[32];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const double2 x = b[i];
                    w[2 * i] = x.x;
                    w[2 * i + 1] = x.y;
                }
#pragma unroll
                for (int h = 2; h < 32; h <<= 1)
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (!(i & h)) {
                            const double x = w[i], y = w[i + h];
                            w[i] = x + y;
                            w[i + h] = x - y;
                        }
#pragma unroll
                for (int i = 0; i < 16; ++i) b[i] = make_double2(w[2 * i], w[2 * i + 1]);
            }
            __syncthreads();
            {  // bits 5 .. L-2 (hi = bit L-1 was done by the producers)
                constexpr int K = 1 << (C::L - 6);
                constexpr int ITEMS = 8 * E / K;
#pragma unroll 1
                for (int it = t; it < ITEMS; it += NT) {
                    const int arr = it / (E / K), rest = it % (E / K);
                    const int lo = rest & 31, hi = rest >> 5;
                    double *b = F + arr * EP + lo + 34 * K * hi;
                    double w[K];
#pragma unroll
                    for (int i = 0; i < K; ++i) w[i] = b[34 * i];
#pragma unroll
                    for (int h = 1; h < K; h <<= 1)
#pragma unroll
                        for (int i = 0; i < K; ++i)
                            if (!(i & h)) {
                                const double x = w[i], y = w[i + h];
                                w[i] = x + y;
                                w[i + h] = x - y;
                            }
#pragma unroll
                    for (int i = 0; i < K; ++i) b[34 * i] = w[i];
                }
            }
            __syncthreads();
            X8_T(4);
            // ---- next block's theta into registers (in flight during the write phase) ----
            const int cb0 = b0, cb1 = b1, cb2 = b2;
            const int64_t un = un_next;
            bool nsplit = false;
            if (un < a.units) {
                nsplit = split_bits((uint32_t)(a.m_begin + un * 8), LOGD, b0, b1, b2);
                if (nsplit) {
                    x8_load<LOGD>(a, un, rank, t, 0, b0, b1, b2, v);
                    x8_stage<LOGD>(a, un, rank, t, 1, b0, b1, b2, stg);
                }
            }
            // ---- write phase: rows with split bits = rank, whole 128-byte lines ----
            const uint32_t m0c = del3(m0, cb0, cb1, cb2);
            const uint32_t rpat = ins3(0u, cb0, cb1, cb2, (uint32_t)rank);
            // a warp writes 8 rows per step, 4 lanes per row: lane (rr, w) stores the
            // 32-byte slot pair w of row rr, so every store instruction covers 8 whole
            // 128-byte lines (the L1 processes 8 lines, not 32 partial ones)
            const int lane = t & 31, warp = t >> 5;
            const int rr = lane >> 2, w = lane & 3;
            // slot s of row r holds mask (r & 7) ^ s.  The lane's slots are 2w, 2w+1; it
            // loads slot sa = 2w + (w & 1) first so that each load instruction mixes
            // odd and even slots: the partner-row loads F_j[rp ^ m0c ^ j] (index
            // (8 g8 ^ m0c) | s) then fall on all 16 bank pairs, 2 wavefronts per
            // instruction instead of 4 (all four loads are conflict-free).
            const int sa = 2 * w + (w & 1), sb = sa ^ 1;
            const int ja = rr ^ sa, jb = rr ^ sb;
            const bool swp = w & 1;  // slot 2w holds the sb value
            const double *Aa = F + ja * EP, *Ab = F + jb * EP;
#pragma unroll 4
            for (int g8 = warp; g8 < E / 8; g8 += NT / 32) {
                const int rp = 8 * g8 + rr;
                const uint32_t r = ins3((uint32_t)rp, cb0, cb1, cb2, 0u) | rpat;
                const double f1a = Aa[pad2_32(rp)], f2a = Aa[pad2_32(rp ^ (int)(m0c + ja))];
                const double f1b = Ab[pad2_32(rp)], f2b = Ab[pad2_32(rp ^ (int)(m0c + jb))];
                const double2 oa = make_double2(a.scale_half * (f1a + f2a), a.scale_half * (f2a - f1a));
                const double2 ob = make_double2(a.scale_half * (f1b + f2b), a.scale_half * (f2b - f1b));
                double2 *dst = a.mu + (int64_t)r * a.S + ((int64_t)(r ^ m0) & smask & ~(int64_t)7) + 2 * w;
                st256_cs(dst, swp ? ob : oa, swp ? oa : ob);
            }
            split = nsplit;
        } else {
            // ---- FULL mode: this CTA transforms its whole mask; partners pull ----
            if (t == 0) {
                fence_proxy_async_smem();
                mbar_expect_tx(barR, (uint32_t)D * sizeof(double));
                const double *src = a.theta + ((u * 8 + rank) << LOGD);
                constexpr uint32_t CH = 16384;
#pragma unroll 1
                for (uint32_t off = 0; off < (uint32_t)D * sizeof(double); off += CH)
                    bulk_load(reinterpret_cast<char *>(F) + off, reinterpret_cast<const char *>(src) + off, CH, barR);
            }
            mbar_wait(barR, parity);
            const uint32_t m = m0 + (uint32_t)rank;
            {  // bits 5..9 with the sign twist; read all (linear), then write padded
                const int g = t >> 5, l = t & 31;  // NT = D / 32 threads = one (group, lane) each
                const int base = g * 1024 + l;
                double w[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const uint32_t av = (uint32_t)(base + 32 * j);
                    const double x = F[base + 32 * j];
                    w[j] = ((__popc(av & m) >> 1) & 1) ? -x : x;
                }
#pragma unroll
                for (int h = 1; h < 32; h <<= 1)
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (!(j & h)) {
                            const double x = w[j], y = w[j + h];
                            w[j] = x + y;
                            w[j + h] = x - y;
                        }
                __syncthreads();
#pragma unroll
                for (int j = 0; j < 32; ++j) F[pad32(base + 32 * j)] = w[j];
            }
            __syncthreads();
            {  // bits 0..4
                double *b = F + 33 * t;
                double w[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) w[i] = b[i];
#pragma unroll
                for (int h = 1; h < 32; h <<= 1)
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (!(i & h)) {
                            const double x = w[i], y = w[i + h];
                            w[i] = x + y;
                            w[i + h] = x - y;
                        }
#pragma unroll
                for (int i = 0; i < 32; ++i) b[i] = w[i];
            }
            if constexpr (LOGD > 10) {  // bits 10..n-1
                __syncthreads();
                constexpr int K = 1 << (LOGD - 10);
#pragma unroll 1
                for (int bse = t; bse < 1024; bse += NT) {
                    double w[K];
#pragma unroll
                    for (int j = 0; j < K; ++j) w[j] = F[pad32(bse + 1024 * j)];
#pragma unroll
                    for (int h = 1; h < K; h <<= 1)
#pragma unroll
                        for (int j = 0; j < K; ++j)
                            if (!(j & h)) {
                                const double x = w[j], y = w[j + h];
                                w[j] = x + y;
                                w[j + h] = x - y;
                            }
#pragma unroll
                    for (int j = 0; j < K; ++j) F[pad32(bse + 1024 * j)] = w[j];
                }
            }
            cluster.sync();  // the 8 transforms are complete and visible to the partners
            // rows [rank d/8, (rank+1) d/8): partners' values through distributed shared memory
#pragma unroll 1
            for (int q = 0; q < 4; ++q) {
                const int r = rank * (D / 8) + t + NT * q;
                double2 *dst = a.mu + (int64_t)r * a.S + ((int64_t)((uint32_t)r ^ m0) & smask & ~(int64_t)7);
                const int rho = r & 7;
#pragma unroll
                for (int J = 0; J < 4; ++J) {
                    const double *A0 = cluster.map_shared_rank(F, 2 * J), *A1 = cluster.map_shared_rank(F, 2 * J + 1);
                    const double f1a = A0[pad32(r)], f2a = A0[pad32(r ^ (int)(m0 + 2 * J))];
                    const double f1b = A1[pad32(r)], f2b = A1[pad32(r ^ (int)(m0 + 2 * J + 1))];
                    const double2 oa = make_double2(a.scale_half * (f1a + f2a), a.scale_half * (f2a - f1a));
                    const double2 ob = make_double2(a.scale_half * (f1b + f2b), a.scale_half * (f2b - f1b));
                    const bool sw = rho & 1;
                    st256_cs(dst + 2 * ((rho >> 1) ^ J), sw ? ob : oa, sw ? oa : ob);
                }
            }
            const int64_t un = un_next;
            if (un < a.units) {
                split = split_bits((uint32_t)(a.m_begin + un * 8), LOGD, b0, b1, b2);
                if (split) {
                    x8_load<LOGD>(a, un, rank, t, 0, b0, b1, b2, v);
                    x8_stage<LOGD>(a, un, rank, t, 1, b0, b1, b2, stg);
                }
            }
        }
        X8_T(5);
        cluster_arrive_relaxed();  // this CTA is done reading its own buffer (and, FULL mode, the partners')
    }
    if (!first) cluster_wait();  // partners may still read this CTA's shared memory (FULL mode)
}

template <typename K>
static int launch_cluster8(K kern, int nt, size_t smem, const X8Args &a, cudaStream_t s) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return LRE_ECUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(8, 1, 1);
    cfg.blockDim = dim3(nt, 1, 1);
    cfg.dynamicSmemBytes = smem;
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
    kern<<<(unsigned)(8 * clusters), nt, smem, s>>>(a);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
}

template <int LOGD>
static int launch_x8(const double *theta, int64_t m_begin, int64_t masks, int64_t S, double *mu, cudaStream_t s) {
    // FULL-first round-robin at n = 14 only: at n <= 13 blocks are cheap next to the
    // serial scan of take() and the synchronised FULL start (n = 13 / 12 / 11
    // measured 6 / 25 / 50% slower than the stride, n = 14 2.6% faster:
    // profiles/r02d_assembly_experiments.txt).  LRE_X8_ORDER=stride|rr overrides (A/B).
    static const int forced = [] {
        const char *v = getenv("LRE_X8_ORDER");
        return !v ? -1 : !strcmp(v, "stride") ? 1 : !strcmp(v, "rr") ? 0 : -1;
    }();
    const int order = forced >= 0 ? forced : LOGD >= 14 ? 0 : 1;
    X8Args a;
    a.theta = theta;
    a.m_begin = m_begin;
    a.S = S;
    a.units = masks / 8;
    a.scale_half = 0.5 * pow(2.0, -LOGD / 2.0);
    a.mu = reinterpret_cast<double2 *>(mu);
    a.order = order;
    return launch_cluster8(assemble_x8_kernel<LOGD>, X8<LOGD>::NT, X8<LOGD>::SMEM, a, s);
}

// the cluster kernel applies to mask-major slices of >= 8 masks at n >= 11
// (LRE_ASM=legacy selects the round-1 kernels for A/B runs)
static bool use_cl8(int layout, int n, int64_t S) {
    static const bool legacy = [] {
        const char *v = getenv("LRE_ASM");
        return v && !strcmp(v, "legacy");
    }();
    return !legacy && layout == LRE_LAYOUT_MASK_MAJOR && n >= 11 && n <= 14 && S >= 8;
}

static int launch_cl8_n(int n, const double *theta, int64_t m_begin, int64_t masks, int64_t S, double *mu,
                        cudaStream_t s) {
    switch (n) {
    case 11: return launch_x8<11>(theta, m_begin, masks, S, mu, s);
    case 12: return launch_x8<12>(theta, m_begin, masks, S, mu, s);
    case 13: return launch_x8<13>(theta, m_begin, masks, S, mu, s);
    case 14: return launch_x8<14>(theta, m_begin, masks, S, mu, s);
    default: return LRE_EUNSUPPORTED;
    }
}

int assemble_impl(const double *theta, int layout, int n, int64_t m_begin, int64_t m_end, double *mu, cudaStream_t s);

// masks [m_begin, m_end) (mask-major slice) written into the column slab of the
// masks [slab_begin, slab_begin + slab_masks): mu_slab[r * slab_masks + c] =
// mu[r, ((r / slab_masks) ^ (slab_begin / slab_masks)) * slab_masks + c] —
// one chunk of a rank's slice assembled as soon as its reduce-scatter chunk lands
#ifdef LRE_X8_PROFILE
extern "C" int lre_x8_profile_dump(void *host, size_t bytes) {
    return cudaMemcpyFromSymbol(host, g_x8_prof, bytes < sizeof(g_x8_prof) ? bytes : sizeof(g_x8_prof)) == cudaSuccess
               ? 0
               : 2;
}
#endif

int assemble_slab_impl(const double *theta, int n, int64_t m_begin, int64_t m_end, int64_t slab_begin,
                       int64_t slab_masks, double *mu, cudaStream_t s) {
    const int64_t masks = m_end - m_begin;
    const int64_t d = (int64_t)1 << n;
    if (slab_masks <= 0 || (slab_masks & (slab_masks - 1)) || slab_begin % slab_masks || slab_begin + slab_masks > d)
        return LRE_EINVAL;
    if (masks <= 0 || (masks & (masks - 1)) || m_begin % masks || m_begin < slab_begin ||
        m_end > slab_begin + slab_masks)
        return LRE_EINVAL;
    if (masks == slab_masks) return assemble_impl(theta, LRE_LAYOUT_MASK_MAJOR, n, m_begin, m_end, mu, s);
    if (!use_cl8(LRE_LAYOUT_MASK_MAJOR, n, masks)) return LRE_EUNSUPPORTED;
    return launch_cl8_n(n, theta, m_begin, masks, slab_masks, mu, s);
}

int assemble_impl(const double *theta, int layout, int n, int64_t m_begin, int64_t m_end, double *mu, cudaStream_t s) {
    const int64_t S = m_end - m_begin;
    const int64_t d = (int64_t)1 << n;
    if (n < 1 || n > 14) return LRE_EUNSUPPORTED;
    if (S <= 0 || (S & (S - 1)) || m_begin % S || m_end > d) return LRE_EINVAL;
    if (use_cl8(layout, n, S)) return launch_cl8_n(n, theta, m_begin, S, S, mu, s);
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
