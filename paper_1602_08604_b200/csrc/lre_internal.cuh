// Internal device helpers shared by the LRE kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdint.h>

#include "../../include/lre_b200.h"

namespace lre {

// ---------------------------------------------------------------------------
// compile-time helpers
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int pow3(int k) { return k <= 0 ? 1 : 3 * pow3(k - 1); }
__host__ __device__ constexpr int popc_c(int x) { return x == 0 ? 0 : (x & 1) + popc_c(x >> 1); }

// global launch counter (bench.py reports it as gpu_launches)
void count_launch(int k = 1);

// multiprocessor count of the current device (grid sizing; cached per device)
int num_sms();

// Philox4x32-10 (counter-based): the record generators key it on (seed) with
// counters (shot, ..., setting), so records do not depend on launch shape.
struct Philox {
    __device__ __forceinline__ static uint4 gen(uint4 c, uint2 k) {
#pragma unroll
        for (int i = 0; i < 10; ++i) {
            const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
            const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
            c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
            k.x += 0x9E3779B9u;
            k.y += 0xBB67AE85u;
        }
        return c;
    }
};


// ---------------------------------------------------------------------------
// count loads: 8 consecutive elements of the counts / intermediate tensor,
// streamed with the evict-first (".cs") policy so they do not displace the
// scattered output lines that L2 is merging.
// ---------------------------------------------------------------------------
template <typename A>
__device__ __forceinline__ void load8(const uint8_t *p, A v[8]) {
    uint2 u = __ldcs(reinterpret_cast<const uint2 *>(p));
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = (A)((u.x >> (8 * i)) & 0xff);
#pragma unroll
    for (int i = 0; i < 4; ++i) v[4 + i] = (A)((u.y >> (8 * i)) & 0xff);
}
template <typename A>
__device__ __forceinline__ void load8(const uint16_t *p, A v[8]) {
    uint4 u = __ldcs(reinterpret_cast<const uint4 *>(p));
    v[0] = (A)(u.x & 0xffff); v[1] = (A)(u.x >> 16);
    v[2] = (A)(u.y & 0xffff); v[3] = (A)(u.y >> 16);
    v[4] = (A)(u.z & 0xffff); v[5] = (A)(u.z >> 16);
    v[6] = (A)(u.w & 0xffff); v[7] = (A)(u.w >> 16);
}
template <typename A>
__device__ __forceinline__ void load8(const int32_t *p, A v[8]) {
    int4 a = __ldcs(reinterpret_cast<const int4 *>(p));
    int4 b = __ldcs(reinterpret_cast<const int4 *>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <typename A>
__device__ __forceinline__ void load8(const int64_t *p, A v[8]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        longlong2 q = __ldcs(reinterpret_cast<const longlong2 *>(p) + i);
        v[2 * i] = (A)q.x;
        v[2 * i + 1] = (A)q.y;
    }
}

// scalar load used by the small (<8 column) tiles
template <typename T> __device__ __forceinline__ int64_t load1(const T *p) { return (int64_t)__ldcs(p); }
template <> __device__ __forceinline__ int64_t load1<uint8_t>(const uint8_t *p) { return (int64_t)*p; }
template <> __device__ __forceinline__ int64_t load1<uint16_t>(const uint16_t *p) {
    return (int64_t)__ldcs(reinterpret_cast<const unsigned short *>(p));
}

// ---------------------------------------------------------------------------
// the per-qubit 6 -> 4 map A (SURVEY §0.1 "separable form"):
//   rows (axis X,Y,Z) x outcome bit -> Pauli digit I,X,Y,Z
//   I = sum of all six, X/Y/Z = (+1 outcome) - (-1 outcome) on that axis.
// ---------------------------------------------------------------------------
template <typename A>
__device__ __forceinline__ void q6to4(A x0, A x1, A y0, A y1, A z0, A z1, A &I, A &X, A &Y, A &Z) {
    I = (x0 + x1) + (y0 + y1) + (z0 + z1);
    X = x0 - x1;
    Y = y0 - y1;
    Z = z0 - z1;
}

// Natural Pauli index i (base-4 digits, qubit 1 most significant) ->
// mask-major index m * 2^n + a with m = X|Y bits and a = Y|Z bits
// (SURVEY §0.1 "symplectic relabel"; reference pauli.py:262-289).
__device__ __forceinline__ uint32_t compact_odd(uint64_t x) {
    // take bits 1,3,5,... of x and pack them
    x = (x >> 1) & 0x5555555555555555ull;
    x = (x | (x >> 1)) & 0x3333333333333333ull;
    x = (x | (x >> 2)) & 0x0f0f0f0f0f0f0f0full;
    x = (x | (x >> 4)) & 0x00ff00ff00ff00ffull;
    x = (x | (x >> 8)) & 0x0000ffff0000ffffull;
    x = (x | (x >> 16)) & 0x00000000ffffffffull;
    return (uint32_t)x;
}
__device__ __forceinline__ uint32_t compact_even(uint64_t x) { return compact_odd(x << 1); }

__device__ __forceinline__ void natural_to_ma(uint64_t i, uint32_t &m, uint32_t &a) {
    uint32_t hi = compact_odd(i);   // digit >= 2  -> Y or Z
    uint32_t lo = compact_even(i);  // digit odd   -> X or Z
    a = hi;
    m = hi ^ lo;                    // X (01) or Y (10)
}

__device__ __forceinline__ uint64_t spread_bits(uint32_t x) {
    uint64_t v = x;
    v = (v | (v << 16)) & 0x0000ffff0000ffffull;
    v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
    v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
    v = (v | (v << 2)) & 0x3333333333333333ull;
    v = (v | (v << 1)) & 0x5555555555555555ull;
    return v;
}
// (m, a) -> natural index: hi bit = a, lo bit = a ^ m
__device__ __forceinline__ uint64_t ma_to_natural(uint32_t m, uint32_t a) {
    return (spread_bits(a) << 1) | spread_bits(a ^ m);
}

// Epilogue factors theta = N * fac[zc], fac[zc] = 2^{-n/2} / shots / 3^zc
// (pipeline.py:138, records.py:62-64) rounded once from the long-double
// quotient: one multiply per output instead of two fp64 divisions (relative
// error <= 2 ulp, the int64 numerators N stay exact).  Every kernel that
// finishes numerators (the last fold pass, lre_finalize) takes the table by
// value and stages it in shared memory (lanes of a warp index different zc;
// divergent constant-bank reads would serialise), so results are bit-identical
// across entry points and the library keeps no per-(n, shots) device state.
struct Factors {
    double f[33];
};
inline Factors make_factors(int n, int64_t shots) {
    Factors fac;
    const long double scale = (long double)pow(2.0, -n / 2.0);
    long double p3 = 1.0L;
    for (int zc = 0; zc < 33; ++zc) {
        fac.f[zc] = (double)(scale / (long double)shots / p3);
        p3 *= 3.0L;
    }
    return fac;
}
// copy the table into shared memory; the caller synchronises before use
__device__ __forceinline__ void stage_factors(double *dst, const Factors &fac) {
    for (int i = threadIdx.x; i < 33; i += blockDim.x) dst[i] = fac.f[i];
}

// ---------------------------------------------------------------------------
// mbarrier / bulk-copy (TMA) helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#ifdef LRE_MBAR_WATCHDOG
    // debug builds: trap (instead of hanging) when a phase never completes
    for (long long it = 0;; ++it) {
        uint32_t ok;
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (it == (1ll << 22)) {
            if ((threadIdx.x & 31) == 0)
                printf("LRE mbarrier watchdog: block %d thread %d bar %p parity %u\n", blockIdx.x, threadIdx.x, bar,
                       parity);
            __trap();
        }
    }
#endif
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LRE_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LRE_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// As mbar_wait, but the waiting threads are suspended (up to `hint_ns` per try) instead of
// spinning: for a producer that waits on a slower consumer, whose warps need the issue slots.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity, uint32_t hint_ns) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LRE_WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra LRE_WAITS_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(hint_ns)
        : "memory");
}
// 1-D bulk copy global -> this CTA's shared memory, completing on `bar`
// (size a multiple of 16 bytes)
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// order this thread's generic-proxy shared-memory accesses before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Mask position of X-mask m in a MASK_MAJOR-family layout (include/lre_b200.h):
// plain MASK_MAJOR is the identity; MASK_CHUNKED(logP, logK) swaps the rank field
// g (top logP bits of m) with the chunk field c (next logK bits), so that chunk c
// of every rank's mask slice is one contiguous block (a reduce-scatter chunk).
__host__ __device__ __forceinline__ uint64_t mask_position(uint64_t m, int n, int layout) {
    if ((layout & 0xff) != 2) return m;
    const int logP = (layout >> 8) & 0xff, logK = (layout >> 16) & 0xff;
    const int logS = n - logP, logJ = logS - logK;
    const uint64_t g = m >> logS, c = (m >> logJ) & ((1ull << logK) - 1), j = m & ((1ull << logJ) - 1);
    return (((c << logP) | g) << logJ) | j;
}
__host__ __device__ __forceinline__ bool layout_is_mask_major(int layout) {
    return layout == LRE_LAYOUT_MASK_MAJOR || (layout & 0xff) == 2;
}

// 3^k as an exact double (k <= 32)
__device__ __forceinline__ double pow3d(int k) {
    double g = 1.0;
    for (int i = 0; i < k; ++i) g *= 3.0;
    return g;
}

}  // namespace lre
