// Step (i) of the LRE hot path on B200: counts (3^n x 2^n) -> theta (4^n).
//
// Reference: pipeline.py:116-138 (step_one_least_squares), _kernels.py:34-56
// (accumulate_fast: per-setting WHT + scatter), pauli.py:153-209 (support
// locations, Gram diagonal).
//
// Step (i) is the tensor map A^{(x)n} applied to the 6^n count tensor
// (SURVEY §0.1 "separable form"): per qubit, the setting digit (X/Y/Z) and
// the outcome bit (+1/-1) of that qubit map to one Pauli digit I/X/Y/Z.
// The map is evaluated in passes, each consuming the lowest-stride qubits of
// its input:
//
//   pass 1  (tile_pass_kernel)  counts -> Y1[aH][c][4^Q1]   Q1 = 6 or 7
//           one tile = 3^Q1 rows x 2^Q1 contiguous columns; its 4^Q1 exact
//           int32 outputs are written contiguously ("tile-major"), so every
//           store is a coalesced 128-byte line.
//   pass k  (vfold_kernel)      X[a][col][V] -> Y[A][B][4^Q][V]   Q <= 3
//           lanes own consecutive elements of the contiguous V axis (the
//           Pauli digits already produced), each thread transforms Q more
//           qubits in registers; reads and writes are 128-byte lines.
//
// All arithmetic is exact integer arithmetic (int16x2 packed, int32, int64);
// the only rounding is the final fp64 epilogue theta = N / shots * 2^{-n/2} /
// 3^{zc} (pipeline.py:138, records.py:64).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "lre_internal.cuh"

namespace lre {

#include "lre_y1rank.inc"
// split Y1 high-part rows: the 1156 used positions padded to a multiple of 32 lanes
static constexpr int LRE_Y1_HROW = 1184;

// ===========================================================================
// epilogue shared by both kernels
// ===========================================================================
enum { OUT_INTER = 0, OUT_THETA = 1, OUT_NUM = 2 };

struct Final {
    void *out;
    int kind;    // OUT_INTER / OUT_THETA / OUT_NUM
    int layout;  // LRE_LAYOUT_* (final outputs only)
    int n;
    int64_t shots;
    Factors fac;  // theta = N * fac[zc] (lre_internal.cuh), staged in shared memory by the final kernels
};

// store a finished fp64 numerator (frequency sources: theta = N * fac[zc], fac from shots = 1)
__device__ __forceinline__ void store_final(const Final &f, const double *sfac, uint64_t nat, double v) {
    uint64_t pos = nat;
    if (layout_is_mask_major(f.layout)) {
        uint32_t m, a;
        natural_to_ma(nat, m, a);
        pos = (mask_position(m, f.n, f.layout) << f.n) | a;
    }
    const int zc = f.n - __popcll((nat | (nat >> 1)) & 0x5555555555555555ull);
    reinterpret_cast<double *>(f.out)[pos] = v * sfac[zc];
}

// store a finished numerator at natural Pauli index `nat`; sfac = the staged fac table
__device__ __forceinline__ void store_final(const Final &f, const double *sfac, uint64_t nat, int64_t v) {
    uint64_t pos = nat;
    if (layout_is_mask_major(f.layout)) {
        uint32_t m, a;
        natural_to_ma(nat, m, a);
        pos = (mask_position(m, f.n, f.layout) << f.n) | a;
    }
    if (f.kind == OUT_NUM) {
        reinterpret_cast<int64_t *>(f.out)[pos] = v;
    } else {
        // zc = number of I (zero) base-4 digits of the natural index
        const int zc = f.n - __popcll((nat | (nat >> 1)) & 0x5555555555555555ull);
        reinterpret_cast<double *>(f.out)[pos] = (double)v * sfac[zc];
    }
}

// ===========================================================================
// pass 1: tile kernel
// ===========================================================================
// A tile of Q = 6 qubits is processed in two levels of three qubits:
//   L1 (warps 0-6): item (rb, g) = 27 consecutive rows x 8 contiguous
//       columns; three qubits reduced in registers -> 64 values, staged.
//   L2 (warps 7-8): one thread per staged value index `dlo`: the 27 x 8
//       staged values of the tile -> three more qubits -> 64 values per
//       thread, written as coalesced lines.
// L1 of sub-tile s overlaps L2 of sub-tile s-1 (double-buffered staging, one
// __syncthreads per sub-tile).  A Q = 7 tile is six Q = 6 sub-tiles (its top
// setting digit r1 x top outcome bit b1) combined by the L2 threads.
//
// SMALL mode (shots <= 1213): L1 keeps two outcomes per 32-bit word
// (w = lo + 65536*hi, exact mod 2^32) so each add works on two counts; the
// staged values fit int16 (|v| <= 27*shots).
constexpr int P1_L1_WARPS = 7;  // 216 L1 items per sub-tile
constexpr int P1_L2_WARPS = 2;  // 64 staged columns
constexpr int P1_THREADS = 32 * (P1_L1_WARPS + P1_L2_WARPS);
constexpr int P1_ITEMS = 216;
constexpr int SMALL_MAX_SHOTS = 1213;  // 27 * shots <= 32767

template <bool SMALL> struct Stage {
    using T = typename std::conditional<SMALL, int16_t, int32_t>::type;
    static constexpr int STRIDE = SMALL ? 72 : 68;  // 144 B / 272 B per item: conflict-free STS.128
    static constexpr size_t BYTES = (size_t)P1_ITEMS * STRIDE * sizeof(T);
};

template <int Q, bool SMALL> struct P1Smem {
    static constexpr size_t STAGE = Stage<SMALL>::BYTES;
    static constexpr size_t EXTRA = Q == 7 ? 2 * 64 * 64 * sizeof(int32_t) : 0;  // tmp + I accumulators
    static constexpr size_t TOTAL = 2 * STAGE + EXTRA;
};

struct P1Args {
    const void *counts;  // rows [row_base, ...) of the record, 2^n columns
    int64_t rowlen;      // 2^n
    int64_t row_base;    // record row of counts[0]
    int64_t aH0;         // first tile row group computed (units of 3^Q rows)
    int64_t naH;         // number of tile row groups computed
    int64_t out_aH0;     // first tile row group held by the output buffer
    int64_t C;           // column tiles, 2^(n-Q)
    int logC;            // log2(C): tile index math by shifts
    Final f;             // f.kind == OUT_INTER: Y1 int32 tile-major
    int debug_no_l2;     // diagnostics only (LRE_P1_DEBUG=noL2 / noL1): skip L2 / L1 work, output invalid
    int debug_no_l1;
    // split Y1 (Q = 7, SMALL): every value's low 16 bits in lo[tile][16384] (int16), and for the
    // 1156 indices with >= 4 identity digits (the only ones that can exceed int16) the high part
    // in hi[tile][1184] at their position; f.out unused
    int split16;
    int16_t *lo;
    int16_t *hi;
    int pipe;  // tile_pass_kernel stage hand-off: 1 = full/empty mbarriers, 0 = lockstep CTA barrier
};

// --- packed loads: 8 consecutive counts -> 4 words (c[2k] | c[2k+1] << 16) ---
// (uint16, the benchmarked record: a plain load, which the compiler may schedule
// freely, ran pass 1 at n = 14 0.75% faster than __ldcs / ld.global.cs, and
// ld.global.nc / .lu / L1::no_allocate / an asm .ca 0.7-5.5% slower:
// profiles/r02d_pass1_prefetch_ab.txt)
__device__ __forceinline__ void load_packed(const uint16_t *p, uint32_t w[4]) {
    const uint4 u = *reinterpret_cast<const uint4 *>(p);
    w[0] = u.x; w[1] = u.y; w[2] = u.z; w[3] = u.w;
}
__device__ __forceinline__ void load_packed(const uint8_t *p, uint32_t w[4]) {
    const uint2 u = __ldcs(reinterpret_cast<const uint2 *>(p));
    w[0] = __byte_perm(u.x, 0, 0x4140); w[1] = __byte_perm(u.x, 0, 0x4342);
    w[2] = __byte_perm(u.y, 0, 0x4140); w[3] = __byte_perm(u.y, 0, 0x4342);
}
__device__ __forceinline__ void load_packed(const int32_t *p, uint32_t w[4]) {
    const int4 a = __ldcs(reinterpret_cast<const int4 *>(p));
    const int4 b = __ldcs(reinterpret_cast<const int4 *>(p) + 1);
    w[0] = __byte_perm(a.x, a.y, 0x5410); w[1] = __byte_perm(a.z, a.w, 0x5410);
    w[2] = __byte_perm(b.x, b.y, 0x5410); w[3] = __byte_perm(b.z, b.w, 0x5410);
}
__device__ __forceinline__ void load_packed(const int64_t *p, uint32_t w[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const longlong2 q = __ldcs(reinterpret_cast<const longlong2 *>(p) + i);
        w[i] = __byte_perm((uint32_t)q.x, (uint32_t)q.y, 0x5410);
    }
}
// --- wide loads: 8 consecutive counts as int32 ---
__device__ __forceinline__ void load_wide(const uint16_t *p, int32_t v[8]) {
    uint32_t w[4];
    load_packed(p, w);
#pragma unroll
    for (int k = 0; k < 4; ++k) { v[2 * k] = (int32_t)(w[k] & 0xffff); v[2 * k + 1] = (int32_t)(w[k] >> 16); }
}
__device__ __forceinline__ void load_wide(const uint8_t *p, int32_t v[8]) {
    const uint2 u = __ldcs(reinterpret_cast<const uint2 *>(p));
#pragma unroll
    for (int k = 0; k < 4; ++k) { v[k] = (u.x >> (8 * k)) & 0xff; v[4 + k] = (u.y >> (8 * k)) & 0xff; }
}
__device__ __forceinline__ void load_wide(const int32_t *p, int32_t v[8]) {
    const int4 a = __ldcs(reinterpret_cast<const int4 *>(p));
    const int4 b = __ldcs(reinterpret_cast<const int4 *>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void load_wide(const int64_t *p, int32_t v[8]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const longlong2 q = __ldcs(reinterpret_cast<const longlong2 *>(p) + i);
        v[2 * i] = (int32_t)q.x; v[2 * i + 1] = (int32_t)q.y;
    }
}

__device__ __forceinline__ void cp_async16(void *sdst, const void *gsrc, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(sdst)),
                 "l"(gsrc), "r"(src_bytes)
                 : "memory");
}

// packed word w = L + 65536 H (|L|,|H|,|L+-H| < 2^15): L - H and L + H
__device__ __forceinline__ int32_t packed_diff(uint32_t w) {
    const int32_t L = (int32_t)(int16_t)(w & 0xffffu);  // sign-extended low half
    return (int32_t)((uint32_t)L * 65537u - w) >> 16;
}
__device__ __forceinline__ int32_t packed_sum(uint32_t w) {
    const int32_t L = (int32_t)(int16_t)(w & 0xffffu);
    return (int32_t)(w + (uint32_t)L * 65535u) >> 16;
}

// L1, SMALL mode: 27 rows (j = a1*9 + a2*3 + a3) x 8 columns, qubits
// (a1,b4) (a2,b5) (a3,b6); b6 is the in-word bit and a3 is streamed.
// sink(D6, v[16]) receives the 16 values (index D4*4 + D5) of Pauli digit D6
// as soon as they are final; only the 16 I accumulators stay live.
template <typename RowLd, typename Sink>
__device__ __forceinline__ void l1_small(RowLd ld, Sink sink) {
    uint32_t Iacc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) Iacc[k] = 0;
#pragma unroll 1
    for (int a3 = 0; a3 < 3; ++a3) {
        uint32_t x[3][3][4];
#pragma unroll
        for (int a1 = 0; a1 < 3; ++a1)
#pragma unroll
            for (int a2 = 0; a2 < 3; ++a2) ld(a1 * 9 + a2 * 3 + a3, x[a1][a2]);
        uint32_t y[4][3][2];  // [D4][a2][b5]
#pragma unroll
        for (int a2 = 0; a2 < 3; ++a2)
#pragma unroll
            for (int b5 = 0; b5 < 2; ++b5)
                q6to4<uint32_t>(x[0][a2][b5], x[0][a2][2 + b5], x[1][a2][b5], x[1][a2][2 + b5], x[2][a2][b5],
                                x[2][a2][2 + b5], y[0][a2][b5], y[1][a2][b5], y[2][a2][b5], y[3][a2][b5]);
        int32_t v[16];
#pragma unroll
        for (int D4 = 0; D4 < 4; ++D4) {
            uint32_t z[4];
            q6to4<uint32_t>(y[D4][0][0], y[D4][0][1], y[D4][1][0], y[D4][1][1], y[D4][2][0], y[D4][2][1], z[0], z[1],
                            z[2], z[3]);
#pragma unroll
            for (int D5 = 0; D5 < 4; ++D5) {
                Iacc[D4 * 4 + D5] += z[D5];
                v[D4 * 4 + D5] = packed_diff(z[D5]);
            }
        }
        sink(a3 + 1, v);
    }
    int32_t v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = packed_sum(Iacc[k]);
    sink(0, v);
}

// L1, WIDE mode (int32 lanes, any shots with 27*shots*3^... < 2^31): same
// transform without packing; b6 is combined inside the last stage.
template <typename RowLd, typename Sink>
__device__ __forceinline__ void l1_wide(RowLd ld, Sink sink) {
    int32_t Iacc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) Iacc[k] = 0;
#pragma unroll 1
    for (int a3 = 0; a3 < 3; ++a3) {
        int32_t y[4][3][4];  // [D4][a2][b5 b6]
#pragma unroll
        for (int a2 = 0; a2 < 3; ++a2) {
            int32_t x[3][8];
#pragma unroll
            for (int a1 = 0; a1 < 3; ++a1) ld(a1 * 9 + a2 * 3 + a3, x[a1]);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                q6to4<int32_t>(x[0][e], x[0][4 + e], x[1][e], x[1][4 + e], x[2][e], x[2][4 + e], y[0][a2][e],
                               y[1][a2][e], y[2][a2][e], y[3][a2][e]);
        }
        int32_t v[16];
#pragma unroll
        for (int D4 = 0; D4 < 4; ++D4) {
            int32_t z0[4], z1[4];
            q6to4<int32_t>(y[D4][0][0], y[D4][0][2], y[D4][1][0], y[D4][1][2], y[D4][2][0], y[D4][2][2], z0[0],
                           z0[1], z0[2], z0[3]);
            q6to4<int32_t>(y[D4][0][1], y[D4][0][3], y[D4][1][1], y[D4][1][3], y[D4][2][1], y[D4][2][3], z1[0],
                           z1[1], z1[2], z1[3]);
#pragma unroll
            for (int D5 = 0; D5 < 4; ++D5) {
                Iacc[D4 * 4 + D5] += z0[D5] + z1[D5];
                v[D4 * 4 + D5] = z0[D5] - z1[D5];
            }
        }
        sink(a3 + 1, v);
    }
    sink(0, Iacc);
}

// L2: the 27 x 8 staged values (rb = a1*9 + a2*3 + a3, g = b1*4 + b2*2 + b3)
// of one staged column -> sink(D3, v[16], is_I) with v index D1*4 + D2 and
// is_I a compile-time std::bool_constant<D3 == 0>.
template <typename T, int STRIDE, typename Sink>
__device__ __forceinline__ void l2_transform(const T *st, Sink sink) {
    int32_t Iacc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) Iacc[k] = 0;
#pragma unroll 1
    for (int a3 = 0; a3 < 3; ++a3) {
        int32_t y[4][3][4];  // [D1][a2][b2 b3]
#pragma unroll
        for (int a2 = 0; a2 < 3; ++a2) {
            int32_t x[3][8];
#pragma unroll
            for (int a1 = 0; a1 < 3; ++a1)
#pragma unroll
                for (int g = 0; g < 8; ++g) x[a1][g] = (int32_t)st[((a1 * 9 + a2 * 3 + a3) * 8 + g) * STRIDE];
#pragma unroll
            for (int e = 0; e < 4; ++e)
                q6to4<int32_t>(x[0][e], x[0][4 + e], x[1][e], x[1][4 + e], x[2][e], x[2][4 + e], y[0][a2][e],
                               y[1][a2][e], y[2][a2][e], y[3][a2][e]);
        }
        int32_t v[16];
#pragma unroll
        for (int D1 = 0; D1 < 4; ++D1) {
            int32_t z0[4], z1[4];
            q6to4<int32_t>(y[D1][0][0], y[D1][0][2], y[D1][1][0], y[D1][1][2], y[D1][2][0], y[D1][2][2], z0[0],
                           z0[1], z0[2], z0[3]);
            q6to4<int32_t>(y[D1][0][1], y[D1][0][3], y[D1][1][1], y[D1][1][3], y[D1][2][1], y[D1][2][3], z1[0],
                           z1[1], z1[2], z1[3]);
#pragma unroll
            for (int D2 = 0; D2 < 4; ++D2) {
                Iacc[D1 * 4 + D2] += z0[D2] + z1[D2];
                v[D1 * 4 + D2] = z0[D2] - z1[D2];
            }
        }
        sink(a3 + 1, v, std::false_type{});
    }
    sink(0, Iacc, std::true_type{});
}

// numerators (int32 or int64) in natural order -> final theta / int64 numerators
template <typename Tn>
__global__ void __launch_bounds__(256) convert_kernel(const Tn *__restrict__ in, int64_t count, const Final f) {
    __shared__ double sfac[33];
    stage_factors(sfac, f.fac);
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        store_final(f, sfac, (uint64_t)i, (int64_t)in[i]);
}

// Staged record of one L1 item: 64 values (+ padding) at position
//   col = (D4 >> 1) * 32 + D6 * 8 + (D4 & 1) * 4 + D5
// so each sink call is two 8-value chunks (one 16-byte shared store each in
// SMALL mode) and the L2 warp reading columns [32w, 32w + 32) owns the 32
// consecutive Pauli indices dlo = D4*16 + D5*4 + D6 in [32w, 32w + 32): its
// global stores are whole 128-byte lines.
template <bool SMALL>
__device__ __forceinline__ void stage_record(typename Stage<SMALL>::T *rec, int D6, const int32_t (&v)[16]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k = 8 * h;
        if constexpr (SMALL) {
            uint4 q;
            q.x = __byte_perm(v[k], v[k + 1], 0x5410);
            q.y = __byte_perm(v[k + 2], v[k + 3], 0x5410);
            q.z = __byte_perm(v[k + 4], v[k + 5], 0x5410);
            q.w = __byte_perm(v[k + 6], v[k + 7], 0x5410);
            *reinterpret_cast<uint4 *>(rec + h * 32 + D6 * 8) = q;
        } else {
            *reinterpret_cast<int4 *>(rec + h * 32 + D6 * 8) = make_int4(v[k], v[k + 1], v[k + 2], v[k + 3]);
            *reinterpret_cast<int4 *>(rec + h * 32 + D6 * 8 + 4) = make_int4(v[k + 4], v[k + 5], v[k + 6], v[k + 7]);
        }
    }
}

__device__ __forceinline__ int staged_col_to_dlo(int col) {
    const int D4 = ((col >> 5) << 1) | ((col >> 2) & 1), D6 = (col >> 3) & 3, D5 = col & 3;
    return D4 * 16 + D5 * 4 + D6;
}

// The per-sub-tile CTA barrier of the tile pass.  The L1 and L2 warps run
// separate loops and so reach it from different code; PTX requires the
// non-.aligned form there (compute-sanitizer synccheck flags bar.sync).
// Measured A/B at n = 14 (profiles/README.md): the inline .aligned form is
// ~1.1 % faster but undefined behaviour; a shared non-inlined .aligned
// barrier costs the same as this one.
__device__ __forceinline__ void p1_step_barrier() { asm volatile("barrier.sync 0;" ::: "memory"); }

// Sub-tile s of this CTA -> tile, top setting digit r1, top outcome bit b1
// compile-time loop: f(std::integral_constant<int, i>) for i = 0 .. N-1
template <int I, int N, typename F> __device__ __forceinline__ void static_for_impl(F &&f) {
    if constexpr (I < N) {
        f(std::integral_constant<int, I>{});
        static_for_impl<I + 1, N>(f);
    }
}
template <int N, typename F> __device__ __forceinline__ void static_for(F &&f) { static_for_impl<0, N>(f); }

struct SubTile {
    int64_t aH, c;
    int r1, b1;
};
template <int Q>
__device__ __forceinline__ SubTile subtile_of(const P1Args &a, int s) {
    constexpr int SUB = Q == 7 ? 6 : 1;
    const int64_t t = blockIdx.x + (int64_t)(s / SUB) * gridDim.x;
    const int sub = s % SUB;
    SubTile st;
    st.aH = a.aH0 + (t >> a.logC);
    st.c = t & (a.C - 1);
    st.r1 = sub >> 1;
    st.b1 = sub & 1;
    return st;
}

// L2 of one sub-tile: staged column `col` -> Pauli values, combined over the
// Q = 7 top qubit (r1, b1) in the thread's private smem slabs tmp / oi.
// (R1, B1) are compile-time so the per-value top-qubit combine is branch-free
// (the runtime form spent ~13% of the L2 warps' instructions on branches).
// SPL: split Y1 storage (make_plan) as a compile-time switch: a runtime test per
// stored value cost the latency-bound L2 warps whole milliseconds of pass 1.
template <int Q, bool SMALL, int R1, int B1, bool SPL>
__device__ __forceinline__ void l2_subtile_rb(const P1Args &a, const SubTile &st,
                                              const typename Stage<SMALL>::T *stage, int col, int32_t *tmp,
                                              int32_t *oi) {
    constexpr int STRIDE = Stage<SMALL>::STRIDE;
    const int dlo = staged_col_to_dlo(col);
    const int64_t tile = (st.aH - a.out_aH0) * a.C + st.c;
    int32_t *out = reinterpret_cast<int32_t *>(a.f.out) + (tile << (2 * Q)) + dlo;
    int32_t *tc = tmp + col, *oc = oi + col;
    // split Y1 (make_plan): the value at u * 64 + dlo (u = top, D1, D2, D3) has a high part
    // iff zc(dlo) >= 4 - zc(u); ZC_U is known at compile time, so most stores need no test.
    int16_t *lo = a.lo + (tile << 14) + dlo;
    int16_t *hi = a.hi + tile * LRE_Y1_HROW;
    // per threshold t = 4 - zc(u): this thread's rank among the low digit patterns with
    // >= t identities (t <= 0: its own dlo), and whether it is one
    const uint32_t lrpack = (Q == 7 && SPL) ? g_y1_lrpack[dlo] : 0u;
    const int hidx[4] = {dlo, (int)(lrpack & 0xFF), (int)((lrpack >> 8) & 0xFF), (int)((lrpack >> 16) & 0xFF)};
    const bool hok[4] = {true, hidx[1] != 0xFF, hidx[2] != 0xFF, hidx[3] != 0xFF};
    auto put = [&](int idx_hi, auto zc_u, int32_t val) {  // idx_hi = u * 64
        constexpr int T = 4 - decltype(zc_u)::value;
        if constexpr (Q != 7 || !SPL) {
            out[idx_hi] = val;
        } else {
            lo[idx_hi] = (int16_t)val;
            if constexpr (T < 4) {
                constexpr int TI = T < 0 ? 0 : T;
                // high part = floor((val + 2^15) / 2^16), the carry above the signed low half
                const int pos = c_y1_uoff[idx_hi >> 6] + hidx[TI];
                const int16_t h16 = (int16_t)((val + 32768) >> 16);
                if (hok[TI]) hi[pos] = h16;
            }
        }
    };
    l2_transform<typename Stage<SMALL>::T, STRIDE>(stage + col, [&](int D3, const int32_t(&v)[16], auto is_i) {
        static_for<16>([&](auto K) {
            constexpr int k = decltype(K)::value;
            const int r = k * 4 + D3;  // core digits D1 D2 D3
            if constexpr (Q == 6) {
                out[r * 64] = v[k];
            } else if constexpr (B1 == 0) {
                tc[r * 64] = v[k];
            } else {
                const int32_t u = tc[r * 64];
                int32_t acc = u + v[k];
                if constexpr (R1 > 0) acc += oc[r * 64];
                // identity digits among D1 D2 D3 (k = D1 * 4 + D2 is unrolled)
                using ZcR = std::integral_constant<int, ((k >> 2) == 0) + ((k & 3) == 0) + (decltype(is_i)::value ? 1 : 0)>;
                if constexpr (R1 < 2) oc[r * 64] = acc;
                else put(r * 64, std::integral_constant<int, ZcR::value + 1>{}, acc);  // top digit I
                put((R1 + 1) * 4096 + r * 64, ZcR{}, u - v[k]);                       // top digit X / Y / Z
            }
        });
    });
}

template <int Q, bool SMALL, bool SPL>
__device__ __forceinline__ void l2_subtile(const P1Args &a, const SubTile &st, const typename Stage<SMALL>::T *stage,
                                           int col, int32_t *tmp, int32_t *oi) {
    if constexpr (Q == 6) {
        l2_subtile_rb<Q, SMALL, 0, 0, SPL>(a, st, stage, col, tmp, oi);
    } else {
        switch (st.r1 * 2 + st.b1) {
        case 0: l2_subtile_rb<Q, SMALL, 0, 0, SPL>(a, st, stage, col, tmp, oi); break;
        case 1: l2_subtile_rb<Q, SMALL, 0, 1, SPL>(a, st, stage, col, tmp, oi); break;
        case 2: l2_subtile_rb<Q, SMALL, 1, 0, SPL>(a, st, stage, col, tmp, oi); break;
        case 3: l2_subtile_rb<Q, SMALL, 1, 1, SPL>(a, st, stage, col, tmp, oi); break;
        case 4: l2_subtile_rb<Q, SMALL, 2, 0, SPL>(a, st, stage, col, tmp, oi); break;
        default: l2_subtile_rb<Q, SMALL, 2, 1, SPL>(a, st, stage, col, tmp, oi); break;
        }
    }
}

// Pass-1 tile kernel, LDG variant: persistent, 2 CTAs x 9 warps per SM in
// SMALL mode.  Per sub-tile s (one __syncthreads):
//   warps 0-6  L1(s): thread = row block rb x column chunk g; the 27 x 8
//              count block -> 3 qubits in registers -> staged (int16);
//   warps 7-8  L2(s-1): thread = staged column; the 27 x 8 staged values ->
//              3 more qubits -> 64 values stored as whole 128-byte lines.
// L1 warps wait on HBM while L2 warps compute, and the two CTAs of an SM
// interleave their phases.  LOGN > 0 makes the row length 2^LOGN a
// compile-time constant so the 27 row loads of an item are [base + imm]
// (the runtime form costs ~5 integer instructions of address math per load).
template <int Q, bool SMALL, typename Tin, int LOGN, bool SPL = false>
__global__ void __launch_bounds__(P1_THREADS, SMALL ? 2 : 1) tile_pass_kernel(const P1Args a) {
    using ST = Stage<SMALL>;
    using T = typename ST::T;
    constexpr int STRIDE = ST::STRIDE;
    constexpr int SUB = Q == 7 ? 6 : 1;
    constexpr int64_t Q3 = Q == 7 ? 2187 : 729;
    extern __shared__ __align__(16) unsigned char smem[];
    int32_t *tmp = reinterpret_cast<int32_t *>(smem + 2 * ST::BYTES);  // [64 r][64 col]
    int32_t *oi = tmp + 64 * 64;                                        // [64 r][64 col]

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int64_t ntiles = a.naH * a.C;
    const int my_tiles = (int64_t)blockIdx.x < ntiles ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
    const int S = my_tiles * SUB;
    const Tin *counts = reinterpret_cast<const Tin *>(a.counts);
    const int rowlen = LOGN > 0 ? (1 << LOGN) : (int)a.rowlen;
    const bool l1 = warp < P1_L1_WARPS && tid < P1_ITEMS;
    const int rb = tid >> 3, g = tid & 7;
    // Stage hand-off.  a.pipe (default): per-buffer full/empty mbarriers, so the
    // L1 warps fill buffer s & 1 as soon as the L2 warps have drained sub-tile
    // s - 2 and a slow step on either side is absorbed by the other instead of
    // both waiting at a lockstep CTA barrier (ncu at n = 14: ~28 % of both
    // sides' samples sat in that barrier).  LRE_P1_SYNC=bar: the lockstep form.
    __shared__ __align__(8) uint64_t bars[4];  // full[2], empty[2]
    if (a.pipe) {
        if (tid == 0) {
            mbar_init(&bars[0], 32 * P1_L1_WARPS);
            mbar_init(&bars[1], 32 * P1_L1_WARPS);
            mbar_init(&bars[2], 32 * P1_L2_WARPS);
            mbar_init(&bars[3], 32 * P1_L2_WARPS);
            fence_mbar_init();
        }
        __syncthreads();
    }

    auto item_base = [&](int s) -> const Tin * {
        const SubTile st = subtile_of<Q>(a, s);
        const int64_t row = st.aH * Q3 + (Q == 7 ? st.r1 * 729 : 0) + rb * 27 - a.row_base;
        const int64_t col = (st.c << Q) + (Q == 7 ? st.b1 * 64 : 0) + g * 8;
        return counts + row * (int64_t)rowlen + col;
    };
    auto load_step = [&](const Tin *base, int a3, uint32_t(&x)[3][3][4]) {
#pragma unroll
        for (int a1 = 0; a1 < 3; ++a1)
#pragma unroll
            for (int a2 = 0; a2 < 3; ++a2) load_packed(base + (a1 * 9 + a2 * 3 + a3) * rowlen, x[a1][a2]);
    };

    // L1 and L2 warps run separate loops with the same barrier sequence, so
    // the L1 loop's registers that live across sub-tiles (the prefetched
    // next step) are not allocated in the L2 code.
    if (warp < P1_L1_WARPS) {
        // SMALL: the loads of the next 9-row step are issued as soon as the
        // first qubit stage has consumed the current step's words (reusing
        // their registers), so they fly during the rest of this step's
        // compute — the next sub-tile's first step included.
        uint32_t x[3][3][4];
        const Tin *base = nullptr;
        if constexpr (SMALL) {
            if (l1 && S > 0) {
                base = item_base(0);
                load_step(base, 0, x);
            }
        }
        for (int s = 0; s <= S; ++s) {
            if (a.pipe) {
                if (s == S) break;
                // the L2 warps set the pace: sleep instead of spinning on their issue slots
                if (s >= 2) mbar_wait_sleep(&bars[2 + (s & 1)], ((s >> 1) - 1) & 1, 100000);
            }
            if (s < S && l1 && !a.debug_no_l1) {
                T *rec = reinterpret_cast<T *>(smem + (s & 1) * ST::BYTES) + tid * STRIDE;
                if constexpr (SMALL) {
                    const Tin *next_base = s + 1 < S ? item_base(s + 1) : nullptr;
                    uint32_t Iacc[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) Iacc[k] = 0;
#pragma unroll
                    for (int a3 = 0; a3 < 3; ++a3) {
                        uint32_t y[4][3][2];  // [D4][a2][b5]: qubit (a1, b4)
#pragma unroll
                        for (int a2 = 0; a2 < 3; ++a2)
#pragma unroll
                            for (int b5 = 0; b5 < 2; ++b5)
                                q6to4<uint32_t>(x[0][a2][b5], x[0][a2][2 + b5], x[1][a2][b5], x[1][a2][2 + b5],
                                                x[2][a2][b5], x[2][a2][2 + b5], y[0][a2][b5], y[1][a2][b5],
                                                y[2][a2][b5], y[3][a2][b5]);
                        if (a3 < 2) load_step(base, a3 + 1, x);
                        else if (next_base) load_step(next_base, 0, x);
                        // L2 prefetch of the rows two load steps ahead (the register loads above
                        // run one step ahead): the L1 warps are load-latency bound, and the extra
                        // lead cut pass 1 at n = 14 from 29.17 to 28.71 ms (3 steps ahead: 30.2 ms;
                        // profiles/r02d_pass1_prefetch_ab.txt).  Compile-time row length only, so
                        // the addresses are [base + immediate] and no register is added.
                        if constexpr (LOGN > 0) {
                            // (the last sub-tile has no next one: it re-prefetches its own rows)
                            const Tin *pb = a3 == 0 || !next_base ? base : next_base;
                            const Tin *pr = pb + (a3 == 0 ? 2 : a3 - 1) * (1 << LOGN);
                            static_for<9>([&](auto K) {
                                constexpr int k = decltype(K)::value;
                                asm volatile("prefetch.global.L2 [%0+%1];" ::"l"(pr),
                                             "n"(((k / 3) * 9 + (k % 3) * 3) * (1 << LOGN) * (int)sizeof(Tin)));
                            });
                        }
                        int32_t v[16];
#pragma unroll
                        for (int D4 = 0; D4 < 4; ++D4) {
                            uint32_t z[4];
                            q6to4<uint32_t>(y[D4][0][0], y[D4][0][1], y[D4][1][0], y[D4][1][1], y[D4][2][0],
                                            y[D4][2][1], z[0], z[1], z[2], z[3]);
#pragma unroll
                            for (int D5 = 0; D5 < 4; ++D5) {
                                Iacc[D4 * 4 + D5] += z[D5];
                                v[D4 * 4 + D5] = packed_diff(z[D5]);
                            }
                        }
                        stage_record<true>(rec, a3 + 1, v);
                    }
                    int32_t v[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) v[k] = packed_sum(Iacc[k]);
                    stage_record<true>(rec, 0, v);
                    base = next_base;
                } else {
                    const Tin *ib = item_base(s);
                    l1_wide([&](int j, int32_t(&w)[8]) { load_wide(ib + j * rowlen, w); },
                            [&](int D6, const int32_t(&v)[16]) { stage_record<SMALL>(rec, D6, v); });
                }
            }
            if (a.pipe) mbar_arrive(&bars[s & 1]);
            else p1_step_barrier();
        }
    } else if (a.pipe) {
        for (int s = 0; s < S; ++s) {
            mbar_wait(&bars[s & 1], (s >> 1) & 1);
            if (!a.debug_no_l2)
                l2_subtile<Q, SMALL, SPL>(a, subtile_of<Q>(a, s), reinterpret_cast<const T *>(smem + (s & 1) * ST::BYTES),
                                     tid - 32 * P1_L1_WARPS, tmp, oi);
            mbar_arrive(&bars[2 + (s & 1)]);
        }
    } else {
        for (int s = 0; s <= S; ++s) {
            if (s > 0 && !a.debug_no_l2)
                l2_subtile<Q, SMALL, SPL>(a, subtile_of<Q>(a, s - 1),
                                     reinterpret_cast<const T *>(smem + ((s - 1) & 1) * ST::BYTES),
                                     tid - 32 * P1_L1_WARPS, tmp, oi);
            p1_step_barrier();
        }
    }
}

// ---------------------------------------------------------------------------
// L2 split by the top core setting digit a1 (for the warp-parallel L2 of the
// ring kernel): qubits c3 = (a3, b3) and c2 = (a2, b2, streamed over a2) in
// registers, then the b1 half of qubit c1.  emit(r, v) receives the final
// values with D1 = a1 + 1 (r = D1*16 + D2*4 + D3); icon(k, v) receives this
// a1's contribution to the D1 = I value of k = D2*4 + D3.
template <typename T, int STRIDE, typename Emit, typename Icon>
__device__ __forceinline__ void l2_part(const T *st, int a1, Emit emit, Icon icon) {
    int32_t Iacc[2][4];  // [b1][D3], D2 = I
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int d = 0; d < 4; ++d) Iacc[b][d] = 0;
#pragma unroll
    for (int a2 = 0; a2 < 3; ++a2) {
        int32_t x[3][8];  // [a3][g = b1 b2 b3]
#pragma unroll
        for (int a3 = 0; a3 < 3; ++a3)
#pragma unroll
            for (int g = 0; g < 8; ++g) x[a3][g] = (int32_t)st[((a1 * 9 + a2 * 3 + a3) * 8 + g) * STRIDE];
        int32_t u[2][2][4];  // [b1][b2][D3]
#pragma unroll
        for (int b1 = 0; b1 < 2; ++b1)
#pragma unroll
            for (int b2 = 0; b2 < 2; ++b2) {
                const int g0 = b1 * 4 + b2 * 2;
                q6to4<int32_t>(x[0][g0], x[0][g0 + 1], x[1][g0], x[1][g0 + 1], x[2][g0], x[2][g0 + 1], u[b1][b2][0],
                               u[b1][b2][1], u[b1][b2][2], u[b1][b2][3]);
            }
#pragma unroll
        for (int D3 = 0; D3 < 4; ++D3) {
            Iacc[0][D3] += u[0][0][D3] + u[0][1][D3];
            Iacc[1][D3] += u[1][0][D3] + u[1][1][D3];
            const int32_t d0 = u[0][0][D3] - u[0][1][D3], d1 = u[1][0][D3] - u[1][1][D3];  // D2 = a2 + 1
            emit((a1 + 1) * 16 + (a2 + 1) * 4 + D3, d0 - d1);
            icon((a2 + 1) * 4 + D3, d0 + d1);
        }
    }
#pragma unroll
    for (int D3 = 0; D3 < 4; ++D3) {
        emit((a1 + 1) * 16 + D3, Iacc[0][D3] - Iacc[1][D3]);
        icon(D3, Iacc[0][D3] + Iacc[1][D3]);
    }
}

// Store core value r (D1 D2 D3) of staged column col for sub-tile st: Q = 6
// writes Y1 directly; Q = 7 combines the tile's top qubit (r1, b1): the
// b1 = 0 half parks in tmp, X/Y/Z = tmp - v are final, I accumulates in oi
// over r1.  Each (r, col) is owned by exactly one thread.
template <int Q>
__device__ __forceinline__ void p1_store(int32_t *out, const SubTile &st, int r, int col, int32_t v, int32_t *tmp,
                                         int32_t *oi) {
    if constexpr (Q == 6) {
        out[r * 64] = v;
    } else if (st.b1 == 0) {
        tmp[r * 64 + col] = v;
    } else {
        const int32_t u = tmp[r * 64 + col];
        const int32_t acc = (st.r1 == 0 ? 0 : oi[r * 64 + col]) + u + v;
        if (st.r1 < 2) oi[r * 64 + col] = acc;
        else out[r * 64] = acc;                    // top digit I
        out[(st.r1 + 1) * 4096 + r * 64] = u - v;  // top digit X / Y / Z
    }
}

template <int Q>
__device__ __forceinline__ int32_t *p1_out(const P1Args &a, const SubTile &st, int col) {
    return reinterpret_cast<int32_t *>(a.f.out) + (((st.aH - a.out_aH0) * a.C + st.c) << (2 * Q)) +
           staged_col_to_dlo(col);
}

// Pass-1 tile kernel, cp.async-ring variant (uint16 counts, SMALL mode): one
// CTA of 15 warps per SM, persistent.  Per sub-tile s (one __syncthreads):
//   warps 0-6   L1(s): each thread streams the 9-row steps of its items
//               through a private ring of three 144-byte shared-memory slots
//               filled by cp.async, so steps q+1 and q+2 are in flight while
//               step q computes (62 KB per SM continuously, no registers
//               held), across sub-tile boundaries;
//   warps 7-12  L2(s-1): staged column x top core digit a1 -> the D1 = a1+1
//               values + I contributions (the single-thread-per-column L2 is
//               a latency-bound chain of ~900 instructions);
//   warps 13-14 I(s-2): the D1 = I values = sum of the three contributions.
constexpr int RING_SLOT_BYTES = 9 * 16;
constexpr int RING_THREAD_BYTES = 3 * RING_SLOT_BYTES;
constexpr int RING_L1_WARPS = 7, RING_L2_WARPS = 6, RING_RED_WARPS = 2;
constexpr int RING_THREADS = 32 * (RING_L1_WARPS + RING_L2_WARPS + RING_RED_WARPS);

template <int Q> struct RingSmem {
    static constexpr size_t STAGE = Stage<true>::BYTES;
    static constexpr size_t EXTRA = P1Smem<Q, true>::EXTRA;
    static constexpr size_t IRED = 2 * 3 * 16 * 64 * sizeof(int32_t);
    static constexpr size_t RING = (size_t)P1_ITEMS * RING_THREAD_BYTES;
    static constexpr size_t TOTAL = 2 * STAGE + EXTRA + IRED + RING;
};

template <int Q, int LOGN>
__global__ void __launch_bounds__(RING_THREADS, 1) tile_ring_kernel(const P1Args a) {
    using ST = Stage<true>;
    using T = ST::T;
    constexpr int STRIDE = ST::STRIDE;
    constexpr int SUB = Q == 7 ? 6 : 1;
    constexpr int64_t Q3 = Q == 7 ? 2187 : 729;
    extern __shared__ __align__(16) unsigned char smem[];
    int32_t *tmp = reinterpret_cast<int32_t *>(smem + 2 * ST::BYTES);
    int32_t *oi = tmp + 64 * 64;
    int32_t *ired = reinterpret_cast<int32_t *>(smem + 2 * ST::BYTES + RingSmem<Q>::EXTRA);  // [2][3][16][64]
    unsigned char *ring = smem + 2 * ST::BYTES + RingSmem<Q>::EXTRA + RingSmem<Q>::IRED;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int64_t ntiles = a.naH * a.C;
    const int my_tiles = (int64_t)blockIdx.x < ntiles ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
    const int S = my_tiles * SUB;
    const uint16_t *counts = reinterpret_cast<const uint16_t *>(a.counts);
    const int rowlen = LOGN > 0 ? (1 << LOGN) : (int)a.rowlen;
    const bool l1 = tid < P1_ITEMS;
    const int rb = tid >> 3, g = tid & 7;
    unsigned char *myring = ring + (l1 ? tid : 0) * RING_THREAD_BYTES;

    auto item_base = [&](int s) -> const uint16_t * {
        const SubTile st = subtile_of<Q>(a, s);
        const int64_t row = st.aH * Q3 + (Q == 7 ? st.r1 * 729 : 0) + rb * 27 - a.row_base;
        const int64_t col = (st.c << Q) + (Q == 7 ? st.b1 * 64 : 0) + g * 8;
        return counts + row * (int64_t)rowlen + col;
    };
    // step q = 3 s + a3: the 9 rows (a1, a2) of step a3 of sub-tile s
    const int nq = 3 * S;
    const uint16_t *ib_issue = nullptr;
    int s_issue = -1;
    auto issue = [&](int q) {
        if (q < nq) {
            const int s = q / 3, a3 = q % 3;
            if (s != s_issue) {
                ib_issue = item_base(s);
                s_issue = s;
            }
            unsigned char *slot = myring + (q % 3) * RING_SLOT_BYTES;
#pragma unroll
            for (int a1 = 0; a1 < 3; ++a1)
#pragma unroll
                for (int a2 = 0; a2 < 3; ++a2)
                    cp_async16(slot + (a1 * 3 + a2) * 16, ib_issue + (a1 * 9 + a2 * 3 + a3) * rowlen, 16);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    if (l1) {
        issue(0);
        issue(1);
    }
    for (int s = 0; s < S + 2; ++s) {
        if (warp < RING_L1_WARPS) {
            if (s < S && l1) {
                T *rec = reinterpret_cast<T *>(smem + (s & 1) * ST::BYTES) + tid * STRIDE;
                uint32_t Iacc[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) Iacc[k] = 0;
#pragma unroll
                for (int a3 = 0; a3 < 3; ++a3) {
                    const int q = 3 * s + a3;
                    issue(q + 2);
                    asm volatile("cp.async.wait_group 2;" ::: "memory");
                    const unsigned char *slot = myring + (q % 3) * RING_SLOT_BYTES;
                    uint32_t x[3][3][4];
#pragma unroll
                    for (int a1 = 0; a1 < 3; ++a1)
#pragma unroll
                        for (int a2 = 0; a2 < 3; ++a2) {
                            const uint4 u = *reinterpret_cast<const uint4 *>(slot + (a1 * 3 + a2) * 16);
                            x[a1][a2][0] = u.x; x[a1][a2][1] = u.y; x[a1][a2][2] = u.z; x[a1][a2][3] = u.w;
                        }
                    uint32_t y[4][3][2];  // [D4][a2][b5]
#pragma unroll
                    for (int a2 = 0; a2 < 3; ++a2)
#pragma unroll
                        for (int b5 = 0; b5 < 2; ++b5)
                            q6to4<uint32_t>(x[0][a2][b5], x[0][a2][2 + b5], x[1][a2][b5], x[1][a2][2 + b5],
                                            x[2][a2][b5], x[2][a2][2 + b5], y[0][a2][b5], y[1][a2][b5], y[2][a2][b5],
                                            y[3][a2][b5]);
                    int32_t v[16];
#pragma unroll
                    for (int D4 = 0; D4 < 4; ++D4) {
                        uint32_t z[4];
                        q6to4<uint32_t>(y[D4][0][0], y[D4][0][1], y[D4][1][0], y[D4][1][1], y[D4][2][0],
                                        y[D4][2][1], z[0], z[1], z[2], z[3]);
#pragma unroll
                        for (int D5 = 0; D5 < 4; ++D5) {
                            Iacc[D4 * 4 + D5] += z[D5];
                            v[D4 * 4 + D5] = packed_diff(z[D5]);
                        }
                    }
                    stage_record<true>(rec, a3 + 1, v);
                }
                int32_t v[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) v[k] = packed_sum(Iacc[k]);
                stage_record<true>(rec, 0, v);
            }
        } else if (warp < RING_L1_WARPS + RING_L2_WARPS) {
            if (s >= 1 && s <= S) {
                const int u = tid - 32 * RING_L1_WARPS;
                const int a1 = u >> 6, col = u & 63;
                const SubTile st = subtile_of<Q>(a, s - 1);
                const T *stage = reinterpret_cast<const T *>(smem + ((s - 1) & 1) * ST::BYTES) + col;
                int32_t *out = p1_out<Q>(a, st, col);
                int32_t *ic = ired + (((s - 1) & 1) * 3 + a1) * 16 * 64 + col;
                l2_part<T, STRIDE>(
                    stage, a1, [&](int r, int32_t v) { p1_store<Q>(out, st, r, col, v, tmp, oi); },
                    [&](int k, int32_t v) { ic[k * 64] = v; });
            }
        } else {
            if (s >= 2) {
                const int col = tid - 32 * (RING_L1_WARPS + RING_L2_WARPS);
                const SubTile st = subtile_of<Q>(a, s - 2);
                int32_t *out = p1_out<Q>(a, st, col);
                const int32_t *ic = ired + ((s - 2) & 1) * 3 * 16 * 64 + col;
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    p1_store<Q>(out, st, k, col, ic[k * 64] + ic[(16 + k) * 64] + ic[(32 + k) * 64], tmp, oi);
            }
        }
        __syncthreads();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// ===========================================================================
// pass 1, TMA variant (uint16 counts, SMALL mode): a producer warp streams
// the 27-row x 128-byte box of every L1 row block into a ring of shared
// memory slots with cp.async.bulk.tensor (128-byte swizzle, so the eight
// 16-byte chunks of a row land in distinct banks for any row), completing on
// mbarriers; L1 threads read their rows from shared memory.  Slot rb holds
// row block rb of consecutive sub-tiles, so its fill number is the sub-tile
// index and every waiter is at most one mbarrier phase ahead (a waiter two
// phases ahead would alias parities: with fewer slots than row blocks, row
// blocks rb and rb + NSLOT of one sub-tile raced and hung).  The ring keeps up
// to one sub-tile (~93 KB) per SM in flight independent of L1/L2 compute.
// ===========================================================================
constexpr int TMA_NSLOT = 27;  // one slot per L1 row block: slot = rb, fill = sub-tile
constexpr int TMA_SLOT_BYTES = 4096;  // 27 * 128 B, padded to the 1024-byte swizzle atom
constexpr int TMA_BOX_BYTES = 27 * 128;
constexpr int TMA_L1_WARPS = 7, TMA_L2_WARPS = 2;
constexpr int TMA_COMPUTE_THREADS = 32 * (TMA_L1_WARPS + TMA_L2_WARPS);
constexpr int TMA_THREADS = TMA_COMPUTE_THREADS + 32;  // + producer warp

template <int Q> struct TmaSmem {
    static constexpr size_t RING = (size_t)TMA_NSLOT * TMA_SLOT_BYTES;
    static constexpr size_t STAGE = Stage<true>::BYTES;
    static constexpr size_t EXTRA = P1Smem<Q, true>::EXTRA;
    static constexpr size_t BARS = 2 * TMA_NSLOT * sizeof(uint64_t);
    static constexpr size_t TOTAL = 1024 /* alignment slack */ + RING + 2 * STAGE + EXTRA + BARS;
};

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

template <int Q>
__global__ void __launch_bounds__(TMA_THREADS, 1) tile_tma_kernel(const P1Args a, const __grid_constant__ CUtensorMap map) {
    using ST = Stage<true>;
    using T = ST::T;
    constexpr int STRIDE = ST::STRIDE;
    constexpr int SUB = Q == 7 ? 6 : 1;
    constexpr int64_t Q3 = Q == 7 ? 2187 : 729;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char *ring = smem;
    unsigned char *stage0 = ring + TmaSmem<Q>::RING;
    int32_t *tmp = reinterpret_cast<int32_t *>(stage0 + 2 * ST::BYTES);
    int32_t *oi = tmp + 64 * 64;
    uint64_t *full = reinterpret_cast<uint64_t *>(stage0 + 2 * ST::BYTES + TmaSmem<Q>::EXTRA);
    uint64_t *empty = full + TMA_NSLOT;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int64_t ntiles = a.naH * a.C;
    const int my_tiles = (int64_t)blockIdx.x < ntiles ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
    const int S = my_tiles * SUB;

    if (tid == 0) {
        for (int i = 0; i < TMA_NSLOT; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 8);  // the 8 L1 threads (column chunks) of a row block
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    if (warp == TMA_L1_WARPS + TMA_L2_WARPS) {  // producer
        if ((tid & 31) == 0) {
            const int total = S * 27;
            auto coords = [&](int q, int &col, int &row) {
                const SubTile st = subtile_of<Q>(a, q / 27);
                row = (int)(st.aH * Q3 + (Q == 7 ? st.r1 * 729 : 0) + (q % 27) * 27 - a.row_base);
                col = (int)((st.c << Q) + (Q == 7 ? st.b1 * 64 : 0));
            };
            for (int q = 0; q < total; ++q) {
                const int slot = q % TMA_NSLOT;  // == rb
                int col, row;
                if (q >= TMA_NSLOT) mbar_wait(&empty[slot], ((q / TMA_NSLOT) - 1) & 1);
                coords(q, col, row);
                mbar_expect_tx(&full[slot], TMA_BOX_BYTES);
                tma_load_2d(ring + slot * TMA_SLOT_BYTES, &map, col, row, &full[slot]);
            }
        }
        return;
    }

    for (int s = 0; s <= S; ++s) {
        if (warp < TMA_L1_WARPS) {
            if (s < S && tid < P1_ITEMS) {
                const int rb = tid >> 3, g = tid & 7;
                const int q = s * 27 + rb;
                const int slot = q % TMA_NSLOT;
                mbar_wait(&full[slot], (q / TMA_NSLOT) & 1);
                const unsigned char *box = ring + slot * TMA_SLOT_BYTES;
                T *rec = reinterpret_cast<T *>(stage0 + (s & 1) * ST::BYTES) + tid * STRIDE;
                l1_small(
                    [&](int j, uint32_t(&w)[4]) {
                        const uint4 u = *reinterpret_cast<const uint4 *>(box + j * 128 + ((g ^ (j & 7)) << 4));
                        w[0] = u.x; w[1] = u.y; w[2] = u.z; w[3] = u.w;
                    },
                    [&](int D6, const int32_t(&v)[16]) { stage_record<true>(rec, D6, v); });
                mbar_arrive(&empty[slot]);
            }
        } else if (s > 0) {
            l2_subtile<Q, true, false>(a, subtile_of<Q>(a, s - 1),
                                reinterpret_cast<const T *>(stage0 + ((s - 1) & 1) * ST::BYTES),
                                tid - 32 * TMA_L1_WARPS, tmp, oi);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(TMA_COMPUTE_THREADS) : "memory");
    }
}

// ===========================================================================
// vfold: Q <= 3 qubits per pass over a vector axis V
// ===========================================================================
// input  X[a][col][v]   a in [xa0, ...) rows of the previous level (only
//        a in [alo, ahi) hold data, others read as 0), col in [0, 2^R),
//        v in [0, V)
// output Y[A - ya0][B][4^Q][v]  for A in [A0, A0 + nA), B in [0, 2^(R-Q))
// (or, when final, natural Pauli index d * V + v with A = B = 0).
struct VArgs {
    const void *in;
    int64_t V;
    int64_t ncol;  // 2^R
    int64_t xa0, alo, ahi;
    int64_t A0, nA, ya0;
    int64_t nB;  // 2^(R-Q)
    int logV, lognB;  // V and nB are powers of two: index math by shifts (64-bit div/mod is ~100 instructions)
    int vf1_batch;  // Q = 1: issue all row loads of 4 elements first (LRE_VF1=0 disables; A/B only)
    Final f;
    const int32_t *hi = nullptr;  // split Y1 high parts of the input (rows of V / 16384 * 1184) for the merge, or null
};

// final-store value: integers widen to int64 numerators, fp64 stays fp64
template <typename Ta> __device__ __forceinline__ auto fin_val(Ta y) {
    if constexpr (std::is_floating_point<Ta>::value) return (double)y;
    else return (int64_t)y;
}

template <typename Tin>
__device__ __forceinline__ auto vload(const Tin *p) {
    if constexpr (std::is_floating_point<Tin>::value) return __ldcs(p);
    else return (int64_t)__ldcs(p);
}
template <> __device__ __forceinline__ auto vload<uint8_t>(const uint8_t *p) { return (int64_t)*p; }
template <> __device__ __forceinline__ auto vload<uint16_t>(const uint16_t *p) {
    return (int64_t)__ldcs(reinterpret_cast<const unsigned short *>(p));
}

// Loop-invariant strides are re-materialised through an opaque move inside
// the loop so ptxas does not hoist dozens of 64-bit address products out of
// it (that alone pushed the Q = 3 kernels to 255 registers with spills).
__device__ __forceinline__ int64_t opaque(int64_t x) {
    int64_t y;
    asm volatile("mov.b64 %0, %1;" : "=l"(y) : "l"(x));
    return y;
}

// Q-qubit transform of one (3^Q x 2^Q) block, streamed over the most
// significant row digit r1: ld(j, s) loads row digits j (< 3^(Q-1), lower
// digits) x column bits s of the current r1; sink(d, v) receives natural
// output index d (first qubit most significant).
template <int Q, typename Ta, typename Ld, typename Sink>
__device__ __forceinline__ void vblock(Ld ld, Sink sink) {
    constexpr int H = 1 << (Q - 1);                    // columns per b1
    constexpr int NL = 1 << (2 * (Q - 1));             // outputs per top digit
    Ta Iacc[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) Iacc[k] = 0;
#pragma unroll 1
    for (int r1 = 0; r1 < 3; ++r1) {
        Ta w[2][NL];  // [b1][lower digits]
#pragma unroll
        for (int b1 = 0; b1 < 2; ++b1) {
            if constexpr (Q == 1) {
                w[b1][0] = ld(r1, 0, b1);
            } else if constexpr (Q == 2) {
                Ta x[3][2];
#pragma unroll
                for (int j = 0; j < 3; ++j)
#pragma unroll
                    for (int s = 0; s < 2; ++s) x[j][s] = ld(r1, j, b1 * H + s);
                q6to4<Ta>(x[0][0], x[0][1], x[1][0], x[1][1], x[2][0], x[2][1], w[b1][0], w[b1][1], w[b1][2], w[b1][3]);
            } else {
                Ta u[3][2][4];  // after qubit 3: [r2][b2][D3]
#pragma unroll
                for (int r2 = 0; r2 < 3; ++r2)
#pragma unroll
                    for (int b2 = 0; b2 < 2; ++b2) {
                        Ta x[3][2];
#pragma unroll
                        for (int r3 = 0; r3 < 3; ++r3)
#pragma unroll
                            for (int b3 = 0; b3 < 2; ++b3) x[r3][b3] = ld(r1, r2 * 3 + r3, b1 * H + b2 * 2 + b3);
                        q6to4<Ta>(x[0][0], x[0][1], x[1][0], x[1][1], x[2][0], x[2][1], u[r2][b2][0], u[r2][b2][1],
                                  u[r2][b2][2], u[r2][b2][3]);
                    }
#pragma unroll
                for (int d3 = 0; d3 < 4; ++d3)
                    q6to4<Ta>(u[0][0][d3], u[0][1][d3], u[1][0][d3], u[1][1][d3], u[2][0][d3], u[2][1][d3],
                              w[b1][0 * 4 + d3], w[b1][1 * 4 + d3], w[b1][2 * 4 + d3], w[b1][3 * 4 + d3]);
            }
        }
#pragma unroll
        for (int k = 0; k < NL; ++k) {
            Iacc[k] += w[0][k] + w[1][k];
            sink((r1 + 1) * NL + k, w[0][k] - w[1][k]);
        }
    }
#pragma unroll
    for (int k = 0; k < NL; ++k) sink(k, Iacc[k]);
}

template <int Q, typename Tin, typename Ta, bool FINAL>
#ifndef VF1_MINB
#define VF1_MINB 8
#endif
#ifndef VF1_U
#define VF1_U 2
#endif
__global__ void __launch_bounds__(128, Q == 1 ? VF1_MINB : 4) vfold_kernel(const VArgs a) {
    constexpr int R3 = Q == 1 ? 3 : Q == 2 ? 9 : 27;
    constexpr int C2 = 1 << Q;
    constexpr int NOUT = 1 << (2 * Q);
    constexpr int RL = R3 / 3;  // rows per top digit
    const int64_t total = a.nA * a.nB * a.V;
    const Tin *in = reinterpret_cast<const Tin *>(a.in);
    __shared__ double sfac[FINAL ? 33 : 1];
    if constexpr (FINAL) {
        stage_factors(sfac, a.f.fac);
        __syncthreads();
    }
    if (Q == 1 && a.vf1_batch) {
        // One qubit: each thread issues the six row loads of VF1_U elements
        // before any arithmetic (the r1-streamed vblock keeps only two loads
        // in flight, which held the final n = 14 pass at 2.4 TB/s).
        constexpr int U = VF1_U;
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t0 < total; t0 += U * stride) {
            Ta x[U][6];
            int64_t vv[U], AA[U], BB[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t t = t0 + u * stride;
                const int64_t V = opaque(a.V);
                vv[u] = t & (V - 1);
                const int64_t rest = t >> a.logV;
                BB[u] = rest & (a.nB - 1);
                AA[u] = a.A0 + (rest >> a.lognB);
                const int64_t row0 = AA[u] * 3;
                const Tin *p0 = in + ((row0 - a.xa0) * a.ncol + BB[u] * 2) * V + vv[u];
                const int64_t rstride = a.ncol * V;
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                    for (int b = 0; b < 2; ++b) {
                        const int64_t row = row0 + r;
                        x[u][2 * r + b] = (t < total && row >= a.alo && row < a.ahi)
                                              ? (Ta)vload<Tin>(p0 + r * rstride + b * V)
                                              : (Ta)0;
                    }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (t0 + u * stride >= total) break;
                const Ta I = (x[u][0] + x[u][1]) + (x[u][2] + x[u][3]) + (x[u][4] + x[u][5]);
                const Ta D[4] = {I, x[u][0] - x[u][1], x[u][2] - x[u][3], x[u][4] - x[u][5]};
                if constexpr (!FINAL) {
                    Ta *out = reinterpret_cast<Ta *>(a.f.out) + ((AA[u] - a.ya0) * a.nB + BB[u]) * 4 * a.V + vv[u];
#pragma unroll
                    for (int d = 0; d < 4; ++d) out[(int64_t)d * a.V] = D[d];
                } else {
#pragma unroll
                    for (int d = 0; d < 4; ++d) store_final(a.f, sfac, (uint64_t)(d * a.V + vv[u]), fin_val(D[d]));
                }
            }
        }
    } else {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t V = opaque(a.V);
        const int64_t v = t & (V - 1);
        const int64_t rest = t >> a.logV;
        const int64_t B = rest & (a.nB - 1);
        const int64_t A = a.A0 + (rest >> a.lognB);
        const int64_t row0 = A * R3;
        const Tin *p0 = in + ((row0 - a.xa0) * a.ncol + B * C2) * V + v;
        const int64_t rstride = a.ncol * V;
        auto ld = [&](int r1, int j, int s) -> Ta {
            const int64_t row = row0 + r1 * RL + j;
            if (row < a.alo || row >= a.ahi) return (Ta)0;
            const Tin *rp = p0 + (int64_t)(r1 * RL + j) * rstride;
            return (Ta)vload<Tin>(rp + (uint32_t)s * (uint32_t)V);
        };
        if constexpr (!FINAL) {
            Ta *out = reinterpret_cast<Ta *>(a.f.out) + ((A - a.ya0) * a.nB + B) * NOUT * V + v;
            vblock<Q, Ta>(ld, [&](int d, Ta y) { out[(int64_t)d * V] = y; });
        } else {
            vblock<Q, Ta>(ld, [&](int d, Ta y) { store_final(a.f, sfac, (uint64_t)(d * V + v), fin_val(y)); });
        }
    }
    }
}

// vfold3: three qubits per pass for int32 data with V >= 32.  Each warp owns
// tasks = (A, B, 32 consecutive v); a task's 27 x 8 input lines are 128-byte
// lines (one per lane-wide v block).  The transform streams over the top row
// digit r1, so the lines arrive as three groups of 9 rows x 8 columns (9 KB)
// through a per-warp ring of three cp.async slots: while group q computes,
// groups q+1 and q+2 are in flight, with no registers held for them.  Every
// lane then runs the r1 step on its v at compile-time shared-memory offsets
// and writes whole 128-byte lines.  (Q = 3 cuts the n = 14 step-(i) traffic
// from 223 GB (7+2+2+2+1) to 210 GB (7+3+3+1); the register-only vfold
// would need 216 runtime-strided 64-bit addresses per thread.)
#ifndef VF3_W
#define VF3_W 8
#endif
#ifndef VF3_S
#define VF3_S 3
#endif
#ifndef VF3_MINB
#define VF3_MINB 1
#endif
constexpr int VF3_WARPS = VF3_W;
constexpr int VF3_GROUP_CHUNKS = 72 * 8;  // 16-byte chunks per r1 group (72 lines x 128 B)
constexpr int VF3_SLOTS = VF3_S;

// Tin = int16_t: the low halves of a split Y1 (lines of 32 v are 64 bytes); int32 otherwise
template <bool FINAL, typename Tin = int32_t>
__global__ void __launch_bounds__(32 * VF3_WARPS, VF3_MINB) vfold3_kernel(const VArgs a) {
    constexpr int CPL = 32 * (int)sizeof(Tin) / 16;  // 16-byte chunks per line of 32 v
    extern __shared__ __align__(16) int4 vsm4[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int4 *ring = vsm4 + warp * VF3_SLOTS * VF3_GROUP_CHUNKS;
    __shared__ double sfac[FINAL ? 33 : 1];
    if constexpr (FINAL) {
        stage_factors(sfac, a.f.fac);
        __syncthreads();
    }
    const int64_t V = a.V;
    const int64_t nvb = V >> 5;
    const int64_t ntask = a.nA * a.nB * nvb;
    const Tin *in = reinterpret_cast<const Tin *>(a.in);
    const int64_t gw = (int64_t)blockIdx.x * VF3_WARPS + warp, nw = (int64_t)gridDim.x * VF3_WARPS;
    const int my_tasks = gw < ntask ? (int)((ntask - 1 - gw) / nw) + 1 : 0;
    const int nq = my_tasks * 3;

    auto task_coords = [&](int i, int64_t &A, int64_t &B, int64_t &v0) {
        const int64_t t = gw + (int64_t)i * nw;
        int64_t rest;
        if (a.logV >= 0) {
            v0 = (t & (nvb - 1)) << 5;
            rest = t >> (a.logV - 5);
        } else {  // V not a power of two (split-Y1 high-part rows): one division per task
            rest = t / nvb;
            v0 = (t - rest * nvb) << 5;
        }
        B = rest & (a.nB - 1);
        A = a.A0 + (rest >> a.lognB);
    };
    auto issue = [&](int q) {
        if (q < nq) {
            int64_t A, B, v0;
            task_coords(q / 3, A, B, v0);
            const int r1 = q % 3;
            const int64_t row0 = A * 27 + r1 * 9;
            const Tin *p0 = in + ((row0 - a.xa0) * a.ncol + B * 8) * V + v0;
            int4 *slot = ring + (q % VF3_SLOTS) * VF3_GROUP_CHUNKS;
#pragma unroll
            for (int k = 0; k < 72 * CPL / 32; ++k) {
                const int id = lane + 32 * k;
                const int L = id / CPL, c = id % CPL, j = L >> 3, s = L & 7;
                const int64_t row = row0 + j;
                const bool ok = row >= a.alo && row < a.ahi;
                cp_async16(slot + id,
                           ok ? (const void *)(p0 + (j * a.ncol + s) * V + c * (16 / (int)sizeof(Tin))) : (const void *)in,
                           ok ? 16 : 0);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

#pragma unroll
    for (int k = 0; k < VF3_SLOTS; ++k) issue(k);
    int32_t Iacc[16];
    // Keep the CTA's warps in step: one named barrier per task while every warp still has
    // one.  With int16 input a task's lines are 64-byte halves of 128-byte lines whose other
    // halves belong to the neighbouring warp's task; warps that drift apart re-fetch whole
    // lines from DRAM (n = 14: up to 2x the reads; with the barrier pass 2 reads 9.17 GB in
    // 2.17 ms instead of 2.6 ms).  int32 passes gain too (n = 14 pass 3: 1.21 -> 1.10 ms):
    // the CTA's eight tasks stay on neighbouring lines of the same rows.
    const int64_t gw_last = (int64_t)blockIdx.x * VF3_WARPS + VF3_WARPS - 1;
    const int cta_tasks = gw_last < ntask ? (int)((ntask - 1 - gw_last) / nw) + 1 : 0;
    for (int q = 0; q < nq; ++q) {
        if (q % 3 == 0 && q / 3 < cta_tasks) asm volatile("bar.sync 1, %0;" ::"n"(32 * VF3_WARPS) : "memory");
        const int r1 = q % 3;
        int64_t A, B, v0;
        task_coords(q / 3, A, B, v0);
        const int64_t v = v0 + lane;
        const int64_t orow = (A - a.ya0) * a.nB + B;
        int32_t *out = nullptr;
        if constexpr (!FINAL) out = reinterpret_cast<int32_t *>(a.f.out) + orow * 64 * V + v;
        asm volatile("cp.async.wait_group %0;" ::"n"(VF3_SLOTS - 1) : "memory");
        __syncwarp();
        const Tin *st = reinterpret_cast<const Tin *>(ring + (q % VF3_SLOTS) * VF3_GROUP_CHUNKS);
        auto x = [&](int j, int s) -> int32_t { return (int32_t)st[(j * 8 + s) * 32 + lane]; };
        auto sink = [&](int d, int32_t y) {
            if constexpr (!FINAL) {
                out[(int64_t)d * V] = y;
            } else {
                store_final(a.f, sfac, (uint64_t)(d * V + v), (int64_t)y);
            }
        };
        if (r1 == 0) {
#pragma unroll
            for (int k = 0; k < 16; ++k) Iacc[k] = 0;
        }
        int32_t w[2][16];  // [b1][D2 D3]
#pragma unroll
        for (int b1 = 0; b1 < 2; ++b1) {
            int32_t u[3][2][4];  // after qubit 3: [r2][b2][D3]
#pragma unroll
            for (int r2 = 0; r2 < 3; ++r2)
#pragma unroll
                for (int b2 = 0; b2 < 2; ++b2) {
                    const int s0 = b1 * 4 + b2 * 2;
                    q6to4<int32_t>(x(r2 * 3 + 0, s0), x(r2 * 3 + 0, s0 + 1), x(r2 * 3 + 1, s0), x(r2 * 3 + 1, s0 + 1),
                                   x(r2 * 3 + 2, s0), x(r2 * 3 + 2, s0 + 1), u[r2][b2][0], u[r2][b2][1], u[r2][b2][2],
                                   u[r2][b2][3]);
                }
#pragma unroll
            for (int d3 = 0; d3 < 4; ++d3)
                q6to4<int32_t>(u[0][0][d3], u[0][1][d3], u[1][0][d3], u[1][1][d3], u[2][0][d3], u[2][1][d3],
                               w[b1][0 * 4 + d3], w[b1][1 * 4 + d3], w[b1][2 * 4 + d3], w[b1][3 * 4 + d3]);
        }
        __syncwarp();
        issue(q + VF3_SLOTS);  // this slot's data is in registers now
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            Iacc[k] += w[0][k] + w[1][k];
            sink((r1 + 1) * 16 + k, w[0][k] - w[1][k]);
        }
        if (r1 == 2) {
#pragma unroll
            for (int k = 0; k < 16; ++k) sink(k, Iacc[k]);
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// ===========================================================================
// host-side planning
// ===========================================================================
static inline int64_t ipow(int64_t b, int e) {
    int64_t r = 1;
    while (e-- > 0) r *= b;
    return r;
}

// |values| after `done` qubits are <= shots * 3^done
static inline bool fits_i32(int64_t shots, int done) {
    double b = (double)shots;
    for (int i = 0; i < done; ++i) b *= 3.0;
    return b <= 2147483647.0;
}

struct Pass {
    int q;            // qubits consumed
    int kind;         // 0 = tile pass (pass 1), 1 = vfold
    int small;        // tile pass: packed mode
    int in_dtype;     // LRE_* of the input
    int acc64;        // vfold accumulates (and stores intermediates) in int64
    int64_t alo, ahi; // valid input rows (previous-level units)
    int64_t A0, nA;   // output row groups computed
    size_t out_bytes; // intermediate output bytes (0 for the final pass)
    size_t hi_off;    // split Y1: byte offset of the high-part plane in the output buffer
};

// byte offset of the int64 numerators a one-pass streaming stage leaves in the workspace
static inline size_t onepass_num_offset(int n) {
    size_t b = 1;
    for (int i = 0; i < n; ++i) b *= 4;
    return (b * sizeof(int32_t) + 255) & ~(size_t)255;
}

struct Plan {
    std::vector<Pass> p;
    size_t ws_bytes = 0;
    size_t off[2] = {0, 0};  // ping-pong buffers for intermediates
    int split = 0;           // split Y1 storage (below)
};

// Split Y1 storage.  Pass 1 (Q = 7) values satisfy |Y1[v]| <= shots * 3^zc(v),
// zc(v) = identity digits of the 7-qubit index v.  With shots * 27 <= 32767
// every value with zc <= 3 fits int16, so Y1 is stored as an int16 plane of
// low halves (lo, 2 B per value) plus, for the 1156 of 16384 indices per tile
// with zc >= 4, the high part hi = (y - lo) / 65536 in a compact int16 plane
// [tile][1184] (lre_y1rank.inc).  Both planes go through the same Q = 3 folds
// (linear, so lo and hi chains stay exact: lo after L levels is bounded by
// 3^L * 32768), and y1_merge_kernel recombines lo + 65536 * hi at the level
// the final pass reads.  Pass 1 writes and pass 2 reads 10.3 GB instead of
// 18.3 GB at n = 14.  Requires: rows of the record sum to shots (the same
// contract the int32 bounds rest on; lre_validate_counts checks it).
static bool split_allowed() {
    static const bool on = [] {
        const char *e = getenv("LRE_Y1SPLIT");
        const char *v = getenv("LRE_P1");
        return !(e && e[0] == '0') && !(v && (!strcmp(v, "ring") || !strcmp(v, "tma")));
    }();
    return on;
}

// first-pass width: the tile pass when it applies, else vfold from raw counts
// vfold passes consume at most two qubits: a thread then needs 36 loads
// (9 rows x 4 columns) whose 64-bit addresses still fit in registers.
constexpr int VFOLD_MAX_Q = 2;

static int first_q(int n, int64_t shots) {
    if (n >= 7 && fits_i32(shots, 7)) return 7;
    if (n >= 6 && fits_i32(shots, 6)) return 6;
    return std::min(VFOLD_MAX_Q, n);
}

Plan make_plan(int n, int64_t shots, int dtype, int64_t w_begin, int64_t w_end) {
    Plan pl;
    int done = 0;
    int64_t lo = w_begin, hi = w_end;
    const int q1 = first_q(n, shots);
    std::vector<int> qs;
    qs.push_back(q1);
    int rem = n - q1;
    int done_q = q1;
    while (rem > 0) {
        // shared-memory staged Q = 3 passes need int32 data and V = 4^done >= 32
        const bool q3 = done_q >= 3 && fits_i32(shots, done_q + 3);
        const int q = std::min(q3 ? 3 : VFOLD_MAX_Q, rem);
        qs.push_back(q);
        rem -= q;
        done_q += q;
    }
    for (size_t i = 0; i < qs.size(); ++i) {
        Pass ps{};
        ps.q = qs[i];
        ps.kind = (i == 0 && ps.q >= 6) ? 0 : 1;
        ps.small = (ps.kind == 0 && shots <= SMALL_MAX_SHOTS) ? 1 : 0;
        ps.in_dtype = i == 0 ? dtype : (pl.p[i - 1].acc64 ? LRE_I64 : LRE_I32);
        const bool last = i + 1 == qs.size();
        ps.acc64 = (ps.kind == 1 && !fits_i32(shots, done + ps.q)) ? 1 : 0;
        ps.alo = lo;
        ps.ahi = hi;
        const int64_t q3 = ipow(3, ps.q);
        ps.A0 = lo / q3;
        ps.nA = (hi + q3 - 1) / q3 - ps.A0;
        const int R = n - done;  // remaining qubits before this pass
        if (!last) {
            const int64_t nB = ipow(2, R - ps.q);
            const size_t elems = (size_t)ps.nA * (size_t)nB * (size_t)ipow(4, done + ps.q);
            ps.out_bytes = elems * (ps.kind == 0 ? 4 : (ps.acc64 ? 8 : 4));
        }
        pl.p.push_back(ps);
        lo = ps.A0;
        hi = ps.A0 + ps.nA;
        done += ps.q;
    }
    {
        const size_t np = pl.p.size();
        bool sp = split_allowed() && np >= 3 && pl.p[0].kind == 0 && pl.p[0].q == 7 && shots >= 1 &&
                  shots * 27 <= 32767 && pl.p[np - 1].in_dtype == LRE_I32;
        for (size_t i = 1; sp && i + 1 < np; ++i) sp = pl.p[i].q == 3 && !pl.p[i].acc64;
        if (sp) {
            pl.split = 1;
            for (size_t i = 0; i + 1 < np; ++i) {
                const size_t eb = i == 0 ? 2 : 4;  // int16 Y1, int32 later levels
                const size_t elems = pl.p[i].out_bytes / 4;
                pl.p[i].hi_off = (elems * eb + 255) & ~(size_t)255;
                pl.p[i].out_bytes = pl.p[i].hi_off + elems / 16384 * LRE_Y1_HROW * eb;
            }
        }
    }
    // intermediates alternate between two buffers
    size_t need[2] = {0, 0};
    for (size_t i = 0; i + 1 < pl.p.size(); ++i) need[i & 1] = std::max(need[i & 1], pl.p[i].out_bytes);
    pl.off[0] = 0;
    pl.off[1] = (need[0] + 255) & ~(size_t)255;
    pl.ws_bytes = pl.off[1] + ((need[1] + 255) & ~(size_t)255);
    // one-pass plans (n <= 2, 6, 7): int32 tile of the tile pass, then (streaming
    // form only) the int64 numerators that lre_step1_stage leaves for _finish
    if (pl.p.size() == 1) pl.ws_bytes = onepass_num_offset(n) + (size_t)ipow(4, n) * sizeof(int64_t);
    return pl;
}

static bool g_pow3_ready = false;

static bool g_disable_tma;
static int g_p1_variant = 1;  // 1 = LDG (default), 0 = cp.async ring (LRE_P1=ring), 2 = TMA (LRE_P1=tma)

static cudaError_t ensure_init() {
    if (!g_pow3_ready) {
        const char *env = getenv("LRE_P1");
        g_p1_variant = env && !strcmp(env, "ring") ? 0 : env && !strcmp(env, "tma") ? 2 : 1;
        g_disable_tma = g_p1_variant != 2;
        g_pow3_ready = true;
    }
    return cudaSuccess;
}

template <int Q, bool SMALL, typename Tin, int LOGN = 0>
static cudaError_t launch_tile(const P1Args &a, cudaStream_t s) {
    auto kern = tile_pass_kernel<Q, SMALL, Tin, LOGN>;
    if constexpr (Q == 7 && SMALL) {
        if (a.split16) kern = tile_pass_kernel<Q, SMALL, Tin, LOGN, true>;
    }
    const size_t smem = P1Smem<Q, SMALL>::TOTAL;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = a.naH * a.C;
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)num_sms() * (SMALL ? 2 : 1));  // persistent
    kern<<<(unsigned)grid, P1_THREADS, smem, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

template <int Q, int LOGN>
static cudaError_t launch_ring(const P1Args &a, cudaStream_t s) {
    auto kern = tile_ring_kernel<Q, LOGN>;
    const size_t smem = RingSmem<Q>::TOTAL;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = a.naH * a.C;
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)num_sms());
    kern<<<(unsigned)grid, RING_THREADS, smem, s>>>(a);
    count_launch();
    return cudaGetLastError();
}


template <int Q, int LOGN>
static cudaError_t launch_u16_small(const P1Args &a, cudaStream_t s) {
    if (g_p1_variant == 1) return launch_tile<Q, true, uint16_t, LOGN>(a, s);
    return launch_ring<Q, LOGN>(a, s);
}

// uint16 SMALL tiles (the benchmark format) get a compile-time row length
template <int Q>
static cudaError_t tile_u16_small(const P1Args &a, cudaStream_t s) {
    switch (a.rowlen) {
    case 1 << 7: return launch_u16_small<Q, 7>(a, s);
    case 1 << 8: return launch_u16_small<Q, 8>(a, s);
    case 1 << 9: return launch_u16_small<Q, 9>(a, s);
    case 1 << 10: return launch_u16_small<Q, 10>(a, s);
    case 1 << 11: return launch_u16_small<Q, 11>(a, s);
    case 1 << 12: return launch_u16_small<Q, 12>(a, s);
    case 1 << 13: return launch_u16_small<Q, 13>(a, s);
    case 1 << 14: return launch_u16_small<Q, 14>(a, s);
    default: return launch_u16_small<Q, 0>(a, s);
    }
}

template <int Q, bool SMALL>
static cudaError_t tile_dtype(int dtype, const P1Args &a, cudaStream_t s) {
    switch (dtype) {
    case LRE_U8: return launch_tile<Q, SMALL, uint8_t>(a, s);
    case LRE_U16:
        if constexpr (SMALL && Q == 7) return tile_u16_small<Q>(a, s);
        return launch_tile<Q, SMALL, uint16_t>(a, s);
    case LRE_I32: return launch_tile<Q, SMALL, int32_t>(a, s);
    case LRE_I64: return launch_tile<Q, SMALL, int64_t>(a, s);
    default: return cudaErrorInvalidValue;
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static cudaError_t encode_counts_map(CUtensorMap *map, const P1Args &a, int Q) {
    if (!g_encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
        if (e != cudaSuccess || qr != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const int64_t q3 = ipow(3, Q);
    const int64_t rows = (a.aH0 + a.naH) * q3 - a.row_base;  // rows held by the counts buffer
    cuuint64_t dims[2] = {(cuuint64_t)a.rowlen, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)a.rowlen * sizeof(uint16_t)};
    cuuint32_t box[2] = {64, 27};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void *>(a.counts), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int Q>
static cudaError_t launch_tma(const P1Args &a, cudaStream_t s) {
    CUtensorMap map;
    cudaError_t e = encode_counts_map(&map, a, Q);
    if (e != cudaSuccess) return e;
    auto kern = tile_tma_kernel<Q>;
    const size_t smem = TmaSmem<Q>::TOTAL;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = a.naH * a.C;
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)num_sms());
    kern<<<(unsigned)grid, TMA_THREADS, smem, s>>>(a, map);
    count_launch();
    return cudaGetLastError();
}

// pass-1 variant for uint16 SMALL tiles: LRE_P1=ldg (default) | ring | tma (A/B measurements)

static cudaError_t run_tile(int q, int small, int dtype, const P1Args &a, cudaStream_t s) {
    if (small && dtype == LRE_U16 && !g_disable_tma && (a.rowlen * 2) % 16 == 0 &&
        ((uintptr_t)a.counts & 15) == 0) {
        if (q == 7) return launch_tma<7>(a, s);
        if (q == 6) return launch_tma<6>(a, s);
    }
#ifdef LRE_ONLY_ONE
    return launch_tile<7, true, uint16_t>(a, s);
#else
    if (q == 7) return small ? tile_dtype<7, true>(dtype, a, s) : tile_dtype<7, false>(dtype, a, s);
    if (q == 6) return small ? tile_dtype<6, true>(dtype, a, s) : tile_dtype<6, false>(dtype, a, s);
    return cudaErrorInvalidValue;
#endif
}

template <int Q, typename Tin, typename Ta>
static cudaError_t launch_vfold(const VArgs &a, cudaStream_t s) {
    const int64_t total = a.nA * a.nB * a.V;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((total + 127) / 128, (int64_t)num_sms() * 16));
    if (a.f.kind == OUT_INTER) vfold_kernel<Q, Tin, Ta, false><<<(unsigned)blocks, 128, 0, s>>>(a);
    else vfold_kernel<Q, Tin, Ta, true><<<(unsigned)blocks, 128, 0, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

template <typename Tin = int32_t>
static cudaError_t launch_vfold3(const VArgs &a, cudaStream_t s) {
    const size_t smem = (size_t)VF3_WARPS * VF3_SLOTS * VF3_GROUP_CHUNKS * sizeof(int4);
    const int64_t tasks = a.nA * a.nB * (a.V >> 5);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((tasks + VF3_WARPS - 1) / VF3_WARPS,
                                                                (int64_t)num_sms() * VF3_MINB));
    cudaError_t e;
    if (a.f.kind == OUT_INTER) {
        auto kern = vfold3_kernel<false, Tin>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        kern<<<(unsigned)grid, 32 * VF3_WARPS, smem, s>>>(a);
    } else {
        if constexpr (!std::is_same<Tin, int32_t>::value) return cudaErrorInvalidValue;
        e = cudaFuncSetAttribute(vfold3_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        vfold3_kernel<true><<<(unsigned)grid, 32 * VF3_WARPS, smem, s>>>(a);
    }
    count_launch();
    return cudaGetLastError();
}

template <typename Tin, typename Ta>
static cudaError_t vfold_q(int q, const VArgs &a, cudaStream_t s) {
    switch (q) {
    case 1: return launch_vfold<1, Tin, Ta>(a, s);
    case 2: return launch_vfold<2, Tin, Ta>(a, s);
    case 3:
        if constexpr (sizeof(Tin) == 4 && sizeof(Ta) == 4) {
            if (a.V >= 32) return launch_vfold3(a, s);
        }
        return cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
    }
}

// Last fold pass (one qubit: the most significant) writing MASK_MAJOR output
// (theta[m * 2^n + a], the layout the n >= 10 assembly bulk-copies mask by
// mask).  Natural digits interleave the m and a bits, so a lane-per-element
// store would scatter 8-byte writes over 2^n-strided mask rows.  A block takes
// 1024 consecutive v (the five lowest qubits complete): (m5, a5) =
// natural_to_ma(v & 1023) covers a full 32 x 32 grid, so after staging the
// 4 x 1024 results in shared memory as [digit][m5][a5] every warp writes runs
// of 32 consecutive doubles (256 B) of one mask row.  Reads: the six
// (setting digit, outcome bit) planes of the input, 4 KB lines.
struct longlong4_pair {
    longlong2 a, b;
};
template <typename Tin, typename Ta, bool NUM>
__global__ void __launch_bounds__(256) final_mm_kernel(const VArgs a) {
    __shared__ int64_t st[4 * 32 * 33];  // exact numerators; theta = N * factor at write-out
    __shared__ double sfac[33];
    if constexpr (!NUM) stage_factors(sfac, a.f.fac);
    const Tin *in = reinterpret_cast<const Tin *>(a.in);
    const int n = a.f.n;
    const int64_t V = a.V;  // 4^(n-1)
    const int64_t nblk = V >> 10;
    const int64_t rstride = a.ncol * V;
    const int vb = 4 * threadIdx.x;
    // Block loads, software-pipelined: block blk + gridDim.x's planes are requested before
    // this block's write-out.  Four consecutive v per thread: one 16-byte (int32) or two
    // (int64) loads per plane.
    using L = typename std::conditional<sizeof(Tin) == 4, int4, longlong4_pair>::type;
    L ld[6];
    // Split Y1 (make_plan): a block's 1024 v hold 16 whole 7-digit u blocks, whose high
    // parts sit at the consecutive compact positions [P0, P1) of every plane row
    // (lre_y1rank.inc, at most 376): thread t loads the six planes' high parts of
    // exceptions P0 + t and P0 + t + 256 (coalesced across threads) with the planes.
    int hx[2][6];
    int hw[2];  // block-local v of this thread's exceptions, or -1
    auto load = [&](int64_t blk) {
        const int64_t v0 = blk << 10;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            const int r = i >> 1, b = i & 1;
            const bool ok = blk < nblk && r >= a.alo && r < a.ahi;
            const Tin *p = in + ((int64_t)r - a.xa0) * rstride + (int64_t)b * V + v0 + vb;
            if constexpr (sizeof(Tin) == 4) {
                ld[i] = ok ? *reinterpret_cast<const int4 *>(p) : make_int4(0, 0, 0, 0);  // plain: 0.02 ms < __ldcs
            } else {
                ld[i].a = ok ? __ldcs(reinterpret_cast<const longlong2 *>(p)) : make_longlong2(0, 0);
                ld[i].b = ok ? __ldcs(reinterpret_cast<const longlong2 *>(p) + 1) : make_longlong2(0, 0);
            }
        }
        hw[0] = hw[1] = -1;
        if (a.hi && blk < nblk) {
            const int u0 = (int)((v0 & 16383) >> 6);
            const int P0 = c_y1_uoff[u0], P1 = u0 + 16 < 256 ? c_y1_uoff[u0 + 16] : LRE_Y1_EXC;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int p = P0 + (int)threadIdx.x + 256 * k;
                if (p < P1) {
                    hw[k] = (int)g_y1_exc_v[p] - (u0 << 6);
                    const int64_t hrow = (v0 >> 14) * LRE_Y1_HROW + p;
#pragma unroll
                    for (int i = 0; i < 6; ++i) {
                        const int r = i >> 1, b = i & 1;
                        hx[k][i] = (r >= a.alo && r < a.ahi)
                                       ? __ldg(a.hi + (((int64_t)r - a.xa0) * a.ncol + b) * ((V >> 14) * LRE_Y1_HROW) + hrow)
                                       : 0;
                    }
                }
            }
        }
    };
    __syncthreads();
    load(blockIdx.x);
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        uint32_t mh, ah;  // mask / a bits of qubits 2 .. n-5 (natural_to_ma of the block index)
        natural_to_ma((uint64_t)blk, mh, ah);
        Tin x[6][4];  // widened to Ta in the fold below
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            if constexpr (sizeof(Tin) == 4) {
                x[i][0] = ld[i].x;
                x[i][1] = ld[i].y;
                x[i][2] = ld[i].z;
                x[i][3] = ld[i].w;
            } else {
                x[i][0] = (Ta)ld[i].a.x;
                x[i][1] = (Ta)ld[i].a.y;
                x[i][2] = (Ta)ld[i].b.x;
                x[i][3] = (Ta)ld[i].b.y;
            }
        }
        uint32_t mt4, at4;  // qubits above the lowest of v = vb + e
        natural_to_ma((uint64_t)threadIdx.x, mt4, at4);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const Ta D[4] = {((Ta)x[0][e] + (Ta)x[1][e]) + ((Ta)x[2][e] + (Ta)x[3][e]) + ((Ta)x[4][e] + (Ta)x[5][e]),
                             (Ta)x[0][e] - (Ta)x[1][e], (Ta)x[2][e] - (Ta)x[3][e], (Ta)x[4][e] - (Ta)x[5][e]};
            // lowest qubit digit e = I, X, Y, Z -> (m, a) bits (0,0), (1,0), (1,1), (0,1)
            const uint32_t m5 = (mt4 << 1) | (uint32_t)(e == 1 || e == 2), a5 = (at4 << 1) | (uint32_t)(e >= 2);
#pragma unroll
            for (int d = 0; d < 4; ++d) st[(d * 32 + m5) * 33 + a5] = (int64_t)D[d];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            if (hw[k] < 0) continue;  // exception: numerator += 65536 * (the same fold of the high parts)
            const int *h = hx[k];
            const int64_t H[4] = {(int64_t)h[0] + h[1] + h[2] + h[3] + h[4] + h[5], (int64_t)h[0] - h[1],
                                  (int64_t)h[2] - h[3], (int64_t)h[4] - h[5]};
            uint32_t mt, at;
            natural_to_ma((uint64_t)(hw[k] >> 2), mt, at);
            const int e = hw[k] & 3;
            const uint32_t m5 = (mt << 1) | (uint32_t)(e == 1 || e == 2), a5 = (at << 1) | (uint32_t)(e >= 2);
#pragma unroll
            for (int d = 0; d < 4; ++d) st[(d * 32 + m5) * 33 + a5] += 65536 * H[d];
        }
        __syncthreads();
        load(blk + gridDim.x);  // in flight during the write-out
        // 128 rows (digit, m5) of 32 values: warp w writes rows w, w + 8, ...
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll 4
        for (int row = warp; row < 128; row += 8) {
            const int d = row >> 5, m5 = row & 31;
            const uint64_t mt = (d == 1 || d == 2), at = (d >= 2);
            const uint64_t m = (mt << (n - 1)) | ((uint64_t)mh << 5) | (uint64_t)m5;
            const uint64_t aa = (at << (n - 1)) | ((uint64_t)ah << 5) | (uint64_t)lane;
            const int64_t N = st[row * 33 + lane];
            const uint64_t pos = (mask_position(m, n, a.f.layout) << n) | aa;
            if constexpr (NUM) reinterpret_cast<int64_t *>(a.f.out)[pos] = N;
            else __stcs(reinterpret_cast<double *>(a.f.out) + pos, (double)N * sfac[n - __popcll(m | aa)]);
        }
        __syncthreads();
    }
}

template <typename Tin, typename Ta, bool NUM> static void launch_fmm_t(const VArgs &a, cudaStream_t s) {
    const int64_t nblk = a.V >> 10;
    // 64 blocks per SM (about 7 loop iterations each at n = 14): ncu sweep of blocks per SM
    // 4 / 8 / 16 / 32 / 64 / 128 / 443 -> 0.86 / 0.83 / 0.79 / 0.77 / 0.755 / 0.754 / 0.81 ms
    const unsigned grid = (unsigned)std::min<int64_t>(nblk, (int64_t)num_sms() * 64);
    final_mm_kernel<Tin, Ta, NUM><<<grid, 256, 0, s>>>(a);
}

static cudaError_t launch_final_mm(int in_dtype, int acc64, const VArgs &a, cudaStream_t s) {
    const bool num = a.f.kind == OUT_NUM;
#define LRE_FMM(TIN, TA)                                                                  \
    do {                                                                                  \
        if (num) launch_fmm_t<TIN, TA, true>(a, s);                                       \
        else launch_fmm_t<TIN, TA, false>(a, s);                                          \
    } while (0)
    if (in_dtype == LRE_I32 && acc64) LRE_FMM(int32_t, int64_t);
    else if (in_dtype == LRE_I32) LRE_FMM(int32_t, int32_t);
    else if (in_dtype == LRE_I64) LRE_FMM(int64_t, int64_t);
    else return cudaErrorInvalidValue;
#undef LRE_FMM
    count_launch();
    return cudaGetLastError();
}

static cudaError_t run_vfold(int q, int in_dtype, int acc64, const VArgs &a, cudaStream_t s) {
#ifdef LRE_ONLY_ONE
    return vfold_q<int32_t, int32_t>(q, a, s);
#endif
    if (acc64) {
        switch (in_dtype) {
        case LRE_U8: return vfold_q<uint8_t, int64_t>(q, a, s);
        case LRE_U16: return vfold_q<uint16_t, int64_t>(q, a, s);
        case LRE_I32: return vfold_q<int32_t, int64_t>(q, a, s);
        case LRE_I64: return vfold_q<int64_t, int64_t>(q, a, s);
        default: return cudaErrorInvalidValue;
        }
    }
    switch (in_dtype) {
    case LRE_U8: return vfold_q<uint8_t, int32_t>(q, a, s);
    case LRE_U16: return vfold_q<uint16_t, int32_t>(q, a, s);
    case LRE_I32: return vfold_q<int32_t, int32_t>(q, a, s);
    case LRE_I64: return vfold_q<int64_t, int32_t>(q, a, s);  // counts bounded by shots < 2^31
    default: return cudaErrorInvalidValue;
    }
}

// The final pass runs final_mm_kernel (one-qubit fold straight into the mask-major layout)
static bool final_is_mm(const Pass &ps, int layout, int n, int done) {
    return ps.q == 1 && layout_is_mask_major(layout) && ipow(4, done) >= 1024 && ps.A0 == 0 && ps.nA == 1 &&
           n - done == 1 && (ps.in_dtype == LRE_I32 || ps.in_dtype == LRE_I64);
}
static bool final_fuses_merge(const Plan &pl, size_t i, int layout, int n, int done) {
    return pl.split && i + 1 == pl.p.size() && final_is_mm(pl.p[i], layout, n, done);
}

// Split Y1 (make_plan): lo[row][v] += 65536 * hi[row][(v >> 14) * 2048 + rank(v & 16383)]
// over the exception indices, in place on the int32 level the final pass reads.
// One thread per exception: hi is read densely, lo touched at 1156 of 16384 v.
__global__ void __launch_bounds__(256) y1_merge_kernel(int32_t *__restrict__ lo, const int32_t *__restrict__ hi,
                                                       int64_t rows, int64_t V) {
    const int64_t per_row = (V >> 14) * LRE_Y1_EXC;
    const int64_t total = rows * per_row;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / per_row, rem = i - row * per_row;
        const int64_t h = rem / LRE_Y1_EXC;
        const int rk = (int)(rem - h * LRE_Y1_EXC);
        int32_t *p = lo + row * V + (h << 14) + g_y1_exc_v[rk];
        const int64_t y = (int64_t)*p + 65536 * (int64_t)hi[row * ((V >> 14) * LRE_Y1_HROW) + h * LRE_Y1_HROW + rk];
        *p = (int32_t)y;
    }
}

// Run passes [first, last) of `pl` (computed rows) with intermediates laid out
// as in `lay` (== pl for one-shot shards; the full-range plan for streaming).
static int run_passes(const Plan &pl, const Plan &lay, size_t first, size_t last, const void *counts,
                      int64_t row_base, int n, int64_t shots, void *ws, void *out, int out_kind, int layout,
                      cudaStream_t stream) {
    if (ensure_init() != cudaSuccess) return LRE_ECUDA;
    const Factors fac = make_factors(n, shots);
    int done = 0;
    for (size_t i = 0; i < first; ++i) done += pl.p[i].q;
    for (size_t i = first; i < last; ++i) {
        const Pass &ps = pl.p[i];
        const Pass &ls = lay.p[i];
        const bool fin = i + 1 == pl.p.size();
        const int R = n - done;
        Final f;
        f.kind = fin ? (out_kind == LRE_OUT_NUM_I64 ? OUT_NUM : OUT_THETA) : OUT_INTER;
        f.out = fin ? out : (void *)((char *)ws + lay.off[i & 1]);
        f.layout = layout;
        f.n = n;
        f.shots = shots;
        f.fac = fac;
        const void *in = i == 0 ? counts : (const void *)((const char *)ws + lay.off[(i - 1) & 1]);
        cudaError_t e;
        if (ps.kind == 0) {
            P1Args a;
            static const int pipe = [] {
                const char *v = getenv("LRE_P1_SYNC");
                return v && !strcmp(v, "bar") ? 0 : 1;
            }();
            a.pipe = pipe;
            a.split16 = 0;
            a.lo = a.hi = nullptr;
            if (lay.split) {
                a.split16 = 1;
                a.lo = reinterpret_cast<int16_t *>(f.out);
                a.hi = reinterpret_cast<int16_t *>((char *)f.out + ls.hi_off);
            }
            a.counts = counts;
            a.rowlen = (int64_t)1 << n;
            a.row_base = row_base;
            a.aH0 = ps.A0;
            a.naH = ps.nA;
            a.out_aH0 = fin ? 0 : ls.A0;
            a.C = ipow(2, R - ps.q);
            a.logC = R - ps.q;
            a.f = f;
            a.f.kind = OUT_INTER;
            {
                const char *dbg = getenv("LRE_P1_DEBUG");
                a.debug_no_l2 = dbg && !strcmp(dbg, "noL2");
                a.debug_no_l1 = dbg && !strcmp(dbg, "noL1");
            }
            if (fin) a.f.out = ws;  // single-pass plan: int32 tile (natural order), converted below
            e = run_tile(ps.q, ps.small, ps.in_dtype, a, stream);
            if (e == cudaSuccess && fin) {
                const int64_t count = ipow(4, n);
                const int64_t blocks = std::min<int64_t>((count + 255) / 256, (int64_t)num_sms() * 8);
                convert_kernel<int32_t><<<(unsigned)blocks, 256, 0, stream>>>(reinterpret_cast<const int32_t *>(ws), count, f);
                count_launch();
                e = cudaGetLastError();
            }
        } else {
            VArgs a;
            a.in = in;
            a.V = ipow(4, done);
            a.ncol = ipow(2, R);
            a.xa0 = i == 0 ? row_base : ls.alo;
            a.alo = ps.alo;
            a.ahi = ps.ahi;
            a.A0 = ps.A0;
            a.nA = ps.nA;
            a.ya0 = fin ? 0 : ls.A0;
            a.nB = ipow(2, R - ps.q);
            a.logV = 2 * done;
            a.lognB = R - ps.q;
            static const int vf1 = [] {
                const char *v = getenv("LRE_VF1");
                return v && v[0] == '0' ? 0 : 1;
            }();
            a.vf1_batch = vf1;
            a.f = f;
            const bool fmm = fin && final_is_mm(ps, layout, n, done);
            a.hi = nullptr;
            if (fmm && lay.split)  // merge of the split high parts fused into the final pass
                a.hi = reinterpret_cast<const int32_t *>((const char *)in + lay.p[i - 1].hi_off);
            if (lay.split && !fin) {
                // lo plane (int16 Y1 at pass 2), then the hi plane: V / 16384 * 1184 lanes per row
                e = i == 1 ? launch_vfold3<int16_t>(a, stream) : launch_vfold3<int32_t>(a, stream);
                if (e == cudaSuccess) {
                    VArgs h = a;
                    h.in = (const char *)in + lay.p[i - 1].hi_off;
                    h.f.out = (char *)f.out + ls.hi_off;
                    h.V = a.V / 16384 * LRE_Y1_HROW;
                    h.logV = -1;  // not a power of two
                    e = i == 1 ? launch_vfold3<int16_t>(h, stream) : launch_vfold3<int32_t>(h, stream);
                }
                if (e == cudaSuccess && i + 2 == pl.p.size() && !final_fuses_merge(pl, i + 1, layout, n, done + ps.q)) {
                    const int64_t rows = ps.nA * a.nB, Vout = a.V * 64;
                    const int64_t total = rows * (Vout >> 14) * LRE_Y1_EXC;
                    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16);
                    y1_merge_kernel<<<(unsigned)blocks, 256, 0, stream>>>(
                        reinterpret_cast<int32_t *>(f.out),
                        reinterpret_cast<const int32_t *>((const char *)f.out + ls.hi_off), rows, Vout);
                    count_launch();
                    e = cudaGetLastError();
                }
            } else {
                e = fmm ? launch_final_mm(ps.in_dtype, ps.acc64, a, stream)
                        : run_vfold(ps.q, ps.in_dtype, ps.acc64, a, stream);
            }
        }
        if (e != cudaSuccess) return e == cudaErrorInvalidValue ? LRE_EUNSUPPORTED : LRE_ECUDA;
        done += ps.q;
    }
    return LRE_OK;
}

int step1_impl(const void *counts, int dtype, int n, int64_t shots, int64_t w_begin, int64_t w_end, void *ws,
               size_t ws_bytes, void *out, int out_kind, int layout, cudaStream_t stream) {
    const Plan pl = make_plan(n, shots, dtype, w_begin, w_end);
    if (ws_bytes < pl.ws_bytes || (pl.ws_bytes && !ws)) return LRE_ENOMEM;
    return run_passes(pl, pl, 0, pl.p.size(), counts, w_begin, n, shots, ws, out, out_kind, layout, stream);
}

// pass 1 of a setting chunk into the full-range workspace (streaming records).
// A one-pass plan (n <= 2, 6, 7) has a shard quantum equal to the whole
// record, so its only chunk is [0, 3^n): stage computes the exact int64
// numerators into the workspace and finish converts them.
int step1_stage_impl(const void *counts, int dtype, int n, int64_t shots, int64_t w_begin, int64_t w_end, void *ws,
                     size_t ws_bytes, cudaStream_t stream) {
    const Plan full = make_plan(n, shots, dtype, 0, ipow(3, n));
    if (ws_bytes < full.ws_bytes || !ws) return LRE_ENOMEM;
    if (full.p.size() < 2) {
        if (w_begin != 0 || w_end != ipow(3, n)) return LRE_EINVAL;
        return run_passes(full, full, 0, 1, counts, 0, n, shots, ws, (char *)ws + onepass_num_offset(n),
                          LRE_OUT_NUM_I64, LRE_LAYOUT_NATURAL, stream);
    }
    const Plan pl = make_plan(n, shots, dtype, w_begin, w_end);
    return run_passes(pl, full, 0, 1, counts, w_begin, n, shots, ws, nullptr, 0, 0, stream);
}

// passes 2.. over the full-range workspace
int step1_finish_impl(void *ws, size_t ws_bytes, int n, int64_t shots, void *out, int out_kind, int layout,
                      cudaStream_t stream) {
    // the count dtype only affects pass 1; any value gives the same later passes
    const Plan full = make_plan(n, shots, LRE_I64, 0, ipow(3, n));
    if (ws_bytes < full.ws_bytes || !ws) return LRE_ENOMEM;
    if (ensure_init() != cudaSuccess) return LRE_ECUDA;
    if (full.p.size() < 2) {
        Final f;
        f.kind = out_kind == LRE_OUT_NUM_I64 ? OUT_NUM : OUT_THETA;
        f.out = out;
        f.layout = layout;
        f.n = n;
        f.shots = shots;
        f.fac = make_factors(n, shots);
        const int64_t count = ipow(4, n);
        const int64_t blocks = std::min<int64_t>((count + 255) / 256, (int64_t)num_sms() * 8);
        convert_kernel<int64_t><<<(unsigned)blocks, 256, 0, stream>>>(
            reinterpret_cast<const int64_t *>((const char *)ws + onepass_num_offset(n)), count, f);
        count_launch();
        return cudaGetLastError() == cudaSuccess ? LRE_OK : LRE_ECUDA;
    }
    return run_passes(full, full, 1, full.p.size(), nullptr, 0, n, shots, ws, out, out_kind, layout, stream);
}

int step1_num_passes(int n, int64_t shots) { return (int)make_plan(n, shots, LRE_I64, 0, ipow(3, n)).p.size(); }

size_t step1_workspace(int n, int64_t shots, int64_t w_begin, int64_t w_end) {
    return make_plan(n, shots, LRE_I64, w_begin, w_end).ws_bytes;
}

// setting shards must align to the first pass's row groups; 3^min(n,7) works
// for every plan (3^q1 divides it)
int64_t shard_quantum(int n, int64_t /*shots*/) { return ipow(3, std::min(n, 7)); }

// ===========================================================================
// step (i) from fp64 frequencies (the reference's source protocol,
// pipeline.py:42-59,84: any object with .frequencies(a, b); ExactFrequencies)
// ===========================================================================
// The same separable A^{(x)n} map in fp64: 2-qubit vfold passes (a final
// 1-qubit pass for odd n).  Records of fp64 frequencies (8 B per entry, 627 GB
// at n = 14) only ever exist chunk by chunk: lre_step1_f64_stage runs the
// first s <= 3 passes of a chunk (its intermediates in `scratch`), the last of
// them writing into the full-range level-s buffer of the workspace;
// lre_step1_f64_finish runs the remaining passes.  theta = N * 2^{-n/2} / 3^zc
// (make_factors with shots = 1: the frequencies are already normalised).
struct F64Plan {
    std::vector<int> q;  // qubits per pass
    int staged = 0;      // passes run per chunk
    int64_t quantum = 1; // chunk alignment (settings)
    size_t ws_off[2] = {0, 0}, ws_bytes = 0;
};

static F64Plan f64_plan(int n) {
    F64Plan pl;
    int rem = n;
    while (rem > 0) {
        const int q = rem >= 2 ? 2 : 1;
        pl.q.push_back(q);
        rem -= q;
    }
    const int P = (int)pl.q.size();
    pl.staged = P == 1 ? 0 : std::min(3, P - 1);
    int S = 0;
    for (int i = 0; i < pl.staged; ++i) S += pl.q[i];
    pl.quantum = ipow(3, S);
    // full-range levels s .. P-1 ping-pong in two buffers (level l: 6^(n-S_l) 4^S_l doubles)
    size_t need[2] = {0, 0};
    int done = S;
    for (int p = pl.staged; p < P; ++p) {
        const size_t lvl = (size_t)ipow(6, n - done) * (size_t)ipow(4, done) * sizeof(double);
        need[(p - pl.staged) & 1] = std::max(need[(p - pl.staged) & 1], lvl);
        done += pl.q[p];
    }
    pl.ws_off[0] = 0;
    pl.ws_off[1] = (need[0] + 255) & ~(size_t)255;
    pl.ws_bytes = pl.ws_off[1] + ((need[1] + 255) & ~(size_t)255);
    return pl;
}

// chunk-local scratch for the first staged passes of a chunk of `rows` settings
static size_t f64_scratch_bytes(const F64Plan &pl, int n, int64_t rows) {
    size_t off = 0;
    int done = 0;
    int64_t r = rows;
    for (int p = 0; p + 1 < pl.staged; ++p) {
        done += pl.q[p];
        r = (r + ipow(3, pl.q[p]) - 1) / ipow(3, pl.q[p]);
        off += (((size_t)r * (size_t)ipow(2, n - done) * (size_t)ipow(4, done) * sizeof(double)) + 255) & ~(size_t)255;
    }
    return off;
}

static cudaError_t f64_pass(int q, const VArgs &a, bool fin, cudaStream_t s) {
    const int64_t total = a.nA * a.nB * a.V;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((total + 127) / 128, (int64_t)num_sms() * 16));
    if (q == 2) {
        if (fin) vfold_kernel<2, double, double, true><<<(unsigned)blocks, 128, 0, s>>>(a);
        else vfold_kernel<2, double, double, false><<<(unsigned)blocks, 128, 0, s>>>(a);
    } else {
        if (fin) vfold_kernel<1, double, double, true><<<(unsigned)blocks, 128, 0, s>>>(a);
        else vfold_kernel<1, double, double, false><<<(unsigned)blocks, 128, 0, s>>>(a);
    }
    count_launch();
    return cudaGetLastError();
}

static VArgs f64_args(int n, int done, int q, const void *in, int64_t xa0, int64_t alo, int64_t ahi, void *out,
                      int64_t ya0, const Final &f) {
    VArgs a;
    a.in = in;
    a.V = ipow(4, done);
    a.ncol = ipow(2, n - done);
    a.xa0 = xa0;
    a.alo = alo;
    a.ahi = ahi;
    const int64_t q3 = ipow(3, q);
    a.A0 = alo / q3;
    a.nA = (ahi + q3 - 1) / q3 - a.A0;
    a.ya0 = ya0;
    a.nB = ipow(2, n - done - q);
    a.logV = 2 * done;
    a.lognB = n - done - q;
    a.vf1_batch = 1;
    a.f = f;
    a.f.out = out;
    return a;
}

size_t step1_f64_workspace(int n) { return f64_plan(n).ws_bytes; }
size_t step1_f64_scratch(int n, int64_t rows) { return f64_scratch_bytes(f64_plan(n), n, rows); }
int64_t step1_f64_quantum(int n) { return f64_plan(n).quantum; }

int step1_f64_stage_impl(const double *freq, int n, int64_t w_begin, int64_t w_end, void *ws, size_t ws_bytes,
                         void *scratch, size_t scratch_bytes, cudaStream_t stream) {
    const F64Plan pl = f64_plan(n);
    if (ensure_init() != cudaSuccess) return LRE_ECUDA;
    if (ws_bytes < pl.ws_bytes || !ws) return LRE_ENOMEM;
    if (scratch_bytes < f64_scratch_bytes(pl, n, w_end - w_begin)) return LRE_ENOMEM;
    const int64_t settings = ipow(3, n);
    if (w_begin % pl.quantum || (w_end % pl.quantum && w_end != settings)) return LRE_EINVAL;
    if (pl.staged == 0) {  // n <= 2: the whole record is level 0 of the workspace
        if (cudaMemcpyAsync((char *)ws + pl.ws_off[0] + (size_t)w_begin * ((size_t)1 << n) * sizeof(double), freq,
                            (size_t)(w_end - w_begin) * ((size_t)1 << n) * sizeof(double), cudaMemcpyDeviceToDevice,
                            stream) != cudaSuccess)
            return LRE_ECUDA;
        return LRE_OK;
    }
    Final f{};
    f.kind = OUT_INTER;
    f.n = n;
    int done = 0;
    int64_t lo = w_begin, hi = w_end;
    const void *in = freq;
    int64_t xa0 = w_begin;
    size_t soff = 0;
    for (int p = 0; p < pl.staged; ++p) {
        const int q = pl.q[p];
        const bool last = p + 1 == pl.staged;
        const int64_t q3 = ipow(3, q);
        const int64_t A0 = lo / q3, A1 = (hi + q3 - 1) / q3;
        void *out;
        int64_t ya0;
        if (last) {
            out = (char *)ws + pl.ws_off[0];
            ya0 = 0;
        } else {
            out = (char *)scratch + soff;
            ya0 = A0;
            soff += (((size_t)(A1 - A0) * (size_t)ipow(2, n - done - q) * (size_t)ipow(4, done + q) * sizeof(double)) +
                     255) & ~(size_t)255;
        }
        const VArgs a = f64_args(n, done, q, in, xa0, lo, hi, out, ya0, f);
        if (f64_pass(q, a, false, stream) != cudaSuccess) return LRE_ECUDA;
        in = out;
        xa0 = ya0;
        lo = A0;
        hi = A1;
        done += q;
    }
    return LRE_OK;
}

int step1_f64_finish_impl(void *ws, size_t ws_bytes, int n, double *theta, int layout, cudaStream_t stream) {
    const F64Plan pl = f64_plan(n);
    if (ensure_init() != cudaSuccess) return LRE_ECUDA;
    if (ws_bytes < pl.ws_bytes || !ws) return LRE_ENOMEM;
    const int P = (int)pl.q.size();
    int done = 0;
    for (int p = 0; p < pl.staged; ++p) done += pl.q[p];
    Final f{};
    f.n = n;
    f.layout = layout;
    f.shots = 1;
    f.fac = make_factors(n, 1);
    for (int p = pl.staged; p < P; ++p) {
        const int q = pl.q[p];
        const bool fin = p + 1 == P;
        const void *in = (const char *)ws + pl.ws_off[(p - pl.staged) & 1];
        void *out = fin ? (void *)theta : (void *)((char *)ws + pl.ws_off[(p - pl.staged + 1) & 1]);
        f.kind = fin ? OUT_THETA : OUT_INTER;
        const int64_t rows = ipow(3, n - done);
        const VArgs a = f64_args(n, done, q, in, 0, 0, rows, out, 0, f);
        if (f64_pass(q, a, fin, stream) != cudaSuccess) return LRE_ECUDA;
        done += q;
    }
    return LRE_OK;
}

}  // namespace lre
