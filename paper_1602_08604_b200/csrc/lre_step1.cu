// Step (i) of the LRE hot path on B200: counts (3^n x 2^n) -> theta (4^n).
//
// Reference: pipeline.py:116-138 (step_one_least_squares), _kernels.py:34-56
// (accumulate_fast: per-setting WHT + scatter) and pauli.py:153-209 (support
// locations, Gram diagonal).
//
// B200 design: step (i) is the tensor map A^{(x)n} on the
// 6^n count tensor, A = the per-qubit 6->4 map (rows X,Y,Z x outcome bit ->
// Pauli digit).  It is evaluated in "fold passes"; a pass consumes the Q
// lowest-stride qubits of its input
//     X[P][3^h][3^Q][2^h][2^Q]  (row-major)
// and writes
//     Y[4^Q][P][3^h][2^h]
// so the next pass again finds its qubits at the lowest strides, and after
// the last pass Y is theta in natural order.  One CTA owns one tile
// (3^Q rows x 2^Q contiguous columns; TPC tiles for small Q) and keeps all
// 4^Q partial sums on chip while streaming the tile from HBM once:
//   Phase A   each thread reduces 3 qubits fully in registers
//             (27 rows x 8 contiguous columns -> 64 values, int32, exact);
//   Phase A2  Walsh-Hadamard butterfly over the tile's column-group bits in
//             shared memory;
//   Phase B   each warp folds the staged row-block digits for one butterfly
//             index t and emits final values (or accumulates the phase digit
//             in shared memory).
// All arithmetic is exact integer arithmetic; the only rounding is the final
// fp64 epilogue theta = N / shots * 2^{-n/2} / 3^{zc}.
#include <algorithm>
#include <cmath>
#include <vector>

#include "lre_internal.cuh"

namespace lre {

__constant__ double c_pow3[33];

struct PassGeom {
    int64_t P;       // finished-digit groups (4^{qubits done})
    int64_t C;       // column blocks (2^h)
    int64_t alo;     // valid input a-range [alo, ahi) within 3^{h+Q}
    int64_t ahi;
    int64_t aloH;    // a_H range of the tiles this launch computes
    int64_t nH;      // number of a_H values computed
    int64_t aHout0;  // a_H of the first row group held by the output buffer
    int64_t nHout;   // number of a_H row groups held by the output buffer
    int64_t RCout;   // P * nHout * C : stride between output slots
    int64_t ntiles;  // P * nH * C
    int64_t rowlen;  // C * 2^Q elements
    int Q;
    int final_pass;
    int out_kind;    // LRE_OUT_*
    int layout;      // LRE_LAYOUT_*
    int n;
    int64_t shots;
    double scale;    // 2^{-n/2}
};

// ---------------------------------------------------------------------------
// epilogue: intermediate store or finished theta / numerators
// ---------------------------------------------------------------------------
// output position of tile t inside one output slot
__device__ __forceinline__ int64_t tile_out_base(const PassGeom &g, int64_t t) {
    const int64_t c = t % g.C;
    const int64_t rest = t / g.C;
    const int64_t aH = g.aloH + rest % g.nH;
    const int64_t p = rest / g.nH;
    return (p * g.nHout + (aH - g.aHout0)) * g.C + c;
}

template <typename Ta>
__device__ __forceinline__ void emit(void *__restrict__ out, const PassGeom &g, int64_t slot, int64_t ob, Ta v) {
    const int64_t idx = slot * g.RCout + ob;
    if (!g.final_pass) {
        reinterpret_cast<Ta *>(out)[idx] = v;
        return;
    }
    uint32_t m, a;
    natural_to_ma((uint64_t)idx, m, a);
    const uint64_t pos = g.layout == LRE_LAYOUT_MASK_MAJOR ? (((uint64_t)m << g.n) | a) : (uint64_t)idx;
    if (g.out_kind == LRE_OUT_NUM_I64) {
        reinterpret_cast<int64_t *>(out)[pos] = (int64_t)v;
    } else {
        const int zc = g.n - __popc(m | a);
        reinterpret_cast<double *>(out)[pos] = ((double)v / (double)g.shots) * g.scale / c_pow3[zc];
    }
}

// ---------------------------------------------------------------------------
// in-thread transform of 3 qubits: 27 rows x 8 contiguous columns -> 64
// values indexed d = d1*16 + d2*4 + d3 (local qubit order, first = slowest
// row digit = most significant column bit).  `sink(off, v[16])` receives the
// 16 values with first digit d1 = off/16 as soon as they are final.
// ---------------------------------------------------------------------------
template <typename Tin, typename Ts, typename RowPtr, typename Sink>
__device__ __forceinline__ void transform3(RowPtr rowptr, int64_t col0, Sink sink) {
    Ts accI[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) accI[i] = 0;
#pragma unroll
    for (int a1 = 0; a1 < 3; ++a1) {
        Ts x[9][8];
#pragma unroll
        for (int r = 0; r < 9; ++r) {
            const Tin *p = rowptr(a1 * 9 + r);
            if (p) {
                load8<Ts>(p + col0, x[r]);
            } else {
#pragma unroll
                for (int c = 0; c < 8; ++c) x[r][c] = 0;
            }
        }
        Ts y[3][4][4];  // [a2][b1 b2][d3]
#pragma unroll
        for (int a2 = 0; a2 < 3; ++a2)
#pragma unroll
            for (int bb = 0; bb < 4; ++bb)
                q6to4<Ts>(x[a2 * 3 + 0][2 * bb], x[a2 * 3 + 0][2 * bb + 1], x[a2 * 3 + 1][2 * bb],
                          x[a2 * 3 + 1][2 * bb + 1], x[a2 * 3 + 2][2 * bb], x[a2 * 3 + 2][2 * bb + 1],
                          y[a2][bb][0], y[a2][bb][1], y[a2][bb][2], y[a2][bb][3]);
        Ts z[2][4][4];  // [b1][d2][d3]
#pragma unroll
        for (int b1 = 0; b1 < 2; ++b1)
#pragma unroll
            for (int d3 = 0; d3 < 4; ++d3)
                q6to4<Ts>(y[0][2 * b1][d3], y[0][2 * b1 + 1][d3], y[1][2 * b1][d3], y[1][2 * b1 + 1][d3],
                          y[2][2 * b1][d3], y[2][2 * b1 + 1][d3], z[b1][0][d3], z[b1][1][d3], z[b1][2][d3],
                          z[b1][3][d3]);
        Ts v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const Ts s0 = z[0][k >> 2][k & 3], s1 = z[1][k >> 2][k & 3];
            accI[k] += s0 + s1;
            v[k] = s0 - s1;
        }
        sink((a1 + 1) * 16, v);
    }
    sink(0, accI);
}

// 2 qubits: 9 rows x 4 columns -> 16 values (d1*4 + d2)
template <typename Tin, typename Ts, typename RowPtr>
__device__ __forceinline__ void transform2(RowPtr rowptr, int64_t col0, Ts out[16]) {
    Ts x[9][4];
#pragma unroll
    for (int r = 0; r < 9; ++r) {
        const Tin *p = rowptr(r);
#pragma unroll
        for (int c = 0; c < 4; ++c) x[r][c] = p ? (Ts)load1<Tin>(p + col0 + c) : (Ts)0;
    }
    Ts y[3][2][4];  // [a1][b1][d2]
#pragma unroll
    for (int a1 = 0; a1 < 3; ++a1)
#pragma unroll
        for (int b1 = 0; b1 < 2; ++b1)
            q6to4<Ts>(x[a1 * 3 + 0][2 * b1], x[a1 * 3 + 0][2 * b1 + 1], x[a1 * 3 + 1][2 * b1],
                      x[a1 * 3 + 1][2 * b1 + 1], x[a1 * 3 + 2][2 * b1], x[a1 * 3 + 2][2 * b1 + 1],
                      y[a1][b1][0], y[a1][b1][1], y[a1][b1][2], y[a1][b1][3]);
#pragma unroll
    for (int d2 = 0; d2 < 4; ++d2)
        q6to4<Ts>(y[0][0][d2], y[0][1][d2], y[1][0][d2], y[1][1][d2], y[2][0][d2], y[2][1][d2], out[0 * 4 + d2],
                  out[1 * 4 + d2], out[2 * 4 + d2], out[3 * 4 + d2]);
}

// 1 qubit: 3 rows x 2 columns -> 4 values
template <typename Tin, typename Ts, typename RowPtr>
__device__ __forceinline__ void transform1(RowPtr rowptr, int64_t col0, Ts out[4]) {
    Ts x[3][2];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const Tin *p = rowptr(r);
        x[r][0] = p ? (Ts)load1<Tin>(p + col0) : (Ts)0;
        x[r][1] = p ? (Ts)load1<Tin>(p + col0 + 1) : (Ts)0;
    }
    q6to4<Ts>(x[0][0], x[0][1], x[1][0], x[1][1], x[2][0], x[2][1], out[0], out[1], out[2], out[3]);
}

// ---------------------------------------------------------------------------
// compile-time fold over QS staged ternary digits for butterfly pattern TS
// (bit QS-1 of TS = first staged digit).  Digits with t=0 are summed (I),
// digits with t=1 are kept (X/Y/Z).  out has 3^popc(TS) entries ordered by
// the kept digits, first staged digit most significant.
// ---------------------------------------------------------------------------
template <int QS, int TS> struct Fold {
    static constexpr int OUT = pow3(popc_c(TS));
    template <typename Ts, typename Ta> __device__ __forceinline__ static void run(const Ts *x, Ta *out) {
        constexpr int TOP = (TS >> (QS - 1)) & 1;
        constexpr int REST = TS & ((1 << (QS - 1)) - 1);
        constexpr int SUB = pow3(QS - 1);
        if constexpr (TOP) {
#pragma unroll
            for (int a = 0; a < 3; ++a) Fold<QS - 1, REST>::run(x + a * SUB, out + a * Fold<QS - 1, REST>::OUT);
        } else {
            Ta s[SUB];
#pragma unroll
            for (int i = 0; i < SUB; ++i) s[i] = (Ta)x[i] + (Ta)x[SUB + i] + (Ta)x[2 * SUB + i];
            Fold<QS - 1, REST>::template run<Ta, Ta>(s, out);
        }
    }
};
template <int TS> struct Fold<0, TS> {
    static constexpr int OUT = 1;
    template <typename Ts, typename Ta> __device__ __forceinline__ static void run(const Ts *x, Ta *out) {
        out[0] = (Ta)x[0];
    }
};

// base-4 staged-digit number of fold output j for pattern TS
template <int QS, int TS> __host__ __device__ constexpr int fold_slot(int j) {
    int d = 0, rem = j, kept = popc_c(TS);
    int div = pow3(kept - 1 < 0 ? 0 : kept - 1);
    for (int k = QS - 1; k >= 0; --k) {  // from first staged digit
        int digit = 0;
        if ((TS >> k) & 1) {
            digit = rem / div + 1;
            rem %= div;
            div = div / 3 > 0 ? div / 3 : 1;
        }
        d = d * 4 + digit;
    }
    return d;
}

// ---------------------------------------------------------------------------
// the fold-pass kernel (Q = 4..7)
// ---------------------------------------------------------------------------
template <int Q, typename Ts> struct FoldCfg {
    static constexpr int QS = (Q - 3 < 3) ? Q - 3 : 3;
    static constexpr int QP = Q - 3 - QS;  // 0 or 1
    static constexpr int NRB = pow3(QS);
    static constexpr int NCG = 1 << (QP + QS);
    static constexpr int NA_MAX = sizeof(Ts) == 4 ? 432 : 216;
    static constexpr int TPC = (NA_MAX / (NRB * NCG)) < 1 ? 1 : NA_MAX / (NRB * NCG);
    static constexpr int NA = TPC * NRB * NCG;
    static constexpr int SP = 68;  // staging record stride in elements (64 + pad)
    static constexpr int THREADS = 512;
    static constexpr int NWARPS = THREADS / 32;
    static constexpr int NPAIRS = TPC * NCG;
    static constexpr size_t STAGE_BYTES = (size_t)NA * SP * sizeof(Ts);
    static_assert(NA <= THREADS, "phase A needs one thread per work item");
    static_assert(QP == 0 || NPAIRS == NWARPS, "phase digits need one pair per warp");
};

template <int QS, int TS, int QP, typename Ts, typename Ta>
__device__ __forceinline__ void phaseB_pair(const Ts *v0, const Ts *v1, void *out, const PassGeom &g, int64_t ob,
                                            int tP, int round, int lane, Ta *O) {
    constexpr int OUT = Fold<QS, TS>::OUT;
    Ta o0[OUT], o1[OUT];
    Fold<QS, TS>::template run<Ts, Ta>(v0, o0);
    Fold<QS, TS>::template run<Ts, Ta>(v1, o1);
    const int di = 2 * lane;
#pragma unroll
    for (int j = 0; j < OUT; ++j) {
        const int dS = fold_slot<QS, TS>(j);
        if (QP == 0 || tP) {
            const int dP = QP == 0 ? 0 : round + 1;  // phase digit: X/Y/Z = round + 1
            const int64_t slot = ((int64_t)dP * (1 << (2 * QS)) + dS) * 64 + di;
            emit<Ta>(out, g, slot, ob, o0[j]);
            emit<Ta>(out, g, slot + 1, ob, o1[j]);
        } else {
            O[dS * 64 + di] += o0[j];
            O[dS * 64 + di + 1] += o1[j];
        }
    }
}

template <int Q, typename Tin, typename Ts, typename Ta>
__global__ void __launch_bounds__(512, 1)
    fold_pass_kernel(const Tin *__restrict__ in, void *__restrict__ out, const PassGeom g) {
    using Cfg = FoldCfg<Q, Ts>;
    constexpr int QS = Cfg::QS, QP = Cfg::QP, NRB = Cfg::NRB, NCG = Cfg::NCG, TPC = Cfg::TPC, SP = Cfg::SP;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Ts *S = reinterpret_cast<Ts *>(smem_raw);
    Ta *O = reinterpret_cast<Ta *>(smem_raw + Cfg::STAGE_BYTES);  // phase-digit accumulators (QP=1)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tile0 = (int64_t)blockIdx.x * TPC;

    if (QP > 0) {
        for (int i = tid; i < (1 << (2 * (Q - 1))); i += Cfg::THREADS) O[i] = 0;
    }

    // phase-A identity of this thread
    const int ta = tid;
    const int cg = ta % NCG;
    const int tl = (ta / NCG) % TPC;
    const int rb = ta / (NCG * TPC);
    const int64_t tA = tile0 + tl;
    const bool activeA = ta < Cfg::NA && tA < g.ntiles;
    int64_t p = 0, aH = 0, c = 0;
    if (activeA) {
        c = tA % g.C;
        const int64_t rest = tA / g.C;
        aH = g.aloH + rest % g.nH;
        p = rest / g.nH;
    }
    const int64_t span = g.ahi - g.alo;
    const Tin *base = in + p * span * g.rowlen;
    const int64_t col0 = c * ((int64_t)1 << Q) + cg * 8;

#pragma unroll 1
    for (int round = 0; round < pow3(QP); ++round) {
        // ---------------- phase A ----------------
        if (activeA) {
            const int64_t a0 = aH * pow3(Q) + ((int64_t)round * NRB + rb) * 27;
            auto rowptr = [&](int j) -> const Tin * {
                const int64_t a = a0 + j;
                return (a >= g.alo && a < g.ahi) ? base + (a - g.alo) * g.rowlen : nullptr;
            };
            Ts *rec = S + (size_t)ta * SP;
            transform3<Tin, Ts>(rowptr, col0, [&](int off, const Ts *v) {
#pragma unroll
                for (int k = 0; k < 16; k += 4) {
                    if constexpr (sizeof(Ts) == 4) {
                        *reinterpret_cast<int4 *>(rec + off + k) = make_int4(v[k], v[k + 1], v[k + 2], v[k + 3]);
                    } else {
                        *reinterpret_cast<longlong2 *>(rec + off + k) = make_longlong2(v[k], v[k + 1]);
                        *reinterpret_cast<longlong2 *>(rec + off + k + 2) = make_longlong2(v[k + 2], v[k + 3]);
                    }
                }
            });
        }
        __syncthreads();
        // ---------------- phase A2: butterfly over the NCG column groups ----------------
        for (int it = tid; it < 16 * NRB * TPC; it += Cfg::THREADS) {
            const int q = it & 15, rt = it >> 4;
            Ts w[NCG][4];
#pragma unroll
            for (int k = 0; k < NCG; ++k) {
                const Ts *src = S + ((size_t)rt * NCG + k) * SP + 4 * q;
#pragma unroll
                for (int e = 0; e < 4; ++e) w[k][e] = src[e];
            }
#pragma unroll
            for (int h = 1; h < NCG; h <<= 1)
#pragma unroll
                for (int k = 0; k < NCG; ++k)
                    if (!(k & h)) {
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const Ts u = w[k][e], v = w[k + h][e];
                            w[k][e] = u + v;
                            w[k + h][e] = u - v;
                        }
                    }
#pragma unroll
            for (int k = 0; k < NCG; ++k) {
                Ts *dst = S + ((size_t)rt * NCG + k) * SP + 4 * q;
#pragma unroll
                for (int e = 0; e < 4; ++e) dst[e] = w[k][e];
            }
        }
        __syncthreads();
        // ---------------- phase B: fold staged digits per butterfly index ----------------
        for (int pair = warp; pair < Cfg::NPAIRS; pair += Cfg::NWARPS) {
            const int tl2 = pair / NCG, to = pair % NCG;
            const int64_t t = tile0 + tl2;
            if (t >= g.ntiles) continue;
            const int64_t ob = tile_out_base(g, t);
            const int tP = to >> QS;
            const int TS = to & ((1 << QS) - 1);
            Ts v0[NRB], v1[NRB];
#pragma unroll
            for (int r = 0; r < NRB; ++r) {
                const Ts *src = S + ((size_t)(r * TPC + tl2) * NCG + to) * SP + 2 * lane;
                v0[r] = src[0];
                v1[r] = src[1];
            }
            switch (TS) {
#define LRE_CASE(X)                                                                                      \
    case X:                                                                                              \
        if constexpr (X < (1 << QS)) phaseB_pair<QS, X, QP, Ts, Ta>(v0, v1, out, g, ob, tP, round, lane, O); \
        break;
                LRE_CASE(0)
                LRE_CASE(1)
                LRE_CASE(2)
                LRE_CASE(3)
                LRE_CASE(4)
                LRE_CASE(5)
                LRE_CASE(6)
                LRE_CASE(7)
#undef LRE_CASE
            default: break;
            }
        }
        __syncthreads();
    }
    if (QP > 0 && tile0 < g.ntiles) {  // flush the d1 = I slots accumulated across rounds
        const int64_t ob = tile_out_base(g, tile0);
        for (int i = tid; i < (1 << (2 * (Q - 1))); i += Cfg::THREADS) emit<Ta>(out, g, i, ob, O[i]);
    }
}

// ---------------------------------------------------------------------------
// small passes (Q <= 3): one thread per tile, everything in registers
// ---------------------------------------------------------------------------
template <int Q, typename Tin, typename Ta>
__global__ void __launch_bounds__(128) small_pass_kernel(const Tin *__restrict__ in, void *__restrict__ out,
                                                          const PassGeom g) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= g.ntiles) return;
    const int64_t c = t % g.C;
    const int64_t rest = t / g.C;
    const int64_t aH = g.aloH + rest % g.nH;
    const int64_t p = rest / g.nH;
    const int64_t span = g.ahi - g.alo;
    const Tin *base = in + p * span * g.rowlen;
    const int64_t a0 = aH * pow3(Q);
    auto rowptr = [&](int j) -> const Tin * {
        const int64_t a = a0 + j;
        return (a >= g.alo && a < g.ahi) ? base + (a - g.alo) * g.rowlen : nullptr;
    };
    const int64_t col0 = c << Q;
    const int64_t ob = tile_out_base(g, t);
    if constexpr (Q == 3) {
        transform3<Tin, Ta>(rowptr, col0, [&](int off, const Ta *v) {
#pragma unroll
            for (int k = 0; k < 16; ++k) emit<Ta>(out, g, off + k, ob, v[k]);
        });
    } else if constexpr (Q == 2) {
        Ta v[16];
        transform2<Tin, Ta>(rowptr, col0, v);
#pragma unroll
        for (int k = 0; k < 16; ++k) emit<Ta>(out, g, k, ob, v[k]);
    } else {
        Ta v[4];
        transform1<Tin, Ta>(rowptr, col0, v);
#pragma unroll
        for (int k = 0; k < 4; ++k) emit<Ta>(out, g, k, ob, v[k]);
    }
}

// ---------------------------------------------------------------------------
// host-side planning
// ---------------------------------------------------------------------------
static inline int64_t ipow(int64_t b, int e) {
    int64_t r = 1;
    while (e-- > 0) r *= b;
    return r;
}

// largest |value| after processing `done` qubits is shots * 3^done
static inline bool fits_i32(int64_t shots, int done) {
    double b = (double)shots;
    for (int i = 0; i < done; ++i) b *= 3.0;
    return b < 2147483647.0;
}

std::vector<int> plan_passes(int n, int64_t shots) {
    std::vector<int> q;
    if (n <= 7) {
        q.push_back(n);
    } else {
        const int k = (n + 6) / 7;
        const int base = n / k, extra = n % k;
        for (int i = 0; i < k; ++i) q.push_back(base + (i < extra ? 1 : 0));
    }
    // Q=7 passes need int32 staging (shots * 3^{done+3} < 2^31); otherwise split
    std::vector<int> out;
    int done = 0;
    for (size_t i = 0; i < q.size(); ++i) {
        int qi = q[i];
        if (qi == 7 && !fits_i32(shots, done + 3)) {
            out.push_back(6);
            done += 6;
            if (i + 1 < q.size()) q[i + 1] += 1;
            else q.push_back(1);
            continue;
        }
        out.push_back(qi);
        done += qi;
    }
    return out;
}

struct PassPlan {
    std::vector<int> q;
    std::vector<int64_t> alo, ahi;   // valid input a-range per pass
    std::vector<size_t> out_bytes;   // intermediate output bytes (non-final)
    std::vector<int> acc64;          // accumulate in int64
    std::vector<int> stage64;        // stage in int64
    size_t ws_bytes = 0;
};

PassPlan make_plan(int n, int64_t shots, int64_t w_begin, int64_t w_end) {
    PassPlan pl;
    pl.q = plan_passes(n, shots);
    int done = 0;
    int64_t lo = w_begin, hi = w_end;
    size_t ws = 0;
    for (size_t i = 0; i < pl.q.size(); ++i) {
        const int Q = pl.q[i];
        const int h = n - done - Q;
        pl.alo.push_back(lo);
        pl.ahi.push_back(hi);
        const int64_t q3 = ipow(3, Q);
        const int64_t loH = lo / q3, hiH = (hi + q3 - 1) / q3;
        const bool last = i + 1 == pl.q.size();
        const bool a64 = last || !fits_i32(shots, done + Q);
        pl.acc64.push_back(a64 ? 1 : 0);
        pl.stage64.push_back(fits_i32(shots, done + std::min(Q, 3)) ? 0 : 1);
        if (!last) {
            const int64_t P = ipow(4, done);
            const size_t elems = (size_t)ipow(4, Q) * (size_t)P * (size_t)(hiH - loH) * (size_t)ipow(2, h);
            const size_t bytes = elems * (a64 ? 8 : 4);
            pl.out_bytes.push_back(bytes);
            ws += (bytes + 255) & ~(size_t)255;
        } else {
            pl.out_bytes.push_back(0);
        }
        lo = loH;
        hi = hiH;
        done += Q;
    }
    pl.ws_bytes = ws;
    return pl;
}

template <typename Tin, typename Ts, typename Ta, int Q>
static cudaError_t launch_fold(const void *in, void *out, const PassGeom &g, cudaStream_t s) {
    using Cfg = FoldCfg<Q, Ts>;
    const size_t smem = Cfg::STAGE_BYTES + (Cfg::QP > 0 ? ((size_t)1 << (2 * (Q - 1))) * sizeof(Ta) : 0);
    auto kern = fold_pass_kernel<Q, Tin, Ts, Ta>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (g.ntiles + Cfg::TPC - 1) / Cfg::TPC;
    kern<<<(unsigned)blocks, Cfg::THREADS, smem, s>>>(reinterpret_cast<const Tin *>(in), out, g);
    count_launch();
    return cudaGetLastError();
}

template <typename Tin, typename Ta, int Q>
static cudaError_t launch_small(const void *in, void *out, const PassGeom &g, cudaStream_t s) {
    const int64_t blocks = (g.ntiles + 127) / 128;
    small_pass_kernel<Q, Tin, Ta><<<(unsigned)blocks, 128, 0, s>>>(reinterpret_cast<const Tin *>(in), out, g);
    count_launch();
    return cudaGetLastError();
}

template <typename Tin, typename Ts, typename Ta>
static cudaError_t dispatch_q(int Q, const void *in, void *out, const PassGeom &g, cudaStream_t s) {
    switch (Q) {
    case 1: return launch_small<Tin, Ta, 1>(in, out, g, s);
    case 2: return launch_small<Tin, Ta, 2>(in, out, g, s);
    case 3: return launch_small<Tin, Ta, 3>(in, out, g, s);
    case 4: return launch_fold<Tin, Ts, Ta, 4>(in, out, g, s);
    case 5: return launch_fold<Tin, Ts, Ta, 5>(in, out, g, s);
    case 6: return launch_fold<Tin, Ts, Ta, 6>(in, out, g, s);
    case 7:
        if constexpr (sizeof(Ts) == 4) return launch_fold<Tin, Ts, Ta, 7>(in, out, g, s);
        return cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
    }
}

template <typename Tin>
static cudaError_t dispatch_types(int st64, int a64, int Q, const void *in, void *out, const PassGeom &g,
                                  cudaStream_t s) {
    if (!a64) return dispatch_q<Tin, int32_t, int32_t>(Q, in, out, g, s);
    if (!st64) return dispatch_q<Tin, int32_t, int64_t>(Q, in, out, g, s);
    return dispatch_q<Tin, int64_t, int64_t>(Q, in, out, g, s);
}

static cudaError_t run_pass(int in_dtype, int st64, int a64, int Q, const void *in, void *out, const PassGeom &g,
                            cudaStream_t s) {
    switch (in_dtype) {
    case LRE_U8: return dispatch_types<uint8_t>(st64, a64, Q, in, out, g, s);
    case LRE_U16: return dispatch_types<uint16_t>(st64, a64, Q, in, out, g, s);
    case LRE_I32: return dispatch_types<int32_t>(st64, a64, Q, in, out, g, s);
    case LRE_I64: return dispatch_types<int64_t>(st64, a64, Q, in, out, g, s);
    default: return cudaErrorInvalidValue;
    }
}

static bool g_pow3_ready = false;

static cudaError_t ensure_constants() {
    if (g_pow3_ready) return cudaSuccess;
    double t[33];
    t[0] = 1.0;
    for (int i = 1; i < 33; ++i) t[i] = t[i - 1] * 3.0;
    cudaError_t e = cudaMemcpyToSymbol(c_pow3, t, sizeof(t));
    if (e == cudaSuccess) g_pow3_ready = true;
    return e;
}

// Run passes [first, last) of the plan for input setting range [w_begin, w_end).
// full_ws: intermediates use the full-range layout (stage/finish streaming);
// otherwise they hold only the row groups this range touches (shards).
static int run_passes(const PassPlan &pl, const PassPlan &full, bool full_ws, size_t first, size_t last,
                      const void *input, int in_dtype, int n, int64_t shots, void *ws, void *out, int out_kind,
                      int layout, cudaStream_t stream) {
    if (ensure_constants() != cudaSuccess) return LRE_ECUDA;
    const PassPlan &lay = full_ws ? full : pl;
    std::vector<size_t> offs;
    size_t off = 0;
    for (size_t i = 0; i < lay.q.size(); ++i) {
        offs.push_back(off);
        off += (lay.out_bytes[i] + 255) & ~(size_t)255;
    }
    int done = 0;
    for (size_t i = 0; i < first; ++i) done += pl.q[i];
    const void *cur = input;
    int cur_dtype = in_dtype;
    if (first > 0) {
        cur = (const char *)ws + offs[first - 1];
        cur_dtype = lay.acc64[first - 1] ? LRE_I64 : LRE_I32;
    }
    for (size_t i = first; i < last; ++i) {
        const int Q = pl.q[i];
        const int h = n - done - Q;
        const bool fin = i + 1 == pl.q.size();
        const int64_t q3 = ipow(3, Q);
        PassGeom g;
        g.P = ipow(4, done);
        g.C = ipow(2, h);
        // compute only the row groups of this range; address the buffers by `lay`
        g.alo = lay.alo[i];
        g.ahi = lay.ahi[i];
        g.aloH = pl.alo[i] / q3;
        g.nH = (pl.ahi[i] + q3 - 1) / q3 - g.aloH;
        if (fin) {
            g.aHout0 = 0;
            g.nHout = 1;
        } else {
            g.aHout0 = lay.alo[i] / q3;
            g.nHout = (lay.ahi[i] + q3 - 1) / q3 - g.aHout0;
        }
        if (i == 0) {  // the counts buffer holds exactly [w_begin, w_end)
            g.alo = pl.alo[0];
            g.ahi = pl.ahi[0];
        }
        g.RCout = g.P * g.nHout * g.C;
        g.ntiles = g.P * g.nH * g.C;
        g.rowlen = g.C << Q;
        g.Q = Q;
        g.final_pass = fin ? 1 : 0;
        g.out_kind = out_kind;
        g.layout = layout;
        g.n = n;
        g.shots = shots;
        g.scale = pow(2.0, -n / 2.0);
        void *dst = fin ? out : (void *)((char *)ws + offs[i]);
        cudaError_t e = run_pass(cur_dtype, pl.stage64[i], pl.acc64[i], Q, cur, dst, g, stream);
        if (e != cudaSuccess) return e == cudaErrorInvalidValue ? LRE_EUNSUPPORTED : LRE_ECUDA;
        if (!fin) {
            cur = dst;
            cur_dtype = pl.acc64[i] ? LRE_I64 : LRE_I32;
        }
        done += Q;
    }
    return LRE_OK;
}

int step1_impl(const void *counts, int dtype, int n, int64_t shots, int64_t w_begin, int64_t w_end, void *ws,
               size_t ws_bytes, void *out, int out_kind, int layout, cudaStream_t stream) {
    const PassPlan pl = make_plan(n, shots, w_begin, w_end);
    if (ws_bytes < pl.ws_bytes || (pl.ws_bytes && !ws)) return LRE_ENOMEM;
    return run_passes(pl, pl, false, 0, pl.q.size(), counts, dtype, n, shots, ws, out, out_kind, layout, stream);
}

// pass 1 of a setting chunk into the full-range workspace
int step1_stage_impl(const void *counts, int dtype, int n, int64_t shots, int64_t w_begin, int64_t w_end, void *ws,
                     size_t ws_bytes, cudaStream_t stream) {
    const PassPlan full = make_plan(n, shots, 0, ipow(3, n));
    if (full.q.size() < 2) return LRE_EUNSUPPORTED;
    if (ws_bytes < full.ws_bytes || !ws) return LRE_ENOMEM;
    const PassPlan pl = make_plan(n, shots, w_begin, w_end);
    if (pl.q != full.q) return LRE_EINVAL;
    return run_passes(pl, full, true, 0, 1, counts, dtype, n, shots, ws, nullptr, 0, 0, stream);
}

// passes 2.. over the full-range workspace
int step1_finish_impl(void *ws, size_t ws_bytes, int n, int64_t shots, void *out, int out_kind, int layout,
                      cudaStream_t stream) {
    const PassPlan full = make_plan(n, shots, 0, ipow(3, n));
    if (full.q.size() < 2) return LRE_EUNSUPPORTED;
    if (ws_bytes < full.ws_bytes || !ws) return LRE_ENOMEM;
    return run_passes(full, full, true, 1, full.q.size(), nullptr, 0, n, shots, ws, out, out_kind, layout, stream);
}

int step1_num_passes(int n, int64_t shots) { return (int)plan_passes(n, shots).size(); }

size_t step1_workspace(int n, int64_t shots, int64_t w_begin, int64_t w_end) {
    return make_plan(n, shots, w_begin, w_end).ws_bytes;
}

int64_t shard_quantum(int n, int64_t shots) { return ipow(3, plan_passes(n, shots)[0]); }

}  // namespace lre
