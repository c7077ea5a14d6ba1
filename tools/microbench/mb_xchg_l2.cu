// Microbenchmark: skeleton of one assembly block per CTA — an all-to-all
// exchange of 16 KB per (sender, receiver) inside a group of 8 CTAs, then a
// write phase of 2048 scattered 128-byte mu lines (256 KB) per CTA.
//   mode 0  DSMEM: 8-CTA clusters, st.async + mbarrier (the x8 design; 15 clusters fit)
//   mode 1  L2:    persistent CTAs (1 per SM, groups of 8), exchange through a
//                  double-buffered global scratch + a release/acquire counter per group
//   mode 2  L2 with st.global.L2::cache_hint evict_last on the scratch
// "X only" / "W only" variants time the two phases alone.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o mb_xchg_l2 mb_xchg_l2.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

constexpr int NT = 512;
constexpr int PART = 16384;
constexpr int BUF = 8 * PART;
constexpr int SMEM = BUF + 64;
constexpr int LOGD = 14;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) {
  uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o;
}
__device__ __forceinline__ void mbar_init(uint64_t *b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
                   smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void st256(double2 *dst, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// the write phase: 2048 rows x 128 B at XOR-diagonal positions (4 lanes per line)
__device__ __forceinline__ void write_phase(double2 *mu, int64_t unit, int part, const double *F) {
  const int64_t d = 1LL << LOGD;
  const int64_t m0 = (unit * 8) & (d - 1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rr = lane >> 2, w = lane & 3;
#pragma unroll 4
  for (int g8 = warp; g8 < 256; g8 += NT / 32) {
    const int64_t r = (int64_t)part * 2048 + 8 * g8 + rr;
    const double f = F[(8 * g8 + rr) * 8 + w];
    st256(mu + r * d + ((r ^ m0) & ~7LL) + 2 * w, f, -f, f + 1, f - 1);
  }
}

template <int MODE, bool X, bool W>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(NT, 1) k_dsmem(int64_t units, double2 *mu) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + BUF);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank(), t = threadIdx.x;
  if (t == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  cl.sync();
  const uint32_t buf_s = smem_u32(sm), bar_s = smem_u32(bar);
  int it = 0;
  for (int64_t u = blockIdx.x / 8; u < units; u += gridDim.x / 8, ++it) {
    if (X) {
      if (t == 0) mbar_expect_tx(bar, BUF);
      for (int k = 0; k < 8; ++k) {
        const int dst = (rank + k) & 7;
        const uint32_t rb = mapa(bar_s, dst);
#pragma unroll
        for (int i = 0; i < PART / 16 / NT; ++i) {
          const int p = t + NT * i;
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                           mapa(buf_s + rank * PART + 16 * p, dst)), "d"((double)p), "d"((double)u), "r"(rb) : "memory");
        }
      }
      mbar_wait(bar, it & 1);
    }
    __syncthreads();
    if (W) write_phase(mu, u, rank, reinterpret_cast<const double *>(sm));
    cl.sync();
  }
}

template <int MODE, bool X, bool W>
__global__ void __launch_bounds__(NT, 1) k_l2(int64_t units, double2 *mu, double2 *scratch, unsigned *counters) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int t = threadIdx.x;
  const int ngroups = gridDim.x / 8;
  const int grp = blockIdx.x / 8, rank = blockIdx.x % 8;
  if (grp >= ngroups) return;
  uint64_t pol = 0;
  if (MODE == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  double2 *sgrp = scratch + (size_t)grp * 2 * (BUF / 16) * 8;  // [buf][dst][src][PART/16]
  int it = 0;
  for (int64_t u = grp; u < units; u += ngroups, ++it) {
    if (X) {
      double2 *sb = sgrp + (size_t)(it & 1) * (BUF / 16) * 8;
      for (int k = 0; k < 8; ++k) {
        const int dst = (rank + k) & 7;
        double2 *o = sb + ((size_t)dst * 8 + rank) * (PART / 16);
#pragma unroll
        for (int i = 0; i < PART / 16 / NT; ++i) {
          const int p = t + NT * i;
          if (MODE == 2)
            asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(o + p), "d"((double)p),
                         "d"((double)u), "l"(pol) : "memory");
          else
            asm volatile("st.global.cg.v2.f64 [%0], {%1, %2};" ::"l"(o + p), "d"((double)p), "d"((double)u) : "memory");
        }
      }
      __syncthreads();
      if (t == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counters + grp) : "memory");
        unsigned v;
        const unsigned target = 8u * (unsigned)(it + 1);
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counters + grp) : "memory");
        } while (v < target);
      }
      __syncthreads();
      const double2 *in = sb + (size_t)rank * 8 * (PART / 16);
      double2 *F2 = reinterpret_cast<double2 *>(sm);
#pragma unroll 4
      for (int i = t; i < BUF / 16; i += NT) {
        double2 v;
        asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(in + i));
        F2[i] = v;
      }
      __syncthreads();
    }
    if (W) write_phase(mu, u, rank, reinterpret_cast<const double *>(sm));
    __syncthreads();
  }
}

template <typename L>
float timeit(L launch) {
  launch();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

template <bool X, bool W>
int run_dsmem(const char *name, int64_t units, double2 *mu) {
  auto k = k_dsmem<0, X, W>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(NT); cfg.dynamicSmemBytes = SMEM;
  cudaLaunchAttribute attr; attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 8; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
  cfg.attrs = &attr; cfg.numAttrs = 1; cfg.gridDim = dim3(8);
  int maxc = 0;
  CK(cudaOccupancyMaxActiveClusters(&maxc, (void *)k, &cfg));
  cfg.gridDim = dim3(8 * maxc);
  const float ms = timeit([&] { cudaLaunchKernelEx(&cfg, k, units, mu); });
  CK(cudaGetLastError());
  printf("%-26s ctas=%3d  %.3f ms  %.2f us/unit/group\n", name, 8 * maxc, ms, ms * 1e3 / ((double)units / maxc));
  return 0;
}

template <int MODE, bool X, bool W>
int run_l2(const char *name, int64_t units, double2 *mu, double2 *scratch, unsigned *ctr, int ctas) {
  auto k = k_l2<MODE, X, W>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  const float ms = timeit([&] {
    cudaMemsetAsync(ctr, 0, 64 * sizeof(unsigned));
    k<<<ctas, NT, SMEM>>>(units, mu, scratch, ctr);
  });
  CK(cudaGetLastError());
  printf("%-26s ctas=%3d  %.3f ms  %.2f us/unit/group\n", name, ctas, ms, ms * 1e3 / ((double)units / (ctas / 8)));
  return 0;
}

// warp-specialised: warps 0-7 run the exchange into the buffer while warps 8-15
// write 256 KB of mu lines (from a second, unchanging source): do DSMEM pushes and
// global stores overlap inside one SM?
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(NT, 1) k_dsmem_ws(int64_t units, double2 *mu) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + BUF);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank(), t = threadIdx.x;
  if (t == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  cl.sync();
  const uint32_t buf_s = smem_u32(sm), bar_s = smem_u32(bar);
  const int64_t d = 1LL << LOGD;
  int it = 0;
  for (int64_t u = blockIdx.x / 8; u < units; u += gridDim.x / 8, ++it) {
    if (t < NT / 2) {
      if (t == 0) mbar_expect_tx(bar, BUF);
      for (int k = 0; k < 8; ++k) {
        const int dst = (rank + k) & 7;
        const uint32_t rb = mapa(bar_s, dst);
#pragma unroll
        for (int i = 0; i < PART / 16 / (NT / 2); ++i) {
          const int p = t + (NT / 2) * i;
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                           mapa(buf_s + rank * PART + 16 * p, dst)), "d"((double)p), "d"((double)u), "r"(rb) : "memory");
        }
      }
      mbar_wait(bar, it & 1);
    } else {
      const int64_t m0 = (u * 8) & (d - 1);
      const int tt = t - NT / 2;
      const int lane = tt & 31, warp = tt >> 5;
      const int rr = lane >> 2, w = lane & 3;
#pragma unroll 4
      for (int g8 = warp; g8 < 256; g8 += NT / 64) {
        const int64_t r = (int64_t)rank * 2048 + 8 * g8 + rr;
        const double f = (double)(g8 + u);
        st256(mu + r * d + ((r ^ m0) & ~7LL) + 2 * w, f, -f, f + 1, f - 1);
      }
    }
    cl.sync();
  }
}

int run_ws(const char *name, int64_t units, double2 *mu) {
  auto k = k_dsmem_ws;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(NT); cfg.dynamicSmemBytes = SMEM;
  cudaLaunchAttribute attr; attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 8; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
  cfg.attrs = &attr; cfg.numAttrs = 1; cfg.gridDim = dim3(8);
  int maxc = 0;
  CK(cudaOccupancyMaxActiveClusters(&maxc, (void *)k, &cfg));
  cfg.gridDim = dim3(8 * maxc);
  const float ms = timeit([&] { cudaLaunchKernelEx(&cfg, k, units, mu); });
  CK(cudaGetLastError());
  printf("%-26s ctas=%3d  %.3f ms  %.2f us/unit/group\n", name, 8 * maxc, ms, ms * 1e3 / ((double)units / maxc));
  return 0;
}

int main() {
  const int64_t d = 1LL << LOGD;
  double2 *mu, *scratch;
  unsigned *ctr;
  CK(cudaMalloc(&mu, 16 * d * d));
  CK(cudaMalloc(&scratch, (size_t)18 * 2 * BUF * 8));
  CK(cudaMalloc(&ctr, 64 * sizeof(unsigned)));
  const int64_t units = 2048 * 8 / 8;  // 2048 blocks of 8 masks, each written by 8 parts: as n = 14
  for (int rep = 0; rep < 2; ++rep) {
    run_ws("dsmem X||W (warp-spec)", units, mu);
    run_dsmem<true, true>("dsmem X+W", units, mu);
    run_dsmem<true, false>("dsmem X only", units, mu);
    run_dsmem<false, true>("dsmem W only", units, mu);
    run_l2<1, true, true>("L2 X+W (144)", units, mu, scratch, ctr, 144);
    run_l2<1, true, false>("L2 X only (144)", units, mu, scratch, ctr, 144);
    run_l2<1, false, true>("L2 W only (144)", units, mu, scratch, ctr, 144);
    run_l2<2, true, true>("L2 evict_last X+W (144)", units, mu, scratch, ctr, 144);
    run_l2<1, true, true>("L2 X+W (120)", units, mu, scratch, ctr, 120);
  }
  return 0;
}
