// Microbenchmark: the assembly's all-to-all exchange inside an 8-CTA cluster.
// Every CTA sends 16 KB to each of the 8 CTAs of its cluster (128 KB in, 128 KB
// out per CTA per round), the receiver waits on its mbarrier (complete_tx), then
// a cluster barrier; R rounds.  Mechanisms:
//   st.async  - 16-byte st.async.shared::cluster per thread (the x8 push)
//   bulk C    - cp.async.bulk.shared::cluster.shared::cta, C-byte chunks, issued by 32 lanes
//   pull      - ld.shared::cluster.v2.f64 from the partners, st.shared locally
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mb_dsmem mb_dsmem.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

constexpr int NT = 512;
constexpr int PART = 16384;            // bytes per (sender, receiver)
constexpr int BUF = 8 * PART;          // receive buffer
constexpr int SRC = PART;              // local source (the same 16 KB sent to everyone)
constexpr int SMEM = BUF + SRC + 64;

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

template <int MODE, int CHUNK>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(NT, 1) xchg(int rounds, double *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char *buf = sm, *src = sm + BUF;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + BUF + SRC);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank(), t = threadIdx.x;
  for (int i = t; i < SRC / 8; i += NT) reinterpret_cast<double *>(src)[i] = i + rank;
  if (t == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  cl.sync();
  const uint32_t buf_s = smem_u32(buf), bar_s = smem_u32(bar), src_s = smem_u32(src);
  for (int it = 0; it < rounds; ++it) {
    if (MODE != 2 && t == 0) mbar_expect_tx(bar, BUF);
    if constexpr (MODE == 0) {
      // thread t sends 16-byte piece p = t + NT * i of its 16 KB to every receiver
      const double2 *s2 = reinterpret_cast<const double2 *>(src);
#pragma unroll 2
      for (int k = 0; k < 8; ++k) {
        const int dst = (rank + k) & 7;
        const uint32_t rb = mapa(bar_s, dst);
#pragma unroll
        for (int i = 0; i < PART / 16 / NT; ++i) {
          const int p = t + NT * i;
          const double2 v = s2[p];
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                           mapa(buf_s + rank * PART + 16 * p, dst)), "d"(v.x), "d"(v.y), "r"(rb) : "memory");
        }
      }
    } else if constexpr (MODE == 1) {
      constexpr int NCH = PART / CHUNK;
      if (t < 32) {
        for (int q = t; q < 8 * NCH; q += 32) {
          const int dst = (rank + q / NCH) & 7, c = q % NCH;
          asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           mapa(buf_s + rank * PART + c * CHUNK, dst)), "r"(src_s + c * CHUNK), "r"(CHUNK), "r"(mapa(bar_s, dst))
                       : "memory");
        }
      }
    } else {
      // pull: thread reads its pieces of every sender's 16 KB source
      double2 *b2 = reinterpret_cast<double2 *>(buf);
#pragma unroll 2
      for (int k = 0; k < 8; ++k) {
        const int from = (rank + k) & 7;
        const uint32_t rs = mapa(src_s, from);
#pragma unroll
        for (int i = 0; i < PART / 16 / NT; ++i) {
          const int p = t + NT * i;
          double2 v;
          asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(rs + 16 * p));
          b2[from * (PART / 16) + p] = v;
        }
      }
    }
    if (MODE != 2) mbar_wait(bar, it & 1);
    // consume a little so nothing is dead
    if (t == 0 && it == rounds - 1) sink[blockIdx.x] = reinterpret_cast<double *>(buf)[rank];
    cl.sync();
  }
}

template <int MODE, int CHUNK>
int run(const char *name, int rounds, double *sink) {
  auto k = xchg<MODE, CHUNK>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = SMEM;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 8; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
  cfg.attrs = &attr; cfg.numAttrs = 1;
  cfg.gridDim = dim3(8);
  int maxc = 0;
  CK(cudaOccupancyMaxActiveClusters(&maxc, (void *)k, &cfg));
  cfg.gridDim = dim3(8 * maxc);
  CK(cudaLaunchKernelEx(&cfg, k, rounds, sink));
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  CK(cudaLaunchKernelEx(&cfg, k, rounds, sink));
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double per = ms * 1e3 / rounds;  // us per round
  printf("%-22s clusters=%d  %.2f us/round  %.1f B/clk/SM in (at 1.965 GHz, 112 KB remote)\n", name, maxc, per,
         (7.0 * PART) / (per * 1e-6) / 1.965e9);
  return 0;
}

int main() {
  double *sink;
  CK(cudaMalloc(&sink, 4096 * 8));
  const int R = 2000;
  run<0, 0>("st.async v2.f64", R, sink);
  run<1, 256>("bulk 256 B", R, sink);
  run<1, 2048>("bulk 2 KB", R, sink);
  run<1, 16384>("bulk 16 KB", R, sink);
  run<2, 0>("pull ld.v2", R, sink);
  run<0, 0>("st.async v2.f64", R, sink);
  return 0;
}
