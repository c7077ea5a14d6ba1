// Microbenchmark: could the SMs the 8-CTA cluster kernel leaves idle (148 - 120 at
// n = 14) assemble blocks on their own?  A solo CTA builds eighth k of a block from
// all 8 masks, so it re-reads the block's 1 MB of theta once per eighth (8x, from L2).
//   (1) L2 re-read rate: C CTAs, each reads its own 1 MB region 8 times (v2 loads)
//   (2) co-residency: the DSMEM skeleton cluster kernel (stream A) with C solo CTAs
//       (stream B) - do both run at once on disjoint SMs?
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o mb_solo mb_solo.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

constexpr int NT = 512;
constexpr int SMEM = 200 * 1024;

__global__ void __launch_bounds__(NT, 1) reread(const double2 *theta, int blocks, int reps, double *sink) {
  extern __shared__ double sm[];
  double acc = 0;
  for (int b = blockIdx.x; b < blocks; b += gridDim.x) {
    const double2 *src = theta + (size_t)b * (1 << 16);  // 1 MB block
    for (int r = 0; r < reps; ++r) {
#pragma unroll 8
      for (int i = threadIdx.x; i < (1 << 16); i += NT) {
        double2 v;
        asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(src + i));
        acc += v.x - v.y;
      }
    }
  }
  if (acc == 1.2345) sink[0] = acc;
  if (threadIdx.x == 0) sm[0] = acc;
}

__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(NT, 1) spin_cluster(long long ns, double *sink) {
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t = t0;
  while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && t == 0) sink[1] = 1;
}
__global__ void __launch_bounds__(NT, 1) spin_solo(long long ns, double *sink) {
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t = t0;
  while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && t == 0) sink[2] = 1;
}

int main() {
  double2 *theta;
  double *sink;
  CK(cudaMalloc(&theta, (size_t)1 << 31));  // 2 GB = 2048 blocks of 1 MB
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(theta, 0, (size_t)1 << 31));
  CK(cudaFuncSetAttribute(reread, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int C : {28, 60, 148}) {
    for (int reps : {1, 8}) {
      const int blocks = C * 8;
      reread<<<C, NT, SMEM>>>(theta, blocks, reps, sink);
      cudaEventRecord(e0);
      reread<<<C, NT, SMEM>>>(theta, blocks, reps, sink);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)blocks * reps * (1 << 20);
      printf("reread C=%3d reps=%d  %.3f ms  %.1f GB/s total  %.1f GB/s per CTA  (%.1f us per 1 MB pass)\n", C, reps, ms,
             bytes / ms / 1e6, bytes / ms / 1e6 / C, ms * 1e3 / (blocks / C * reps));
    }
  }
  // co-residency: 15 clusters of 8 (120 CTAs) + 28 solo CTAs, 200 KB smem each, 1 ms each
  CK(cudaFuncSetAttribute(spin_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  CK(cudaFuncSetAttribute(spin_solo, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  cudaStream_t sa, sb;
  cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking);
  for (int solo : {0, 28, 29, 36}) {
    cudaEventRecord(e0, sa);
    cudaStreamWaitEvent(sb, e0, 0);
    spin_cluster<<<120, NT, SMEM, sa>>>(1000000, sink);
    if (solo) spin_solo<<<solo, NT, SMEM, sb>>>(1000000, sink);
    cudaEvent_t ej;
    cudaEventCreate(&ej);
    cudaEventRecord(ej, sb);
    cudaStreamWaitEvent(sa, ej, 0);
    cudaEventRecord(e1, sa);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("co-residency: 120 cluster CTAs + %d solo CTAs (1 ms each): %.3f ms\n", solo, ms);
  }
  return 0;
}
